// tkd_sgemm.cu -- the IEEE-fp32 (TDC_MATH_FP32) TKD layer on CUDA cores as three
// register-blocked "GEMM with taps" launches over the whole GPU (variant 6, simt3_fp32):
//
//   stage 1 (a1)  X'g[phase grid row] = X[pixel] . U_in            M = B H W,   K = C,      N = D1
//   stage 2 (a2)  Z[out] = sum_tap X'g[row(out) + off(tap)] . core[tap]
//                                                                  M = B Hq Wq, K = D1/tap, N = D2
//   stage 3 (a3)  Y[out] = Z[out] . U_out^T (+ bias)               M = B H' W', K = D2,     N = N
//
// The core convolution is the paper's per-thread sum over (c, r, s) as an
// implicit GEMM: the zero-bordered X' "phase grid" (stride s split into s*s planes, same
// layout as the tensor-core path) turns every tap into a constant row
// offset of the A operand, so the K loop over (tap, channel) streams A tiles without
// index arithmetic per element.  Each CTA computes a BM x BN output tile (64x128, 128x64
// or 256x32 by the stage's width) with 128 threads, each thread an 8 x 8 register block
// (64 FFMA per four 16-byte shared-memory reads); K streams through a 3-deep cp.async
// ring in steps of 16 and an under-filled stage splits K over grid.z with a deterministic
// reduce.  fp32 FFMA throughout, so integer-valued layers are bit-exact and the error is
// the fp32 rounding of each stage.
// The old single-kernel SIMT path (tkd_simt.cu) remains for channel counts the vector
// loads cannot take (C % 4 != 0).
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "internal.h"

namespace tdc {


__device__ __forceinline__ bool sg_out_row(const SgemmArgs &g, int m, long long *dst) {
    if (m >= g.M) return false;
    if (g.remap == 0) {
        *dst = m;
        return true;
    }
    if (g.remap == 1) {  // input pixel (b, y, x) -> its phase-grid row
        const int x = m % g.W;
        const int t = m / g.W;
        const int y = t % g.H;
        const int b = t / g.H;
        const int uy = y + g.p, ux = x + g.p;
        const int ph = g.phase_idx[(uy % g.s) * g.s + (ux % g.s)];
        if (ph < 0) return false;  // a phase no tap reads
        *dst = (long long)ph * g.phase_rows + ((long long)b * g.Hq + uy / g.s) * g.Wq + ux / g.s;
        return true;
    }
    // remap 2: phase-grid output position -> compact output pixel (junk rows skipped)
    const int ox = m % g.Wq;
    const int t = m / g.Wq;
    const int oy = t % g.Hq;
    const int b = t / g.Hq;
    if (oy >= g.Ho || ox >= g.Wo) return false;
    *dst = ((long long)b * g.Ho + oy) * g.Wo + ox;
    return true;
}

// Row iterator for the epilogue: the destination row of output row m and of the rows
// after it (x advances with carries), so a run of consecutive rows costs one division.
struct SgRowIter {
    int b, y, x;
    __device__ __forceinline__ void start(const SgemmArgs &g, int m) {
        const int w = g.remap == 2 ? g.Wq : g.W, h = g.remap == 2 ? g.Hq : g.H;
        x = m % w;
        const int t = m / w;
        y = t % h;
        b = t / h;
    }
    __device__ __forceinline__ void next(const SgemmArgs &g) {
        const int w = g.remap == 2 ? g.Wq : g.W, h = g.remap == 2 ? g.Hq : g.H;
        if (++x == w) {
            x = 0;
            if (++y == h) { y = 0; ++b; }
        }
    }
    __device__ __forceinline__ bool dst(const SgemmArgs &g, int m, long long *d) const {
        if (m >= g.M) return false;
        if (g.remap == 0) { *d = m; return true; }
        if (g.remap == 1) {
            const int uy = y + g.p, ux = x + g.p;
            const int ph = g.phase_idx[(uy % g.s) * g.s + (ux % g.s)];
            if (ph < 0) return false;
            *d = (long long)ph * g.phase_rows + ((long long)b * g.Hq + uy / g.s) * g.Wq + ux / g.s;
            return true;
        }
        if (y >= g.Ho || x >= g.Wo) return false;
        *d = ((long long)b * g.Ho + y) * g.Wo + x;
        return true;
    }
};

__device__ __forceinline__ void sg_cp16(uint32_t dst, const void *src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void sg_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void sg_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

constexpr int kSgBK = 16;     // K per pipeline step
constexpr int kSgStages = 3;  // cp.async ring depth

// A stage: BM rows x 16 floats (four 16-byte units per row), unit u stored at
// u ^ ((u >> 5) & 7): the eight rows a warp's lanes read at one k-quad (rows 8 apart)
// land in eight different 16-byte bank groups.
__device__ __forceinline__ int sg_swz(int u) { return u ^ ((u >> 5) & 7); }

template <int BM, int BN>
constexpr int sg_smem_bytes() {
    return kSgStages * (BM * kSgBK + kSgBK * BN) * 4;
}

// One CTA of (BM/8)(BN/8) = 128 threads per output tile (and K piece, grid.z, when the
// stage splits K).  Each thread holds an 8 x 8 register block: rows ty*8 .. ty*8+7
// (consecutive, so the epilogue's row remap is one division per thread), columns tx*4..
// and BN/2 + tx*4.. (each B fragment read of a warp is one conflict-free line).  Operands
// stream through a 3-deep cp.async ring and land untransposed (A[row][k..k+3] fragments,
// four k per read): per 16-wide K-step a thread issues BM/32 + BN/32 16-byte copies and
// 1024 FFMA.  Split K: every piece stores its partial tile and tdc_sgemm_reduce_kernel
// sums the pieces in piece order (deterministic) and runs the epilogue.
template <int BM, int BN>
__global__ void __launch_bounds__((BM / 8) * (BN / 8), 3) tdc_sgemm_taps_kernel(const SgemmArgs g) {
    constexpr int TX = BN / 8, TY = BM / 8, NT = TX * TY;
    static_assert(NT == 128, "thread layout");
    constexpr int LX = TX < 8 ? TX : 8, LY = 32 / LX, WX = TX / LX;
    constexpr int AU = BM * (kSgBK / 4) / NT;  // A 16-byte units per thread per step
    constexpr int BU = kSgBK * BN / 4 / NT;    // B units per thread per step
    static_assert(AU >= 1 && BU >= 1, "load split");
    extern __shared__ __align__(16) float sg_smem[];
    float *As = sg_smem;                           // [stage][BM*16] swizzled units
    float *Bs = sg_smem + kSgStages * BM * kSgBK;  // [stage][16][BN]
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int tx = (warp % WX) * LX + lane % LX, ty = (warp / WX) * LY + lane / LX;
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int ksteps = g.K / kSgBK, iters_all = g.taps * ksteps;
    const int it0 = (int)((long long)blockIdx.z * iters_all / gridDim.z);
    const int it1 = (int)((long long)(blockIdx.z + 1) * iters_all / gridDim.z);
    const uint32_t sA = (uint32_t)__cvta_generic_to_shared(As), sB = (uint32_t)__cvta_generic_to_shared(Bs);

    // loader: next step to fetch (tap ltap, channel offset lk0), advanced without division
    int lit = it0, ltap = it0 / ksteps, lk0 = (it0 - ltap * ksteps) * kSgBK;
    auto issue = [&](int slot) {
        if (lit < it1) {
#pragma unroll
            for (int j = 0; j < AU; ++j) {
                const int u = tid + j * NT, row = u >> 2, c = u & 3;
                const int m = m0 + row;
                const int k = lk0 + c * 4;
                const float *src = g.A + ((long long)(m < g.M ? m : 0) + g.a_off[ltap]) * g.lda + k;
                sg_cp16(sA + (uint32_t)(slot * BM * kSgBK + sg_swz(u) * 4) * 4, src, !g.kmask || k < g.K_valid);
            }
#pragma unroll
            for (int j = 0; j < BU; ++j) {
                const int u = tid + j * NT, k = u / (BN / 4), n = (u % (BN / 4)) * 4;
                const float *src = g.B + ((long long)ltap * g.K + lk0 + k) * g.ldb + n0 + n;
                sg_cp16(sB + (uint32_t)(slot * kSgBK * BN + k * BN + n) * 4, src, true);
            }
            lk0 += kSgBK;
            if (lk0 == g.K) {
                lk0 = 0;
                ++ltap;
            }
            ++lit;
        }
        sg_commit();  // (empty groups keep the wait_group count uniform)
    };
    auto lcol = [&](int j) { return (j < 4 ? 0 : BN / 2 - 4) + tx * 4 + j; };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

#pragma unroll
    for (int st = 0; st < kSgStages - 1; ++st) issue(st);
    int slot = 0;
    for (int it = it0; it < it1; ++it) {
        sg_wait<kSgStages - 2>();
        __syncthreads();  // this step landed for every thread; the previous slot is free
        issue(slot == 0 ? kSgStages - 1 : slot - 1);
        const float *a_s = As + slot * BM * kSgBK;
        const float *b_s = Bs + slot * kSgBK * BN;
#pragma unroll
        for (int kq = 0; kq < 4; ++kq) {
            float4 a4[8];
#pragma unroll
            for (int i = 0; i < 8; ++i)
                a4[i] = *reinterpret_cast<const float4 *>(a_s + sg_swz((ty * 8 + i) * 4 + kq) * 4);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const float4 b0 = *reinterpret_cast<const float4 *>(b_s + (kq * 4 + kk) * BN + lcol(0));
                const float4 b1 = *reinterpret_cast<const float4 *>(b_s + (kq * 4 + kk) * BN + lcol(4));
                const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float av = kk == 0 ? a4[i].x : kk == 1 ? a4[i].y : kk == 2 ? a4[i].z : a4[i].w;
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av, b[j], acc[i][j]);
                }
            }
        }
        slot = slot == kSgStages - 1 ? 0 : slot + 1;
    }
    sg_wait<0>();

    if (gridDim.z > 1) {  // split K: partial tile to the workspace; tdc_sgemm_reduce_kernel finishes
        float *part = g.part + ((long long)(blockIdx.y * gridDim.x + blockIdx.x) * gridDim.z + blockIdx.z) * BM * BN;
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; j += 4)
                __stcg(reinterpret_cast<float4 *>(part + (ty * 8 + i) * BN + lcol(j)),
                       make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]));
        return;
    }

    // epilogue: row remap, + bias, fp32 float4 stores (each output element written once)
    float bv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int n = n0 + lcol(j);
        bv[j] = (g.bias && n < g.N) ? __ldg(g.bias + n) : 0.f;
    }
    const bool vec = (g.ldc & 3) == 0;
    SgRowIter ri;
    ri.start(g, m0 + ty * 8);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        long long dr;
        if (ri.dst(g, m0 + ty * 8 + i, &dr)) {
            float *dst = g.C + dr * g.ldc + n0;
#pragma unroll
            for (int j = 0; j < 8; j += 4) {
                const int c = lcol(j);
                const float4 v = make_float4(acc[i][j] + bv[j], acc[i][j + 1] + bv[j + 1], acc[i][j + 2] + bv[j + 2],
                                             acc[i][j + 3] + bv[j + 3]);
                if (vec && n0 + c + 4 <= g.N) {
                    *reinterpret_cast<float4 *>(dst + c) = v;
                } else {
                    if (n0 + c < g.N) dst[c] = v.x;
                    if (n0 + c + 1 < g.N) dst[c + 1] = v.y;
                    if (n0 + c + 2 < g.N) dst[c + 2] = v.z;
                    if (n0 + c + 3 < g.N) dst[c + 3] = v.w;
                }
            }
        }
        ri.next(g);
    }
}

// Split-K finish: one thread per (tile row, 4 columns) sums the pieces in piece order
// (deterministic), adds the bias, remaps the row and stores a float4.
__global__ void __launch_bounds__(256) tdc_sgemm_reduce_kernel(const SgemmArgs g, int bm, int bn, int mt) {
    const int q4 = bn / 4;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // (tile, row, col quad)
    const long long per = (long long)bm * q4;
    const long long tile = e / per;
    if (tile >= (long long)mt * ((g.N + bn - 1) / bn)) return;
    const int rc = (int)(e - tile * per), row = rc / q4, col = (rc % q4) * 4;
    const int tm = (int)(tile % mt), tn = (int)(tile / mt);
    const int n = tn * bn + col;
    SgRowIter ri;
    const int m = tm * bm + row;
    long long dr;
    if (n >= g.N || m >= g.M) return;
    ri.start(g, m);
    if (!ri.dst(g, m, &dr)) return;
    const int KS = g.ksplit;
    const float *pp = g.part + tile * KS * (long long)bm * bn + row * bn + col;
    float4 v = __ldcg(reinterpret_cast<const float4 *>(pp));
    for (int z = 1; z < KS; ++z) {
        const float4 w = __ldcg(reinterpret_cast<const float4 *>(pp + (long long)z * bm * bn));
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        v.w += w.w;
    }
    float o[4] = {v.x, v.y, v.z, v.w};
    float *dst = g.C + dr * g.ldc;
    if (n + 4 <= g.N && (g.ldc & 3) == 0) {
        if (g.bias)
            for (int j = 0; j < 4; ++j) o[j] += __ldg(g.bias + n + j);
        *reinterpret_cast<float4 *>(dst + n) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
        for (int j = 0; j < 4 && n + j < g.N; ++j) dst[n + j] = o[j] + (g.bias ? __ldg(g.bias + n + j) : 0.f);
    }
}

cudaError_t sgemm_taps_launch(const SgemmArgs &g, cudaStream_t st) {
    auto go = [&](auto kernel, auto bm_c, auto bn_c) {
        constexpr int bm = decltype(bm_c)::value, bn = decltype(bn_c)::value;
        constexpr int smem = sg_smem_bytes<bm, bn>();
        const int mt = (g.M + bm - 1) / bm, nt = (g.N + bn - 1) / bn;
        if (mt <= 0 || nt <= 0) return cudaSuccess;
        dim3 grid(mt, nt, g.ksplit > 1 ? g.ksplit : 1);
        kernel<<<grid, (bm / 8) * (bn / 8), smem, st>>>(g);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess || g.ksplit <= 1) return e;
        const long long n = (long long)mt * nt * bm * (bn / 4);
        tdc_sgemm_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, bm, bn, mt);
        return cudaGetLastError();
    };
    using I64 = std::integral_constant<int, 64>;
    using I128 = std::integral_constant<int, 128>;
    using I256 = std::integral_constant<int, 256>;
    using I32 = std::integral_constant<int, 32>;
    switch (g.tile) {
        case 0: return go(tdc_sgemm_taps_kernel<64, 128>, I64{}, I128{});
        case 1: return go(tdc_sgemm_taps_kernel<128, 64>, I128{}, I64{});
        default: return go(tdc_sgemm_taps_kernel<256, 32>, I256{}, I32{});
    }
}

// Opt the kernels into their dynamic shared memory on the current device (plan time).
cudaError_t sgemm_prepare() {
    cudaError_t e = cudaFuncSetAttribute(tdc_sgemm_taps_kernel<64, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         sg_smem_bytes<64, 128>());
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tdc_sgemm_taps_kernel<128, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 sg_smem_bytes<128, 64>());
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(tdc_sgemm_taps_kernel<256, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 sg_smem_bytes<256, 32>());
    return e;
}

// Co-resident CTAs of a tile shape on this device (the persistent grid size).
int sgemm_ctas(int tile, int num_sms) {
    int per_sm = 0;
    cudaError_t e;
    switch (tile) {
        case 0:
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tdc_sgemm_taps_kernel<64, 128>, 128,
                                                              sg_smem_bytes<64, 128>());
            break;
        case 1:
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tdc_sgemm_taps_kernel<128, 64>, 128,
                                                              sg_smem_bytes<128, 64>());
            break;
        default:
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tdc_sgemm_taps_kernel<256, 32>, 128,
                                                              sg_smem_bytes<256, 32>());
    }
    if (e != cudaSuccess || per_sm < 1) per_sm = 1;
    return per_sm * num_sms;
}

// Tile shapes (8 x 8 outputs per thread, 128 threads, 3 CTAs per SM): 0 64x128, 1 128x64,
// 2 256x32.
static constexpr int kSgBM[3] = {64, 128, 256}, kSgBN[3] = {128, 64, 32};
static long long sg_tiles(long long M, int N, int t) {
    return ((M + kSgBM[t] - 1) / kSgBM[t]) * ((N + kSgBN[t] - 1) / kSgBN[t]);
}

// Tile shape for a stage: the one whose width fits N (wider outputs take several tiles).
int sgemm_pick_tile(long long M, int N, int num_sms) {
    (void)M;
    (void)num_sms;
    return N > 64 ? 0 : (N > 32 ? 1 : 2);
}
// K pieces for a stage whose tiles under-fill the GPU: the count (1..8, >= 4 K-steps each)
// minimising waves(tiles * ks over `ctas` co-resident CTAs) * (steps per piece + 2), a
// split paying ~3 steps for the partial store and the reduce launch.
int sgemm_pick_ksplit(long long M, int N, int K, int taps, int tile, int ctas) {
    const long long tiles = sg_tiles(M, N, tile);
    const int iters = taps * (K / kSgBK);
    int best = 1;
    double best_cost = 1e30;
    for (int ks = 1; ks <= 8 && (ks == 1 || iters / ks >= 4); ++ks) {
        const double waves = (double)((tiles * ks + ctas - 1) / ctas);
        const double cost = waves * ((iters + ks - 1) / ks + 2.0) + (ks > 1 ? 3.0 : 0.0);
        if (cost < best_cost * 0.95) {
            best_cost = cost;
            best = ks;
        }
    }
    return best;
}
long long sgemm_tiles(long long M, int N, int tile) { return sg_tiles(M, N, tile); }
long long sgemm_part_floats(long long M, int N, int tile, int ksplit) {
    if (ksplit <= 1) return 0;
    return sg_tiles(M, N, tile) * (long long)ksplit * kSgBM[tile] * kSgBN[tile];
}

}  // namespace tdc
