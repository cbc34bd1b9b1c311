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
// index arithmetic per element.  Each CTA computes a BM x BN output tile with 256 threads,
// each thread a TM x TN register block (64 FFMA per 16 floats read from shared memory at
// 128 x 128); K is staged through double-buffered shared memory in steps of 8 with the next
// step's global loads in flight during the current step's FMAs.  fp32 FFMA throughout, so
// integer-valued layers are bit-exact and the error is the fp32 rounding of each stage.
// The old single-kernel SIMT path (tkd_simt.cu) remains for channel counts the vector
// loads cannot take (C % 4 != 0).
#include <cuda_runtime.h>

#include "internal.h"

namespace tdc {

constexpr int kSgThreads = 256;
constexpr int kSgBK = 8;

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

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__(kSgThreads) tdc_sgemm_taps_kernel(const SgemmArgs g) {
    static_assert((BM / TM) * (BN / TN) == kSgThreads, "thread layout");
    constexpr int AL = BM * kSgBK / (4 * kSgThreads);  // float4 loads of A per thread per K-step
    constexpr int BL = (BN * kSgBK + 4 * kSgThreads - 1) / (4 * kSgThreads);
    __shared__ __align__(16) float As[2][kSgBK][BM + 4];
    __shared__ __align__(16) float Bs[2][kSgBK][BN];
    const int tid = threadIdx.x;
    const int tx = tid % (BN / TN), ty = tid / (BN / TN);
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    const int ksteps = g.K / kSgBK, iters_all = g.taps * ksteps;
    // split-K (few output tiles): this CTA's slice of the (tap, K-step) loop
    const int it0 = (int)((long long)blockIdx.z * iters_all / gridDim.z);
    const int it1 = (int)((long long)(blockIdx.z + 1) * iters_all / gridDim.z);

    float4 ra[AL], rb[BL > 0 ? BL : 1];
    auto load = [&](int it) {
        const int tap = it / ksteps, k0 = (it - tap * ksteps) * kSgBK;
#pragma unroll
        for (int i = 0; i < AL; ++i) {
            const int e = (tid + i * kSgThreads) * 4, row = e / kSgBK, kq = e % kSgBK;
            const int m = m0 + row;
            const float *src = g.A + ((long long)(m < g.M ? m : 0) + g.a_off[tap]) * g.lda + k0 + kq;
            ra[i] = (g.kmask && k0 + kq + 4 > g.K_valid)
                        ? make_float4(k0 + kq < g.K_valid ? src[0] : 0.f, k0 + kq + 1 < g.K_valid ? src[1] : 0.f,
                                      k0 + kq + 2 < g.K_valid ? src[2] : 0.f, 0.f)
                        : __ldg(reinterpret_cast<const float4 *>(src));
        }
#pragma unroll
        for (int i = 0; i < BL; ++i) {
            const int e = (tid + i * kSgThreads) * 4;
            if (e < kSgBK * BN) {
                const int k = e / BN, n = e % BN;
                rb[i] = __ldg(reinterpret_cast<const float4 *>(g.B + ((long long)tap * g.K + k0 + k) * g.ldb + n0 + n));
            }
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int i = 0; i < AL; ++i) {
            const int e = (tid + i * kSgThreads) * 4, row = e / kSgBK, kq = e % kSgBK;
            As[buf][kq][row] = ra[i].x;
            As[buf][kq + 1][row] = ra[i].y;
            As[buf][kq + 2][row] = ra[i].z;
            As[buf][kq + 3][row] = ra[i].w;
        }
#pragma unroll
        for (int i = 0; i < BL; ++i) {
            const int e = (tid + i * kSgThreads) * 4;
            if (e < kSgBK * BN) *reinterpret_cast<float4 *>(&Bs[buf][e / BN][e % BN]) = rb[i];
        }
    };

    float acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

    load(it0);
    store(0);
    __syncthreads();
    for (int it = it0; it < it1; ++it) {
        const int buf = (it - it0) & 1;
        if (it + 1 < it1) load(it + 1);  // next K-step's global loads overlap these FMAs
#pragma unroll
        for (int k = 0; k < kSgBK; ++k) {
            float a[TM], b[TN];
#pragma unroll
            for (int i = 0; i < TM; i += 4) {
                const float4 v = *reinterpret_cast<const float4 *>(&As[buf][k][ty * TM + i]);
                a[i] = v.x; a[i + 1] = v.y; a[i + 2] = v.z; a[i + 3] = v.w;
            }
            if (TN % 4 == 0) {
#pragma unroll
                for (int j = 0; j < TN; j += 4) {
                    const float4 v = *reinterpret_cast<const float4 *>(&Bs[buf][k][tx * TN + j]);
                    b[j] = v.x; b[j + 1] = v.y; b[j + 2] = v.z; b[j + 3] = v.w;
                }
            } else {
#pragma unroll
                for (int j = 0; j < TN; ++j) b[j] = Bs[buf][k][tx * TN + j];
            }
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        if (it + 1 < it1) {
            store(buf ^ 1);
            __syncthreads();
        }
    }

    if (gridDim.z > 1) {  // split-K: partial tile to the workspace; tdc_sgemm_reduce_kernel finishes
        float *part = g.part + ((long long)(blockIdx.y * gridDim.x + blockIdx.x) * gridDim.z + blockIdx.z) * BM * BN;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
            for (int j = 0; j < TN; j += (TN % 4 == 0 ? 4 : 1)) {
                float *dst = part + (ty * TM + i) * BN + tx * TN + j;
                if (TN % 4 == 0)
                    *reinterpret_cast<float4 *>(dst) = make_float4(acc[i][j], acc[i][j + 1], acc[i][j + 2], acc[i][j + 3]);
                else
                    *dst = acc[i][j];
            }
        return;
    }

    // epilogue: row remap, + bias, fp32 stores (each output element written once)
    const int nbase = n0 + tx * TN;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        long long dr;
        if (!sg_out_row(g, m0 + ty * TM + i, &dr)) continue;
        float *dst = g.C + dr * g.ldc + nbase;
        float v[TN];
#pragma unroll
        for (int j = 0; j < TN; ++j) v[j] = acc[i][j] + ((g.bias && nbase + j < g.N) ? __ldg(g.bias + nbase + j) : 0.f);
        if (TN % 4 == 0 && nbase + TN <= g.N && (g.ldc & 3) == 0) {
#pragma unroll
            for (int j = 0; j < TN; j += 4)
                *reinterpret_cast<float4 *>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < TN; ++j)
                if (nbase + j < g.N) dst[j] = v[j];
        }
    }
}

// Split-K reduction: partial tiles summed in split order (deterministic), then the row
// remap, bias and the single store of every output element.
__global__ void __launch_bounds__(256) tdc_sgemm_reduce_kernel(const SgemmArgs g, int bm, int bn, int mt) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // (tile, row, col)
    const int KS = g.ksplit;
    const long long per = (long long)bm * bn;
    const long long tile = e / per;
    if (tile >= (long long)mt * ((g.N + bn - 1) / bn)) return;
    const int rc = (int)(e - tile * per), row = rc / bn, col = rc % bn;
    const int tm = (int)(tile % mt), tn = (int)(tile / mt);
    const int n = tn * bn + col;
    long long dr;
    if (n >= g.N || !sg_out_row(g, tm * bm + row, &dr)) return;
    const float *pp = g.part + tile * KS * per + rc;
    float v = 0.f;
    for (int z = 0; z < KS; ++z) v += pp[z * per];
    if (g.bias) v += __ldg(g.bias + n);
    g.C[dr * g.ldc + n] = v;
}

cudaError_t sgemm_taps_launch(const SgemmArgs &g, cudaStream_t st) {
    auto go = [&](auto kernel, int bm, int bn) {
        const int mt = (g.M + bm - 1) / bm, nt = (g.N + bn - 1) / bn;
        dim3 grid(mt, nt, g.ksplit > 1 ? g.ksplit : 1);
        kernel<<<grid, kSgThreads, 0, st>>>(g);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess || g.ksplit <= 1) return e;
        const long long n = (long long)mt * nt * bm * bn;
        tdc_sgemm_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, bm, bn, mt);
        return cudaGetLastError();
    };
    switch (g.tile) {
        case 0: return go(tdc_sgemm_taps_kernel<128, 128, 8, 8>, 128, 128);
        case 1: return go(tdc_sgemm_taps_kernel<128, 64, 8, 4>, 128, 64);
        default: return go(tdc_sgemm_taps_kernel<256, 32, 16, 2>, 256, 32);
    }
}

// Tile shape for a stage: 128 x 128 (8 x 8 per thread) for wide outputs, 128 x 64 for
// N <= 64, 256 x 32 for N <= 32; a wide stage with fewer than 2 CTAs per SM takes 128 x 64.
int sgemm_pick_tile(long long M, int N, int num_sms) {
    int t = N > 64 ? 0 : (N > 32 ? 1 : 2);
    if (t == 0 && ((M + 127) / 128) * ((N + 127) / 128) < 2LL * num_sms) t = 1;
    return t;
}
// K pieces for a stage whose tiles leave the GPU under-filled: about 2 CTAs per SM, each
// piece >= 4 K-steps, <= 8 pieces.  Workspace floats: tiles * pieces * BM * BN.
int sgemm_pick_ksplit(long long M, int N, int K, int taps, int tile, int num_sms) {
    const int bm = tile == 2 ? 256 : 128, bn = tile == 0 ? 128 : (tile == 1 ? 64 : 32);
    const long long tiles = ((M + bm - 1) / bm) * ((N + bn - 1) / bn);
    const int iters = taps * (K / kSgBK);
    int ks = 1;
    while (ks < 8 && tiles * (ks + 1) <= 2LL * num_sms && iters / (ks + 1) >= 4) ++ks;
    return ks;
}
long long sgemm_part_floats(long long M, int N, int tile, int ksplit) {
    if (ksplit <= 1) return 0;
    const int bm = tile == 2 ? 256 : 128, bn = tile == 0 ? 128 : (tile == 1 ? 64 : 32);
    return ((M + bm - 1) / bm) * ((N + bn - 1) / bn) * (long long)ksplit * bm * bn;
}

}  // namespace tdc
