// tkd_tc.cu -- the TKD layer on 5th-generation tensor cores (tcgen05, kind::tf32).
//
// One kernel, tdc_tc_gemm_kernel, computes a "GEMM with taps":
//
//     Out[m][n] = sum_{tap} sum_k A[m + a_off[tap]][k] * Bt[b_off[tap] + n][k]   (+ bias[n])
//
// and the three stages of the layer (include/tdc.h) are three instances of it:
//
//   stage 1 (a1): A = X (NHWC rows = pixels, K = C), Bt = U_in^T, one tap; the
//                 epilogue scatters each pixel's D1 ranks into a zero-bordered
//                 "phase grid" X'g (below) -- zero padding for free (reading R6).
//   stage 2 (a2): A = X'g, Bt = core re-laid out per tap, K*K taps whose row
//                 offsets are constants on the phase grid, so the core
//                 convolution is an implicit GEMM with pure TMA
//                 row-shifted loads; the epilogue compacts valid rows into Z.
//   stage 3 (a3): A = Z, Bt = U_out (N x D2 is already K-major), one tap,
//                 bias in the epilogue, rows written straight to Y (NHWC).
//
// Phase grid (stride s, pad p): padded coordinate u = y + p splits into phase
// u % s and position u / s; tap (r, t) of output (oy, ox) reads phase
// (r % s, t % s) at (oy + r / s, ox + t / s).  With every image laid out as an
// Hq x Wq block (Hq = ceil((H+2p)/s)), the read row is (output-grid row) +
// constant, which is exactly what a TMA box at a shifted row coordinate loads.
//
// Kernel anatomy (one 128 x BN output tile per CTA, 6 warps):
//   warp 0  TMA producer: A (128 rows x 32 fp32, 128B-swizzled) and Bt (BN x 32)
//           per (tap, 32-wide K chunk) into an S-stage mbarrier ring;
//   warp 1  TMEM allocation + single-thread tcgen05.mma issue (4 x K=8 per
//           chunk), tcgen05.commit frees ring slots / signals the epilogue;
//   warps 2-5  epilogue: tcgen05.ld 32x32b (one TMEM lane = one output row per
//           thread), bias, row remap, vectorised global stores.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.h"
#include "sm100.cuh"

namespace tdc {

using namespace sm100;

constexpr int kTcThreads = 192;
constexpr int kBM = 128;
constexpr int kBK = 32;                      // fp32 elements per K chunk = one 128 B swizzle row
constexpr int kATileBytes = kBM * kBK * 4;   // 16 KB

__device__ __forceinline__ bool remap_row(const TcGemmArgs &g, int m, long long *dst) {
    if (m >= g.M) return false;
    if (g.remap == 0) {
        *dst = m;
        return true;
    }
    if (g.remap == 1) {  // compact input pixel -> phase grid row
        const int x = m % g.W;
        const int t = m / g.W;
        const int y = t % g.H;
        const int b = t / g.H;
        const int uy = y + g.p, ux = x + g.p;
        const int ph = (uy % g.s) * g.s + (ux % g.s);
        *dst = (long long)ph * g.phase_rows + ((long long)b * g.Hq + uy / g.s) * g.Wq + ux / g.s;
        return true;
    }
    // remap == 2: output grid row -> compact output pixel (skip junk rows)
    const int ox = m % g.Wq;
    const int t = m / g.Wq;
    const int oy = t % g.Hq;
    const int b = t / g.Hq;
    if (oy >= g.Ho || ox >= g.Wo) return false;
    *dst = ((long long)b * g.Ho + oy) * g.Wo + ox;
    return true;
}

__global__ void __launch_bounds__(kTcThreads, 1)
tdc_tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB, const TcGemmArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for the 128B-swizzle atoms
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = g.stages, BN = g.BN;
    const int b_tile_bytes = BN * kBK * 4;
    uint8_t *a_tiles = smem;
    uint8_t *b_tiles = smem + (size_t)S * kATileBytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(b_tiles + (size_t)S * b_tile_bytes);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kBM, n0 = blockIdx.y * BN;
    const uint32_t ncols = BN < 32 ? 32 : BN;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
    }
    if (warp == 1) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int iters = g.taps * g.kchunks;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            const uint32_t bytes = kATileBytes + b_tile_bytes;
            for (int i = 0; i < iters; ++i) {
                const int st = i % S;
                const uint32_t ph = (i / S) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&full[st], bytes);
                const int tap = i / g.kchunks, kc = i - tap * g.kchunks;
                tma_load_2d(a_tiles + (size_t)st * kATileBytes, &mapA, &full[st], kc * kBK,
                            m0 + g.a_off[tap]);
                tma_load_2d(b_tiles + (size_t)st * b_tile_bytes, &mapB, &full[st], kc * kBK,
                            g.b_off[tap] + n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer (single thread)
            const uint32_t idesc = idesc_tf32(kBM, BN);
            for (int i = 0; i < iters; ++i) {
                const int st = i % S;
                const uint32_t ph = (i / S) & 1;
                mbar_wait(&full[st], ph);
                tc_fence_after();
                const uint32_t a0 = smem_u32(a_tiles + (size_t)st * kATileBytes);
                const uint32_t b0 = smem_u32(b_tiles + (size_t)st * b_tile_bytes);
#pragma unroll
                for (int j = 0; j < kBK / 8; ++j) {  // K = 8 tf32 = 32 B per MMA
                    mma_tf32(tmem, sdesc_kmajor_sw128(a0 + j * 32), sdesc_kmajor_sw128(b0 + j * 32),
                             idesc, (i | j) != 0);
                }
                mma_commit(&empty[st]);
            }
            mma_commit(tfull);
        }
    } else {  // ------------------------------ epilogue warps 2..5
        mbar_wait(tfull, 0);
        tc_fence_after();
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int row = q * 32 + lane;
        long long dst_row;
        const bool valid = remap_row(g, m0 + row, &dst_row);
        float *dst = valid ? (g.planar_stride ? g.out + dst_row * 4 : g.out + dst_row * g.ldo)
                           : nullptr;
        for (int c = 0; c < BN; c += 32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, r);
            tmem_ld_wait();
            const int n = n0 + c;
            if (!valid || n >= g.Nn) continue;
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if (g.bias) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (n + j < g.Nn) v[j] += __ldg(&g.bias[n + j]);
            }
            if (g.planar_stride) {  // [col/4][row][4]: lanes = consecutive rows -> coalesced
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4 *>(dst + (long long)((n + j) >> 2) * g.planar_stride) =
                        make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else if (n + 32 <= g.Nn && (g.ldo & 3) == 0) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                    *reinterpret_cast<float4 *>(dst + n + j) =
                        make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
            } else {
                for (int j = 0; j < 32 && n + j < g.Nn; ++j) dst[n + j] = v[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, ncols);
}


// ---------------------------------------------------------------------------
// Stage 2 with a resident X' band: the core convolution as an
// implicit GEMM whose A operand is never re-fetched per tap.  Per 32-channel
// chunk kc of D1, the rows [m0, m0 + band_rows) of every phase plane are
// bulk-copied once into shared memory in the no-swizzle K-major layout
// [phase][kg][row][4 fp32] (a "core matrix" = 8 rows x 16 B); tap (r, t) is
// then just a descriptor whose start address is shifted by the tap's constant
// row offset (r/s)*Wq + t/s -- the 8-row groups stay 128 B apart (SBO) and the
// K-adjacent 4-channel planes band_rows*16 B apart (LBO).  Weights arrive as
// pre-blocked [8][BN][4] chunks (plan-time re-layout, the CRSN idea P:L338-340).
constexpr int kCoreThreads = 192;

__host__ __device__ inline int core_a_slot_bytes(int nphase, int band_rows) {
    return nphase * 8 * band_rows * 16;
}

int tc_core_smem_bytes(int BN, int nphase, int band_rows, int b_stages) {
    return 1024 + 2 * core_a_slot_bytes(nphase, band_rows) + b_stages * BN * 128 +
           (4 + 2 * b_stages + 1) * 8 + 16;
}

__global__ void __launch_bounds__(kCoreThreads, 1) tdc_tc_core_kernel(const TcCoreArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int BN = g.BN, SB = g.b_stages;
    const int a_bytes = core_a_slot_bytes(g.nphase, g.band_rows);
    const int b_bytes = BN * 128;
    uint8_t *a_slots = smem;
    uint8_t *b_slots = smem + 2 * (size_t)a_bytes;
    uint64_t *a_full = reinterpret_cast<uint64_t *>(b_slots + (size_t)SB * b_bytes);
    uint64_t *a_empty = a_full + 2;
    uint64_t *b_full = a_empty + 2;
    uint64_t *b_empty = b_full + SB;
    uint64_t *tfull = b_empty + SB;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kBM, nt = blockIdx.y, n0 = nt * BN;
    const uint32_t ncols = BN < 32 ? 32 : BN;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < SB; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        mbar_init(tfull, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t band_bytes = (uint32_t)g.band_rows * 16;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- bulk-copy producer
            int it = 0;
            for (int kc = 0; kc < g.kchunks; ++kc) {
                const int sa = kc & 1;
                mbar_wait(&a_empty[sa], ((kc >> 1) & 1) ^ 1);
                mbar_arrive_expect_tx(&a_full[sa], (uint32_t)a_bytes);
                uint8_t *dst = a_slots + (size_t)sa * a_bytes;
                for (int ph = 0; ph < g.nphase; ++ph)
                    for (int kg = 0; kg < 8; ++kg) {
                        const float *src = g.xg + (long long)(kc * 8 + kg) * g.plane_stride +
                                           ((long long)g.phase_src[ph] * g.phase_rows + m0) * 4;
                        bulk_load(dst + (size_t)(ph * 8 + kg) * band_bytes, src, band_bytes,
                                  &a_full[sa]);
                    }
                for (int tap = 0; tap < g.taps; ++tap, ++it) {
                    const int sb = it % SB;
                    mbar_wait(&b_empty[sb], ((it / SB) & 1) ^ 1);
                    mbar_arrive_expect_tx(&b_full[sb], (uint32_t)b_bytes);
                    const float *src =
                        g.w + ((long long)(tap * g.kchunks + kc) * g.ntiles + nt) * BN * 32;
                    bulk_load(b_slots + (size_t)sb * b_bytes, src, (uint32_t)b_bytes, &b_full[sb]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer
            const uint32_t idesc = idesc_tf32(kBM, BN);
            int it = 0;
            for (int kc = 0; kc < g.kchunks; ++kc) {
                const int sa = kc & 1;
                mbar_wait(&a_full[sa], (kc >> 1) & 1);
                const uint32_t a0 = smem_u32(a_slots + (size_t)sa * a_bytes);
                for (int tap = 0; tap < g.taps; ++tap, ++it) {
                    const int sb = it % SB;
                    mbar_wait(&b_full[sb], (it / SB) & 1);
                    tc_fence_after();
                    const uint32_t b0 = smem_u32(b_slots + (size_t)sb * b_bytes);
                    const uint32_t abase = a0 + (uint32_t)g.tap_phase[tap] * 8 * band_bytes +
                                           (uint32_t)g.tap_off[tap] * 16;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {  // K = 8 = two 4-channel planes
                        const uint64_t ad = sdesc_kmajor_none(abase + j * 2 * band_bytes, band_bytes, 128);
                        const uint64_t bd = sdesc_kmajor_none(b0 + j * 2 * BN * 16, BN * 16, 128);
                        mma_tf32(tmem, ad, bd, idesc, (kc | tap | j) != 0);
                    }
                    mma_commit(&b_empty[sb]);
                }
                mma_commit(&a_empty[sa]);
            }
            mma_commit(tfull);
        }
    } else {  // ------------------------------ epilogue warps 2..5: Z compact rows
        mbar_wait(tfull, 0);
        tc_fence_after();
        const int q = warp & 3;
        const int m = m0 + q * 32 + lane;
        bool valid = m < g.M;
        long long dst_row = 0;
        if (valid) {
            const int ox = m % g.Wq;
            const int t = m / g.Wq;
            const int oy = t % g.Hq;
            const int b = t / g.Hq;
            valid = oy < g.Ho && ox < g.Wo;
            dst_row = ((long long)b * g.Ho + oy) * g.Wo + ox;
        }
        float *dst = g.z + dst_row * g.ldz;
        for (int c = 0; c < BN; c += 32) {
            uint32_t r[32];
            tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + c, r);
            tmem_ld_wait();
            if (!valid || n0 + c >= g.Nn) continue;
#pragma unroll
            for (int j = 0; j < 32; j += 4)
                *reinterpret_cast<float4 *>(dst + n0 + c + j) =
                    make_float4(__uint_as_float(r[j]), __uint_as_float(r[j + 1]),
                                __uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, ncols);
}

cudaError_t tc_core_launch(const TcCoreArgs &g, cudaStream_t st) {
    const int smem = tc_core_smem_bytes(g.BN, g.nphase, g.band_rows, g.b_stages);
    cudaError_t e =
        cudaFuncSetAttribute(tdc_tc_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.M + kBM - 1) / kBM, g.ntiles);
    tdc_tc_core_kernel<<<grid, kCoreThreads, smem, st>>>(g);
    return cudaGetLastError();
}

int tc_smem_bytes(int BN, int stages) {
    return 1024 /*align slack*/ + stages * (kATileBytes + BN * kBK * 4) + (2 * stages + 1) * 8 + 16;
}

int tc_pick_stages(int BN, int iters, int max_smem) {
    int s = 8;
    while (s > 2 && tc_smem_bytes(BN, s) > max_smem) --s;
    if (s > iters) s = iters < 2 ? 2 : iters;
    return s;
}

// ----------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D fp32 row-major [rows][pitch] matrix, K extent k_extent, box {32, box_rows}, 128B swizzle.
bool make_tma_2d(CUtensorMap *map, const float *base, long long rows, int k_extent, int pitch,
                 int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)k_extent, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
    cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims,
                     strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool make_tma_4d_nhwc(CUtensorMap *map, const float *x, int C, int W, int H, int B, int box_w,
                      int box_h) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
    cuuint32_t box[4] = {32, (cuuint32_t)box_w, (cuuint32_t)box_h, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(x), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

cudaError_t tc_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapB, const TcGemmArgs &g,
                           int grid_n, cudaStream_t st) {
    const int smem = tc_smem_bytes(g.BN, g.stages);
    cudaError_t e =
        cudaFuncSetAttribute(tdc_tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    dim3 grid((g.M + kBM - 1) / kBM, grid_n);
    tdc_tc_gemm_kernel<<<grid, kTcThreads, smem, st>>>(mapA, mapB, g);
    return cudaGetLastError();
}

}  // namespace tdc
