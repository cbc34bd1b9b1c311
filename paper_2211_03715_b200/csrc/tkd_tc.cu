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
        float *dst = valid ? g.out + dst_row * g.ldo : nullptr;
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
            if (n + 32 <= g.Nn && (g.ldo & 3) == 0) {
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
