// tkd_bf16.cu -- the 3-launch TKD path in 3xBF16 (TDC_MATH_3XBF16): fp32-grade
// accuracy from bf16 tensor-core products.
//
// Every operand x is split into bf16 hi = RN(x) and lo = RN(x - hi)
// (|x - hi - lo| <= 2^-17 |x|) and each product is hi*hi + hi*lo + lo*hi,
// accumulated in fp32 in TMEM (the dropped lo*lo term is ~2^-16 relative;
// ~1e-5 max-normalized on the ResNet-18 shapes vs the 1e-4 tolerance).  A
// kind::f16 tcgen05.mma covers K = 16 for about the cost of a K = 8 kind::tf32
// one, so this needs half the MMA instructions of 3xTF32.
//
// Same structure as tkd_tc.cu (persistent kernels, double-buffered TMEM
// accumulators, coalesced epilogues), with these operand formats:
//   stage 1  A = X: fp32 NHWC by TMA (two 32-channel boxes = one 64-channel
//            chunk) into a staging area; a converter warpgroup writes the bf16
//            hi/lo tiles in the 128B-swizzled K-major layout.  B = U_in^T bf16.
//            Epilogue: X' hi/lo, planar bf16 [c/8][row][8] (16-byte rows).
//   stage 2  the core convolution on a shared-memory X' band (planar bf16,
//            K = 16 = two 8-channel planes per MMA); epilogue: Z hi/lo bf16
//            row-major [row][D2p].
//   stage 3  A = Z hi/lo by TMA (bf16 boxes {64, 128}), B = U_out bf16,
//            epilogue writes fp32 Y (+bias).
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"
#include "tkd_common.cuh"

namespace tdc {

using namespace sm100;

#ifdef TDC_TIMELINE
__device__ unsigned long long g_tdc_bf_tl[4 * 64 * 8];
__device__ unsigned int g_tdc_bf_seq;
__device__ __forceinline__ void bftl(int seq, int it, int ev) {
    if (blockIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_bf_tl[((seq & 3) * 64 + it) * 8 + ev] = t;
    }
}
extern "C" int tdc_debug_bf_timeline(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_bf_tl, sizeof(unsigned long long) * n);
}
#define BFTL(seq, it, ev) bftl((seq), (it), (ev))
#else
#define BFTL(seq, it, ev) ((void)0)
#endif

constexpr int kBM16 = 128;
constexpr int kBK16 = 64;                       // bf16 elements per K chunk = one 128 B row
constexpr int kATile16 = kBM16 * kBK16 * 2;     // 16 KB per hi or lo tile
constexpr int kStage32 = kBM16 * 32 * 4 * 2;    // fp32 staging of one 64-channel chunk (2 boxes)
constexpr int kEpiScratch16 = 4 * 4096;

// 32 rows x 64 bytes (32 bf16) per warp, row `lane` held by lane `lane` as 16
// packed words; transposed through shared memory so each global store covers
// eight full 64-byte row segments.
__device__ __forceinline__ void warp_store_block32_b16(float *scratch, const uint32_t (&w)[16],
                                                       void *row_ptr, int lane) {
    const uint32_t base = smem_u32(scratch);
#pragma unroll
    for (int c = 0; c < 4; ++c)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                         base + (uint32_t)(lane * 4 + (c ^ (lane & 3))) * 16),
                     "r"(w[4 * c]), "r"(w[4 * c + 1]), "r"(w[4 * c + 2]), "r"(w[4 * c + 3])
                     : "memory");
    __syncwarp();
    const int c = lane & 3;
    uint4 val[4];
    unsigned long long dst[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = i * 8 + (lane >> 2);
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(val[i].x), "=r"(val[i].y), "=r"(val[i].z), "=r"(val[i].w)
                     : "r"(base + (uint32_t)(r * 4 + (c ^ (r & 3))) * 16));
        dst[i] = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(row_ptr), r);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (dst[i])
            asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(
                             reinterpret_cast<uint4 *>(dst[i]) + c),
                         "r"(val[i].x), "r"(val[i].y), "r"(val[i].z), "r"(val[i].w)
                         : "memory");
    __syncwarp();
}

// ============================================================ GEMM (stages 1, 3)
constexpr int kConvThreads16 = 256;  // 8 converter warps (stage 1 is converter-paced otherwise)

template <bool CONVERT>
__global__ void __launch_bounds__(CONVERT ? 192 + kConvThreads16 : 192, 1)
tdc_bf_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapAlo,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapBlo,
                   const TcGemmArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = g.stages, BN = g.BN;
    const uint32_t b_tile = (uint32_t)BN * kBK16 * 2;
    const uint32_t half = kATile16 + b_tile;                  // hi -> lo offset
    const uint32_t slot_bytes = 2 * half + (CONVERT ? kStage32 : 0);
    // slot: A hi | B hi | A lo | B lo | [fp32 staging of A]
    float *epi_scratch = reinterpret_cast<float *>(smem + (size_t)S * slot_bytes);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * slot_bytes + kEpiScratch16);
    uint64_t *conv = full + S;
    uint64_t *empty = conv + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ncols = 32;
    while ((int)ncols < BN) ncols *= 2;
    const int mtiles = (g.M + kBM16 - 1) / kBM16;
    const int num_tiles = mtiles * g.ntiles;
    const int iters = g.taps * g.kchunks;
#ifdef TDC_TIMELINE
    const int seq = (int)*(volatile unsigned int *)&g_tdc_bf_seq;
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&conv[i], kConvThreads16);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ------------------------------------- TMA producer
        const uint32_t bytes = 2 * kATile16 + 2 * b_tile;  // staging fp32 == A hi + A lo bytes
        Ring r(S);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tit) {
            const int m0 = (t % mtiles) * kBM16, n0 = (t / mtiles) * BN;
            int tap = 0, kc = 0;
            for (int i = 0; i < iters; ++i, r.next()) {
                mbar_wait(&empty[r.slot], r.phase ^ 1);
                if (i == 0 && lane == 0) BFTL(seq, tit, 0);  // producer issues tile
                if (elect_one()) {
                    uint8_t *base = smem + (size_t)r.slot * slot_bytes;
                    mbar_arrive_expect_tx(&full[r.slot], bytes);
                    if (CONVERT) {  // fp32 X: channels [64kc, 64kc+32) and [64kc+32, 64kc+64)
                        tma_load_2d(base + 2 * half, &mapA, &full[r.slot], kc * 64, m0 + g.a_off[tap]);
                        tma_load_2d(base + 2 * half + kStage32 / 2, &mapA, &full[r.slot], kc * 64 + 32,
                                    m0 + g.a_off[tap]);
                    } else {
                        tma_load_2d(base, &mapA, &full[r.slot], kc * kBK16, m0 + g.a_off[tap]);
                        tma_load_2d(base + half, &mapAlo, &full[r.slot], kc * kBK16, m0 + g.a_off[tap]);
                    }
                    tma_load_2d(base + kATile16, &mapB, &full[r.slot], kc * kBK16, g.b_off[tap] + n0);
                    tma_load_2d(base + half + kATile16, &mapBlo, &full[r.slot], kc * kBK16,
                                g.b_off[tap] + n0);
                }
                __syncwarp();
                if (++kc == g.kchunks) {
                    kc = 0;
                    ++tap;
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------ MMA issuer
        const uint32_t idesc = idesc_bf16(kBM16, BN);
        const uint64_t da = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t db = sdesc_kmajor_sw128(smem_u32(smem + kATile16));
        const uint32_t lo = half >> 4;
        Ring r(S), acc(2);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next(), ++tit) {
            mbar_wait(&tempty[acc.slot], acc.phase ^ 1);
            tc_fence_after();
            if (lane == 0) BFTL(seq, tit, 1);  // MMA: accumulator free
            const uint32_t d = tmem + acc.slot * ncols;
            for (int i = 0; i < iters; ++i, r.next()) {
                mbar_wait(CONVERT ? &conv[r.slot] : &full[r.slot], r.phase);
                tc_fence_after();
                if (i == 0 && lane == 0) BFTL(seq, tit, 2);  // MMA: operands ready
                if (elect_one()) {
                    const uint64_t a = da + ((r.slot * slot_bytes) >> 4);
                    const uint64_t b = db + ((r.slot * slot_bytes) >> 4);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {  // K = 16 bf16 = 32 B per MMA
                        mma_bf16(d, a + j * 2, b + j * 2, idesc, (i | j) != 0);
                        mma_bf16(d, a + j * 2, b + lo + j * 2, idesc, 1);  // hi * lo
                        mma_bf16(d, a + lo + j * 2, b + j * 2, idesc, 1);  // lo * hi
                    }
                    mma_commit(&empty[r.slot]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(&tfull[acc.slot]);
            __syncwarp();
            if (lane == 0) BFTL(seq, tit, 3);  // MMA: issued
        }
    } else if (warp < 6) {  // --------------------------------- epilogue
        const int q = warp & 3;
        float *scratch = epi_scratch + q * 1024;
        Ring acc(2);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next(), ++tit) {
            const int m0 = (t % mtiles) * kBM16, n0 = (t / mtiles) * BN;
            mbar_wait(&tfull[acc.slot], acc.phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) BFTL(seq, tit, 4);  // epilogue: accumulator ready
            long long dst_row = 0;
            const bool valid = remap_row(g, m0 + q * 32 + lane, &dst_row);
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(src + c, r);
                tmem_ld_wait();
                const int n = n0 + c;
                if (n >= g.Nn) continue;  // warp-uniform
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                if (g.out_bf16) {  // X' hi/lo planar bf16: plane n/8 at (plane * stride + row) * 8
                    if (valid) {
                        __nv_bfloat16 *hi = reinterpret_cast<__nv_bfloat16 *>(g.out);
                        __nv_bfloat16 *lo = reinterpret_cast<__nv_bfloat16 *>(g.out_lo);
#pragma unroll
                        for (int pl = 0; pl < 4; ++pl) {
                            uint4 h, l;
                            split_bf16x8(v + 8 * pl, h, l);
                            const long long off = ((long long)((n >> 3) + pl) * g.planar_stride + dst_row) * 8;
                            *reinterpret_cast<uint4 *>(hi + off) = h;
                            *reinterpret_cast<uint4 *>(lo + off) = l;
                        }
                    }
                } else {  // fp32 Y (+bias), row-major, coalesced through shared memory
                    if (g.bias) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n + j < g.Nn) v[j] += __ldg(&g.bias[n + j]);
                    }
                    float *dst = g.out + dst_row * g.ldo;
                    if (n + 32 <= g.Nn && (g.ldo & 3) == 0) {
                        warp_store_block32(scratch, v, valid ? dst + n : nullptr, lane);
                    } else if (valid) {
                        for (int j = 0; j < 32 && n + j < g.Nn; ++j) dst[n + j] = v[j];
                    }
                }
            }
            tc_fence_before();
            mbar_arrive_relaxed(&tempty[acc.slot]);
            if (warp == 2 && lane == 0) BFTL(seq, tit, 5);  // epilogue: done
        }
    } else if (CONVERT) {  // --------------- converter: fp32 staging -> bf16 hi/lo tiles
        const int tid = threadIdx.x - 192;
        Ring r(S);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tit) {
            for (int i = 0; i < iters; ++i, r.next()) {
                mbar_wait(&full[r.slot], r.phase);
                if (i == 0 && tid == 0) BFTL(seq, tit, 6);  // converter: X landed
                const uint32_t base = smem_u32(smem + (size_t)r.slot * slot_bytes);
                const uint32_t stage = base + 2 * half;
#pragma unroll
                for (int k = 0; k < 1024 / kConvThreads16; ++k) {
                    const int item = k * kConvThreads16 + tid;  // row r, 8-channel chunk c8
                    const int row = item >> 3, c8 = item & 7;
                    const uint32_t box = stage + (uint32_t)(c8 >> 2) * (kStage32 / 2) + row * 128;
                    const int j0 = (c8 & 3) * 2;              // fp32 16-byte chunk index in the box
                    const float4 f0 = ld_shared_v4(box + ((j0 ^ (row & 7)) << 4));
                    const float4 f1 = ld_shared_v4(box + (((j0 + 1) ^ (row & 7)) << 4));
                    const float v[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
                    uint4 h, l;
                    split_bf16x8(v, h, l);
                    const uint32_t dsto = row * 128 + ((c8 ^ (row & 7)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + dsto), "r"(h.x),
                                 "r"(h.y), "r"(h.z), "r"(h.w)
                                 : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + half + dsto),
                                 "r"(l.x), "r"(l.y), "r"(l.z), "r"(l.w)
                                 : "memory");
                }
                fence_proxy_async_smem();
                mbar_arrive(&conv[r.slot]);
                if (i == iters - 1 && tid == 0) BFTL(seq, tit, 7);  // converter: done
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * ncols);
#ifdef TDC_TIMELINE
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_tdc_bf_seq, 1u);
#endif
}

int bf_smem_bytes(int BN, int stages, int convert) {
    const int half = kATile16 + BN * kBK16 * 2;
    return 1024 + stages * (2 * half + (convert ? kStage32 : 0)) + kEpiScratch16 +
           (3 * stages + 4) * 8 + 16;
}

int bf_pick_stages(int BN, int max_smem, int convert) {
    int s = 6;
    while (s > 2 && bf_smem_bytes(BN, s, convert) > max_smem) --s;
    return s;
}

cudaError_t bf_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapAlo, const CUtensorMap &mapB,
                           const CUtensorMap &mapBlo, const TcGemmArgs &g, int grid, cudaStream_t st) {
    const int smem = bf_smem_bytes(g.BN, g.stages, g.a_convert);
    cudaError_t e;
    if (g.a_convert) {
        e = cudaFuncSetAttribute(tdc_bf_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(tdc_bf_gemm_kernel<true>, grid, 192 + kConvThreads16, smem, st, mapA, mapAlo, mapB, mapBlo, g);
    } else {
        e = cudaFuncSetAttribute(tdc_bf_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(tdc_bf_gemm_kernel<false>, grid, 192, smem, st, mapA, mapAlo, mapB, mapBlo, g);
    }
    return cudaGetLastError();
}

// ============================================================ core conv (stage 2)
__host__ __device__ inline int bf_core_a_half(int nphase, int band_rows) {
    return nphase * 4 * band_rows * 16;  // 4 planes of 8 bf16 channels per 32-channel chunk
}

int bf_core_smem_bytes(int BN, int nphase, int band_rows, int b_stages) {
    return 1024 + 2 * 2 * bf_core_a_half(nphase, band_rows) + b_stages * 2 * BN * 64 + kEpiScratch16 +
           (4 + 2 * b_stages + 4) * 8 + 16;
}

__global__ void __launch_bounds__(192, 1) tdc_bf_core_kernel(const TcCoreArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int BN = g.BN, SB = g.b_stages;
    const uint32_t a_half = bf_core_a_half(g.nphase, g.band_rows);
    const uint32_t a_bytes = 2 * a_half;
    const uint32_t b_half = BN * 64;  // [4 planes][BN][8 bf16]
    const uint32_t b_bytes = 2 * b_half;
    uint8_t *a_slots = smem;
    uint8_t *b_slots = smem + 2 * (size_t)a_bytes;
    float *epi_scratch = reinterpret_cast<float *>(b_slots + (size_t)SB * b_bytes);
    uint64_t *a_full = reinterpret_cast<uint64_t *>(b_slots + (size_t)SB * b_bytes + kEpiScratch16);
    uint64_t *a_empty = a_full + 2;
    uint64_t *b_full = a_empty + 2;
    uint64_t *b_empty = b_full + SB;
    uint64_t *tfull = b_empty + SB;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ncols = 32;
    while ((int)ncols < BN) ncols *= 2;
    const int mtiles = (g.M + kBM16 - 1) / kBM16;
    const int num_tiles = mtiles * g.ntiles;
    const __nv_bfloat16 *xg = reinterpret_cast<const __nv_bfloat16 *>(g.xg);
    const __nv_bfloat16 *xg_lo = reinterpret_cast<const __nv_bfloat16 *>(g.xg_lo);
    const __nv_bfloat16 *w = reinterpret_cast<const __nv_bfloat16 *>(g.w);
    const __nv_bfloat16 *w_lo = reinterpret_cast<const __nv_bfloat16 *>(g.w_lo);

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
        }
        for (int i = 0; i < SB; ++i) {
            mbar_init(&b_full[i], 1);
            mbar_init(&b_empty[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, 2 * ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_slot;
    const uint32_t band_bytes = (uint32_t)g.band_rows * 16;

    if (warp == 0) {  // ---------------------------------- bulk-copy producer
        Ring ra(2), rb(SB);
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
            const int m0 = (t % mtiles) * kBM16, nt = t / mtiles;
            for (int kc = 0; kc < g.kchunks; ++kc, ra.next()) {
                mbar_wait(&a_empty[ra.slot], ra.phase ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&a_full[ra.slot], a_bytes);
                    uint8_t *dst = a_slots + (size_t)ra.slot * a_bytes;
                    for (int ph = 0; ph < g.nphase; ++ph)
                        for (int kg = 0; kg < 4; ++kg) {
                            const long long off = ((long long)(kc * 4 + kg) * g.plane_stride +
                                                   (long long)g.phase_src[ph] * g.phase_rows + m0) * 8;
                            bulk_load(dst + (size_t)(ph * 4 + kg) * band_bytes, xg + off, band_bytes,
                                      &a_full[ra.slot]);
                            bulk_load(dst + a_half + (size_t)(ph * 4 + kg) * band_bytes, xg_lo + off,
                                      band_bytes, &a_full[ra.slot]);
                        }
                }
                __syncwarp();
                for (int tap = 0; tap < g.taps; ++tap, rb.next()) {
                    mbar_wait(&b_empty[rb.slot], rb.phase ^ 1);
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&b_full[rb.slot], b_bytes);
                        const long long woff =
                            ((long long)(tap * g.kchunks + kc) * g.ntiles + nt) * BN * 32;
                        uint8_t *dst = b_slots + (size_t)rb.slot * b_bytes;
                        bulk_load(dst, w + woff, b_half, &b_full[rb.slot]);
                        bulk_load(dst + b_half, w_lo + woff, b_half, &b_full[rb.slot]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------ MMA issuer
        const uint32_t idesc = idesc_bf16(kBM16, BN);
        const uint64_t da = sdesc_kmajor_none(smem_u32(a_slots), band_bytes, 128);
        const uint64_t db = sdesc_kmajor_none(smem_u32(b_slots), BN * 16, 128);
        Ring ra(2), rb(SB), acc(2);
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next()) {
            mbar_wait(&tempty[acc.slot], acc.phase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc.slot * ncols;
            bool first = true;
            for (int kc = 0; kc < g.kchunks; ++kc, ra.next()) {
                mbar_wait(&a_full[ra.slot], ra.phase);
                for (int tap = 0; tap < g.taps; ++tap, rb.next()) {
                    mbar_wait(&b_full[rb.slot], rb.phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t a =
                            da + ((ra.slot * a_bytes + (uint32_t)g.tap_phase[tap] * 4 * band_bytes +
                                   (uint32_t)g.tap_off[tap] * 16) >> 4);
                        const uint64_t b = db + ((rb.slot * b_bytes) >> 4);
#pragma unroll
                        for (int j = 0; j < 2; ++j) {  // K = 16 = two 8-channel planes
                            const uint64_t aj = a + ((j * 2 * band_bytes) >> 4);
                            const uint64_t bj = b + ((j * 2 * BN * 16) >> 4);
                            mma_bf16(d, aj, bj, idesc, !(first && j == 0));
                            mma_bf16(d, aj, bj + (b_half >> 4), idesc, 1);
                            mma_bf16(d, aj + (a_half >> 4), bj, idesc, 1);
                        }
                        mma_commit(&b_empty[rb.slot]);
                    }
                    __syncwarp();
                    first = false;
                }
                if (elect_one()) mma_commit(&a_empty[ra.slot]);
                __syncwarp();
            }
            if (elect_one()) mma_commit(&tfull[acc.slot]);
            __syncwarp();
        }
    } else {  // ------------------------------ epilogue warps 2..5: Z hi/lo bf16
        const int q = warp & 3;
        float *scratch = epi_scratch + q * 1024;
        __nv_bfloat16 *z = reinterpret_cast<__nv_bfloat16 *>(g.z);
        __nv_bfloat16 *z_lo = reinterpret_cast<__nv_bfloat16 *>(g.z_lo);
        Ring acc(2);
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next()) {
            const int m0 = (t % mtiles) * kBM16, n0 = (t / mtiles) * BN;
            mbar_wait(&tfull[acc.slot], acc.phase);
            tc_fence_after();
            const int m = m0 + q * 32 + lane;
            bool valid = m < g.M;
            long long dst_row = 0;
            if (valid) {
                const int ox = m % g.Wq;
                const int tt = m / g.Wq;
                const int oy = tt % g.Hq;
                const int b = tt / g.Hq;
                valid = oy < g.Ho && ox < g.Wo;
                dst_row = ((long long)b * g.Ho + oy) * g.Wo + ox;
            }
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(src + c, r);
                tmem_ld_wait();
                if (n0 + c >= g.Nn) continue;  // warp-uniform
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                uint32_t hw[16], lw[16];
#pragma unroll
                for (int pl = 0; pl < 4; ++pl) {
                    uint4 h, l;
                    split_bf16x8(v + 8 * pl, h, l);
                    hw[4 * pl] = h.x; hw[4 * pl + 1] = h.y; hw[4 * pl + 2] = h.z; hw[4 * pl + 3] = h.w;
                    lw[4 * pl] = l.x; lw[4 * pl + 1] = l.y; lw[4 * pl + 2] = l.z; lw[4 * pl + 3] = l.w;
                }
                const long long off = dst_row * g.ldz + n0 + c;
                warp_store_block32_b16(scratch, hw, valid ? (void *)(z + off) : nullptr, lane);
                warp_store_block32_b16(scratch, lw, valid ? (void *)(z_lo + off) : nullptr, lane);
            }
            tc_fence_before();
            mbar_arrive_relaxed(&tempty[acc.slot]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * ncols);
}

cudaError_t bf_core_launch(const TcCoreArgs &g, int grid, cudaStream_t st) {
    const int smem = bf_core_smem_bytes(g.BN, g.nphase, g.band_rows, g.b_stages);
    cudaError_t e = cudaFuncSetAttribute(tdc_bf_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(tdc_bf_core_kernel, grid, 192, smem, st, g);
}

}  // namespace tdc
