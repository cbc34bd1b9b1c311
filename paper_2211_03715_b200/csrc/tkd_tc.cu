// tkd_tc.cu -- the TKD layer as three tcgen05 launches (the "3-launch" path).
//
// Used where the fused kernel (tkd_fused.cu) does not pay off -- small images
// with large ranks, whose weights dwarf a tile's activations -- and for the
// fp32-accurate 3xTF32 math mode on every shape.
//
//   stage 1 (a1)  tdc_tc_gemm_kernel: A = X (NHWC rows = pixels, K = C) by TMA,
//                 Bt = U_in^T; the epilogue scatters each pixel's D1 ranks into the
//                 zero-bordered "phase grid" X'g, stored planar [kg][row][4] so
//                 stage 2 can bulk-copy row bands (reading R6: zero padding).
//   stage 2 (a2)  tdc_tc_core_kernel: per 32-channel chunk of D1 the X' band of a
//                 128-row output tile is copied into shared memory ONCE; each of
//                 the K*K taps is a descriptor whose start is shifted by the tap's
//                 constant row offset (r/s)*Wq + t/s -- the core convolution
//                  as an implicit GEMM without per-tap data movement.
//   stage 3 (a3)  tdc_tc_gemm_kernel: A = Z, Bt = U_out (N x D2 is K-major), bias
//                 in the epilogue, rows written straight to Y (NHWC).
//
// 3xTF32 (TDC_MATH_3XTF32): every operand is split x = hi + lo with
// hi = cvt.rna.tf32(x) and lo = x - hi (exact in fp32), and each product is
// hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM (~5e-7 max-normalized
// error on the R18 shapes vs ~5e-4 for one TF32 product).  Weights are split at
// plan time, X' and Z by the producing epilogue, and the user's X by a converter
// warpgroup between the TMA landing and the MMA.
//
// Kernel anatomy (one 128 x BN output tile per CTA):
//   warp 0      producer (TMA / bulk copies) into an S-stage mbarrier ring;
//   warp 1      TMEM owner + MMA issue (warp-uniform loop, one elected lane);
//   warps 2-5   epilogue: tcgen05.ld 32x32b, one TMEM lane = one output row;
//   warps 6-9   (3xTF32 stage 1 only) converter: hi in place, lo alongside.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.h"
#include "sm100.cuh"
#include "tkd_common.cuh"

namespace tdc {

using namespace sm100;

constexpr int kBM = 128;
constexpr int kBK = 32;                     // fp32 elements per K chunk = one 128 B swizzle row
constexpr int kATileBytes = kBM * kBK * 4;  // 16 KB

#ifdef TDC_TIMELINE
// Debug build only: per-CTA %globaltimer stamps [cta][8] of the GEMM kernel.
__device__ unsigned long long g_tdc_gemm_tl[4096 * 8];
__device__ __forceinline__ void gtl(int ev) {
    const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (cta < 4096) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_gemm_tl[cta * 8 + ev] = t;
    }
}
extern "C" int tdc_debug_gemm_timeline(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_gemm_tl, sizeof(unsigned long long) * n);
}
#define GTL(ev) gtl(ev)
// per-tile events of CTA 0: [launch seq % 4][tile iter][8]
__device__ unsigned long long g_tdc_tile_tl[4 * 64 * 8];
__device__ unsigned int g_tdc_launch_seq;
__device__ __forceinline__ void ttl(int seq, int it, int ev) {
    if (blockIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_tile_tl[((seq & 3) * 64 + it) * 8 + ev] = t;
    }
}
extern "C" int tdc_debug_tile_timeline(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_tile_tl, sizeof(unsigned long long) * n);
}
#define TTL(seq, it, ev) ttl((seq), (it), (ev))
#else
#define GTL(ev) ((void)0)
#define TTL(seq, it, ev) ((void)0)
#endif

__device__ __forceinline__ void split4(const float *v, float4 *hi, float4 *lo) {
    const float4 h = make_float4(rna_tf32(v[0]), rna_tf32(v[1]), rna_tf32(v[2]), rna_tf32(v[3]));
    *hi = h;
    *lo = make_float4(v[0] - h.x, v[1] - h.y, v[2] - h.z, v[3] - h.w);
}

// Store 32 consecutive output columns of one row (optionally split into hi/lo).
__device__ __forceinline__ void store_row32(float *dst, float *dst_lo, long long planar, int n,
                                            int Nn, bool ldo_vec, const float (&v)[32], bool split) {
    if (planar) {  // [col/4][row][4]: lanes = consecutive rows -> coalesced
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            const long long off = (long long)((n + j) >> 2) * planar;
            if (split)
                split4(v + j, reinterpret_cast<float4 *>(dst + off), reinterpret_cast<float4 *>(dst_lo + off));
            else
                *reinterpret_cast<float4 *>(dst + off) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
    } else if (n + 32 <= Nn && ldo_vec) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) {
            if (split)
                split4(v + j, reinterpret_cast<float4 *>(dst + n + j),
                       reinterpret_cast<float4 *>(dst_lo + n + j));
            else
                *reinterpret_cast<float4 *>(dst + n + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            if (n + j >= Nn) continue;
            if (split) {
                const float h = rna_tf32(v[j]);
                dst[n + j] = h;
                dst_lo[n + j] = v[j] - h;
            } else {
                dst[n + j] = v[j];
            }
        }
    }
}

// ============================================================ GEMM with taps
// Persistent: each CTA walks tiles t = blockIdx.x, += gridDim.x (M-tile fastest,
// so concurrently running CTAs share a weight tile in L2).  The TMEM accumulator
// is double-buffered, so the epilogue of tile i (TMEM -> global) overlaps the
// loads and MMAs of tile i+1 and HBM sees reads and writes interleaved instead
// of the lock-step load/compute/store waves of a one-tile-per-CTA launch.
constexpr int kEpiScratch = 4 * 4096;  // 4 epilogue warps x 32x32 fp32 transpose blocks

template <bool SPLIT>
__global__ void __launch_bounds__(SPLIT ? 320 : 192, 1)
tdc_tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapAlo,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapBlo,
                   const TcGemmArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int S = g.stages, BN = g.BN;
    const uint32_t b_tile = (uint32_t)BN * kBK * 4;
    const uint32_t slot_bytes = (SPLIT ? 2 : 1) * (kATileBytes + b_tile);
    // slot layout: A hi | B hi | [A lo | B lo]
    float *epi_scratch = reinterpret_cast<float *>(smem + (size_t)S * slot_bytes);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)S * slot_bytes + kEpiScratch);
    uint64_t *conv = full + S;
    uint64_t *empty = conv + S;
    uint64_t *tfull = empty + S;    // [2]
    uint64_t *tempty = tfull + 2;   // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ncols = 32;  // TMEM allocations are powers of two >= 32
    while ((int)ncols < BN) ncols *= 2;
    const bool convert = SPLIT && g.a_convert;
    const int mtiles = (g.M + kBM - 1) / kBM;
    const int num_tiles = mtiles * g.ntiles;
    const int iters = g.taps * g.kchunks;
    if (threadIdx.x == 0) GTL(0);  // CTA start
#ifdef TDC_TIMELINE
    const int seq = (int)*(volatile unsigned int *)&g_tdc_launch_seq;
#endif

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&conv[i], 128);
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
    if (threadIdx.x == 0) GTL(1);  // setup done (barriers + TMEM)
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ------------------------------------- TMA producer
        const uint32_t bytes = (SPLIT && !convert ? 2 : 1) * kATileBytes + (SPLIT ? 2 : 1) * b_tile;
        Ring r(S);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tit) {
            const int m0 = (t % mtiles) * kBM, n0 = (t / mtiles) * BN;
            int tap = 0, kc = 0;
            if (lane == 0) TTL(seq, tit, 0);  // producer starts tile
            for (int i = 0; i < iters; ++i, r.next()) {
                mbar_wait(&empty[r.slot], r.phase ^ 1);
                if (elect_one()) {
                    uint8_t *base = smem + (size_t)r.slot * slot_bytes;
                    mbar_arrive_expect_tx(&full[r.slot], bytes);
                    tma_load_2d(base, &mapA, &full[r.slot], kc * kBK, m0 + g.a_off[tap]);
                    tma_load_2d(base + kATileBytes, &mapB, &full[r.slot], kc * kBK, g.b_off[tap] + n0);
                    if (SPLIT) {
                        if (!convert)
                            tma_load_2d(base + kATileBytes + b_tile, &mapAlo, &full[r.slot], kc * kBK,
                                        m0 + g.a_off[tap]);
                        tma_load_2d(base + 2 * kATileBytes + b_tile, &mapBlo, &full[r.slot], kc * kBK,
                                    g.b_off[tap] + n0);
                    }
                }
                __syncwarp();
                if (++kc == g.kchunks) {
                    kc = 0;
                    ++tap;
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------ MMA issuer
        const uint32_t idesc = idesc_tf32(kBM, BN);
        const uint64_t da = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t db = sdesc_kmajor_sw128(smem_u32(smem + kATileBytes));
        const uint32_t lo_off = (kATileBytes + b_tile) >> 4;  // hi -> lo, 16-byte units
        Ring r(S), acc(2);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next(), ++tit) {
            mbar_wait(&tempty[acc.slot], acc.phase ^ 1);  // epilogue drained this buffer
            tc_fence_after();
            if (lane == 0) TTL(seq, tit, 1);  // MMA: accumulator free
            const uint32_t d = tmem + acc.slot * ncols;
            for (int i = 0; i < iters; ++i, r.next()) {
                mbar_wait(convert ? &conv[r.slot] : &full[r.slot], r.phase);
                tc_fence_after();
                if (i == 0 && lane == 0) GTL(2);  // first operands ready
                if (elect_one()) {
                    const uint64_t a = da + ((r.slot * slot_bytes) >> 4);
                    const uint64_t b = db + ((r.slot * slot_bytes) >> 4);
#pragma unroll
                    for (int j = 0; j < kBK / 8; ++j) {  // K = 8 tf32 = 32 B per MMA
                        mma_tf32(d, a + j * 2, b + j * 2, idesc, (i | j) != 0);
                        if (SPLIT) {
                            mma_tf32(d, a + j * 2, b + lo_off + j * 2, idesc, 1);  // hi * lo
                            mma_tf32(d, a + lo_off + j * 2, b + j * 2, idesc, 1);  // lo * hi
                        }
                    }
                    mma_commit(&empty[r.slot]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(&tfull[acc.slot]);
            __syncwarp();
            if (lane == 0) GTL(3);  // all MMAs of the tile issued
            if (lane == 0) TTL(seq, tit, 2);  // MMA: all issued
        }
    } else if (warp < 6) {  // --------------------------------- epilogue
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        float *scratch = epi_scratch + q * 1024;
        const bool rowmajor_vec = !g.planar_stride && (g.ldo & 3) == 0;
        Ring acc(2);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next(), ++tit) {
            const int m0 = (t % mtiles) * kBM, n0 = (t / mtiles) * BN;
            mbar_wait(&tfull[acc.slot], acc.phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) GTL(4);  // accumulator ready
            if (warp == 2 && lane == 0) TTL(seq, tit, 3);  // epilogue: accumulator ready
            long long dst_row = 0;
            const bool valid = remap_row(g, m0 + q * 32 + lane, &dst_row);
            const long long off = g.planar_stride ? dst_row * 4 : dst_row * g.ldo;
            float *dst = g.out + off;
            float *dst_lo = (SPLIT && g.out_lo) ? g.out_lo + off : nullptr;
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(src + c, r);
                tmem_ld_wait();
                if (c == 0 && warp == 2 && lane == 0) TTL(seq, tit, 6);  // first TMEM block loaded
                const int n = n0 + c;
                if (n >= g.Nn) continue;  // warp-uniform
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                if (g.bias) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (n + j < g.Nn) v[j] += __ldg(&g.bias[n + j]);
                }
                if (rowmajor_vec && n + 32 <= g.Nn) {  // coalesced through shared memory
                    if (dst_lo) {
                        float h[32], l[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            h[j] = rna_tf32(v[j]);
                            l[j] = v[j] - h[j];
                        }
                        warp_store_block32(scratch, h, valid ? dst + n : nullptr, lane);
                        warp_store_block32(scratch, l, valid ? dst_lo + n : nullptr, lane);
                    } else {
                        warp_store_block32(scratch, v, valid ? dst + n : nullptr, lane);
                    }
                } else if (valid) {
                    store_row32(dst, dst_lo, g.planar_stride, n, g.Nn, (g.ldo & 3) == 0, v,
                                dst_lo != nullptr);
                }
                if (c == 0 && warp == 2 && lane == 0) TTL(seq, tit, 7);  // first block stored
            }
            tc_fence_before();
            mbar_arrive_relaxed(&tempty[acc.slot]);
            if (warp == 2 && lane == 0) GTL(5);  // epilogue stores issued
            if (warp == 2 && lane == 0) TTL(seq, tit, 4);  // epilogue done
        }
    } else if (convert) {  // ------------------------ converter (3xTF32 stage 1)
        const int tid = threadIdx.x - 192;  // 0..127: each owns 128 contiguous bytes of A
        Ring r(S);
        int tit = 0;
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++tit) {
            for (int i = 0; i < iters; ++i, r.next()) {
                mbar_wait(&full[r.slot], r.phase);
                if (tid == 0 && i == 0) TTL(seq, tit, 5);  // converter: first chunk landed
                float4 *a = reinterpret_cast<float4 *>(smem + (size_t)r.slot * slot_bytes);
                float4 *lo = reinterpret_cast<float4 *>(smem + (size_t)r.slot * slot_bytes +
                                                        kATileBytes + b_tile);
#pragma unroll
                for (int j = 0; j < 8; ++j) {  // elementwise (the 128B swizzle is irrelevant);
                    const int k = j * 128 + tid;  // consecutive lanes -> consecutive 16 B
                    const float4 v = a[k];
                    const float vv[4] = {v.x, v.y, v.z, v.w};
                    split4(vv, &a[k], &lo[k]);
                }
                fence_proxy_async_smem();
                mbar_arrive(&conv[r.slot]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * ncols);
    if (threadIdx.x == 64) GTL(6);  // CTA end
#ifdef TDC_TIMELINE
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_tdc_launch_seq, 1u);
#endif
}

int tc_smem_bytes(int BN, int stages, int split) {
    return 1024 /*align slack*/ + stages * (split ? 2 : 1) * (kATileBytes + BN * kBK * 4) +
           kEpiScratch + (3 * stages + 4) * 8 + 16;
}

int persistent_occupancy(int smem_bytes, int bn) {
    int ncols = 32;
    while (ncols < bn) ncols *= 2;
    const int by_tmem = 512 / (2 * ncols);
    const int by_smem = (228 * 1024) / (smem_bytes + 1024);
    int occ = by_tmem < by_smem ? by_tmem : by_smem;
    return occ < 1 ? 1 : occ;
}

int tc_pick_stages(int BN, int iters, int max_smem, int split) {
    int s = 8;
    while (s > 2 && tc_smem_bytes(BN, s, split) > max_smem) --s;
    (void)iters;  // persistent: the ring also prefetches the next tile
    return s;
}

// ============================================================ core conv (stage 2)
constexpr int kCoreThreads = 192;

__host__ __device__ inline int core_a_slot_bytes(int nphase, int band_rows) {
    return nphase * 8 * band_rows * 16;
}

int tc_core_smem_bytes(int BN, int nphase, int band_rows, int b_stages, int split) {
    const int f = split ? 2 : 1;
    return 1024 + 2 * f * core_a_slot_bytes(nphase, band_rows) + b_stages * f * BN * 128 +
           kEpiScratch + (4 + 2 * b_stages + 4) * 8 + 16;
}

template <bool SPLIT>
__global__ void __launch_bounds__(kCoreThreads, 1) tdc_tc_core_kernel(const TcCoreArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int BN = g.BN, SB = g.b_stages;
    const uint32_t a_half = core_a_slot_bytes(g.nphase, g.band_rows);  // hi -> lo
    const uint32_t a_bytes = a_half * (SPLIT ? 2 : 1);
    const uint32_t b_half = BN * 128;
    const uint32_t b_bytes = b_half * (SPLIT ? 2 : 1);
    uint8_t *a_slots = smem;
    uint8_t *b_slots = smem + 2 * (size_t)a_bytes;
    float *epi_scratch = reinterpret_cast<float *>(b_slots + (size_t)SB * b_bytes);
    uint64_t *a_full = reinterpret_cast<uint64_t *>(b_slots + (size_t)SB * b_bytes + kEpiScratch);
    uint64_t *a_empty = a_full + 2;
    uint64_t *b_full = a_empty + 2;
    uint64_t *b_empty = b_full + SB;
    uint64_t *tfull = b_empty + SB;  // [2]
    uint64_t *tempty = tfull + 2;    // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ncols = 32;  // TMEM allocations are powers of two >= 32
    while ((int)ncols < BN) ncols *= 2;
    const int mtiles = (g.M + kBM - 1) / kBM;
    const int num_tiles = mtiles * g.ntiles;

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
            const int m0 = (t % mtiles) * kBM, nt = t / mtiles;
            for (int kc = 0; kc < g.kchunks; ++kc, ra.next()) {
                mbar_wait(&a_empty[ra.slot], ra.phase ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&a_full[ra.slot], a_bytes);
                    uint8_t *dst = a_slots + (size_t)ra.slot * a_bytes;
                    for (int ph = 0; ph < g.nphase; ++ph)
                        for (int kg = 0; kg < 8; ++kg) {
                            const long long off = (long long)(kc * 8 + kg) * g.plane_stride +
                                                  ((long long)g.phase_src[ph] * g.phase_rows + m0) * 4;
                            bulk_load(dst + (size_t)(ph * 8 + kg) * band_bytes, g.xg + off, band_bytes,
                                      &a_full[ra.slot]);
                            if (SPLIT)
                                bulk_load(dst + a_half + (size_t)(ph * 8 + kg) * band_bytes,
                                          g.xg_lo + off, band_bytes, &a_full[ra.slot]);
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
                        bulk_load(dst, g.w + woff, b_half, &b_full[rb.slot]);
                        if (SPLIT) bulk_load(dst + b_half, g.w_lo + woff, b_half, &b_full[rb.slot]);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {  // ------------------------------ MMA issuer
        const uint32_t idesc = idesc_tf32(kBM, BN);
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
                            da + ((ra.slot * a_bytes + (uint32_t)g.tap_phase[tap] * 8 * band_bytes +
                                   (uint32_t)g.tap_off[tap] * 16) >> 4);
                        const uint64_t b = db + ((rb.slot * b_bytes) >> 4);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {  // K = 8 = two 4-channel planes
                            const uint64_t aj = a + ((j * 2 * band_bytes) >> 4);
                            const uint64_t bj = b + ((j * 2 * BN * 16) >> 4);
                            mma_tf32(d, aj, bj, idesc, !(first && j == 0));
                            if (SPLIT) {
                                mma_tf32(d, aj, bj + (b_half >> 4), idesc, 1);
                                mma_tf32(d, aj + (a_half >> 4), bj, idesc, 1);
                            }
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
    } else {  // --------------------------------- epilogue warps 2..5: Z compact
        const int q = warp & 3;
        float *scratch = epi_scratch + q * 1024;
        Ring acc(2);
        for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, acc.next()) {
            const int m0 = (t % mtiles) * kBM, n0 = (t / mtiles) * BN;
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
            float *dst = g.z + dst_row * g.ldz;
            float *dst_lo = SPLIT ? g.z_lo + dst_row * g.ldz : nullptr;
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(src + c, r);
                tmem_ld_wait();
                if (n0 + c >= g.Nn) continue;  // warp-uniform
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                if (SPLIT) {
                    float h[32], l[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        h[j] = rna_tf32(v[j]);
                        l[j] = v[j] - h[j];
                    }
                    warp_store_block32(scratch, h, valid ? dst + n0 + c : nullptr, lane);
                    warp_store_block32(scratch, l, valid ? dst_lo + n0 + c : nullptr, lane);
                } else {
                    warp_store_block32(scratch, v, valid ? dst + n0 + c : nullptr, lane);
                }
            }
            tc_fence_before();
            mbar_arrive_relaxed(&tempty[acc.slot]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 2 * ncols);
}

cudaError_t tc_core_launch(const TcCoreArgs &g, int grid, cudaStream_t st) {
    const int smem = tc_core_smem_bytes(g.BN, g.nphase, g.band_rows, g.b_stages, g.split);
    cudaError_t e;
    if (g.split) {
        e = cudaFuncSetAttribute(tdc_tc_core_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(tdc_tc_core_kernel<true>, grid, kCoreThreads, smem, st, g);
    } else {
        e = cudaFuncSetAttribute(tdc_tc_core_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(tdc_tc_core_kernel<false>, grid, kCoreThreads, smem, st, g);
    }
    return cudaGetLastError();
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

bool make_tma_2d_bf16(CUtensorMap *map, const void *base, long long rows, int k_extent, int pitch,
                      int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)k_extent, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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

cudaError_t tc_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapAlo,
                           const CUtensorMap &mapB, const CUtensorMap &mapBlo, const TcGemmArgs &g,
                           int grid, cudaStream_t st) {
    const int smem = tc_smem_bytes(g.BN, g.stages, g.split);
    cudaError_t e;
    if (g.split) {
        e = cudaFuncSetAttribute(tdc_tc_gemm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(tdc_tc_gemm_kernel<true>, grid, 320, smem, st, mapA, mapAlo, mapB, mapBlo, g);
    } else {
        e = cudaFuncSetAttribute(tdc_tc_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(tdc_tc_gemm_kernel<false>, grid, 192, smem, st, mapA, mapAlo, mapB, mapBlo, g);
    }
    return cudaGetLastError();
}

}  // namespace tdc
