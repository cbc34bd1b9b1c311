// tkd_fused.cu -- the whole TKD layer (§8(a) rows a1-a4) in ONE persistent
// tcgen05 kernel: HBM sees X once and Y once; X' lives in shared memory and Z in
// tensor memory.
//
// Work unit ("tile"): R output rows of one image.  Its input band is
// Rin = s*(R-1) + K rows x Wp = W + 2p columns, loaded by TMA straight from
// the NHWC input with the padding columns/rows zero-filled out of bounds
// (reading R6: zero-padding X == zero-padding X' because stage 1 is linear).
//
//   stage 1 (a1)  acc1[px][a] = sum_c X[px][c] U_in[c][a]        SS-MMA, A = X band
//                 (128B-swizzled TMA tiles), B = U_in^T chunks, ceil(Rin*Wp/128)
//                 accumulator blocks in TMEM.
//   epilogue 1    tcgen05.ld acc1 -> st.shared into the X' "phase grid" in
//                 no-swizzle K-major planar form [kg][row][4 fp32]: input
//                 pixel (yy, xx) goes to phase (yy%s, xx%s), row (yy/s)*Wq + xx/s.
//   stage 2 (a2)  acc2[m][q] = sum_{tap,a} X'[m + off(tap)][a] core[tap][a][q]:
//                 the core convolution as an implicit GEMM whose A
//                 descriptors are the X' planes shifted by each tap's constant
//                 row offset -- no data movement per tap.
//   stage 3 (a3)  acc3[m][n] = sum_q acc2[m][q] U_out[n][q]: TS-MMA, A read
//                 directly from the stage-2 accumulator in TMEM (lane = row,
//                 column = q), so Z never leaves tensor memory.
//   epilogue 3 (a4)  tcgen05.ld acc3 (+bias) -> each output element written once
//                 to Y (NHWC), no atomics (contrast P:L368-372).
//
// Warp roles (12 warps, one CTA per SM, persistent over tiles):
//   warp 0    X producer: TMA X-band chunks (32 channels each) into an
//             XS-deep ring; it runs ahead, so the next tile's band streams in
//             while the current tile is in stages 2-3.
//   warp 1    TMEM owner + single-thread MMA issue for all three stages.
//   warp 2    weight producer: bulk copies of pre-blocked weight chunks
//             (plan-time re-layout, the CRSN idea P:L338-340) into a WS-deep
//             ring, in exactly the order the MMA thread consumes them.
//   warps 4-7 epilogue 1 (on the critical path: S1 -> epi1 -> S2 -> S3);
//   warps 8-11 epilogue 3, off the critical path thanks to a double-buffered
//             stage-3 accumulator (TMEM lane quarter = warp % 4 in both groups).
#include "internal.h"
#include "sm100.cuh"

namespace tdc {

using namespace sm100;

constexpr int kFusedThreads = 384;  // 12 warps

#ifdef TDC_TIMELINE
// Debug build only: %globaltimer stamps of pipeline events for CTA 0.
__device__ unsigned long long g_tdc_timeline[64 * 32];
__device__ __forceinline__ void tl_mark(int tile_iter, int ev) {
    if (blockIdx.x == 0 && tile_iter < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_timeline[tile_iter * 32 + ev] = t;
    }
}
#define TL(it, ev) tl_mark((it), (ev))
#else
#define TL(it, ev) ((void)0)
#endif
constexpr uint32_t kXBlockBytes = 128 * 128;  // 128 rows x 32 fp32

__host__ __device__ inline int fused_w_slot_bytes(const FusedArgs &g) {
    int r = g.D1s > g.D2s ? g.D1s : g.D2s;
    r = r > g.Nh ? r : g.Nh;
    return r * 128;
}

constexpr int kEpiScratchF = 4 * 4096;  // epilogue-3 warps' 32x32 transpose blocks

int fused_smem_bytes(const FusedArgs &g) {
    return 1024 + g.XS * g.nblk1 * (int)kXBlockBytes + g.WS * fused_w_slot_bytes(g) +
           g.TR * g.D1s * 4 + kEpiScratchF + (2 * g.XS + 2 * g.WS + 6) * 8 + 16;
}

__global__ void __launch_bounds__(kFusedThreads, 1)
tdc_tkd_fused_tc_kernel(const __grid_constant__ CUtensorMap mapX, const FusedArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t x_slot = g.nblk1 * kXBlockBytes;
    const uint32_t w_slot = (uint32_t)fused_w_slot_bytes(g);
    uint8_t *x_ring = smem;
    uint8_t *w_ring = x_ring + (size_t)g.XS * x_slot;
    uint8_t *x1 = w_ring + (size_t)g.WS * w_slot;
    float *epi_scratch = reinterpret_cast<float *>(x1 + (size_t)g.TR * g.D1s * 4);
    uint64_t *x_full = reinterpret_cast<uint64_t *>(x1 + (size_t)g.TR * g.D1s * 4 + kEpiScratchF);
    uint64_t *x_empty = x_full + g.XS;
    uint64_t *w_full = x_empty + g.XS;
    uint64_t *w_empty = w_full + g.WS;
    uint64_t *acc1_full = w_empty + g.WS;
    uint64_t *x1_ready = acc1_full + 1;
    uint64_t *acc3_full = x1_ready + 1;   // [2]
    uint64_t *acc3_empty = acc3_full + 2; // [2]
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc3_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < g.XS; ++i) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_empty[i], 1);
        }
        for (int i = 0; i < g.WS; ++i) {
            mbar_init(&w_full[i], 1);
            mbar_init(&w_empty[i], 1);
        }
        mbar_init(acc1_full, 1);
        mbar_init(x1_ready, 128);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&acc3_full[i], 1);
            mbar_init(&acc3_empty[i], 128);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) tma_prefetch(&mapX);
    if (warp == 1) tmem_alloc(tmem_slot, (uint32_t)g.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_slot;

    const int kc1 = g.c_chunks, kc2 = g.D1s / 32, kc3 = g.D2s / 32;
    const uint32_t x_bytes = (uint32_t)g.Rin * g.Wp * 128;

    // Producer and MMA roles run their loops on the whole warp (warp-uniform
    // control flow, so descriptors live in uniform registers) and let one
    // elected lane issue each TMA / bulk copy / tcgen05.mma / commit.
    if (warp == 0) {  // ============================ X-band producer (TMA)
        Ring xr(g.XS);
        int it = 0;
        for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++it) {
            const int b = tile / g.tiles_per_img;
            const int oy0 = (tile - b * g.tiles_per_img) * g.R;
            const int y0 = oy0 * g.s - g.p;
            for (int kc = 0; kc < kc1; ++kc, xr.next()) {
                mbar_wait(&x_empty[xr.slot], xr.phase ^ 1);
                if (lane == 0 && kc == 0) TL(it, 0);  // X slot free, issuing chunk 0
                if (elect_one()) {
                    mbar_arrive_expect_tx(&x_full[xr.slot], x_bytes);
                    tma_load_4d(x_ring + (size_t)xr.slot * x_slot, &mapX, &x_full[xr.slot], kc * 32,
                                -g.p, y0, b);
                }
                __syncwarp();
            }
        }
    } else if (warp == 2) {  // ===================== weight-chunk producer (bulk copies)
        Ring wr(g.WS);
        auto push_w = [&](const float *src, uint32_t bytes) {
            mbar_wait(&w_empty[wr.slot], wr.phase ^ 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(&w_full[wr.slot], bytes);
                bulk_load(w_ring + (size_t)wr.slot * w_slot, src, bytes, &w_full[wr.slot]);
            }
            __syncwarp();
            wr.next();
        };
        const uint32_t b1 = g.D1s * 128, b2 = g.D2s * 128, b3 = g.Nh * 128;
        int it = 0;
        for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++it) {
            const float *src = g.w;
            if (lane == 0) TL(it, 1);  // weight producer starts this tile's chunks
            for (int kc = 0; kc < kc1; ++kc, src += g.D1s * 32) push_w(src, b1);
            for (int i = 0; i < kc2 * g.KK; ++i, src += g.D2s * 32) push_w(src, b2);
            for (int i = 0; i < g.nhalves * kc3; ++i, src += g.Nh * 32) push_w(src, b3);
        }
    } else if (warp == 1) {  // ===================== MMA issuer
        const uint32_t id1 = idesc_tf32(128, g.D1s), id2 = idesc_tf32(128, g.D2s),
                       id3 = idesc_tf32(128, g.Nh);
        const uint32_t tr16 = (uint32_t)g.TR * 16;
        const uint32_t lbo1 = g.D1s * 16, lbo2 = g.D2s * 16, lbo3 = g.Nh * 16;
        // descriptor templates; per-use offsets are added to the start-address field (16 B units)
        const uint64_t dx0 = sdesc_kmajor_sw128(smem_u32(x_ring));
        const uint64_t dw1 = sdesc_kmajor_none(smem_u32(w_ring), lbo1, 128);
        const uint64_t dw2 = sdesc_kmajor_none(smem_u32(w_ring), lbo2, 128);
        const uint64_t dw3 = sdesc_kmajor_none(smem_u32(w_ring), lbo3, 128);
        const uint64_t dx1 = sdesc_kmajor_none(smem_u32(x1), tr16, 128);
        Ring xr(g.XS), wr(g.WS), a3(g.nbuf3);
        uint32_t tpar = 0;
        int it = 0;
        for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, tpar ^= 1, ++it) {
            if (lane == 0) TL(it, 2);  // MMA: tile start
            // ---- stage 1: acc1[blk] = X band . U_in
            for (int kc = 0; kc < kc1; ++kc, xr.next(), wr.next()) {
                mbar_wait(&x_full[xr.slot], xr.phase);
                if (lane == 0 && kc == 0) TL(it, 3);  // X chunk 0 landed
                mbar_wait(&w_full[wr.slot], wr.phase);
                if (lane == 0 && kc == 0) TL(it, 4);  // W chunk 0 landed
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t ax = dx0 + ((xr.slot * x_slot) >> 4);
                    const uint64_t bw = dw1 + ((wr.slot * w_slot) >> 4);
                    // K-steps round-robin over independent accumulators (blk, j % P1)
                    // so consecutive MMAs never wait on each other's accumulate.
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        for (int blk = 0; blk < g.nblk1; ++blk)
                            mma_tf32(tmem + (blk * g.P1 + (j % g.P1)) * g.D1s,
                                     ax + ((blk * kXBlockBytes + j * 32) >> 4),
                                     bw + ((j * 2 * lbo1) >> 4), id1, (kc > 0) | (j >= g.P1));
                    mma_commit(&x_empty[xr.slot]);
                    mma_commit(&w_empty[wr.slot]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(acc1_full);
            __syncwarp();
            if (lane == 0) TL(it, 5);  // S1 issued
            // ---- stage 2 (needs X' from epilogue 1; acc2 reuses acc1's columns)
            mbar_wait(x1_ready, tpar);
            tc_fence_after();
            if (lane == 0) TL(it, 6);  // X' ready
            {
                int idx = 0;  // MMA index in stage 2; chain = idx % P2 (independent accumulators)
                for (int kc = 0; kc < kc2; ++kc)
                    for (int tap = 0; tap < g.KK; ++tap, wr.next()) {
                        if (lane == 0 && kc == 0 && tap < 9) TL(it, 14 + tap);  // before W wait
                        mbar_wait(&w_full[wr.slot], wr.phase);
                        tc_fence_after();
                        if (elect_one()) {
                            const uint64_t ad =
                                dx1 + (((uint32_t)(g.tap_phase[tap] * g.PR + g.tap_off[tap]) * 16 +
                                        (uint32_t)kc * 8 * tr16) >> 4);
                            const uint64_t bw = dw2 + ((wr.slot * w_slot) >> 4);
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                mma_tf32(tmem + ((idx + j) % g.P2) * g.D2s, ad + ((j * 2 * tr16) >> 4),
                                         bw + ((j * 2 * lbo2) >> 4), id2, idx + j >= g.P2);
                            mma_commit(&w_empty[wr.slot]);
                        }
                        __syncwarp();
                        idx += 4;
                    }
            }
            if (lane == 0) TL(it, 7);  // S2 issued
            // ---- stage 3: A = acc2 straight from TMEM
            for (int h = 0; h < g.nhalves; ++h, a3.next()) {
                mbar_wait(&acc3_empty[a3.slot], a3.phase ^ 1);
                tc_fence_after();
                if (lane == 0 && h == 0) TL(it, 8);  // acc3 buffer free
                const uint32_t acc3 = tmem + g.acc3_col + a3.slot * g.P3 * g.Nh;
                int idx = 0;
                for (int kc = 0; kc < kc3; ++kc, wr.next()) {
                    mbar_wait(&w_full[wr.slot], wr.phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint64_t bw = dw3 + ((wr.slot * w_slot) >> 4);
                        // Z = sum of the P2 stage-2 partials; by linearity each partial is
                        // multiplied into acc3 directly (TS-MMA, A from TMEM).
                        for (int c = 0; c < g.P2; ++c)
#pragma unroll
                            for (int j = 0; j < 4; ++j, ++idx)
                                mma_tf32_ts(acc3 + (idx % g.P3) * g.Nh,
                                            tmem + c * g.D2s + kc * 32 + j * 8,
                                            bw + ((j * 2 * lbo3) >> 4), id3, idx >= g.P3);
                        mma_commit(&w_empty[wr.slot]);
                    } else {
                        idx += 4 * g.P2;
                    }
                    __syncwarp();
                }
                if (elect_one()) mma_commit(&acc3_full[a3.slot]);
                __syncwarp();
            }
            if (lane == 0) TL(it, 9);  // S3 issued
        }
    } else if (warp >= 4 && warp < 8) {  // ======= epilogue 1: acc1 -> X' (critical path)
        const int q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t x1a = smem_u32(x1);
        const int band = g.Rin * g.Wp;
        uint32_t tcount = 0;
        for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++tcount) {
            mbar_wait(acc1_full, tcount & 1);
            tc_fence_after();
            if (warp == 4 && lane == 0) TL((int)tcount, 10);  // acc1 full seen
            for (int blk = 0; blk < g.nblk1; ++blk) {
                const int i = blk * 128 + q * 32 + lane;
                int dest = -1;
                if (i < band) {
                    const int yy = i / g.Wp, xx = i - yy * g.Wp;
                    const int ph = g.phase_idx[(yy % g.s) * g.s + (xx % g.s)];
                    if (ph >= 0) dest = ph * g.PR + (yy / g.s) * g.Wq + xx / g.s;
                }
                for (int c = 0; c < g.D1s; c += 32) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(tmem + lane_base + blk * g.P1 * g.D1s + c, r);
                    tmem_ld_wait();
                    for (int pp = 1; pp < g.P1; ++pp) {
                        uint32_t r2[32];
                        tmem_ld_32x32b_x32(tmem + lane_base + (blk * g.P1 + pp) * g.D1s + c, r2);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
                    }
                    if (dest >= 0) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            st_shared_v4(x1a + ((uint32_t)(c / 4 + j) * g.TR + dest) * 16,
                                         __uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                         __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3]));
                    }
                }
            }
            fence_proxy_async_smem();
            tc_fence_before();
            mbar_arrive(x1_ready);
            if (warp == 4 && lane == 0) TL((int)tcount, 11);  // X' written
        }
    } else if (warp >= 8) {  // ================= epilogue 3: acc3 (+bias) -> Y
        const int q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const bool vec = (g.N & 3) == 0;
        Ring a3(g.nbuf3);
        int it = 0;
        for (int tile = blockIdx.x; tile < g.num_tiles; tile += gridDim.x, ++it) {
            const int b = tile / g.tiles_per_img;
            const int oy0 = (tile % g.tiles_per_img) * g.R;
            const int m = q * 32 + lane;
            const int oy = oy0 + m / g.Wq, ox = m % g.Wq;
            const bool valid = m < g.R * g.Wq && oy < g.Ho && ox < g.Wo;
            float *dst = g.y + (((long long)b * g.Ho + oy) * g.Wo + ox) * g.N;
            for (int h = 0; h < g.nhalves; ++h, a3.next()) {
                const uint32_t ab = a3.slot;
                mbar_wait(&acc3_full[ab], a3.phase);
                tc_fence_after();
                if (warp == 8 && lane == 0 && h == 0) TL(it, 12);  // acc3 full seen
                const uint32_t acc3 = tmem + lane_base + g.acc3_col + ab * g.P3 * g.Nh;
                float *scratch = epi_scratch + q * 1024;
                for (int c = 0; c < g.Nh; c += 32) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(acc3 + c, r);
                    tmem_ld_wait();
                    for (int pp = 1; pp < g.P3; ++pp) {
                        uint32_t r2[32];
                        tmem_ld_32x32b_x32(acc3 + pp * g.Nh + c, r2);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            r[j] = __float_as_uint(__uint_as_float(r[j]) + __uint_as_float(r2[j]));
                    }
                    const int n = h * g.Nh + c;
                    if (n >= g.N) continue;  // warp-uniform
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        v[j] = __uint_as_float(r[j]) + (g.bias && n + j < g.N ? __ldg(g.bias + n + j) : 0.f);
                    if (vec && n + 32 <= g.N) {  // coalesced through shared memory
                        warp_store_block32(scratch, v, valid ? dst + n : nullptr, lane);
                    } else if (valid) {
                        _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n + j < g.N) dst[n + j] = v[j];
                    }
                }
                tc_fence_before();
                mbar_arrive_relaxed(&acc3_empty[ab]);
            }
            if (warp == 8 && lane == 0) TL(it, 13);  // Y stored
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, (uint32_t)g.tmem_cols);
}

// 4-D NHWC view (C, W, H, B) of x, box {32, Wp, Rin, 1}, 128-byte swizzle.
bool fused_make_x_map(CUtensorMap *map, const float *x, const FusedArgs &g) {
    return make_tma_4d_nhwc(map, x, g.C, g.W, g.H, g.B, g.Wp, g.Rin);
}

#ifdef TDC_TIMELINE
extern "C" int tdc_debug_timeline(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_timeline, sizeof(unsigned long long) * n);
}
#endif

cudaError_t fused_launch(const CUtensorMap &mapX, const FusedArgs &g, int grid,
                         cudaStream_t st) {
    const int smem = fused_smem_bytes(g);
    cudaError_t e = cudaFuncSetAttribute(tdc_tkd_fused_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(tdc_tkd_fused_tc_kernel, grid, kFusedThreads, smem, st, mapX, g);
}

}  // namespace tdc
