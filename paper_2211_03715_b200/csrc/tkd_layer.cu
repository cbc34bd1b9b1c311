// tkd_layer.cu -- the whole 3xBF16 TKD layer in ONE
// persistent tcgen05 kernel: HBM sees X once, Y once and the weights once; the
// intermediates X' (stage 1 -> 2) and Z (stage 2 -> 3) never leave the SM.
//
// Work unit ("tile"): R output rows of one image (M = R*Wq <= 128 accumulator rows,
// output position m = yo*Wq + xo).  A CTA walks a contiguous range of tiles, so
// consecutive tiles of an image share all but R of their core-input rows: the X'
// band is a ring of phase rows in shared memory and each tile computes stage 1
// only for its R new rows (plus the K-1 halo rows where a CTA starts or an image
// begins) -- the paper's "input tile loaded once into shared memory"
// carried across tiles.
//
//   stage 1 (a1)  acc1[px][a] = sum_c X[px][c] U_in[c][a] on blocks of rpb padded
//                 input rows x Wp columns, TMA-loaded (4-D NHWC box, out-of-bounds
//                 zero fill = the zero padding, reading R6) as fp32 and split in
//                 place into bf16 hi/lo by the converter warps; B = [U_in hi | lo]
//                 so one N = 2*D1 MMA gives hi*hi and hi*lo, one N = D1 MMA lo*hi.
//   epilogue 1    acc1 -> X' = hi-part + lo-part -> bf16 hi/lo -> the band ring
//                 (no-swizzle K-major planes [plane][row][16 B]); a ring row also
//                 written at its mirror position + NR when < R+e, so every
//                 tile's window of R+e+1 rows is contiguous (one descriptor).
//   stage 2 (a2)  acc2[m][q] = sum_{tap,a} X'[m + off(tap)][a] core[q][a][tap]:
//                 each tap a row-shifted descriptor of the band.
//   epilogue 2    acc2 -> Z hi/lo bf16 -> shared memory.
//   stage 3 (a3)  acc3[m][n] = sum_q Z[m][q] U_out[n][q] (+bias, +residual, ReLU).
//   epilogue 3    acc3 -> Y (NHWC), every output element written once, no atomics
//                 (contrast P:L368-372).
//
// Band ring: NR = 2R + e phase rows (e = (K-1)/s).  Tile t's window starts at ring
// row start(t) = start(t-1) + R (mod NR).  A regular tile writes R new rows into the
// ring rows tile t-2 used (E1 waits for S2(t-2)); a tile that starts an image writes
// R+e rows, the first e of which tile t-1 still reads (E1 waits for S2(t-1)).  The
// row after a window (its "guard") is read only by the junk columns/rows of the
// tile, so the next tile may overwrite it while the MMAs run.
//
// Warp roles (20 warps, one CTA per SM):
//   0 producer (weights once, then X blocks by TMA)   1 MMA issue of the core (stage 2)
//   2-5 epilogue 1   6-9 epilogue 2   10-13 epilogue 3   14-17 converters
//   18 / 19 MMA issue of stage 1 / stage 3 -- one issuing thread per stage, so no stage's
//   hand-off waits ever hold back another stage's MMAs
#include <cuda.h>
#include <cuda_bf16.h>

#include "internal.h"
#include "sm100.cuh"
#include "tkd_common.cuh"

namespace tdc {

using namespace sm100;

#ifdef TDC_TIMELINE
// Debug build only: %globaltimer stamps of pipeline events of one CTA (g_tdc_ltl_cta), per
// local tile (< 32) -- read by scripts/layer_timeline.py.
__device__ unsigned long long g_tdc_ltl[32 * 24];
__device__ int g_tdc_ltl_cta;
__device__ __forceinline__ void ltl(bool on, int t, int ev) {
    if (on && t < 32) {
        unsigned long long v;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
        g_tdc_ltl[t * 24 + ev] = v;
    }
}
extern "C" int tdc_debug_layer_timeline(unsigned long long *host, int n, int cta) {
    cudaMemcpyToSymbol(g_tdc_ltl_cta, &cta, sizeof(int));
    return (int)cudaMemcpyFromSymbol(host, g_tdc_ltl, sizeof(unsigned long long) * n);
}
#define LTL(t, ev) ltl(tl_on, (t), (ev))
#else
#define LTL(t, ev) ((void)0)
#endif

#if defined(TDC_DEBUG_KNOBS) || defined(TDC_TIMELINE)
#define LKNOB(bit) (g.knobs & (bit))
#else
#define LKNOB(bit) 0
#endif

constexpr int kLayerThreads = 640;  // 20 warps
constexpr int kS1Warp = 18;         // stage-1 MMA issue
constexpr int kS3Warp = 19;         // stage-3 MMA issue
#if defined(TDC_DEBUG_KNOBS) || defined(TDC_TIMELINE)
#define S3_FIRST LKNOB(512)
#else
#define S3_FIRST 0
#endif

// Epilogue-side waits.  Debug knob 256 swaps the suspend-hint wait for the plain one.
#if defined(TDC_DEBUG_KNOBS) || defined(TDC_TIMELINE)
#define ewait(bar, par) (LKNOB(256) ? mbar_wait((bar), (par)) : mbar_wait_sleep((bar), (par)))
#else
#define ewait(bar, par) mbar_wait_sleep((bar), (par))
#endif
constexpr uint32_t kEpiScr = 4 * 4096;

struct LayerSmem {
    uint32_t xs, w1, w2, w3, band, z, scr, xch, bars, total;
};

__host__ __device__ inline LayerSmem layer_smem(const BfLayerArgs &g) {
    LayerSmem s;
    uint32_t o = 0;
    s.xs = o;   o += (uint32_t)g.XS * 2 * g.XR * 128;
    s.w1 = o;   o += (uint32_t)g.cchunks * 2 * g.D1s * 128;
    s.w2 = o;   o += (uint32_t)(g.D1s / 32) * g.KK * 4 * 2 * g.D2s * 16;
    s.w3 = o;   o += (uint32_t)(g.D2s / 8) * 2 * g.N3p * 16;
    s.band = o; o += 2u * (g.D1s / 8) * g.NRB * g.Wq * 16;
    s.z = o;    o += g.xt ? 0u : 2u * 2u * (g.D2s / 8) * g.ZR * 16;  // two Z buffers (hi | lo each)
    s.scr = o;  o += kEpiScr;
    s.xch = o;  o += g.tn ? 2 * 4 * 16 * 4 : 0;  // TN: epilogue-2 row exchange
    s.bars = o; o += 64 * 8 + 16;
    s.total = o + 1024;  // + alignment slack of the dynamic shared memory base
    return s;
}
int bf_layer_smem_bytes(const BfLayerArgs &g) { return (int)layer_smem(g).total; }

struct TileGeo {
    int b, j, ylo, yhi, nb;
    bool fresh;
    int x0;  // first output column of the tile's strip (variant 5b; 0 elsewhere)
};
// Tile k of the CTA whose range starts at k0: image b, row block j, the new band
// (phase) rows [ylo, yhi) it computes, and the number of stage-1 blocks.  s = 1.
__device__ __forceinline__ TileGeo tile_geo(const BfLayerArgs &g, int k, int k0) {
    TileGeo t;
    t.b = k / g.T;
    t.j = k - t.b * g.T;
    t.fresh = (t.j == 0) || (k == k0);
    t.ylo = t.fresh ? t.j * g.R : t.j * g.R + g.e;
    t.yhi = t.j * g.R + g.R + g.e;
    t.nb = (t.yhi - t.ylo + g.rpb - 1) / g.rpb;
    t.x0 = 0;
    return t;
}

// KT: core size K at compile time (3), or 0 = any K.  TN ("tap pairs along N", K = 3,
// D2 = 32): taps (r,0) and (r,1) of a core row share one A operand -- B = [C(r,0) lo | hi |
// C(r,1) hi | lo], N = 4*D2 -- and tap (r,2) is the row-shifted A of the same accumulator
// block 0, so stage 2 issues 24 MMAs per tile instead of 36 (and a quarter fewer band
// re-reads); tap (r,1)'s accumulator block is shifted by one row in epilogue 2
// (Z[m] = blk0[m] + blk1[m + 1]: a lane shuffle plus one row exchanged between the
// epilogue warps).  Stage 3 then drops its hi|lo concatenation so every accumulator
// stays double-buffered in the 512 TMEM columns.
template <int KT, bool TN>
__global__ void __launch_bounds__(kLayerThreads, 1)
tdc_bf_layer_kernel(const __grid_constant__ CUtensorMap mapX, const BfLayerArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const LayerSmem L = layer_smem(g);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *x_full = bars, *x_empty = bars + 4, *conv = bars + 8;   // XS <= 4
    uint64_t *w_full = bars + 12;
    uint64_t *a1_full = bars + 13, *a1_empty = bars + 15;
    uint64_t *band_ready = bars + 17, *band_free = bars + 19;
    uint64_t *a2_full = bars + 21, *a2_empty = bars + 23;
    uint64_t *z_full = bars + 25, *z_empty = bars + 27;
    uint64_t *a3_full = bars + 29, *a3_empty = bars + 31;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 40);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef TDC_TIMELINE
    const bool tl_on = (int)blockIdx.x == *(volatile int *)&g_tdc_ltl_cta;  // read once
    if (threadIdx.x == 0) LTL(0, 21);  // kernel entry
#endif
    if (threadIdx.x == 0) {
        for (int i = 0; i < g.XS; ++i) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_empty[i], 1);
            mbar_init(&conv[i], 128);
        }
        mbar_init(w_full, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a1_full[i], 1);
            mbar_init(&a1_empty[i], 128);
            mbar_init(&band_ready[i], 128);
            mbar_init(&band_free[i], 1);
            mbar_init(&a2_full[i], 1);
            mbar_init(&a2_empty[i], 128);
            mbar_init(&a3_full[i], 1);
            mbar_init(&a3_empty[i], 128);
            mbar_init(&z_full[i], 128);
            mbar_init(&z_empty[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) tma_prefetch(&mapX);
    if (warp == 1) tmem_alloc(tmem_slot, (uint32_t)g.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) LTL(0, 22);  // setup done (barriers, TMEM)

    // contiguous tile range of this CTA (sliding band within it)
    const int k0 = (int)((long long)blockIdx.x * g.num_tiles / gridDim.x);
    const int k1 = (int)((long long)(blockIdx.x + 1) * g.num_tiles / gridDim.x);
    const int nt = k1 - k0;
    // TN: acc2 is 4*D2s wide (two tap blocks x [hi part | lo part]); stage 3 then skips the hi|lo
    // concatenation (3 MMAs into N3p columns instead of 2 into 2*N3p) to stay within 512 columns
    constexpr int NA1 = 2, NA2 = 2;     // acc1 / acc2 buffers
    const bool s3cat = !TN && g.ncat3;  // stage 3 with [hi | lo] U_out along N (2 MMAs, 2*N3p columns)
    const uint32_t acc1_cols = 2 * g.D1s, acc2_cols = (TN ? 4 : 2) * g.D2s, acc3_cols = (s3cat ? 2 : 1) * g.N3p;
    const uint32_t acc2_base = NA1 * acc1_cols, acc3_base = acc2_base + NA2 * acc2_cols;
    const uint32_t plane_stride = (uint32_t)g.NRB * g.Wq * 16;   // bytes between band planes
    const uint32_t band_half = (uint32_t)(g.D1s / 8) * plane_stride;  // hi -> lo
    const uint32_t zhalf = (uint32_t)(g.D2s / 8) * g.ZR * 16;      // Z hi -> lo
    const uint32_t xslot = 2u * g.XR * 128, xhalf = (uint32_t)g.XR * 128;  // X slot; hi -> lo tile

    if (warp == 0) {  // =============================================== producer
        const int w1b = (int)(L.w2 - L.w1), w2b = (int)(L.w3 - L.w2), w3b = (int)(L.band - L.w3);
        auto load_split = [&](uint8_t *dst, const void *src, uint32_t bytes) {
            const uint32_t piece = 16384;
            for (uint32_t o = (uint32_t)lane * piece; o < bytes; o += 32 * piece)
                bulk_load(dst + o, reinterpret_cast<const uint8_t *>(src) + o, bytes - o < piece ? bytes - o : piece,
                          w_full);
        };
        if (lane == 0) mbar_arrive_expect_tx(w_full, (uint32_t)(w1b + w2b + w3b));
        __syncwarp();
        load_split(smem + L.w1, g.w1, w1b);
        load_split(smem + L.w2, g.w2, w2b);
        load_split(smem + L.w3, g.w3, w3b);
        __syncwarp();
        pdl_wait();  // X may be written by the previous kernel in the stream
        const uint32_t box_bytes = (uint32_t)g.rpb * g.Wp * 128;
        // L2 prefetch cursor kPF blocks ahead of the loads: the staging ring holds only XS
        // blocks, too few to cover HBM latency at full bandwidth, so the loads should hit L2
        int pk = k0, pblk = 0;
        auto prefetch_next = [&]() {
            if (pk >= k1) return;
            const TileGeo pg = tile_geo(g, pk, k0);
            if (lane == 0)
                for (int cc = 0; cc < g.cchunks; ++cc) {
                    tma_prefetch_l2_4d(&mapX, cc * 64, -g.p, pg.ylo + pblk * g.rpb - g.p, pg.b);
                    tma_prefetch_l2_4d(&mapX, cc * 64 + 32, -g.p, pg.ylo + pblk * g.rpb - g.p, pg.b);
                }
            if (++pblk == pg.nb) {
                pblk = 0;
                ++pk;
            }
        };
        for (int i = 0; i < g.pf_blocks; ++i) prefetch_next();
        Ring xr(g.XS);
        for (int k = k0; k < k1; ++k) {
            const TileGeo tg = tile_geo(g, k, k0);
            for (int blk = 0; blk < tg.nb; ++blk) {
                const int u0 = tg.ylo + blk * g.rpb;  // padded row (s = 1: = phase row)
                prefetch_next();
                for (int cc = 0; cc < g.cchunks; ++cc, xr.next()) {
                    mbar_wait(&x_empty[xr.slot], xr.phase ^ 1);
                    if (lane == 0 && blk == 0 && cc == 0) LTL(k - k0, 0);  // producer: X load issued
                    if (LKNOB(128) && (k > k0 + 1)) {  // debug: no X traffic after the first tiles
                        if (elect_one()) mbar_arrive(&x_full[xr.slot]);
                        __syncwarp();
                        continue;
                    }
                    if (elect_one()) {
                        uint8_t *dst = smem + L.xs + (size_t)xr.slot * xslot;
                        mbar_arrive_expect_tx(&x_full[xr.slot], 2 * box_bytes);
                        tma_load_4d(dst, &mapX, &x_full[xr.slot], cc * 64, -g.p, u0 - g.p, tg.b);
                        tma_load_4d(dst + xhalf, &mapX, &x_full[xr.slot], cc * 64 + 32, -g.p, u0 - g.p, tg.b);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1 || warp == kS1Warp || warp == kS3Warp) {  // ============== MMA issue
        const uint32_t id1 = idesc_bf16(128, 2 * g.D1s), id1h = idesc_bf16(128, g.D1s);
        const uint32_t id2 = idesc_bf16(128, 2 * g.D2s), id2h = idesc_bf16(128, g.D2s);
        const uint32_t id3 = idesc_bf16(128, 2 * g.N3p), id3h = idesc_bf16(128, g.N3p);
        const uint64_t dx = sdesc_kmajor_sw128(smem_u32(smem + L.xs));
        const uint64_t dw1 = sdesc_kmajor_sw128(smem_u32(smem + L.w1));
        const uint64_t dband = sdesc_kmajor_none(smem_u32(smem + L.band), plane_stride, 128);
        const uint64_t dw2 = sdesc_kmajor_none(smem_u32(smem + L.w2), 2 * g.D2s * 16, 128);
        const uint64_t dw2tn = sdesc_kmajor_none(smem_u32(smem + L.w2), 6 * g.D2s * 16, 128);
        const uint32_t id2tn = idesc_bf16(128, 4 * g.D2s), id2tnh = idesc_bf16(128, 2 * g.D2s);
        const uint64_t dz = sdesc_kmajor_none(smem_u32(smem + L.z), g.ZR * 16, 128);
        const uint64_t dw3 = sdesc_kmajor_none(smem_u32(smem + L.w3), 2 * g.N3p * 16, 128);
        const uint32_t w1_chunk = (uint32_t)2 * g.D1s * 128;
        const uint32_t w2_tap = (uint32_t)4 * 2 * g.D2s * 16, w2_plane2 = (uint32_t)2 * 2 * g.D2s * 16;
        const uint32_t w3_plane2 = (uint32_t)2 * 2 * g.N3p * 16;
        const int kc2 = g.D1s / 32, k3 = g.D2s / 16;
        Ring xr(g.XS);
        uint32_t ublk = 0;  // stage-1 block counter (acc1 buffer = ublk & 1)
        mbar_wait(w_full, 0);
        if (warp == kS1Warp && lane == 0) LTL(0, 23);  // weights landed
        int s1_tile = 0;  // (timeline) local tile of the next stage-1 block
        auto s1_block = [&]() {
            const uint32_t ab = NA1 == 1 ? 0u : (ublk & 1), aph = NA1 == 1 ? (ublk & 1) : ((ublk >> 1) & 1);
            if (lane == 0) LTL(s1_tile, 13);  // MMA: S1 block start
            mbar_wait(&a1_empty[ab], aph ^ 1);
            tc_fence_after();
            if (lane == 0) LTL(s1_tile, 14);  // MMA: S1 acc1 free
            const uint32_t d = tmem + ab * acc1_cols;
            for (int cc = 0; cc < g.cchunks; ++cc, xr.next()) {
                mbar_wait(&conv[xr.slot], xr.phase);
                tc_fence_after();
                if (lane == 0) LTL(s1_tile, 15);  // MMA: S1 X converted
                if (elect_one()) {
                    const uint64_t a = dx + ((xr.slot * xslot) >> 4);
                    const uint64_t b = dw1 + ((cc * w1_chunk) >> 4);
#pragma unroll
                    for (int j = 0; j < (LKNOB(32) ? 0 : 4); ++j) {  // K = 16 bf16 = 32 B per MMA
                        mma_bf16(d, a + j * 2, b + j * 2, id1, (cc > 0) || (j > 0));   // hi * [hi | lo]
                        mma_bf16(d, a + (xhalf >> 4) + j * 2, b + j * 2, id1h, 1);  // lo * hi
                    }
                    mma_commit(&x_empty[xr.slot]);
                }
                __syncwarp();
            }
            if (elect_one()) mma_commit(&a1_full[ab]);
            __syncwarp();
            ++ublk;
            if (lane == 0) LTL(s1_tile, 2);  // MMA: S1 block issued
        };
        auto s2 = [&](int t, uint32_t start) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;                       // band ring
            const uint32_t ab2 = NA2 == 1 ? 0u : sb, aph2 = NA2 == 1 ? (t & 1) : sph;  // acc2
            mbar_wait(&band_ready[sb], sph);
            mbar_wait(&a2_empty[ab2], aph2 ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc2_base + ab2 * acc2_cols;
            const uint64_t arow = dband + start * (uint32_t)g.Wq;  // 16-byte units
            if (TN) {
                const uint32_t wq = (uint32_t)g.Wq, p2a = (2 * plane_stride) >> 4, lo_a = band_half >> 4;
                const uint32_t wr = (4 * 6 * g.D2s * 16) >> 4, p2b = (2 * 6 * g.D2s * 16) >> 4;  // per row r / K16
                const uint32_t rows16 = ((uint32_t)g.D2s * 16) >> 4;  // one D2s-row group of B
                for (int kc = 0; kc < (LKNOB(16) ? 0 : kc2); ++kc) {
                    const uint64_t ak = arow + (uint32_t)kc * ((4 * plane_stride) >> 4);
                    const uint64_t bk = dw2tn + (uint32_t)kc * 3 * wr;
                    if (elect_one()) {
#pragma unroll
                        for (int r = 0; r < 3; ++r)
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                const uint64_t aj = ak + r * wq + j * p2a, bj = bk + r * wr + j * p2b;
                                // taps (r,0),(r,1): hi x [C0 lo | C0 hi | C1 hi | C1 lo] -> cols [0, 4*D2)
                                mma_bf16(d, aj, bj, id2tn, (kc > 0) || r || j);
                                // lo x [C0 hi | C1 hi] -> cols [D2, 3*D2) (block 0 group 1, block 1 group 0)
                                mma_bf16(d + g.D2s, aj + lo_a, bj + rows16, id2tnh, 1);
                                // tap (r,2): A shifted by 2 rows, into block 0: hi x [C2 hi | C2 lo], lo x C2 hi
                                mma_bf16(d, aj + 2, bj + 4 * rows16, id2, 1);
                                mma_bf16(d, aj + 2 + lo_a, bj + 4 * rows16, id2h, 1);
                            }
                    }
                    __syncwarp();
                }
                if (elect_one()) {
                    mma_commit(&band_free[sb]);
                    mma_commit(&a2_full[ab2]);
                }
            } else if (KT > 0) {
                // compile-time taps: every descriptor is the converged, warp-uniform row base
                // plus r*Wq + t (16-byte rows), so the MMAs issue back to back from uniform
                // registers instead of each waiting on a parameter load + R2UR chain
                const uint32_t wq = (uint32_t)g.Wq, p2a = (2 * plane_stride) >> 4, lo_a = band_half >> 4;
                const uint32_t wt = w2_tap >> 4, p2b = w2_plane2 >> 4;
                for (int kc = 0; kc < (LKNOB(16) ? 0 : kc2); ++kc) {
                    const uint64_t ak = arow + (uint32_t)kc * ((4 * plane_stride) >> 4);
                    const uint64_t bk = dw2 + (uint32_t)kc * (KT * KT) * wt;
                    if (elect_one()) {
#pragma unroll
                        for (int r = 0; r < KT; ++r)
#pragma unroll
                            for (int tt = 0; tt < KT; ++tt)
#pragma unroll
                                for (int j = 0; j < 2; ++j) {
                                    const uint64_t aj = ak + r * wq + tt + j * p2a;
                                    const uint64_t bj = bk + (r * KT + tt) * wt + j * p2b;
                                    mma_bf16(d, aj, bj, id2, (kc > 0) || r || tt || j);  // hi * [hi | lo]
                                    mma_bf16(d, aj + lo_a, bj, id2h, 1);                  // lo * hi
                                }
                    }
                    __syncwarp();
                }
                if (elect_one()) {
                    mma_commit(&band_free[sb]);
                    mma_commit(&a2_full[ab2]);
                }
            } else if (elect_one()) {
                uint32_t acc = 0;
                for (int kc = 0; kc < kc2; ++kc)
#pragma unroll 1
                    for (int tap = 0; tap < g.KK; ++tap) {
                        const uint64_t a = arow + (((uint32_t)(kc * 4) * plane_stride + (uint32_t)g.tap_off[tap] * 16) >> 4);
                        const uint64_t b = dw2 + (((uint32_t)(kc * g.KK + tap) * w2_tap) >> 4);
#pragma unroll
                        for (int j = 0; j < 2; ++j) {  // K = 16 = two 8-channel planes
                            const uint64_t aj = a + ((j * 2 * plane_stride) >> 4), bj = b + ((j * w2_plane2) >> 4);
                            mma_bf16(d, aj, bj, id2, acc);                      // hi * [hi | lo]
                            mma_bf16(d, aj + (band_half >> 4), bj, id2h, 1);    // lo * hi
                            acc = 1;
                        }
                    }
                mma_commit(&band_free[sb]);
                mma_commit(&a2_full[ab2]);
            }
            __syncwarp();
        };
        auto s3 = [&](int t) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            mbar_wait(&z_full[sb], sph);
            mbar_wait(&a3_empty[sb], sph ^ 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t d = tmem + acc3_base + sb * acc3_cols;
                const uint64_t zs = dz + ((sb * 2 * zhalf) >> 4);
                for (int j = 0; j < (LKNOB(64) ? 0 : k3); ++j) {
                    const uint64_t a = zs + ((j * 2 * g.ZR * 16) >> 4), b = dw3 + ((j * w3_plane2) >> 4);
                    if (!s3cat) {  // hi*hi, hi*lo, lo*hi into the same N3p columns (half the TMEM reads)
                        mma_bf16(d, a, b, id3h, j > 0);
                        mma_bf16(d, a, b + ((g.N3p * 16) >> 4), id3h, 1);
                        mma_bf16(d, a + (zhalf >> 4), b, id3h, 1);
                    } else {
                        mma_bf16(d, a, b, id3, j > 0);
                        mma_bf16(d, a + (zhalf >> 4), b, id3h, 1);
                    }
                }
                mma_commit(&z_empty[sb]);
                mma_commit(&a3_full[sb]);
            }
            __syncwarp();
        };
        if (warp == 1) {  // the core stream: S2(t) as soon as its band is ready
            uint32_t start = 0;
            for (int t = 0; t < nt; ++t) {
                if (lane == 0) LTL(t, 11);  // MMA: S2(t) about to wait
                s2(t, start);
                if (lane == 0) LTL(t, 3);   // MMA: S2(t) issued
                start += g.R;
                if (start >= (uint32_t)g.NR) start -= g.NR;
            }
        } else if (warp == kS1Warp) {  // stage 1 runs ahead (2 acc1 buffers), never behind stage 3
            for (int t = 0; t < nt; ++t) {
                s1_tile = t;
                const int nb = tile_geo(g, k0 + t, k0).nb;
                for (int blk = 0; blk < nb; ++blk) s1_block();
            }
        } else {  // stage 3: waits only for epilogue 2's Z
            for (int t = 0; t < nt; ++t) {
                s3(t);
                if (lane == 0) LTL(t, 4);  // MMA: S3 issued
            }
        }
    } else if (warp < 6) {  // ========================= epilogue 1: acc1 -> X' band ring
        const int q = warp & 3;  // TMEM lane quarter this warp may access = warp % 4
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t bandA = smem_u32(smem + L.band);
        const int i = q * 32 + lane;  // block row = TMEM lane
        const int yy = i / g.Wp, xx = i - yy * g.Wp;
        uint32_t ublk = 0;
        int start = 0;
        for (int t = 0; t < nt; ++t) {
            const TileGeo tg = tile_geo(g, k0 + t, k0);
            for (int blk = 0; blk < tg.nb; ++blk, ++ublk) {
                const uint32_t ab = NA1 == 1 ? 0u : (ublk & 1), aph = NA1 == 1 ? (ublk & 1) : ((ublk >> 1) & 1);
                if (blk == 0 && t > 0) {  // ring rows about to be overwritten are no longer read
                    const int tw = tg.fresh ? t - 1 : t - 2;
                    if (tw >= 0) ewait(&band_free[tw & 1], (tw >> 1) & 1);
                }
                ewait(&a1_full[ab], aph);
                tc_fence_after();
                if (threadIdx.x == 64 && blk == 0) LTL(t, 5);  // E1: acc1 full seen
                const int y = tg.ylo + blk * g.rpb + yy;  // phase (= padded) row of this lane's pixel
                const bool valid = i < g.rpb * g.Wp && y < tg.yhi;
                int slot = start + (y - tg.j * g.R);
                if (slot >= g.NR) slot -= g.NR;
                const bool mirror = slot < g.NRB - g.NR;
                const uint32_t pos = (uint32_t)(slot * g.Wq + xx) * 16;
                const uint32_t pos2 = pos + (uint32_t)g.NR * g.Wq * 16;
                for (int c = 0; c < g.D1s; c += 16) {
                    uint32_t r0[16], r1[16];
                    tmem_ld_32x32b_x16(tmem + lane_base + ab * acc1_cols + c, r0);
                    tmem_ld_32x32b_x16(tmem + lane_base + ab * acc1_cols + g.D1s + c, r1);
                    tmem_ld_wait();
                    if (!valid || LKNOB(4)) continue;
                    float v[16];
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
#pragma unroll
                    for (int pl = 0; pl < 2; ++pl) {
                        uint4 h, l;
                        split_bf16x8(v + 8 * pl, h, l);
                        const uint32_t po = (uint32_t)(c / 8 + pl) * plane_stride;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + po + pos), "r"(h.x),
                                     "r"(h.y), "r"(h.z), "r"(h.w) : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + band_half + po + pos),
                                     "r"(l.x), "r"(l.y), "r"(l.z), "r"(l.w) : "memory");
                        if (mirror) {
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + po + pos2), "r"(h.x),
                                         "r"(h.y), "r"(h.z), "r"(h.w) : "memory");
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + band_half + po + pos2),
                                         "r"(l.x), "r"(l.y), "r"(l.z), "r"(l.w) : "memory");
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive_relaxed(&a1_empty[ab]);
            }
            fence_proxy_async_smem();  // X' (generic writes) -> visible to the MMAs (async proxy)
            mbar_arrive(&band_ready[t & 1]);
            if (threadIdx.x == 64) LTL(t, 6);  // E1: band ready
            start += g.R;
            if (start >= g.NR) start -= g.NR;
        }
    } else if (warp < 10) {  // ======================= epilogue 2: acc2 -> Z hi/lo (smem)
        const int q = warp & 3;  // TMEM lane quarter this warp may access = warp % 4
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const int r = q * 32 + lane;
        const bool zrow = r < g.ZR;  // Z planes hold ZR rows (rows beyond: junk MMA rows)
        float *xbuf = reinterpret_cast<float *>(smem + L.xch);  // TN: [chunk 2][quarter 4][16]
        for (int t = 0; t < nt; ++t) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            const uint32_t ab2 = NA2 == 1 ? 0u : sb, aph2 = NA2 == 1 ? (t & 1) : sph;
            const uint32_t zb = smem_u32(smem + L.z) + sb * 2 * zhalf;
            ewait(&a2_full[ab2], aph2);
            tc_fence_after();
            if (threadIdx.x == 192) LTL(t, 7);  // E2: acc2 full seen
            if (TN) {  // Z[m] = blk0[m] + blk1[m + 1], each block = group 0 + group 1 (D2s = 32)
                const uint32_t a2 = tmem + lane_base + acc2_base + ab2 * acc2_cols;
                uint4 h0[4], l0[4];
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    const int c = ch * 16;
                    float p0[16], p1[16];
                    {
                        uint32_t r0[16], r1[16], r2[16], r3[16];
                        tmem_ld_32x32b_x16(a2 + c, r0);
                        tmem_ld_32x32b_x16(a2 + g.D2s + c, r1);
                        tmem_ld_32x32b_x16(a2 + 2 * g.D2s + c, r2);
                        tmem_ld_32x32b_x16(a2 + 3 * g.D2s + c, r3);
                        tmem_ld_wait();
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) {
                            p0[jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
                            p1[jj] = __uint_as_float(r2[jj]) + __uint_as_float(r3[jj]);
                        }
                    }
                    if (ch == 1) {  // every TMEM read of this tile done: S2(t+2) may overwrite acc2
                        tc_fence_before();
                        mbar_arrive_relaxed(&a2_empty[ab2]);
                    }
                    // row m+1 of lane 31 lives in the next lane quarter (lane 0): exchange it
                    float *mine = xbuf + (ch * 4 + q) * 16, *next = xbuf + (ch * 4 + ((q + 1) & 3)) * 16;
                    if (lane == 0)
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) mine[jj] = p1[jj];
                    asm volatile("bar.sync 3, 128;" ::: "memory");
                    float v[16];
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        float s1 = __shfl_down_sync(0xffffffffu, p1[jj], 1);
                        if (lane == 31) s1 = next[jj];
                        v[jj] = p0[jj] + s1;
                    }
                    split_bf16x8(v, h0[2 * ch], l0[2 * ch]);
                    split_bf16x8(v + 8, h0[2 * ch + 1], l0[2 * ch + 1]);
                }
                ewait(&z_empty[sb], sph ^ 1);  // S3 two tiles back has read this Z buffer
                if (!LKNOB(8) && zrow)
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) {
                        const uint32_t o = ((uint32_t)pl * g.ZR + r) * 16;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + o), "r"(h0[pl].x),
                                     "r"(h0[pl].y), "r"(h0[pl].z), "r"(h0[pl].w) : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + zhalf + o), "r"(l0[pl].x),
                                     "r"(l0[pl].y), "r"(l0[pl].z), "r"(l0[pl].w) : "memory");
                    }
                fence_proxy_async_smem();
                mbar_arrive(&z_full[sb]);
                if (threadIdx.x == 192) LTL(t, 8);
                continue;
            }
            // the first 32 columns are read and split before waiting for the Z buffer, so the
            // S3(t-1) -> E2(t) -> S3(t) hand-off carries only the shared-memory stores
            uint4 h0[4], l0[4];
#pragma unroll
            for (int c = 0; c < 32; c += 16) {
                uint32_t r0[16], r1[16];
                tmem_ld_32x32b_x16(tmem + lane_base + acc2_base + ab2 * acc2_cols + c, r0);
                tmem_ld_32x32b_x16(tmem + lane_base + acc2_base + ab2 * acc2_cols + g.D2s + c, r1);
                tmem_ld_wait();
                float v[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
                split_bf16x8(v, h0[c / 8], l0[c / 8]);
                split_bf16x8(v + 8, h0[c / 8 + 1], l0[c / 8 + 1]);
            }
            ewait(&z_empty[sb], sph ^ 1);  // S3 two tiles back has read this Z buffer
            if (threadIdx.x == 192) LTL(t, 12);  // E2: Z buffer free
            if (!LKNOB(8) && zrow)
#pragma unroll
                for (int pl = 0; pl < 4; ++pl) {
                    const uint32_t o = ((uint32_t)pl * g.ZR + r) * 16;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + o), "r"(h0[pl].x),
                                 "r"(h0[pl].y), "r"(h0[pl].z), "r"(h0[pl].w) : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + zhalf + o), "r"(l0[pl].x),
                                 "r"(l0[pl].y), "r"(l0[pl].z), "r"(l0[pl].w) : "memory");
                }
            for (int c = 32; c < g.D2s; c += 16) {
                uint32_t r0[16], r1[16];
                tmem_ld_32x32b_x16(tmem + lane_base + acc2_base + ab2 * acc2_cols + c, r0);
                tmem_ld_32x32b_x16(tmem + lane_base + acc2_base + ab2 * acc2_cols + g.D2s + c, r1);
                tmem_ld_wait();
                float v[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
                if (LKNOB(8) || !zrow) continue;
#pragma unroll
                for (int pl = 0; pl < 2; ++pl) {  // Z planes [c/8 + pl][row r][16 B]: lanes = rows, no conflicts
                    uint4 h, l;
                    split_bf16x8(v + 8 * pl, h, l);
                    const uint32_t o = ((uint32_t)(c / 8 + pl) * g.ZR + r) * 16;
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + o), "r"(h.x), "r"(h.y),
                                 "r"(h.z), "r"(h.w) : "memory");
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + zhalf + o), "r"(l.x),
                                 "r"(l.y), "r"(l.z), "r"(l.w) : "memory");
                }
            }
            tc_fence_before();
            mbar_arrive_relaxed(&a2_empty[ab2]);
            fence_proxy_async_smem();
            mbar_arrive(&z_full[sb]);
            if (threadIdx.x == 192) LTL(t, 8);  // E2: Z written
        }
    } else if (warp < 14) {  // ======================= epilogue 3: acc3 (+bias, res, relu) -> Y
        const int q = warp & 3;  // TMEM lane quarter this warp may access = warp % 4
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        float *scratch = reinterpret_cast<float *>(smem + L.scr) + q * 1024;
        const int m = q * 32 + lane;
        const int yo = m / g.Wq, xo = m - yo * g.Wq;
        const bool vec = (g.N & 3) == 0;
        for (int t = 0; t < nt; ++t) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            const int k = k0 + t, b = k / g.T, j = k - b * g.T;
            const int oy = j * g.R + yo;
            const bool valid = yo < g.R && oy < g.Ho && xo < g.Wo;
            const long long orow = ((long long)b * g.Ho + oy) * g.Wo + xo;
            float *dst = g.y + orow * g.N;
            ewait(&a3_full[sb], sph);
            tc_fence_after();
            if (threadIdx.x == 320) LTL(t, 9);  // E3: acc3 full seen
            for (int c = 0; c < g.N3p; c += 32) {
                float v[32];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    uint32_t r0[16], r1[16];
                    tmem_ld_32x32b_x16(tmem + lane_base + acc3_base + sb * acc3_cols + c + 16 * hh, r0);
                    if (s3cat) tmem_ld_32x32b_x16(tmem + lane_base + acc3_base + sb * acc3_cols + g.N3p + c + 16 * hh, r1);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj)
                        v[16 * hh + jj] = s3cat ? __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]) : __uint_as_float(r0[jj]);
                }
                if (c >= g.N) continue;  // warp-uniform
                epi_bias_res_relu<32>(v, c, g.N, g.bias, (g.res && valid) ? g.res + orow * g.N : nullptr, g.relu);
                if (LKNOB(1)) {
                } else if (vec && c + 32 <= g.N) {
                    warp_store_block32(scratch, v, valid ? dst + c : nullptr, lane);
                } else if (valid) {
                    _Pragma("unroll") for (int jj = 0; jj < 32; ++jj) if (c + jj < g.N) dst[c + jj] = v[jj];
                }
            }
            tc_fence_before();
            mbar_arrive_relaxed(&a3_empty[sb]);
            if (threadIdx.x == 320) LTL(t, 10);  // E3: Y stored
        }
    } else {  // ======================= converters: fp32 staging -> bf16 hi/lo A tiles (in place)
        // thread = block row: reads its row's 64 fp32 channels (two 128B-swizzled 32-channel
        // boxes), then overwrites the same two 128-byte rows with the row's bf16 hi (first
        // 16 KB) and lo (second 16 KB) -- each thread touches only its own rows, no barrier.
        const int row = threadIdx.x - 14 * 32;
        const bool crow = row < g.XR;  // slot rows (the MMA's rows beyond XR are junk)
        Ring xr(g.XS);
        for (int k = k0; k < k1; ++k) {
            const TileGeo tg = tile_geo(g, k, k0);
            for (int blk = 0; blk < tg.nb; ++blk)
                for (int cc = 0; cc < g.cchunks; ++cc, xr.next()) {
                    mbar_wait(&x_full[xr.slot], xr.phase);
                    if (row == 0 && blk == tg.nb - 1 && cc == g.cchunks - 1) LTL(k - k0, 20);  // X landed (last block)
                    const uint32_t base = smem_u32(smem + L.xs + (size_t)xr.slot * xslot);
                    if (LKNOB(2) || !crow) {
                        mbar_arrive(&conv[xr.slot]);
                        continue;
                    }
                    // box 0 row (channels 0-31) -> hi chunks 0-3 written at once (its own row
                    // of the hi tile overlays exactly the fp32 row just read); lo chunks 0-3
                    // overlay the box-1 row, so they wait until that row has been read
                    uint4 lo_keep[4];
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        float v[32];
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const float4 f = ld_shared_v4(base + hf * xhalf + row * 128 + ((jj ^ (row & 7)) << 4));
                            v[4 * jj] = f.x; v[4 * jj + 1] = f.y; v[4 * jj + 2] = f.z; v[4 * jj + 3] = f.w;
                        }
#pragma unroll
                        for (int g8 = 0; g8 < 4; ++g8) {
                            uint4 h, l;
                            split_bf16x8(v + 8 * g8, h, l);
                            const int c8 = 4 * hf + g8;
                            const uint32_t o = row * 128 + ((c8 ^ (row & 7)) << 4);
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + o), "r"(h.x),
                                         "r"(h.y), "r"(h.z), "r"(h.w) : "memory");
                            if (hf == 0) {
                                lo_keep[g8] = l;
                            } else {
                                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + xhalf + o),
                                             "r"(l.x), "r"(l.y), "r"(l.z), "r"(l.w) : "memory");
                            }
                        }
                    }
#pragma unroll
                    for (int g8 = 0; g8 < 4; ++g8) {
                        const uint32_t o = row * 128 + ((g8 ^ (row & 7)) << 4);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + xhalf + o),
                                     "r"(lo_keep[g8].x), "r"(lo_keep[g8].y), "r"(lo_keep[g8].z), "r"(lo_keep[g8].w)
                                     : "memory");
                    }
                    fence_proxy_async_smem();
                    mbar_arrive(&conv[xr.slot]);
                    if ((row & 31) == 0 && blk == tg.nb - 1 && cc == g.cchunks - 1) LTL(k - k0, row == 0 ? 1 : 16 + row / 32);  // converter warp done
                }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (g.dbg && blockIdx.x == 0)  // debug dump of the CTA's shared memory (layout = layer_smem)
        for (uint32_t o = threadIdx.x * 16; o + 16 <= L.total - 1024; o += kLayerThreads * 16)
            *reinterpret_cast<uint4 *>(g.dbg + o) = *reinterpret_cast<const uint4 *>(smem + o);
    if (warp == 1) tmem_dealloc(tmem, (uint32_t)g.tmem_cols);
}

// Incremental tile walk of a CTA's contiguous range (tile_geo without a division per tile:
// the epilogue / converter warps are issue-bound).  nbf / nbr: stage-1 blocks of a fresh /
// regular tile.
// Tiles of an image are ordered (strip, row block), so consecutive tiles of a strip slide the
// band ring down its rows.
struct TileWalk {
    int b, strip, j;
    bool first = true;
    __device__ TileWalk(const BfLayerArgs &g, int k0) {
        b = k0 / g.T;
        const int rem = k0 - b * g.T;
        strip = rem / g.TH;
        j = rem - strip * g.TH;
    }
    __device__ __forceinline__ TileGeo geo(const BfLayerArgs &g, int nbf, int nbr) const {
        TileGeo t;
        t.b = b;
        t.j = j;
        t.fresh = first || j == 0;
        t.ylo = j * g.R + (t.fresh ? 0 : g.e);
        t.yhi = j * g.R + g.R + g.e;
        t.nb = t.fresh ? nbf : nbr;
        t.x0 = strip * g.sw;
        return t;
    }
    __device__ __forceinline__ void next(const BfLayerArgs &g) {
        first = false;
        if (++j == g.TH) {
            j = 0;
            if (++strip == g.nstrips) {
                strip = 0;
                ++b;
            }
        }
    }
};

// Variant 5b: the tap-pair layer kernel with the stage-1 and stage-3 A operands in TENSOR
// memory.  The kernel above is bound by shared-memory bandwidth (~415 KB of shared-memory
// traffic per 56x56 tile at 128 B/cycle ~ 1.65 us against a measured ~1.95 us tile period):
// every SS-MMA re-reads its A tile from shared memory.  Here
//   * the converters split X into bf16 hi/lo straight into a TMEM slot (tcgen05.st) and
//     release the fp32 staging slot as soon as they have read it, and stage 1 is a TS-MMA
//     (A = X hi / lo from TMEM): no bf16 X tile is written to or read from shared memory;
//   * epilogue 2 writes Z hi/lo back into the first D2s columns of the acc2 buffer it has
//     just read, and stage 3 is a TS-MMA reading Z from there (acc2 is released by the
//     stage-3 commit): Z never touches shared memory;
//   * the freed Z buffers become a third fp32 staging slot.
// TMEM: X 2 x 64 | acc1 2*D1s | acc2 2 x 4*D2s | acc3 N3p columns (R18 56x56: 512); acc1 and
// acc3 are single-buffered -- epilogues 1 and 3 read the whole accumulator into registers
// and release it before their shared-memory / global stores.  K = 3, D1s = D2s = 32,
// N3p <= 64 (the layer's ranks / channels are what the single-buffer register reads allow).
__global__ void __launch_bounds__(kLayerThreads, 1)
tdc_bf_layer_tm_kernel(const __grid_constant__ CUtensorMap mapX, const BfLayerArgs g) {
    constexpr int KT = 3;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const LayerSmem L = layer_smem(g);
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + L.bars);
    uint64_t *x_full = bars, *x_empty = bars + 4;      // fp32 staging ring (XS <= 4)
    uint64_t *xt_full = bars + 8, *xt_empty = bars + 10;  // TMEM X slots (2)
    uint64_t *w_full = bars + 12;
    uint64_t *a1_full = bars + 13, *a1_empty = bars + 15;
    uint64_t *band_ready = bars + 17, *band_free = bars + 19;
    uint64_t *a2_full = bars + 21, *a2_empty = bars + 23;
    uint64_t *z_full = bars + 25;
    uint64_t *a3_full = bars + 29;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 40);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef TDC_TIMELINE
    const bool tl_on = (int)blockIdx.x == *(volatile int *)&g_tdc_ltl_cta;
    if (threadIdx.x == 0) LTL(0, 21);
#endif
    // epilogue / converter / producer waits back off (debug knob 256: plain spin)
#define BWAIT(bar, par) (LKNOB(256) ? mbar_wait((bar), (par)) : mbar_wait_backoff<128>((bar), (par)))
    const int nbf = (g.R + g.e + g.rpb - 1) / g.rpb, nbr = (g.R + g.rpb - 1) / g.rpb;
    if (threadIdx.x == 0) {
        for (int i = 0; i < g.XS; ++i) {
            mbar_init(&x_full[i], 1);
            mbar_init(&x_empty[i], 128);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&xt_full[i], 128);
            mbar_init(&xt_empty[i], 1);
            mbar_init(&band_ready[i], 128);
            mbar_init(&band_free[i], 1);
            mbar_init(&a2_full[i], 1);
            mbar_init(&a2_empty[i], 128);  // epilogue 3 (acc3 lives in the acc2 buffer)
            mbar_init(&a1_full[i], 1);
            mbar_init(&a1_empty[i], 128);
            mbar_init(&a3_full[i], 1);
            mbar_init(&z_full[i], 128);
        }
        mbar_init(w_full, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) tma_prefetch(&mapX);
    if (warp == 1) tmem_alloc(tmem_slot, (uint32_t)g.tmem_cols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) LTL(0, 22);

    const int k0 = (int)(blockIdx.x * (unsigned)g.num_tiles / gridDim.x);  // num_tiles * grid < 2^32 (plan)
    const int k1 = (int)((blockIdx.x + 1) * (unsigned)g.num_tiles / gridDim.x);
    const int nt = k1 - k0;
    // TMEM columns
    // TMEM columns: X slots [0, 128) | acc1 x 2 | acc2 x 2; the acc2 buffer of tile t also holds,
    // once epilogue 2 has read it, Z hi/lo (columns [64, 96)) and then acc3 (columns [0, N3p))
    const uint32_t acc1_base = 128, acc2_cols = 4 * g.D2s, acc1_cols = 2 * g.D1s;
    const uint32_t acc2_base = acc1_base + 2 * acc1_cols, z_off = 64;
    const uint32_t plane_stride = (uint32_t)g.NRB * g.Wq * 16;
    const uint32_t band_half = (uint32_t)(g.D1s / 8) * plane_stride;
    const uint32_t xslot = 2u * g.XR * 128, xhalf = (uint32_t)g.XR * 128;

    if (warp == 0) {  // =============================================== producer
        const int w1b = (int)(L.w2 - L.w1), w2b = (int)(L.w3 - L.w2), w3b = (int)(L.band - L.w3);
        auto load_split = [&](uint8_t *dst, const void *src, uint32_t bytes) {
            const uint32_t piece = 16384;
            for (uint32_t o = (uint32_t)lane * piece; o < bytes; o += 32 * piece)
                bulk_load(dst + o, reinterpret_cast<const uint8_t *>(src) + o, bytes - o < piece ? bytes - o : piece,
                          w_full);
        };
        if (lane == 0) mbar_arrive_expect_tx(w_full, (uint32_t)(w1b + w2b + w3b));
        __syncwarp();
        load_split(smem + L.w1, g.w1, w1b);
        load_split(smem + L.w2, g.w2, w2b);
        load_split(smem + L.w3, g.w3, w3b);
        __syncwarp();
        pdl_wait();
        const uint32_t box_bytes = (uint32_t)g.rpb * g.Wp * 128;
        // no L2 prefetch here: the three fp32 staging slots cover the load latency (TDC_LAYER_PF
        // measured no gain), and the prefetch loop was ~1400 instructions of code
        Ring xr(g.XS);
        TileWalk tw(g, k0);
        for (int k = k0; k < k1; ++k, tw.next(g)) {
            const TileGeo tg = tw.geo(g, nbf, nbr);
            for (int blk = 0; blk < tg.nb; ++blk) {
                const int u0 = tg.ylo + blk * g.rpb;
                for (int cc = 0; cc < g.cchunks; ++cc, xr.next()) {
                    BWAIT(&x_empty[xr.slot], xr.phase ^ 1);
                    if (lane == 0 && blk == 0 && cc == 0) LTL(k - k0, 0);
                    if (LKNOB(128) && (k > k0 + 1)) {  // debug: no X traffic after the first tiles
                        if (elect_one()) mbar_arrive(&x_full[xr.slot]);
                        __syncwarp();
                        continue;
                    }
                    if (elect_one()) {
                        uint8_t *dst = smem + L.xs + (size_t)xr.slot * xslot;
                        mbar_arrive_expect_tx(&x_full[xr.slot], 2 * box_bytes);
                        tma_load_4d(dst, &mapX, &x_full[xr.slot], cc * 64, tg.x0 - g.p, u0 - g.p, tg.b);
                        tma_load_4d(dst + xhalf, &mapX, &x_full[xr.slot], cc * 64 + 32, tg.x0 - g.p, u0 - g.p, tg.b);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1 || warp == kS1Warp || warp == kS3Warp) {  // ============== MMA issue
        const uint32_t id1 = idesc_bf16(128, 2 * g.D1s), id1h = idesc_bf16(128, g.D1s);
        const uint32_t id2 = idesc_bf16(128, 2 * g.D2s), id2h = idesc_bf16(128, g.D2s);
        const uint32_t id3h = idesc_bf16(128, g.N3p);
        const uint64_t dw1 = sdesc_kmajor_sw128(smem_u32(smem + L.w1));
        const uint64_t dband = sdesc_kmajor_none(smem_u32(smem + L.band), plane_stride, 128);
        const uint64_t dw2tn = sdesc_kmajor_none(smem_u32(smem + L.w2), 6 * g.D2s * 16, 128);
        const uint32_t id2tn = idesc_bf16(128, 4 * g.D2s), id2tnh = idesc_bf16(128, 2 * g.D2s);
        const uint64_t dw3 = sdesc_kmajor_none(smem_u32(smem + L.w3), 2 * g.N3p * 16, 128);
        const uint32_t w1_chunk = (uint32_t)2 * g.D1s * 128;
        const uint32_t w3_plane2 = (uint32_t)2 * 2 * g.N3p * 16;
        const int kc2 = g.D1s / 32, k3 = g.D2s / 16;
        mbar_wait(w_full, 0);
        if (warp == kS1Warp && lane == 0) LTL(0, 23);
        if (warp == 1) {  // the core stream (stage 2): tap pairs along N, as in the kernel above
            uint32_t start = 0;
            for (int t = 0; t < nt; ++t) {
                if (lane == 0) LTL(t, 11);
                const uint32_t sb = t & 1, sph = (t >> 1) & 1;
                mbar_wait(&band_ready[sb], sph);
                mbar_wait(&a2_empty[sb], sph ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc2_base + sb * acc2_cols;
                const uint32_t wq = (uint32_t)g.Wq, p2a = (2 * plane_stride) >> 4, lo_a = band_half >> 4;
                const uint32_t wr = (4 * 6 * g.D2s * 16) >> 4, p2b = (2 * 6 * g.D2s * 16) >> 4;
                const uint32_t rows16 = ((uint32_t)g.D2s * 16) >> 4;
                const bool wrap = g.R == 1;  // ring rows wrap (no mirror rows, see the planner)
                for (int kc = 0; kc < (LKNOB(16) ? 0 : kc2); ++kc) {
                    const uint64_t ak = dband + (uint32_t)kc * ((4 * plane_stride) >> 4);
                    const uint64_t bk = dw2tn + (uint32_t)kc * KT * wr;
                    if (elect_one()) {
                        // rolled over the core rows: the whole kernel's per-tile code does not fit the
                        // 32 KB instruction cache, and a smaller stream measured faster
#pragma unroll 1
                        for (int r = 0; r < KT; ++r) {
                            uint32_t row = start + r;
                            if (wrap && row >= (uint32_t)g.NR) row -= g.NR;
#pragma unroll
                            for (int j = 0; j < 2; ++j) {
                                const uint64_t aj = ak + row * wq + j * p2a, bj = bk + r * wr + j * p2b;
                                mma_bf16(d, aj, bj, id2tn, (kc > 0) || r || j);
                                mma_bf16(d + g.D2s, aj + lo_a, bj + rows16, id2tnh, 1);
                                mma_bf16(d, aj + 2, bj + 4 * rows16, id2, 1);
                                mma_bf16(d, aj + 2 + lo_a, bj + 4 * rows16, id2h, 1);
                            }
                        }
                    }
                    __syncwarp();
                }
                if (elect_one()) {
                    mma_commit(&band_free[sb]);
                    mma_commit(&a2_full[sb]);
                }
                __syncwarp();
                if (lane == 0) LTL(t, 3);
                start += g.R;
                if (start >= (uint32_t)g.NR) start -= g.NR;
            }
        } else if (warp == kS1Warp) {  // stage 1: A = X hi / lo from TMEM slots
            Ring xt(2);
            uint32_t ublk = 0;
            for (int t = 0; t < nt; ++t) {
                const int nb = (t == 0 || (k0 + t) % g.TH == 0) ? nbf : nbr;
                for (int blk = 0; blk < nb; ++blk, ++ublk) {
                    if (lane == 0 && blk == 0) LTL(t, 13);
                    const uint32_t ab = ublk & 1, aph = (ublk >> 1) & 1;
                    mbar_wait(&a1_empty[ab], aph ^ 1);
                    tc_fence_after();
                    const uint32_t d = tmem + acc1_base + ab * acc1_cols;
                    for (int cc = 0; cc < g.cchunks; ++cc, xt.next()) {
                        mbar_wait(&xt_full[xt.slot], xt.phase);
                        tc_fence_after();
                        if (elect_one()) {
                            const uint32_t a = tmem + xt.slot * 64;
                            const uint64_t b = dw1 + ((cc * w1_chunk) >> 4);
#pragma unroll
                            for (int j = 0; j < (LKNOB(32) ? 0 : 4); ++j) {  // K = 16 channels = 8 TMEM columns
                                mma_bf16_ts(d, a + j * 8, b + j * 2, id1, (cc > 0) || (j > 0));  // hi * [hi | lo]
                                mma_bf16_ts(d, a + 32 + j * 8, b + j * 2, id1h, 1);            // lo * hi
                            }
                            mma_commit(&xt_empty[xt.slot]);
                        }
                        __syncwarp();
                    }
                    if (elect_one()) mma_commit(&a1_full[ab]);
                    __syncwarp();
                    if (lane == 0 && blk == nb - 1) LTL(t, 2);
                }
            }
        } else {  // stage 3: A = Z hi / lo from the first D2s columns of the acc2 buffer
            for (int t = 0; t < nt; ++t) {
                const uint32_t sb = t & 1, sph = (t >> 1) & 1;
                mbar_wait(&z_full[sb], sph);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t d = tmem + acc2_base + sb * acc2_cols, z = d + z_off;
                    for (int j = 0; j < (LKNOB(64) ? 0 : k3); ++j) {
                        const uint64_t b = dw3 + ((j * w3_plane2) >> 4);
                        // Z channels [16j, 16j+16): hi in columns [16j, 16j+8), lo in [16j+8, 16j+16)
                        mma_bf16_ts(d, z + j * 16, b, id3h, j > 0);                          // hi * hi
                        mma_bf16_ts(d, z + j * 16, b + ((g.N3p * 16) >> 4), id3h, 1);         // hi * lo
                        mma_bf16_ts(d, z + j * 16 + 8, b, id3h, 1);                          // lo * hi
                    }
                    mma_commit(&a3_full[sb]);
                }
                __syncwarp();
                if (lane == 0) LTL(t, 4);
            }
        }
    } else if (warp < 6) {  // ========================= epilogue 1: acc1 -> X' band ring
        const int q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t bandA = smem_u32(smem + L.band);
        const int i = q * 32 + lane;
        const int yy = i / g.Wp, xx = i - yy * g.Wp;
        uint32_t ublk = 0;
        int start = 0;
        TileWalk tw(g, k0);
        for (int t = 0; t < nt; ++t, tw.next(g)) {
            const TileGeo tg = tw.geo(g, nbf, nbr);
            for (int blk = 0; blk < tg.nb; ++blk, ++ublk) {
                if (blk == 0 && t > 0) {
                    const int tb = tg.fresh ? t - 1 : t - 2;
                    if (tb >= 0) BWAIT(&band_free[tb & 1], (tb >> 1) & 1);
                }
                const uint32_t ab = ublk & 1, aph = (ublk >> 1) & 1;
                BWAIT(&a1_full[ab], aph);
                tc_fence_after();
                if (threadIdx.x == 64 && blk == 0) LTL(t, 5);
                uint32_t r0[2][16], r1[2][16];  // D1s = 32: hi part | lo part, two 16-column halves
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    tmem_ld_32x32b_x16(tmem + lane_base + acc1_base + ab * acc1_cols + 16 * h, r0[h]);
                    tmem_ld_32x32b_x16(tmem + lane_base + acc1_base + ab * acc1_cols + g.D1s + 16 * h, r1[h]);
                }
                tmem_ld_wait();
                tc_fence_before();
                mbar_arrive_relaxed(&a1_empty[ab]);  // acc1 buffer free for stage-1 block ublk + 2
                const int y = tg.ylo + blk * g.rpb + yy;
                const bool valid = i < g.rpb * g.Wp && y < tg.yhi;
                if (valid && !LKNOB(4)) {
                    int slot = start + (y - tg.j * g.R);
                    if (slot >= g.NR) slot -= g.NR;
                    const bool mirror = slot < g.NRB - g.NR;
                    const uint32_t pos = (uint32_t)(slot * g.Wq + xx) * 16;
                    const uint32_t pos2 = pos + (uint32_t)g.NR * g.Wq * 16;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float v[16];
#pragma unroll
                        for (int jj = 0; jj < 16; ++jj) v[jj] = __uint_as_float(r0[h][jj]) + __uint_as_float(r1[h][jj]);
#pragma unroll
                        for (int pl = 0; pl < 2; ++pl) {
                            uint4 hh, ll;
                            split_bf16x8(v + 8 * pl, hh, ll);
                            const uint32_t po = (uint32_t)(2 * h + pl) * plane_stride;
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + po + pos), "r"(hh.x),
                                         "r"(hh.y), "r"(hh.z), "r"(hh.w) : "memory");
                            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + band_half + po + pos),
                                         "r"(ll.x), "r"(ll.y), "r"(ll.z), "r"(ll.w) : "memory");
                            if (mirror) {
                                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + po + pos2),
                                             "r"(hh.x), "r"(hh.y), "r"(hh.z), "r"(hh.w) : "memory");
                                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(bandA + band_half + po + pos2),
                                             "r"(ll.x), "r"(ll.y), "r"(ll.z), "r"(ll.w) : "memory");
                            }
                        }
                    }
                }
            }
            fence_proxy_async_smem();
            mbar_arrive(&band_ready[t & 1]);
            if (threadIdx.x == 64) LTL(t, 6);
            start += g.R;
            if (start >= g.NR) start -= g.NR;
        }
    } else if (warp < 10) {  // ======================= epilogue 2: acc2 -> Z hi/lo (TMEM)
        const int q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        float *xbuf = reinterpret_cast<float *>(smem + L.xch);  // [chunk 2][quarter 4][16]
        for (int t = 0; t < nt; ++t) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            BWAIT(&a2_full[sb], sph);
            tc_fence_after();
            if (threadIdx.x == 192) LTL(t, 7);
            const uint32_t a2 = tmem + lane_base + acc2_base + sb * acc2_cols;
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {  // Z[m] = blk0[m] + blk1[m + 1] (tap pairs, see above)
                const int c = ch * 16;
                float p0[16], p1[16];
                {
                    uint32_t r0[16], r1[16], r2[16], r3[16];
                    tmem_ld_32x32b_x16(a2 + c, r0);
                    tmem_ld_32x32b_x16(a2 + g.D2s + c, r1);
                    tmem_ld_32x32b_x16(a2 + 2 * g.D2s + c, r2);
                    tmem_ld_32x32b_x16(a2 + 3 * g.D2s + c, r3);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        p0[jj] = __uint_as_float(r0[jj]) + __uint_as_float(r1[jj]);
                        p1[jj] = __uint_as_float(r2[jj]) + __uint_as_float(r3[jj]);
                    }
                }
                const uint32_t mine = smem_u32(xbuf + (ch * 4 + q) * 16),
                               next = smem_u32(xbuf + (ch * 4 + ((q + 1) & 3)) * 16);
                if (lane == 0)
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4)
                        st_shared_v4(mine + 16 * j4, p1[4 * j4], p1[4 * j4 + 1], p1[4 * j4 + 2], p1[4 * j4 + 3]);
                asm volatile("bar.sync 3, 128;" ::: "memory");
                float nx[16];
                if (lane == 31)
#pragma unroll
                    for (int j4 = 0; j4 < 4; ++j4) {
                        const float4 f = ld_shared_v4(next + 16 * j4);
                        nx[4 * j4] = f.x; nx[4 * j4 + 1] = f.y; nx[4 * j4 + 2] = f.z; nx[4 * j4 + 3] = f.w;
                    }
                float v[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                    float s1 = __shfl_down_sync(0xffffffffu, p1[jj], 1);
                    if (lane == 31) s1 = nx[jj];
                    v[jj] = p0[jj] + s1;
                }
                uint32_t zh[8], zl[8];
#pragma unroll
                for (int g8 = 0; g8 < 2; ++g8) {
                    uint4 hh, ll;
                    split_bf16x8(v + 8 * g8, hh, ll);
                    zh[4 * g8] = hh.x; zh[4 * g8 + 1] = hh.y; zh[4 * g8 + 2] = hh.z; zh[4 * g8 + 3] = hh.w;
                    zl[4 * g8] = ll.x; zl[4 * g8 + 1] = ll.y; zl[4 * g8 + 2] = ll.z; zl[4 * g8 + 3] = ll.w;
                }
                // Z channels [c, c+16): hi -> columns [c, c+8), lo -> [c+8, c+16) of the buffer
                // just read -- columns this warp has already loaded for its own lanes (chunk 0
                // read [0,16) of every block, so chunk 0's Z cannot clobber chunk 1's inputs)
                if (!LKNOB(8)) {
                    tmem_st_32x32b_x8(a2 + z_off + c, zh);
                    tmem_st_32x32b_x8(a2 + z_off + c + 8, zl);
                }
            }
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&z_full[sb]);
            if (threadIdx.x == 192) LTL(t, 8);
        }
    } else if (warp < 14) {  // ======================= epilogue 3: acc3 (+bias, res, relu) -> Y
        const int q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        float *scratch = reinterpret_cast<float *>(smem + L.scr) + q * 1024;
        const int m = q * 32 + lane;
        const int yo = m / g.Wq, xo = m - yo * g.Wq;
        const bool vec = (g.N & 3) == 0;
        const int nch = g.N3p / 32;  // 1 or 2
        TileWalk e3w(g, k0);
        for (int t = 0; t < nt; ++t) {
            const int b = e3w.b, j = e3w.j, ox = e3w.strip * g.sw + xo;
            e3w.next(g);
            const int oy = j * g.R + yo;
            const bool valid = yo < g.R && oy < g.Ho && xo < g.sw && ox < g.Wo;
            const long long orow = ((long long)b * g.Ho + oy) * g.Wo + ox;
            float *dst = g.y + orow * g.N;
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            const uint32_t a3 = tmem + lane_base + acc2_base + sb * acc2_cols;
            BWAIT(&a3_full[sb], sph);
            tc_fence_after();
            if (threadIdx.x == 320) LTL(t, 9);
            // chunk by chunk; acc3 is released once its last chunk has been read, so stage 3 of
            // the next tile overlaps the last chunk's stores
            for (int c2 = 0; c2 < nch; ++c2) {
                const int c = 32 * c2;
                float v[32];
                {
                    uint32_t r0[16], r1[16];
                    tmem_ld_32x32b_x16(a3 + c, r0);
                    tmem_ld_32x32b_x16(a3 + c + 16, r1);
                    tmem_ld_wait();
#pragma unroll
                    for (int jj = 0; jj < 16; ++jj) {
                        v[jj] = __uint_as_float(r0[jj]);
                        v[16 + jj] = __uint_as_float(r1[jj]);
                    }
                }
                if (c2 == nch - 1) {
                    tc_fence_before();
                    mbar_arrive_relaxed(&a2_empty[sb]);  // the acc2 buffer is free for S2(t + 2)
                }
                if (c >= g.N) continue;  // warp-uniform
                epi_bias_res_relu<32>(v, c, g.N, g.bias, (g.res && valid) ? g.res + orow * g.N : nullptr, g.relu);
                if (LKNOB(1)) {
                } else if (vec && c + 32 <= g.N) {
                    warp_store_block32(scratch, v, valid ? dst + c : nullptr, lane);
                } else if (valid) {
                    _Pragma("unroll") for (int jj = 0; jj < 32; ++jj) if (c + jj < g.N) dst[c + jj] = v[jj];
                }
            }
            if (threadIdx.x == 320) LTL(t, 10);
        }
    } else {  // ======================= converters: fp32 staging -> bf16 hi/lo in a TMEM slot
        const int q = warp & 3;  // TMEM lane quarter = warp % 4; thread = X block row
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const int row = q * 32 + lane;
        const bool crow = row < g.XR;
        Ring xr(g.XS), xt(2);
        TileWalk tw(g, k0);
        for (int k = k0; k < k1; ++k, tw.next(g)) {
            const TileGeo tg = tw.geo(g, nbf, nbr);
            for (int blk = 0; blk < tg.nb; ++blk)
                for (int cc = 0; cc < g.cchunks; ++cc, xr.next(), xt.next()) {
                    BWAIT(&x_full[xr.slot], xr.phase);
                    if (row == 0 && blk == tg.nb - 1 && cc == g.cchunks - 1) LTL(k - k0, 20);
                    BWAIT(&xt_empty[xt.slot], xt.phase ^ 1);
                    tc_fence_after();
                    const uint32_t base = smem_u32(smem + L.xs + (size_t)xr.slot * xslot);
                    const uint32_t tx = tmem + lane_base + xt.slot * 64;
#pragma unroll 1
                    for (int hf = 0; hf < (LKNOB(2) ? 0 : 2); ++hf) {  // box hf = channels 32*hf .. 32*hf + 31
                        float v[32];
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (crow) f = ld_shared_v4(base + hf * xhalf + row * 128 + ((jj ^ (row & 7)) << 4));
                            v[4 * jj] = f.x; v[4 * jj + 1] = f.y; v[4 * jj + 2] = f.z; v[4 * jj + 3] = f.w;
                        }
                        uint32_t h[16], l[16];
#pragma unroll
                        for (int g8 = 0; g8 < 4; ++g8) {
                            uint4 hh, ll;
                            split_bf16x8(v + 8 * g8, hh, ll);
                            h[4 * g8] = hh.x; h[4 * g8 + 1] = hh.y; h[4 * g8 + 2] = hh.z; h[4 * g8 + 3] = hh.w;
                            l[4 * g8] = ll.x; l[4 * g8 + 1] = ll.y; l[4 * g8 + 2] = ll.z; l[4 * g8 + 3] = ll.w;
                        }
                        tmem_st_32x32b_x16(tx + 16 * hf, h);       // hi: columns [0, 32)
                        tmem_st_32x32b_x16(tx + 32 + 16 * hf, l);  // lo: columns [32, 64)
                    }
                    mbar_arrive(&x_empty[xr.slot]);  // the fp32 staging slot has been read
                    tmem_st_wait();
                    tc_fence_before();
                    mbar_arrive(&xt_full[xt.slot]);
                    if ((row & 31) == 0 && blk == tg.nb - 1 && cc == g.cchunks - 1) LTL(k - k0, row == 0 ? 1 : 16 + row / 32);
                }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (g.dbg && blockIdx.x == 0)
        for (uint32_t o = threadIdx.x * 16; o + 16 <= L.total - 1024; o += blockDim.x * 16)
            *reinterpret_cast<uint4 *>(g.dbg + o) = *reinterpret_cast<const uint4 *>(smem + o);
    if (warp == 1) tmem_dealloc(tmem, (uint32_t)g.tmem_cols);
#undef BWAIT
}

cudaError_t bf_layer_launch(const CUtensorMap &mapX, const BfLayerArgs &g, int grid, cudaStream_t st) {
    const int smem = bf_layer_smem_bytes(g);
    auto go = [&](auto kernel) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(kernel, grid, kLayerThreads, smem, st, mapX, g);
    };
    if (g.xt) return go(tdc_bf_layer_tm_kernel);
    if (g.tn) return go(tdc_bf_layer_kernel<3, true>);
    return g.K == 3 ? go(tdc_bf_layer_kernel<3, false>) : go(tdc_bf_layer_kernel<0, false>);
}

}  // namespace tdc
