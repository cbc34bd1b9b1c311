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
#include <type_traits>
#include <cuda_bf16.h>

#include <cstdlib>

#include "internal.h"
#include "sm100.cuh"
#include "tkd_common.cuh"

namespace tdc {

using namespace sm100;

// Debug knobs (TDC_CORE_DBG / TDC_GEMM_DBG bits, TDC_Y_DIRECT) exist only in debug builds
// (-DTDC_DEBUG_KNOBS, implied by the timeline build): the production kernels carry no
// knob branches in their hot loops (smaller code).
#if defined(TDC_DEBUG_KNOBS) || defined(TDC_TIMELINE)
#define TDC_DBG(g, bit) ((g).dbg & (bit))
#define TDC_YDIRECT(g) ((g).y_direct)
#else
#define TDC_DBG(g, bit) 0
#define TDC_YDIRECT(g) 0
#endif

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
__device__ unsigned long long g_tdc_bfc_tl[64 * 12];
__device__ __forceinline__ void bfctl(int it, int ev) {
    if (blockIdx.x == 0 && it < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_bfc_tl[it * 12 + ev] = t;
    }
}
extern "C" int tdc_debug_bfc_timeline(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_bfc_tl, sizeof(unsigned long long) * n);
}
#define BFCTL(it, ev) bfctl((it), (ev))
__device__ unsigned long long g_tdc_bfc_tap[128 * 2];
__device__ __forceinline__ void bfctap(int i, int ev) {
    if (blockIdx.x == 0 && i < 128) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_bfc_tap[i * 2 + ev] = t;
    }
}
extern "C" int tdc_debug_bfc_taps(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_bfc_tap, sizeof(unsigned long long) * n);
}
#define BFCTAP(i, ev) bfctap((i), (ev))
// per-CTA [start, after-prologue, end] stamps of the last core launch
__device__ unsigned long long g_tdc_bfc_span[1024 * 4];
__device__ __forceinline__ void bfcspan(int ev) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_tdc_bfc_span[blockIdx.x * 4 + ev] = t;
}
extern "C" int tdc_debug_bfc_span(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_bfc_span, sizeof(unsigned long long) * n);
}
#define BFCSPAN(ev) bfcspan(ev)
// per-CTA [start, after-prologue, end] of the gemm launches: [launch seq % 4][cta][4]
__device__ unsigned long long g_tdc_bfg_span[4 * 1024 * 4];
__device__ __forceinline__ void bfgspan(int seq, int ev) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x < 1024) g_tdc_bfg_span[((seq & 3) * 1024 + blockIdx.x) * 4 + ev] = t;
}
extern "C" int tdc_debug_bfg_span(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_bfg_span, sizeof(unsigned long long) * n);
}
#define BFGSPAN(seq, ev) bfgspan((seq), (ev))
// per-chunk events of CTA 0's first tile of the gemm launches: [seq % 4][chunk < 64][4]:
// 0 producer issued the chunk's A, 1 converter saw it land, 2 converter done, 3 MMAs issued
__device__ unsigned long long g_tdc_bfk[4 * 64 * 4];
__device__ __forceinline__ void bfk(int seq, int tit, int i, int ev) {
    if (blockIdx.x == 0 && tit == 0 && i < 64) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_tdc_bfk[((seq & 3) * 64 + i) * 4 + ev] = t;
    }
}
extern "C" int tdc_debug_bf_chunks(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_bfk, sizeof(unsigned long long) * n);
}
#define BFK(seq, it, i, ev) bfk((seq), (it), (i), (ev))
#else
#define BFK(seq, it, i, ev) ((void)0)
#define BFGSPAN(seq, ev) ((void)0)
#define BFCSPAN(ev) ((void)0)
#define BFCTAP(i, ev) ((void)0)
#define BFTL(seq, it, ev) ((void)0)
#define BFCTL(it, ev) ((void)0)
#endif

constexpr int kBM16 = 128;
constexpr int kBK16 = 64;                       // bf16 elements per K chunk = one 128 B row
constexpr int kATile16 = kBM16 * kBK16 * 2;     // 16 KB per hi or lo tile
constexpr int kStage32 = kBM16 * 32 * 4 * 2;    // fp32 staging of one 64-channel chunk (2 boxes)
constexpr int kEpiScratch16 = 4 * 4096;
// fp32-output GEMMs (stage 3, model dense convs): each epilogue warp owns a ring of
// kYRing 4 KB buffers; 32 x 32 output blocks are staged there (128B-swizzled) and
// stored by TMA with up to kYRing - 1 stores in flight, and the residual block of the
// next chunk is TMA-loaded into the ring ahead of use (no synchronous global reads).
// (ring of 4 for stage 3; 2 for the converting dense convs of the model path, whose fp32
// staging ring already takes most of shared memory)
constexpr int kYRing = 4;
// ring depth: stage 3 (not converting) 4; converting fp32-output GEMMs g.yring (2 or 4)
__host__ __device__ inline int bf_yring(bool convert, int yring) { return convert ? (yring > 2 ? 4 : 2) : kYRing; }
__host__ __device__ inline int bf_epi_bytes(bool convert, bool out_bf16, int yring) {
    return (convert && out_bf16) ? kEpiScratch16 : 4 * bf_yring(convert, yring) * 4096;
}
// cp.async.bulk.wait_group.read with a run-time count (0..3)
__device__ __forceinline__ void bulk_wait_read_upto(int n) {
    switch (n) {
        case 0: bulk_wait_group_read<0>(); break;
        case 1: bulk_wait_group_read<1>(); break;
        case 2: bulk_wait_group_read<2>(); break;
        default: bulk_wait_group_read<3>(); break;
    }
}

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

// ------------------------------------------------ split-K over a cluster (DSMEM)
// Each CTA of a cluster of CS (<= kMaxSplit) CTAs accumulates a K range of the same
// output tile; the fp32 partials go to shared memory ([128 rows][W cols], 16-byte
// chunks swizzled by row % 8), and after a cluster handshake CTA r sums rows
// [r*128/CS, (r+1)*128/CS) over ranks 0..CS-1 in that fixed order (deterministic).
constexpr int kMaxSplit = 4;

__device__ __forceinline__ void red_store_row32(uint32_t red_a, int W, int row, int c, const float *v) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int j4 = c / 4 + j;
        st_shared_v4(red_a + (uint32_t)(row * W + 4 * (j4 ^ (row & 7))) * 4, v[4 * j], v[4 * j + 1], v[4 * j + 2],
                     v[4 * j + 3]);
    }
}
// v[0..7] = sum over ranks of columns [8*c8, 8*c8 + 8) of row rw (all loads issued first)
__device__ __forceinline__ void red_sum8(uint32_t red_a, int W, int CS, int rw, int c8, float *v) {
    float4 f[2 * kMaxSplit];
    const uint32_t o0 = (uint32_t)(rw * W + 4 * ((2 * c8) ^ (rw & 7))) * 4;
    const uint32_t o1 = (uint32_t)(rw * W + 4 * ((2 * c8 + 1) ^ (rw & 7))) * 4;
#pragma unroll
    for (int k = 0; k < kMaxSplit; ++k)
        if (k < CS) {
            const uint32_t base = mapa_shared(red_a, k);
            f[2 * k] = ld_dsmem_v4(base + o0);
            f[2 * k + 1] = ld_dsmem_v4(base + o1);
        }
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.f;
#pragma unroll
    for (int k = 0; k < kMaxSplit; ++k)
        if (k < CS) {
            v[0] += f[2 * k].x; v[1] += f[2 * k].y; v[2] += f[2 * k].z; v[3] += f[2 * k].w;
            v[4] += f[2 * k + 1].x; v[5] += f[2 * k + 1].y; v[6] += f[2 * k + 1].z; v[7] += f[2 * k + 1].w;
        }
}
__device__ __forceinline__ void red_signal(uint64_t *bar, int CS) {
    for (int k = 0; k < CS; ++k) mbar_arrive_cluster(mapa_shared(smem_u32(bar), k));
}

// ------------------------------------------------ split-K through L2 ("gsplit")
// The K loop of an output tile is cut into GS fixed pieces (independent of the batch,
// so a B = 1 forward equals a slice of a B = 32 one bit for bit).  Each (tile, piece)
// is a work unit of the persistent grid; piece p > 0 writes its fp32 partial tile to
// a plan-owned L2 workspace ([c/4][row][4] float4 planes, lane = row: coalesced) and
// raises a flag; piece 0 (the lowest unit index of the tile) waits for the flags,
// adds the partials in piece order (deterministic) and runs the normal epilogue, then
// clears the flags for the next launch.  Units are dealt round-robin, so a piece-0
// CTA only ever waits on units of higher index held by other CTAs: with all CTAs
// co-resident (persistent grid) and grid >= GS this cannot deadlock.
__device__ __forceinline__ void epi_bar128() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void gs_store32(float *slot, int c, int row, const float *v) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
        st_global_v4(slot + ((size_t)(c / 4 + j) * 128 + row) * 4,
                     make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]));
}
__device__ __forceinline__ void gs_add32(const float *slot, int c, int row, float *v) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const float4 f = __ldcg(reinterpret_cast<const float4 *>(slot + ((size_t)(c / 4 + j) * 128 + row) * 4));
        v[4 * j] += f.x; v[4 * j + 1] += f.y; v[4 * j + 2] += f.z; v[4 * j + 3] += f.w;
    }
}
__device__ __forceinline__ void gs_wait(const int *flag) {
    int v;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if (v) break;
        __nanosleep(32);
    }
}
// after every epilogue thread stored its part of the partial: publish it
__device__ __forceinline__ void gs_publish(int *flag, bool leader) {
    __threadfence();
    epi_bar128();
    if (leader) asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flag), "r"(1) : "memory");
}

// ============================================================ GEMM (stages 1, 3)
constexpr int kConvThreads16 = 256;  // 8 converter warps (stage 1 is converter-paced otherwise)
constexpr int kXT = 2;                // converting GEMMs: X hi/lo TMEM slots (64 columns each)

// KS: 0 plain, 1 cluster split-K, 2 split-K through L2; OB: bf16 planar X' output (stage 1)
// rather than fp32 -- each instantiation carries only the epilogue code it runs.
template <bool CONVERT, int KS, bool OB>
__global__ void __launch_bounds__(CONVERT ? 192 + kConvThreads16 : 192, 1)
tdc_bf_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapAlo,
                   const __grid_constant__ CUtensorMap mapB, const __grid_constant__ CUtensorMap mapBlo,
                   const __grid_constant__ CUtensorMap mapY, const __grid_constant__ CUtensorMap mapR,
                   const TcGemmArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int BN = g.BN;
    const int SX = CONVERT ? g.xstages : 0;  // fp32 staging ring depth (converting GEMMs)
    const int S = CONVERT ? SX : g.stages;   // operand ring depth
    const int SB = CONVERT ? g.bstages : 0;  // converting GEMMs: separate weight ring depth
    const uint32_t b_tile = (uint32_t)BN * kBK16 * 2;
    // non-CONVERT slot: A hi | B hi | A lo | B lo (one TMA ring);
    // CONVERT: the fp32 staging slot is converted IN PLACE into A hi | A lo (the 32 KB of
    // a 128 x 64 fp32 chunk hold exactly its two 16 KB bf16 tiles), so the staging ring is
    // the operand ring; B (hi | lo) has a separate ring the producer fills ahead.
    const uint32_t half = CONVERT ? kATile16 : kATile16 + b_tile;   // A hi -> A lo
    const uint32_t slot_bytes = CONVERT ? (uint32_t)kStage32 : 2 * half;
    const uint32_t bslot = 2 * b_tile;
    // [SX fp32 staging = operand slots | S operand slots][SB B slots][epilogue scratch][red][barriers]
    uint8_t *xstage = smem;
    uint8_t *ops = CONVERT ? xstage : smem;
    uint8_t *bring = smem + (size_t)(CONVERT ? SX : S) * slot_bytes;
    float *epi_scratch = reinterpret_cast<float *>(bring + (size_t)SB * bslot);
    // split-K (cluster of CS CTAs over K): fp32 partial tile [128][BN], float4-swizzled
    const int CS = (KS == 1 && g.ksplit > 1) ? g.ksplit : 1;
    float *red = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(epi_scratch) + bf_epi_bytes(CONVERT, OB, g.yring));
    uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(red) +
                                                  (CS > 1 ? (size_t)128 * BN * 4 : 0));
    uint64_t *conv = full + S;       // CONVERT: A hi/lo written by the converter
    uint64_t *empty = conv + S;      // operand slot consumed by the MMAs
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint64_t *xfull = tempty + 2;    // CONVERT: fp32 X landed in a staging slot
    uint64_t *xempty = xfull + SX;   // CONVERT: staging slot converted
    uint64_t *bfull = xempty + SX;      // CONVERT: B ring
    uint64_t *bempty = bfull + SB;
    uint64_t *red_ready = bempty + SB;  // split-K: all CS partials of the tile written
    uint64_t *red_free = red_ready + 1; // split-K: all CS readers done with this CTA's partial
    uint64_t *rbar = red_free + 1;      // fp32 output: residual block landed in ring buffer [warp][slot]
    uint64_t *xt_full = rbar + 4 * kYRing, *xt_empty = xt_full + kXT;  // CONVERT: TMEM X slots
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(xt_empty + kXT);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t ncols = 32;
    while ((int)ncols < BN) ncols *= 2;
    // CONVERT: the converters write X hi/lo into kXT TMEM slots of 64 columns after the two
    // accumulators, and stage 1 is a TS-MMA -- the fp32 staging slot is free as soon as it has
    // been read, and no bf16 X tile goes through shared memory
    const uint32_t xt_base = 2 * ncols;
    uint32_t tcols = 2 * ncols + (CONVERT ? 64u * kXT : 0u);
    {
        uint32_t p2 = 32;
        while (p2 < tcols) p2 *= 2;
        tcols = p2;
    }
    const int mtiles = (g.M + kBM16 - 1) / kBM16;
    const int num_tiles = mtiles * g.ntiles;
    const int iters = g.taps * g.kchunks;
    const int crank = CS > 1 ? (int)cluster_ctarank() : 0;
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;  // cluster id / count
    const int ci0 = crank * iters / CS, ci1 = (crank + 1) * iters / CS;  // cluster split: this CTA's K range
    const int GS = (KS == 2 && g.gsplit > 1) ? g.gsplit : 1;              // split-K through L2
    const int num_units = num_tiles * GS;
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
        for (int i = 0; i < SX; ++i) {
            mbar_init(&xfull[i], 1);
            mbar_init(&xempty[i], kConvThreads16);  // the converters have read the fp32 slot
        }
        for (int i = 0; i < kXT; ++i) {
            mbar_init(&xt_full[i], kConvThreads16);  // hi/lo written to the TMEM slot
            mbar_init(&xt_empty[i], 1);             // the MMAs that read it completed
        }
        for (int i = 0; i < SB; ++i) {
            mbar_init(&bfull[i], 1);
            mbar_init(&bempty[i], 1);
        }
        mbar_init(red_ready, CS * 128);
        mbar_init(red_free, CS * 128);
        for (int i = 0; i < 4 * kYRing; ++i) mbar_init(&rbar[i], 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA);
        tma_prefetch(&mapB);
    }
    if (threadIdx.x == 0) BFGSPAN(seq, 0);
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    if (CS > 1) cluster_sync();  // peers' barriers initialised before any remote arrive
    tc_fence_after();
    pdl_wait();
    pdl_launch_dependents();
    if (threadIdx.x == 0) BFGSPAN(seq, 1);
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {  // ------------------------------------- TMA producer
        Ring r(CONVERT ? SX : S), rb(CONVERT ? SB : 1);
        int tit = 0;
        for (int u = cid; u < num_units; u += ncl, ++tit) {
            const int t = u / GS, pc = u - t * GS;
            const int i0 = GS > 1 ? pc * iters / GS : ci0, i1 = GS > 1 ? (pc + 1) * iters / GS : ci1;
            const int m0 = (t % mtiles) * kBM16, n0 = (t / mtiles) * BN;
            int tap = i0 / g.kchunks, kc = i0 % g.kchunks;
            for (int i = i0; i < i1; ++i, r.next()) {
                if (CONVERT) {  // fp32 X: channels [64kc, 64kc+32) and [64kc+32, 64kc+64)
                    mbar_wait(&xempty[r.slot], r.phase ^ 1);
                    if (i == i0 && lane == 0) BFTL(seq, tit, 0);  // producer issues tile
                    if (lane == 0) BFK(seq, tit, i - i0, 0);
                    if (elect_one()) {
                        uint8_t *dst = xstage + (size_t)r.slot * kStage32;
                        mbar_arrive_expect_tx(&xfull[r.slot], kStage32);
                        tma_load_2d(dst, &mapA, &xfull[r.slot], kc * 64, m0 + g.a_off[tap]);
                        tma_load_2d(dst + kStage32 / 2, &mapA, &xfull[r.slot], kc * 64 + 32, m0 + g.a_off[tap]);
                    }
                    __syncwarp();
                    mbar_wait(&bempty[rb.slot], rb.phase ^ 1);
                    if (elect_one()) {
                        uint8_t *bs = bring + (size_t)rb.slot * bslot;
                        mbar_arrive_expect_tx(&bfull[rb.slot], bslot);
                        tma_load_2d(bs, &mapB, &bfull[rb.slot], kc * kBK16, g.b_off[tap] + n0);
                        tma_load_2d(bs + b_tile, &mapBlo, &bfull[rb.slot], kc * kBK16, g.b_off[tap] + n0);
                    }
                    rb.next();
                } else {
                    mbar_wait(&empty[r.slot], r.phase ^ 1);
                    if (i == i0 && lane == 0) BFTL(seq, tit, 0);
                    if (elect_one()) {
                        uint8_t *base = ops + (size_t)r.slot * slot_bytes;
                        mbar_arrive_expect_tx(&full[r.slot], 2 * kATile16 + 2 * b_tile);
                        tma_load_2d(base, &mapA, &full[r.slot], kc * kBK16, m0 + g.a_off[tap]);
                        tma_load_2d(base + half, &mapAlo, &full[r.slot], kc * kBK16, m0 + g.a_off[tap]);
                        tma_load_2d(base + kATile16, &mapB, &full[r.slot], kc * kBK16, g.b_off[tap] + n0);
                        tma_load_2d(base + half + kATile16, &mapBlo, &full[r.slot], kc * kBK16,
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
        const uint32_t idesc = idesc_bf16(kBM16, BN);
        const uint64_t da = sdesc_kmajor_sw128(smem_u32(ops));
        const uint64_t db = sdesc_kmajor_sw128(smem_u32(CONVERT ? bring : ops + kATile16));
        const uint32_t lo = half >> 4, blo = (CONVERT ? b_tile : half) >> 4;
        Ring r(CONVERT ? kXT : S), acc(2), rb(CONVERT ? SB : 1);
        int tit = 0;
        for (int u = cid; u < num_units; u += ncl, acc.next(), ++tit) {
            const int pc = u % GS;
            const int i0 = GS > 1 ? pc * iters / GS : ci0, i1 = GS > 1 ? (pc + 1) * iters / GS : ci1;
            mbar_wait(&tempty[acc.slot], acc.phase ^ 1);
            tc_fence_after();
            if (lane == 0) BFTL(seq, tit, 1);  // MMA: accumulator free
            const uint32_t d = tmem + acc.slot * ncols;
            for (int i = i0; i < i1; ++i, r.next()) {
                if (CONVERT) {
                    mbar_wait(&xt_full[r.slot], r.phase);
                    mbar_wait(&bfull[rb.slot], rb.phase);
                } else {
                    mbar_wait(&full[r.slot], r.phase);
                }
                tc_fence_after();
                if (i == i0 && lane == 0) BFTL(seq, tit, 2);  // MMA: operands ready
                if (elect_one()) {
                    const uint64_t b = db + (((CONVERT ? rb.slot * bslot : r.slot * slot_bytes)) >> 4);
                    if (CONVERT) {  // A = X hi (columns [0, 32)) / lo ([32, 64)) of TMEM slot r
                        const uint32_t xa = tmem + xt_base + r.slot * 64;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {  // K = 16 channels = 8 TMEM columns
                            mma_bf16_ts(d, xa + j * 8, b + j * 2, idesc, (i != i0) || (j != 0));
                            mma_bf16_ts(d, xa + j * 8, b + blo + j * 2, idesc, 1);  // hi * lo
                            mma_bf16_ts(d, xa + 32 + j * 8, b + j * 2, idesc, 1);   // lo * hi
                        }
                        mma_commit(&xt_empty[r.slot]);
                        mma_commit(&bempty[rb.slot]);
                    } else {
                        const uint64_t a = da + ((r.slot * slot_bytes) >> 4);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {  // K = 16 bf16 = 32 B per MMA
                            mma_bf16(d, a + j * 2, b + j * 2, idesc, (i != i0) || (j != 0));
                            mma_bf16(d, a + j * 2, b + blo + j * 2, idesc, 1);  // hi * lo
                            mma_bf16(d, a + lo + j * 2, b + j * 2, idesc, 1);   // lo * hi
                        }
                        mma_commit(&empty[r.slot]);
                    }
                }
                __syncwarp();
                if (lane == 0) BFK(seq, tit, i - i0, 3);
                if (CONVERT) rb.next();
            }
            if (elect_one()) mma_commit(&tfull[acc.slot]);
            __syncwarp();
            if (lane == 0) BFTL(seq, tit, 3);  // MMA: issued
        }
    } else if (warp < 6) {  // --------------------------------- epilogue
        const int q = warp & 3;
        const int NR = bf_yring(CONVERT, g.yring), LA = NR / 2;  // ring depth, residual lookahead
        float *scratch = epi_scratch + q * (OB ? 1024 : NR * 1024);
        // fp32 output ring (tma_y): chunk counter of this warp -> buffer and residual parity
        const bool ring = !OB && g.tma_y && (g.ldo & 3) == 0;
        const bool rres = ring && g.res && !TDC_DBG(g, 2);
        const uint32_t ring_s = smem_u32(scratch);
        uint32_t yc = 0;
        auto full_chunk = [&](int n) { return n + 32 <= g.Nn; };
        // TMA-load the residual block (columns n, rows r0..r0+31) into ring buffer of chunk k;
        // `pend` = TMA stores that may still be reading when the buffer's last store is done
        // `pend`: committed stores that may still be reading when this buffer's last one is done
        auto res_load = [&](uint32_t k, int n, int r0, int pend) {
            if (lane == 0) {
                bulk_wait_read_upto(pend);
                const uint32_t b = k % NR;
                mbar_arrive_expect_tx(&rbar[q * kYRing + b], 4096);
                tma_load_2d(scratch + b * 1024, &mapR, &rbar[q * kYRing + b], n, r0);
            }
        };
        Ring acc(2);
        int tit = 0;
        for (int u = cid; u < num_units; u += ncl, acc.next(), ++tit) {
            const int t = u / GS, pc = u - t * GS;
            const int m0 = (t % mtiles) * kBM16, n0 = (t / mtiles) * BN;
            // the tile's first residual block is in flight while the MMAs finish
            if (rres && (GS == 1 || pc == 0))
                for (int j = 0; j < LA && j * 32 < BN && full_chunk(n0 + 32 * j); ++j)
                    res_load(yc + j, n0 + 32 * j, m0 + q * 32, NR - 1 - j);
            mbar_wait(&tfull[acc.slot], acc.phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) BFTL(seq, tit, 4);  // epilogue: accumulator ready
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            if (CS > 1) {  // ---- split-K: partial -> own smem, reduce a row slice over the cluster
                const int row = q * 32 + lane, tid = row;
                const uint32_t red_a = smem_u32(red);
                const uint32_t tpar = (uint32_t)(tit & 1);
                mbar_wait_cluster(red_free, tpar ^ 1);  // peers done reading the previous partial
                for (int c = 0; c < BN; c += 32) {
                    uint32_t rr[32];
                    tmem_ld_32x32b_x32(src + c, rr);
                    tmem_ld_wait();
                    red_store_row32(red_a, BN, row, c, reinterpret_cast<const float *>(rr));
                }
                tc_fence_before();
                mbar_arrive_relaxed(&tempty[acc.slot]);
                fence_release_smem_cluster();
                red_signal(red_ready, CS);
                mbar_wait_cluster(red_ready, tpar);
                const int r0 = crank * 128 / CS, r1 = (crank + 1) * 128 / CS, nr = r1 - r0;
                const int g8 = BN / 8;
                for (int u = tid; u < nr * g8; u += 128) {
                    // bf16 planar output: consecutive threads take consecutive rows of one plane;
                    // fp32 row-major output: consecutive threads take consecutive columns of a row
                    const int rl = OB ? u % nr : u / g8, c8 = OB ? u / nr : u % g8;
                    const int rw = r0 + rl;
                    float v[8];
                    red_sum8(red_a, BN, CS, rw, c8, v);
                    long long dst_row = 0;
                    const bool valid = remap_row(g, m0 + rw, &dst_row);
                    const int n = n0 + 8 * c8;
                    if (!valid || n >= g.Nn) continue;
                    if (OB) {
                        uint4 h, l;
                        split_bf16x8(v, h, l);
                        const long long off = ((long long)(n >> 3) * g.planar_stride + dst_row) * 8;
                        *reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(g.out) + off) = h;
                        *reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(g.out_lo) + off) = l;
                    } else {
                        float *dst = g.out + dst_row * g.ldo + n;
                        epi_bias_res_relu<8>(v, n, g.Nn, g.bias, g.res ? g.res + dst_row * g.ldo : nullptr, g.relu);
                        if (n + 8 <= g.Nn && (g.ldo & 3) == 0) {
                            st_global_v4(dst, make_float4(v[0], v[1], v[2], v[3]));
                            st_global_v4(dst + 4, make_float4(v[4], v[5], v[6], v[7]));
                        } else {
                            _Pragma("unroll") for (int j = 0; j < 8; ++j) if (n + j < g.Nn) dst[j] = v[j];
                        }
                    }
                }
                red_signal(red_free, CS);
                if (warp == 2 && lane == 0) BFTL(seq, tit, 5);
                continue;
            }
            if (GS > 1 && pc > 0) {  // ---- split-K piece: fp32 partial -> L2 workspace
                float *slot = g.part + (size_t)(t * (GS - 1) + pc - 1) * 128 * BN;
                for (int c = 0; c < BN; c += 32) {
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(src + c, r);
                    tmem_ld_wait();
                    gs_store32(slot, c, q * 32 + lane, reinterpret_cast<const float *>(r));
                }
                tc_fence_before();
                mbar_arrive_relaxed(&tempty[acc.slot]);
                gs_publish(g.flags + t * (GS - 1) + pc - 1, warp == 2 && lane == 0);
                continue;
            }
            if (GS > 1)
                for (int pp = 1; pp < GS; ++pp) gs_wait(g.flags + t * (GS - 1) + pp - 1);
            long long dst_row = 0;
            const bool valid = remap_row(g, m0 + q * 32 + lane, &dst_row);
            for (int c = 0; c < BN; c += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(src + c, r);
                tmem_ld_wait();
                const int n = n0 + c;
                if (n >= g.Nn) continue;  // warp-uniform
                float v[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                for (int pp = 1; pp < GS; ++pp)  // partials in piece order (deterministic)
                    gs_add32(g.part + (size_t)(t * (GS - 1) + pp - 1) * 128 * BN, c, q * 32 + lane, v);
                if (OB) {  // X' hi/lo planar bf16: plane n/8 at (plane * stride + row) * 8
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
                } else if (ring && full_chunk(n)) {  // fp32 Y through the per-warp TMA ring
                    const uint32_t b = yc % NR, buf = ring_s + b * 4096;
                    const bool nxt = c + 32 * LA < BN && full_chunk(n + 32 * LA);
                    if (rres && nxt) res_load(yc + LA, n + 32 * LA, m0 + q * 32, NR - LA - 1);
                    else if (!rres && lane == 0) bulk_wait_read_upto(NR - 1);  // buffer b free
                    __syncwarp();
                    if (rres) {
                        mbar_wait(&rbar[q * kYRing + b], (yc / NR) & 1);
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4) {
                            const float4 f = ld_shared_v4(buf + (uint32_t)(lane * 128 + ((j4 ^ (lane & 7)) << 4)));
                            v[4 * j4] += f.x; v[4 * j4 + 1] += f.y; v[4 * j4 + 2] += f.z; v[4 * j4 + 3] += f.w;
                        }
                    }
                    epi_bias_res_relu<32>(v, n, g.Nn, g.bias, nullptr, g.relu);
                    if (!TDC_DBG(g, 1)) {
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4)
                            st_shared_v4(buf + (uint32_t)(lane * 128 + ((j4 ^ (lane & 7)) << 4)), v[4 * j4],
                                         v[4 * j4 + 1], v[4 * j4 + 2], v[4 * j4 + 3]);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&mapY, scratch + b * 1024, n, m0 + q * 32);
                            bulk_commit_group();
                        }
                    } else {
                        __syncwarp();
                        if (lane == 0) bulk_commit_group();  // keep the group count in step
                    }
                    ++yc;
                } else {  // fp32 Y (+bias, +residual, ReLU), row-major, coalesced through shared memory
                    const bool full = n + 32 <= g.Nn && (g.ldo & 3) == 0;
                    if (TDC_DBG(g, 1)) continue;
                    if (g.res && full && !TDC_DBG(g, 2)) {  // residual block read coalesced, then per-lane rows
                        float rv[32];
                        warp_load_block32(scratch, rv, valid ? g.res + dst_row * g.ldo + n : nullptr, lane);
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] += rv[j];
                        epi_bias_res_relu<32>(v, n, g.Nn, g.bias, nullptr, g.relu);
                    } else {
                        epi_bias_res_relu<32>(v, n, g.Nn, g.bias,
                                              (g.res && valid) ? g.res + dst_row * g.ldo : nullptr, g.relu);
                    }
                    float *dst = g.out + dst_row * g.ldo;
                    if (g.tma_y && full) {  // stage the 32x32 block (128B-swizzled box) and TMA-store it
                        const uint32_t sb = smem_u32(scratch);
                        if (lane == 0) bulk_wait_group_read0();  // this warp's previous block was read
                        __syncwarp();
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4)
                            st_shared_v4(sb + (uint32_t)(lane * 128 + ((j4 ^ (lane & 7)) << 4)), v[4 * j4],
                                         v[4 * j4 + 1], v[4 * j4 + 2], v[4 * j4 + 3]);
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            tma_store_2d(&mapY, scratch, n, m0 + q * 32);
                            bulk_commit_group();
                        }
                    } else if (n + 32 <= g.Nn && (g.ldo & 3) == 0) {
                        warp_store_block32(scratch, v, valid ? dst + n : nullptr, lane);
                    } else if (valid) {
                        _Pragma("unroll") for (int j = 0; j < 32; ++j) if (n + j < g.Nn) dst[n + j] = v[j];
                    }
                }
            }
            tc_fence_before();
            mbar_arrive_relaxed(&tempty[acc.slot]);
            if (GS > 1) {  // every epilogue thread has read the partials: clear the flags
                epi_bar128();
                if (warp == 2 && lane == 0)
                    for (int pp = 1; pp < GS; ++pp) g.flags[t * (GS - 1) + pp - 1] = 0;
            }
            if (warp == 2 && lane == 0) BFTL(seq, tit, 5);  // epilogue: done
        }
        if (g.tma_y && lane == 0) bulk_wait_group0();  // TMA stores complete before the CTA retires
        (void)res_load;
    } else if (CONVERT) {  // ----------------- converter: fp32 staging -> bf16 hi/lo in a TMEM slot
        // thread = (row, 32-channel half): row = this warp's TMEM lane quarter (warp % 4) x 32 +
        // lane, half = which 4 of the 8 converter warps; reads its 128 B of the fp32 box, writes
        // 16 hi and 16 lo columns (bf16 pairs) of the row's TMEM lane
        const int tid = threadIdx.x - 192;
        const int q = warp & 3, hf = tid >> 7, row = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        Ring rx(SX), xt(kXT);
        int tit = 0;
        for (int u = cid; u < num_units; u += ncl, ++tit) {
            const int pc = u % GS;
            const int i0 = GS > 1 ? pc * iters / GS : ci0, i1 = GS > 1 ? (pc + 1) * iters / GS : ci1;
            for (int i = i0; i < i1; ++i, rx.next(), xt.next()) {
                mbar_wait(&xfull[rx.slot], rx.phase);
                if (i == i0 && tid == 0) BFTL(seq, tit, 6);  // converter: X landed
                if (tid == 0) BFK(seq, tit, i - i0, 1);
                const uint32_t box = smem_u32(xstage + (size_t)rx.slot * kStage32) + (uint32_t)hf * (kStage32 / 2) +
                                     row * 128;
                float v[32];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 f = ld_shared_v4(box + ((j ^ (row & 7)) << 4));
                    v[4 * j] = f.x; v[4 * j + 1] = f.y; v[4 * j + 2] = f.z; v[4 * j + 3] = f.w;
                }
                mbar_arrive(&xempty[rx.slot]);  // the fp32 slot has been read: the next TMA may land
                uint32_t h[16], l[16];
#pragma unroll
                for (int g8 = 0; g8 < 4; ++g8) {
                    uint4 hh, ll;
                    split_bf16x8(v + 8 * g8, hh, ll);
                    h[4 * g8] = hh.x; h[4 * g8 + 1] = hh.y; h[4 * g8 + 2] = hh.z; h[4 * g8 + 3] = hh.w;
                    l[4 * g8] = ll.x; l[4 * g8 + 1] = ll.y; l[4 * g8 + 2] = ll.z; l[4 * g8 + 3] = ll.w;
                }
                mbar_wait(&xt_empty[xt.slot], xt.phase ^ 1);
                tc_fence_after();
                const uint32_t tx = tmem + lane_base + xt_base + xt.slot * 64;
                tmem_st_32x32b_x16(tx + 16 * hf, h);       // hi: channels 32hf.. -> columns 16hf..
                tmem_st_32x32b_x16(tx + 32 + 16 * hf, l);  // lo: columns 32 + 16hf..
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(&xt_full[xt.slot]);
                if (tid == 0) BFK(seq, tit, i - i0, 2);
                if (i == i1 - 1 && tid == 0) BFTL(seq, tit, 7);  // converter: done
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CS > 1) cluster_sync();  // no CTA leaves while a peer may still read its partial
    if (threadIdx.x == 0) BFGSPAN(seq, 2);
    if (warp == 1) tmem_dealloc(tmem, tcols);
#ifdef TDC_TIMELINE
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&g_tdc_bf_seq, 1u);
#endif
}

// xstages > 0 (converting stage 1): xstages fp32 staging slots, `stages` A slots and
// bstages weight slots; otherwise `stages` combined A|B slots.
int bf_smem_bytes(int BN, int stages, int xstages, int ksplit, int bstages, int fp32_out) {
    // fp32_out (converting GEMMs only): 0 = bf16 X' output, else the output ring depth (2 or 4)
    const int b_tile = BN * kBK16 * 2;
    // converting GEMMs: A is converted in place in the fp32 staging slots (stages == xstages)
    const int ops = xstages ? bstages * 2 * b_tile : stages * 2 * (kATile16 + b_tile);
    return 1024 + xstages * kStage32 + ops + bf_epi_bytes(xstages > 0, xstages > 0 && !fp32_out, fp32_out) +
           (ksplit > 1 ? 128 * BN * 4 : 0) +
           (3 * stages + 4 + 2 * xstages + 2 * bstages + 2 + 4 * kYRing + 2 * kXT) * 8 + 16;
}

// Ring depths: operand slots (and, for the converting stage 1, the fp32 staging and
// weight rings).
int bf_pick_stages(int BN, int max_smem, int convert, int *xstages, int ksplit, int *bstages, int fp32_out) {
    if (convert) {  // staging (= operand) ring first, then the weight ring
        static const int sx_max = std::getenv("TDC_GEMM_SX") ? std::atoi(std::getenv("TDC_GEMM_SX")) : 6;  // A/B knob
        int sx = sx_max < 2 ? 2 : (sx_max > 6 ? 6 : sx_max), sb = 4;
        while (sb > 2 && bf_smem_bytes(BN, sx, sx, ksplit, sb, fp32_out) > max_smem) --sb;
        while (sx > 2 && bf_smem_bytes(BN, sx, sx, ksplit, sb, fp32_out) > max_smem) --sx;
        if (xstages) *xstages = sx;
        if (bstages) *bstages = sb;
        return sx;
    }
    int s = 6, sx = 0, sb = 0;
    while (s > 2 && bf_smem_bytes(BN, s, sx, ksplit, sb, fp32_out) > max_smem) --s;
    if (xstages) *xstages = sx;
    if (bstages) *bstages = sb;
    return s;
}

cudaError_t bf_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapAlo, const CUtensorMap &mapB,
                           const CUtensorMap &mapBlo, const CUtensorMap &mapY, const TcGemmArgs &g, int grid,
                           cudaStream_t st, const CUtensorMap *mapR) {
    if (!mapR) mapR = &mapY;
    if (g.a_convert && g.BN > 128) return cudaErrorInvalidValue;  // TMEM: 2 accumulators + 2 X slots <= 512 columns
    const int smem = bf_smem_bytes(g.BN, g.stages, g.a_convert ? g.xstages : 0, g.ksplit, g.a_convert ? g.bstages : 0,
                                   g.out_bf16 ? 0 : bf_yring(true, g.yring));
    // the cluster split-K variant is a separate instantiation, so the default kernels carry
    // none of its code (smaller hot loops)
    auto go = [&](auto kernel, int threads) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl_cluster(kernel, grid, threads, smem, st, g.ksplit, mapA, mapAlo, mapB, mapBlo, mapY, *mapR,
                                  g);
    };
    const int ks = g.ksplit > 1 ? 1 : (g.gsplit > 1 ? 2 : 0);
    const int th = 192 + kConvThreads16;
    if (g.a_convert && g.out_bf16)  // stage 1
        return ks == 1 ? go(tdc_bf_gemm_kernel<true, 1, true>, th)
                       : (ks == 2 ? go(tdc_bf_gemm_kernel<true, 2, true>, th) : go(tdc_bf_gemm_kernel<true, 0, true>, th));
    if (g.a_convert)  // model dense convolutions (fp32 out)
        return ks == 1 ? go(tdc_bf_gemm_kernel<true, 1, false>, th)
                       : (ks == 2 ? go(tdc_bf_gemm_kernel<true, 2, false>, th)
                                  : go(tdc_bf_gemm_kernel<true, 0, false>, th));
    return ks == 1 ? go(tdc_bf_gemm_kernel<false, 1, false>, 192)
                   : (ks == 2 ? go(tdc_bf_gemm_kernel<false, 2, false>, 192)
                              : go(tdc_bf_gemm_kernel<false, 0, false>, 192));
}

// ============================================================ core conv (stage 2)
// Per tile (128 phase-grid rows x BN output channels) and 32-channel chunk kc: the
// X' band (hi and lo, every phase the taps use) arrives as 8*nphase plane copies
// issued from different producer lanes (the TMA engine overlaps copies from
// different threads; one thread's copies are ~100-200 cycles apart);
// the weights arrive as one large copy per (kc, tap group) -- or stay resident for
// the CTA's lifetime when they fit -- and every tap is a row-shifted descriptor.
__host__ __device__ inline uint32_t bf_core_a_half(int nphase, int band_rows) {
    return (uint32_t)nphase * 4 * band_rows * 16;  // 4 planes of 8 bf16 channels per chunk
}

int bf_core_smem_bytes(int BN, int nphase, int band_rows, int tg, int w_slots, int ksplit) {
    return 1024 + 2 * 2 * (int)bf_core_a_half(nphase, band_rows) + w_slots * tg * BN * 128 + kEpiScratch16 +
           (ksplit > 1 ? 128 * BN * 4 : 0) + (10 + 2 * w_slots) * 8 + 16;
}

__host__ __device__ inline int bf_pow2_cols(int c) {
    int n = 32;
    while (n < c) n *= 2;
    return n;
}
// Fused variant: + two Z hi|lo tile buffers [BN/8 planes][128 rows][16 B] x 2 and the
// resident U_out hi|lo panel [BN/8 planes][2*N3p rows][16 B], + 9 barriers.
__host__ __device__ inline int bf_core3_zbuf(const BfCoreArgs &g) { return (g.BN / 8) * 128 * 16 * 2; }
__host__ __device__ inline int bf_core3_w3(const BfCoreArgs &g) { return (g.BN / 8) * 2 * g.N3p * 16; }
// + the second epilogue-3 warp group's transpose scratch (kEpiScratch16)
int bf_core3_smem_bytes(const BfCoreArgs &g) {
    return bf_core_smem_bytes(g.BN, g.nphase, g.band_rows, g.tg, g.w_slots, 1) + 2 * bf_core3_zbuf(g) +
           bf_core3_w3(g) + kEpiScratch16 + 9 * 8;
}
__host__ __device__ inline int bf_core3_tmem(const BfCoreArgs &g) {
    const int a2 = bf_pow2_cols(g.ncat ? 2 * g.BN : g.BN), a3 = bf_pow2_cols(g.ncat3 ? 2 * g.N3p : g.N3p);
    return bf_pow2_cols(2 * a2 + 2 * a3);
}
int bf_core3_tmem_cols(const BfCoreArgs &g) { return bf_core3_tmem(g); }

// F3 = false: stage 2 alone, Z hi/lo to global (the 3-launch path).
// F3 = true:  stage 2 + stage 3 in one kernel ("core3"): the Z tile is split into
// bf16 hi/lo by the epilogue-2 warps straight into shared memory, stage 3 multiplies
// it with the resident U_out panel, epilogue-3 warps write Y (+bias).  Z never
// touches HBM.  MMA issue is software-pipelined: S2(tile i) then S3(tile i-1).
// KS: 0 plain, 1 cluster split-K, 2 split-K through L2 (stage 2 alone); RES: the fused
// stage-3 epilogue adds a residual (model path) -- compiled only where used.
template <bool F3, int KS, bool RES>
// F3: 14 warps -- epilogue 3 is split over two groups of four warps (each stores half of the
// output columns), as the Y stores were the fused kernel's slowest stage
__global__ void __launch_bounds__(F3 ? 448 : 192, 1) tdc_bf_core_kernel(const BfCoreArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int BN = g.BN, WS = g.w_slots, TG = g.tg;
    const uint32_t band_bytes = (uint32_t)g.band_rows * 16;
    const uint32_t a_half = bf_core_a_half(g.nphase, g.band_rows);
    const uint32_t a_bytes = 2 * a_half;
    const uint32_t w_tap = (uint32_t)BN * 128;  // [4 planes][2BN rows][16 B]
    const uint32_t w_slot = (uint32_t)TG * w_tap;
    const uint32_t zbuf = F3 ? (uint32_t)bf_core3_zbuf(g) : 0u, zhalf = zbuf / 2;
    const uint32_t w3_bytes = F3 ? (uint32_t)bf_core3_w3(g) : 0u;
    uint8_t *a_slots = smem;
    uint8_t *w_slots = smem + 2 * (size_t)a_bytes;
    float *epi_scratch = reinterpret_cast<float *>(w_slots + (size_t)WS * w_slot);
    uint8_t *zs = reinterpret_cast<uint8_t *>(epi_scratch) + (F3 ? 2 : 1) * kEpiScratch16;  // F3: 2 Z buffers
    const int CS = (!F3 && KS == 1 && g.ksplit > 1) ? g.ksplit : 1;           // split-K cluster size
    float *red = reinterpret_cast<float *>(zs);                              // split-K partial [128][BN]
    const uint32_t red_bytes = CS > 1 ? (uint32_t)128 * BN * 4 : 0u;
    uint8_t *w3s = zs + 2 * (size_t)zbuf + red_bytes;                        // F3: U_out panel
    uint64_t *a_full = reinterpret_cast<uint64_t *>(w3s + w3_bytes);
    uint64_t *a_empty = a_full + 2;
    uint64_t *tfull = a_empty + 2;
    uint64_t *tempty = tfull + 2;
    uint64_t *w_full = tempty + 2;
    uint64_t *w_empty = w_full + WS;
    uint64_t *red_ready = w_empty + WS;  // split-K handshake
    uint64_t *red_free = red_ready + 1;
    uint64_t *z_full = red_free + 1;   // F3 only from here on
    uint64_t *z_empty = z_full + 2;
    uint64_t *t3full = z_empty + 2;
    uint64_t *t3empty = t3full + 2;
    uint64_t *w3_full = t3empty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(F3 ? w3_full + 1 : z_full);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int acc_cols = g.ncat ? 2 * BN : BN;
    const uint32_t ncols = bf_pow2_cols(acc_cols);                      // one acc2 buffer
    const uint32_t ncols3 = F3 ? bf_pow2_cols(g.ncat3 ? 2 * g.N3p : g.N3p) : 0u;
    const uint32_t tcols = F3 ? (uint32_t)bf_core3_tmem(g) : 2 * ncols;
    const int mtiles = (g.M + kBM16 - 1) / kBM16;
    const int num_tiles = mtiles * g.ntiles;
    const bool resident = g.w_resident != 0;
    const int crank = CS > 1 ? (int)cluster_ctarank() : 0;
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;                 // cluster id / count
    const int ck0 = crank * g.kchunks / CS, ck1 = (crank + 1) * g.kchunks / CS;  // cluster split: chunks
    const int GS = (!F3 && KS == 2 && g.gsplit > 1) ? g.gsplit : 1;                // split-K through L2
    const int num_units = num_tiles * GS;

    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128);
            if (F3) {
                mbar_init(&z_full[i], 128);
                mbar_init(&z_empty[i], 1);
                mbar_init(&t3full[i], 1);
                mbar_init(&t3empty[i], 256);  // both epilogue-3 warp groups
            }
        }
        for (int i = 0; i < WS; ++i) {
            mbar_init(&w_full[i], 1);
            mbar_init(&w_empty[i], 1);
        }
        if (F3) mbar_init(w3_full, 1);
        mbar_init(red_ready, CS * 128);
        mbar_init(red_free, CS * 128);
        fence_mbar_init();
    }
    if (threadIdx.x == 0) BFCSPAN(0);
    if (warp == 1) tmem_alloc(tmem_slot, tcols);
    tc_fence_before();
    __syncthreads();
    if (CS > 1) cluster_sync();  // peers' barriers initialised before any remote arrive
    tc_fence_after();
    // pdl_wait() is taken by the producer alone, after it has issued the plan-owned weight
    // loads: every other role only consumes what the producer's loads bring in.
    pdl_launch_dependents();
    if (threadIdx.x == 0) BFCSPAN(1);
    const uint32_t tmem = *tmem_slot;

    // phase-grid row m -> compact output row (b, oy, ox), or invalid
    auto out_row = [&](int m, long long *dst_row) {
        if (m >= g.M) return false;
        const int ox = m % g.Wq;
        const int tt = m / g.Wq;
        const int oy = tt % g.Hq;
        const int b = tt / g.Hq;
        *dst_row = ((long long)b * g.Ho + oy) * g.Wo + ox;
        return oy < g.Ho && ox < g.Wo;
    };

    if (warp == 0) {  // ---------------------------------- bulk-copy producer
        const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(g.w);
        // copy `bytes` to smem in <= 16 KB pieces issued from different lanes
        auto load_split = [&](uint8_t *dst, const uint8_t *src, uint32_t bytes, uint64_t *bar) {
            if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
            __syncwarp();
            const uint32_t piece = 16384;
            for (uint32_t o = (uint32_t)lane * piece; o < bytes; o += 32 * piece)
                bulk_load(dst + o, src + o, bytes - o < piece ? bytes - o : piece, bar);
            __syncwarp();
        };
        if (F3) load_split(w3s, reinterpret_cast<const uint8_t *>(g.w3), w3_bytes, w3_full);
        if (resident)  // ntiles == 1: every (kc, group) slice once, for the CTA's lifetime
            for (int i = 0; i < WS; ++i)
                load_split(w_slots + (size_t)i * w_slot, wsrc + (size_t)i * w_slot, w_slot, &w_full[i]);
        pdl_wait();  // X' is written by the previous kernel (stage 1)
        Ring ra(2), rw(WS);
        int tit = 0;
        for (int u = cid; u < num_units; u += ncl, ++tit) {
            const int t = u / GS, pc = u - t * GS;
            const int k0 = GS > 1 ? pc * g.kchunks / GS : ck0, k1 = GS > 1 ? (pc + 1) * g.kchunks / GS : ck1;
            const int m0 = (t % mtiles) * kBM16, nt = t / mtiles;
            for (int kc = k0; kc < k1; ++kc, ra.next()) {
                if (!TDC_DBG(g, 1024) || tit < 2) mbar_wait_sleep(&a_empty[ra.slot], ra.phase ^ 1);
                if (kc == k0 && lane == 0) BFCTL(tit, 0);  // producer: band issue
                const bool stale = TDC_DBG(g, 4) && tit >= 2;  // debug: keep the stale band
                if (lane == 0) mbar_arrive_expect_tx(&a_full[ra.slot], stale ? 0u : a_bytes);
                __syncwarp();
                uint8_t *dst = a_slots + (size_t)ra.slot * a_bytes;
                for (int c = stale ? 32 * 64 : lane; c < g.nphase * 8; c += 32) {  // (phase, plane, hi/lo)
                    const int ph = c >> 3, kg = (c >> 1) & 3, lo = c & 1;
                    const long long off =
                        ((long long)(kc * 4 + kg) * g.plane_rows + (long long)g.phase_src[ph] * g.phase_rows + m0) * 8;
                    bulk_load(dst + lo * a_half + (size_t)(ph * 4 + kg) * band_bytes, (lo ? g.xg_lo : g.xg) + off,
                              band_bytes, &a_full[ra.slot]);
                }
                __syncwarp();
                if (!resident)
                    for (int grp = 0; grp < g.ngroups; ++grp, rw.next()) {
                        mbar_wait(&w_empty[rw.slot], rw.phase ^ 1);
                        if (tit == 0 && lane == 0) BFCTAP(kc * g.ngroups + grp, 0);
                        const long long slice = ((long long)kc * g.ntiles + nt) * g.ngroups + grp;
                        load_split(w_slots + (size_t)rw.slot * w_slot, wsrc + slice * w_slot, w_slot,
                                   &w_full[rw.slot]);
                    }
            }
        }
    } else if (warp == 1) {  // ------------------------------ MMA issuer
        const uint32_t idesc = idesc_bf16(kBM16, acc_cols);
        // ncat: X' lo x C hi alone (N = BN: 48 instead of 64 cycles per MMA at BN = 64, and 2 KB
        // less B traffic) -- the lo x lo product of an N = 2*BN MMA is below the split's error
        const uint32_t idesc_h = idesc_bf16(kBM16, BN);
        const uint64_t da = sdesc_kmajor_none(smem_u32(a_slots), band_bytes, 128);
        const uint64_t db = sdesc_kmajor_none(smem_u32(w_slots), 2 * BN * 16, 128);
        const uint32_t a_lo = a_half >> 4, b_lo = (BN * 16) >> 4;
        // stage 3 (F3): A = Z tile planar [plane][128][16 B], B = U_out [plane][2*N3p][16 B]
        const uint32_t id3 = F3 ? idesc_bf16(kBM16, g.ncat3 ? 2 * g.N3p : g.N3p) : 0u;
        const uint64_t dz = sdesc_kmajor_none(smem_u32(zs), 128 * 16, 128);
        const uint64_t dw3 = sdesc_kmajor_none(smem_u32(w3s), 2 * g.N3p * 16, 128);
        const uint32_t z_lo = zhalf >> 4, b3_lo = (g.N3p * 16) >> 4;
        const int k3 = BN / 16;
        // Per-tap A start offsets (16-byte units, relative to a band slot), hoisted out of
        // the tile loop: with the 3x3 core (one group of 9 taps) the tap loop below is
        // fully unrolled, so each MMA costs one uniform add -- the issuing thread must
        // keep up with ~48-cycle MMAs.
        const uint32_t wtap16 = w_tap >> 4, plane2a = (2 * band_bytes) >> 4, plane2b = (2 * 2 * BN * 16) >> 4;
        Ring ra(2), rw(WS), acc(2), zr(2), a3(2);
        int tit = 0;
        bool pending = false;  // F3: S3 of the previous tile still to issue
        if (F3) mbar_wait(w3_full, 0);
        for (int u = cid;; u += ncl, ++tit) {
            const bool have = u < num_units;
            const int pc = u % GS;
            const int k0 = GS > 1 ? pc * g.kchunks / GS : ck0, k1 = GS > 1 ? (pc + 1) * g.kchunks / GS : ck1;
            if (have) {
                if (!TDC_DBG(g, 16)) mbar_wait(&tempty[acc.slot], acc.phase ^ 1);
                tc_fence_after();
                if (lane == 0) BFCTL(tit, 1);  // MMA: accumulator free
                const uint32_t d = tmem + acc.slot * ncols;
                uint32_t accum = 0;
                for (int kc = k0; kc < k1; ++kc, ra.next()) {
                    if (!TDC_DBG(g, 512) || tit == 0) mbar_wait(&a_full[ra.slot], ra.phase);  // dbg 512: stale bands
                    if (kc == k0 && lane == 0) BFCTL(tit, 2);  // MMA: band landed
                    for (int grp = 0; grp < g.ngroups; ++grp) {
                        int ws;
                        if (resident) {
                            ws = kc * g.ngroups + grp;
                            if (!TDC_DBG(g, 1024) || tit == 0) mbar_wait(&w_full[ws], 0);
                        } else {
                            ws = rw.slot;
                            mbar_wait(&w_full[ws], rw.phase);
                        }
                        tc_fence_after();
                        if (tit == 0 && lane == 0) BFCTAP(kc * g.ngroups + grp, 1);
                        if (TG == 9 && g.ngroups == 1) {  // 3x3 core: fully unrolled taps
                            // Descriptor bases computed in converged code from warp-uniform values
                            // (kernel parameters, ring cursors) so they live in uniform registers;
                            // the hi|lo concatenation branch is hoisted out of the stream.  The tap
                            // loop stays rolled: the fully unrolled stream measured slower (code
                            // size).
                            const uint64_t aslot = da + ((ra.slot * a_bytes) >> 4);
                            const uint64_t bslot = db + ((ws * w_slot) >> 4);
                            auto stream = [&](auto ncat) {
                                if (elect_one()) {
#pragma unroll 1
                                    for (int tt = 0; tt < 9; ++tt) {
                                        const uint64_t a = aslot + (((uint32_t)g.tap_phase[tt] * 4 * band_bytes +
                                                                     (uint32_t)g.tap_off[tt] * 16) >> 4);
                                        const uint64_t b = bslot + tt * wtap16;
#pragma unroll
                                        for (int j = 0; j < 2; ++j) {
                                            const uint64_t aj = a + j * plane2a, bj = b + j * plane2b;
                                            mma_bf16(d, aj, bj, idesc, accum);
                                            if (decltype(ncat)::value) {
                                                mma_bf16(d, aj + a_lo, bj, idesc_h, 1);
                                            } else {
                                                mma_bf16(d, aj, bj + b_lo, idesc, 1);
                                                mma_bf16(d, aj + a_lo, bj, idesc, 1);
                                            }
                                            accum = 1;
                                        }
                                    }
                                    if (!resident) mma_commit(&w_empty[ws]);
                                }
                            };
                            if (g.ncat) stream(std::integral_constant<bool, true>());
                            else stream(std::integral_constant<bool, false>());
                        } else if (elect_one()) {
                            for (int tt = 0; tt < TG; ++tt) {
                                const int tap = grp * TG + tt;
                                const uint64_t a =
                                    da + ((ra.slot * a_bytes + (uint32_t)g.tap_phase[tap] * 4 * band_bytes +
                                           (uint32_t)g.tap_off[tap] * 16) >> 4);
                                const uint64_t b = db + ((ws * w_slot + tt * w_tap) >> 4);
#pragma unroll
                                for (int j = 0; j < 2; ++j) {  // K = 16 = two 8-channel planes
                                    const uint64_t aj = a + ((j * 2 * band_bytes) >> 4);
                                    const uint64_t bj = b + ((j * 2 * 2 * BN * 16) >> 4);
                                    if (g.ncat) {  // [hi | lo] along N: hi*hi, hi*lo | lo*hi
                                        mma_bf16(d, aj, bj, idesc, accum);
                                        mma_bf16(d, aj + a_lo, bj, idesc_h, 1);
                                    } else {
                                        mma_bf16(d, aj, bj, idesc, accum);
                                        mma_bf16(d, aj, bj + b_lo, idesc, 1);
                                        mma_bf16(d, aj + a_lo, bj, idesc, 1);
                                    }
                                    accum = 1;
                                }
                            }
                            if (!resident) mma_commit(&w_empty[ws]);
                        }
                        __syncwarp();
                        accum = 1;
                        if (!resident) rw.next();
                    }
                    if (!TDC_DBG(g, 1024) && elect_one()) mma_commit(&a_empty[ra.slot]);  // dbg 1024: none
                    __syncwarp();
                }
                if (elect_one()) mma_commit(&tfull[acc.slot]);
                __syncwarp();
                acc.next();
                if (lane == 0) BFCTL(tit, 3);  // MMA: all issued
            }
            if (F3 && pending && !TDC_DBG(g, 256)) {  // ---- stage 3 of the previous tile (dbg 256: none)
                mbar_wait(&t3empty[a3.slot], a3.phase ^ 1);
                if (lane == 0) BFCTL(tit - 1, 6);  // S3: acc3 buffer free
                mbar_wait(&z_full[zr.slot], zr.phase);
                tc_fence_after();
                if (lane == 0) BFCTL(tit - 1, 7);  // S3: Z ready, issuing
                if (elect_one()) {
                    const uint32_t d3 = tmem + 2 * ncols + a3.slot * ncols3;
                    if (TDC_DBG(g, 8)) {  // debug: no stage-3 MMAs
                        mma_commit(&z_empty[zr.slot]);
                        mma_commit(&t3full[a3.slot]);
                    } else {
                    const uint64_t az = dz + ((zr.slot * zbuf) >> 4);
                    for (int j = 0; j < k3; ++j) {
                        const uint64_t aj = az + ((j * 2 * 128 * 16) >> 4);
                        const uint64_t bj = dw3 + ((j * 2 * 2 * g.N3p * 16) >> 4);
                        if (g.ncat3) {
                            mma_bf16(d3, aj, bj, id3, j > 0);
                            mma_bf16(d3, aj + z_lo, bj, id3, 1);
                        } else {
                            mma_bf16(d3, aj, bj, id3, j > 0);
                            mma_bf16(d3, aj, bj + b3_lo, id3, 1);
                            mma_bf16(d3, aj + z_lo, bj, id3, 1);
                        }
                    }
                    mma_commit(&z_empty[zr.slot]);
                    mma_commit(&t3full[a3.slot]);
                    }
                }
                __syncwarp();
                zr.next();
                a3.next();
            }
            if (!have) break;
            pending = true;
        }
    } else if (warp < 6) {  // ------------------ epilogue warps 2..5: acc2 -> Z hi/lo bf16
        const int q = warp & 3;
        float *scratch = epi_scratch + q * 1024;
        __nv_bfloat16 *z = reinterpret_cast<__nv_bfloat16 *>(g.z);
        __nv_bfloat16 *z_lo = reinterpret_cast<__nv_bfloat16 *>(g.z_lo);
        const int r = q * 32 + lane;  // tile row = TMEM lane
        Ring acc(2), zr(2);
        int tit = 0;
        for (int u = cid; u < num_units; u += ncl, acc.next(), zr.next(), ++tit) {
            const int t = u / GS, pc = u - t * GS;
            const int m0 = (t % mtiles) * kBM16, n0 = (t / mtiles) * BN;
            mbar_wait_sleep(&tfull[acc.slot], acc.phase);
            tc_fence_after();
            if (warp == 2 && lane == 0) BFCTL(tit, 4);  // epilogue: accumulator ready
            if (!F3 && CS > 1) {  // ---- split-K: partial -> own smem, reduce a row slice
                const uint32_t red_a = smem_u32(red), tpar = (uint32_t)(tit & 1);
                const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
                mbar_wait_cluster(red_free, tpar ^ 1);
                for (int c = 0; c < BN; c += 32) {
                    uint32_t rr[32];
                    float v[32];
                    tmem_ld_32x32b_x32(src + c, rr);
                    if (g.ncat) {
                        uint32_t r2[32];
                        tmem_ld_32x32b_x32(src + BN + c, r2);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]) + __uint_as_float(r2[j]);
                    } else {
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
                    }
                    red_store_row32(red_a, BN, r, c, v);
                }
                tc_fence_before();
                mbar_arrive_relaxed(&tempty[acc.slot]);
                fence_release_smem_cluster();
                red_signal(red_ready, CS);
                mbar_wait_cluster(red_ready, tpar);
                const int r0 = crank * 128 / CS, r1 = (crank + 1) * 128 / CS, nr = r1 - r0, g8 = BN / 8;
                for (int u = r; u < nr * g8; u += 128) {  // Z row-major: threads along columns
                    const int rw = r0 + u / g8, c8 = u % g8;
                    float v[8];
                    red_sum8(red_a, BN, CS, rw, c8, v);
                    long long dr = 0;
                    const int n = n0 + 8 * c8;
                    if (!out_row(m0 + rw, &dr) || n >= g.Nn) continue;
                    uint4 h, l;
                    split_bf16x8(v, h, l);
                    *reinterpret_cast<uint4 *>(z + dr * g.ldz + n) = h;
                    *reinterpret_cast<uint4 *>(z_lo + dr * g.ldz + n) = l;
                }
                red_signal(red_free, CS);
                continue;
            }
            long long dst_row = 0;
            const bool valid = out_row(m0 + r, &dst_row);
            if (F3 && !TDC_DBG(g, 256)) mbar_wait_sleep(&z_empty[zr.slot], zr.phase ^ 1);
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            const uint32_t zb = smem_u32(zs) + zr.slot * zbuf;
            const bool gpart = GS > 1 && pc > 0;  // split-K piece: fp32 partial -> L2 workspace
            if (GS > 1 && pc == 0)
                for (int pp = 1; pp < GS; ++pp) gs_wait(g.flags + t * (GS - 1) + pp - 1);
            for (int c = 0; c < (TDC_DBG(g, 32) ? 0 : BN); c += 32) {
                uint32_t rr[32];
                float v[32];
                tmem_ld_32x32b_x32(src + c, rr);
                if (g.ncat) {
                    uint32_t r2[32];
                    tmem_ld_32x32b_x32(src + BN + c, r2);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]) + __uint_as_float(r2[j]);
                } else {
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
                }
                if (gpart) {
                    gs_store32(g.part + (size_t)(t * (GS - 1) + pc - 1) * 128 * BN, c, r, v);
                    continue;
                }
                for (int pp = 1; pp < GS; ++pp)  // partials in piece order (deterministic)
                    gs_add32(g.part + (size_t)(t * (GS - 1) + pp - 1) * 128 * BN, c, r, v);
                if (F3 && TDC_DBG(g, 2)) {
                } else if (F3) {  // Z hi/lo planes [c/8 + pl][row r][16 B] (conflict-free: lanes = rows)
#pragma unroll
                    for (int pl = 0; pl < 4; ++pl) {
                        uint4 h, l;
                        split_bf16x8(v + 8 * pl, h, l);
                        const uint32_t o = ((uint32_t)(c / 8 + pl) * 128 + r) * 16;
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + o), "r"(h.x), "r"(h.y),
                                     "r"(h.z), "r"(h.w)
                                     : "memory");
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(zb + zhalf + o), "r"(l.x),
                                     "r"(l.y), "r"(l.z), "r"(l.w)
                                     : "memory");
                    }
                } else {
                    if (n0 + c >= g.Nn) continue;  // warp-uniform
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
            }
            tc_fence_before();
            mbar_arrive_relaxed(&tempty[acc.slot]);
            if (gpart) {
                gs_publish(g.flags + t * (GS - 1) + pc - 1, warp == 2 && lane == 0);
            } else if (GS > 1) {  // every epilogue thread has read the partials: clear the flags
                epi_bar128();
                if (warp == 2 && lane == 0)
                    for (int pp = 1; pp < GS; ++pp) g.flags[t * (GS - 1) + pp - 1] = 0;
            }
            if (F3) {
                fence_proxy_async_smem();  // Z (generic writes) -> visible to the MMA (async proxy)
                mbar_arrive(&z_full[zr.slot]);
            }
            if (warp == 2 && lane == 0) BFCTL(tit, 5);  // epilogue: done
        }
    } else if (F3) {  // ------------------------- epilogue warps 6..13: acc3 (+bias) -> Y
        const int q = warp & 3, grp = (warp - 6) >> 2;  // group 0: warps 6-9, group 1: warps 10-13
        float *scratch = epi_scratch + (warp - 6) * 1024;
        const int chalf = ((g.N3p / 32 + 1) / 2) * 32;  // output columns per group (whole 32-column chunks)
        Ring a3(2);
        int tit = 0;
        for (int t = TDC_DBG(g, 256) ? num_tiles : cid; t < num_tiles; t += ncl, a3.next(), ++tit) {
            const int m0 = (t % mtiles) * kBM16;
            mbar_wait_sleep(&t3full[a3.slot], a3.phase);
            tc_fence_after();
            if (warp == 6 && lane == 0) BFCTL(tit, 8);  // E3: acc3 ready
            long long dst_row = 0;
            const bool valid = out_row(m0 + q * 32 + lane, &dst_row);
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + 2 * ncols + a3.slot * ncols3;
            float *dst = g.y + dst_row * g.N3;
            const int c_end = (grp + 1) * chalf < g.N3p ? (grp + 1) * chalf : g.N3p;
            for (int c = grp * chalf; c < (TDC_DBG(g, 64) ? 0 : c_end); c += 32) {  // dbg 64: no E3 TMEM loads
                uint32_t rr[32];
                float v[32];
                tmem_ld_32x32b_x32(src + c, rr);
                if (g.ncat3) {
                    uint32_t r2[32];
                    tmem_ld_32x32b_x32(src + g.N3p + c, r2);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]) + __uint_as_float(r2[j]);
                } else {
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]);
                }
                if (c >= g.N3 || TDC_DBG(g, 1)) continue;  // warp-uniform
                if (RES && g.res && c + 32 <= g.N3 && (g.N3 & 3) == 0) {  // coalesced residual block
                    float rv[32];
                    warp_load_block32(scratch, rv, valid ? g.res + dst_row * g.N3 + c : nullptr, lane);
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] += rv[j];
                    epi_bias_res_relu<32>(v, c, g.N3, g.bias, nullptr, g.relu);
                } else {
                    epi_bias_res_relu<32>(v, c, g.N3, g.bias, (RES && g.res && valid) ? g.res + dst_row * g.N3 : nullptr,
                                          g.relu);
                }
                if (c + 32 <= g.N3 && (g.N3 & 3) == 0) {
                    if (TDC_YDIRECT(g)) {  // each lane stores its own row: no shared-memory traffic
                        if (valid)
#pragma unroll
                            for (int j = 0; j < 8; ++j)
                                st_global_v4(dst + c + 4 * j, make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2],
                                                                          v[4 * j + 3]));
                    } else {
                        warp_store_block32(scratch, v, valid ? dst + c : nullptr, lane);
                    }
                } else if (valid) {
                    _Pragma("unroll") for (int j = 0; j < 32; ++j) if (c + j < g.N3) dst[c + j] = v[j];
                }
            }
            tc_fence_before();
            mbar_arrive_relaxed(&t3empty[a3.slot]);
            if (warp == 6 && lane == 0) BFCTL(tit, 9);  // E3: Y stored
        }
    }
    tc_fence_before();
    __syncthreads();
    if (CS > 1) cluster_sync();  // no CTA leaves while a peer may still read its partial
    if (threadIdx.x == 0) BFCSPAN(2);
    if (warp == 1) tmem_dealloc(tmem, tcols);
}

// ============================================================ core conv, CTA pair
// Stage 2 alone on a CTA PAIR (cta_group::2, M = 256): the two CTAs of a cluster run the M
// tiles 2p and 2p + 1 of the same N tile, and the leader issues every MMA for both.  B (the
// core weights, N = 2*BN = [hi | lo]) is split along N between the pair: CTA 0 holds the hi
// rows of each (chunk, tap, plane), CTA 1 the lo rows, so each SM streams HALF of the weight
// slice per 32-channel chunk while its tensor core does the same MMA work -- the deep layers'
// core kernels are bound by that per-SM weight streaming (~40-60 GB/s per SM measured;
// DESIGN.md §8, §7d).  A (the X' band) is per CTA: each loads its own tile's band.
// Hand-offs: each CTA's producer signals its own full barriers; the peer's idle MMA warp
// relays "peer slot full" to the leader (remote arrive); the leader's commits are
// multicast to both CTAs' empty / accumulator-full barriers; the peer's epilogue releases
// the accumulator on the leader's barrier.  3x3 core (9 taps in one weight slice), streamed
// weights, Z hi/lo to global like tdc_bf_core_kernel<false, 0, false>.
// per (chunk, N tile) and CTA: [tap][plane][BN rows: own half of [C hi | C lo]] followed by
// [tap][plane][BN/2 rows: this CTA's half of C hi] (the B of the X' lo x C hi MMA, N = BN)
__host__ __device__ inline uint32_t bf_core2_wslot(int BN) { return 9u * 4u * (uint32_t)(BN + BN / 2) * 16u; }
// a_slots: band ring depth (2 or 3: the MMAs of chunk k+2 cannot start before chunk k's band slot is
// free, so a third slot keeps the producer ahead when the weights leave room for it)
int bf_core2_smem_bytes(int BN, int nphase, int band_rows, int w_slots, int a_slots) {
    return 1024 + a_slots * 2 * (int)bf_core_a_half(nphase, band_rows) + w_slots * (int)bf_core2_wslot(BN) +
           kEpiScratch16 + (13 + 3 * w_slots) * 8 + 16;
}

__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// commit the leader's MMAs to the barrier at this smem offset in BOTH CTAs of the pair
__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)3)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote_release(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_acq_cluster(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAITQ_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAITQ_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

#ifdef TDC_TIMELINE
// Debug build only: per-chunk events of the first unit of CTA pair 0 (scripts/core2_timeline.py):
// [kc][0] producer issues the weight half (leader), [1] leader sees its weights, [2] leader sees
// the peer's weights, [3] leader has issued the chunk's MMAs, [4] peer producer issue
__device__ unsigned long long g_tdc_c2tl[64 * 8];
extern "C" int tdc_debug_core2_timeline(unsigned long long *host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_tdc_c2tl, sizeof(unsigned long long) * n);
}
#define C2TL(kc, ev)                                                                         \
    do {                                                                                     \
        if (blockIdx.x < 2 && (kc) < 64) {                                                   \
            unsigned long long v_;                                                           \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_));                           \
            g_tdc_c2tl[(kc) * 8 + (ev)] = v_;                                                \
        }                                                                                    \
    } while (0)
#else
#define C2TL(kc, ev) ((void)0)
#endif
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1) tdc_bf_core2_kernel(const BfCoreArgs g) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int BN = g.BN, WS = g.w_slots, AS = g.a_slots;
    const uint32_t band_bytes = (uint32_t)g.band_rows * 16;
    const uint32_t a_half = bf_core_a_half(g.nphase, g.band_rows), a_bytes = 2 * a_half;
    const uint32_t w_slot = bf_core2_wslot(BN), w_tap = (uint32_t)BN * 64;  // [tap][4 planes][BN rows][16 B]
    const uint32_t w_extra = 9u * w_tap, x_tap = (uint32_t)BN * 32;        // then [tap][4 planes][BN/2][16 B]
    uint8_t *a_slots = smem;
    uint8_t *w_slots = smem + (size_t)AS * a_bytes;
    float *epi_scratch = reinterpret_cast<float *>(w_slots + (size_t)WS * w_slot);
    uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(epi_scratch) + kEpiScratch16);
    uint64_t *a_full = bars, *a_empty = bars + 3, *a_peer = bars + 6, *tfull = bars + 9, *tempty = bars + 11;
    uint64_t *w_full = bars + 13, *w_empty = w_full + WS, *w_peer = w_empty + WS;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(w_peer + WS);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int ncols = 2 * BN;  // one accumulator buffer: [hi-weight products | lo-weight products]
    uint32_t tcols = 32;
    while ((int)tcols < 2 * ncols) tcols *= 2;
    const int mtiles = (g.M + kBM16 - 1) / kBM16, mpairs = (mtiles + 1) / 2;
    const int num_units = mpairs * g.ntiles;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (threadIdx.x == 0) {
        for (int i = 0; i < AS; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], 1);
            mbar_init(&a_peer[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 128 + 4);  // own epilogue threads + one arrive per peer epilogue warp
        }
        for (int i = 0; i < WS; ++i) {
            mbar_init(&w_full[i], 1);
            mbar_init(&w_empty[i], 1);
            mbar_init(&w_peer[i], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tcols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // both CTAs' barriers initialised, TMEM allocated
    tc_fence_after();
    pdl_launch_dependents();
    const uint32_t tmem = *tmem_slot;

    auto out_row = [&](int m, long long *dst_row) {
        if (m >= g.M) return false;
        const int ox = m % g.Wq;
        const int tt = m / g.Wq;
        const int oy = tt % g.Hq;
        const int b = tt / g.Hq;
        *dst_row = ((long long)b * g.Ho + oy) * g.Wo + ox;
        return oy < g.Ho && ox < g.Wo;
    };

    if (warp == 0) {  // ---------------------------------- bulk-copy producer (both CTAs)
        const uint8_t *wsrc = reinterpret_cast<const uint8_t *>(g.w);
        pdl_wait();  // X' is written by the previous kernel (stage 1)
        Ring ra(AS), rw(WS);
        for (int u = cid; u < num_units; u += ncl) {
            const int pr = u % mpairs, nt = u / mpairs;
            const int m0 = (2 * pr + (int)rank) * kBM16;  // a phantom tile (odd tile count) reads slack rows
            for (int kc = 0; kc < g.kchunks; ++kc, ra.next(), rw.next()) {
                mbar_wait_sleep(&a_empty[ra.slot], ra.phase ^ 1);
                if (lane == 0) mbar_arrive_expect_tx(&a_full[ra.slot], a_bytes);
                __syncwarp();
                uint8_t *dst = a_slots + (size_t)ra.slot * a_bytes;
                for (int c = lane; c < g.nphase * 8; c += 32) {  // (phase, plane, hi/lo)
                    const int ph = c >> 3, kg = (c >> 1) & 3, lo = c & 1;
                    const long long off =
                        ((long long)(kc * 4 + kg) * g.plane_rows + (long long)g.phase_src[ph] * g.phase_rows + m0) * 8;
                    bulk_load(dst + lo * a_half + (size_t)(ph * 4 + kg) * band_bytes, (lo ? g.xg_lo : g.xg) + off,
                              band_bytes, &a_full[ra.slot]);
                }
                __syncwarp();
                mbar_wait(&w_empty[rw.slot], rw.phase ^ 1);
                if (lane == 0 && u == cid) C2TL(kc, leader ? 0 : 4);
                if (lane == 0) mbar_arrive_expect_tx(&w_full[rw.slot], w_slot);
                __syncwarp();
                // this CTA's half (rank 0: hi rows, rank 1: lo rows) of the (kc, nt) slice
                const uint8_t *src = wsrc + (((size_t)kc * g.ntiles + nt) * 2 + rank) * w_slot;
                for (uint32_t o = (uint32_t)lane * 16384; o < w_slot; o += 32 * 16384)
                    bulk_load(w_slots + (size_t)rw.slot * w_slot + o, src + o, w_slot - o < 16384 ? w_slot - o : 16384,
                              &w_full[rw.slot]);
                __syncwarp();
            }
        }
    } else if (warp == 1 && !leader) {  // ------------- peer: relay "my slot is full" to the leader
        const uint32_t a_peer_l = mapa_shared(smem_u32(a_peer), 0), w_peer_l = mapa_shared(smem_u32(w_peer), 0);
        Ring ra(AS), rw(WS);
        for (int u = cid; u < num_units; u += ncl)
            for (int kc = 0; kc < g.kchunks; ++kc, ra.next(), rw.next()) {
                // cheap release (no GPU-scope membar): the TMA writes are complete
                mbar_wait(&a_full[ra.slot], ra.phase);
                if (lane == 0) {
                    fence_release_smem_cluster();
                    mbar_arrive_cluster(a_peer_l + ra.slot * 8);
                }
                mbar_wait(&w_full[rw.slot], rw.phase);
                if (lane == 0) {
                    fence_release_smem_cluster();
                    mbar_arrive_cluster(w_peer_l + rw.slot * 8);
                }
                __syncwarp();
            }
    } else if (warp == 1) {  // ---------------------------- leader: MMA issue for the pair
        const uint32_t idesc = idesc_bf16(2 * kBM16, ncols), idesc_h = idesc_bf16(2 * kBM16, BN);
        const uint64_t da = sdesc_kmajor_none(smem_u32(a_slots), band_bytes, 128);
        const uint64_t db = sdesc_kmajor_none(smem_u32(w_slots), BN * 16, 128);
        const uint64_t dbx = sdesc_kmajor_none(smem_u32(w_slots + w_extra), BN / 2 * 16, 128);
        const uint32_t a_lo = a_half >> 4, wtap16 = w_tap >> 4, xtap16 = x_tap >> 4;
        const uint32_t plane2a = (2 * band_bytes) >> 4, plane2b = (2 * BN * 16) >> 4, plane2x = (BN * 16) >> 4;
        Ring ra(AS), rw(WS), acc(2);
        for (int u = cid; u < num_units; u += ncl, acc.next()) {
            mbar_wait_acq_cluster(&tempty[acc.slot], acc.phase ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc.slot * ncols;
            uint32_t accum = 0;
            for (int kc = 0; kc < g.kchunks; ++kc, ra.next(), rw.next()) {
                mbar_wait(&a_full[ra.slot], ra.phase);
                mbar_wait_cluster(&a_peer[ra.slot], ra.phase);
                mbar_wait(&w_full[rw.slot], rw.phase);
                if (lane == 0 && u == cid) C2TL(kc, 1);
                mbar_wait_cluster(&w_peer[rw.slot], rw.phase);
                if (lane == 0 && u == cid) C2TL(kc, 2);
                tc_fence_after();
                const uint64_t aslot = da + ((ra.slot * a_bytes) >> 4);
                const uint64_t bslot = db + ((rw.slot * w_slot) >> 4), xslot = dbx + ((rw.slot * w_slot) >> 4);
                if (elect_one()) {
#pragma unroll 1
                    for (int tt = 0; tt < 9; ++tt) {
                        const uint64_t a = aslot + (((uint32_t)g.tap_phase[tt] * 4 * band_bytes +
                                                     (uint32_t)g.tap_off[tt] * 16) >> 4);
                        const uint64_t b = bslot + tt * wtap16, x = xslot + tt * xtap16;
#pragma unroll
                        for (int j = 0; j < 2; ++j) {  // K = 16 = two 8-channel planes
                            const uint64_t aj = a + j * plane2a;
                            mma_bf16_pair(d, aj, b + j * plane2b, idesc, accum);      // X' hi x [C hi | C lo]
                            mma_bf16_pair(d, aj + a_lo, x + j * plane2x, idesc_h, 1);  // X' lo x C hi
                            accum = 1;
                        }
                    }
                    mma_commit_pair(&w_empty[rw.slot]);
                    mma_commit_pair(&a_empty[ra.slot]);
                }
                __syncwarp();
                if (lane == 0 && u == cid) C2TL(kc, 3);
            }
            if (elect_one()) mma_commit_pair(&tfull[acc.slot]);
            __syncwarp();
        }
    } else if (warp < 6) {  // ------------------ epilogue warps 2..5 (both CTAs): acc -> Z hi/lo
        const int q = warp & 3;
        float *scratch = epi_scratch + q * 1024;
        __nv_bfloat16 *z = reinterpret_cast<__nv_bfloat16 *>(g.z);
        __nv_bfloat16 *z_lo = reinterpret_cast<__nv_bfloat16 *>(g.z_lo);
        const int r = q * 32 + lane;  // tile row = TMEM lane
        const uint32_t tempty_l = mapa_shared(smem_u32(tempty), 0);
        Ring acc(2);
        for (int u = cid; u < num_units; u += ncl, acc.next()) {
            const int pr = u % mpairs, nt = u / mpairs;
            const int m0 = (2 * pr + (int)rank) * kBM16, n0 = nt * BN;
            mbar_wait_sleep(&tfull[acc.slot], acc.phase);
            tc_fence_after();
            long long dst_row = 0;
            const bool valid = out_row(m0 + r, &dst_row);
            const uint32_t src = tmem + ((uint32_t)(q * 32) << 16) + acc.slot * ncols;
            for (int c = 0; c < BN; c += 32) {
                uint32_t rr[32], r2[32];
                float v[32];
                tmem_ld_32x32b_x32(src + c, rr);
                tmem_ld_32x32b_x32(src + BN + c, r2);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(rr[j]) + __uint_as_float(r2[j]);
                if (n0 + c >= g.Nn) continue;  // warp-uniform
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
            if (leader) {
                mbar_arrive_relaxed(&tempty[acc.slot]);
            } else {
                __syncwarp();
                if (lane == 0) mbar_arrive_remote_release(tempty_l + acc.slot * 8);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();  // the leader's MMAs read the peer's shared memory: nobody leaves early
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
}

cudaError_t bf_core2_launch(const BfCoreArgs &g, int grid, cudaStream_t st) {
    const int smem = bf_core2_smem_bytes(g.BN, g.nphase, g.band_rows, g.w_slots, g.a_slots);
    cudaError_t e = cudaFuncSetAttribute(tdc_bf_core2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(tdc_bf_core2_kernel, grid, 192, smem, st, g);  // cluster dims are static (2)
}

cudaError_t bf_core_launch(const BfCoreArgs &g, int grid, cudaStream_t st) {
    const int smem = bf_core_smem_bytes(g.BN, g.nphase, g.band_rows, g.tg, g.w_slots, g.ksplit);
    auto go = [&](auto kernel) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl_cluster(kernel, grid, 192, smem, st, g.ksplit, g);
    };
    return g.ksplit > 1 ? go(tdc_bf_core_kernel<false, 1, false>)
                        : (g.gsplit > 1 ? go(tdc_bf_core_kernel<false, 2, false>) : go(tdc_bf_core_kernel<false, 0, false>));
}

cudaError_t bf_core3_launch(const BfCoreArgs &g, int grid, cudaStream_t st) {
    const int smem = bf_core3_smem_bytes(g);
    auto go = [&](auto kernel) {
        cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        return launch_pdl(kernel, grid, 448, smem, st, g);
    };
    return g.res ? go(tdc_bf_core_kernel<true, 0, true>) : go(tdc_bf_core_kernel<true, 0, false>);
}

}  // namespace tdc
