// internal.h -- device-side parameter blocks and launchers shared by the
// C-ABI (tdc_api.cu) and the kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

namespace tdc {

// Packed weights produced at plan time (§8(a) row a0; CRSN idea).
//   uin   [C][D1p]            stage-1 factor, rank fastest (zero-padded ranks)
//   core  [K*K][D1p][D2p]     core, tap-major, out-rank fastest ("CRSN" order)
//   uoutT [D2p][Np]           stage-3 factor transposed, channel fastest
//   bias  [Np] or null
struct SimtWeights {
    const float *uin, *core, *uoutT, *bias;
    int D1p, D2p, Np;
};

struct LayerDims {
    int B, C, H, W, N, K, stride, pad, Ho, Wo;
};

struct SimtTile {
    int oth, otw;   // output tile (pixels)
    int ih, iw;     // input halo tile = (ot-1)*s + K
    int ck;         // channel chunk for stage 1
    int tiles_h, tiles_w;
    int smem_bytes;
};

// Chooses the output tile for the SIMT variant; returns false if nothing fits.
bool simt_choose_tile(const LayerDims &d, int D1p, int D2p, int max_smem, SimtTile *t);
// x, y NHWC.  Launches one kernel.
cudaError_t simt_fused_launch(const LayerDims &d, const SimtWeights &w, const SimtTile &t,
                              const float *x, float *y, int batch, cudaStream_t st);

// ---- tensor-core (tcgen05) GEMM with taps: see tkd_tc.cu ----
constexpr int kMaxTaps = 49;
struct TcGemmArgs {
    int M, Nn, kchunks, taps, BN, stages;
    int a_off[kMaxTaps], b_off[kMaxTaps];
    float *out;
    int ldo;
    const float *bias;
    int remap;  // 0 identity, 1 pixel -> phase grid, 2 output grid -> compact
    int H, W, s, p, Hq, Wq, Ho, Wo;
    long long phase_rows;
    long long planar_stride;  // >0: epilogue writes planar [col/4][row][4] with this plane stride (floats)
    int split;        // 1: 3xTF32 (hi*hi + hi*lo + lo*hi), fp32-grade accuracy
    int a_convert;    // split only: 1 = A lo computed in-kernel from A (user input); 0 = loaded
    float *out_lo;    // split only: epilogue also writes the lo part of the output (next stage's A lo)
    int ntiles;       // N tiles (persistent kernel walks mtiles x ntiles)
    int out_bf16;     // 3xBF16 stage 1: out/out_lo are bf16 planar [c/8][row][8], planar_stride in rows
    int xstages;      // 3xBF16 stage 1: depth of the fp32 staging ring (separate from `stages`)
    int ksplit;       // 3xBF16: >1 = split K over a cluster of ksplit CTAs, DSMEM reduction
    int bstages;      // 3xBF16 stage 1: depth of the weight (B) ring
    const float *res; // fp32 output only: residual added before the activation (ld = ldo), or null
    int relu;         // fp32 output only: ReLU after bias/residual
    int dbg;          // debug (TDC_GEMM_DBG): 1 skip the fp32 output stores, 2 skip residual reads
    int tma_y;        // fp32 output (remap 0, ldo == Nn): full 32x32 blocks stored by TMA (mapY)
    int yring;        // 3xBF16 converting GEMM with fp32 output: TMA output ring depth (2 or 4)
    int gsplit;       // 3xBF16: >1 = split K into gsplit pieces, partials reduced through L2
    float *part;      // gsplit: fp32 partial tiles [tiles][gsplit-1][BN/4][128][4]
    int *flags;       // gsplit: one flag per (tile, piece > 0), zero between launches
};

// Stage-2 core convolution with a shared-memory-resident X' band (tkd_tc.cu):
// X' planar [kg][rows_total][4]; weights pre-blocked [tap][kc][ntile][8][BN][4].
struct TcCoreArgs {
    const float *xg;          // X' planar grid
    long long plane_stride;   // floats between kg planes (rows_total * 4)
    const float *w;           // blocked core weights
    float *z;                 // Z compact [B*Ho*Wo][ldz]
    int ldz, Nn;              // Z pitch, valid output columns (D2s)
    int M;                    // output-grid rows this launch
    int kchunks, taps, ntiles, BN, nphase, band_rows, b_stages;
    long long phase_rows;
    int tap_phase[kMaxTaps], tap_off[kMaxTaps];
    int phase_src[kMaxTaps];   // global phase index of compact phase i
    int Hq, Wq, Ho, Wo;
    int split;                 // 3xTF32
    const float *xg_lo;        // split: X' lo planes
    const float *w_lo;         // split: blocked core weights, lo parts
    float *z_lo;               // split: Z lo (next stage's A lo)
};


int tc_core_smem_bytes(int BN, int nphase, int band_rows, int b_stages, int split);
cudaError_t tc_core_launch(const TcCoreArgs &g, int grid, cudaStream_t st);
// CTAs per SM for a persistent kernel given its smem and TMEM (2 x ncols) footprint.
int persistent_occupancy(int smem_bytes, int bn);
int tc_smem_bytes(int BN, int stages, int split);
int tc_pick_stages(int BN, int iters, int max_smem, int split);
bool make_tma_2d(CUtensorMap *map, const float *base, long long rows, int k_extent, int pitch,
                 int box_rows);
cudaError_t tc_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapAlo,
                           const CUtensorMap &mapB, const CUtensorMap &mapBlo, const TcGemmArgs &g,
                           int grid, cudaStream_t st);

// ---- fused single-kernel TKD layer (tkd_fused.cu) ----
struct FusedArgs {
    int B, H, W, C, N, Ho, Wo, K, KK, s, p;
    int R, Rin, Wp, Wq;          // output rows per tile; input band rows/cols; phase-grid width
    int tiles_per_img, num_tiles;
    int nblk1, c_chunks;         // stage-1 accumulator blocks (128 rows); C/32 chunks
    int D1s, D2s, Nh, nhalves;   // padded ranks; stage-3 columns per pass
    int nph, PR, TR;             // X' phases, phase-plane stride (rows), total rows
    int tap_phase[kMaxTaps], tap_off[kMaxTaps];
    int phase_idx[kMaxTaps];     // (py*s+px) -> compact phase or -1
    const float *w;              // [U_in chunks][core chunks][U_out chunks], blocked [8][rows][4]
    const float *bias;
    float *y;
    int XS, WS;                  // ring depths (X chunks, weight chunks)
    int acc3_col, tmem_cols, nbuf3;   // stage-3 accumulator column, TMEM size, buffers
    int P1, P2, P3;  // independent accumulator chains per stage (hide MMA accumulate latency)
};
int fused_smem_bytes(const FusedArgs &g);
bool make_tma_4d_nhwc(CUtensorMap *map, const float *x, int C, int W, int H, int B, int box_w,
                      int box_h);
bool fused_make_x_map(CUtensorMap *map, const float *x, const FusedArgs &g);
cudaError_t fused_launch(const CUtensorMap &mapX, const FusedArgs &g, int grid, cudaStream_t st);

// ---- 3xBF16 variant of the 3-launch path (tkd_bf16.cu) ----
// fp32_out: a converting (xstages > 0) GEMM with fp32 output (model dense convs) reserves
// its TMA output ring of fp32_out (2 or 4) buffers per warp; stage 1 (bf16 X') passes 0.
int bf_smem_bytes(int BN, int stages, int xstages, int ksplit, int bstages, int fp32_out = 0);
int bf_pick_stages(int BN, int max_smem, int convert, int *xstages, int ksplit, int *bstages, int fp32_out = 0);
// mapR: fp32-output GEMMs with a residual and tma_y: TMA map of the residual (same
// geometry as mapY); null = no residual map (mapY is passed in its place).
cudaError_t bf_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapAlo, const CUtensorMap &mapB,
                           const CUtensorMap &mapBlo, const CUtensorMap &mapY, const TcGemmArgs &g, int grid,
                           cudaStream_t st, const CUtensorMap *mapR = nullptr);
// 3xBF16 stage-2 core convolution (tkd_bf16.cu).  X' hi/lo planar bf16
// [D1s/8][rows_total][8]; weights blocked [kc][ntile][group][tg taps][plane 4][2BN][8]
// with rows 0..BN-1 = hi and BN..2BN-1 = lo, so one bulk copy moves a whole
// (kc, tap-group) slice and, when 2BN <= 128, one N = 2BN MMA covers hi and lo.
struct BfCoreArgs {
    const uint16_t *xg, *xg_lo;
    long long plane_rows;     // rows_total: rows between 8-channel planes
    const uint16_t *w;
    uint16_t *z, *z_lo;       // Z hi/lo [B*Ho*Wo][ldz]
    int ldz, Nn, M;
    int kchunks, taps, ntiles, BN, nphase, band_rows;
    int tg, ngroups, w_slots, w_resident, ncat;
    long long phase_rows;
    int tap_phase[kMaxTaps], tap_off[kMaxTaps], phase_src[kMaxTaps];
    int Hq, Wq, Ho, Wo;
    // fused stage 3 (tdc_bf_core3_kernel): Z stays on chip, Y = Z . U_out^T (+bias)
    const uint16_t *w3;       // U_out blocked [D2s/8 planes][2*N3p rows: hi | lo][8], resident
    const float *bias;
    float *y;                 // Y [B*Ho*Wo][N3]
    int N3, N3p, ncat3;       // output channels, padded (mult. of 16), hi|lo concat in one MMA
    int ksplit;               // >1: split the D1 chunks over a cluster (stage 2 alone, not fused)
    int a_slots;              // CTA-pair kernel (tdc_bf_core2_kernel): band ring depth (2 or 3)
    int y_direct;             // fused stage 3: lanes store their own Y rows (no smem transpose)
    const float *res;         // fused stage 3: residual [B*Ho*Wo][N3] added before the activation
    int relu;                 // fused stage 3: ReLU after bias/residual
    int dbg;                  // debug (TDC_CORE_DBG): 1 skip Y stores, 2 skip Z smem writes,
                              // 4 skip band reloads after the first tile, 8 skip S3 MMAs,
                              // 16 no acc2-free wait, 32 no E2 TMEM loads, 64 no E3 TMEM loads,
                              // 256 no stage 3 at all (no S3 waits/commits, E3 idle), 512 MMA warp
                              // does not wait for bands after the first tile, 1024 (with 512) no
                              // per-tile weight wait or band-slot commit
    int gsplit;               // stage 2 alone: >1 = split the D1 chunks into gsplit pieces (L2 partials)
    float *part;              // gsplit: fp32 partial tiles [tiles][gsplit-1][BN/4][128][4]
    int *flags;               // gsplit: one flag per (tile, piece > 0)
};
int bf_core_smem_bytes(int BN, int nphase, int band_rows, int tg, int w_slots, int ksplit);
int bf_core3_smem_bytes(const BfCoreArgs &g);
int bf_core3_tmem_cols(const BfCoreArgs &g);
cudaError_t bf_core3_launch(const BfCoreArgs &g, int grid, cudaStream_t st);
cudaError_t bf_core_launch(const BfCoreArgs &g, int grid, cudaStream_t st);
// stage 2 on CTA pairs (cta_group::2, tdc_bf_core2_kernel): weights [kc][ntile][half hi|lo][tap][plane][BN][8]
int bf_core2_smem_bytes(int BN, int nphase, int band_rows, int w_slots, int a_slots);
cudaError_t bf_core2_launch(const BfCoreArgs &g, int grid, cudaStream_t st);
bool make_tma_2d_bf16(CUtensorMap *map, const void *base, long long rows, int k_extent, int pitch,
                      int box_rows);

// Single-launch 3xBF16 TKD layer (tkd_layer.cu): stage 1 -> X' band ring in shared
// memory -> core -> Z in shared memory -> stage 3, one persistent kernel.  Stride 1.
struct BfLayerArgs {
    int B, H, W, C, N, K, KK, s, p, Ho, Wo, Wp, Wq, Hq;
    int R, e, T;              // output rows per tile (R*Wq <= 128), (K-1)/s, tiles per image
    int TH, nstrips, sw;      // row blocks per image, column strips (Wp > 128: 128-position
                              // strips of sw = 128 - (K-1) output columns; else 1 strip, sw = Wo)
    int rpb;                  // padded input rows per stage-1 block (rpb*Wp <= 128)
    int NR, NRB;              // band ring rows (2R+e) and buffer rows incl. the mirror rows
    int XR, ZR;               // rows of an X staging tile / a Z plane (multiples of 8, <= 128)
    int tn;                   // 1: K = 3, D2s = 32, the 3 taps of a core row along N (tkd_layer.cu)
    int xt;                   // 1 (with tn): X hi/lo and Z hi/lo in tensor memory, stages 1 and 3 as TS-MMAs
    int ncat3;                // 1: stage 3 as [hi | lo] along N (2 MMAs, 2*N3p accumulator columns)
    int cchunks;              // 64-channel chunks of C (TMA zero-fills channels >= C)
    int D1s, D2s, N3p;        // ranks / output channels padded to multiples of 32
    int XS;                   // X staging ring depth (<= 4)
    int pf_blocks;            // stage-1 blocks the producer's L2 prefetch runs ahead of its loads
    int num_tiles;            // batch * T for this call
    int tmem_cols;
    int tap_off[kMaxTaps];    // r*Wq + t
    const uint16_t *w1;       // U_in per 64-channel chunk: [2*D1s rows: hi | lo][64] bf16, 128B-swizzled image
    const uint16_t *w2;       // core [D1s/32][tap][plane 4][2*D2s rows: hi | lo][8]
    const uint16_t *w3;       // U_out [D2s/8][2*N3p rows: hi | lo][8]
    const float *bias;        // [N] or null
    const float *res;         // residual [B*Ho*Wo][N] or null (model path)
    int relu;
    float *y;                 // [B*Ho*Wo][N]
    uint8_t *dbg;             // debug: CTA 0 copies its shared memory here at exit (null = off)
    int knobs;                // debug builds only (TDC_LAYER_DBG): 1 no Y stores, 2 no X conversion,
                              // 4 no band writes, 8 no Z writes, 16/32/64 no S2/S1/S3 MMAs,
                              // 128 no X loads after the first tiles (results wrong by design)
};
int bf_layer_smem_bytes(const BfLayerArgs &g);
cudaError_t bf_layer_launch(const CUtensorMap &mapX, const BfLayerArgs &g, int grid, cudaStream_t st);
// IEEE-fp32 3-launch path on CUDA cores (tkd_sgemm.cu): C[out(m)] = sum_tap A[m + a_off[tap]] . B[tap]
struct SgemmArgs {
    const float *A;           // rows of K (padded to 8) fp32, row stride lda
    long long lda;
    int M, K, taps;           // output rows, K per tap (multiple of 8), taps
    int kmask, K_valid;       // 1: columns >= K_valid of A are read as 0 (stage 1, C % 8 != 0)
    long long a_off[kMaxTaps];// per-tap row offset (phase plane + tap shift)
    const float *B;           // [taps][K][ldb] fp32, zero-padded to the N tiles
    int ldb, N;
    float *C;                 // output rows, stride ldc; columns >= N untouched
    int ldc;
    const float *bias;        // [N] or null
    int remap;                // 0 identity, 1 input pixel -> phase grid row, 2 phase grid -> compact
    int H, W, s, p, Hq, Wq, Ho, Wo;
    long long phase_rows;
    int phase_idx[kMaxTaps];  // (py*s+px) -> compact phase or -1
    int tile;                 // 0: 64x128, 1: 128x64, 2: 256x32 (8x8 per thread, 128 threads)
    int ksplit;               // > 1: K split over grid.z, partial tiles in `part`, reduce kernel
    float *part;
    int ctas;                 // co-resident CTAs of the tile shape (split-K choice)
};
cudaError_t sgemm_taps_launch(const SgemmArgs &g, cudaStream_t st);
cudaError_t sgemm_prepare();
int sgemm_pick_tile(long long M, int N, int num_sms);
int sgemm_pick_ksplit(long long M, int N, int K, int taps, int tile, int ctas);
long long sgemm_tiles(long long M, int N, int tile);
int sgemm_ctas(int tile, int num_sms);
long long sgemm_part_floats(long long M, int N, int tile, int ksplit);
// NCHW <-> NHWC for the NCHW API layout.
cudaError_t nchw_to_nhwc(const float *src, float *dst, int B, int C, int H, int W,
                         cudaStream_t st);
cudaError_t nhwc_to_nchw(const float *src, float *dst, int B, int C, int H, int W,
                         cudaStream_t st);

// Launch a tcgen05 kernel with programmatic dependent launch (PDL) when enabled
// (default; TDC_NO_PDL=1 disables): the kernel's prologue (barrier init, TMEM
// alloc, descriptor prefetch) overlaps the tail of the previous kernel in the
// stream; the kernel calls griddepcontrol.wait before touching global memory.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), int grid, int block, int smem, cudaStream_t st,
                       Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
// Same, with a thread-block cluster of `cluster` CTAs along x (grid a multiple of it).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_cluster(void (*kernel)(KArgs...), int grid, int block, int smem, cudaStream_t st,
                               int cluster, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int n = 0;
    if (cluster > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = (unsigned)cluster;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    if (pdl_enabled()) {
        attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

}  // namespace tdc
