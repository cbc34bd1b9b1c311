// internal.h -- device-side parameter blocks and launchers shared by the
// C-ABI (tdc_api.cu) and the kernels.  Not part of the public ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

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
};
int tc_smem_bytes(int BN, int stages);
int tc_pick_stages(int BN, int iters, int max_smem);
bool make_tma_2d(CUtensorMap *map, const float *base, long long rows, int k_extent, int pitch,
                 int box_rows);
cudaError_t tc_gemm_launch(const CUtensorMap &mapA, const CUtensorMap &mapB, const TcGemmArgs &g,
                           int grid_n, cudaStream_t st);

// NCHW <-> NHWC for the NCHW API layout.
cudaError_t nchw_to_nhwc(const float *src, float *dst, int B, int C, int H, int W,
                         cudaStream_t st);
cudaError_t nhwc_to_nchw(const float *src, float *dst, int B, int C, int H, int W,
                         cudaStream_t st);

}  // namespace tdc
