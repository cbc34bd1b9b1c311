// tkd_simt.cu -- fused three-stage TKD layer on CUDA cores (fp32 FFMA).
//
// One CTA = one image b x one output tile (oth x otw pixels) x all N output
// channels.  The three stages of the layer (include/tdc.h; north_star) run
// back to back inside the CTA and the rank-sized intermediates never touch HBM:
//
//   stage 1 (a1)  X'[p][a] for every pixel p of the (ih x iw) input halo tile,
//                 K-loop over C in chunks of ck staged in shared memory; X' is
//                 accumulated in shared memory.  Out-of-image halo pixels load
//                 0, which is the core's zero padding (reading R6).
//   stage 2 (a2)  Z[o][q] = sum_{r,t,a} X'[(oy*s+r)*iw + ox*s+t][a] * core[r,t][a][q],
//                 the paper's core convolution as a gather from
//                 the shared X' tile with CRSN-ordered weights.
//   stage 3 (a3)  Y[o][n] = sum_q Z[o][q] * U_out[n][q] (+ bias), written once
//                 per output element with coalesced NHWC stores (a4) -- no
//                 atomics, unlike the paper's C-split.
//
// Every stage is a register-blocked 4 x 4 micro-tile GEMM: each thread owns 4
// rows (pixels) x 4 columns (ranks / channels), so each shared-memory value
// read feeds 4 FMAs.  This is the always-correct fp32 variant; the tcgen05
// variant (tkd_tc.cu) is the fast path where the stages are real contractions.
#include "internal.h"

namespace tdc {

constexpr int kSimtThreads = 256;

__host__ __device__ inline int round_up4(int v) { return (v + 3) & ~3; }

struct SimtSmem {
    int xs, us, x1s, zs, total;  // float offsets
};

__host__ __device__ inline SimtSmem simt_smem_layout(int P, int M, int ck, int D1p, int D2p) {
    SimtSmem s;
    s.xs = 0;
    s.us = round_up4(P * (ck + 1));
    s.x1s = s.us + ck * D1p;
    s.zs = round_up4(s.x1s + P * (D1p + 1));
    s.total = s.zs + M * (D2p + 1);
    return s;
}

__global__ void __launch_bounds__(kSimtThreads)
tdc_tkd_fused_simt_kernel(LayerDims d, SimtWeights w, SimtTile t,
                          const float *__restrict__ x, float *__restrict__ y) {
    extern __shared__ __align__(16) float smem[];
    const int tid = threadIdx.x;
    const int P = t.ih * t.iw;
    const int M = t.oth * t.otw;
    const int D1p = w.D1p, D2p = w.D2p;
    const int LDX = t.ck + 1, LD1 = D1p + 1, LD2 = D2p + 1;
    const SimtSmem L = simt_smem_layout(P, M, t.ck, D1p, D2p);
    float *xs = smem + L.xs;
    float *us = smem + L.us;
    float *x1s = smem + L.x1s;
    float *zs = smem + L.zs;

    const int b = blockIdx.y;
    const int th = blockIdx.x / t.tiles_w, tw = blockIdx.x % t.tiles_w;
    const int oy0 = th * t.oth, ox0 = tw * t.otw;
    const int iy0 = oy0 * d.stride - d.pad, ix0 = ox0 * d.stride - d.pad;

    // ---------------- stage 1: X' = X . U_in over the halo tile ----------------
    const int nt1 = D1p >> 2, T1 = ((P + 3) >> 2) * nt1;
    for (int c0 = 0; c0 < d.C; c0 += t.ck) {
        __syncthreads();
        for (int e = tid; e < P * t.ck; e += kSimtThreads) {
            const int p = e / t.ck, cc = e - p * t.ck;
            const int iy = iy0 + p / t.iw, ix = ix0 + p % t.iw, c = c0 + cc;
            float v = 0.f;
            if (c < d.C && iy >= 0 && iy < d.H && ix >= 0 && ix < d.W)
                v = __ldg(&x[(((size_t)b * d.H + iy) * d.W + ix) * d.C + c]);
            xs[p * LDX + cc] = v;
        }
        for (int e = tid; e < t.ck * D1p; e += kSimtThreads) {
            const int cc = e / D1p;
            us[e] = (c0 + cc < d.C) ? __ldg(&w.uin[(size_t)c0 * D1p + e]) : 0.f;
        }
        __syncthreads();
        const int kc = min(t.ck, d.C - c0);
        for (int tile = tid; tile < T1; tile += kSimtThreads) {
            const int mt = tile / nt1, nt = tile - mt * nt1;
            int prow[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) prow[i] = min(mt * 4 + i, P - 1);
            float acc[4][4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    acc[i][j] = (c0 == 0) ? 0.f : x1s[prow[i] * LD1 + nt * 4 + j];
            for (int cc = 0; cc < kc; ++cc) {
                const float4 bv = *reinterpret_cast<const float4 *>(&us[cc * D1p + nt * 4]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float av = xs[prow[i] * LDX + cc];
                    acc[i][0] = fmaf(av, bv.x, acc[i][0]);
                    acc[i][1] = fmaf(av, bv.y, acc[i][1]);
                    acc[i][2] = fmaf(av, bv.z, acc[i][2]);
                    acc[i][3] = fmaf(av, bv.w, acc[i][3]);
                }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                if (mt * 4 + i < P)
#pragma unroll
                    for (int j = 0; j < 4; ++j) x1s[prow[i] * LD1 + nt * 4 + j] = acc[i][j];
        }
    }
    __syncthreads();

    // ---------------- stage 2: core K x K convolution D1 -> D2 -----------------
    const int nt2 = D2p >> 2, T2 = ((M + 3) >> 2) * nt2;
    const int KK = d.K * d.K;
    for (int tile = tid; tile < T2; tile += kSimtThreads) {
        const int mt = tile / nt2, nt = tile - mt * nt2;
        int pbase[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int o = min(mt * 4 + i, M - 1);
            const int oy = o / t.otw, ox = o - oy * t.otw;
            pbase[i] = (oy * d.stride) * t.iw + ox * d.stride;
        }
        float acc[4][4] = {};
        for (int tap = 0; tap < KK; ++tap) {
            const int r = tap / d.K, tt = tap - r * d.K;
            const int poff = r * t.iw + tt;
            const float *cw = w.core + (size_t)tap * D1p * D2p + nt * 4;
            for (int a = 0; a < D1p; ++a) {
                const float4 bv = __ldg(reinterpret_cast<const float4 *>(cw + (size_t)a * D2p));
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float av = x1s[(pbase[i] + poff) * LD1 + a];
                    acc[i][0] = fmaf(av, bv.x, acc[i][0]);
                    acc[i][1] = fmaf(av, bv.y, acc[i][1]);
                    acc[i][2] = fmaf(av, bv.z, acc[i][2]);
                    acc[i][3] = fmaf(av, bv.w, acc[i][3]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (mt * 4 + i < M)
#pragma unroll
                for (int j = 0; j < 4; ++j) zs[(mt * 4 + i) * LD2 + nt * 4 + j] = acc[i][j];
    }
    __syncthreads();

    // ---------------- stage 3: Y = Z . U_out^T (+ bias), NHWC store ------------
    const int Np = w.Np;
    const int nt3 = Np >> 2, T3 = ((M + 3) >> 2) * nt3;
    const bool vec_store = (d.N & 3) == 0;
    for (int tile = tid; tile < T3; tile += kSimtThreads) {
        const int mt = tile / nt3, nt = tile - mt * nt3;
        int orow[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) orow[i] = min(mt * 4 + i, M - 1);
        float acc[4][4] = {};
        for (int q = 0; q < D2p; ++q) {
            const float4 bv = __ldg(reinterpret_cast<const float4 *>(w.uoutT + (size_t)q * Np + nt * 4));
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float av = zs[orow[i] * LD2 + q];
                acc[i][0] = fmaf(av, bv.x, acc[i][0]);
                acc[i][1] = fmaf(av, bv.y, acc[i][1]);
                acc[i][2] = fmaf(av, bv.z, acc[i][2]);
                acc[i][3] = fmaf(av, bv.w, acc[i][3]);
            }
        }
        float4 bb = make_float4(0.f, 0.f, 0.f, 0.f);
        if (w.bias) bb = __ldg(reinterpret_cast<const float4 *>(w.bias + nt * 4));
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int o = mt * 4 + i;
            if (o >= M) continue;
            const int oy = oy0 + o / t.otw, ox = ox0 + o % t.otw;
            if (oy >= d.Ho || ox >= d.Wo) continue;
            float *dst = y + (((size_t)b * d.Ho + oy) * d.Wo + ox) * d.N + nt * 4;
            const float4 v = make_float4(acc[i][0] + bb.x, acc[i][1] + bb.y,
                                         acc[i][2] + bb.z, acc[i][3] + bb.w);
            if (vec_store) {
                *reinterpret_cast<float4 *>(dst) = v;
            } else {
                const float vv[4] = {v.x, v.y, v.z, v.w};
                for (int j = 0; j < 4 && nt * 4 + j < d.N; ++j) dst[j] = vv[j];
            }
        }
    }
}

bool simt_choose_tile(const LayerDims &d, int D1p, int D2p, int max_smem, SimtTile *t) {
    static const int cand[][2] = {{8, 8}, {8, 4}, {4, 4}, {4, 2}, {2, 2}, {2, 1}, {1, 1}};
    const int ck = d.C < 32 ? d.C : 32;
    for (auto &c : cand) {
        const int oth = c[0] < d.Ho ? c[0] : d.Ho;
        const int otw = c[1] < d.Wo ? c[1] : d.Wo;
        const int ih = (oth - 1) * d.stride + d.K, iw = (otw - 1) * d.stride + d.K;
        const SimtSmem L = simt_smem_layout(ih * iw, oth * otw, ck, D1p, D2p);
        const long bytes = (long)L.total * 4;
        if (bytes <= max_smem) {
            t->oth = oth;
            t->otw = otw;
            t->ih = ih;
            t->iw = iw;
            t->ck = ck;
            t->tiles_h = (d.Ho + oth - 1) / oth;
            t->tiles_w = (d.Wo + otw - 1) / otw;
            t->smem_bytes = (int)bytes;
            return true;
        }
    }
    return false;
}

cudaError_t simt_fused_launch(const LayerDims &d, const SimtWeights &w, const SimtTile &t,
                              const float *x, float *y, int batch, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(tdc_tkd_fused_simt_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         t.smem_bytes);
    if (e != cudaSuccess) return e;
    dim3 grid(t.tiles_h * t.tiles_w, batch);
    tdc_tkd_fused_simt_kernel<<<grid, kSimtThreads, t.smem_bytes, st>>>(d, w, t, x, y);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Layout conversion for the NCHW API layout (paper statement).
// 32 x 32 shared-memory transpose per (b, plane) so both sides stay coalesced.
__global__ void tdc_nchw_to_nhwc_kernel(const float *__restrict__ src, float *__restrict__ dst,
                                        int C, int HW) {
    __shared__ float tile[32][33];
    const int b = blockIdx.z;
    const int c0 = blockIdx.y * 32, s0 = blockIdx.x * 32;
    const float *s = src + (size_t)b * C * HW;
    float *o = dst + (size_t)b * C * HW;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int c = c0 + i, sp = s0 + threadIdx.x;
        if (c < C && sp < HW) tile[i][threadIdx.x] = s[(size_t)c * HW + sp];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int sp = s0 + i, c = c0 + threadIdx.x;
        if (c < C && sp < HW) o[(size_t)sp * C + c] = tile[threadIdx.x][i];
    }
}

__global__ void tdc_nhwc_to_nchw_kernel(const float *__restrict__ src, float *__restrict__ dst,
                                        int C, int HW) {
    __shared__ float tile[32][33];
    const int b = blockIdx.z;
    const int s0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    const float *s = src + (size_t)b * C * HW;
    float *o = dst + (size_t)b * C * HW;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int sp = s0 + i, c = c0 + threadIdx.x;
        if (c < C && sp < HW) tile[i][threadIdx.x] = s[(size_t)sp * C + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int c = c0 + i, sp = s0 + threadIdx.x;
        if (c < C && sp < HW) o[(size_t)c * HW + sp] = tile[threadIdx.x][i];
    }
}

cudaError_t nchw_to_nhwc(const float *src, float *dst, int B, int C, int H, int W,
                         cudaStream_t st) {
    const int HW = H * W;
    dim3 grid((HW + 31) / 32, (C + 31) / 32, B), block(32, 8);
    tdc_nchw_to_nhwc_kernel<<<grid, block, 0, st>>>(src, dst, C, HW);
    return cudaGetLastError();
}

cudaError_t nhwc_to_nchw(const float *src, float *dst, int B, int C, int H, int W,
                         cudaStream_t st) {
    const int HW = H * W;
    dim3 grid((C + 31) / 32, (HW + 31) / 32, B), block(32, 8);
    tdc_nhwc_to_nchw_kernel<<<grid, block, 0, st>>>(src, dst, C, HW);
    return cudaGetLastError();
}

}  // namespace tdc
