// tdc_model.cu -- whole-network inference over the TKD layer:
// an ordered op list (include/tdc.h "models") planned once, run as a sequence of
// kernels on one stream.  TKD layers go through the layer C-ABI with the residual /
// ReLU epilogue fused into their last stage; dense convolutions and the classifier
// run on the same tcgen05 3xBF16 GEMM kernel as the layer's stage 1 (im2col first
// when K > 1 or stride > 1); pools are small fp32 kernels.  BN is folded into the
// weights and a bias at create time.
#include "../../include/tdc.h"
#include "internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

namespace tdc {
uint16_t bf16_bits(float x);      // tdc_api.cu
float bf16_float(uint16_t b);
tdc_status set_error(tdc_status s, const char *msg);
int num_sms_of(int device);
int max_smem_of(int device);
}  // namespace tdc

namespace {

constexpr float kBnEps = 1e-5f;

int div_up(int a, int b) { return (a + b - 1) / b; }
int round_up(int v, int m) { return (v + m - 1) / m * m; }

tdc_status mfail(tdc_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    return tdc::set_error(s, buf);
}
tdc_status mcuda(cudaError_t e, const char *what) {
    return mfail(e == cudaErrorMemoryAllocation ? TDC_ERR_OUT_OF_MEMORY : TDC_ERR_CUDA, "%s: %s", what,
                 cudaGetErrorString(e));
}

// ------------------------------------------------------------------ aux kernels
// im2col, NHWC: row (b, oy, ox), column (r*K + t)*C + c; zero outside the image and in
// the padded columns [K*K*C, ld).
__global__ void tdc_im2col_kernel(const float *__restrict__ x, float *__restrict__ out, int B, int H, int W, int C,
                                  int K, int s, int p, int Ho, int Wo, int ld) {
    const long long total = (long long)B * Ho * Wo * ld;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(i % ld);
        const long long row = i / ld;
        float v = 0.f;
        if (col < K * K * C) {
            const int c = col % C, rt = col / C, t = rt % K, r = rt / K;
            const int ox = (int)(row % Wo), oy = (int)((row / Wo) % Ho), b = (int)(row / ((long long)Wo * Ho));
            const int y = oy * s - p + r, xx = ox * s - p + t;
            if (y >= 0 && y < H && xx >= 0 && xx < W) v = x[(((long long)b * H + y) * W + xx) * C + c];
        }
        out[i] = v;
    }
}

__global__ void tdc_maxpool_kernel(const float *__restrict__ x, float *__restrict__ out, int B, int H, int W, int C,
                                   int K, int s, int p, int Ho, int Wo) {
    const long long total = (long long)B * Ho * Wo * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % C);
        const long long pix = i / C;
        const int ox = (int)(pix % Wo), oy = (int)((pix / Wo) % Ho), b = (int)(pix / ((long long)Wo * Ho));
        float m = -INFINITY;
        for (int r = 0; r < K; ++r) {
            const int y = oy * s - p + r;
            if (y < 0 || y >= H) continue;
            for (int t = 0; t < K; ++t) {
                const int xx = ox * s - p + t;
                if (xx < 0 || xx >= W) continue;
                m = fmaxf(m, x[(((long long)b * H + y) * W + xx) * C + c]);
            }
        }
        out[i] = m;
    }
}

// float4 variants with 32-bit index arithmetic (C % 4 == 0, fewer than 2^31 vectors): the
// scalar kernels above spend most of their time in 64-bit div/mod per element.
__global__ void tdc_im2col4_kernel(const float4 *__restrict__ x, float4 *__restrict__ out, int B, int H, int W,
                                   int C4, int K, int s, int p, int Ho, int Wo, int ld4) {
    const int total = B * Ho * Wo * ld4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int col = i % ld4, row = i / ld4;
        float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
        if (col < K * K * C4) {
            const int c = col % C4, rt = col / C4, t = rt % K, r = rt / K;
            const int ox = row % Wo, t2 = row / Wo, oy = t2 % Ho, b = t2 / Ho;
            const int y = oy * s - p + r, xx = ox * s - p + t;
            if (y >= 0 && y < H && xx >= 0 && xx < W) v = __ldg(x + (((size_t)b * H + y) * W + xx) * C4 + c);
        }
        out[i] = v;
    }
}
__global__ void tdc_maxpool4_kernel(const float4 *__restrict__ x, float4 *__restrict__ out, int B, int H, int W,
                                    int C4, int K, int s, int p, int Ho, int Wo) {
    const int total = B * Ho * Wo * C4;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int c = i % C4, pix = i / C4, ox = pix % Wo, t2 = pix / Wo, oy = t2 % Ho, b = t2 / Ho;
        float4 m = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        for (int r = 0; r < K; ++r) {
            const int y = oy * s - p + r;
            if (y < 0 || y >= H) continue;
            for (int t = 0; t < K; ++t) {
                const int xx = ox * s - p + t;
                if (xx < 0 || xx >= W) continue;
                const float4 v = __ldg(x + (((size_t)b * H + y) * W + xx) * C4 + c);
                m.x = fmaxf(m.x, v.x); m.y = fmaxf(m.y, v.y); m.z = fmaxf(m.z, v.z); m.w = fmaxf(m.w, v.w);
            }
        }
        out[i] = m;
    }
}

// one block per (image, 256-channel slice): fixed-order sum over H*W (deterministic)
__global__ void tdc_avgpool_kernel(const float *__restrict__ x, float *__restrict__ out, int HW, int C) {
    const int b = blockIdx.y;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const float *p = x + (long long)b * HW * C + c;
    float s = 0.f;
    for (int i = 0; i < HW; ++i) s += p[(long long)i * C];
    out[(long long)b * C + c] = s / (float)HW;
}

// Direct fp32 convolution for thin inputs (C <= 4: the stem), one thread per output
// pixel and 64 output channels in registers; weights [K][K][C][N] (BN folded) staged in
// shared memory and read as broadcasts.  Avoids a K*K*C-wide im2col round trip.
constexpr int kDirectCo = 64;
__global__ void __launch_bounds__(128) tdc_direct_conv_kernel(const float *__restrict__ x,
                                                               const float *__restrict__ w,
                                                               const float *__restrict__ bias, float *__restrict__ y,
                                                               int B, int H, int W, int C, int N, int K, int s, int p,
                                                               int Ho, int Wo, int relu) {
    extern __shared__ float ws[];
    const int KKC = K * K * C;
    const int n0 = blockIdx.y * kDirectCo;
    const int nc = min(kDirectCo, N - n0);
    for (int i = threadIdx.x; i < KKC * kDirectCo; i += blockDim.x) {
        const int n = i % kDirectCo, k = i / kDirectCo;
        ws[i] = n < nc ? w[(size_t)k * N + n0 + n] : 0.f;
    }
    __syncthreads();
    const long long pix = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= (long long)B * Ho * Wo) return;
    const int ox = (int)(pix % Wo), oy = (int)((pix / Wo) % Ho), b = (int)(pix / ((long long)Wo * Ho));
    float acc[kDirectCo];
#pragma unroll
    for (int n = 0; n < kDirectCo; ++n) acc[n] = 0.f;
    for (int r = 0; r < K; ++r) {
        const int iy = oy * s - p + r;
        if (iy < 0 || iy >= H) continue;
        for (int t = 0; t < K; ++t) {
            const int ix = ox * s - p + t;
            if (ix < 0 || ix >= W) continue;
            const float *xp = x + (((long long)b * H + iy) * W + ix) * C;
            for (int c = 0; c < C; ++c) {
                const float xv = __ldg(xp + c);
                const float *wr = ws + ((r * K + t) * C + c) * kDirectCo;
#pragma unroll
                for (int n = 0; n < kDirectCo; ++n) acc[n] = fmaf(xv, wr[n], acc[n]);
            }
        }
    }
    float *yp = y + pix * N + n0;
    for (int n = 0; n < nc; n += 4) {
        float4 v;
        v.x = acc[n] + (bias ? bias[n0 + n] : 0.f);
        v.y = acc[n + 1] + (bias ? bias[n0 + n + 1] : 0.f);
        v.z = acc[n + 2] + (bias ? bias[n0 + n + 2] : 0.f);
        v.w = acc[n + 3] + (bias ? bias[n0 + n + 3] : 0.f);
        if (relu) {
            v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
        }
        *reinterpret_cast<float4 *>(yp + n) = v;
    }
}

// The 3-channel stems (ResNet 7x7/2, VGG 3x3/1) with 64 outputs, specialised: a block
// computes a 16 x 16 output tile from a zero-padded input patch staged in shared memory
// (no bounds checks in the loop).  Warp w owns output channels [16w, 16w + 16) (so its
// weight reads are broadcasts), lane l 8 pixels of tile column l % 16: per tap and input
// channel, 8 scalar x loads and 4 float4 weight loads feed 128 FMAs.  The finished tile
// is transposed through shared memory and written as contiguous 8 KB pixel rows.
constexpr int kStemTH = 16, kStemTW = 16, kStemPL = 8;  // tile rows, cols; pixels per lane
template <int K, int S>
__host__ __device__ constexpr int stem_smem_floats() {
    return (K * K * 3 * 64 + ((kStemTH - 1) * S + K) * ((kStemTW - 1) * S + K) * 3) > kStemTH * kStemTW * 64
               ? (K * K * 3 * 64 + ((kStemTH - 1) * S + K) * ((kStemTW - 1) * S + K) * 3)
               : kStemTH * kStemTW * 64;
}
template <int K, int S>
__global__ void __launch_bounds__(128, 3) tdc_stem_kernel(const float *__restrict__ x, const float *__restrict__ w,
                                                        const float *__restrict__ bias, float *__restrict__ y, int H,
                                                        int W, int p, int Ho, int Wo, int relu) {
    constexpr int C = 3, N = 64, PH = (kStemTH - 1) * S + K, PW = (kStemTW - 1) * S + K;
    extern __shared__ float sm[];
    float *ws = sm;                    // [K*K*C][64]
    float *xs = sm + K * K * C * N;    // [PH][PW][C], zero outside the image
    const int tiles_x = (Wo + kStemTW - 1) / kStemTW, tiles_y = (Ho + kStemTH - 1) / kStemTH;
    const int tx = blockIdx.x % tiles_x, ty = (blockIdx.x / tiles_x) % tiles_y, b = blockIdx.x / (tiles_x * tiles_y);
    for (int i = threadIdx.x; i < K * K * C * N / 4; i += blockDim.x)
        reinterpret_cast<float4 *>(ws)[i] = __ldg(reinterpret_cast<const float4 *>(w) + i);
    const int iy0 = ty * kStemTH * S - p, ix0 = tx * kStemTW * S - p;
    for (int i = threadIdx.x; i < PH * PW; i += blockDim.x) {
        const int py = i / PW, px = i % PW, iy = iy0 + py, ix = ix0 + px;
        const bool in = iy >= 0 && iy < H && ix >= 0 && ix < W;
        const float *src = x + (((size_t)b * H + (in ? iy : 0)) * W + (in ? ix : 0)) * C;
#pragma unroll
        for (int c = 0; c < C; ++c) xs[i * C + c] = in ? __ldg(src + c) : 0.f;
    }
    __syncthreads();
    const int wq = threadIdx.x >> 5, lane = threadIdx.x & 31, col = lane & 15, rh = lane >> 4;
    float acc[kStemPL][16];  // lane's pixels: tile rows rh*8 .. rh*8+7 of column col
#pragma unroll
    for (int i = 0; i < kStemPL; ++i)
#pragma unroll
        for (int n = 0; n < 16; ++n) acc[i][n] = 0.f;
#pragma unroll 1
    for (int r = 0; r < K; ++r) {
#pragma unroll
        for (int t = 0; t < K; ++t)
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const float4 *wr = reinterpret_cast<const float4 *>(ws + ((r * K + t) * C + c) * N + 16 * wq);
                const float4 w0 = wr[0], w1 = wr[1], w2 = wr[2], w3 = wr[3];
                const float wv[16] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w,
                                      w2.x, w2.y, w2.z, w2.w, w3.x, w3.y, w3.z, w3.w};
#pragma unroll
                for (int i = 0; i < kStemPL; ++i) {
                    const float xv = xs[(((rh * kStemPL + i) * S + r) * PW + col * S + t) * C + c];
#pragma unroll
                    for (int n = 0; n < 16; ++n) acc[i][n] = fmaf(xv, wv[n], acc[i][n]);
                }
            }
    }
    __syncthreads();  // done with the weights / patch: reuse shared memory for the output tile
    float *ys = sm;   // [TH][TW][64], 16-byte chunks of a pixel rotated by the pixel index
#pragma unroll
    for (int i = 0; i < kStemPL; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int px = (rh * kStemPL + i) * kStemTW + col, ch4 = (wq * 4 + j + px) & 15;
            float4 v = make_float4(acc[i][4 * j] + bias[16 * wq + 4 * j], acc[i][4 * j + 1] + bias[16 * wq + 4 * j + 1],
                                   acc[i][4 * j + 2] + bias[16 * wq + 4 * j + 2], acc[i][4 * j + 3] + bias[16 * wq + 4 * j + 3]);
            if (relu) {
                v.x = fmaxf(v.x, 0.f); v.y = fmaxf(v.y, 0.f); v.z = fmaxf(v.z, 0.f); v.w = fmaxf(v.w, 0.f);
            }
            reinterpret_cast<float4 *>(ys)[px * 16 + ch4] = v;
        }
    __syncthreads();
    const int ox0 = tx * kStemTW, nx = min(kStemTW, Wo - ox0);
    for (int i = 0; i < kStemTH; ++i) {
        const int oy = ty * kStemTH + i;
        if (oy >= Ho) break;
        float4 *dst = reinterpret_cast<float4 *>(y + (((size_t)b * Ho + oy) * Wo + ox0) * N);
        for (int e = threadIdx.x; e < nx * 16; e += blockDim.x) {  // contiguous row of nx pixels
            const int px = i * kStemTW + e / 16, ch4 = e % 16;
            dst[e] = reinterpret_cast<const float4 *>(ys)[px * 16 + ((ch4 + px) & 15)];
        }
    }
}

template <int K, int S>
cudaError_t stem_launch(const float *x, const float *w, const float *bias, float *y, int B, int H, int W, int p,
                        int Ho, int Wo, int relu, cudaStream_t st) {
    const int smem = stem_smem_floats<K, S>() * 4;
    cudaError_t e = cudaFuncSetAttribute(tdc_stem_kernel<K, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    const int blocks = B * ((Ho + kStemTH - 1) / kStemTH) * ((Wo + kStemTW - 1) / kStemTW);
    tdc_stem_kernel<K, S><<<blocks, 128, smem, st>>>(x, w, bias, y, H, W, p, Ho, Wo, relu);
    return cudaGetLastError();
}

int ew_grid(long long n) { return (int)std::min<long long>(div_up((int)std::min<long long>(n, 1LL << 30), 256), 148 * 16); }

// ------------------------------------------------------------------ dense GEMM op
struct DenseOp {
    int Kdim = 0;            // GEMM K (C for a plain 1x1, else the padded im2col row)
    bool im2col = false;
    bool direct = false;     // thin input (C <= 4, N % 4 == 0): tdc_direct_conv_kernel
    float *d_wdirect = nullptr;  // [K][K][C][N] fp32, BN folded, then the bias
    uint16_t *d_w = nullptr;  // [hi | lo] bf16 panels [R][K64], then fp32 bias
    float *d_gs = nullptr;    // split-K through L2: partial tiles | flags (few-tile long-K GEMMs)
    float *d_bias = nullptr;
    tdc::TcGemmArgs args;
    CUtensorMap mapA, mapB, mapBlo;
    const float *mapA_src = nullptr;
    long long mapA_rows = 0;  // the A map's row extent = this call's rows (loads past it zero-fill)
    CUtensorMap mapY;        // TMA map of the output (tma_y), re-encoded when dst changes
    const float *mapY_dst = nullptr;
    long long mapY_rows = 0;  // the map's row extent = this call's rows (TMA stores clip there)
    CUtensorMap mapR;        // TMA map of the residual (tma_y with a residual)
    const float *mapR_src = nullptr;
    long long mapR_rows = 0;
};

}  // namespace

struct ModelOp {
    tdc_model_op d;
    int H = 0, W = 0, C = 0, Ho = 0, Wo = 0, Co = 0;
    tdc_conv_plan_t tkd = nullptr;
    DenseOp dense;
};

struct tdc_model_s {
    std::vector<ModelOp> ops;
    std::vector<float *> act;  // act[id]: id 0 = the caller's input (not owned)
    float *scratch = nullptr;  // im2col buffer
    int max_batch = 0, device = 0, num_sms = 148, max_smem = 0;
};

namespace {

struct Guard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit Guard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~Guard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

// BN fold: y = g/sqrt(v+eps) * (conv + b - m) + beta  ->  scale, bias'
void bn_fold(const tdc_model_op &o, int Co, std::vector<double> &scale, std::vector<double> &bias) {
    scale.assign(Co, 1.0);
    bias.assign(Co, 0.0);
    for (int n = 0; n < Co; ++n) {
        const double b0 = o.bias ? o.bias[n] : 0.0;
        if (o.bn) {
            const double g = o.bn[n], be = o.bn[Co + n], m = o.bn[2 * Co + n], v = o.bn[3 * Co + n];
            scale[n] = g / std::sqrt(v + (double)kBnEps);
            bias[n] = scale[n] * (b0 - m) + be;
        } else {
            bias[n] = b0;
        }
    }
}

// `o` is the caller's op (host weight pointers valid only during tdc_model_create)
tdc_status plan_dense(tdc_model_s *m, ModelOp &op, const tdc_model_op &o) {
    DenseOp &g = op.dense;
    const int K = o.kind == TDC_OP_FC ? 1 : o.kernel;
    const int C = op.C, N = op.Co;
    if (o.kind == TDC_OP_CONV && o.res < 0 && C <= 4 && N % 4 == 0 && K * K * C * kDirectCo * 4 <= 96 * 1024) {
        g.direct = true;
        std::vector<double> scale, bias;
        bn_fold(o, N, scale, bias);
        std::vector<float> h((size_t)K * K * C * N + N);
        for (int n = 0; n < N; ++n) {
            for (int c = 0; c < C; ++c)
                for (int r = 0; r < K; ++r)
                    for (int t = 0; t < K; ++t)
                        h[((size_t)(r * K + t) * C + c) * N + n] =
                            (float)(scale[n] * o.w[(((size_t)n * C + c) * K + r) * K + t]);
            h[(size_t)K * K * C * N + n] = (float)bias[n];
        }
        cudaError_t e = cudaMalloc(&g.d_wdirect, h.size() * sizeof(float));
        if (e == cudaSuccess) e = cudaMemcpy(g.d_wdirect, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice);
        if (e != cudaSuccess) return mcuda(e, "direct conv weights");
        return TDC_OK;
    }
    g.im2col = !(K == 1 && o.stride == 1 && o.pad == 0 && C % 4 == 0);
    g.Kdim = g.im2col ? round_up(K * K * C, 32) : C;
    const int K64 = round_up(g.Kdim, 64);
    const long long Mmax = (long long)m->max_batch * op.Ho * op.Wo;
    if (Mmax > (1LL << 31) - 256) return mfail(TDC_ERR_UNSUPPORTED, "op too large (M=%lld rows)", Mmax);
    int BN = 32;
    const int bn_cap = std::getenv("TDC_DENSE_BN") ? std::atoi(std::getenv("TDC_DENSE_BN")) : 128;
    while (BN < N && BN < bn_cap) BN *= 2;
    // (N tile, split-K pieces) from a streaming model: every K chunk of a
    // work unit moves 32 KB of fp32 A and 256*BN B bytes into the SM; A is re-read once per
    // N tile and B once per M tile.  A CTA streams at ~40 GB/s and the chip at ~5 TB/s
    // (measured on these kernels), so time ~ max(per-CTA bytes / 40 GB/s, all bytes /
    // 5 TB/s) + the split-K fix-up traffic.  Pieces > 1 only when K is long (>= 8 chunks).
    int gsp = 1;
    {
        const int mt = div_up((int)Mmax, 128), kch = K64 / 64, top = BN;
        const bool gs_ok = kch >= 8 && !std::getenv("TDC_DENSE_NO_GSPLIT");
        double best = 1e30;
        int bbn = BN;
        for (int b = top; b >= 32 && b >= top / 4; b /= 2)
            for (int gq = 1; gq <= (gs_ok ? std::min(8, kch / 4) : 1); ++gq) {
                const long long units = (long long)mt * div_up(N, b) * gq;
                const double unit_bytes = (double)div_up(kch, gq) * (32768.0 + 256.0 * b);
                const double waves = (double)div_up((int)units, m->num_sms);
                const double t = std::max(waves * unit_bytes / 40e3, units * unit_bytes / 5e6) +
                                 (gq > 1 ? 2.0 + (gq - 1) * (double)mt * div_up(N, b) * 128 * b * 8 / 5e6 : 0.0);
                if (t < best * 0.97) {
                    best = t;
                    bbn = b;
                    gsp = gq;
                }
            }
        BN = bbn;
    }
    const int R = round_up(N, BN);
    std::vector<double> scale, bias;
    bn_fold(o, N, scale, bias);
    const size_t nw = (size_t)R * K64;
    std::vector<uint16_t> hb(2 * nw, 0);
    for (int n = 0; n < N; ++n)
        for (int r = 0; r < K; ++r)
            for (int t = 0; t < K; ++t)
                for (int c = 0; c < C; ++c) {
                    const double wv = (o.kind == TDC_OP_FC ? (double)o.w[(size_t)n * C + c]
                                                           : (double)o.w[(((size_t)n * C + c) * K + r) * K + t]) *
                                      scale[n];
                    const float f = (float)wv;
                    const size_t col = g.im2col ? (size_t)(r * K + t) * C + c : (size_t)c;
                    const uint16_t hi = tdc::bf16_bits(f);
                    hb[(size_t)n * K64 + col] = hi;
                    hb[nw + (size_t)n * K64 + col] = tdc::bf16_bits(f - tdc::bf16_float(hi));
                }
    const size_t wbytes = hb.size() * sizeof(uint16_t), nb = round_up(N, 4);
    cudaError_t e = cudaMalloc(&g.d_w, wbytes + nb * sizeof(float));
    if (e != cudaSuccess) return mcuda(e, "cudaMalloc(dense weights)");
    e = cudaMemcpy(g.d_w, hb.data(), wbytes, cudaMemcpyHostToDevice);
    std::vector<float> bf(nb, 0.f);
    for (int n = 0; n < N; ++n) bf[n] = (float)bias[n];
    g.d_bias = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(g.d_w) + wbytes);
    if (e == cudaSuccess) e = cudaMemcpy(g.d_bias, bf.data(), nb * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return mcuda(e, "cudaMemcpy(dense weights)");
    std::memset(&g.args, 0, sizeof g.args);
    tdc::TcGemmArgs &a = g.args;
    a.Nn = N; a.kchunks = K64 / 64; a.taps = 1; a.BN = BN; a.remap = 0; a.a_convert = 1; a.out_bf16 = 0;
    a.ldo = N; a.bias = g.d_bias; a.relu = o.relu; a.ntiles = R / BN; a.ksplit = 1;
    // output ring: 2 buffers per epilogue warp (residual block loaded one chunk ahead);
    // TDC_DENSE_RING=4 asks for 4 (two chunks ahead) if shared memory allows
    a.yring = 2;  // shared memory goes to the fp32 staging ring first (measured)
    if (const char *ev = std::getenv("TDC_DENSE_RING")) a.yring = std::atoi(ev) > 2 ? 4 : 2;
    a.stages = tdc::bf_pick_stages(BN, m->max_smem, 1, &a.xstages, 1, &a.bstages, a.yring);
    if (tdc::bf_smem_bytes(BN, a.stages, a.xstages, 1, a.bstages, a.yring) > m->max_smem) {
        a.yring = 2;
        a.stages = tdc::bf_pick_stages(BN, m->max_smem, 1, &a.xstages, 1, &a.bstages, a.yring);
    }
    if (const char *dbg = std::getenv("TDC_GEMM_DBG")) a.dbg = std::atoi(dbg);
    {
        const char *ev = std::getenv("TDC_NO_TMA_Y");
        a.tma_y = N % 4 == 0 && !(ev && ev[0] && ev[0] != '0');
    }
    // Split-K through L2 (gsplit) for the few-tile, long-K GEMMs (classifiers, the VGG FC1
    // 7x7 conv): the K loop is cut into fixed pieces spread over the idle SMs; the piece-0
    // CTA adds the partials in piece order (deterministic) and runs the epilogue.
    {
        const long long tiles = (long long)div_up((int)Mmax, 128) * (R / BN);
        if (gsp > 1) {
            const size_t parts = (size_t)tiles * (gsp - 1) * 128 * BN, flags = (size_t)tiles * (gsp - 1);
            e = cudaMalloc(&g.d_gs, parts * sizeof(float) + flags * sizeof(int));
            if (e == cudaSuccess) e = cudaMemset(g.d_gs, 0, parts * sizeof(float) + flags * sizeof(int));
            if (e != cudaSuccess) return mcuda(e, "cudaMalloc(dense split-K workspace)");
            a.gsplit = gsp;
            a.part = g.d_gs;
            a.flags = reinterpret_cast<int *>(g.d_gs + parts);
        }
    }
    if (!tdc::make_tma_2d_bf16(&g.mapB, g.d_w, R, K64, K64, BN) ||
        !tdc::make_tma_2d_bf16(&g.mapBlo, g.d_w + nw, R, K64, K64, BN))
        return mfail(TDC_ERR_CUDA, "cuTensorMapEncodeTiled failed (dense weights)");
    return TDC_OK;
}

tdc_status run_dense(tdc_model_s *m, ModelOp &op, const float *src, float *dst, const float *res, int batch,
                     cudaStream_t st) {
    DenseOp &g = op.dense;
    const tdc_model_op &o = op.d;
    const long long M = (long long)batch * op.Ho * op.Wo;
    if (g.direct && op.C == 3 && op.Co == 64 && !std::getenv("TDC_NO_STEM") &&
        ((o.kernel == 7 && o.stride == 2) || (o.kernel == 3 && o.stride == 1))) {
        const float *wd = g.d_wdirect, *bd = g.d_wdirect + (size_t)o.kernel * o.kernel * 3 * 64;
        cudaError_t e = o.kernel == 7
                            ? stem_launch<7, 2>(src, wd, bd, dst, batch, op.H, op.W, o.pad, op.Ho, op.Wo, o.relu, st)
                            : stem_launch<3, 1>(src, wd, bd, dst, batch, op.H, op.W, o.pad, op.Ho, op.Wo, o.relu, st);
        if (e != cudaSuccess) return mcuda(e, "stem conv launch");
        return TDC_OK;
    }
    if (g.direct) {
        const int K = o.kernel, C = op.C, N = op.Co;
        const int smem = K * K * C * kDirectCo * 4;
        cudaError_t e = cudaFuncSetAttribute(tdc_direct_conv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return mcuda(e, "direct conv attribute");
        dim3 grid((unsigned)div_up((int)M, 128), (unsigned)div_up(N, kDirectCo));
        tdc_direct_conv_kernel<<<grid, 128, smem, st>>>(src, g.d_wdirect, g.d_wdirect + (size_t)K * K * C * N, dst,
                                                        batch, op.H, op.W, C, N, K, o.stride, o.pad, op.Ho, op.Wo,
                                                        o.relu);
        e = cudaGetLastError();
        if (e != cudaSuccess) return mcuda(e, "direct conv launch");
        return TDC_OK;
    }
    const float *A = src;
    if (g.im2col) {
        const int K = o.kind == TDC_OP_FC ? 1 : o.kernel;
        const long long n = M * g.Kdim;
        if (op.C % 4 == 0 && g.Kdim % 4 == 0 && n / 4 < (1LL << 31))
            tdc_im2col4_kernel<<<ew_grid(n / 4), 256, 0, st>>>(reinterpret_cast<const float4 *>(src),
                                                                reinterpret_cast<float4 *>(m->scratch), batch, op.H,
                                                                op.W, op.C / 4, K, o.stride, o.pad, op.Ho, op.Wo,
                                                                g.Kdim / 4);
        else
            tdc_im2col_kernel<<<ew_grid(n), 256, 0, st>>>(src, m->scratch, batch, op.H, op.W, op.C, K, o.stride,
                                                           o.pad, op.Ho, op.Wo, g.Kdim);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return mcuda(e, "im2col launch");
        A = m->scratch;
    }
    // extent = this call's rows, so the last M tile of a partial batch is zero-filled instead
    // of reading past a caller's input sized for `batch`
    if (A != g.mapA_src || M != g.mapA_rows) {
        if (!tdc::make_tma_2d(&g.mapA, A, M, g.Kdim, g.Kdim, 128))
            return mfail(TDC_ERR_INVALID_ARGUMENT, "cuTensorMapEncodeTiled rejected a dense-op input (16-byte aligned?)");
        g.mapA_src = A;
        g.mapA_rows = M;
    }
    tdc::TcGemmArgs a = g.args;
    a.M = (int)M;
    a.out = dst;
    a.res = res;
    const int smem = tdc::bf_smem_bytes(a.BN, a.stages, a.xstages, 1, a.bstages, a.yring);
    const long long tiles = (long long)div_up((int)M, 128) * a.ntiles * std::max(1, a.gsplit);
    // split-K: at most one CTA per SM, so every CTA is co-resident (piece-0 CTAs wait on others)
    const long long cap = a.gsplit > 1 ? (long long)m->num_sms
                                       : (long long)m->num_sms * tdc::persistent_occupancy(smem, a.BN);
    const int grid = (int)std::max<long long>(1, std::min(tiles, cap));
    if (a.tma_y && (dst != g.mapY_dst || M != g.mapY_rows)) {
        // extent = this call's rows: the last tile's 32-row blocks past M are clipped, not
        // written past a partial batch
        if (!tdc::make_tma_2d(&g.mapY, dst, M, op.Co, op.Co, 32))
            return mfail(TDC_ERR_INVALID_ARGUMENT, "cuTensorMapEncodeTiled rejected a dense-op output");
        g.mapY_dst = dst;
        g.mapY_rows = M;
    }
    if (a.tma_y && res && (res != g.mapR_src || M != g.mapR_rows)) {
        if (!tdc::make_tma_2d(&g.mapR, res, M, op.Co, op.Co, 32))
            return mfail(TDC_ERR_INVALID_ARGUMENT, "cuTensorMapEncodeTiled rejected a residual input");
        g.mapR_src = res;
        g.mapR_rows = M;
    }
    cudaError_t e = tdc::bf_gemm_launch(g.mapA, g.mapA, g.mapB, g.mapBlo, a.tma_y ? g.mapY : g.mapA, a, grid, st,
                                        (a.tma_y && res) ? &g.mapR : nullptr);
    if (e != cudaSuccess) return mcuda(e, "dense GEMM launch");
    return TDC_OK;
}

void destroy(tdc_model_s *m) {
    for (auto &op : m->ops) {
        if (op.tkd) tdc_conv_plan_destroy(op.tkd);
        if (op.dense.d_w) cudaFree(op.dense.d_w);
        if (op.dense.d_gs) cudaFree(op.dense.d_gs);
        if (op.dense.d_wdirect) cudaFree(op.dense.d_wdirect);
    }
    for (size_t i = 1; i < m->act.size(); ++i)
        if (m->act[i]) cudaFree(m->act[i]);
    if (m->scratch) cudaFree(m->scratch);
    delete m;
}

}  // namespace

extern "C" {

tdc_status tdc_model_create(const tdc_model_op *ops, int32_t n_ops, int32_t max_batch, int32_t device,
                            tdc_model_t *out) {
    if (!out) return mfail(TDC_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (!ops || n_ops < 1) return mfail(TDC_ERR_INVALID_ARGUMENT, "need at least one op");
    if (max_batch < 1) return mfail(TDC_ERR_INVALID_ARGUMENT, "max_batch must be >= 1");
    Guard guard(device);
    if (guard.err != cudaSuccess) return mcuda(guard.err, "cudaSetDevice");
    tdc_model_s *m = new tdc_model_s;
    m->max_batch = max_batch;
    m->device = device;
    m->num_sms = tdc::num_sms_of(device);
    m->max_smem = tdc::max_smem_of(device);
    m->ops.resize(n_ops);
    m->act.assign(n_ops + 1, nullptr);
    // geometry of every id: id 0 = first op's input
    std::vector<int> gh(n_ops + 1), gw(n_ops + 1), gc(n_ops + 1);
    gh[0] = ops[0].height; gw[0] = ops[0].width; gc[0] = ops[0].c_in;
    size_t scratch = 0;
    for (int i = 0; i < n_ops; ++i) {
        const tdc_model_op &o = ops[i];
        ModelOp &op = m->ops[i];
        op.d = o;
        op.d.w = op.d.u_in = op.d.u_out = op.d.bias = op.d.bn = nullptr;
        auto bad = [&](const char *why) {
            destroy(m);
            return mfail(TDC_ERR_INVALID_ARGUMENT, "op %d: %s", i, why);
        };
        if (o.src < 0 || o.src > i) return bad("src id must refer to the input (0) or an earlier op");
        if (o.res < -1 || o.res > i) return bad("res id must be -1 or refer to an earlier op");
        if (o.c_in != gc[o.src] || o.height != gh[o.src] || o.width != gw[o.src])
            return bad("input geometry (c_in, height, width) does not match the src activation");
        op.H = o.height; op.W = o.width; op.C = o.c_in;
        switch (o.kind) {
            case TDC_OP_CONV:
            case TDC_OP_TKD:
            case TDC_OP_MAXPOOL:
                if (o.kernel < 1 || o.stride < 1 || o.pad < 0 || o.kernel > o.height + 2 * o.pad ||
                    o.kernel > o.width + 2 * o.pad)
                    return bad("kernel/stride/pad out of range");
                op.Ho = (o.height + 2 * o.pad - o.kernel) / o.stride + 1;
                op.Wo = (o.width + 2 * o.pad - o.kernel) / o.stride + 1;
                op.Co = o.kind == TDC_OP_MAXPOOL ? o.c_in : o.c_out;
                break;
            case TDC_OP_AVGPOOL:
                op.Ho = op.Wo = 1;
                op.Co = o.c_in;
                break;
            case TDC_OP_FC:
                if (o.height != 1 || o.width != 1) return bad("FC needs a 1x1 input (use AVGPOOL first)");
                op.Ho = op.Wo = 1;
                op.Co = o.c_out;
                break;
            default:
                return bad("unknown op kind");
        }
        if (op.Co < 1) return bad("c_out must be positive");
        if ((o.kind == TDC_OP_CONV || o.kind == TDC_OP_TKD || o.kind == TDC_OP_FC) && !o.w)
            return bad("weights missing");
        if (o.kind == TDC_OP_TKD && (!o.u_in || !o.u_out)) return bad("TKD factors missing");
        if (o.res >= 0 && (gc[o.res] != op.Co || gh[o.res] != op.Ho || gw[o.res] != op.Wo))
            return bad("residual geometry does not match the output");
        if (o.res >= 0 && (o.kind == TDC_OP_MAXPOOL || o.kind == TDC_OP_AVGPOOL)) return bad("pools take no residual");
        gh[i + 1] = op.Ho; gw[i + 1] = op.Wo; gc[i + 1] = op.Co;
        const size_t elems = (size_t)max_batch * op.Ho * op.Wo * op.Co;
        cudaError_t e = cudaMalloc(&m->act[i + 1], elems * sizeof(float));
        if (e != cudaSuccess) {
            destroy(m);
            return mcuda(e, "cudaMalloc(activation)");
        }
        tdc_status s = TDC_OK;
        if (o.kind == TDC_OP_TKD) {
            std::vector<double> scale, bias;
            bn_fold(o, op.Co, scale, bias);
            std::vector<float> uo((size_t)op.Co * o.rank_out), bb(op.Co);
            for (int n = 0; n < op.Co; ++n) {
                for (int q = 0; q < o.rank_out; ++q)
                    uo[(size_t)n * o.rank_out + q] = (float)(scale[n] * o.u_out[(size_t)n * o.rank_out + q]);
                bb[n] = (float)bias[n];
            }
            tdc_conv_desc d;
            std::memset(&d, 0, sizeof d);
            d.batch = max_batch; d.c_in = o.c_in; d.height = o.height; d.width = o.width; d.c_out = o.c_out;
            d.rank_in = o.rank_in; d.rank_out = o.rank_out; d.kernel = o.kernel; d.stride = o.stride;
            d.pad = o.pad; d.layout = TDC_LAYOUT_NHWC; d.math = TDC_MATH_3XBF16;
            s = tdc_conv_plan(&d, o.w, o.u_in, uo.data(), bb.data(), device, &op.tkd);
            if (s == TDC_OK) {
                tdc_plan_info info;
                tdc_conv_plan_query(op.tkd, &info);
                if (info.variant != 4 && info.variant != 5)  // 3-launch or single-launch 3xBF16
                    s = mfail(TDC_ERR_UNSUPPORTED, "op %d: TKD layer did not get the 3xBF16 tensor-core plan", i);
            }
        } else if (o.kind == TDC_OP_CONV || o.kind == TDC_OP_FC) {
            s = plan_dense(m, op, o);
            if (s == TDC_OK && op.dense.im2col)
                scratch = std::max(scratch, (size_t)max_batch * op.Ho * op.Wo * op.dense.Kdim);
        }
        if (s != TDC_OK) {
            std::string msg = tdc_last_error();
            destroy(m);
            return tdc::set_error(s, msg.c_str());
        }
    }
    if (scratch) {
        cudaError_t e = cudaMalloc(&m->scratch, scratch * sizeof(float));
        if (e != cudaSuccess) {
            destroy(m);
            return mcuda(e, "cudaMalloc(im2col scratch)");
        }
    }
    *out = m;
    return TDC_OK;
}

tdc_status tdc_model_forward(tdc_model_t m, const float *x, int32_t batch, float *out, void *stream) {
    if (!m) return mfail(TDC_ERR_INVALID_ARGUMENT, "model is NULL");
    if (!x || !out) return mfail(TDC_ERR_INVALID_ARGUMENT, "x/out is NULL");
    if (batch < 1 || batch > m->max_batch)
        return mfail(TDC_ERR_INVALID_ARGUMENT, "batch %d outside [1, %d]", batch, m->max_batch);
    Guard guard(m->device);
    if (guard.err != cudaSuccess) return mcuda(guard.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    const int n = (int)m->ops.size();
    auto ptr = [&](int id) -> float * {
        if (id == 0) return const_cast<float *>(x);
        return id == n ? out : m->act[id];
    };
    for (int i = 0; i < n; ++i) {
        ModelOp &op = m->ops[i];
        const tdc_model_op &o = op.d;
        const float *src = ptr(o.src);
        float *dst = ptr(i + 1);
        const float *res = o.res >= 0 ? ptr(o.res) : nullptr;
        tdc_status s = TDC_OK;
        cudaError_t e = cudaSuccess;
        switch (o.kind) {
            case TDC_OP_TKD:
                s = tdc_conv_forward_ex(op.tkd, src, dst, batch, res, o.relu, stream);
                break;
            case TDC_OP_CONV:
            case TDC_OP_FC:
                s = run_dense(m, op, src, dst, res, batch, st);
                break;
            case TDC_OP_MAXPOOL: {
                const long long tot = (long long)batch * op.Ho * op.Wo * op.Co;
                if (op.C % 4 == 0 && tot / 4 < (1LL << 31))
                    tdc_maxpool4_kernel<<<ew_grid(tot / 4), 256, 0, st>>>(
                        reinterpret_cast<const float4 *>(src), reinterpret_cast<float4 *>(dst), batch, op.H, op.W,
                        op.C / 4, o.kernel, o.stride, o.pad, op.Ho, op.Wo);
                else
                    tdc_maxpool_kernel<<<ew_grid(tot), 256, 0, st>>>(src, dst, batch, op.H, op.W, op.C, o.kernel,
                                                                     o.stride, o.pad, op.Ho, op.Wo);
                e = cudaGetLastError();
                break;
            }
            case TDC_OP_AVGPOOL: {
                dim3 grid(div_up(op.C, 256), batch);
                tdc_avgpool_kernel<<<grid, 256, 0, st>>>(src, dst, op.H * op.W, op.C);
                e = cudaGetLastError();
                break;
            }
        }
        if (e != cudaSuccess) return mcuda(e, "pool launch");
        if (s != TDC_OK) {
            std::string msg = tdc_last_error();
            return mfail(s, "op %d: %s", i, msg.c_str());
        }
    }
    return TDC_OK;
}

tdc_status tdc_model_output_shape(tdc_model_t m, int32_t op, int32_t *h, int32_t *w, int32_t *c) {
    if (!m || !h || !w || !c) return mfail(TDC_ERR_INVALID_ARGUMENT, "NULL argument");
    if (op >= (int)m->ops.size()) return mfail(TDC_ERR_INVALID_ARGUMENT, "op %d out of range", op);
    const ModelOp &o = m->ops[op < 0 ? m->ops.size() - 1 : (size_t)op];
    *h = o.Ho;
    *w = o.Wo;
    *c = o.Co;
    return TDC_OK;
}

tdc_status tdc_model_destroy(tdc_model_t m) {
    if (!m) return TDC_OK;
    Guard guard(m->device);
    destroy(m);
    return TDC_OK;
}

}  // extern "C"
