// tdc_api.cu -- the C-ABI of include/tdc.h: validation, plan-time weight
// re-layout (§8(a) row a0), variant selection and forward dispatch.
#include "../../include/tdc.h"
#include "internal.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

namespace tdc {
bool pdl_enabled() {
    static const bool on = [] {
        const char *v = std::getenv("TDC_NO_PDL");
        return !(v && v[0] && v[0] != '0');
    }();
    return on;
}
}  // namespace tdc

namespace {

thread_local std::string g_last_error;

tdc_status fail(tdc_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

tdc_status cuda_fail(cudaError_t e, const char *what) {
    if (e == cudaErrorMemoryAllocation)
        return fail(TDC_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
    return fail(TDC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// Restores the caller's current device on scope exit.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

int round_up(int v, int m) { return (v + m - 1) / m * m; }

tdc_status validate_desc(const tdc_conv_desc *d, int *ho, int *wo) {
    if (!d) return fail(TDC_ERR_INVALID_ARGUMENT, "desc is NULL");
    if (d->batch < 1 || d->c_in < 1 || d->height < 1 || d->width < 1 || d->c_out < 1 ||
        d->rank_in < 1 || d->rank_out < 1 || d->kernel < 1)
        return fail(TDC_ERR_INVALID_ARGUMENT,
                    "all sizes must be positive (batch=%d C=%d H=%d W=%d N=%d D1=%d D2=%d K=%d)",
                    d->batch, d->c_in, d->height, d->width, d->c_out, d->rank_in, d->rank_out,
                    d->kernel);
    if (d->rank_in > d->c_in || d->rank_out > d->c_out)
        return fail(TDC_ERR_INVALID_ARGUMENT,
                    "rank bounds violated: need 1 <= D1 <= C and 1 <= D2 <= N (D1=%d C=%d D2=%d N=%d)",
                    d->rank_in, d->c_in, d->rank_out, d->c_out);
    if (d->stride < 1 || d->pad < 0)
        return fail(TDC_ERR_INVALID_ARGUMENT, "need stride >= 1 and pad >= 0 (stride=%d pad=%d)",
                    d->stride, d->pad);
    if (d->kernel > d->height + 2 * d->pad || d->kernel > d->width + 2 * d->pad)
        return fail(TDC_ERR_INVALID_ARGUMENT, "kernel %d exceeds padded input %dx%d", d->kernel,
                    d->height + 2 * d->pad, d->width + 2 * d->pad);
    if (d->layout != TDC_LAYOUT_NCHW && d->layout != TDC_LAYOUT_NHWC)
        return fail(TDC_ERR_INVALID_ARGUMENT, "unknown layout %d", d->layout);
    if (d->math < TDC_MATH_FP32 || d->math > TDC_MATH_3XBF16)
        return fail(TDC_ERR_INVALID_ARGUMENT, "unknown math mode %d", d->math);
    const long long elems_in = (long long)d->batch * d->c_in * d->height * d->width;
    if (elems_in > (1LL << 40))
        return fail(TDC_ERR_INVALID_ARGUMENT, "input too large (%lld elements)", elems_in);
    *ho = (d->height + 2 * d->pad - d->kernel) / d->stride + 1;
    *wo = (d->width + 2 * d->pad - d->kernel) / d->stride + 1;
    return TDC_OK;
}

}  // namespace

struct tdc_conv_plan_s {
    tdc_conv_desc desc;
    int device = 0;
    tdc::LayerDims dims;
    int D1p = 0, D2p = 0, Np = 0;
    int variant = 0;
    // packed device weights (one allocation)
    float *d_weights = nullptr;
    size_t weight_bytes = 0;
    tdc::SimtWeights simt;
    tdc::SimtTile simt_tile;
    // NCHW conversion workspace, host-forward staging
    float *d_ws_in = nullptr, *d_ws_out = nullptr;
    size_t ws_bytes = 0;
    float *d_stage_x = nullptr, *d_stage_y = nullptr;
    cudaStream_t s_in = nullptr, s_out = nullptr;  // host-forward pipeline: copy streams
    cudaEvent_t ev[17] = {};                       // per-chunk H2D / forward done, entry
    // tensor-core variant (variant 2): three tcgen05 GEMM-with-taps launches
    struct TcStage {
        tdc::TcGemmArgs args;
        CUtensorMap mapA, mapB, mapAlo, mapBlo;
        int grid_n = 1;
    } tc[3];
    // fused single-kernel variant (variant 3)
    tdc::FusedArgs fargs;
    float *d_fw = nullptr;
    CUtensorMap fmapX;
    const float *f_last_x = nullptr;
    int fgrid = 0, num_sms = 148;
    bool tc_core = false;          // stage 2 uses the band-resident core kernel
    bool split = false;            // 3xTF32
    bool bf16x3 = false;           // 3xBF16 (variant 4 uses tc[] maps + core_args, bf16 formats)

    tdc::TcCoreArgs core_args;
    tdc::BfCoreArgs bf_core;
    bool fuse3 = false;            // 3xBF16: core + stage 3 in one kernel (Z on chip)
    tdc_plan_hints hints = {-1, 0, 0, 0, 0, 0, 0, 0, 0, 0, -1};  // planner overrides (tdc_conv_plan_ex)
    int latency_mode = 0;          // 3xBF16 3-launch plan for a small batch (plan_bf16)
    bool core2 = false;            // 3xBF16 stage 2 on CTA pairs (tdc_bf_core2_kernel)
    void *d_c2w = nullptr;         // its weight image [kc][ntile][hi|lo][tap][plane][BN][8]
    CUtensorMap mapY3;             // 3xBF16 stage 3: TMA map of the output (per y pointer)
    const float *last_y3 = nullptr;
    long long last_y3_rows = 0;
    CUtensorMap mapR3;             // 3xBF16 stage 3: TMA map of the residual (tdc_conv_forward_ex)
    const float *last_r3 = nullptr;
    long long last_r3_rows = 0;
    float *d_tc_w = nullptr;       // Bt1 | Bt2 | Bt3 | bias
    float *d_xg = nullptr;         // X' phase grids (zero borders)
    float *d_z = nullptr;          // Z compact
    float *d_gs = nullptr;         // 3xBF16 split-K through L2: partial tiles | flags
    size_t tc_ws_bytes = 0;
    const float *tc_last_x = nullptr;
    int tc_last_x_batch = 0;
    int max_smem = 0;
    // IEEE-fp32 three-launch CUDA-core path (variant 6, tkd_sgemm.cu)
    tdc::SgemmArgs sg[3];
    float *d_sg = nullptr;         // B1 | B2 | B3 | bias | X' phase grid | Z
    float *d_sg_part = nullptr;    // split-K partial tiles
    // single-launch 3xBF16 layer (variant 5, tkd_layer.cu)
    tdc::BfLayerArgs bl;
    CUtensorMap lmapX;
    const float *l_last_x = nullptr;
    int l_last_batch = 0;
};

namespace {


int div_up(int a, int b) { return (a + b - 1) / b; }

// Round-to-nearest (ties away) to tf32: clear the low 13 mantissa bits.
// fp32 -> bf16 round-to-nearest-even, returned as the bf16 bit pattern.
uint16_t bf16_bits_host(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) return (uint16_t)(u >> 16);
    u += 0x7fffu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
float bf16_to_float_host(uint16_t b) {
    const uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

float tf32_round_host(float x) {
    uint32_t u;
    std::memcpy(&u, &x, 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & ~0x1fffu;
    float r;
    std::memcpy(&r, &u, 4);
    return r;
}

// Plan the tcgen05 3-launch variant: weight re-layout (a0), workspaces, tensor
// maps.  split = 3xTF32 (hi/lo operands everywhere).
tdc_status plan_tc(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                   const float *bias, bool split) {
    const tdc_conv_desc &d = p->desc;
    const int C = d.c_in, N = d.c_out, D1 = d.rank_in, D2 = d.rank_out, K = d.kernel;
    const int s = d.stride, pad = d.pad, H = d.height, W = d.width;
    const int Ho = p->dims.Ho, Wo = p->dims.Wo, Bm = d.batch;
    const int Cs = round_up(C, 32), D1s = round_up(D1, 32), D2s = round_up(D2, 32);
    const int Hq = div_up(H + 2 * pad, s), Wq = div_up(W + 2 * pad, s);
    const long long phase_rows = (long long)Bm * Hq * Wq;
    const long long M1 = (long long)Bm * H * W, M2 = phase_rows, M3 = (long long)Bm * Ho * Wo;
    if (M1 > (1LL << 31) - 256 || M2 * s * s > (1LL << 31) - 256)
        return fail(TDC_ERR_UNSUPPORTED, "batch too large for the tensor-core variant");
    const int sp = split ? 1 : 0;
    // Widest N tile: a tcgen05.mma costs ~130-150 cycles whatever N <= 256 is
    // (DESIGN.md §8), so N = 256 does 8x the work of N = 32 per instruction.
    // Parallelism lost to wide tiles is restored with split-K below.
    // N tile: a power of two (it is also the TMEM allocation), narrowed while the
    // stage has fewer than 2 tiles per SM so small-image stages spread over the GPU.
    auto pick = [&](int nn, long long mrows) {
        int b = 32;
        while (b < nn && b < 256) b *= 2;
        while (b > 64 && div_up((int)mrows, 128) * (long long)div_up(nn, b) < 2 * p->num_sms) b /= 2;
        return b;
    };
    int BN1 = pick(D1s, M1);
    int BN2 = pick(D2s, M2);
    const int BN3 = pick(N, M3);
    const int KK = K * K;

    // Stage-2 kernel choice: band-resident core kernel if its two A slots fit.
    const int maxoff = ((K - 1) / s) * Wq + (K - 1) / s;
    const int band_rows = round_up(128 + maxoff, 8);
    int phase_of[tdc::kMaxTaps], nphase = 0, phase_src[tdc::kMaxTaps];
    {
        // phase id (r % s) * s + (t % s) ranges over s*s values, not K*K
        std::vector<int> idx_of((size_t)s * s, -1);
        for (int r = 0; r < K; ++r)
            for (int t = 0; t < K; ++t) {
                const int ph = (r % s) * s + (t % s);
                if (idx_of[ph] < 0) {
                    idx_of[ph] = nphase;
                    phase_src[nphase++] = ph;
                }
                phase_of[r * K + t] = idx_of[ph];
            }
    }
    int core_stages = 4;
    for (;;) {
        while (core_stages > 2 &&
               tdc::tc_core_smem_bytes(BN2, nphase, band_rows, core_stages, sp) > p->max_smem)
            --core_stages;
        if (BN2 <= 64 || tdc::tc_core_smem_bytes(BN2, nphase, band_rows, core_stages, sp) <= p->max_smem)
            break;
        BN2 /= 2;  // narrower tile so the band + weight ring fit
        core_stages = 4;
    }
    p->tc_core = tdc::tc_core_smem_bytes(BN2, nphase, band_rows, core_stages, sp) <= p->max_smem;
    const int R1 = round_up(D1s, BN1), R2 = round_up(D2s, BN2), R3 = round_up(N, BN3);
    const int k2chunks = D1s / 32, nt2 = R2 / BN2;
    const long long rows_total = (long long)s * s * phase_rows + band_rows + 128;

    // ---- a0: K-major weight panels, zero padded (CRSN idea) ----
    const size_t n1 = (size_t)R1 * Cs, n2 = (size_t)KK * R2 * D1s, n3 = (size_t)R3 * D2s,
                 nb = (size_t)round_up(N, 4);
    const size_t nw = n1 + n2 + n3;  // one copy (hi or plain)
    std::vector<float> h(nw * (split ? 2 : 1) + nb, 0.f);
    float *b1 = h.data(), *b2 = b1 + n1, *b3 = b2 + n2;
    float *hb = h.data() + nw * (split ? 2 : 1);
    for (int a = 0; a < D1; ++a)
        for (int c = 0; c < C; ++c) b1[(size_t)a * Cs + c] = u_in[(size_t)c * D1 + a];
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t)
            for (int q = 0; q < D2; ++q)
                for (int a = 0; a < D1; ++a) {
                    const float v = core[(((size_t)q * D1 + a) * K + r) * K + t];
                    const int tap = r * K + t;
                    if (p->tc_core) {
                        // blocked [tap][kc][ntile][kg8][BN][4] no-swizzle K-major chunks
                        const int kc = a / 32, kg = (a % 32) / 4, e = a % 4;
                        const int ntl = q / BN2, n = q % BN2;
                        b2[((((size_t)(tap * k2chunks + kc) * nt2 + ntl) * 8 + kg) * BN2 + n) * 4 + e] = v;
                    } else {
                        b2[((size_t)tap * R2 + q) * D1s + a] = v;
                    }
                }
    for (int n = 0; n < N; ++n)
        for (int q = 0; q < D2; ++q) b3[(size_t)n * D2s + q] = u_out[(size_t)n * D2 + q];
    if (split)  // hi = RN-to-tf32 (low 13 mantissa bits cleared), lo = w - hi (exact)
        for (size_t i = 0; i < nw; ++i) {
            const float hi = tf32_round_host(h[i]);
            h[nw + i] = h[i] - hi;
            h[i] = hi;
        }
    if (bias)
        for (int n = 0; n < N; ++n) hb[n] = bias[n];
    cudaError_t e = cudaMalloc(&p->d_tc_w, h.size() * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tc weights)");
    e = cudaMemcpy(p->d_tc_w, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(tc weights)");
    p->weight_bytes += h.size() * sizeof(float);

    // ---- workspaces: X' phase grids (zero borders, never written there) and Z ----
    const size_t xg_elems = p->tc_core ? (size_t)rows_total * D1s : (size_t)s * s * phase_rows * D1s;
    const size_t z_elems = (size_t)M3 * D2s;
    const int f = split ? 2 : 1;
    e = cudaMalloc(&p->d_xg, f * xg_elems * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&p->d_z, f * z_elems * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tc workspace)");
    e = cudaMemset(p->d_xg, 0, f * xg_elems * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(X' grid)");
    p->tc_ws_bytes = f * (xg_elems + z_elems) * sizeof(float);
    float *xg_lo = split ? p->d_xg + xg_elems : nullptr;
    float *z_lo = split ? p->d_z + z_elems : nullptr;

    auto base_args = [&](tdc::TcGemmArgs &g) {
        std::memset(&g, 0, sizeof g);
        g.H = H; g.W = W; g.s = s; g.p = pad; g.Hq = Hq; g.Wq = Wq; g.Ho = Ho; g.Wo = Wo;
        g.phase_rows = phase_rows;
        g.split = sp;
    };
    const float *dB1 = p->d_tc_w, *dB2 = dB1 + n1, *dB3 = dB2 + n2;
    const float *dB1lo = split ? dB1 + nw : nullptr, *dB2lo = split ? dB2 + nw : nullptr,
                *dB3lo = split ? dB3 + nw : nullptr;
    const float *dbias = p->d_tc_w + nw * f;
    const char *enc_err = "cuTensorMapEncodeTiled failed";
    // stage 1: A = X (per forward), Bt1; out = X' grid (planar for the core kernel)
    {
        auto &st = p->tc[0];
        base_args(st.args);
        st.args.M = (int)M1; st.args.Nn = D1s; st.args.kchunks = Cs / 32; st.args.taps = 1;
        st.args.BN = BN1; st.args.out = p->d_xg; st.args.ldo = D1s; st.args.remap = 1;
        st.args.planar_stride = p->tc_core ? rows_total * 4 : 0;
        st.args.a_convert = 1;
        st.args.out_lo = xg_lo;
        st.args.stages = tdc::tc_pick_stages(BN1, Cs / 32, p->max_smem, sp);
        st.grid_n = R1 / BN1;
        st.args.ntiles = st.grid_n;
        if (!tdc::make_tma_2d(&st.mapB, dB1, R1, Cs, Cs, BN1) ||
            (split && !tdc::make_tma_2d(&st.mapBlo, dB1lo, R1, Cs, Cs, BN1)))
            return fail(TDC_ERR_CUDA, "%s (stage-1 weights)", enc_err);
        st.mapAlo = st.mapB;  // unused (converter computes A lo)
        if (!split) st.mapBlo = st.mapB;
    }
    // stage 2
    if (p->tc_core) {
        tdc::TcCoreArgs &g = p->core_args;
        std::memset(&g, 0, sizeof g);
        g.xg = p->d_xg; g.plane_stride = rows_total * 4; g.w = dB2; g.z = p->d_z;
        g.ldz = D2s; g.Nn = D2s; g.M = (int)M2; g.kchunks = k2chunks; g.taps = KK;
        g.ntiles = nt2; g.BN = BN2; g.nphase = nphase; g.band_rows = band_rows;
        g.b_stages = core_stages; g.phase_rows = phase_rows;
        for (int r = 0; r < K; ++r)
            for (int t = 0; t < K; ++t) {
                g.tap_phase[r * K + t] = phase_of[r * K + t];
                g.tap_off[r * K + t] = (r / s) * Wq + (t / s);
            }
        for (int i = 0; i < nphase; ++i) g.phase_src[i] = phase_src[i];
        g.Hq = Hq; g.Wq = Wq; g.Ho = Ho; g.Wo = Wo;
        g.split = sp; g.xg_lo = xg_lo; g.w_lo = dB2lo; g.z_lo = z_lo;
    } else {
        auto &st = p->tc[1];
        base_args(st.args);
        st.args.M = (int)M2; st.args.Nn = D2s; st.args.kchunks = D1s / 32; st.args.taps = KK;
        st.args.BN = BN2; st.args.out = p->d_z; st.args.ldo = D2s; st.args.remap = 2;
        st.args.out_lo = z_lo;
        for (int r = 0; r < K; ++r)
            for (int t = 0; t < K; ++t) {
                const int ph = (r % s) * s + (t % s);
                st.args.a_off[r * K + t] = (int)(ph * phase_rows + (r / s) * Wq + (t / s));
                st.args.b_off[r * K + t] = (r * K + t) * R2;
            }
        st.args.stages = tdc::tc_pick_stages(BN2, KK * D1s / 32, p->max_smem, sp);
        st.grid_n = R2 / BN2;
        st.args.ntiles = st.grid_n;
        if (!tdc::make_tma_2d(&st.mapA, p->d_xg, (long long)s * s * phase_rows, D1s, D1s, 128) ||
            !tdc::make_tma_2d(&st.mapB, dB2, (long long)KK * R2, D1s, D1s, BN2))
            return fail(TDC_ERR_CUDA, "%s (stage 2)", enc_err);
        if (split) {
            if (!tdc::make_tma_2d(&st.mapAlo, xg_lo, (long long)s * s * phase_rows, D1s, D1s, 128) ||
                !tdc::make_tma_2d(&st.mapBlo, dB2lo, (long long)KK * R2, D1s, D1s, BN2))
                return fail(TDC_ERR_CUDA, "%s (stage 2 lo)", enc_err);
        } else {
            st.mapAlo = st.mapA;
            st.mapBlo = st.mapB;
        }
    }
    // stage 3: A = Z, Bt3 = U_out; out = Y (per forward), bias
    {
        auto &st = p->tc[2];
        base_args(st.args);
        st.args.M = (int)M3; st.args.Nn = N; st.args.kchunks = D2s / 32; st.args.taps = 1;
        st.args.BN = BN3; st.args.ldo = N; st.args.remap = 0; st.args.bias = bias ? dbias : nullptr;
        st.args.stages = tdc::tc_pick_stages(BN3, D2s / 32, p->max_smem, sp);
        st.grid_n = R3 / BN3;
        st.args.ntiles = st.grid_n;
        if (!tdc::make_tma_2d(&st.mapA, p->d_z, M3, D2s, D2s, 128) ||
            !tdc::make_tma_2d(&st.mapB, dB3, R3, D2s, D2s, BN3))
            return fail(TDC_ERR_CUDA, "%s (stage 3)", enc_err);
        if (split) {
            if (!tdc::make_tma_2d(&st.mapAlo, z_lo, M3, D2s, D2s, 128) ||
                !tdc::make_tma_2d(&st.mapBlo, dB3lo, R3, D2s, D2s, BN3))
                return fail(TDC_ERR_CUDA, "%s (stage 3 lo)", enc_err);
        } else {
            st.mapAlo = st.mapA;
            st.mapBlo = st.mapB;
        }
    }
    p->variant = 2;
    p->split = split;
    return TDC_OK;
}

// Plan the 3xBF16 3-launch variant (fp32-grade accuracy, bf16 tensor cores).
// Returns TDC_OK with *used = false when the band-resident core kernel does not
// fit (the caller then plans 3xTF32 instead).
tdc_status plan_bf16_impl(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                          const float *bias, bool *used);
tdc_status plan_bf16(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                     const float *bias, bool *used) {
    const tdc_plan_hints saved = p->hints;
    const tdc_status st = plan_bf16_impl(p, core, u_in, u_out, bias, used);
    if (st != TDC_OK || !*used) {  // latency-mode hints belong to this variant only
        p->hints = saved;
        p->latency_mode = 0;
    }
    return st;
}
tdc_status plan_bf16_impl(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                          const float *bias, bool *used) {
    *used = false;
    const tdc_conv_desc &d = p->desc;
    const int C = d.c_in, N = d.c_out, D1 = d.rank_in, D2 = d.rank_out, K = d.kernel;
    const int s = d.stride, pad = d.pad, H = d.height, W = d.width;
    const int Ho = p->dims.Ho, Wo = p->dims.Wo, Bm = d.batch;
    if (C % 4 || K * K > tdc::kMaxTaps) return TDC_OK;
    const int C64 = round_up(C, 64), D1s = round_up(D1, 32), D2s = round_up(D2, 32),
              D2p = round_up(D2, 64);
    const int Hq = div_up(H + 2 * pad, s), Wq = div_up(W + 2 * pad, s);
    const long long phase_rows = (long long)Bm * Hq * Wq;
    const long long M1 = (long long)Bm * H * W, M2 = phase_rows, M3 = (long long)Bm * Ho * Wo;
    if (M1 > (1LL << 31) - 256 || M2 * s * s > (1LL << 31) - 256) return TDC_OK;
    {   // Latency mode (small batches): when even 32-wide core N tiles leave half of the SMs
        // idle, every kernel is a chain of a few tiles and its length, not throughput, sets the
        // time -- 32-wide N tiles everywhere and the core's K split over a 4-CTA cluster
        // (batch 1, scripts/b1_sweep_hints2.sh: 7x7 24.8 -> 18.4 us, 14x14 17.5 -> 14.4 us,
        // 28x28 s1 13.8 -> 12.8 us).  Only without explicit planner hints.
        tdc_plan_hints &h = p->hints;
        const bool none = h.core3 < 0 && h.fused_layer < 0 && !h.bn_stage1 && !h.bn_core && !h.bn_stage3 &&
                          !h.ksplit_stage1 && !h.ksplit_core && !h.ksplit_stage3 && !h.gsplit_stage1 &&
                          !h.gsplit_core && !h.gsplit_stage3;
        const char *ev = std::getenv("TDC_NO_LATENCY_MODE");
        if (none && !(ev && ev[0] && ev[0] != '0') &&
            (long long)div_up((int)M2, 128) * div_up(D2s, 32) * 2 <= p->num_sms) {
            h.bn_stage1 = h.bn_core = h.bn_stage3 = 32;
            if (D1s / 32 >= 2) h.ksplit_core = 4;
            h.core3 = 0;
            p->latency_mode = 1;
        }
    }
    auto pick = [&](int nn, long long mrows) {
        int b = 32;
        while (b < nn && b < 256) b *= 2;
        while (b > 64 && div_up((int)mrows, 128) * (long long)div_up(nn, b) < 2 * p->num_sms) b /= 2;
        return b;
    };
    int BN1 = std::min(pick(D1s, M1), 128), BN3 = pick(N, M3);  // stage 1: 2 accumulators + 2 TMEM X slots <= 512 columns
    int BN2 = pick(D2s, M2);
    // few output tiles (deep / strided layers): a narrower core N tile while the grid still
    // fits one wave -- twice the CTAs streaming weight slices (14x14 s2: 26.8 -> 24.6 us,
    // profiles/r02_tiling_search_r18_b32.json)
    while (BN2 > 32 && (long long)div_up((int)M2, 128) * div_up(D2s, BN2 / 2) <= p->num_sms) BN2 /= 2;
    // Split K over a thread-block cluster (DSMEM reduction, deterministic order) when the
    // output tiles alone leave SMs idle: pick (BN, cluster size) maximising busy SMs,
    // larger BN on ties.  Opt-in (TDC_SPLITK=1): on the R18 shapes the per-tile
    // cluster handshake costs more than the shorter K loop saves.
    int ks1 = 1, ks3 = 1;
    {
        const char *ev = std::getenv("TDC_SPLITK");
        const bool off = !(ev && ev[0] && ev[0] != '0');
        auto split_pick = [&](long long mrows, int nn, int bn_max, int iters, int *bn) {
            const long long tiles0 = (long long)div_up((int)mrows, 128) * div_up(nn, *bn);
            if (off || tiles0 >= p->num_sms) return 1;
            int best_bn = *bn, best_cs = 1;
            long long best_u = tiles0;
            int b = 32;
            while (b < nn && b < bn_max) b *= 2;
            for (; b >= 32; b /= 2) {
                const long long tiles = (long long)div_up((int)mrows, 128) * div_up(nn, b);
                int cs = 1;
                for (int c = 2; c <= 4 && c <= iters; ++c)
                    if (tiles * c <= p->num_sms) cs = c;
                const long long u = std::min<long long>(tiles * cs, p->num_sms);
                if (u > best_u) {
                    best_u = u;
                    best_bn = b;
                    best_cs = cs;
                }
            }
            *bn = best_bn;
            return best_cs;
        };
        ks1 = split_pick(M1, D1s, 64, C64 / 64, &BN1);
        ks3 = split_pick(M3, N, 128, D2p / 64, &BN3);
    }
    {   // planner overrides (tdc_conv_plan_ex; NEXT-3 autotune)
        const tdc_plan_hints &h = p->hints;
        auto pow2 = [](int v) {
            int b = 32;
            while (b < v && b < 256) b *= 2;
            return b;
        };
        if (h.bn_stage1 > 0) BN1 = std::min(pow2(h.bn_stage1), 128);
        if (h.bn_stage3 > 0) BN3 = pow2(h.bn_stage3);
        if (h.ksplit_stage1 > 0) ks1 = std::max(1, std::min({h.ksplit_stage1, 4, C64 / 64}));
        if (h.ksplit_stage3 > 0) ks3 = std::max(1, std::min({h.ksplit_stage3, 4, D2p / 64}));
    }
    // narrow N tiles until the GEMM kernels' rings fit shared memory (stage 1 also holds
    // the fp32 staging ring: BN <= 128 there)
    for (;;) {
        int xs = 0, bs = 0;
        const int st = tdc::bf_pick_stages(BN1, p->max_smem, 1, &xs, ks1, &bs);
        if (BN1 <= 32 || tdc::bf_smem_bytes(BN1, st, xs, ks1, bs) <= p->max_smem) break;
        BN1 /= 2;
    }
    for (;;) {
        const int st = tdc::bf_pick_stages(BN3, p->max_smem, 0, nullptr, ks3, nullptr);
        if (BN3 <= 32 || tdc::bf_smem_bytes(BN3, st, 0, ks3, 0) <= p->max_smem) break;
        BN3 /= 2;
    }
    // Split-K through L2 (gsplit): when the output tiles alone leave SMs
    // idle, pick (N tile, pieces) minimising waves x K iterations per piece x the cost of
    // one iteration (measured MMA issue cost + operand loads) + a fix-up
    // cost per split; the planner's own choice stands unless this is >= 5 % cheaper.
    const char *gev = std::getenv("TDC_GSPLIT");
    const bool gs_off = !(gev && gev[0] && gev[0] != '0');  // opt-in: measured slower on R18 (§8c)
    auto mma_cyc = [](int n) { return n <= 64 ? (n <= 32 ? 44.0 : 48.0) : n / 2.0; };
    auto gs_choose = [&](long long mrows, int nn, int iters, int bn_max, bool bn_fixed, int *bn, int hint,
                         auto iter_cost) {
        const long long mt = div_up((int)mrows, 128);
        auto cost = [&](int b, int gsp) {
            const long long units = mt * div_up(nn, b) * gsp;
            return (double)div_up((int)units, p->num_sms) * div_up(iters, gsp) * iter_cost(b) +
                   (gsp > 1 ? 2500.0 : 0.0);
        };
        if (hint > 0) return std::max(1, std::min(hint, std::min(iters, 8)));
        if (gs_off) return 1;
        int best_bn = *bn, best_gs = 1;
        double best = cost(*bn, 1) * 0.95;
        int top = 32;
        while (top < nn && top < bn_max) top *= 2;
        for (int b = bn_fixed ? *bn : top; b >= (bn_fixed ? *bn : 32); b /= 2)
            for (int gsp = 1; gsp <= std::min(iters, 8); ++gsp) {
                const double t = cost(b, gsp);
                if (t < best) {
                    best = t;
                    best_bn = b;
                    best_gs = gsp;
                }
            }
        *bn = best_bn;
        return best_gs;
    };
    auto gemm_iter = [&](int b) { return 12.0 * mma_cyc(b) + (32768.0 + 256.0 * b) / 64.0; };
    int gs1 = 1, gs3 = 1, gs2 = 1;
    if (ks1 == 1) {
        gs1 = gs_choose(M1, D1s, C64 / 64, 128, p->hints.bn_stage1 > 0, &BN1, p->hints.gsplit_stage1, gemm_iter);
        for (;;) {  // the chosen N tile must still fit
            int xs = 0, bs = 0;
            const int st = tdc::bf_pick_stages(BN1, p->max_smem, 1, &xs, 1, &bs);
            if (BN1 <= 32 || tdc::bf_smem_bytes(BN1, st, xs, 1, bs) <= p->max_smem) break;
            BN1 /= 2;
        }
    }
    const int KK = K * K;
    const int maxoff = ((K - 1) / s) * Wq + (K - 1) / s;
    const int band_rows = round_up(128 + maxoff, 8);
    int phase_of[tdc::kMaxTaps], nphase = 0, phase_src[tdc::kMaxTaps];
    {
        // phase id (r % s) * s + (t % s) ranges over s*s values, not K*K
        std::vector<int> idx_of((size_t)s * s, -1);
        for (int r = 0; r < K; ++r)
            for (int t = 0; t < K; ++t) {
                const int ph = (r % s) * s + (t % s);
                if (idx_of[ph] < 0) {
                    idx_of[ph] = nphase;
                    phase_src[nphase++] = ph;
                }
                phase_of[r * K + t] = idx_of[ph];
            }
    }
    // Stage-2 weight staging: one bulk copy per (kc, tap group) slice
    // of tg taps x [4 planes][2*BN2 rows (hi | lo)][8]; resident for the CTA's
    // lifetime when the whole N tile fits, otherwise a ring of w_slots slices.
    const int k2chunks = D1s / 32;
    int tg = 0, w_slots = 0, resident = 0, nt2 = 0;
    // debug overrides of the streamed-weight ring: taps per slice / maximum ring depth
    const int env_tg = std::getenv("TDC_CORE_TG") ? std::atoi(std::getenv("TDC_CORE_TG")) : 0;
    const int ws_max = std::getenv("TDC_CORE_WS") ? std::max(2, std::atoi(std::getenv("TDC_CORE_WS"))) : 4;
    // Fused core + stage 3 (Z stays on chip) when the whole D2 fits one N tile, the
    // U_out panel is resident and both double-buffered accumulators fit in TMEM.
    const int N3p = round_up(N, 32), ncat3 = 2 * N3p <= 128 && !std::getenv("TDC_NO_NCAT3");
    int fuse3 = 0;
    {
        const char *ev = std::getenv("TDC_NO_FUSE3");
        const char *e2f = std::getenv("TDC_CORE2");  // A/B knob: 2 = the CTA-pair core instead of core3
        const bool off = (ev && ev[0] && ev[0] != '0') || p->hints.core3 == 0 || (e2f && e2f[0] == '2') ||
                         (p->hints.bn_core > 0 && p->hints.bn_core < D2s) || p->hints.ksplit_core > 1;
        int bn = 32;
        while (bn < D2s) bn *= 2;
        if (!off && bn <= 128 && (ncat3 ? 2 * N3p : N3p) <= 256) {
            tdc::BfCoreArgs t;
            std::memset(&t, 0, sizeof t);
            t.BN = bn; t.nphase = nphase; t.band_rows = band_rows; t.N3p = N3p;
            t.ncat = 2 * bn <= 128; t.ncat3 = ncat3;
            if (tdc::bf_core3_tmem_cols(t) <= 512) {
                t.tg = KK; t.w_slots = k2chunks;
                if (tdc::bf_core3_smem_bytes(t) <= p->max_smem) {
                    tg = KK; w_slots = k2chunks; resident = 1;
                } else {
                    for (int g = KK; g >= 1 && !tg; --g) {
                        if (KK % g || (env_tg > 0 && g != env_tg)) continue;
                        for (int ws = ws_max; ws >= 2; --ws) {
                            t.tg = g; t.w_slots = ws;
                            if (tdc::bf_core3_smem_bytes(t) <= p->max_smem) {
                                tg = g; w_slots = ws;
                                break;
                            }
                        }
                    }
                }
                if (tg) {
                    fuse3 = 1;
                    BN2 = bn;
                    nt2 = 1;
                }
            }
        }
    }
    // Stage-2 split-K (opt-in, TDC_SPLITK=1): when the output tiles leave SMs idle, pick
    // (BN2, cluster size) minimising a simple cost model: waves x chunks-per-CTA x MMA
    // cycles per chunk (measured issue cost) + a handshake overhead.
    int ks2 = 1;
    {
        const char *ev = std::getenv("TDC_SPLITK");
        const bool on = ev && ev[0] && ev[0] != '0';
        const long long mt = div_up((int)M2, 128);
        if (on && !fuse3 && mt * div_up(D2s, BN2) < p->num_sms) {
            auto mma = [](int n) { return n <= 64 ? (n <= 32 ? 44.0 : 48.0) : n / 2.0; };
            double best = 1e30;
            int bn_top = 32;
            while (bn_top < D2s && bn_top < 128) bn_top *= 2;
            for (int bn = bn_top; bn >= 32; bn /= 2) {
                const double per_kc = 2.0 * KK * (2 * bn <= 128 ? 2 * mma(2 * bn) : 3 * mma(bn));
                const long long tiles = mt * div_up(D2s, bn);
                for (int cs = 1; cs <= 4 && cs <= k2chunks; ++cs) {
                    if (cs > 1 && tiles * cs > p->num_sms) break;
                    const long long per_cta = div_up((int)tiles, std::max(1, p->num_sms / cs));
                    const double t = per_cta * div_up(k2chunks, cs) * per_kc + (cs > 1 ? 3000.0 : 0.0);
                    if (t < best - 1.0) {
                        best = t;
                        BN2 = bn;
                        ks2 = cs;
                    }
                }
            }
        }
    }
    if (!fuse3) {
        const tdc_plan_hints &h = p->hints;
        if (h.bn_core > 0) {
            BN2 = 32;
            while (BN2 < h.bn_core && BN2 < 256) BN2 *= 2;
        }
        if (h.ksplit_core > 0) ks2 = std::max(1, std::min({h.ksplit_core, 4, k2chunks}));
        if (ks2 == 1) {
            auto core_iter = [&](int b) {
                return 2.0 * KK * (2 * b <= 128 ? 2 * mma_cyc(2 * b) : 3 * mma_cyc(b)) + KK * b * 128.0 / 48.0;
            };
            gs2 = gs_choose(M2, D2s, k2chunks, 128, h.bn_core > 0, &BN2, h.gsplit_core, core_iter);
        }
        if (ks3 == 1) {
            gs3 = gs_choose(M3, N, D2p / 64, 128, h.bn_stage3 > 0, &BN3, h.gsplit_stage3, gemm_iter);
            for (;;) {
                const int stg = tdc::bf_pick_stages(BN3, p->max_smem, 0, nullptr, 1, nullptr);
                if (BN3 <= 32 || tdc::bf_smem_bytes(BN3, stg, 0, 1, 0) <= p->max_smem) break;
                BN3 /= 2;
            }
        }
    }
    for (; !fuse3 && BN2 >= 32; BN2 /= 2) {
        nt2 = div_up(D2s, BN2);
        if (ks2 == 1 && nt2 == 1 &&
            tdc::bf_core_smem_bytes(BN2, nphase, band_rows, KK, k2chunks, 1) <= p->max_smem) {
            tg = KK;
            w_slots = k2chunks;
            resident = 1;
            break;
        }
        for (int g = KK; g >= 1 && !tg; --g) {
            if (KK % g || (env_tg > 0 && g != env_tg)) continue;
            for (int ws = ws_max; ws >= 2; --ws)
                if (tdc::bf_core_smem_bytes(BN2, nphase, band_rows, g, ws, ks2) <= p->max_smem) {
                    tg = g;
                    w_slots = ws;
                    break;
                }
        }
        if (tg) break;
    }
    if (!tg) return TDC_OK;
    const int ngroups = KK / tg;
    const int ncat = 2 * BN2 <= 128;  // one N = 2*BN2 MMA covers the hi and lo weights
    const int R1 = round_up(D1s, BN1), R2 = nt2 * BN2, R3 = round_up(N, BN3);
    const long long rows_total = (long long)s * s * phase_rows + band_rows + 128;

    // ---- a0: bf16 hi/lo weight panels (CRSN idea) ----
    // stages 1/3: [all hi][all lo] K-major panels; stage 2: hi/lo interleaved slices.
    const size_t n1 = (size_t)R1 * C64, n3 = (size_t)R3 * D2p, nw = n1 + n3;
    const size_t n2 = (size_t)KK * R2 * D1s;  // per hi or lo
    const size_t n3f = fuse3 ? (size_t)BN2 * 2 * N3p : 0;  // fused stage-3 panel (hi|lo rows)
    std::vector<float> wf(nw, 0.f);  // fp32 staging in the final element order
    float *w1 = wf.data(), *w3 = w1 + n1;
    for (int a = 0; a < D1; ++a)
        for (int c = 0; c < C; ++c) w1[(size_t)a * C64 + c] = u_in[(size_t)c * D1 + a];
    for (int n = 0; n < N; ++n)
        for (int q = 0; q < D2; ++q) w3[(size_t)n * D2p + q] = u_out[(size_t)n * D2 + q];
    std::vector<uint16_t> hb(2 * nw + 2 * n2 + n3f, 0);
    for (size_t i = 0; i < nw; ++i) {
        const uint16_t hi = bf16_bits_host(wf[i]);
        hb[i] = hi;
        hb[nw + i] = bf16_bits_host(wf[i] - bf16_to_float_host(hi));
    }
    uint16_t *w2 = hb.data() + 2 * nw;
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t)
            for (int q = 0; q < D2; ++q)
                for (int a = 0; a < D1; ++a) {
                    // [kc][ntile][group][tt][plane(4)][2*BN2][8]: row n = hi, BN2 + n = lo
                    const int kc = a / 32, pl = (a % 32) / 8, e = a % 8, tap = r * K + t;
                    const int ntl = q / BN2, n = q % BN2, grp = tap / tg, tt = tap % tg;
                    const size_t base =
                        (((((size_t)kc * nt2 + ntl) * ngroups + grp) * tg + tt) * 4 + pl) * 2 * BN2;
                    const float v = core[(((size_t)q * D1 + a) * K + r) * K + t];
                    const uint16_t hi = bf16_bits_host(v);
                    w2[(base + n) * 8 + e] = hi;
                    w2[(base + BN2 + n) * 8 + e] = bf16_bits_host(v - bf16_to_float_host(hi));
                }
    if (fuse3) {  // [D2/8 planes][2*N3p rows: hi n | lo N3p + n][8]
        uint16_t *w3f = w2 + 2 * n2;
        for (int n = 0; n < N; ++n)
            for (int q = 0; q < D2; ++q) {
                const float v = u_out[(size_t)n * D2 + q];
                const uint16_t hi = bf16_bits_host(v);
                const size_t row = (size_t)(q / 8) * 2 * N3p;
                w3f[(row + n) * 8 + q % 8] = hi;
                w3f[(row + N3p + n) * 8 + q % 8] = bf16_bits_host(v - bf16_to_float_host(hi));
            }
    }
    const size_t wbytes = hb.size() * sizeof(uint16_t), nbias = round_up(N, 4);
    cudaError_t e = cudaMalloc(&p->d_tc_w, wbytes + nbias * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(bf16 weights)");
    e = cudaMemcpy(p->d_tc_w, hb.data(), wbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && bias) {
        std::vector<float> bb(nbias, 0.f);
        for (int n = 0; n < N; ++n) bb[n] = bias[n];
        e = cudaMemcpy(reinterpret_cast<uint8_t *>(p->d_tc_w) + wbytes, bb.data(), nbias * sizeof(float),
                       cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(bf16 weights)");
    p->weight_bytes += wbytes + nbias * sizeof(float);
    const uint16_t *wb = reinterpret_cast<const uint16_t *>(p->d_tc_w);
    const uint16_t *dB1 = wb, *dB3 = wb + n1, *dB2 = wb + 2 * nw;
    const uint16_t *dB1lo = dB1 + nw, *dB3lo = dB3 + nw;
    const float *dbias =
        bias ? reinterpret_cast<const float *>(reinterpret_cast<uint8_t *>(p->d_tc_w) + wbytes) : nullptr;

    // ---- workspaces: X' hi/lo planar bf16 (zero borders), Z hi/lo bf16 [M3][D2p] ----
    const size_t xg_elems = (size_t)rows_total * D1s, z_elems = fuse3 ? 0 : (size_t)M3 * D2p;
    e = cudaMalloc(&p->d_xg, 2 * xg_elems * sizeof(uint16_t));
    if (e == cudaSuccess && z_elems) e = cudaMalloc(&p->d_z, 2 * z_elems * sizeof(uint16_t));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(bf16 workspace)");
    e = cudaMemset(p->d_xg, 0, 2 * xg_elems * sizeof(uint16_t));
    if (e == cudaSuccess && z_elems)
        e = cudaMemset(p->d_z, 0, 2 * z_elems * sizeof(uint16_t));  // pad columns stay 0
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemset(bf16 workspace)");
    p->tc_ws_bytes = 2 * (xg_elems + z_elems) * sizeof(uint16_t);
    uint16_t *xg = reinterpret_cast<uint16_t *>(p->d_xg), *xg_lo = xg + xg_elems;
    uint16_t *z = reinterpret_cast<uint16_t *>(p->d_z), *z_lo = z + z_elems;
    // split-K through L2: fp32 partial tiles of pieces 1..gs-1 and one flag each (zeroed
    // here; every launch leaves them zero)
    const long long gt1 = (long long)div_up((int)M1, 128) * (R1 / BN1), gt2 = (long long)div_up((int)M2, 128) * nt2,
                    gt3 = fuse3 ? 0 : (long long)div_up((int)M3, 128) * (R3 / BN3);
    const size_t gp1 = gs1 > 1 ? (size_t)gt1 * (gs1 - 1) * 128 * BN1 : 0,
                 gp2 = (!fuse3 && gs2 > 1) ? (size_t)gt2 * (gs2 - 1) * 128 * BN2 : 0,
                 gp3 = gs3 > 1 ? (size_t)gt3 * (gs3 - 1) * 128 * BN3 : 0;
    const size_t gf1 = gs1 > 1 ? (size_t)gt1 * (gs1 - 1) : 0, gf2 = gp2 ? (size_t)gt2 * (gs2 - 1) : 0,
                 gf3 = gs3 > 1 ? (size_t)gt3 * (gs3 - 1) : 0;
    float *gpart1 = nullptr, *gpart2 = nullptr, *gpart3 = nullptr;
    int *gflag1 = nullptr, *gflag2 = nullptr, *gflag3 = nullptr;
    if (gp1 + gp2 + gp3) {
        const size_t gbytes = (gp1 + gp2 + gp3) * sizeof(float) + (gf1 + gf2 + gf3) * sizeof(int);
        e = cudaMalloc(&p->d_gs, gbytes);
        if (e == cudaSuccess) e = cudaMemset(p->d_gs, 0, gbytes);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(split-K workspace)");
        p->tc_ws_bytes += gbytes;
        gpart1 = p->d_gs;
        gpart2 = gpart1 + gp1;
        gpart3 = gpart2 + gp2;
        gflag1 = reinterpret_cast<int *>(gpart3 + gp3);
        gflag2 = gflag1 + gf1;
        gflag3 = gflag2 + gf2;
    }

    auto base_args = [&](tdc::TcGemmArgs &g) {
        std::memset(&g, 0, sizeof g);
        g.H = H; g.W = W; g.s = s; g.p = pad; g.Hq = Hq; g.Wq = Wq; g.Ho = Ho; g.Wo = Wo;
        g.phase_rows = phase_rows;
    };
    const char *enc_err = "cuTensorMapEncodeTiled failed (3xBF16)";
    {   // stage 1: A = X fp32 (map per forward, 32-channel boxes), B = U_in^T bf16
        auto &st = p->tc[0];
        base_args(st.args);
        st.args.M = (int)M1; st.args.Nn = D1s; st.args.kchunks = C64 / 64; st.args.taps = 1;
        st.args.BN = BN1; st.args.remap = 1; st.args.a_convert = 1; st.args.out_bf16 = 1;
        st.args.out = reinterpret_cast<float *>(xg); st.args.out_lo = reinterpret_cast<float *>(xg_lo);
        st.args.planar_stride = rows_total;  // rows
        st.args.ksplit = ks1;
        if (gp1) {
            st.args.gsplit = gs1;
            st.args.part = gpart1;
            st.args.flags = gflag1;
        }
        st.args.stages = tdc::bf_pick_stages(BN1, p->max_smem, 1, &st.args.xstages, ks1, &st.args.bstages);
        st.grid_n = R1 / BN1;
        st.args.ntiles = st.grid_n;
        if (!tdc::make_tma_2d_bf16(&st.mapB, dB1, R1, C64, C64, BN1) ||
            !tdc::make_tma_2d_bf16(&st.mapBlo, dB1lo, R1, C64, C64, BN1))
            return fail(TDC_ERR_CUDA, "%s (stage 1)", enc_err);
    }
    {   // stage 2: band-resident core kernel on bf16 planes
        tdc::BfCoreArgs &g = p->bf_core;
        std::memset(&g, 0, sizeof g);
        g.xg = xg;
        g.xg_lo = xg_lo;
        g.plane_rows = rows_total;
        g.w = dB2;
        g.z = z;
        g.z_lo = z_lo;
        g.ldz = D2p; g.Nn = D2s; g.M = (int)M2; g.kchunks = k2chunks; g.taps = KK;
        g.ntiles = nt2; g.BN = BN2; g.nphase = nphase; g.band_rows = band_rows;
        g.tg = tg; g.ngroups = ngroups; g.w_slots = w_slots; g.w_resident = resident; g.ncat = ncat;
        g.ksplit = ks2;
        if (gp2) {
            g.gsplit = gs2;
            g.part = gpart2;
            g.flags = gflag2;
        }
        g.phase_rows = phase_rows;
        for (int r = 0; r < K; ++r)
            for (int t = 0; t < K; ++t) {
                g.tap_phase[r * K + t] = phase_of[r * K + t];
                g.tap_off[r * K + t] = (r / s) * Wq + (t / s);
            }
        for (int i = 0; i < nphase; ++i) g.phase_src[i] = phase_src[i];
        g.Hq = Hq; g.Wq = Wq; g.Ho = Ho; g.Wo = Wo;
        if (fuse3) {
            const char *dbg = std::getenv("TDC_CORE_DBG");
            g.dbg = dbg ? std::atoi(dbg) : 0;
            const char *yd = std::getenv("TDC_Y_DIRECT");
            g.y_direct = yd && yd[0] && yd[0] != '0';
            g.w3 = dB2 + 2 * n2;
            g.bias = dbias;
            g.N3 = N; g.N3p = N3p; g.ncat3 = ncat3;
        }
        // Stage 2 on CTA pairs (cta_group::2): each SM streams half of every weight slice.
        // For the streamed-weight 3x3 cores (deep layers), whose time is the per-SM weight
        // streaming, not the MMAs.  TDC_CORE2=0 disables.
        const char *e2 = std::getenv("TDC_CORE2");
        const int mt2 = div_up((int)M2, 128);
        if (!fuse3 && !(e2 && e2[0] == '0') && KK == 9 && (!resident || (e2 && e2[0] == '2')) && ks2 == 1 &&
            gs2 <= 1 &&
            2 * BN2 <= 256 && mt2 >= 2 && p->hints.ksplit_core <= 0 && p->hints.gsplit_core <= 0) {
            int ws2 = 0, as2 = 0;
            const char *eas = std::getenv("TDC_CORE2_AS");  // A/B knob: band ring depth (2 or 3)
            const char *ews = std::getenv("TDC_CORE2_WS");  // A/B knob: maximum weight slots
            const int ws_top = ews ? std::max(3, std::min(6, std::atoi(ews))) : 6;
            for (int as = eas ? std::max(2, std::min(3, std::atoi(eas))) : 3; as >= 2 && !ws2; --as)
                for (int ws = ws_top; ws >= 3 && !ws2; --ws)
                    if (tdc::bf_core2_smem_bytes(BN2, nphase, band_rows, ws, as) <= p->max_smem) {
                        ws2 = ws;
                        as2 = as;
                    }
            if (!ws2 && tdc::bf_core2_smem_bytes(BN2, nphase, band_rows, 2, 2) <= p->max_smem) ws2 = as2 = 2;
            if (ws2) {
                // per (kc, ntile, CTA half h): [tap][plane][BN2 rows: h ? C lo : C hi][8] followed by
                // [tap][plane][BN2/2 rows: C hi rows h*BN2/2 ..][8] (B of the X' lo x C hi MMA)
                const size_t slot_el = (size_t)9 * 4 * (BN2 + BN2 / 2) * 8, main_el = (size_t)9 * 4 * BN2 * 8;
                const size_t nc2 = (size_t)k2chunks * nt2 * 2 * slot_el;
                std::vector<uint16_t> c2(nc2, 0);
                for (int r = 0; r < K; ++r)
                    for (int t = 0; t < K; ++t)
                        for (int q = 0; q < D2; ++q)
                            for (int a = 0; a < D1; ++a) {
                                const int kc = a / 32, pl = (a % 32) / 8, e8 = a % 8, tap = r * K + t;
                                const int ntl = q / BN2, n = q % BN2;
                                const float v = core[(((size_t)q * D1 + a) * K + r) * K + t];
                                const uint16_t hi = bf16_bits_host(v);
                                const uint16_t lo = bf16_bits_host(v - bf16_to_float_host(hi));
                                for (int half = 0; half < 2; ++half) {
                                    const size_t slot = (((size_t)kc * nt2 + ntl) * 2 + half) * slot_el;
                                    c2[slot + (((size_t)tap * 4 + pl) * BN2 + n) * 8 + e8] = half ? lo : hi;
                                }
                                const int hx = n / (BN2 / 2), nx = n % (BN2 / 2);  // the CTA holding this C hi row
                                const size_t slot = (((size_t)kc * nt2 + ntl) * 2 + hx) * slot_el;
                                c2[slot + main_el + (((size_t)tap * 4 + pl) * (BN2 / 2) + nx) * 8 + e8] = hi;
                            }
                cudaError_t ce = cudaMalloc(&p->d_c2w, nc2 * sizeof(uint16_t));
                if (ce == cudaSuccess) ce = cudaMemcpy(p->d_c2w, c2.data(), nc2 * sizeof(uint16_t), cudaMemcpyHostToDevice);
                if (ce != cudaSuccess) return cuda_fail(ce, "core weights for the CTA-pair kernel");
                p->weight_bytes += nc2 * sizeof(uint16_t);
                g.w = reinterpret_cast<const uint16_t *>(p->d_c2w);
                g.w_slots = ws2;
                g.a_slots = as2;
                p->core2 = true;
            }
        }
    }
    p->fuse3 = fuse3 != 0;
    if (!fuse3) {   // stage 3: A = Z hi/lo bf16, B = U_out bf16; out = Y fp32 (+bias)
        auto &st = p->tc[2];
        base_args(st.args);
        st.args.M = (int)M3; st.args.Nn = N; st.args.kchunks = D2p / 64; st.args.taps = 1;
        st.args.BN = BN3; st.args.ldo = N; st.args.remap = 0; st.args.bias = dbias;
        st.args.ksplit = ks3;
        if (gp3) {
            st.args.gsplit = gs3;
            st.args.part = gpart3;
            st.args.flags = gflag3;
        }
        st.args.stages = tdc::bf_pick_stages(BN3, p->max_smem, 0, nullptr, ks3, nullptr);
        {
            const char *ev = std::getenv("TDC_NO_TMA_Y");
            st.args.tma_y = ks3 == 1 && N % 4 == 0 && !(ev && ev[0] && ev[0] != '0');
        }
        st.grid_n = R3 / BN3;
        st.args.ntiles = st.grid_n;
        if (!tdc::make_tma_2d_bf16(&st.mapA, z, M3, D2p, D2p, 128) ||
            !tdc::make_tma_2d_bf16(&st.mapAlo, z_lo, M3, D2p, D2p, 128) ||
            !tdc::make_tma_2d_bf16(&st.mapB, dB3, R3, D2p, D2p, BN3) ||
            !tdc::make_tma_2d_bf16(&st.mapBlo, dB3lo, R3, D2p, D2p, BN3))
            return fail(TDC_ERR_CUDA, "%s (stage 3)", enc_err);
    }
    p->tc_core = true;
    p->bf16x3 = true;
    p->variant = 4;
    *used = true;
    return TDC_OK;
}

// Plan the IEEE-fp32 path (variant 6): three register-blocked GEMM-with-taps launches on
// CUDA cores over the whole GPU (tkd_sgemm.cu).  Needs 16-byte pixel rows (C % 4 == 0);
// otherwise the single-kernel SIMT variant stays.
tdc_status plan_sgemm(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                      const float *bias, bool *used) {
    *used = false;
    const tdc_conv_desc &d = p->desc;
    const int C = d.c_in, N = d.c_out, D1 = d.rank_in, D2 = d.rank_out, K = d.kernel;
    const int s = d.stride, pad = d.pad, H = d.height, W = d.width, Bm = d.batch;
    const int Ho = p->dims.Ho, Wo = p->dims.Wo, KK = K * K;
    {
        const char *ev = std::getenv("TDC_NO_SGEMM");
        if (ev && ev[0] && ev[0] != '0') return TDC_OK;
    }
    if (C % 4 || KK > tdc::kMaxTaps) return TDC_OK;
    const int K1 = round_up(C, 16), D1p = round_up(D1, 16), D2p = round_up(D2, 16);  // K-step 16
    const int ldb1 = round_up(D1p, 128), ldb2 = round_up(D2, 128), ldb3 = round_up(N, 128);
    const int Hq = div_up(H + 2 * pad, s), Wq = div_up(W + 2 * pad, s);
    const long long phase_rows = (long long)Bm * Hq * Wq;
    const long long M1 = (long long)Bm * H * W, M2 = phase_rows, M3 = (long long)Bm * Ho * Wo;
    std::vector<int> idx_of((size_t)s * s, -1);
    int phase_of[tdc::kMaxTaps], nphase = 0;
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t) {
            const int ph = (r % s) * s + (t % s);
            if (idx_of[ph] < 0) idx_of[ph] = nphase++;
            phase_of[r * K + t] = idx_of[ph];
        }
    if (s * s > tdc::kMaxTaps || nphase * M2 + 1024 > (1LL << 31) || M1 > (1LL << 31) - 256) return TDC_OK;
    const long long maxoff = (long long)((K - 1) / s) * Wq + (K - 1) / s;
    const long long xg_rows = nphase * phase_rows + maxoff + 512;
    const size_t nb1 = (size_t)K1 * ldb1, nb2 = (size_t)KK * D1p * ldb2, nb3 = (size_t)D2p * ldb3,
                 nbias = round_up(N, 4), nxg = (size_t)xg_rows * D1p, nz = (size_t)(M3 + 512) * D2p;
    // ---- a0: weight re-layout (CRSN idea), zero-padded to the tiles ----
    std::vector<float> hw(nb1 + nb2 + nb3 + nbias, 0.f);
    float *b1 = hw.data(), *b2 = b1 + nb1, *b3 = b2 + nb2, *bb = b3 + nb3;
    for (int c = 0; c < C; ++c)
        for (int a = 0; a < D1; ++a) b1[(size_t)c * ldb1 + a] = u_in[(size_t)c * D1 + a];
    for (int q = 0; q < D2; ++q)
        for (int a = 0; a < D1; ++a)
            for (int r = 0; r < K; ++r)
                for (int t = 0; t < K; ++t)
                    b2[((size_t)(r * K + t) * D1p + a) * ldb2 + q] = core[(((size_t)q * D1 + a) * K + r) * K + t];
    for (int n = 0; n < N; ++n)
        for (int q = 0; q < D2; ++q) b3[(size_t)q * ldb3 + n] = u_out[(size_t)n * D2 + q];
    if (bias)
        for (int n = 0; n < N; ++n) bb[n] = bias[n];
    const size_t wbytes = hw.size() * sizeof(float), tot = wbytes + (nxg + nz) * sizeof(float);
    cudaError_t e = tdc::sgemm_prepare();
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(fp32 GEMM)");
    e = cudaMalloc(&p->d_sg, tot);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(fp32 weights + workspace)");
    e = cudaMemcpy(p->d_sg, hw.data(), wbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemset(p->d_sg + hw.size(), 0, (nxg + nz) * sizeof(float));  // zero borders / pads
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(fp32 weights)");
    p->weight_bytes += wbytes;
    p->tc_ws_bytes += (nxg + nz) * sizeof(float);
    float *dB1 = p->d_sg, *dB2 = dB1 + nb1, *dB3 = dB2 + nb2, *dbias = dB3 + nb3, *xg = dbias + nbias, *z = xg + nxg;
    for (auto &a : p->sg) {
        std::memset(&a, 0, sizeof a);
        a.H = H; a.W = W; a.s = s; a.p = pad; a.Hq = Hq; a.Wq = Wq; a.Ho = Ho; a.Wo = Wo;
        a.phase_rows = phase_rows;
        for (int i = 0; i < tdc::kMaxTaps; ++i) a.phase_idx[i] = i < s * s ? idx_of[i] : -1;
        a.taps = 1;
    }
    tdc::SgemmArgs &s1 = p->sg[0], &s2 = p->sg[1], &s3 = p->sg[2];
    s1.lda = C; s1.M = (int)M1; s1.K = K1; s1.kmask = K1 != C; s1.K_valid = C; s1.B = dB1; s1.ldb = ldb1;
    s1.N = D1p; s1.C = xg; s1.ldc = D1p; s1.remap = 1;
    s2.A = xg; s2.lda = D1p; s2.M = (int)M2; s2.K = D1p; s2.taps = KK; s2.B = dB2; s2.ldb = ldb2;
    s2.N = D2; s2.C = z; s2.ldc = D2p; s2.remap = 2;
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t)
            s2.a_off[r * K + t] = (long long)phase_of[r * K + t] * phase_rows + (r / s) * Wq + t / s;
    s3.A = z; s3.lda = D2p; s3.M = (int)M3; s3.K = D2p; s3.B = dB3; s3.ldb = ldb3; s3.N = N; s3.ldc = N;
    s3.bias = bias ? dbias : nullptr; s3.remap = 0;
    // tiles and split-K pieces for the plan's batch (a smaller batch keeps them: bit-identical
    // results for a partial batch); one partial workspace shared by the three stages
    long long part = 0;
    const char *ev_t = std::getenv("TDC_SG_TILES"), *ev_k = std::getenv("TDC_SG_KSPLIT");  // tuning: "t1,t2,t3"
    for (int i = 0; i < 3; ++i) {
        tdc::SgemmArgs &a = p->sg[i];
        a.tile = tdc::sgemm_pick_tile(a.M, a.N, p->num_sms);
        if (ev_t && (int)std::strlen(ev_t) > 2 * i && ev_t[2 * i] >= '0' && ev_t[2 * i] <= '2') a.tile = ev_t[2 * i] - '0';
        a.ctas = tdc::sgemm_ctas(a.tile, p->num_sms);
        a.ksplit = tdc::sgemm_pick_ksplit(a.M, a.N, a.K, a.taps, a.tile, a.ctas);
        if (ev_k && (int)std::strlen(ev_k) > 2 * i && ev_k[2 * i] >= '1' && ev_k[2 * i] <= '8') a.ksplit = ev_k[2 * i] - '0';
        a.ksplit = std::min(a.ksplit, std::max(1, a.taps * (a.K / 16)));
        part = std::max(part, tdc::sgemm_part_floats(a.M, a.N, a.tile, a.ksplit));
    }
    if (part) {  // partial tiles of the split stages (one workspace, stages run in order)
        float *pw = nullptr;
        e = cudaMalloc(&pw, part * sizeof(float));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(fp32 split-K workspace)");
        p->d_sg_part = pw;
        p->tc_ws_bytes += part * sizeof(float);
        for (auto &a : p->sg) a.part = pw;
    }
    p->variant = 6;
    *used = true;
    return TDC_OK;
}

tdc_status forward_sgemm(tdc_conv_plan_s *p, const float *x, float *y, int batch, cudaStream_t st) {
    const tdc::LayerDims &d = p->dims;
    tdc::SgemmArgs a1 = p->sg[0], a2 = p->sg[1], a3 = p->sg[2];
    a1.A = x;
    a1.M = batch * d.H * d.W;
    a2.M = batch * a2.Hq * a2.Wq;
    a3.M = batch * d.Ho * d.Wo;
    a3.C = y;
    cudaError_t e = tdc::sgemm_taps_launch(a1, st);
    if (e == cudaSuccess) e = tdc::sgemm_taps_launch(a2, st);
    if (e == cudaSuccess) e = tdc::sgemm_taps_launch(a3, st);
    if (e != cudaSuccess) return cuda_fail(e, "fp32 CUDA-core GEMM launch");
    return TDC_OK;
}

// Plan the single-launch 3xBF16 layer kernel (variant 5): stage 1, the core and stage 3
// in one persistent kernel with X' and Z on chip.  Used when the
// layer has stride 1, its ranks / output channels fit one tile (<= 128, hi|lo
// concatenated in one MMA), all weights stay resident in shared memory next to the
// band ring and X staging, and the accumulators fit TMEM; *used = false otherwise.
tdc_status plan_layer(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                      const float *bias, bool *used) {
    *used = false;
    const tdc_conv_desc &d = p->desc;
    const int C = d.c_in, N = d.c_out, D1 = d.rank_in, D2 = d.rank_out, K = d.kernel;
    const int s = d.stride, pad = d.pad, H = d.height, W = d.width;
    {
        const char *ev = std::getenv("TDC_NO_LAYER"), *ev3 = std::getenv("TDC_NO_FUSE3");
        const tdc_plan_hints &h = p->hints;
        if ((ev && ev[0] && ev[0] != '0') || (ev3 && ev3[0] && ev3[0] != '0') || h.fused_layer == 0) return TDC_OK;
        // auto: an explicit choice for the three-launch kernels (tile, split or fusion
        // override) asks for those kernels
        const bool other = h.core3 == 0 || h.bn_stage1 > 0 || h.bn_core > 0 || h.bn_stage3 > 0 ||
                           h.ksplit_stage1 > 0 || h.ksplit_core > 0 || h.ksplit_stage3 > 0 || h.gsplit_stage1 > 0 ||
                           h.gsplit_core > 0 || h.gsplit_stage3 > 0;
        if (h.fused_layer < 0 && other) return TDC_OK;
    }
    if (s != 1 || C % 4 || K * K > tdc::kMaxTaps) return TDC_OK;
    const int Wp = W + 2 * pad, Hp = H + 2 * pad;
    const int D1s = round_up(D1, 32), D2s = round_up(D2, 32), N3p = round_up(N, 32);
    // rows wider than one 128-row tile: column strips of 128 padded positions, one output row
    // per tile -- only the TMEM-operand kernel (variant 5b) walks strips
    const char *ex0 = std::getenv("TDC_LAYER_XT");
    const bool strips = Wp > 128;
    if (strips && !(K == 3 && D1s == 32 && D2s == 32 && N3p <= 64 && !(ex0 && ex0[0] == '0'))) return TDC_OK;
    if (D1s > 128 || D2s > 128 || N3p > 128) return TDC_OK;
    tdc::BfLayerArgs g;
    std::memset(&g, 0, sizeof g);
    g.B = d.batch; g.H = H; g.W = W; g.C = C; g.N = N; g.K = K; g.KK = K * K; g.s = s; g.p = pad;
    g.Ho = p->dims.Ho; g.Wo = p->dims.Wo; g.Wp = Wp; g.Wq = Wp; g.Hq = Hp;
    g.nstrips = 1;
    g.sw = g.Wo;
    if (strips) {
        g.Wp = g.Wq = 128;
        g.sw = 128 - (K - 1);
        g.nstrips = div_up(g.Wo, g.sw);
    }
    g.R = std::min(128 / g.Wp, g.Ho);
    g.e = K - 1;
    if (g.R < 1) return TDC_OK;
    g.TH = div_up(g.Ho, g.R);
    g.T = g.TH * g.nstrips;
    g.rpb = g.R;
    g.NR = 2 * g.R + g.e;
    {   // windows start at multiples of gcd(R, NR) below NR; the last one (+ its guard row)
        // must be contiguous: NRB = max start + R + e + 1, mirror rows = NRB - NR
        int a = g.R, b = g.NR;
        while (b) { const int t = a % b; a = b; b = t; }
        g.NRB = g.NR - a + g.R + g.e + 1;
    }
    g.XR = round_up(g.R * g.Wp, 8);   // rpb = R: one block = R padded rows
    g.ZR = round_up(g.R * g.Wq, 8);
    if (g.XR > 128 || g.ZR > 128) return TDC_OK;
    g.cchunks = div_up(C, 64);
    g.D1s = D1s; g.D2s = D2s; g.N3p = N3p;
    {   // taps along N (K = 3, D2s = 32): 1 acc1 + 1 acc2 of 6*D2s columns + 2 acc3
        const char *ev = std::getenv("TDC_LAYER_TN");  // A/B knob: 0 disables
        g.tn = K == 3 && D2s == 32 && 4 * D1s + 8 * D2s + 2 * N3p <= 512 && !(ev && ev[0] == '0');
        const char *e3 = std::getenv("TDC_LAYER_NCAT3");  // A/B knob
        g.ncat3 = e3 ? (e3[0] == '1') : 1;
        // X and Z in tensor memory (variant 5b): TMEM = X 2x64 | acc1 | 2 acc2 | one acc3
        const char *ex = std::getenv("TDC_LAYER_XT");  // A/B knob: 0 disables
        g.xt = g.tn && D1s == 32 && N3p <= 64 && 128 + 4 * D1s + 8 * D2s <= 512 && !(ex && ex[0] == '0');
        if (strips && !g.xt) return TDC_OK;
        // one output row per tile: a tap's A spans one ring row (+ 2 positions that only feed
        // junk columns), so the 5b kernel wraps rows instead of mirroring them
        if (g.xt && g.R == 1) g.NRB = g.NR;
    }
    const int tcols = g.xt ? 128 + 4 * D1s + 8 * D2s
                           : g.tn ? 4 * D1s + 8 * D2s + 2 * N3p : 4 * D1s + 4 * D2s + (g.ncat3 ? 4 : 2) * N3p;
    if (tcols > 512) return TDC_OK;
    g.tmem_cols = 32;
    while (g.tmem_cols < tcols) g.tmem_cols *= 2;
    g.XS = 0;
    const char *xs_env = std::getenv("TDC_LAYER_XS");  // A/B knob: maximum X staging depth
    // 5b: two staging slots measured faster than three (56^2 batch 32: 18.75 vs 19.6 us) -- the
    // converters free a slot as soon as they have read it, and the freed 30 KB go to L1
    for (int xs = xs_env ? std::max(2, std::min(4, std::atoi(xs_env))) : (g.xt ? 2 : 4); xs >= 2 && !g.XS; --xs) {
        g.XS = xs;
        if (tdc::bf_layer_smem_bytes(g) > p->max_smem) g.XS = 0;
    }
    if (!g.XS) return TDC_OK;
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t) g.tap_off[r * K + t] = r * g.Wq + t;

    // ---- a0: bf16 hi/lo operand images (CRSN idea) ----
    const int KK = K * K, C64 = g.cchunks * 64;
    const size_t n1 = (size_t)g.cchunks * 2 * D1s * 64;           // U_in, swizzled per chunk
    const size_t n2 = (size_t)(D1s / 32) * KK * 4 * 2 * D2s * 8;   // core
    const size_t n3 = (size_t)(D2s / 8) * 2 * N3p * 8;             // U_out
    std::vector<uint16_t> hb(n1 + n2 + n3, 0);
    auto split = [](float v, uint16_t *hi, uint16_t *lo) {
        *hi = bf16_bits_host(v);
        *lo = bf16_bits_host(v - bf16_to_float_host(*hi));
    };
    uint16_t *w1 = hb.data(), *w2 = w1 + n1, *w3 = w2 + n2;
    for (int cc = 0; cc < g.cchunks; ++cc)      // [cc][row: hi a | lo D1s + a][64 ch], 128B swizzle
        for (int a = 0; a < D1; ++a)
            for (int k = 0; k < 64; ++k) {
                const int c = cc * 64 + k;
                if (c >= C) continue;
                uint16_t hi, lo;
                split(u_in[(size_t)c * D1 + a], &hi, &lo);
                for (int hl = 0; hl < 2; ++hl) {
                    const int row = hl * D1s + a;
                    const size_t at = ((size_t)cc * 2 * D1s + row) * 64 + (size_t)(((k / 8) ^ (row & 7)) * 8 + k % 8);
                    w1[at] = hl ? lo : hi;
                }
            }
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t)
            for (int q = 0; q < D2; ++q)
                for (int a = 0; a < D1; ++a) {
                    uint16_t hi, lo;
                    split(core[(((size_t)q * D1 + a) * K + r) * K + t], &hi, &lo);
                    const int tap = r * K + t, kc = a / 32, pl = (a % 32) / 8, e8 = a % 8;
                    if (g.tn) {  // [kc][r][plane][rows: C(r,0) lo | C(r,0) hi | C(r,1) hi | C(r,1) lo | C(r,2) hi | lo][8]
                        static const int hi_grp[3] = {1, 2, 4}, lo_grp[3] = {0, 3, 5};
                        const size_t base = (((size_t)kc * K + r) * 4 + pl) * 6 * D2s;
                        w2[(base + hi_grp[t] * D2s + q) * 8 + e8] = hi;
                        w2[(base + lo_grp[t] * D2s + q) * 8 + e8] = lo;
                    } else {     // [kc][tap][plane][row: hi q | lo D2s + q][8]
                        const size_t base = (((size_t)kc * KK + tap) * 4 + pl) * 2 * D2s;
                        w2[(base + q) * 8 + e8] = hi;
                        w2[(base + D2s + q) * 8 + e8] = lo;
                    }
                }
    for (int n = 0; n < N; ++n)                 // [plane q/8][row: hi n | lo N3p + n][8]
        for (int q = 0; q < D2; ++q) {
            uint16_t hi, lo;
            split(u_out[(size_t)n * D2 + q], &hi, &lo);
            const size_t row = (size_t)(q / 8) * 2 * N3p;
            w3[(row + n) * 8 + q % 8] = hi;
            w3[(row + N3p + n) * 8 + q % 8] = lo;
        }
    (void)C64;
    const size_t wbytes = hb.size() * sizeof(uint16_t), nbias = round_up(N, 4);
    cudaError_t e = cudaMalloc(&p->d_tc_w, wbytes + nbias * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(layer weights)");
    e = cudaMemcpy(p->d_tc_w, hb.data(), wbytes, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && bias) {
        std::vector<float> bb(nbias, 0.f);
        for (int n = 0; n < N; ++n) bb[n] = bias[n];
        e = cudaMemcpy(reinterpret_cast<uint8_t *>(p->d_tc_w) + wbytes, bb.data(), nbias * sizeof(float),
                       cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(layer weights)");
    p->weight_bytes += wbytes + nbias * sizeof(float);
    const uint16_t *wb = reinterpret_cast<const uint16_t *>(p->d_tc_w);
    g.w1 = wb;
    g.w2 = wb + n1;
    g.w3 = wb + n1 + n2;
    g.bias = bias ? reinterpret_cast<const float *>(reinterpret_cast<uint8_t *>(p->d_tc_w) + wbytes) : nullptr;
    {
        const char *kn = std::getenv("TDC_LAYER_DBG");  // honoured by the debug builds only
        g.knobs = kn ? std::atoi(kn) : 0;
        const char *pf = std::getenv("TDC_LAYER_PF");   // L2 prefetch distance (blocks), A/B knob
        g.pf_blocks = pf ? std::atoi(pf) : 4;
    }
    p->bl = g;
    p->l_last_x = nullptr;
    p->variant = 5;
    *used = true;
    return TDC_OK;
}

tdc_status forward_layer(tdc_conv_plan_s *p, const float *x, float *y, int batch, cudaStream_t st,
                         const float *res = nullptr, int relu = 0) {
    tdc::BfLayerArgs g = p->bl;
    if (x != p->l_last_x || batch != p->l_last_batch) {
        // box {32 ch, Wp, rpb rows}: the padding columns/rows are out of bounds -> zeros
        if (!tdc::make_tma_4d_nhwc(&p->lmapX, x, g.C, g.W, g.H, batch, g.Wp, g.rpb))
            return fail(TDC_ERR_INVALID_ARGUMENT, "cuTensorMapEncodeTiled rejected x (needs 16-byte aligned pointer)");
        p->l_last_x = x;
        p->l_last_batch = batch;
    }
    g.B = batch;
    g.num_tiles = batch * g.T;
    g.y = y;
    g.res = res;
    g.relu = relu;
    const int grid = std::max(1, std::min(g.num_tiles, p->num_sms));
    if ((long long)g.num_tiles * grid >= (1LL << 32))  // the kernel splits tiles in 32-bit arithmetic
        return fail(TDC_ERR_INVALID_ARGUMENT, "batch too large for the single-launch layer kernel");
    cudaError_t e = tdc::bf_layer_launch(p->lmapX, g, grid, st);
    if (e != cudaSuccess) return cuda_fail(e, "3xBF16 single-launch layer kernel");
    return TDC_OK;
}

tdc_status forward_bf16(tdc_conv_plan_s *p, const float *x, float *y, int batch, cudaStream_t st,
                        const float *res = nullptr, int relu = 0) {
    const tdc::LayerDims &d = p->dims;
    auto &s1 = p->tc[0], &s3 = p->tc[2];
    if (x != p->tc_last_x || batch != p->tc_last_x_batch) {
        // extent = this call's images: a partial last tile is zero-filled, not read past x
        if (!tdc::make_tma_2d(&s1.mapA, x, (long long)batch * d.H * d.W, d.C, d.C, 128))
            return fail(TDC_ERR_INVALID_ARGUMENT,
                        "cuTensorMapEncodeTiled rejected x (needs 16-byte aligned pointer)");
        p->tc_last_x = x;
        p->tc_last_x_batch = batch;
    }
    tdc::TcGemmArgs a1 = s1.args, a3 = s3.args;
    a1.M = batch * d.H * d.W;
    a3.M = batch * d.Ho * d.Wo;
    a3.out = y;
    a3.res = res;
    a3.relu = relu;
    tdc::BfCoreArgs c = p->bf_core;
    c.res = res;
    c.relu = relu;
    c.M = batch * a1.Hq * a1.Wq;
    auto grid = [&](long long M, int ntiles, int smem, int bn) {
        const long long tiles = (long long)div_up((int)M, 128) * ntiles;
        const long long cap = (long long)p->num_sms * tdc::persistent_occupancy(smem, bn);
        return (int)std::max<long long>(1, std::min(tiles, cap));
    };
    // split-K launches: clusters of ksplit CTAs, one cluster per output tile (persistent);
    // split-K through L2 (gsplit): one unit per (tile, piece), at most one CTA per SM so that
    // every CTA is co-resident (a piece-0 CTA waits for its other pieces)
    auto grid_ks = [&](long long M, int ntiles, int smem, int bn, int ks, int gs = 1) {
        if (gs > 1)
            return (int)std::max<long long>(1, std::min<long long>((long long)div_up((int)M, 128) * ntiles * gs,
                                                                   p->num_sms));
        if (ks <= 1) return grid(M, ntiles, smem, bn);
        const long long tiles = (long long)div_up((int)M, 128) * ntiles;
        const long long cap = (long long)p->num_sms * tdc::persistent_occupancy(smem, bn) / ks;
        return (int)(std::max<long long>(1, std::min(tiles, cap)) * ks);
    };
    cudaError_t e = tdc::bf_gemm_launch(
        s1.mapA, s1.mapA, s1.mapB, s1.mapBlo, s1.mapA, a1,
        grid_ks(a1.M, a1.ntiles, tdc::bf_smem_bytes(a1.BN, a1.stages, a1.xstages, a1.ksplit, a1.bstages), a1.BN, a1.ksplit,
                a1.gsplit), st);
    if (e != cudaSuccess) return cuda_fail(e, "3xBF16 stage-1 launch");
    if (p->fuse3) {
        c.y = y;
        e = tdc::bf_core3_launch(c, grid(c.M, c.ntiles, tdc::bf_core3_smem_bytes(c), tdc::bf_core3_tmem_cols(c) / 2),
                                 st);
        if (e != cudaSuccess) return cuda_fail(e, "3xBF16 fused core+stage-3 launch");
        return TDC_OK;
    }
    if (p->core2) {  // one CTA pair per (pair of M tiles, N tile), persistent over the units
        const long long units = (long long)div_up(div_up((int)c.M, 128), 2) * c.ntiles;
        e = tdc::bf_core2_launch(c, 2 * (int)std::max<long long>(1, std::min<long long>(units, p->num_sms / 2)), st);
    } else {
        e = tdc::bf_core_launch(
            c, grid_ks(c.M, c.ntiles, tdc::bf_core_smem_bytes(c.BN, c.nphase, c.band_rows, c.tg, c.w_slots, c.ksplit),
                       c.ncat ? 2 * c.BN : c.BN, c.ksplit, c.gsplit), st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "3xBF16 stage-2 launch");
    if (a3.tma_y && (y != p->last_y3 || a3.M != p->last_y3_rows)) {
        // extent = this call's rows, so the stores of the last tile clip at the batch end
        if (!tdc::make_tma_2d(&p->mapY3, y, a3.M, d.N, d.N, 32))
            return fail(TDC_ERR_INVALID_ARGUMENT, "cuTensorMapEncodeTiled rejected y (16-byte aligned pointer?)");
        p->last_y3 = y;
        p->last_y3_rows = a3.M;
    }
    if (a3.tma_y && res && (res != p->last_r3 || a3.M != p->last_r3_rows)) {  // residual blocks by TMA
        if (!tdc::make_tma_2d(&p->mapR3, res, a3.M, d.N, d.N, 32))
            return fail(TDC_ERR_INVALID_ARGUMENT, "cuTensorMapEncodeTiled rejected residual (16-byte aligned?)");
        p->last_r3 = res;
        p->last_r3_rows = a3.M;
    }
    e = tdc::bf_gemm_launch(
        s3.mapA, s3.mapAlo, s3.mapB, s3.mapBlo, p->mapY3, a3,
        grid_ks(a3.M, a3.ntiles, tdc::bf_smem_bytes(a3.BN, a3.stages, 0, a3.ksplit, 0), a3.BN, a3.ksplit, a3.gsplit), st,
        res ? &p->mapR3 : nullptr);
    if (e != cudaSuccess) return cuda_fail(e, "3xBF16 stage-3 launch");
    return TDC_OK;
}

// Plan the fused single-kernel variant; returns TDC_OK and sets variant 3 if the
// layer fits the kernel's shared-memory / tensor-memory budget, otherwise leaves
// the plan untouched (caller falls back to the three-launch variant).
tdc_status plan_fused(tdc_conv_plan_s *p, const float *core, const float *u_in, const float *u_out,
                      const float *bias, bool *used) {
    *used = false;
    const tdc_conv_desc &d = p->desc;
    const int C = d.c_in, N = d.c_out, D1 = d.rank_in, D2 = d.rank_out, K = d.kernel;
    const int s = d.stride, pad = d.pad, H = d.height, W = d.width;
    const int Ho = p->dims.Ho, Wo = p->dims.Wo;
    const int D1s = round_up(D1, 32), D2s = round_up(D2, 32);
    if (C % 4 || D1s > 256 || D2s > 256 || K * K > tdc::kMaxTaps || s * s > tdc::kMaxTaps)
        return TDC_OK;
    const int Wp = W + 2 * pad, Wq = div_up(Wp, s);
    if (Wp > 256 || Wq > 128) return TDC_OK;
    const int kc1 = div_up(C, 32);
    int Nh = N < 256 ? round_up(N, 16) : 256;
    const int nhalves = div_up(N, Nh);
    // compact phases used by the taps
    int phase_idx[tdc::kMaxTaps], nph = 0;
    for (int i = 0; i < tdc::kMaxTaps; ++i) phase_idx[i] = -1;
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t) {
            const int ph = (r % s) * s + (t % s);
            if (phase_idx[ph] < 0) phase_idx[ph] = nph++;
        }
    const int maxoff = ((K - 1) / s) * Wq + (K - 1) / s;

    tdc::FusedArgs best;
    bool found = false;
    const int rmax = std::min(Ho, 128 / Wq);
    for (int R = rmax; R >= 1; --R) {
        tdc::FusedArgs g;
        std::memset(&g, 0, sizeof g);
        g.B = d.batch; g.H = H; g.W = W; g.C = C; g.N = N; g.Ho = Ho; g.Wo = Wo; g.K = K;
        g.KK = K * K; g.s = s; g.p = pad; g.R = R; g.Rin = s * (R - 1) + K; g.Wp = Wp; g.Wq = Wq;
        if (g.Rin > 256) continue;
        g.tiles_per_img = div_up(Ho, R);
        g.num_tiles = d.batch * g.tiles_per_img;
        g.nblk1 = div_up(g.Rin * Wp, 128);
        g.c_chunks = kc1;
        g.D1s = D1s; g.D2s = D2s; g.Nh = Nh; g.nhalves = nhalves;
        g.nph = nph;
        g.PR = round_up(div_up(g.Rin, s) * Wq, 8);
        g.TR = s == 1 ? std::max(g.Rin * Wp, 128 + maxoff)
                      : (nph - 1) * g.PR + std::max(g.PR, 128 + maxoff);
        g.TR = round_up(g.TR, 8);
        // TMEM: acc1 [nblk1][P1][D1s] and acc2 [P2][D2s] share columns (acc2 is written
        // only after epilogue 1 drained acc1); acc3 [nbuf3][P3][Nh] is separate.
        auto tmem_need = [&](int P1, int P2, int P3, int nb) {
            return std::max(g.nblk1 * P1 * D1s, P2 * D2s) + nb * P3 * Nh;
        };
        // Independent accumulator chains measured to give no gain (tcgen05.mma
        // issue cost is ~130-150 cycles per instruction regardless, see
        // DESIGN.md "tensor-core cost model"), so one chain per stage.
        g.P1 = 1;
        g.P2 = 1;
        g.P3 = 1;
        g.nbuf3 = 2;
        while (tmem_need(g.P1, g.P2, g.P3, g.nbuf3) > 512) {
            if (g.P3 > 1) --g.P3;
            else if (g.P1 > 1) --g.P1;
            else if (g.P2 > 2) g.P2 /= 2;
            else if (g.nbuf3 > 1) --g.nbuf3;
            else if (g.P2 > 1) --g.P2;
            else break;
        }
        const int cols = tmem_need(g.P1, g.P2, g.P3, g.nbuf3);
        if (cols > 512) continue;
        g.acc3_col = std::max(g.nblk1 * g.P1 * D1s, g.P2 * D2s);
        g.tmem_cols = 32;
        while (g.tmem_cols < cols) g.tmem_cols *= 2;
        // ring depths: as deep as shared memory allows (X: up to two tiles ahead)
        g.WS = 4;
        g.XS = std::max(2, std::min(2 * kc1, 8));
        while (g.XS > 2 && tdc::fused_smem_bytes(g) > p->max_smem) --g.XS;
        if (tdc::fused_smem_bytes(g) > p->max_smem) {
            g.WS = 2;
            if (tdc::fused_smem_bytes(g) > p->max_smem) continue;
        }
        while (g.WS < 8) {
            ++g.WS;
            if (tdc::fused_smem_bytes(g) > p->max_smem) { --g.WS; break; }
        }
        if (!found || (best.num_tiles < p->num_sms && g.num_tiles > best.num_tiles)) {
            best = g;
            found = true;
        }
        if (best.num_tiles >= p->num_sms) break;
    }
    if (!found) return TDC_OK;
    tdc::FusedArgs &g = best;
    // The kernel streams every weight chunk once per tile (from L2).  When that
    // outweighs the tile's own activation traffic (small images, large ranks),
    // the three-launch variant -- whose GEMM tiles reuse weights across more
    // rows -- is the better choice.
    {
        const double wbytes = (double)(kc1 * D1s + (D1s / 32) * K * K * D2s +
                                       g.nhalves * (D2s / 32) * Nh) * 128.0;
        const double abytes = ((double)g.Rin * W * C + (double)g.R * Wo * N) * 4.0;
        if (wbytes > 2.5 * abytes && !getenv("TDC_FORCE_FUSED")) return TDC_OK;
    }
    for (int r = 0; r < K; ++r)
        for (int t = 0; t < K; ++t) {
            g.tap_phase[r * K + t] = phase_idx[(r % s) * s + (t % s)];
            g.tap_off[r * K + t] = (r / s) * Wq + (t / s);
        }
    for (int i = 0; i < tdc::kMaxTaps; ++i) g.phase_idx[i] = phase_idx[i];

    // ---- a0: blocked weight chunks [8][rows][4] in consumption order ----
    const int KK = K * K, kc2 = D1s / 32, kc3 = D2s / 32;
    const size_t n1 = (size_t)kc1 * D1s * 32, n2 = (size_t)kc2 * KK * D2s * 32,
                 n3 = (size_t)nhalves * kc3 * Nh * 32, nb = (size_t)round_up(N, 4);
    std::vector<float> h(n1 + n2 + n3 + nb, 0.f);
    float *w1 = h.data(), *w2 = w1 + n1, *w3 = w2 + n2, *hb = w3 + n3;
    for (int c = 0; c < C; ++c)
        for (int a = 0; a < D1; ++a) {
            const int kc = c / 32, kg = (c % 32) / 4, e = c % 4;
            w1[(((size_t)kc * 8 + kg) * D1s + a) * 4 + e] = u_in[(size_t)c * D1 + a];
        }
    for (int q = 0; q < D2; ++q)
        for (int a = 0; a < D1; ++a)
            for (int r = 0; r < K; ++r)
                for (int t = 0; t < K; ++t) {
                    const int kc = a / 32, kg = (a % 32) / 4, e = a % 4, tap = r * K + t;
                    w2[((((size_t)kc * KK + tap) * 8 + kg) * D2s + q) * 4 + e] =
                        core[(((size_t)q * D1 + a) * K + r) * K + t];
                }
    for (int n = 0; n < N; ++n)
        for (int q = 0; q < D2; ++q) {
            const int hh = n / Nh, nn = n % Nh, kc = q / 32, kg = (q % 32) / 4, e = q % 4;
            w3[((((size_t)hh * kc3 + kc) * 8 + kg) * Nh + nn) * 4 + e] = u_out[(size_t)n * D2 + q];
        }
    if (bias)
        for (int n = 0; n < N; ++n) hb[n] = bias[n];
    cudaError_t e = cudaMalloc(&p->d_fw, h.size() * sizeof(float));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(fused weights)");
    e = cudaMemcpy(p->d_fw, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(fused weights)");
    p->weight_bytes += h.size() * sizeof(float);
    g.w = p->d_fw;
    g.bias = bias ? p->d_fw + n1 + n2 + n3 : nullptr;
    p->fargs = g;
    p->variant = 3;
    *used = true;
    return TDC_OK;
}

tdc_status forward_fused(tdc_conv_plan_s *p, const float *x, float *y, int batch, cudaStream_t st) {
    if (x != p->f_last_x) {
        if (!tdc::fused_make_x_map(&p->fmapX, x, p->fargs))
            return fail(TDC_ERR_INVALID_ARGUMENT,
                        "cuTensorMapEncodeTiled rejected x (needs a 16-byte aligned pointer)");
        p->f_last_x = x;
    }
    tdc::FusedArgs g = p->fargs;
    g.y = y;
    g.num_tiles = batch * g.tiles_per_img;
    const int grid = std::min(g.num_tiles, p->num_sms);
    cudaError_t e = tdc::fused_launch(p->fmapX, g, grid, st);
    if (e != cudaSuccess) return cuda_fail(e, "fused tcgen05 kernel launch");
    return TDC_OK;
}

tdc_status forward_tc(tdc_conv_plan_s *p, const float *x, float *y, int batch, cudaStream_t st) {
    const tdc::LayerDims &d = p->dims;
    auto &s1 = p->tc[0], &s2 = p->tc[1], &s3 = p->tc[2];
    if (x != p->tc_last_x || batch != p->tc_last_x_batch) {
        // extent = this call's images: a partial last tile is zero-filled, not read past x
        if (!tdc::make_tma_2d(&s1.mapA, x, (long long)batch * d.H * d.W, d.C, d.C, 128))
            return fail(TDC_ERR_INVALID_ARGUMENT,
                        "cuTensorMapEncodeTiled rejected x (needs 16-byte aligned pointer)");
        p->tc_last_x = x;
        p->tc_last_x_batch = batch;
    }
    tdc::TcGemmArgs a1 = s1.args, a2 = s2.args, a3 = s3.args;
    a1.M = batch * d.H * d.W;
    const int Hq = a1.Hq, Wq = a1.Wq;  // stage-1 args always carry the grid geometry
    a2.M = batch * Hq * Wq;
    a3.M = batch * d.Ho * d.Wo;
    a3.out = y;
    if (p->split) s1.mapAlo = s1.mapA;  // unused by the converter path; any valid map
    auto grid_of = [&](const tdc::TcGemmArgs &a) {
        const long long tiles = (long long)div_up(a.M, 128) * a.ntiles;
        const long long cap = (long long)p->num_sms *
                              tdc::persistent_occupancy(tdc::tc_smem_bytes(a.BN, a.stages, a.split), a.BN);
        return (int)std::max<long long>(1, std::min(tiles, cap));
    };
    cudaError_t e = tdc::tc_gemm_launch(s1.mapA, s1.mapAlo, s1.mapB, s1.mapBlo, a1, grid_of(a1), st);
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 stage-1 launch");
    if (p->tc_core) {
        tdc::TcCoreArgs c = p->core_args;
        c.M = a2.M;
        const long long tiles = (long long)div_up(c.M, 128) * c.ntiles;
        const long long cap = (long long)p->num_sms *
                              tdc::persistent_occupancy(tdc::tc_core_smem_bytes(c.BN, c.nphase, c.band_rows,
                                                                                c.b_stages, c.split), c.BN);
        e = tdc::tc_core_launch(c, (int)std::max<long long>(1, std::min(tiles, cap)), st);
        if (e != cudaSuccess)
            return fail(TDC_ERR_CUDA, "tcgen05 core launch: %s (M=%d ntiles=%d BN=%d smem=%d nphase=%d band=%d stages=%d)",
                        cudaGetErrorString(e), c.M, c.ntiles, c.BN,
                        tdc::tc_core_smem_bytes(c.BN, c.nphase, c.band_rows, c.b_stages, c.split), c.nphase,
                        c.band_rows, c.b_stages);
    } else {
        e = tdc::tc_gemm_launch(s2.mapA, s2.mapAlo, s2.mapB, s2.mapBlo, a2, grid_of(a2), st);
    }
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 stage-2 launch");
    e = tdc::tc_gemm_launch(s3.mapA, s3.mapAlo, s3.mapB, s3.mapBlo, a3, grid_of(a3), st);
    if (e != cudaSuccess) return cuda_fail(e, "tcgen05 stage-3 launch");
    return TDC_OK;
}

}  // namespace

extern "C" {

const char *tdc_version(void) { return "tdc-b200 0.1.0 (sm_100a)"; }

const char *tdc_status_string(tdc_status s) {
    switch (s) {
        case TDC_OK: return "ok";
        case TDC_ERR_INVALID_ARGUMENT: return "invalid argument";
        case TDC_ERR_UNSUPPORTED: return "unsupported";
        case TDC_ERR_CUDA: return "CUDA error";
        case TDC_ERR_OUT_OF_MEMORY: return "out of memory";
        case TDC_ERR_INTERNAL: return "internal error";
    }
    return "unknown status";
}

const char *tdc_last_error(void) { return g_last_error.c_str(); }

tdc_status tdc_conv_output_shape(const tdc_conv_desc *desc, int32_t *h_out, int32_t *w_out) {
    if (!h_out || !w_out) return fail(TDC_ERR_INVALID_ARGUMENT, "h_out/w_out is NULL");
    int ho, wo;
    tdc_status s = validate_desc(desc, &ho, &wo);
    if (s != TDC_OK) return s;
    *h_out = ho;
    *w_out = wo;
    return TDC_OK;
}

tdc_status tdc_conv_plan(const tdc_conv_desc *desc, const float *core, const float *u_in,
                         const float *u_out, const float *bias, int32_t device,
                         tdc_conv_plan_t *out) {
    return tdc_conv_plan_ex(desc, core, u_in, u_out, bias, nullptr, device, out);
}

tdc_status tdc_conv_plan_ex(const tdc_conv_desc *desc, const float *core, const float *u_in,
                            const float *u_out, const float *bias, const tdc_plan_hints *hints,
                            int32_t device, tdc_conv_plan_t *out) {
    if (!out) return fail(TDC_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    int ho, wo;
    tdc_status s = validate_desc(desc, &ho, &wo);
    if (s != TDC_OK) return s;
    if (!core || !u_in || !u_out)
        return fail(TDC_ERR_INVALID_ARGUMENT, "core, u_in and u_out must be non-NULL host arrays");
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (device < 0 || device >= ndev)
        return fail(TDC_ERR_INVALID_ARGUMENT, "device %d out of range (%d devices)", device, ndev);
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
    if (prop.major != 10 || prop.minor != 0)
        return fail(TDC_ERR_UNSUPPORTED, "device %d is sm_%d%d; this library is built for sm_100a only",
                    device, prop.major, prop.minor);

    DeviceGuard guard(device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");

    tdc_conv_plan_s *p = new (std::nothrow) tdc_conv_plan_s();
    if (!p) return fail(TDC_ERR_OUT_OF_MEMORY, "host allocation of plan failed");
    p->desc = *desc;
    p->device = device;
    if (hints) p->hints = *hints;
    const tdc_conv_desc &d = *desc;
    p->dims = tdc::LayerDims{d.batch, d.c_in, d.height, d.width, d.c_out, d.kernel,
                             d.stride, d.pad, ho, wo};
    const int C = d.c_in, N = d.c_out, D1 = d.rank_in, D2 = d.rank_out, K = d.kernel;
    p->D1p = round_up(D1, 4);
    p->D2p = round_up(D2, 4);
    p->Np = round_up(N, 4);
    const int D1p = p->D1p, D2p = p->D2p, Np = p->Np;

    // ---- a0: offline re-layout (CRSN idea), zero-padded ranks ----
    const size_t n_uin = (size_t)C * D1p, n_core = (size_t)K * K * D1p * D2p,
                 n_uout = (size_t)D2p * Np, n_bias = (size_t)Np;
    std::vector<float> h((n_uin + n_core + n_uout + n_bias), 0.f);
    float *h_uin = h.data(), *h_core = h_uin + n_uin, *h_uout = h_core + n_core,
          *h_bias = h_uout + n_uout;
    for (int c = 0; c < C; ++c)
        for (int a = 0; a < D1; ++a) h_uin[(size_t)c * D1p + a] = u_in[(size_t)c * D1 + a];
    for (int q = 0; q < D2; ++q)
        for (int a = 0; a < D1; ++a)
            for (int r = 0; r < K; ++r)
                for (int t = 0; t < K; ++t)
                    h_core[((size_t)(r * K + t) * D1p + a) * D2p + q] =
                        core[(((size_t)q * D1 + a) * K + r) * K + t];
    for (int n = 0; n < N; ++n)
        for (int q = 0; q < D2; ++q) h_uout[(size_t)q * Np + n] = u_out[(size_t)n * D2 + q];
    if (bias)
        for (int n = 0; n < N; ++n) h_bias[n] = bias[n];

    p->weight_bytes = h.size() * sizeof(float);
    e = cudaMalloc(&p->d_weights, p->weight_bytes);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaMalloc(weights)");
    }
    e = cudaMemcpy(p->d_weights, h.data(), p->weight_bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        tdc_conv_plan_destroy(p);
        return cuda_fail(e, "cudaMemcpy(weights)");
    }
    p->simt = tdc::SimtWeights{p->d_weights, p->d_weights + n_uin,
                               p->d_weights + n_uin + n_core,
                               bias ? p->d_weights + n_uin + n_core + n_uout : nullptr, D1p, D2p,
                               Np};

    // ---- variant selection ----
    const int max_smem = (int)prop.sharedMemPerBlockOptin;
    p->max_smem = max_smem;
    if (!tdc::simt_choose_tile(p->dims, D1p, D2p, max_smem, &p->simt_tile)) {
        tdc_conv_plan_destroy(p);
        return fail(TDC_ERR_UNSUPPORTED, "ranks D1=%d D2=%d too large for the fused kernel's "
                    "shared-memory budget (%d bytes)", D1, D2, max_smem);
    }
    p->variant = 1;
    // Tensor-core variant: TMA needs 16-byte row pitches (C % 4 == 0) and at most
    // kMaxTaps taps; otherwise the plan keeps the (more accurate) fp32 variant.
    p->num_sms = prop.multiProcessorCount;
    bool fused = false;
    if (d.math == TDC_MATH_TF32 && !getenv("TDC_DISABLE_FUSED")) {
        s = plan_fused(p, core, u_in, u_out, bias, &fused);
        if (s != TDC_OK) {
            tdc_conv_plan_destroy(p);
            return s;
        }
    }
    if (d.math == TDC_MATH_FP32) {
        bool sg = false;
        s = plan_sgemm(p, core, u_in, u_out, bias, &sg);
        if (s != TDC_OK) {
            tdc_conv_plan_destroy(p);
            return s;
        }
    }
    bool bf = false;
    if (d.math == TDC_MATH_3XBF16) {
        s = plan_layer(p, core, u_in, u_out, bias, &bf);
        if (s != TDC_OK) {
            tdc_conv_plan_destroy(p);
            return s;
        }
    }
    if (d.math == TDC_MATH_3XBF16 && !bf) {
        s = plan_bf16(p, core, u_in, u_out, bias, &bf);
        if (s != TDC_OK) {
            tdc_conv_plan_destroy(p);
            return s;
        }
    }
    if (!fused && !bf && d.math != TDC_MATH_FP32 && C % 4 == 0 && K * K <= tdc::kMaxTaps) {
        s = plan_tc(p, core, u_in, u_out, bias, d.math != TDC_MATH_TF32);
        if (s != TDC_OK) {
            tdc_conv_plan_destroy(p);
            return s;
        }
    }

    if (d.layout == TDC_LAYOUT_NCHW) {
        const size_t in_b = (size_t)d.batch * C * d.height * d.width * sizeof(float);
        const size_t out_b = (size_t)d.batch * N * ho * wo * sizeof(float);
        e = cudaMalloc(&p->d_ws_in, in_b);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_ws_out, out_b);
        if (e != cudaSuccess) {
            tdc_conv_plan_destroy(p);
            return cuda_fail(e, "cudaMalloc(NCHW workspace)");
        }
        p->ws_bytes = in_b + out_b;
    }
    *out = p;
    return TDC_OK;
}

tdc_status tdc_conv_plan_query(tdc_conv_plan_t p, tdc_plan_info *info) {
    if (!p || !info) return fail(TDC_ERR_INVALID_ARGUMENT, "plan/info is NULL");
    std::memset(info, 0, sizeof *info);
    info->h_out = p->dims.Ho;
    info->w_out = p->dims.Wo;
    info->variant = p->variant;
    const bool tc = p->variant == 2 || p->variant == 4, fz = p->variant == 3;
    std::snprintf(info->variant_name, sizeof info->variant_name, "%s",
                  p->variant == 6 ? "simt3_fp32" : p->variant == 5 ? "layer_3xbf16_fused" :
                  p->variant == 4 ? (p->fuse3 ? "tc2_3xbf16_core3" : p->core2 ? "tc3_3xbf16_pair" : "tc3_3xbf16_band") : fz ? "fused_tc_tf32"
                     : tc ? (p->split ? (p->tc_core ? "tc3_3xtf32_band" : "tc3_3xtf32")
                                      : (p->tc_core ? "tc3_tf32_band" : "tc3_tf32"))
                          : "fused_simt_fp32");
    info->launches_per_forward =
        (tc ? (p->variant == 4 && p->fuse3 ? 2 : 3) : 1) + (p->desc.layout == TDC_LAYOUT_NCHW ? 2 : 0);
    info->concurrent_forward = (p->desc.layout == TDC_LAYOUT_NHWC && !tc) ? 1 : 0;
    info->tile_h = p->simt_tile.oth;
    info->tile_w = p->simt_tile.otw;
    info->threads_per_cta = 256;
    info->smem_bytes_per_cta = p->simt_tile.smem_bytes;
    info->ctas_per_image = (int64_t)p->simt_tile.tiles_h * p->simt_tile.tiles_w;
    info->workspace_bytes = (int64_t)(p->ws_bytes + p->tc_ws_bytes);
    if (tc) {
        info->tile_h = 128;
        info->tile_w = p->tc[1].args.BN;
        info->threads_per_cta = 192;
        info->smem_bytes_per_cta = tdc::tc_smem_bytes(p->tc[1].args.BN, p->tc[1].args.stages, p->split);
        info->ctas_per_image = 0;
    }
    if (p->variant == 4) {  // stage-2 (core) kernel geometry
        const tdc::BfCoreArgs &c = p->bf_core;
        info->bn_stage1 = p->tc[0].args.BN;
        info->ksplit_stage1 = std::max(1, p->tc[0].args.ksplit);
        info->bn_core = c.BN;
        info->ksplit_core = std::max(1, c.ksplit);
        info->bn_stage3 = p->fuse3 ? c.N3p : p->tc[2].args.BN;
        info->ksplit_stage3 = p->fuse3 ? 1 : std::max(1, p->tc[2].args.ksplit);
        info->core3 = p->fuse3 ? 1 : 0;
        info->gsplit_stage1 = std::max(1, p->tc[0].args.gsplit);
        info->gsplit_core = std::max(1, c.gsplit);
        info->gsplit_stage3 = p->fuse3 ? 1 : std::max(1, p->tc[2].args.gsplit);
        info->tile_w = c.BN;
        info->threads_per_cta = p->fuse3 ? 448 : 192;
        info->smem_bytes_per_cta = p->fuse3   ? tdc::bf_core3_smem_bytes(c)
                                   : p->core2 ? tdc::bf_core2_smem_bytes(c.BN, c.nphase, c.band_rows, c.w_slots, c.a_slots)
                                              : tdc::bf_core_smem_bytes(c.BN, c.nphase, c.band_rows, c.tg, c.w_slots,
                                                                        c.ksplit);
    }
    if (fz) {
        info->tile_h = p->fargs.R;
        info->tile_w = p->fargs.Wo;
        info->threads_per_cta = 384;
        info->smem_bytes_per_cta = tdc::fused_smem_bytes(p->fargs);
        info->ctas_per_image = p->fargs.tiles_per_img;  // tiles per image (persistent grid)
        info->concurrent_forward = p->desc.layout == TDC_LAYOUT_NHWC ? 1 : 0;
    }
    if (p->variant == 6) {
        info->launches_per_forward = 3 + (p->desc.layout == TDC_LAYOUT_NCHW ? 2 : 0);
        info->concurrent_forward = 0;
        info->threads_per_cta = 256;
        info->ctas_per_image = 0;
    }
    if (p->variant == 5) {
        const tdc::BfLayerArgs &g = p->bl;
        info->launches_per_forward = 1 + (p->desc.layout == TDC_LAYOUT_NCHW ? 2 : 0);
        info->tile_h = g.R;
        info->tile_w = g.Wo;
        info->threads_per_cta = 640;
        info->smem_bytes_per_cta = tdc::bf_layer_smem_bytes(g);
        info->ctas_per_image = g.T;  // tiles per image (persistent grid)
        info->bn_stage1 = g.D1s;
        info->bn_core = g.D2s;
        info->bn_stage3 = g.N3p;
        info->ksplit_stage1 = info->ksplit_core = info->ksplit_stage3 = 1;
        info->gsplit_stage1 = info->gsplit_core = info->gsplit_stage3 = 1;
        info->core3 = 1;
    }
    info->weight_bytes = (int64_t)p->weight_bytes;
    return TDC_OK;
}

tdc_status tdc_conv_forward(tdc_conv_plan_t p, const float *x, float *y, int32_t batch,
                            void *stream) {
    if (!p) return fail(TDC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (!x || !y) return fail(TDC_ERR_INVALID_ARGUMENT, "x and y must be non-NULL device pointers");
    if (batch < 1 || batch > p->desc.batch)
        return fail(TDC_ERR_INVALID_ARGUMENT, "batch %d outside [1, %d] of this plan", batch,
                    p->desc.batch);
    const tdc::LayerDims &d = p->dims;
    const size_t in_elems = (size_t)batch * d.C * d.H * d.W;
    const size_t out_elems = (size_t)batch * d.N * d.Ho * d.Wo;
    if ((const char *)x < (const char *)(y + out_elems) &&
        (const char *)y < (const char *)(x + in_elems))
        return fail(TDC_ERR_INVALID_ARGUMENT, "x and y must not alias");
    DeviceGuard guard(p->device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    if (p->desc.layout == TDC_LAYOUT_NHWC) {
        if (p->variant == 6) return forward_sgemm(p, x, y, batch, st);
        if (p->variant == 5) return forward_layer(p, x, y, batch, st);
        if (p->variant == 4) return forward_bf16(p, x, y, batch, st);
        if (p->variant == 3) return forward_fused(p, x, y, batch, st);
        if (p->variant == 2) return forward_tc(p, x, y, batch, st);
        e = tdc::simt_fused_launch(d, p->simt, p->simt_tile, x, y, batch, st);
        if (e != cudaSuccess) return cuda_fail(e, "fused SIMT kernel launch");
        return TDC_OK;
    }
    e = tdc::nchw_to_nhwc(x, p->d_ws_in, batch, d.C, d.H, d.W, st);
    if (e != cudaSuccess) return cuda_fail(e, "NCHW->NHWC launch");
    if (p->variant == 6) {
        tdc_status s = forward_sgemm(p, p->d_ws_in, p->d_ws_out, batch, st);
        if (s != TDC_OK) return s;
    } else if (p->variant == 5) {
        tdc_status s = forward_layer(p, p->d_ws_in, p->d_ws_out, batch, st);
        if (s != TDC_OK) return s;
    } else if (p->variant == 4) {
        tdc_status s = forward_bf16(p, p->d_ws_in, p->d_ws_out, batch, st);
        if (s != TDC_OK) return s;
    } else if (p->variant == 3) {
        tdc_status s = forward_fused(p, p->d_ws_in, p->d_ws_out, batch, st);
        if (s != TDC_OK) return s;
    } else if (p->variant == 2) {
        tdc_status s = forward_tc(p, p->d_ws_in, p->d_ws_out, batch, st);
        if (s != TDC_OK) return s;
    } else {
        e = tdc::simt_fused_launch(d, p->simt, p->simt_tile, p->d_ws_in, p->d_ws_out, batch, st);
        if (e != cudaSuccess) return cuda_fail(e, "fused SIMT kernel launch");
    }
    e = tdc::nhwc_to_nchw(p->d_ws_out, y, batch, d.N, d.Ho, d.Wo, st);
    if (e != cudaSuccess) return cuda_fail(e, "NHWC->NCHW launch");
    return TDC_OK;
}

tdc_status tdc_conv_forward_ex(tdc_conv_plan_t p, const float *x, float *y, int32_t batch,
                               const float *residual, int32_t relu, void *stream) {
    if (!residual && !relu) return tdc_conv_forward(p, x, y, batch, stream);
    if (!p) return fail(TDC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (!x || !y) return fail(TDC_ERR_INVALID_ARGUMENT, "x/y is NULL");
    if (batch < 1 || batch > p->desc.batch)
        return fail(TDC_ERR_INVALID_ARGUMENT, "batch %d outside [1, %d] of this plan", batch, p->desc.batch);
    if ((p->variant != 4 && p->variant != 5) || p->desc.layout != TDC_LAYOUT_NHWC)
        return fail(TDC_ERR_UNSUPPORTED,
                    "residual/relu epilogue needs an NHWC plan in TDC_MATH_3XBF16 (this plan: variant %d)",
                    p->variant);
    {   // x / residual must not overlap y (ranges, not just equal pointers)
        const tdc::LayerDims &d = p->dims;
        const char *y0 = (const char *)y, *y1 = (const char *)(y + (size_t)batch * d.N * d.Ho * d.Wo);
        const char *x0 = (const char *)x, *x1 = (const char *)(x + (size_t)batch * d.C * d.H * d.W);
        if (x0 < y1 && y0 < x1) return fail(TDC_ERR_INVALID_ARGUMENT, "x and y must not alias");
        if (residual) {
            const char *r0 = (const char *)residual, *r1 = (const char *)(residual + (size_t)batch * d.N * d.Ho * d.Wo);
            if (r0 < y1 && y0 < r1) return fail(TDC_ERR_INVALID_ARGUMENT, "residual must not overlap y");
        }
    }
    DeviceGuard guard(p->device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
    if (p->variant == 5) return forward_layer(p, x, y, batch, (cudaStream_t)stream, residual, relu);
    return forward_bf16(p, x, y, batch, (cudaStream_t)stream, residual, relu);
}

namespace {

// Host-buffer forward, shared by tdc_conv_forward_host and tdc_conv_forward_host_many:
// validation, plan-owned staging buffers and the copy streams / events.
tdc_status host_prepare(tdc_conv_plan_t p, const float *x_host, const float *y_host, int32_t batch) {
    if (!p) return fail(TDC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (!x_host || !y_host) return fail(TDC_ERR_INVALID_ARGUMENT, "x_host/y_host is NULL");
    if (batch < 1 || batch > p->desc.batch)
        return fail(TDC_ERR_INVALID_ARGUMENT, "batch %d outside [1, %d] of this plan", batch,
                    p->desc.batch);
    const tdc::LayerDims &d = p->dims;
    cudaError_t e = cudaSuccess;
    if (!p->d_stage_x) {
        const size_t max_in = (size_t)p->desc.batch * d.C * d.H * d.W * sizeof(float);
        const size_t max_out = (size_t)p->desc.batch * d.N * d.Ho * d.Wo * sizeof(float);
        // + 256 pixel rows of slack: a chunk of the pipeline below starts mid-buffer
        e = cudaMalloc(&p->d_stage_x, max_in + (size_t)256 * d.C * sizeof(float));
        if (e == cudaSuccess) e = cudaMalloc(&p->d_stage_y, max_out);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(host-forward staging)");
    }
    if (!p->s_in) {
        e = cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking);
        for (int i = 0; e == cudaSuccess && i < 17; ++i) e = cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate/cudaEventCreate (host-forward pipeline)");
    }
    return TDC_OK;
}

// Pipeline one forward over image chunks (images are independent): the H2D
// copy of chunk k+1 (s_in) and the D2H copy of chunk k-1 (s_out) overlap the forward of
// chunk k on `st`, so the two link directions run concurrently instead of back to back.
// Chunks of >= ~2 MB of traffic, at most 8.  `ev` is a ring of 16 events (each is waited
// on right after it is recorded, so the ring can wrap); *evi is its cursor.
tdc_status host_enqueue(tdc_conv_plan_t p, const float *x_host, float *y_host, int32_t batch, cudaStream_t st,
                        cudaStream_t s_in, cudaStream_t s_out, cudaEvent_t *ev, int *evi) {
    const tdc::LayerDims &d = p->dims;
    const size_t in_b = (size_t)batch * d.C * d.H * d.W * sizeof(float);
    const size_t out_b = (size_t)batch * d.N * d.Ho * d.Wo * sizeof(float);
    const size_t in_img = in_b / batch, out_img = out_b / batch;
    const int nch = std::max(1, std::min<int>({batch, 8, (int)((in_b + out_b) / (2u << 20))}));
    cudaError_t e;
    for (int k = 0; k < nch; ++k) {
        const int b0 = (int)((long long)k * batch / nch), nb = (int)((long long)(k + 1) * batch / nch) - b0;
        float *dx = p->d_stage_x + b0 * (in_img / sizeof(float)), *dy = p->d_stage_y + b0 * (out_img / sizeof(float));
        cudaEvent_t e_in = ev[(*evi)++ & 15], e_fw = ev[(*evi)++ & 15];
        e = cudaMemcpyAsync(dx, reinterpret_cast<const uint8_t *>(x_host) + b0 * in_img, nb * in_img,
                            cudaMemcpyHostToDevice, s_in);
        if (e == cudaSuccess) e = cudaEventRecord(e_in, s_in);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, e_in, 0);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(H2D)");
        const tdc_status s = tdc_conv_forward(p, dx, dy, nb, st);
        if (s != TDC_OK) return s;
        e = cudaEventRecord(e_fw, st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(s_out, e_fw, 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(reinterpret_cast<uint8_t *>(y_host) + b0 * out_img, dy, nb * out_img,
                                cudaMemcpyDeviceToHost, s_out);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    }
    return TDC_OK;
}

tdc_status host_begin(tdc_conv_plan_t p, cudaStream_t st) {  // earlier work on `st` comes first
    cudaError_t e = cudaEventRecord(p->ev[16], st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_in, p->ev[16], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(p->s_out, p->ev[16], 0);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventRecord/cudaStreamWaitEvent");
    return TDC_OK;
}

tdc_status host_finish(tdc_conv_plan_t p, cudaStream_t st) {
    cudaError_t e = cudaStreamSynchronize(p->s_out);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return TDC_OK;
}

}  // namespace

tdc_status tdc_conv_forward_host(tdc_conv_plan_t p, const float *x_host, float *y_host,
                                 int32_t batch, void *stream) {
    if (!p) return fail(TDC_ERR_INVALID_ARGUMENT, "plan is NULL");
    // staging buffers, copy streams and events are created on the plan's device
    DeviceGuard guard(p->device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
    tdc_status s = host_prepare(p, x_host, y_host, batch);
    if (s != TDC_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((s = host_begin(p, st)) != TDC_OK) return s;
    int evi = 0;
    if ((s = host_enqueue(p, x_host, y_host, batch, st, p->s_in, p->s_out, p->ev, &evi)) != TDC_OK) return s;
    return host_finish(p, st);
}

tdc_status tdc_conv_forward_host_many(const tdc_conv_plan_t *plans, const float *const *x_hosts,
                                      float *const *y_hosts, const int32_t *batches, int32_t n, void *stream) {
    if (!plans || !x_hosts || !y_hosts || !batches || n < 1)
        return fail(TDC_ERR_INVALID_ARGUMENT, "plans/x_hosts/y_hosts/batches NULL or n < 1");
    for (int i = 0; i < n; ++i) {  // one device for all plans, checked before any allocation
        if (!plans[i]) return fail(TDC_ERR_INVALID_ARGUMENT, "plan %d is NULL", i);
        if (plans[i]->device != plans[0]->device)
            return fail(TDC_ERR_INVALID_ARGUMENT, "plan %d is on device %d, plan 0 on %d", i, plans[i]->device,
                        plans[0]->device);
    }
    tdc_conv_plan_t p0 = plans[0];
    DeviceGuard guard(p0->device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
    for (int i = 0; i < n; ++i) {
        const tdc_status s = host_prepare(plans[i], x_hosts[i], y_hosts[i], batches[i]);
        if (s != TDC_OK) return s;
    }
    cudaStream_t st = (cudaStream_t)stream;
    tdc_status s = host_begin(p0, st);
    if (s != TDC_OK) return s;
    int evi = 0;  // one chunk stream across all n forwards: copies of one overlap the next's
    for (int i = 0; i < n; ++i)
        if ((s = host_enqueue(plans[i], x_hosts[i], y_hosts[i], batches[i], st, p0->s_in, p0->s_out, p0->ev,
                              &evi)) != TDC_OK)
            return s;
    return host_finish(p0, st);
}

// Debug only (not in tdc.h): run the single-launch layer kernel with CTA 0's shared
// memory copied to dbg_dev (device, >= smem bytes) at exit.  Returns the layout offsets
// (xs, w1, w2, w3, band, z) in off[6].
tdc_status tdc_debug_layer_forward(tdc_conv_plan_t p, const float *x, float *y, int32_t batch, void *dbg_dev,
                                   int32_t *off) {
    if (!p || p->variant != 5) return fail(TDC_ERR_INVALID_ARGUMENT, "not a single-launch layer plan");
    DeviceGuard guard(p->device);
    p->bl.dbg = reinterpret_cast<uint8_t *>(dbg_dev);
    const tdc_status s = forward_layer(p, x, y, batch, nullptr);
    p->bl.dbg = nullptr;
    const tdc::BfLayerArgs &g = p->bl;
    const int XS = g.XS;
    off[0] = 0;
    off[1] = XS * 2 * g.XR * 128;
    off[2] = off[1] + g.cchunks * 2 * g.D1s * 128;
    off[3] = off[2] + (g.D1s / 32) * g.KK * 4 * 2 * g.D2s * 16;
    off[4] = off[3] + (g.D2s / 8) * 2 * g.N3p * 16;
    off[5] = off[4] + 2 * (g.D1s / 8) * g.NRB * g.Wq * 16;  // Z buffer 0
    return s;
}

tdc_status tdc_conv_plan_destroy(tdc_conv_plan_t p) {
    if (!p) return TDC_OK;
    DeviceGuard guard(p->device);
    cudaFree(p->d_weights);
    cudaFree(p->d_ws_in);
    cudaFree(p->d_ws_out);
    cudaFree(p->d_stage_x);
    cudaFree(p->d_stage_y);
    if (p->s_in) {
        cudaStreamDestroy(p->s_in);
        cudaStreamDestroy(p->s_out);
        for (cudaEvent_t ev : p->ev) cudaEventDestroy(ev);
    }
    cudaFree(p->d_tc_w);
    cudaFree(p->d_fw);
    cudaFree(p->d_xg);
    cudaFree(p->d_z);
    cudaFree(p->d_gs);
    cudaFree(p->d_sg);
    cudaFree(p->d_sg_part);
    cudaFree(p->d_c2w);
    delete p;
    return TDC_OK;
}

}  // extern "C"

// ---- helpers for the model runtime (tdc_model.cu)
namespace tdc {
uint16_t bf16_bits(float x) { return bf16_bits_host(x); }
float bf16_float(uint16_t b) { return bf16_to_float_host(b); }
tdc_status set_error(tdc_status s, const char *msg) { return fail(s, "%s", msg); }
int num_sms_of(int device) {
    int v = 148;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) v = 148;
    return v;
}
int max_smem_of(int device) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) v = 232448;
    return v;
}
}  // namespace tdc
