// tdc_api.cu -- the C-ABI of include/tdc.h: validation, plan-time weight
// re-layout (§8(a) row a0), variant selection and forward dispatch.
#include "../../include/tdc.h"
#include "internal.h"

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

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
    if (d->math < TDC_MATH_FP32 || d->math > TDC_MATH_TF32)
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
};

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
    if (desc->math != TDC_MATH_FP32)
        return fail(TDC_ERR_UNSUPPORTED, "math mode %d is not available in this build", desc->math);

    DeviceGuard guard(device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");

    tdc_conv_plan_s *p = new (std::nothrow) tdc_conv_plan_s();
    if (!p) return fail(TDC_ERR_OUT_OF_MEMORY, "host allocation of plan failed");
    p->desc = *desc;
    p->device = device;
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
    if (!tdc::simt_choose_tile(p->dims, D1p, D2p, max_smem, &p->simt_tile)) {
        tdc_conv_plan_destroy(p);
        return fail(TDC_ERR_UNSUPPORTED, "ranks D1=%d D2=%d too large for the fused kernel's "
                    "shared-memory budget (%d bytes)", D1, D2, max_smem);
    }
    p->variant = 1;

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
    std::snprintf(info->variant_name, sizeof info->variant_name, "%s", "fused_simt_fp32");
    info->launches_per_forward = p->desc.layout == TDC_LAYOUT_NCHW ? 3 : 1;
    info->concurrent_forward = p->desc.layout == TDC_LAYOUT_NHWC ? 1 : 0;
    info->tile_h = p->simt_tile.oth;
    info->tile_w = p->simt_tile.otw;
    info->threads_per_cta = 256;
    info->smem_bytes_per_cta = p->simt_tile.smem_bytes;
    info->ctas_per_image = (int64_t)p->simt_tile.tiles_h * p->simt_tile.tiles_w;
    info->workspace_bytes = (int64_t)p->ws_bytes;
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
        e = tdc::simt_fused_launch(d, p->simt, p->simt_tile, x, y, batch, st);
        if (e != cudaSuccess) return cuda_fail(e, "fused SIMT kernel launch");
        return TDC_OK;
    }
    e = tdc::nchw_to_nhwc(x, p->d_ws_in, batch, d.C, d.H, d.W, st);
    if (e != cudaSuccess) return cuda_fail(e, "NCHW->NHWC launch");
    e = tdc::simt_fused_launch(d, p->simt, p->simt_tile, p->d_ws_in, p->d_ws_out, batch, st);
    if (e != cudaSuccess) return cuda_fail(e, "fused SIMT kernel launch");
    e = tdc::nhwc_to_nchw(p->d_ws_out, y, batch, d.N, d.Ho, d.Wo, st);
    if (e != cudaSuccess) return cuda_fail(e, "NHWC->NCHW launch");
    return TDC_OK;
}

tdc_status tdc_conv_forward_host(tdc_conv_plan_t p, const float *x_host, float *y_host,
                                 int32_t batch, void *stream) {
    if (!p) return fail(TDC_ERR_INVALID_ARGUMENT, "plan is NULL");
    if (!x_host || !y_host) return fail(TDC_ERR_INVALID_ARGUMENT, "x_host/y_host is NULL");
    if (batch < 1 || batch > p->desc.batch)
        return fail(TDC_ERR_INVALID_ARGUMENT, "batch %d outside [1, %d] of this plan", batch,
                    p->desc.batch);
    const tdc::LayerDims &d = p->dims;
    const size_t in_b = (size_t)batch * d.C * d.H * d.W * sizeof(float);
    const size_t out_b = (size_t)batch * d.N * d.Ho * d.Wo * sizeof(float);
    DeviceGuard guard(p->device);
    if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice");
    cudaError_t e;
    if (!p->d_stage_x) {
        const size_t max_in = (size_t)p->desc.batch * d.C * d.H * d.W * sizeof(float);
        const size_t max_out = (size_t)p->desc.batch * d.N * d.Ho * d.Wo * sizeof(float);
        e = cudaMalloc(&p->d_stage_x, max_in);
        if (e == cudaSuccess) e = cudaMalloc(&p->d_stage_y, max_out);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(host-forward staging)");
    }
    cudaStream_t st = (cudaStream_t)stream;
    e = cudaMemcpyAsync(p->d_stage_x, x_host, in_b, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(H2D)");
    tdc_status s = tdc_conv_forward(p, p->d_stage_x, p->d_stage_y, batch, stream);
    if (s != TDC_OK) return s;
    e = cudaMemcpyAsync(y_host, p->d_stage_y, out_b, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpyAsync(D2H)");
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
    return TDC_OK;
}

tdc_status tdc_conv_plan_destroy(tdc_conv_plan_t p) {
    if (!p) return TDC_OK;
    DeviceGuard guard(p->device);
    cudaFree(p->d_weights);
    cudaFree(p->d_ws_in);
    cudaFree(p->d_ws_out);
    cudaFree(p->d_stage_x);
    cudaFree(p->d_stage_y);
    delete p;
    return TDC_OK;
}

}  // extern "C"
