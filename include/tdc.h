/*
 * tdc.h -- C-ABI of the B200-native Tucker-format (TKD) convolution library
 * (libtdc.so, built from paper_2211_03715_b200/csrc for sm_100a).
 *
 * The operation (BASELINE.json north_star): a TKD convolution
 * layer, the Tucker-2 format of a K x K convolution ("truncates ...
 * mode-1 and mode-2 matricization"; Eq. tkd2 referenced there), evaluated as
 * three stages
 *
 *   stage 1  X'[b,h,w,a] = sum_c U_in[c,a] X[b,c,h,w]                 (1x1, C -> D1)
 *   stage 2  Z[b,q,i,j]  = sum_a sum_r sum_t core[q,a,r,t]
 *                              X'[b, i*s-p+r, j*s-p+t, a]              (K x K, D1 -> D2)
 *   stage 3  Y[b,n,i,j]  = sum_q U_out[n,q] Z[b,q,i,j] (+ bias[n])      (1x1, D2 -> N)
 *
 * which equals one convolution with the reconstructed kernel
 * W[n,c,r,t] = sum_{a,q} U_out[n,q] core[q,a,r,t] U_in[c,a] (Eq. tkd2).
 * Stage 2 is the paper's "core convolution" (§5).  Conventions
 * (DESIGN.md readings): cross-correlation (R4); stride and zero padding act on
 * the core stage only (R5, R6); H' = floor((H + 2p - K)/s) + 1; B is batch and
 * N output channels (R3).
 *
 * Threading: all calls are thread-safe on distinct plans.  A plan is immutable
 * after creation; tdc_conv_forward may run concurrently on different streams
 * only when tdc_plan_info.concurrent_forward is 1 (NHWC plans; NCHW plans use
 * a plan-owned conversion workspace).
 *
 * Errors: every call returns a tdc_status; nothing throws or aborts across the
 * ABI.  On failure tdc_last_error() (thread-local) holds a one-line message.
 * Asynchronous device faults surface at the caller's next synchronisation.
 */
#ifndef TDC_H
#define TDC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TDC_OK = 0,
    TDC_ERR_INVALID_ARGUMENT = 1, /* bad size, rank bound, null pointer, batch > plan  */
    TDC_ERR_UNSUPPORTED = 2,      /* device is not sm_100 / math mode not available    */
    TDC_ERR_CUDA = 3,             /* a CUDA runtime/driver call or launch failed        */
    TDC_ERR_OUT_OF_MEMORY = 4,    /* device or host allocation failed                   */
    TDC_ERR_INTERNAL = 5
} tdc_status;

typedef enum {
    TDC_LAYOUT_NCHW = 0, /* the paper's statement; converted on device    */
    TDC_LAYOUT_NHWC = 1  /* fast path: channel-fastest, what the kernels read/write */
} tdc_layout;

typedef enum {
    TDC_MATH_FP32 = 0,   /* fp32 FFMA on CUDA cores (the paper's precision); tol 1e-4 */
    TDC_MATH_3XTF32 = 1, /* tcgen05 TF32 with hi/lo split (3 products); tol 1e-4            */
    TDC_MATH_TF32 = 2,   /* tcgen05 TF32, one product; tol 1e-2 (north_star)                */
    TDC_MATH_3XBF16 = 3  /* tcgen05 bf16 with hi/lo split (3 products, lo*lo dropped):
                          * ~2^-16 relative per product -- NOT IEEE fp32 (about 40x the fp32
                          * kernel's error on the same layer) but within the 1e-4
                          * max-normalized tolerance; integer layers bit-exact             */
} tdc_math;

/* Layer descriptor.  All sizes > 0; 1 <= rank_in <= c_in and
 * 1 <= rank_out <= c_out; kernel <= height + 2*pad and
 * kernel <= width + 2*pad; stride >= 1; pad >= 0. */
typedef struct {
    int32_t batch;             /* B: maximum batch this plan serves                 */
    int32_t c_in, height, width; /* C, H, W of the input                            */
    int32_t c_out;             /* N: output channels                                 */
    int32_t rank_in, rank_out; /* D1, D2: Tucker ranks                               */
    int32_t kernel;            /* K: core filter is K x K                            */
    int32_t stride, pad;       /* of the core convolution (stage 2)                  */
    int32_t layout;            /* tdc_layout of x and y                              */
    int32_t math;              /* tdc_math                                           */
} tdc_conv_desc;

typedef struct tdc_conv_plan_s *tdc_conv_plan_t;

/* Read-only description of what a plan will launch (for benches and tests). */
typedef struct {
    int32_t h_out, w_out;          /* H', W'                                          */
    int32_t variant;               /* 1 = fused fp32 SIMT, 2 = fused tcgen05          */
    char variant_name[48];
    int32_t launches_per_forward;  /* kernels tdc_conv_forward enqueues                */
    int32_t concurrent_forward;    /* 1 if forwards on distinct streams may overlap    */
    int32_t tile_h, tile_w;        /* output pixels per CTA tile                       */
    int32_t threads_per_cta;
    int32_t smem_bytes_per_cta;
    int64_t ctas_per_image;        /* CTAs launched per image by the main kernel       */
    int64_t workspace_bytes;       /* device bytes owned by the plan beyond weights    */
    int64_t weight_bytes;          /* packed device weight bytes                       */
    /* TDC_MATH_3XBF16 tile choices (0 elsewhere): N tile of stage 1 / the core / stage 3,
     * cluster split-K sizes, 1 if stage 3 is fused into the core kernel */
    int32_t bn_stage1, bn_core, bn_stage3;
    int32_t ksplit_stage1, ksplit_core, ksplit_stage3;
    int32_t core3;
    /* split-K through L2 (1 = off): K pieces of stage 1 / the core / stage 3 */
    int32_t gsplit_stage1, gsplit_core, gsplit_stage3;
} tdc_plan_info;

/* Planner overrides for TDC_MATH_3XBF16 (the analytical planner
 * vs exhaustive measured autotune).  -1 / 0 = the planner's own choice.  Requested N
 * tiles (32/64/128/256) are narrowed if they do not fit shared memory / TMEM; a
 * requested fusion that does not fit falls back to the unfused kernels; split-K
 * sizes are clamped to [1, 4] and to the number of K chunks.  The chosen values are
 * reported by tdc_conv_plan_query. */
typedef struct {
    int32_t core3;                         /* -1 auto, 0 never, 1 when it fits      */
    int32_t bn_stage1, bn_core, bn_stage3; /* 0 auto                               */
    int32_t ksplit_stage1, ksplit_core, ksplit_stage3; /* 0 auto, 1 off, 2..4     */
    int32_t gsplit_stage1, gsplit_core, gsplit_stage3; /* split-K through L2:
                                              0 auto, 1 off, 2..8 pieces (clamped to K chunks).
                                              The piece-0 CTA of a tile spins until the other
                                              pieces publish: the grid is capped at one CTA per
                                              SM and REQUIRES every CTA to be co-resident, so do
                                              not combine with MPS SM limits, green contexts or
                                              a concurrent persistent kernel on the same GPU.
                                              The model path enables it for long-K classifier
                                              GEMMs; set TDC_DENSE_NO_GSPLIT=1 to disable it there. */
    int32_t fused_layer;                   /* TDC_MATH_3XBF16: the single-launch layer kernel
                                              (stage 1 + core + stage 3, X' and Z on chip):
                                              -1 auto (when it fits and no other field asks
                                              for the three-launch kernels), 0 never, 1 when
                                              it fits                                      */
} tdc_plan_hints;

const char *tdc_version(void);
const char *tdc_status_string(tdc_status s);
/* Thread-local one-line message for the last failing call on this thread. */
const char *tdc_last_error(void);

/* H' and W' for a descriptor; validates it first. */
tdc_status tdc_conv_output_shape(const tdc_conv_desc *desc, int32_t *h_out, int32_t *w_out);

/* Plan a layer on CUDA device `device` (§8(a) row a0).  core (D2 x D1 x K x K),
 * u_in (C x D1), u_out (N x D2) and bias (N, or NULL) are HOST fp32 arrays,
 * row-major; they are copied and re-laid out (the CRSN idea, P:L338-340:
 * "format conversion can be completely done offline once") so the caller may
 * free them on return.  No kernel runs.  Returns UNSUPPORTED if the device is
 * not compute capability 10.0 or the math mode is not built. */
tdc_status tdc_conv_plan(const tdc_conv_desc *desc, const float *core,
                         const float *u_in, const float *u_out,
                         const float *bias, int32_t device, tdc_conv_plan_t *out);

tdc_status tdc_conv_plan_query(tdc_conv_plan_t plan, tdc_plan_info *info);

/* tdc_conv_plan with planner overrides (hints may be NULL = tdc_conv_plan). */
tdc_status tdc_conv_plan_ex(const tdc_conv_desc *desc, const float *core,
                            const float *u_in, const float *u_out, const float *bias,
                            const tdc_plan_hints *hints, int32_t device,
                            tdc_conv_plan_t *out);

/* Forward (§8(a) rows a1-a4), asynchronous on `stream` (a cudaStream_t; NULL =
 * legacy default stream).  x: DEVICE fp32, batch x C x H x W in desc.layout;
 * y: DEVICE fp32, batch x N x H' x W' in the same layout, fully overwritten.
 * 1 <= batch <= desc.batch; x and y must not alias.  The caller owns x, y and
 * the stream. */
tdc_status tdc_conv_forward(tdc_conv_plan_t plan, const float *x, float *y,
                            int32_t batch, void *stream);

/* End-to-end forward with HOST buffers: copies x to the device, runs
 * tdc_conv_forward on plan-owned device buffers, copies y back and waits for
 * the stream.  Host buffers should be pinned for asynchronous copies. */
tdc_status tdc_conv_forward_host(tdc_conv_plan_t plan, const float *x_host,
                                 float *y_host, int32_t batch, void *stream);

/* n end-to-end forwards with HOST buffers in one call (plans on one device; a plan may
 * appear more than once only if its forwards need not overlap -- they share its staging
 * buffers, so list distinct plans).  Equivalent to n tdc_conv_forward_host calls, but the
 * image chunks of all n forwards form one pipeline: the host->device copy of the next
 * forward and the device->host copy of the previous one overlap the current forward.
 * Waits for completion.  Errors as tdc_conv_forward_host, for the first failing plan. */
tdc_status tdc_conv_forward_host_many(const tdc_conv_plan_t *plans, const float *const *x_hosts,
                                      float *const *y_hosts, const int32_t *batches, int32_t n,
                                      void *stream);

tdc_status tdc_conv_plan_destroy(tdc_conv_plan_t plan);

/* Forward with the model-path epilogue fused into the last stage (SURVEY §8(f)
 * NEXT-1: "BN folded into U_out and bias; ReLU and residual fused into stage-3
 * epilogues"): y = act(layer(x) + bias + residual), act = ReLU if relu != 0.
 * residual: DEVICE fp32 with y's shape and layout, or NULL; it may not alias y.
 * Only NHWC plans in TDC_MATH_3XBF16 support residual/relu (UNSUPPORTED
 * otherwise); with residual == NULL and relu == 0 this is tdc_conv_forward. */
tdc_status tdc_conv_forward_ex(tdc_conv_plan_t plan, const float *x, float *y,
                               int32_t batch, const float *residual, int32_t relu,
                               void *stream);

/* ------------------------------------------------------------------ models
 * Whole-network inference (Tucker ResNet / VGG) as an
 * ordered list of ops over NHWC fp32 activations.  Activation ids: 0 is the
 * model input (batch x H x W x C), op i (0-based) writes id i + 1; the output of
 * the last op is the model output.  Every op computes in 3xBF16 (fp32-grade
 * tensor-core products, tolerance 1e-4 per layer) or FP32 where noted.
 *   TDC_OP_CONV    dense K x K conv (stride, pad) of src; w = [c_out][c_in][K][K]
 *                  (im2col + tcgen05 GEMM; 1 x 1 stride 1 is a plain GEMM)
 *   TDC_OP_TKD     Tucker-2 conv (the TKD layer): w = core [D2][D1][K][K],
 *                  u_in [c_in][D1], u_out [c_out][D2]
 *   TDC_OP_MAXPOOL K x K max pool (stride, pad; padding never wins), fp32
 *   TDC_OP_AVGPOOL global average pool -> batch x 1 x 1 x c_in, fp32
 *   TDC_OP_FC      fully connected on a batch x 1 x 1 x c_in input; w = [c_out][c_in]
 * Conv/TKD/FC outputs: y = act(BN(conv(src)) + bias + res), BN folded at create
 * time from bn = [4][c_out] (gamma, beta, mean, var; eps 1e-5) or none (NULL);
 * res = activation id added before the activation (same shape as the output)
 * or -1; act = ReLU if relu. */
typedef enum {
    TDC_OP_CONV = 0,
    TDC_OP_TKD = 1,
    TDC_OP_MAXPOOL = 2,
    TDC_OP_AVGPOOL = 3,
    TDC_OP_FC = 4
} tdc_op_kind;

typedef struct {
    int32_t kind;
    int32_t src, res;                    /* activation ids (res = -1: none) */
    int32_t c_in, c_out, height, width;  /* input geometry of one image */
    int32_t kernel, stride, pad;
    int32_t rank_in, rank_out;           /* TDC_OP_TKD: D1, D2 */
    int32_t relu;
    const float *w, *u_in, *u_out;       /* HOST, see above */
    const float *bias;                   /* HOST [c_out] or NULL */
    const float *bn;                     /* HOST [4][c_out] or NULL */
} tdc_model_op;

typedef struct tdc_model_s *tdc_model_t;

/* Build a model on `device` for batches up to max_batch: validates the op graph
 * (geometry of every src/res id), folds BN, plans every layer and allocates every
 * activation buffer (device memory owned by the model).  Host arrays are copied. */
tdc_status tdc_model_create(const tdc_model_op *ops, int32_t n_ops, int32_t max_batch,
                            int32_t device, tdc_model_t *out);

/* x: DEVICE fp32 NHWC batch x H x W x C (the first op's input geometry);
 * out: DEVICE fp32, batch x (last op's output) NHWC, fully overwritten.
 * Asynchronous on `stream`; 1 <= batch <= max_batch. */
tdc_status tdc_model_forward(tdc_model_t model, const float *x, int32_t batch, float *out,
                             void *stream);

/* Output geometry of op `op` (or of the model if op < 0): per-image H, W, C. */
tdc_status tdc_model_output_shape(tdc_model_t model, int32_t op, int32_t *h, int32_t *w,
                                  int32_t *c);

tdc_status tdc_model_destroy(tdc_model_t model);

#ifdef __cplusplus
}
#endif
#endif /* TDC_H */
