/*
 * tdc_oracle.h -- fp64 CPU oracle for the Tucker-format (TKD) convolution layer.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path may include, link or
 * call this.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs use it.  It shares no code, header, table or helper with
 * the CUDA path (paper_2211_03715_b200/csrc) and never reads its outputs.
 *
 * Notation: B batch, C input channels, N output channels,
 * D1/D2 Tucker ranks, K core filter size (R = S = K), s stride, p pad.
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn.
 *
 * All arrays are row-major fp64.  Every function returns 0 on success and a
 * negative value on an invalid argument (null pointer, non-positive size,
 * output size < 1).  Loops accumulate in one fixed ascending order with plain
 * multiply-then-add (built with -ffp-contract=off), so results are
 * bit-identical for any OpenMP thread count.
 *
 * Parity status per function:
 *   tdc_oracle_conv7         pinned (closed forms S:L136/S:L163, torch fp64 conv2d,
 *                             scatter brute force, impulse convention)
 *   tdc_oracle_tkd_stages    pinned (≡ reconstructed-kernel conv, identity factors,
 *                             numpy matmul for the 1x1 stages, integer exactness)
 *   tdc_oracle_reconstruct   pinned (hand-enumerated 2x2x1x1 case, zero core,
 *                             einsum-free brute force)
 *   tdc_oracle_tkd_point     pinned (bit-identical to tdc_oracle_tkd_stages)
 */
#ifndef TDC_ORACLE_H
#define TDC_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* H' = floor((H + 2p - K)/s) + 1  (standard conv output size). */
int tdc_oracle_out_dim(int h, int k, int stride, int pad);

/* Seven-loop direct cross-correlation (P:L322-325 per-thread work equation,
 * read as cross-correlation per DESIGN.md reading R4):
 *   y[b,n,i,j] = sum_c sum_r sum_t x[b,c,i*s-p+r, j*s-p+t] * w[n,c,r,t]
 * with out-of-range input positions contributing zero (zero padding).
 * x: B x C x H x W, w: N x C x R x S, y: B x N x H' x W'. */
int tdc_oracle_conv7(const double *x, int B, int C, int H, int W,
                     const double *w, int N, int R, int S,
                     int stride, int pad, double *y);

/* Eq. tkd2 (referenced at P:L693, "recover back to the projected tensor"):
 *   w_rec[n,c,r,t] = sum_a sum_q u_out[n,q] * core[q,a,r,t] * u_in[c,a]
 * core: D2 x D1 x K x K, u_in: C x D1, u_out: N x D2, w_rec: N x C x K x K. */
int tdc_oracle_reconstruct(const double *core, const double *u_in,
                           const double *u_out, int C, int N, int D1, int D2,
                           int K, double *w_rec);

/* Three-stage TKD layer (BASELINE.json north_star), each stage a conv7:
 *   stage 1: x1 = conv7(x,  w1, 1, 0),  w1[a,c,0,0] = u_in[c,a]      (C -> D1)
 *   stage 2: z  = conv7(x1, core, s, p)                               (D1 -> D2)
 *   stage 3: y  = conv7(z,  w3, 1, 0) (+ bias[n]), w3[n,q,0,0] = u_out[n,q]
 * x1 (B x D1 x H x W) and z (B x D2 x H' x W') may be NULL; bias may be NULL. */
int tdc_oracle_tkd_stages(const double *x, int B, int C, int H, int W,
                          const double *core, int D1, int D2, int K,
                          const double *u_in, const double *u_out, int N,
                          const double *bias, int stride, int pad,
                          double *x1, double *z, double *y);

/* One output element y[b,n,i,j] of the three-stage layer, evaluated over its
 * receptive field only, with the same per-stage summation order as
 * tdc_oracle_tkd_stages (so the two agree bit for bit).  Used for sampled
 * parity at full benchmark sizes. */
int tdc_oracle_tkd_point(const double *x, int B, int C, int H, int W,
                         const double *core, int D1, int D2, int K,
                         const double *u_in, const double *u_out, int N,
                         const double *bias, int stride, int pad,
                         int b, int n, int i, int j, double *out);

/* OpenMP thread control (0 = leave the runtime default). */
void tdc_oracle_set_threads(int n);
int tdc_oracle_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
