/*
 * tdc_oracle.c -- plain, slow, obviously correct fp64 CPU oracle for the
 * Tucker-format (TKD) convolution layer.  See tdc_oracle.h for the contract.
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs.  Shares no code with the
 * CUDA path.  Build: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC.
 *
 * Every loop nest below is the textbook definition written out, in ascending
 * index order, with no blocking, fusion or reordering.  OpenMP only splits
 * independent output planes (b, n), so every output element is computed by
 * exactly one thread in exactly the same order whatever the thread count.
 */
#include "tdc_oracle.h"

#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int tdc_oracle_out_dim(int h, int k, int stride, int pad) {
    if (h < 1 || k < 1 || stride < 1 || pad < 0) return -1;
    if (h + 2 * pad - k < 0) return -1;
    return (h + 2 * pad - k) / stride + 1;
}

/* Y(n,th,tw) = sum_c sum_r sum_s I(c, .., ..) * K(n,c,r,s).
 * Index convention: cross-correlation, input row i*s - p + r (R4). */
int tdc_oracle_conv7(const double *x, int B, int C, int H, int W,
                     const double *w, int N, int R, int S,
                     int stride, int pad, double *y) {
    if (!x || !w || !y) return -1;
    if (B < 1 || C < 1 || H < 1 || W < 1 || N < 1 || R < 1 || S < 1) return -1;
    const int Ho = tdc_oracle_out_dim(H, R, stride, pad);
    const int Wo = tdc_oracle_out_dim(W, S, stride, pad);
    if (Ho < 1 || Wo < 1) return -1;
    long planes = (long)B * N;
#pragma omp parallel for schedule(static)
    for (long bn = 0; bn < planes; ++bn) {
        const int b = (int)(bn / N);
        const int n = (int)(bn % N);
        for (int i = 0; i < Ho; ++i) {
            for (int j = 0; j < Wo; ++j) {
                double acc = 0.0;
                for (int c = 0; c < C; ++c) {
                    for (int r = 0; r < R; ++r) {
                        const int hi = i * stride - pad + r;
                        if (hi < 0 || hi >= H) continue;
                        for (int t = 0; t < S; ++t) {
                            const int wi = j * stride - pad + t;
                            if (wi < 0 || wi >= W) continue;
                            const double xv = x[(((long)b * C + c) * H + hi) * W + wi];
                            const double wv = w[(((long)n * C + c) * R + r) * S + t];
                            acc = acc + xv * wv;
                        }
                    }
                }
                y[(((long)b * N + n) * Ho + i) * Wo + j] = acc;
            }
        }
    }
    return 0;
}

/* Eq. tkd2: K_hat[c,n,r,t] = sum_{a,q} core[q,a,r,t] U1[c,a] U2[n,q];
 * stored here out-channel first (N x C x K x K) for use with conv7. */
int tdc_oracle_reconstruct(const double *core, const double *u_in,
                           const double *u_out, int C, int N, int D1, int D2,
                           int K, double *w_rec) {
    if (!core || !u_in || !u_out || !w_rec) return -1;
    if (C < 1 || N < 1 || D1 < 1 || D2 < 1 || K < 1) return -1;
    for (int n = 0; n < N; ++n)
        for (int c = 0; c < C; ++c)
            for (int r = 0; r < K; ++r)
                for (int t = 0; t < K; ++t) {
                    double acc = 0.0;
                    for (int a = 0; a < D1; ++a)
                        for (int q = 0; q < D2; ++q) {
                            const double g = core[(((long)q * D1 + a) * K + r) * K + t];
                            acc = acc + u_out[(long)n * D2 + q] * g * u_in[(long)c * D1 + a];
                        }
                    w_rec[(((long)n * C + c) * K + r) * K + t] = acc;
                }
    return 0;
}

/* North_star three-stage layer: 1x1 (C->D1), KxK core (D1->D2, stride, pad),
 * 1x1 (D2->N).  Stride and pad apply to the core only (R5, R6). */
int tdc_oracle_tkd_stages(const double *x, int B, int C, int H, int W,
                          const double *core, int D1, int D2, int K,
                          const double *u_in, const double *u_out, int N,
                          const double *bias, int stride, int pad,
                          double *x1, double *z, double *y) {
    if (!x || !core || !u_in || !u_out || !y) return -1;
    if (B < 1 || C < 1 || H < 1 || W < 1 || N < 1 || D1 < 1 || D2 < 1 || K < 1)
        return -1;
    const int Ho = tdc_oracle_out_dim(H, K, stride, pad);
    const int Wo = tdc_oracle_out_dim(W, K, stride, pad);
    if (Ho < 1 || Wo < 1) return -1;

    int rc = -2;
    double *w1 = (double *)malloc(sizeof(double) * (size_t)D1 * C);
    double *w3 = (double *)malloc(sizeof(double) * (size_t)N * D2);
    double *x1b = x1 ? x1 : (double *)malloc(sizeof(double) * (size_t)B * D1 * H * W);
    double *zb = z ? z : (double *)malloc(sizeof(double) * (size_t)B * D2 * Ho * Wo);
    if (!w1 || !w3 || !x1b || !zb) goto done;

    /* w1[a,c,0,0] = U_in[c,a]  (U1 in C x D1) */
    for (int a = 0; a < D1; ++a)
        for (int c = 0; c < C; ++c) w1[(long)a * C + c] = u_in[(long)c * D1 + a];
    /* w3[n,q,0,0] = U_out[n,q] (U2 in N x D2, P:L693 read as N x D2) */
    for (int n = 0; n < N; ++n)
        for (int q = 0; q < D2; ++q) w3[(long)n * D2 + q] = u_out[(long)n * D2 + q];

    if (tdc_oracle_conv7(x, B, C, H, W, w1, D1, 1, 1, 1, 0, x1b)) goto done;
    if (tdc_oracle_conv7(x1b, B, D1, H, W, core, D2, K, K, stride, pad, zb)) goto done;
    if (tdc_oracle_conv7(zb, B, D2, Ho, Wo, w3, N, 1, 1, 1, 0, y)) goto done;
    if (bias) {
        for (int b = 0; b < B; ++b)
            for (int n = 0; n < N; ++n)
                for (long e = 0; e < (long)Ho * Wo; ++e)
                    y[((long)b * N + n) * Ho * Wo + e] =
                        y[((long)b * N + n) * Ho * Wo + e] + bias[n];
    }
    rc = 0;
done:
    free(w1);
    free(w3);
    if (!x1) free(x1b);
    if (!z) free(zb);
    return rc;
}

int tdc_oracle_tkd_point(const double *x, int B, int C, int H, int W,
                         const double *core, int D1, int D2, int K,
                         const double *u_in, const double *u_out, int N,
                         const double *bias, int stride, int pad,
                         int b, int n, int i, int j, double *out) {
    if (!x || !core || !u_in || !u_out || !out) return -1;
    const int Ho = tdc_oracle_out_dim(H, K, stride, pad);
    const int Wo = tdc_oracle_out_dim(W, K, stride, pad);
    if (Ho < 1 || Wo < 1) return -1;
    if (b < 0 || b >= B || n < 0 || n >= N || i < 0 || i >= Ho || j < 0 || j >= Wo)
        return -1;
    double *zq = (double *)malloc(sizeof(double) * (size_t)D2);
    if (!zq) return -2;
    /* stage 2 for every q at (i, j); stage-1 values recomputed per tap with the
     * same c-ascending order conv7 uses for the 1x1 stage. */
    for (int q = 0; q < D2; ++q) {
        double acc = 0.0;
        for (int a = 0; a < D1; ++a) {
            for (int r = 0; r < K; ++r) {
                const int hi = i * stride - pad + r;
                if (hi < 0 || hi >= H) continue;
                for (int t = 0; t < K; ++t) {
                    const int wi = j * stride - pad + t;
                    if (wi < 0 || wi >= W) continue;
                    double x1v = 0.0;
                    for (int c = 0; c < C; ++c)
                        x1v = x1v + x[(((long)b * C + c) * H + hi) * W + wi] *
                                        u_in[(long)c * D1 + a];
                    acc = acc + x1v * core[(((long)q * D1 + a) * K + r) * K + t];
                }
            }
        }
        zq[q] = acc;
    }
    double y = 0.0;
    for (int q = 0; q < D2; ++q) y = y + zq[q] * u_out[(long)n * D2 + q];
    if (bias) y = y + bias[n];
    *out = y;
    free(zq);
    return 0;
}

void tdc_oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int tdc_oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
