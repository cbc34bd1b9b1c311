// tkd_common.cuh -- device helpers shared by the tcgen05 kernels of the
// 3-launch path (tkd_tc.cu: TF32 / 3xTF32; tkd_bf16.cu: 3xBF16).
#pragma once
#include <cuda_bf16.h>
#include <stdint.h>

#include "internal.h"

namespace tdc {

__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ bool remap_row(const TcGemmArgs &g, int m, long long *dst) {
    if (m >= g.M) return false;
    if (g.remap == 0) {
        *dst = m;
        return true;
    }
    if (g.remap == 1) {  // compact input pixel -> phase grid row
        const int x = m % g.W;
        const int t = m / g.W;
        const int y = t % g.H;
        const int b = t / g.H;
        const int uy = y + g.p, ux = x + g.p;
        const int ph = (uy % g.s) * g.s + (ux % g.s);
        *dst = (long long)ph * g.phase_rows + ((long long)b * g.Hq + uy / g.s) * g.Wq + ux / g.s;
        return true;
    }
    // remap == 2: output grid row -> compact output pixel (skip junk rows)
    const int ox = m % g.Wq;
    const int t = m / g.Wq;
    const int oy = t % g.Hq;
    const int b = t / g.Hq;
    if (oy >= g.Ho || ox >= g.Wo) return false;
    *dst = ((long long)b * g.Ho + oy) * g.Wo + ox;
    return true;
}


// bf16 split of 8 values: x = hi + lo with hi = RN_bf16(x), lo = RN_bf16(x - hi)
// (|x - hi - lo| <= 2^-17 |x|); packed two per 32-bit word, element 2i low.
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 t = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t *>(&t);
}
__device__ __forceinline__ void split_bf16x8(const float *v, uint4 &hi, uint4 &lo) {
    // hi packed first (one cvt.rn.bf16x2 per pair), then unpacked by bit moves (bf16 -> fp32 is
    // exact): 24 instructions per 8 values instead of 32 (the epilogues are issue-bound)
    uint32_t h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        h[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
        const float h0 = __uint_as_float(h[j] << 16), h1 = __uint_as_float(h[j] & 0xffff0000u);
        l[j] = pack_bf16x2(v[2 * j] - h0, v[2 * j + 1] - h1);
    }
    hi = make_uint4(h[0], h[1], h[2], h[3]);
    lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Model-path epilogue (tdc_model_*): y = v + bias[n] + residual[row][n], then ReLU.
// `res_row` points at the residual row (same layout as the output) or is null; the
// tail beyond nn is left untouched.
template <int W>
__device__ __forceinline__ void epi_bias_res_relu(float *v, int n, int nn, const float *bias, const float *res_row,
                                                  int relu) {
    if (bias) {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (n + j < nn) v[j] += __ldg(&bias[n + j]);
    }
    if (res_row) {
#pragma unroll
        for (int j = 0; j < W; ++j)
            if (n + j < nn) v[j] += __ldg(&res_row[n + j]);
    }
    if (relu) {
#pragma unroll
        for (int j = 0; j < W; ++j) v[j] = fmaxf(v[j], 0.f);
    }
}

}  // namespace tdc
