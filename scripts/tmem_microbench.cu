// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM on sm_100a, with 1, 2,
// 4 and 8 warps reading (each warp its own lane quarter), shapes 32x32b.x16 / .x32.
// Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

template <int X32>
__global__ void bench(int iters, int nwarps, long long *out, float *sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    float acc = 0.f;
    long long t0 = clock64();
    if (warp < nwarps) {
        const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
        for (int it = 0; it < iters; ++it) {
            if (X32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(base + (it & 3) * 32, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
            } else {
                uint32_t r[16];
                tmem_ld_32x32b_x16(base + (it & 7) * 16, r);
                tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) acc += __uint_as_float(r[j]);
            }
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    long long *d, h[148];
    float *sink;
    cudaMalloc(&d, sizeof(long long) * 148);
    cudaMalloc(&sink, sizeof(float) * 148 * 256);
    const int iters = 4096;
    for (int x32 = 0; x32 < 2; ++x32)
        for (int nw : {1, 2, 4, 8}) {
            if (x32) bench<1><<<148, 256>>>(iters, nw, d, sink);
            else bench<0><<<148, 256>>>(iters, nw, d, sink);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
            const double bytes = (double)nw * iters * 32 * (x32 ? 32 : 16) * 4;
            printf("x%d, %d warps: %.1f B/cycle/SM (%lld cycles) %s\n", x32 ? 32 : 16, nw, bytes / mx, mx,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
