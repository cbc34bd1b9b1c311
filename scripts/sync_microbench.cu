// Microbenchmark: cost of the MMA thread's per-tile synchronisation primitives on
// sm_100a -- mbarrier try_wait on an already completed phase, tcgen05.commit to an
// mbarrier (no MMAs outstanding), tcgen05 fences, elect.sync -- alone and with 17
// other warps of the CTA sleeping in try_wait (the fused layer kernel's situation).
// Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

template <int MODE>
__global__ void bench(int iters, long long *out, int nwarps_sleep) {
    __shared__ uint64_t bars[8];
    __shared__ uint64_t park;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
        mbar_init(&park, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(&slot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 0) {
        // complete phase 0 of bars[0..3] so waits on parity 0 succeed at once
        if (threadIdx.x == 0)
            for (int i = 0; i < 4; ++i) mbar_arrive(&bars[i]);
        __syncwarp();
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if (MODE & 1) {  // 6 waits on completed phases
#pragma unroll
                for (int i = 0; i < 6; ++i) mbar_wait(&bars[i & 3], 0);
            }
            if (MODE & 2) {  // 6 commits (no MMAs outstanding) to barriers 4..7
                if (elect_one()) {
#pragma unroll
                    for (int i = 0; i < 6; ++i) mma_commit(&bars[4 + (i & 3)]);
                }
                __syncwarp();
            }
            if (MODE & 4) {  // fences + elect
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    tc_fence_after();
                    if (elect_one()) asm volatile("" ::: "memory");
                    __syncwarp();
                }
            }
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
        if (threadIdx.x == 0) mbar_arrive(&park);
    } else if (warp <= nwarps_sleep) {
        mbar_wait_sleep(&park, 0);  // sleep until warp 0 is done
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(slot, 32);
}

template <int MODE>
void run(int nsleep) {
    long long *d, h[148];
    cudaMalloc(&d, sizeof(long long) * 148);
    bench<MODE><<<148, 576>>>(2000, d, nsleep);
    bench<MODE><<<148, 576>>>(2000, d, nsleep);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(long long) * 148, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("mode %d (waits %d, commits %d, fences %d), %2d sleeping warps: %6lld cycles/iteration %s\n", MODE,
           MODE & 1, (MODE >> 1) & 1, (MODE >> 2) & 1, nsleep, mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int ns : {0, 17}) {
        run<1>(ns);
        run<2>(ns);
        run<4>(ns);
        run<7>(ns);
    }
    return 0;
}
