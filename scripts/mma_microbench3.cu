// Microbenchmark v3: tcgen05.mma.cta_group::2 (CTA pair, M = 256) issue cost vs N,
// next to cta_group::1 M = 128, to decide whether pairing SMs pays for the
// small-N (rank 32-128) MMAs of the TKD layer.  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) bench2(int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<float *>(smem)[i] = 0.001f * (i % 7);
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = slot;
    long long t0 = clock64();
    if (warp == 0 && rank == 0 && threadIdx.x == 0) {
        const uint64_t ad = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_kmajor_sw128(smem_u32(smem + 32768));
        const uint32_t id = idesc_bf16(256, N);
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(ad + k * 2), "l"(bd + k * 2), "r"(id), "r"(1)
                    : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3)
            : "memory");
    }
    if (warp == 0) {
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int N>
void run(long long *d) {
    auto k = bench2<N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    const int iters = 4096, grid = 148;
    k<<<grid, 128, 66 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; i += 2) mx = h[i] > mx ? h[i] : mx;
    printf("bf16 cta_group::2 M=256 N=%3d  %7.1f cyc/mma (pair)  %6.0f MAC/cyc/SM  %s\n", N, mx / iters,
           256.0 * N * 16 * iters / mx / 2, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8 * 512);
    run<32>(d);
    run<64>(d);
    run<128>(d);
    run<256>(d);
    return 0;
}
