// Microbenchmark v4: is the ~45-cycle floor of small-N tcgen05.mma (cta_group::1) a
// per-accumulator dependency (read-modify-write of the same TMEM D) or an issue floor?
// Back-to-back MMAs rotate over NACC distinct accumulators (column blocks of N).
// SS: A and B from shared memory (128B swizzle); TS: A from TMEM.  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

template <int M, int N, int TS, int NACC>
__global__ void bench(int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<float *>(smem)[i] = 0.001f * (i % 7);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint64_t ad = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_kmajor_sw128(smem_u32(smem + 32768));
        const uint32_t id = idesc_bf16(M, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t d = tmem + (k % NACC) * N;
                if (TS) mma_bf16_ts(d, tmem + 384 + (k & 3) * 8, bd + (k & 3) * 2, id, 1);
                else mma_bf16(d, ad + (k & 3) * 2, bd + (k & 3) * 2, id, 1);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int M, int N, int TS, int NACC>
void run(int grid, long long *d) {
    const int iters = 8192;
    auto k = bench<M, N, TS, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    k<<<grid, 128, 66 * 1024>>>(iters, d);
    k<<<grid, 128, 66 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(long long) * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cyc = mx / iters;
    printf("bf16 M=%3d N=%3d %s NACC=%d  %7.1f cyc/mma  floor %5.1f  %s\n", M, N, TS ? "TS" : "SS", NACC,
           cyc, (M < 128 ? 128 : M) * N / 256.0, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *d;
    cudaMalloc(&d, sizeof(long long) * 148);
    const int g = 148;
    run<128, 32, 0, 1>(g, d); run<128, 32, 0, 2>(g, d); run<128, 32, 0, 4>(g, d); run<128, 32, 0, 8>(g, d);
    run<128, 32, 1, 1>(g, d); run<128, 32, 1, 2>(g, d); run<128, 32, 1, 4>(g, d); run<128, 32, 1, 8>(g, d);
    run<128, 64, 0, 1>(g, d); run<128, 64, 0, 2>(g, d); run<128, 64, 0, 4>(g, d);
    run<128, 64, 1, 1>(g, d); run<128, 64, 1, 2>(g, d); run<128, 64, 1, 4>(g, d);
    run<128, 96, 0, 1>(g, d); run<128, 96, 0, 2>(g, d);
    run<128, 96, 1, 1>(g, d); run<128, 96, 1, 2>(g, d);
    run<128, 128, 0, 1>(g, d); run<128, 128, 0, 2>(g, d);
    run<128, 128, 1, 1>(g, d); run<128, 128, 1, 2>(g, d);
    run<128, 256, 0, 1>(g, d); run<128, 256, 1, 1>(g, d);
    run<64, 64, 0, 1>(g, d); run<64, 64, 0, 4>(g, d); run<64, 128, 0, 2>(g, d); run<64, 256, 0, 1>(g, d);
    run<64, 256, 1, 1>(g, d);
    return 0;
}
