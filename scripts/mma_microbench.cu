// Microbenchmark: cycles per tcgen05.mma.kind::tf32 (M=128, cta_group::1) as a
// function of N, operand layout (128B swizzle vs no swizzle), SS vs TS (A in
// TMEM) and the number of independent accumulators.  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

__global__ void bench(int mode, int N, int nacc, int iters, long long *out, int bf, int M) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
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
    if (warp == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t id = bf ? idesc_bf16(M, N) : idesc_tf32(M, N);
        uint64_t ad, bd;
        if (mode == 0 || mode == 2) {  // sw128 A / sw128 B  (mode 2: A from TMEM)
            ad = sdesc_kmajor_sw128(a);
            bd = sdesc_kmajor_sw128(b);
        } else if (mode == 1) {  // no swizzle both
            ad = sdesc_kmajor_none(a, 128 * 16, 128);
            bd = sdesc_kmajor_none(b, N * 16, 128);
        } else {  // sw128 A, no-swizzle B
            ad = sdesc_kmajor_sw128(a);
            bd = sdesc_kmajor_none(b, N * 16, 128);
        }
        __syncwarp();
        long long t0 = clock64();
        if (elect_one()) {
            for (int i = 0; i < iters; ++i) {
                const uint32_t acc = tmem + (i % nacc) * N;
                if (bf) {
                    if (mode == 2)
                        mma_bf16_ts(acc, tmem + 256 + (i & 3) * 8, bd, id, i >= nacc);
                    else
                        mma_bf16(acc, ad + ((i & 3) * 2), bd + ((i & 3) * 2), id, i >= nacc);
                } else if (mode == 2)
                    mma_tf32_ts(acc, tmem + 256 + (i & 3) * 8, bd, id, i >= nacc);
                else
                    mma_tf32(acc, ad + ((i & 3) * 2), bd + ((i & 3) * 2), id, i >= nacc);
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    long long *d;
    cudaMalloc(&d, 8 * 256);
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const char *names[] = {"SS sw128/sw128", "SS none/none", "TS  tmem/sw128", "SS sw128/none"};
    const int iters = 2048;
    for (int bf : {0, 1})
    for (int M : {64, 128})
    for (int grid : {148}) {
        for (int mode = 0; mode < 1; ++mode)
            for (int N : {32, 64, 128, 256})
                for (int nacc : {1, 2}) {
                    if (N * nacc > (mode == 2 ? 256 : 512)) continue;
                    bench<<<grid, 128, 100 * 1024>>>(mode, N, nacc, iters, d, bf, M);
                    cudaError_t e = cudaDeviceSynchronize();
                    long long h[256];
                    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
                    double mx = 0;
                    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
                    printf("M=%d %s grid %3d %-16s N=%3d nacc=%d  %7.1f cyc/mma  (%5.0f MAC/cyc/SM) %s\n", M, bf ? "bf16" : "tf32", grid,
                           names[mode], N, nacc, mx / iters, (double)M * N * (bf ? 16 : 8) * iters / mx,
                           e == cudaSuccess ? "" : cudaGetErrorString(e));
                }
    }
    return 0;
}
