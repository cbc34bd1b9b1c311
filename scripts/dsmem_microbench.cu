// Microbenchmark: DSMEM (ld.shared::cluster) load latency and throughput in a cluster of
// 2 CTAs, vs local ld.shared.  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

template <int REMOTE, int ILP>
__global__ void __cluster_dims__(2, 1, 1) bench(int iters, long long *out, float *sink) {
    __shared__ __align__(16) float buf[64 * 128];
    for (int i = threadIdx.x; i < 64 * 128; i += blockDim.x) buf[i] = i;
    cluster_sync();
    const uint32_t peer = cluster_ctarank() ^ 1;
    const uint32_t base = REMOTE ? mapa_shared(smem_u32(buf), peer) : smem_u32(buf);
    float acc = 0.f;
    uint32_t off = threadIdx.x * 16;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        float4 v[ILP];
#pragma unroll
        for (int k = 0; k < ILP; ++k) {
            const uint32_t a = base + ((off + k * 2048u) & 0x7FF0u);
            if (REMOTE)
                v[k] = ld_dsmem_v4(a);
            else
                v[k] = ld_shared_v4(a);
        }
#pragma unroll
        for (int k = 0; k < ILP; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
        off = (off + 4096u + (uint32_t)(acc == 12345.f)) & 0x7FF0u;  // dependent address chain
    }
    long long t1 = clock64();
    cluster_sync();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 1.f) sink[threadIdx.x] = acc;
}

template <int R, int ILP>
void run(long long *d, float *sink, int threads) {
    const int iters = 256, grid = 148;
    bench<R, ILP><<<grid, threads>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%s ILP %d threads %3d: %7.1f cyc/iter  %6.1f B/cyc/SM %s\n", R ? "DSMEM" : "local", ILP, threads,
           mx / iters, 16.0 * ILP * threads * iters / mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *d;
    float *sink;
    cudaMalloc(&d, 8 * 256);
    cudaMalloc(&sink, 4 * 1024);
    for (int t : {32, 128}) {
        run<0, 1>(d, sink, t); run<0, 8>(d, sink, t);
        run<1, 1>(d, sink, t); run<1, 4>(d, sink, t); run<1, 8>(d, sink, t);
    }
    return 0;
}
