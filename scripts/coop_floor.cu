// Microbenchmark: device time of an empty cooperative kernel with 0 or 2 grid barriers
// (atomic count + generation), in a CUDA graph and with plain launches.  Debug tool.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned bar[2];
__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ void gsync(unsigned &gen, int mode) {
    __syncthreads();
    if (threadIdx.x == 0) {
        if (mode == 0) {
            __threadfence();
            if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) { bar[0] = 0; __threadfence(); atomicAdd(&bar[1], 1u); }
            else while (ld_acq(&bar[1]) == gen) __nanosleep(20);
            __threadfence();
        } else {
            unsigned old;
            asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&bar[0]) : "memory");
            if (old == gridDim.x - 1) {
                asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" :: "l"(&bar[0]) : "memory");
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(&bar[1]) : "memory");
            } else {
                while (ld_acq(&bar[1]) == gen) { if (mode == 2) __nanosleep(20); }
            }
        }
        ++gen;
    }
    __syncthreads();
}
__global__ void k(int nsync, int mode) {
    unsigned gen = 0;
    if (threadIdx.x == 0) gen = ld_acq(&bar[1]);
    for (int i = 0; i < nsync; ++i) gsync(gen, mode);
}
int main() {
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int coop = 0; coop < 2; ++coop)
        for (int grid : {16, 148})
            for (int ns : {0, 2, 12, 22}) for (int mode : {0, 1, 2}) {
                if (!coop && ns) continue;
                if (!ns && mode) continue;
                auto launch = [&]() {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(256); cfg.stream = s;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
                    cfg.attrs = at; cfg.numAttrs = coop;
                    return cudaLaunchKernelEx(&cfg, k, ns, mode);
                };
                for (int g = 0; g < 2; ++g) {
                    const int n = 100;
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0); cudaEventCreate(&e1);
                    cudaGraphExec_t ge = nullptr;
                    if (g) {
                        cudaGraph_t gr;
                        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                        for (int i = 0; i < n; ++i) launch();
                        cudaStreamEndCapture(s, &gr);
                        if (cudaGraphInstantiate(&ge, gr, 0) != cudaSuccess) { printf("instantiate failed\n"); continue; }
                        cudaGraphLaunch(ge, s);
                    } else {
                        for (int i = 0; i < 10; ++i) launch();
                    }
                    cudaStreamSynchronize(s);
                    cudaEventRecord(e0, s);
                    if (g) for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
                    else for (int i = 0; i < 5 * n; ++i) launch();
                    cudaEventRecord(e1, s);
                    cudaEventSynchronize(e1);
                    float ms; cudaEventElapsedTime(&ms, e0, e1);
                    printf("mode=%d coop=%d grid=%3d syncs=%d %s: %.2f us per kernel (%s)\n", mode, coop, grid, ns, g ? "graph" : "plain", ms * 1e3 / (5 * n), cudaGetErrorString(cudaGetLastError()));
                }
            }
    return 0;
}
