// Microbenchmark: device time per kernel of a chain of N dependent tiny kernels captured in a
// CUDA graph, with and without programmatic dependent launch (PDL), 1 and 148 CTAs.
// Debug tool, not product.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 graph_floor.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int *p, int pdl) {
    if (pdl) asm volatile("griddepcontrol.launch_dependents;");
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += 1;
}

int main() {
    int *d;
    cudaMalloc(&d, 4);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int pdl = 0; pdl < 2; ++pdl)
        for (int grid : {1, 148}) {
            for (int threads : {128, 640}) {
                cudaGraph_t g;
                cudaGraphExec_t ge;
                const int n = 200;
                cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
                for (int i = 0; i < n; ++i) {
                    cudaLaunchConfig_t cfg = {};
                    cfg.gridDim = dim3(grid);
                    cfg.blockDim = dim3(threads);
                    cfg.stream = s;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                    at[0].val.programmaticStreamSerializationAllowed = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = pdl ? 1 : 0;
                    cudaLaunchKernelEx(&cfg, k_empty, d, pdl);
                }
                cudaStreamEndCapture(s, &g);
                cudaGraphInstantiate(&ge, g, 0);
                cudaGraphLaunch(ge, s);
                cudaStreamSynchronize(s);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0, s);
                for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
                cudaEventRecord(e1, s);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("pdl=%d grid=%3d threads=%3d: %.3f us per kernel\n", pdl, grid, threads, ms * 1e3 / (5 * n));
                cudaGraphExecDestroy(ge);
                cudaGraphDestroy(g);
            }
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
