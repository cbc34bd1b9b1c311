// Microbenchmark: per-SM throughput of 1-D bulk copies (cp.async.bulk) and 2-D tensor
// TMA loads from an L2-resident buffer into a shared-memory ring, vs copy size and
// ring depth.  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

__global__ void bench_bulk(const uint8_t *src, int bytes, int depth, int iters, long long *out, int src_span) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        uint32_t phase = 0;
        for (int i = 0; i < iters; ++i) {
            const int s = i % depth;
            if (i >= depth) {
                mbar_wait(&bar[s], phase);
                if (s == depth - 1) phase ^= 1;
            }
            mbar_arrive_expect_tx(&bar[s], bytes);
            const size_t off = ((size_t)(blockIdx.x * 7 + i) * bytes) & (size_t)(src_span - 1);
            bulk_load(smem + (size_t)s * bytes, src + off, bytes, &bar[s]);
        }
        // drain
        for (int i = iters; i < iters + depth; ++i) {
            const int s = i % depth;
            mbar_wait(&bar[s], phase);
            if (s == depth - 1) phase ^= 1;
        }
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
}

// nw issuing warps, each with its own ring of `depth` slots of `bytes`.
__global__ void bench_bulk_mw(const uint8_t *src, int bytes, int depth, int iters, long long *out, int src_span) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[4][16];
    const int w = threadIdx.x / 32, nw = blockDim.x / 32;
    if (threadIdx.x % 32 == 0) {
        for (int i = 0; i < depth; ++i) mbar_init(&bar[w][i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    long long t0 = clock64();
    if (threadIdx.x % 32 == 0) {
        uint8_t *ring = smem + (size_t)w * depth * bytes;
        uint32_t phase = 0;
        for (int i = 0; i < iters; ++i) {
            const int s = i % depth;
            if (i >= depth) {
                mbar_wait(&bar[w][s], phase);
                if (s == depth - 1) phase ^= 1;
            }
            mbar_arrive_expect_tx(&bar[w][s], bytes);
            const size_t off = ((size_t)(blockIdx.x * 7 + w * 3 + i) * bytes) & (size_t)(src_span - 1);
            bulk_load(ring + (size_t)s * bytes, src + off, bytes, &bar[w][s]);
        }
        for (int i = iters; i < iters + depth; ++i) {
            const int s = i % depth;
            mbar_wait(&bar[w][s], phase);
            if (s == depth - 1) phase ^= 1;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

// 2-D tensor TMA: box {64 bf16, rows} (128B swizzle) from a [span/128][64] bf16 map.
__global__ void bench_tma2d(const __grid_constant__ CUtensorMap map, int rows, int depth, int iters, long long *out,
                            int total_rows) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[16];
    const int bytes = rows * 128;
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long t0 = clock64();
        uint32_t phase = 0;
        for (int i = 0; i < iters; ++i) {
            const int s = i % depth;
            if (i >= depth) {
                mbar_wait(&bar[s], phase);
                if (s == depth - 1) phase ^= 1;
            }
            mbar_arrive_expect_tx(&bar[s], bytes);
            const int r0 = (int)(((long long)(blockIdx.x * 7 + i) * rows) & (total_rows - 1)) & ~(rows - 1);
            tma_load_2d(smem + (size_t)s * bytes, &map, &bar[s], 0, r0);
        }
        for (int i = iters; i < iters + depth; ++i) {
            const int s = i % depth;
            mbar_wait(&bar[s], phase);
            if (s == depth - 1) phase ^= 1;
        }
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
}

// Batched: issue `depth` copies back-to-back (one mbarrier each), then wait for all;
// also records the cycles spent issuing vs waiting.
__global__ void bench_batch(const uint8_t *src, int bytes, int depth, int batches, long long *out, int src_span) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[16];
    if (threadIdx.x == 0) {
        for (int i = 0; i < depth; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long issue = 0, wait = 0;
        long long t0 = clock64();
        for (int b = 0; b < batches; ++b) {
            long long a = clock64();
            for (int s = 0; s < depth; ++s) {
                mbar_arrive_expect_tx(&bar[s], bytes);
                const size_t off = ((size_t)(blockIdx.x * 7 + b * depth + s) * bytes) & (size_t)(src_span - 1);
                bulk_load(smem + (size_t)s * bytes, src + off, bytes, &bar[s]);
            }
            long long c = clock64();
            for (int s = 0; s < depth; ++s) mbar_wait(&bar[s], b & 1);
            long long e = clock64();
            issue += c - a;
            wait += e - c;
        }
        long long t1 = clock64();
        out[blockIdx.x * 3] = t1 - t0;
        out[blockIdx.x * 3 + 1] = issue;
        out[blockIdx.x * 3 + 2] = wait;
    }
}

// Ring where each iteration's `depth`... no: lanes 0..nl-1 of one warp each issue one
// copy per round (own mbarrier), then every lane waits for all; rounds back to back.
__global__ void bench_lanes(const uint8_t *src, int bytes, int nl, int rounds, long long *out, int src_span) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar[32];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < nl) mbar_init(&bar[threadIdx.x], 1);
    if (threadIdx.x == 0) fence_mbar_init();
    __syncthreads();
    if (threadIdx.x < 32) {
        long long t0 = clock64();
        for (int b = 0; b < rounds; ++b) {
            if (lane < nl) {
                mbar_arrive_expect_tx(&bar[lane], bytes);
                const size_t off = ((size_t)(blockIdx.x * 7 + b * nl + lane) * bytes) & (size_t)(src_span - 1);
                bulk_load(smem + (size_t)lane * bytes, src + off, bytes, &bar[lane]);
            }
            __syncwarp();
            for (int s = 0; s < nl; ++s) mbar_wait(&bar[s], b & 1);
            __syncwarp();
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
}

int main() {
    const int span = 32 << 20;  // 32 MB source: L2 resident after the first pass
    uint8_t *src;
    cudaMalloc(&src, span + (1 << 20));
    cudaMemset(src, 1, span + (1 << 20));
    long long *d;
    cudaMalloc(&d, 8 * 1024);
    cudaFuncSetAttribute(bench_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int grid : {148})
        for (int bytes : {1024, 4096, 16384})
            for (int depth : {1, 2, 8}) {
                if ((long long)bytes * depth > 190 * 1024) continue;
                const int iters = 2048;
                for (int rep = 0; rep < 2; ++rep)
                    bench_bulk<<<grid, 32, 200 * 1024>>>(src, bytes, depth, iters, d, span);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[1024];
                cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
                double mx = 0;
                for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
                printf("bulk grid %3d  %5d B x depth %2d: %6.1f B/cyc/SM  (%6.0f cyc/copy) chip %5.0f B/cyc %s\n", grid,
                       bytes, depth, (double)bytes * iters / mx, mx / iters, (double)bytes * iters / mx * grid,
                       e == cudaSuccess ? "" : cudaGetErrorString(e));
            }
    cudaFuncSetAttribute(bench_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int bytes : {1024, 4096, 16384})
        for (int depth : {1, 4, 8, 12}) {
            if ((long long)bytes * depth > 190 * 1024) continue;
            const int batches = 256, grid = 148;
            for (int rep = 0; rep < 2; ++rep)
                bench_batch<<<grid, 32, 200 * 1024>>>(src, bytes, depth, batches, d, span);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[1024];
            cudaMemcpy(h, d, 8 * 3 * grid, cudaMemcpyDeviceToHost);
            printf("batch %5d B x %2d: %7.0f cyc/batch (issue %6.0f, wait %6.0f)  %6.1f B/cyc/SM %s\n", bytes, depth,
                   (double)h[0] / batches, (double)h[1] / batches, (double)h[2] / batches,
                   (double)bytes * depth * batches / h[0], e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    cudaFuncSetAttribute(bench_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int bytes : {2048, 4096, 8192})
        for (int nl : {1, 4, 8, 16}) {
            if ((long long)bytes * nl > 190 * 1024) continue;
            const int rounds = 256, grid = 148;
            for (int rep = 0; rep < 2; ++rep)
                bench_lanes<<<grid, 32, 200 * 1024>>>(src, bytes, nl, rounds, d, span);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[1024];
            cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("lanes %5d B x %2d lanes: %7.0f cyc/round  %6.1f B/cyc/SM %s\n", bytes, nl, mx / rounds,
                   (double)bytes * nl * rounds / mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    cudaFuncSetAttribute(bench_bulk_mw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int nw : {1, 2, 4})
        for (int bytes : {4096, 16384}) {
            const int depth = 4, iters = 1024, grid = 148;
            if ((long long)bytes * depth * nw > 190 * 1024) continue;
            for (int rep = 0; rep < 2; ++rep)
                bench_bulk_mw<<<grid, 32 * nw, 200 * 1024>>>(src, bytes, depth, iters, d, span);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[1024];
            cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("bulk %d warps  %5d B x depth %2d: %6.1f B/cyc/SM %s\n", nw, bytes, depth,
                   (double)bytes * iters * nw / mx, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    // tensor map over the buffer
    CUtensorMap map;
    const int total_rows = span / 128;
    cuuint64_t dims[2] = {64, (cuuint64_t)total_rows};
    cuuint64_t strides[1] = {128};
    cuuint32_t estr[2] = {1, 1};
    cudaFuncSetAttribute(bench_tma2d, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int rows : {32, 64, 128, 256})
        for (int depth : {2, 4, 8}) {
            if (rows * 128 * depth > 190 * 1024) continue;
            cuuint32_t box[2] = {64, (cuuint32_t)rows};
            CUresult r = cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
            const int iters = 1024, grid = 148;
            for (int rep = 0; rep < 2; ++rep)
                bench_tma2d<<<grid, 32, 200 * 1024>>>(map, rows, depth, iters, d, total_rows);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[1024];
            cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("tma2d box %3d x 128 B (%5d B) x depth %d: %6.1f B/cyc/SM  (%5.0f cyc/copy) %s\n", rows, rows * 128,
                   depth, (double)rows * 128 * iters / mx, mx / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
