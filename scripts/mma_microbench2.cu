// Microbenchmark v2: issue throughput of back-to-back tcgen05.mma (cta_group::1)
// with everything compile-time (no runtime branches around the MMA, descriptors
// precomputed in uniform registers), to separate the tensor-pipe floor from
// issue-loop overheads.  Debug tool, not product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2211_03715_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "sm100.cuh"

using namespace tdc::sm100;

// TS: A from TMEM (cols 256..), SS: A from smem (sw128 K-major).
template <int BF, int M, int N, int TS, int ELECT, int COLS>
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
    if (warp == 0) tmem_alloc(&slot, COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (warp == 0) {
        const uint64_t ad = sdesc_kmajor_sw128(smem_u32(smem));
        const uint64_t bd = sdesc_kmajor_sw128(smem_u32(smem + 32768));
        const uint32_t id = BF ? idesc_bf16(M, N) : idesc_tf32(M, N);
        __syncwarp();
        long long t0 = clock64();
        if (ELECT) {
            for (int i = 0; i < iters; i += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (elect_one()) {
                        if (TS) {
                            if (BF) mma_bf16_ts(tmem, tmem + 256 + k * 8, bd + k * 2, id, 1);
                            else mma_tf32_ts(tmem, tmem + 256 + k * 8, bd + k * 2, id, 1);
                        } else {
                            if (BF) mma_bf16(tmem, ad + k * 2, bd + k * 2, id, 1);
                            else mma_tf32(tmem, ad + k * 2, bd + k * 2, id, 1);
                        }
                    }
                    __syncwarp();
                }
            }
            if (elect_one()) mma_commit(&bar);
        } else if (threadIdx.x == 0) {
            for (int i = 0; i < iters; i += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (TS) {
                        if (BF) mma_bf16_ts(tmem, tmem + 256 + k * 8, bd + k * 2, id, 1);
                        else mma_tf32_ts(tmem, tmem + 256 + k * 8, bd + k * 2, id, 1);
                    } else {
                        if (BF) mma_bf16(tmem, ad + k * 2, bd + k * 2, id, 1);
                        else mma_tf32(tmem, ad + k * 2, bd + k * 2, id, 1);
                    }
                }
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
    if (warp == 0) tmem_dealloc(tmem, COLS);
}

// Layout / commit study (bf16, M = 128, SS): LAYOUT 0 = 128B swizzle, 1 = no swizzle
// (core-matrix interleave as the core kernel: A LBO = band plane stride, B LBO = N*16);
// CE = commit to an mbarrier every CE MMAs (0 = only at the end).
template <int N, int LAYOUT, int CE>
__global__ void bench_lc(int iters, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, cbar[4];
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<float *>(smem)[i] = 0.001f * (i % 7);
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        for (int i = 0; i < 4; ++i) mbar_init(&cbar[i], 1);
        fence_mbar_init();
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        uint64_t ad, bd;
        if (LAYOUT == 0) {
            ad = sdesc_kmajor_sw128(smem_u32(smem));
            bd = sdesc_kmajor_sw128(smem_u32(smem + 32768));
        } else {
            ad = sdesc_kmajor_none(smem_u32(smem), 3968, 128);
            bd = sdesc_kmajor_none(smem_u32(smem + 32768), N * 16, 128);
        }
        const uint32_t id = idesc_bf16(128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 6) {
#pragma unroll
            for (int k = 0; k < 6; ++k) mma_bf16(tmem, ad + (k & 1) * 2, bd + (k % 3) * 2, id, 1);
            if (CE) mma_commit(&cbar[(i / 6) & 3]);
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

template <int N, int LAYOUT, int CE>
void run_lc(long long *d) {
    auto k = bench_lc<N, LAYOUT, CE>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    const int iters = 6 * 682, grid = 148;
    k<<<grid, 128, 66 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("bf16 M=128 N=%3d %s commit/%d: %7.1f cyc/mma %s\n", N, LAYOUT ? "no-swizzle" : "sw128     ", CE ? 6 : 0,
           mx / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

// A start-address offset study (bf16, M = 128, SS, no commits): LAYOUT 1 = no swizzle
// with A start shifted by OFF bytes (row shifts of 16 B as the core kernel's taps);
// LAYOUT 0 = 128B swizzle with A shifted by OFF bytes (multiples of 128 = whole rows)
// and the descriptor base-offset field set to (addr >> 7) & 7.
template <int N, int LAYOUT>
__global__ void bench_off(int iters, int off, long long *out) {
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
        uint64_t ad, bd;
        const uint32_t a_addr = smem_u32(smem) + off;
        if (LAYOUT == 0) {
            ad = sdesc_kmajor_sw128(a_addr) | ((uint64_t)((a_addr >> 7) & 7) << 49);
            bd = sdesc_kmajor_sw128(smem_u32(smem + 40960));
        } else {
            ad = sdesc_kmajor_none(a_addr, 3968, 128);
            bd = sdesc_kmajor_none(smem_u32(smem + 40960), N * 16, 128);
        }
        const uint32_t id = idesc_bf16(128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; i += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16(tmem, ad + (k & 1) * 2, bd + (k & 1) * 2, id, 1);
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

template <int N, int LAYOUT>
void run_off(long long *d, int off) {
    auto k = bench_off<N, LAYOUT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    const int iters = 4096, grid = 148;
    k<<<grid, 128, 66 * 1024>>>(iters, off, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("bf16 M=128 N=%3d %s A offset %4d B: %7.1f cyc/mma %s\n", N, LAYOUT ? "no-swizzle" : "sw128+base", off,
           mx / iters, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

// The core kernel's exact MMA pattern: A = X' band planes (no swizzle, LBO = band plane
// stride 3968 B), per-tap row-shifted start (tap_off = r*58 + t rows), hi/lo halves
// 63.5 KB apart; B = [hi|lo] weight rows (N = 64, LBO = 1 KB); 2 K16 steps x 2 MMAs per
// tap, 9 taps, commit per tile.  VAR 0: as the kernel; 1: no row shift; 2: A_hi only.
template <int VAR>
__global__ void bench_core(int tiles, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, cbar0;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) {
        if (VAR >= 6) {  // random bf16 pairs (hash of the index), magnitudes ~ N(0,1) like real data
            uint32_t h = (uint32_t)i * 2654435761u ^ (blockIdx.x * 40503u);
            h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
            const uint32_t lo = 0x3c00u | (h & 0x807fu) | ((h >> 7) & 0x0180u);
            const uint32_t hi = 0x3c00u | ((h >> 16) & 0x807fu) | ((h >> 23) & 0x0180u);
            reinterpret_cast<uint32_t *>(smem)[i] = lo | (hi << 16);
        } else {
            reinterpret_cast<float *>(smem)[i] = 0.001f * (i % 7);
        }
    }
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&cbar0, 1);
        fence_mbar_init();
        mbar_arrive(&cbar0);
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t band_bytes = 248 * 16, a_half = 4 * band_bytes;
        const uint64_t da = sdesc_kmajor_none(smem_u32(smem), band_bytes, 128);
        const uint64_t db = sdesc_kmajor_none(smem_u32(smem + 2 * 2 * a_half), 2 * 32 * 16, 128);
        const uint32_t id = idesc_bf16(128, 64);
        long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            uint32_t accum = 0;
            if (VAR == 4) {  // per tile: wait a completed barrier + tcgen05 fence (as the kernel)
                mbar_wait(&cbar0, 0);
                tc_fence_after();
            }
            for (int tap = 0; tap < 9; ++tap) {
                if (VAR == 3) tc_fence_after();
                const uint32_t off = VAR == 1 ? 0u : (uint32_t)((tap / 3) * 58 + tap % 3) * 16;
                const uint64_t a = da + (off >> 4);
                const uint64_t b = db + ((tap * 32 * 128) >> 4);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint64_t aj = a + ((j * 2 * band_bytes) >> 4);
                    const uint64_t bj = b + ((j * 2 * 2 * 32 * 16) >> 4);
                    mma_bf16(tmem + (t & 1) * 64, aj, bj, id, accum);
                    mma_bf16(tmem + (t & 1) * 64, VAR == 2 ? aj : aj + (a_half >> 4), bj, id, 1);
                    accum = 1;
                }
            }
            mma_commit(&bar);
            if (VAR == 5) mbar_wait(&bar, t & 1);  // serialize tiles: the pipe drains each tile
        }
        mbar_wait(&bar, (tiles - 1) & 1);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

// Same MMA stream with interference from 4 other warps: INT 1 = tcgen05.ld x32 loops on
// other TMEM columns; 2 = ld/st.shared.v4 streams; 3 = both; 4 = 1-D bulk copies
// (global -> smem, 16 KB) issued by one other warp.
template <int INT>
__global__ void bench_core_int(int tiles, long long *out, const uint8_t *gsrc, volatile int *stop) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar, cbar;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<float *>(smem)[i] = 0.001f * (i % 7);
    const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&cbar, 1);
        fence_mbar_init();
        done = 0;
    }
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc(&slot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t band_bytes = 248 * 16, a_half = 4 * band_bytes;
        const uint64_t da = sdesc_kmajor_none(smem_u32(smem), band_bytes, 128);
        const uint64_t db = sdesc_kmajor_none(smem_u32(smem + 2 * 2 * a_half), 2 * 32 * 16, 128);
        const uint32_t id = idesc_bf16(128, 64);
        long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            uint32_t accum = 0;
            for (int tap = 0; tap < 9; ++tap) {
                const uint32_t off = (uint32_t)((tap / 3) * 58 + tap % 3) * 16;
                const uint64_t a = da + (off >> 4);
                const uint64_t b = db + ((tap * 32 * 128) >> 4);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const uint64_t aj = a + ((j * 2 * band_bytes) >> 4);
                    const uint64_t bj = b + ((j * 2 * 2 * 32 * 16) >> 4);
                    mma_bf16(tmem + (t & 1) * 64, aj, bj, id, accum);
                    mma_bf16(tmem + (t & 1) * 64, aj + (a_half >> 4), bj, id, 1);
                    accum = 1;
                }
            }
            mma_commit(&bar);
        }
        mbar_wait(&bar, (tiles - 1) & 1);
        long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        done = 1;
        if (INT == 5) mbar_arrive(&cbar);
    } else if ((warp >= 4 && warp < 8) || (INT == 5 && warp != 0)) {
        const int q = warp & 3;
        float acc = 0.f;
        uint32_t it = 0;
        while (!done) {
            if (INT & 1) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem + ((uint32_t)(q * 32) << 16) + 256 + (it & 3) * 32, r);
                tmem_ld_wait();
                acc += __uint_as_float(r[lane & 31]);
            }
            if (INT & 2) {
                const uint32_t base = smem_u32(smem + 150 * 1024) + (uint32_t)((q * 32 + lane) * 16);
                float4 v = ld_shared_v4(base + (it & 7) * 2048);
                st_shared_v4(base + ((it + 3) & 7) * 2048, v.x + 1.f, v.y, v.z, v.w);
                acc += v.x;
            }
            if (INT == 5) {  // mbarrier try_wait spinning on a barrier that completes at the end
                mbar_wait(&cbar, 0);
                break;
            }
            if (INT == 4 && warp == 4 && lane == 0) {
                mbar_arrive_expect_tx(&cbar, 16384);
                bulk_load(smem + 160 * 1024, gsrc + (size_t)((blockIdx.x * 131 + it) & 1023) * 16384, 16384, &cbar);
                mbar_wait(&cbar, it & 1);
            }
            ++it;
        }
        if (acc == 12345.f) out[1000] = 1;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

template <int INT>
void run_core_int(long long *d, const uint8_t *g) {
    auto k = bench_core_int<INT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
    const int tiles = 64, grid = 148;
    k<<<grid, INT == 5 ? 320 : 256, 201 * 1024>>>(tiles, d, g, nullptr);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("core pattern + interference %d: %7.1f cyc/tile  %6.1f cyc/mma %s\\n", INT, mx / tiles, mx / tiles / 36,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int VAR>
void run_core(long long *d) {
    auto k = bench_core<VAR>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 201 * 1024);
    const int tiles = getenv("MB_TILES") ? atoi(getenv("MB_TILES")) : 64, grid = 148;
    k<<<grid, 128, 201 * 1024>>>(tiles, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("core pattern VAR %d: %7.1f cyc/tile  %6.1f cyc/mma %s\n", VAR, mx / tiles, mx / tiles / 36,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

template <int BF, int M, int N, int TS, int ELECT>
void run(long long *d, int ctas_per_sm) {
    auto k = ctas_per_sm == 1 ? bench<BF, M, N, TS, ELECT, 512> : bench<BF, M, N, TS, ELECT, 256>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
    const int iters = 4096, grid = 148 * ctas_per_sm;
    k<<<grid, 128, 66 * 1024>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[512];
    cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
    double mx = 0, sum = 0;
    for (int i = 0; i < grid; ++i) {
        mx = h[i] > mx ? h[i] : mx;
        sum += h[i];
    }
    const double kk = BF ? 16 : 8;
    printf("[%d CTA/SM] %s M=%3d N=%3d %s %s  %7.1f cyc/mma (max)  %7.1f (mean)  %6.0f MAC/cyc/SM  floor %5.1f %s\n",
           ctas_per_sm, BF ? "bf16" : "tf32", M, N, TS ? "TS" : "SS", ELECT ? "elect-warp" : "thread0   ",
           mx / iters, sum / grid / iters, M * N * kk * iters / mx * ctas_per_sm, (M < 128 ? 128 : M) * N / 256.0,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
    long long *d;
    cudaMalloc(&d, 8 * 512);
    if (getenv("MB_CORE_ONLY")) {  // the core kernel's MMA pattern only (MB_TILES tiles per CTA)
        run_core<0>(d); run_core<6>(d);
        return 0;
    }
#define ALLN(BF, M, TS, E) run<BF, M, 32, TS, E>(d, 1); run<BF, M, 64, TS, E>(d, 1); \
    run<BF, M, 128, TS, E>(d, 1); run<BF, M, 256, TS, E>(d, 1);
    run_core<0>(d); run_core<1>(d); run_core<2>(d); run_core<3>(d); run_core<4>(d); run_core<5>(d); run_core<6>(d);
    {
        uint8_t *g;
        cudaMalloc(&g, 17 << 20);
        cudaMemset(g, 0, 17 << 20);
        long long *d2;
        cudaMalloc(&d2, 8 * 1024);
        run_core_int<0>(d2, g); run_core_int<1>(d2, g); run_core_int<2>(d2, g); run_core_int<3>(d2, g);
        run_core_int<4>(d2, g);
        run_core_int<5>(d2, g);
    }
    for (int off : {0, 16, 32, 48, 64, 112}) run_off<32, 1>(d, off);
    for (int off : {0, 16, 32, 64}) run_off<64, 1>(d, off);
    for (int off : {0, 16, 64}) run_off<128, 1>(d, off);
    for (int off : {0, 128, 256, 384, 640}) run_off<32, 0>(d, off);
    for (int off : {0, 128, 384}) run_off<64, 0>(d, off);
    for (int off : {0, 128}) run_off<128, 0>(d, off);
    run_lc<32, 0, 0>(d); run_lc<32, 0, 1>(d); run_lc<32, 1, 0>(d); run_lc<32, 1, 1>(d);
    run_lc<64, 0, 0>(d); run_lc<64, 0, 1>(d); run_lc<64, 1, 0>(d); run_lc<64, 1, 1>(d);
    run_lc<128, 0, 0>(d); run_lc<128, 1, 0>(d); run_lc<128, 1, 1>(d);
    ALLN(1, 128, 0, 0)
    ALLN(1, 128, 0, 1)
    ALLN(1, 128, 1, 0)
    ALLN(1, 64, 0, 0)
    ALLN(0, 128, 0, 0)
    ALLN(0, 128, 1, 0)
    run<1, 128, 32, 0, 0>(d, 2);
    run<1, 128, 64, 0, 0>(d, 2);
    run<1, 128, 128, 0, 0>(d, 2);
    return 0;
}
