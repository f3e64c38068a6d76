// Microbenchmark: cost of the K1 grid barrier and of one column scan phase on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/grid_barrier tools/micro/grid_barrier.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2407_20474_b200/csrc/fz_kernels.cuh"

__global__ void __launch_bounds__(1024) bar_only(unsigned int *counter, int iters, unsigned long long *t)
{
    unsigned int target = 0;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int k = 0; k < iters; ++k) fzk::grid_barrier(counter, target);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) t[0] = t1 - t0;
}

__global__ void __launch_bounds__(1024) scan_only(const uint64_t *src, uint64_t *dst, uint64_t N, uint64_t g, int iters,
                                                  unsigned long long *t)
{
    __shared__ uint64_t sm[40];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int k = 0; k < iters; ++k) fzk::block_column_scan(src, dst, N, g, blockIdx.x, sm);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(1024) scan_w_only(const uint64_t *src, uint64_t *dst, uint64_t N, uint64_t g,
                                                    int iters, unsigned long long *t)
{
    __shared__ uint64_t sm[40];
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int k = 0; k < iters; ++k)
        fzk::block_column_scan_w([=](uint64_t x) { return __ldcg(src + x); }, dst, N, g, blockIdx.x, sm);
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) t[blockIdx.x] = t1 - t0;
}

int main()
{
    unsigned int *counter;
    unsigned long long *t;
    cudaMalloc(&counter, 4);
    cudaMalloc(&t, 8 * 1024);
    for (int blocks : {16, 64, 148}) {
        cudaMemset(counter, 0, 4);
        int iters = 100;
        void *args[] = {&counter, &iters, &t};
        cudaLaunchCooperativeKernel((void *)bar_only, blocks, 1024, args, 0, 0);
        cudaDeviceSynchronize();
        unsigned long long h;
        cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost);
        printf("grid barrier, %3d CTAs: %.2f us per barrier (%s)\n", blocks, h / 1e3 / iters,
               cudaGetErrorString(cudaGetLastError()));
    }
    uint64_t N = 30233;
    uint64_t *src, *dst;
    cudaMalloc(&src, N * 8);
    cudaMalloc(&dst, N * 8);
    cudaMemset(src, 0, N * 8);
    for (uint64_t g : {11ull, 19ull, 101ull}) {
        int iters = 20;
        scan_only<<<g, 1024>>>(src, dst, N, g, iters, t);
        cudaDeviceSynchronize();
        unsigned long long h[128];
        cudaMemcpy(h, t, 8 * g, cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (uint64_t i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("column scan N=%llu g=%llu: %.2f us per scan (max over columns)\n", (unsigned long long)N,
               (unsigned long long)g, mx / 1e3 / iters);
        scan_w_only<<<g, 1024>>>(src, dst, N, g, iters, t);
        cudaDeviceSynchronize();
        cudaMemcpy(h, t, 8 * g, cudaMemcpyDeviceToHost);
        mx = 0;
        for (uint64_t i = 0; i < g; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("column scan (warp-segmented) N=%llu g=%llu: %.2f us per scan (max over columns)\n",
               (unsigned long long)N, (unsigned long long)g, mx / 1e3 / iters);
        {   // check: both scans give the same table on a non-trivial source
            std::vector<uint64_t> hs(N);
            for (uint64_t x = 0; x < N; ++x) hs[x] = (x * 2654435761ull) % 1000;
            cudaMemcpy(src, hs.data(), N * 8, cudaMemcpyHostToDevice);
            scan_only<<<g, 1024>>>(src, dst, N, g, 1, t);
            std::vector<uint64_t> a(N), b(N);
            cudaMemcpy(a.data(), dst, N * 8, cudaMemcpyDeviceToHost);
            scan_w_only<<<g, 1024>>>(src, dst, N, g, 1, t);
            cudaMemcpy(b.data(), dst, N * 8, cudaMemcpyDeviceToHost);
            printf("  tables equal: %s\n", a == b ? "yes" : "NO");
        }
    }
    return 0;
}
