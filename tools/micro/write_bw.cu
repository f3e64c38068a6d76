// Microbenchmark: achievable HBM write bandwidth on this B200 for a pure 16-B streaming-store fill
// (the roofline ceiling of K5 materialize), and a copy for comparison.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill(uint4 *p, size_t n, uint32_t v)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i), "r"(v) : "memory");
}
__global__ void copy(const uint4 *__restrict__ a, uint4 *b, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

int main()
{
    const size_t bytes = 1600010896ull & ~15ull, n = bytes / 16;
    uint4 *p, *q;
    cudaMalloc(&p, bytes);
    cudaMalloc(&q, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bpsm : {2, 4, 8, 16}) {
        for (int it = 0; it < 3; ++it) fill<<<sms * bpsm, 256>>>(p, n, it);
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) fill<<<sms * bpsm, 256>>>(p, n, it);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("fill 1.6 GB, %2d CTAs/SM x 256: %.1f us  %.0f GB/s\n", bpsm, ms * 100, bytes / (ms / 10 / 1e3) / 1e9);
    }
    for (int it = 0; it < 3; ++it) copy<<<sms * 8, 256>>>(p, q, n);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) copy<<<sms * 8, 256>>>(p, q, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 1.6 GB: %.1f us  %.0f GB/s (read+write)\n", ms * 100, 2 * bytes / (ms / 10 / 1e3) / 1e9);
    return 0;
}
