// Microbenchmark: achievable HBM write bandwidth on this B200 for a pure 16-B streaming-store fill
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/micro/write_bw tools/micro/write_bw.cu
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

// K5's store pattern: each warp owns one contiguous region (a slice) and writes it front to back in
// batches of 4 x 512 B (4 chunks of 32 rows x 16 B), with `slices` regions taken in order by a queue
__global__ void region_fill(uint4 *p, size_t n, size_t per_slice, size_t slices, unsigned long long *queue, uint32_t v)
{
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned long long s = 0;
        if (lane == 0) s = atomicAdd(queue, 1ull);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= slices) break;
        const size_t b = s * per_slice, e = (b + per_slice < n) ? b + per_slice : n;
        for (size_t i = b + lane; i < e; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + 32 * u < e)
                    asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
        }
    }
}

// the same with static round-robin slices (warp w takes slices w, w + nw, ...): no queue atomics
__global__ void region_fill_static(uint4 *p, size_t n, size_t per_slice, size_t slices, uint32_t v)
{
    const int lane = threadIdx.x & 31;
    const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t s = w; s < slices; s += nw) {
        const size_t b = s * per_slice, e = (b + per_slice < n) ? b + per_slice : n;
        for (size_t i = b + lane; i < e; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + 32 * u < e)
                    asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
        }
    }
}

// store-cache-hint variants of the static region fill: 0 = .cs (K5), 1 = default (.wb), 2 = .L2::evict_last-free
template <int V>
__global__ void region_fill_v(uint4 *p, size_t n, size_t per_slice, size_t slices, uint32_t v)
{
    const int lane = threadIdx.x & 31;
    const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5, nw = ((size_t)gridDim.x * blockDim.x) >> 5;
    for (size_t s = w; s < slices; s += nw) {
        const size_t b = s * per_slice, e = (b + per_slice < n) ? b + per_slice : n;
        for (size_t i = b + lane; i < e; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + 32 * u < e) {
                    if (V == 0)
                        asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
                    else if (V == 1)
                        asm volatile("st.global.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
                    else
                        asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
                }
        }
    }
}

template <int V>
float time_v(uint4 *p, size_t n, size_t per, size_t slices, int grid, cudaEvent_t e0, cudaEvent_t e1)
{
    for (int it = 0; it < 3; ++it) region_fill_v<V><<<grid, 256>>>(p, n, per, slices, it);
    cudaEventRecord(e0);
    for (int it = 0; it < 10; ++it) region_fill_v<V><<<grid, 256>>>(p, n, per, slices, it);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / 10;
}

// K5's pattern with a non-persistent grid: CTA b takes the contiguous slice range [b S / nb, (b+1) S / nb),
// its warps round-robin inside it; more CTAs than resident ones (several waves, like the grid-stride fill)
__global__ void region_fill_waves(uint4 *p, size_t n, size_t per_slice, size_t slices, uint32_t v)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    const size_t s0 = slices * blockIdx.x / gridDim.x, s1 = slices * (blockIdx.x + 1) / gridDim.x;
    for (size_t s = s0 + wib; s < s1; s += nwb) {
        const size_t b = s * per_slice, e = (b + per_slice < n) ? b + per_slice : n;
        for (size_t i = b + lane; i < e; i += 128) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + 32 * u < e)
                    asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
        }
    }
}

// the same address order with persistent CTAs: CTA b runs the virtual CTAs v = b, b + grid, .. (V of them)
__global__ void region_fill_virtual(uint4 *p, size_t n, size_t per_slice, size_t slices, size_t V, uint32_t v)
{
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
    for (size_t vb = blockIdx.x; vb < V; vb += gridDim.x) {
        const size_t s0 = slices * vb / V, s1 = slices * (vb + 1) / V;
        for (size_t s = s0 + wib; s < s1; s += nwb) {
            const size_t b = s * per_slice, e = (b + per_slice < n) ? b + per_slice : n;
            for (size_t i = b + lane; i < e; i += 128) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (i + 32 * u < e)
                        asm volatile("st.global.cs.v4.u32 [%0], {%1, %1, %1, %1};" ::"l"(p + i + 32 * u), "r"(v) : "memory");
            }
        }
    }
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
    {
        unsigned long long *queue;
        cudaMalloc(&queue, 8);
        for (size_t slices : {(size_t)75759, (size_t)4736, (size_t)sms * 4 * 8 * 64}) {
            const size_t per = (n + slices - 1) / slices;
            for (int it = 0; it < 3; ++it) {
                cudaMemset(queue, 0, 8);
                region_fill<<<sms * 4, 256>>>(p, n, per, slices, queue, it);
            }
            float tot = 0;
            for (int it = 0; it < 10; ++it) {
                cudaMemset(queue, 0, 8);
                cudaEventRecord(e0);
                region_fill<<<sms * 4, 256>>>(p, n, per, slices, queue, it);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                tot += ms;
            }
            printf("region fill 1.6 GB, %zu slices (warp-owned, 2 KB batches), 4 CTAs/SM x 256: %.1f us  %.0f GB/s\n",
                   slices, tot * 100, bytes / (tot / 10 / 1e3) / 1e9);
            for (int it = 0; it < 3; ++it) region_fill_static<<<sms * 4, 256>>>(p, n, per, slices, it);
            cudaEventRecord(e0);
            for (int it = 0; it < 10; ++it) region_fill_static<<<sms * 4, 256>>>(p, n, per, slices, it);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms2;
            cudaEventElapsedTime(&ms2, e0, e1);
            printf("region fill 1.6 GB, %zu slices, static round-robin, 4 CTAs/SM x 256: %.1f us  %.0f GB/s\n", slices,
                   ms2 * 100, bytes / (ms2 / 10 / 1e3) / 1e9);
        }
    }
    for (int bpsm : {4, 8}) {
        const size_t slices = 75759, per = (n + slices - 1) / slices;
        const float a = time_v<0>(p, n, per, slices, sms * bpsm, e0, e1), b = time_v<1>(p, n, per, slices, sms * bpsm, e0, e1),
                    c = time_v<2>(p, n, per, slices, sms * bpsm, e0, e1);
        printf("region fill (75759 static slices, %d CTAs/SM): st.cs %.1f us, st (wb) %.1f us, st.L1::no_allocate %.1f us\n",
               bpsm, a * 1e3, b * 1e3, c * 1e3);
    }
    for (int waves : {1, 2, 4, 8}) {
        const size_t slices = 75759, per = (n + slices - 1) / slices;
        const int grid = sms * 4 * waves;
        for (int it = 0; it < 3; ++it) region_fill_waves<<<grid, 256>>>(p, n, per, slices, it);
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) region_fill_waves<<<grid, 256>>>(p, n, per, slices, it);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("region fill, 75759 slices in per-CTA contiguous ranges, %d x 4 CTAs/SM (4 resident): %.1f us\n", waves,
               ms * 100);
    }
    for (int waves : {1, 4, 8, 16}) {
        const size_t slices = 75759, per = (n + slices - 1) / slices;
        const int grid = sms * 4;
        const size_t V = (size_t)grid * waves;
        for (int it = 0; it < 3; ++it) region_fill_virtual<<<grid, 256>>>(p, n, per, slices, V, it);
        cudaEventRecord(e0);
        for (int it = 0; it < 10; ++it) region_fill_virtual<<<grid, 256>>>(p, n, per, slices, V, it);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("region fill, persistent 4 CTAs/SM running %d x virtual CTAs in order: %.1f us\n", waves, ms * 100);
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
