// fz_kernels.cuh -- sm_100a kernels of the factorization-set engine.
//
// Everything here is integer work (no tensor cores: nothing is a dense
// contraction).  Kernel map:
//   K1  k1_tables       count pass: suffix tables S_i, prefix tables W_i, card,
//                       CSR offsets (K2) -- one CTA, column scans over the
//                       residue classes of g_i.
//   K3a k3_links        per memo row: the source row of the copy-increment and
//                       the incremented index (fully parallel; depends only on
//                       the count tables).
//   K3b k3_fill_single  the dimensionwise recurrence Z(x) = U_i incr_i(Z_{>=i}(x-g_i))
//       k3_fill_grid    (Alg. 2/3 PAPER.md:139-192) in elementwise
//                       batches of b = min(tail g); one CTA with
//                       the live window in a shared-memory ring, or the whole grid
//                       with a grid barrier between batches for huge memos.
//   K4  k4_plan         slice planner: unrank each slice start (rows or leading
//                       prefixes) to its leading prefix + memo offset.
//   K5  k5_walk         enumerator: nextCandidate over the leading coordinates
//                       (PAPER.md:203-222, 238-265), innermost leading coordinate
//                       across the 32 lanes, memo blocks flattened across the warp
//                       so that every store instruction writes 32 consecutive rows.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/fz.h"

namespace fzk {

constexpr int kMaxD = FZ_MAX_D;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kLinkMask = (1ull << 56) - 1;

struct Gens {
    uint32_t g[kMaxD];
};

// Slice descriptor written by K4, read by K5.  64 bytes.
struct Slice {
    uint64_t begin;       // MAT/HASH: first row, relative to the shard start; COUNT: first prefix, relative
    uint64_t len;         // rows (MAT/HASH) or leading prefixes (COUNT) in the slice
    uint64_t k0;          // offset of the first row inside the first prefix's memo block
    uint32_t a[kMaxD];    // leading prefix (a_1..a_L) of the first block
};
static_assert(sizeof(Slice) == 64, "slice layout");

struct PlanParams {
    uint64_t n;
    uint64_t top;
    uint64_t shard_begin;   // global index (row or prefix) of this shard's first unit
    uint64_t shard_len;     // units in this shard
    uint64_t slice_len;     // units per slice
    uint64_t nslices;
    int d, t, L, mode;
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src)
{
    uint32_t lo = __shfl_sync(kFull, (uint32_t)v, src);
    uint32_t hi = __shfl_sync(kFull, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint32_t lo = __shfl_xor_sync(kFull, (uint32_t)v, o);
        uint32_t hi = __shfl_xor_sync(kFull, (uint32_t)(v >> 32), o);
        v += ((uint64_t)hi << 32) | lo;
    }
    return v;
}

__device__ __forceinline__ uint64_t ld_cg_u64(const uint64_t *p) { return __ldcg(p); }

// Column-wise inclusive scan used by the count pass:
//   dst[x] = src[x] + dst[x - g]   (x >= g),   dst[x] = src[x]   (x < g),  x in [0, N).
// Viewing [0, N) as a row-major matrix with g columns, this is an inclusive
// scan down every column (= every residue class mod g).  Three phases: per
// (column, row segment) partial sums; a warp-level scan of the segment sums of
// each column; re-scan of each segment with its offset.  One CTA.
__device__ void column_scan(const uint64_t *src, uint64_t *dst, uint64_t N, uint64_t g, uint64_t *sm)
{
    const int nt = blockDim.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const uint64_t cols_total = g < N ? g : N;
    const uint64_t rows = (N + g - 1) / g;
    for (uint64_t c0 = 0; c0 < cols_total; c0 += (uint64_t)nt) {
        const int ncols = (int)((cols_total - c0) < (uint64_t)nt ? (cols_total - c0) : (uint64_t)nt);
        const int nseg = nt / ncols;
        const uint64_t R = (rows + nseg - 1) / nseg;
        const int ci = tid % ncols, seg = tid / ncols;
        const bool active = seg < nseg;
        const uint64_t col = c0 + ci;
        uint64_t s = 0;
        if (active) {
            uint64_t k0 = (uint64_t)seg * R, k1 = k0 + R < rows ? k0 + R : rows;
#pragma unroll 8
            for (uint64_t k = k0; k < k1; ++k) {
                uint64_t x = k * g + col;
                if (x < N) s += ld_cg_u64(src + x);
            }
        }
        sm[tid] = s;
        __syncthreads();
        // phase 2: exclusive scan of the nseg segment sums of each column (warp per column)
        for (int c = warp; c < ncols; c += nwarps) {
            uint64_t carry = 0;
            for (int s0 = 0; s0 < nseg; s0 += 32) {
                int sg = s0 + lane;
                uint64_t v = sg < nseg ? sm[sg * ncols + c] : 0;
                uint64_t inc = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    uint64_t u = shfl_u64(inc, (lane - o) & 31);
                    if (lane >= o) inc += u;
                }
                if (sg < nseg) sm[sg * ncols + c] = carry + inc - v;
                carry += shfl_u64(inc, 31);
            }
        }
        __syncthreads();
        if (active) {
            uint64_t run = sm[tid];
            uint64_t k0 = (uint64_t)seg * R, k1 = k0 + R < rows ? k0 + R : rows;
#pragma unroll 8
            for (uint64_t k = k0; k < k1; ++k) {
                uint64_t x = k * g + col;
                if (x < N) {
                    run += ld_cg_u64(src + x);
                    dst[x] = run;
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K1 + K2
// S level i (0-based, i = 0..d) at S + i*top: S_i[x] = |Z(x; g_i..g_{d-1})|, S_d[x] = [x = 0].
// W level j (j = 0..L) at W + j*top: W_j[x] = #{(a_j..a_{L-1}) : sum a g <= x}, W_L[x] = 1.
// card[x] = S_L[x] (u32), off[x] = sum_{y<x} card[y], off[top] = entries.
__global__ void __launch_bounds__(1024) k1_tables(Gens G, int d, int L, uint64_t top, uint64_t *S, uint64_t *W,
                                                   uint32_t *card, uint64_t *off)
{
    __shared__ uint64_t sm[1024];
    const int nt = blockDim.x, tid = threadIdx.x;
    for (uint64_t x = tid; x < top; x += nt) {
        S[(uint64_t)d * top + x] = (x == 0) ? 1ull : 0ull;
        if (W) W[(uint64_t)L * top + x] = 1ull;
    }
    __syncthreads();
    for (int i = d - 1; i >= 0; --i) column_scan(S + (uint64_t)(i + 1) * top, S + (uint64_t)i * top, top, G.g[i], sm);
    if (W)
        for (int j = L - 1; j >= 0; --j)
            column_scan(W + (uint64_t)(j + 1) * top, W + (uint64_t)j * top, top, G.g[j], sm);
    const uint64_t *cardS = S + (uint64_t)L * top;
    for (uint64_t x = tid; x < top; x += nt) card[x] = (uint32_t)ld_cg_u64(cardS + x);
    // K2: CSR offsets = exclusive scan of card; inclusive scan into off[1..top]
    column_scan(cardS, off + 1, top, 1, sm);
    if (tid == 0) off[0] = 0;
}

// ---------------------------------------------------------------------- K3a
// links[off[x] + q] = (src row) | (i << 56) for every row q of Z(x; tail), x in [1, top).
// Block i (0-based tail index) of Z(x) starts at card[x] - S_{L+i}[x]; its k-th
// row is incr_i of row off[y] + card[y] - S_{L+i}[y] + k = off[y+1] - S_{L+i}[y] + k
// of Z(y), y = x - g_{L+i}  ("beginning index of Z_{>=i}").
__global__ void __launch_bounds__(256) k3_links(Gens G, int L, int t, uint64_t top, const uint64_t *__restrict__ S,
                                                 const uint64_t *__restrict__ off, uint64_t *__restrict__ links)
{
    const int lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if (gw == 0 && lane == 0) links[0] = ~0ull;   // Memo[0] = [0]: the base case row
    for (uint64_t x = 1 + gw; x < top; x += nw) {
        const uint64_t base = __ldg(off + x);
        const uint64_t c = __ldg(off + x + 1) - base;
        if (c == 0) continue;
        for (uint64_t q = lane; q < c; q += 32) {
            int i = 0;
            uint64_t st = 0;
            for (int j = t - 1; j >= 1; --j) {
                uint64_t sj = c - __ldg(S + (uint64_t)(L + j) * top + x);
                if (sj <= q) { i = j; st = sj; break; }
            }
            const uint64_t y = x - G.g[L + i];
            const uint64_t src = __ldg(off + y + 1) - __ldg(S + (uint64_t)(L + i) * top + y) + (q - st);
            links[base + q] = src | ((uint64_t)i << 56);
        }
    }
}

template <int T>
__device__ __forceinline__ void incr_word(uint32_t (&w)[T], int i)
{
#pragma unroll
    for (int j = 0; j < T; ++j) w[j] += (j == i) ? 1u : 0u;
}

// ---------------------------------------------------------------------- K3b
// One CTA runs the batches in order; within a batch every row is independent
// (elementwise x factorizationwise parallelism).  Rows of the
// live window (the last max(tail g) x-blocks) are read from a shared-memory
// ring when RING (fill mode 1), else from global memory written earlier by
// this same CTA (mode 2).  The links of batch k+1 and the batch boundary of
// batch k+2 are prefetched while batch k runs, so the per-batch critical path is
// ring load -> increment -> ring/global store -> __syncthreads.
template <int T, bool RING>
__global__ void __launch_bounds__(1024) k3_fill_single(const uint64_t *__restrict__ off,
                                                        const uint64_t *__restrict__ links, uint32_t *rows,
                                                        uint64_t top, uint32_t b, uint64_t ring_mask)
{
    constexpr int MAXR = 4;
    extern __shared__ uint32_t ring[];
    const uint64_t nt = blockDim.x, tid = threadIdx.x;
    auto bend = [&](uint64_t x0) -> uint64_t {   // off[] at the end of the batch starting at x0
        uint64_t x1 = x0 + b;
        return __ldg(off + (x1 < top ? x1 : top));
    };
    uint64_t R0 = 0, R1 = bend(0);
    uint64_t R2 = ((uint64_t)b < top) ? bend(b) : R1;
    uint64_t pf[MAXR];
#pragma unroll
    for (int j = 0; j < MAXR; ++j) {
        uint64_t r = R0 + tid + j * nt;
        pf[j] = r < R1 ? __ldg(links + r) : 0;
    }
    auto process = [&](uint64_t r, uint64_t link) {
        uint32_t w[T];
        if (link == ~0ull) {
#pragma unroll
            for (int j = 0; j < T; ++j) w[j] = 0;
        } else {
            const uint64_t src = link & kLinkMask;
            const int i = (int)(link >> 56);
            if (RING) {
                const uint32_t *s = ring + (src & ring_mask) * T;
#pragma unroll
                for (int j = 0; j < T; ++j) w[j] = s[j];
            } else {
                const uint32_t *s = rows + src * T;
#pragma unroll
                for (int j = 0; j < T; ++j) w[j] = s[j];
            }
            incr_word<T>(w, i);
        }
        if (RING) {
            uint32_t *dr = ring + (r & ring_mask) * T;
#pragma unroll
            for (int j = 0; j < T; ++j) dr[j] = w[j];
        }
        uint32_t *dg = rows + r * T;
#pragma unroll
        for (int j = 0; j < T; ++j) dg[j] = w[j];
    };
    for (uint64_t x0 = 0; x0 < top; x0 += b) {
        // prefetch: links of the next batch, boundary of the batch after it
        uint64_t nf[MAXR];
#pragma unroll
        for (int j = 0; j < MAXR; ++j) {
            uint64_t r = R1 + tid + j * nt;
            nf[j] = r < R2 ? __ldg(links + r) : 0;
        }
        const uint64_t R3 = (x0 + 2ull * b < top) ? bend(x0 + 2ull * b) : R2;
#pragma unroll
        for (int j = 0; j < MAXR; ++j) {
            uint64_t r = R0 + tid + j * nt;
            if (r < R1) process(r, pf[j]);
        }
        for (uint64_t r = R0 + tid + MAXR * nt; r < R1; r += nt) process(r, __ldg(links + r));
        __syncthreads();
        R0 = R1;
        R1 = R2;
        R2 = R3;
#pragma unroll
        for (int j = 0; j < MAXR; ++j) pf[j] = nf[j];
    }
}

// Grid barrier for a cooperative launch (all CTAs co-resident).  `counter`
// grows monotonically; `target` is the per-CTA running target.
__device__ __forceinline__ void grid_barrier(unsigned int *counter, unsigned int &target)
{
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(counter, 1u);
        unsigned int v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
            if ((int)(v - target) >= 0) break;
            __nanosleep(64);
        }
        __threadfence();
    }
    __syncthreads();
}

// Whole-grid variant (fill mode 3, memos with many rows per batch): the row
// -> (x, block, source) mapping is computed inline, sources are read through L2.
template <int T>
__global__ void __launch_bounds__(256) k3_fill_grid(Gens G, int L, uint64_t top, uint32_t b,
                                                     const uint64_t *__restrict__ S,
                                                     const uint64_t *__restrict__ off, uint32_t *rows,
                                                     unsigned int *counter)
{
    const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t ng = (uint64_t)gridDim.x * blockDim.x;
    unsigned int target = 0;
    for (uint64_t x0 = 0; x0 < top; x0 += b) {
        const uint64_t x1 = (x0 + b < top) ? x0 + b : top;
        const uint64_t R0 = __ldg(off + x0), R1 = __ldg(off + x1);
        for (uint64_t r = R0 + gt; r < R1; r += ng) {
            uint32_t w[T];
            if (r == 0) {
#pragma unroll
                for (int j = 0; j < T; ++j) w[j] = 0;
            } else {
                // x: largest x in [x0, x1) with off[x] <= r
                uint64_t lo = x0, hi = x1 - 1;
                while (lo < hi) {
                    uint64_t mid = (lo + hi + 1) >> 1;
                    if (__ldg(off + mid) <= r) lo = mid; else hi = mid - 1;
                }
                const uint64_t x = lo, q = r - __ldg(off + x);
                const uint64_t c = __ldg(off + x + 1) - __ldg(off + x);
                int i = 0;
                uint64_t st = 0;
                for (int j = T - 1; j >= 1; --j) {
                    uint64_t sj = c - __ldg(S + (uint64_t)(L + j) * top + x);
                    if (sj <= q) { i = j; st = sj; break; }
                }
                const uint64_t y = x - G.g[L + i];
                const uint64_t src = __ldg(off + y + 1) - __ldg(S + (uint64_t)(L + i) * top + y) + (q - st);
                const uint32_t *s = rows + src * T;
#pragma unroll
                for (int j = 0; j < T; ++j) w[j] = __ldcg(s + j);
                incr_word<T>(w, i);
            }
            uint32_t *dg = rows + r * T;
#pragma unroll
            for (int j = 0; j < T; ++j) dg[j] = w[j];
        }
        grid_barrier(counter, target);
    }
}

// ----------------------------------------------------------------------- K4
// Warp-cooperative unranking.  `Tb` points at level 0 of a table with levels
// of `top` entries; level j counts the units (rows for S, prefixes for W) of a
// subtree: F_j(a) = Tb[j][r - a g_j] = units with a'_j >= a under the current
// prefix.  At each level a_j = max{a : F_j(a) > R}, then R -= F_j(a_j + 1).
// Returns the remaining R (offset inside the memo block for S; 0 for W).
__device__ uint64_t unrank(const uint64_t *__restrict__ Tb, uint64_t top, const Gens &G, int L, uint64_t n,
                           uint64_t R, uint32_t *a)
{
    const int lane = threadIdx.x & 31;
    uint64_t r = n;
    for (int j = 0; j < L; ++j) {
        const uint64_t *Tj = Tb + (uint64_t)j * top;
        const uint64_t gj = G.g[j];
        const uint64_t amax = r / gj;
        uint64_t lo = 0, hi = amax;
        while (lo < hi) {
            const uint64_t step = (hi - lo + 31) / 32;
            const uint64_t cand = lo + (uint64_t)(lane + 1) * step;
            const bool pred = cand <= hi && __ldg(Tj + (r - cand * gj)) > R;
            const unsigned bal = __ballot_sync(kFull, pred);
            const int m = __popc(bal);
            const uint64_t nlo = lo + (uint64_t)m * step;
            uint64_t nhi = lo + (uint64_t)(m + 1) * step - 1;
            if (nhi > hi) nhi = hi;
            lo = nlo;
            hi = nhi;
        }
        a[j] = (uint32_t)lo;
        const uint64_t fnext = (lo + 1 <= amax) ? __ldg(Tj + (r - (lo + 1) * gj)) : 0;
        R -= fnext;
        r -= lo * gj;
    }
    return R;
}

__global__ void __launch_bounds__(256) k4_plan(Gens G, PlanParams P, const uint64_t *__restrict__ S,
                                                const uint64_t *__restrict__ W, Slice *slices, uint64_t *result)
{
    const int lane = threadIdx.x & 31;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    if (gw == 0 && lane < 2) result[lane] = 0;
    const bool count_mode = (P.mode == FZ_COUNT);
    for (uint64_t s = gw; s < P.nslices; s += nw) {
        const uint64_t rel = s * P.slice_len;
        const uint64_t len = (P.shard_len - rel) < P.slice_len ? (P.shard_len - rel) : P.slice_len;
        uint32_t a[kMaxD];
        for (int j = 0; j < kMaxD; ++j) a[j] = 0;
        const uint64_t k0 = unrank(count_mode ? W : S, P.top, G, P.L, P.n, P.shard_begin + rel, a);
        if (lane == 0) {
            Slice sl;
            sl.begin = rel;
            sl.len = len;
            sl.k0 = count_mode ? 0 : k0;
            for (int j = 0; j < kMaxD; ++j) sl.a[j] = a[j];
            slices[s] = sl;
        }
    }
}

// ----------------------------------------------------------------------- K5
// Order-sensitive row hash (reading R17), the product's own
// implementation.
template <int D>
__device__ __forceinline__ uint64_t row_hash(uint64_t k, const uint32_t (&w)[D])
{
    uint64_t x = (k + 1) * 0x9E3779B97F4A7C15ull;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        x = (x ^ (uint64_t)w[j]) * 0xBF58476D1CE4E5B9ull;
        x ^= x >> 29;
    }
    x ^= (uint64_t)D;
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDull;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ull;
    x ^= x >> 33;
    return x;
}

template <int T>
__device__ __forceinline__ void load_tail(const uint32_t *__restrict__ p, uint32_t *w)
{
    if constexpr (T == 2) {
        uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        w[0] = v.x; w[1] = v.y;
    } else if constexpr (T == 4) {
        uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
    } else {
#pragma unroll
        for (int j = 0; j < T; ++j) w[j] = __ldg(p + j);
    }
}

template <int D>
__device__ __forceinline__ void store_row(uint32_t *p, const uint32_t (&w)[D])
{
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 4) {
            uint4 v = make_uint4(w[j], w[j + 1], w[j + 2], w[j + 3]);
            __stcs(reinterpret_cast<uint4 *>(p + j), v);
        }
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2) {
            uint2 v = make_uint2(w[j], w[j + 1]);
            __stcs(reinterpret_cast<uint2 *>(p + j), v);
        }
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) __stcs(p + j, w[j]);
    }
}

struct BlockInfo {      // one non-empty memo block of the current warp round (16 B)
    uint64_t memo_row;  // first memo row to copy (off[p] + k offset)
    uint32_t start;     // first output row of the block, relative to the round
    uint32_t v;         // innermost leading coordinate a_L of the block
};

constexpr int kWalkThreads = 256;

template <int D, int T, int MODE>
__global__ void __launch_bounds__(kWalkThreads) k5_walk(Gens G, PlanParams P, const Slice *__restrict__ slices,
                                                         const uint32_t *__restrict__ card,
                                                         const uint64_t *__restrict__ off,
                                                         const uint32_t *__restrict__ memo, uint32_t *out,
                                                         uint64_t row_base, uint64_t *result)
{
    constexpr int L = D - T;
    static_assert(L >= 1, "at least one leading coordinate");
    __shared__ BlockInfo binfo[kWalkThreads / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t n = P.n;
    const uint64_t gL = G.g[L - 1];
    uint64_t acc_rows = 0, acc_hash = 0;
    BlockInfo *bi = binfo[wib];

    for (uint64_t s = gw; s < P.nslices; s += nw) {
        const Slice sl = slices[s];
        uint32_t a[L];
#pragma unroll
        for (int j = 0; j < L; ++j) a[j] = sl.a[j];
        uint64_t r_in = n;
#pragma unroll
        for (int j = 0; j < L - 1; ++j) r_in -= (uint64_t)a[j] * G.g[j];
        int64_t v = a[L - 1];
        uint64_t kfirst = sl.k0;
        uint64_t left = sl.len;
        uint64_t outpos = sl.begin;
        while (left > 0) {
            const int64_t vv = v - lane;
            const bool valid = vv >= 0;
            const uint64_t p = valid ? r_in - (uint64_t)vv * gL : 0;
            uint32_t c = valid ? __ldg(card + p) : 0u;
            if constexpr (MODE == FZ_COUNT) {
                const uint64_t nvalid = (v + 1) < 32 ? (uint64_t)(v + 1) : 32ull;
                const uint64_t take = nvalid < left ? nvalid : left;
                if ((uint64_t)lane < take) acc_rows += c;
                left -= take;
            } else {
                uint64_t mrow = valid ? __ldg(off + p) : 0;
                if (lane == 0) {
                    c -= (uint32_t)kfirst;
                    mrow += kfirst;
                }
                kfirst = 0;
                uint32_t incl = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    uint32_t u = __shfl_up_sync(kFull, incl, o);
                    if (lane >= o) incl += u;
                }
                const uint32_t excl = incl - c;
                const uint32_t total = __shfl_sync(kFull, incl, 31);
                const uint32_t use = (uint64_t)total < left ? total : (uint32_t)left;
                const uint32_t cc = excl >= use ? 0u : (c < use - excl ? c : use - excl);
                const unsigned nz = __ballot_sync(kFull, cc > 0);
                if (cc > 0) {
                    const int e = __popc(nz & ((1u << lane) - 1));
                    bi[e].memo_row = mrow;
                    bi[e].start = excl;
                    bi[e].v = (uint32_t)vv;
                }
                __syncwarp();
                // flattened copy: rows q0 + lane of the round, owner block via block-start bitmask
                int e0 = 0;
                for (uint32_t q0 = 0; q0 < use; q0 += 32) {
                    const unsigned bit = (cc > 0 && excl >= q0 && excl - q0 < 32) ? (1u << (excl - q0)) : 0u;
                    const unsigned M = __reduce_or_sync(kFull, bit);
                    if (q0 != 0) e0 += (int)(M & 1u);
                    const uint32_t q = q0 + lane;
                    if (q < use) {
                        const int e = e0 + __popc(M & ((2u << lane) - 2u));
                        const BlockInfo info = bi[e];
                        uint32_t w[D];
#pragma unroll
                        for (int j = 0; j < L - 1; ++j) w[j] = a[j];
                        w[L - 1] = info.v;
                        if constexpr (T > 0) {
                            uint32_t tw[T];
                            load_tail<T>(memo + (info.memo_row + (q - info.start)) * T, tw);
#pragma unroll
                            for (int j = 0; j < T; ++j) w[L + j] = tw[j];
                        }
                        if constexpr (MODE == FZ_MATERIALIZE) {
                            store_row<D>(out + (outpos + q) * (uint64_t)D, w);
                        } else {
                            acc_hash += row_hash<D>(row_base + outpos + q, w);
                        }
                    }
                    e0 += __popc(M & 0xfffffffeu);
                }
                __syncwarp();
                acc_rows += (lane == 0) ? use : 0;
                outpos += use;
                left -= use;
            }
            if (left == 0) break;
            if (v >= 32) {
                v -= 32;
                continue;
            }
            // carry: nextCandidate over the outer leading coordinates:
            // rightmost nonzero index i < L-1, a_i--, later coordinates restart at their maximum.
            int i = -1;
#pragma unroll
            for (int j = 0; j < L - 1; ++j)
                if (a[j] > 0) i = j;
            if (i < 0) break;   // end of stream
            uint64_t r = n;
#pragma unroll
            for (int j = 0; j < L - 1; ++j) {
                if (j == i) a[j] -= 1;
                if (j > i) a[j] = (uint32_t)(r / G.g[j]);
                r -= (uint64_t)a[j] * G.g[j];
            }
            r_in = r;
            v = (int64_t)(r / gL);
        }
    }
    acc_rows = warp_sum_u64(acc_rows);
    acc_hash = warp_sum_u64(acc_hash);
    if (lane == 0) {
        atomicAdd((unsigned long long *)result, (unsigned long long)acc_rows);
        if (MODE == FZ_HASH) atomicAdd((unsigned long long *)(result + 1), (unsigned long long)acc_hash);
    }
}

}  // namespace fzk
