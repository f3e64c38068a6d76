// fz_kernels.cuh -- sm_100a kernels of the factorization-set engine.
//
// Everything here is integer work (no tensor cores: nothing is a dense
// contraction).  Kernel map:
//   K1  k1_tables       count pass + CSR + links, one cooperative grid: suffix
//                       tables S_i and prefix tables W_i by column scans over the
//                       residue classes of g_i, card
//                       and CSR offsets (K2) -- also in a residue-major copy for
//                       the walk -- and, per memo row, the copy-increment source
//                       ("link") of the recurrence.
//   K3  k3_fill_ring    the dimensionwise recurrence Z(x) = U_i incr_i(Z_{>=i}(x-g_i))
//       k3_fill_l2      (Alg. 2/3) in elementwise
//       k3_fill_grid    batches of b = min(tail g): one CTA with
//                       the live window in a shared-memory ring and TMA-prefetched
//                       links; one CTA through L2; or the whole grid with a grid
//                       barrier between batches for huge memos.
//   K4  k4_plan         slice planner: unrank each slice start (rows or leading
//                       prefixes) to its leading prefix + memo offset.
//   K5  k5_walk         enumerator: nextCandidate over the leading coordinates
//                       (PAPER.md:203-222, 238-265), innermost leading coordinate
//                       across the 32 lanes (contiguous in the residue-major
//                       tables), memo blocks flattened across the warp so that every
//                       store instruction writes 32 consecutive rows.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/fz.h"

namespace fzk {

constexpr int kMaxD = FZ_MAX_D;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint64_t kLinkMask = (1ull << 56) - 1;
constexpr uint32_t kRingIdxBits = 27;
constexpr uint32_t kZeroLink32 = 0xffffffffu;

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

// Plan header (first 256 B of a plan workspace): written by K4, read by K5.
struct PlanHdr {
    uint64_t result[2];    // {rows, hash}: K5 accumulators
    uint64_t err;          // nonzero: the output buffer is too small (nothing written)
    uint64_t total_units;  // rows (MAT/HASH) or leading prefixes (COUNT) of all of Z(n)
    uint64_t shard_begin;  // first unit of this shard
    uint64_t shard_len;    // units in this shard
    uint64_t slice_len;    // units per slice
    uint64_t nslices;
    uint64_t row_begin;    // global row index of the shard's first row
    uint64_t rows;         // rows of Z(n) in this shard
    unsigned long long next_slice;   // K5 work queue (slices are claimed with atomicAdd)
    uint64_t gss_warps;    // != 0: guided slices (COUNT pair walk): rounds of gss_warps slices, each round
                           // half the size of the last, down to slice_len (gss_begin); 0: uniform slices
    uint64_t rbeta;        // != 0 (MATERIALIZE / HASH, k5_walk): slices are ranges of walk COST units -- one per
                           // row plus rbeta per leading prefix the walk visits -- instead of rows (unrank_cost)
};
static_assert(sizeof(PlanHdr) <= 256, "plan header");

struct PlanArgs {
    uint64_t n;
    uint64_t top;
    uint64_t max_slices;
    uint64_t floor_len;
    int mode, shard, nshards, L;
    int pairs;           // COUNT pair walk: units are cost ranks of the C tables, cut at outer prefixes
    uint64_t wg;         // pair walk: warps of the K5 grid (guided slice rounds)
    uint64_t gss_tail;   // pair walk: the last slices are ~ 1/gss_tail of a warp's share
    uint64_t rbeta;      // MATERIALIZE / HASH with k5_walk: cost of a visited leading prefix in rows (0: row slices)
};

// Guided slices (pair walk): round r has `wg` slices of (len >> (r + 1)) / wg units each, until that
// size drops to `fl`; the rest is cut into slices of fl units.  First unit of slice i (clamped to len).
__host__ __device__ __forceinline__ uint64_t gss_begin(uint64_t i, uint64_t len, uint64_t wg, uint64_t fl)
{
    uint64_t B = 0;
    for (int r = 0; r < 63; ++r) {
        const uint64_t z = (len >> (r + 1)) / wg;
        if (z <= fl) {
            B += i * fl;
            break;
        }
        if (i < wg) {
            B += i * z;
            break;
        }
        B += wg * z;
        i -= wg;
    }
    return B < len ? B : len;
}

__host__ __device__ __forceinline__ uint64_t gss_count(uint64_t len, uint64_t wg, uint64_t fl)
{
    uint64_t B = 0, ns = 0;
    for (int r = 0; r < 63; ++r) {
        const uint64_t z = (len >> (r + 1)) / wg;
        if (z <= fl) return ns + (len - B + fl - 1) / fl;
        B += wg * z;
        ns += wg;
    }
    return ns;
}

// x / g for x < 2^32 by the precomputed magic M = ceil(2^64 / g) (M = 0 encodes g = 1): the error of
// x M / 2^64 against x / g is below x / 2^64 < 1 / g, so the floor is exact.
__device__ __forceinline__ uint32_t fdiv(uint32_t x, uint64_t M) { return M ? (uint32_t)__umul64hi(x, M) : x; }

struct ProgGens {     // closed form of Z(x; g, h), g = g_{d-2}, h = g_{d-1}
    uint32_t g, h, e, g1, h1, inv;   // e = gcd(g, h), g1 = g/e, h1 = h/e, inv = g1^{-1} mod h1
    uint64_t mg, mh, me, mh1;        // fdiv magics of g, h, e, h1 (0 encodes 1)
};

// Z(x; g, h) in descending lex order: rows (w0 - j h1, l0 + j g1), j < count
__device__ __forceinline__ uint32_t prog_block(const ProgGens &P, uint32_t x, uint32_t &w0, uint32_t &l0)
{
    const uint32_t xe = fdiv(x, P.me);
    if (x != xe * P.e) return 0;
    const uint32_t a = xe - fdiv(xe, P.mh1) * P.h1;          // (x / e) mod h1
    uint32_t ws;                                               // w == ws (mod h1)
    if (P.h1 <= 0xffffu) {
        const uint32_t pr = a * P.inv;                         // < h1^2 < 2^32
        ws = pr - fdiv(pr, P.mh1) * P.h1;
    } else {
        ws = (uint32_t)(((uint64_t)a * P.inv) % P.h1);
    }
    const uint32_t wmax = fdiv(x, P.mg);
    if (wmax < ws) return 0;
    const uint32_t dw = wmax - ws;
    w0 = wmax - (dw - fdiv(dw, P.mh1) * P.h1);
    l0 = fdiv(x - w0 * P.g, P.mh);
    return fdiv(w0, P.mh1) + 1;
}

// |Z(x; g, h)| in closed form (the count of prog_block)
__device__ __forceinline__ uint64_t prog_count(const ProgGens &P, uint32_t x)
{
    uint32_t w0, l0;
    return prog_block(P, x, w0, l0);
}

// Pointers and sizes of the count tables (all in the memo workspace).
struct Tables {
    uint64_t *S;        // (d+1) x top, natural layout
    uint64_t *W;        // (L+1) x top
    uint64_t *off;      // top+1, natural layout (CSR of the memo)
    uint32_t *cardT;    // top, residue-major w.r.t. m = g_L (innermost leading generator)
    uint64_t *offT;     // top, residue-major
    uint64_t *chunk;    // gridDim scratch for the offset scan
    void *links;        // entries (u32 ring links or u64 row links), or nullptr
    uint64_t top;       // tables cover x < top
    uint64_t ltop;      // memo rows cover x < ltop <= top (topOfMemo; partial memo when < top)
    uint32_t m;         // g_L
    uint64_t R;         // rows per residue column = ceil(top / m)
    int d, L, t;
    int link_mode;      // 0 none, 1 u32 ring-relative, 2 u64 absolute
    uint64_t ring_mask;
    ProgGens P;         // closed form of the last two generators (S_{d-2})
    uint32_t *rows;     // memo rows (the last tail level is written by K2 stage B), or nullptr
    uint8_t lg_a[kMaxD], lg_b[kMaxD];   // fill mode 5: log2 lanes per x of the chain-list / block passes, per level
    uint64_t *trace;    // diagnostics: per-CTA phase timestamps [grid][16][2] (FZ_K1_TRACE), or nullptr
    uint64_t *C;        // COUNT cost tables C_0..C_{L-3} ((L-2) x top, L >= 3), or nullptr
    uint64_t beta;      // COUNT cost of one innermost run beyond its card lookups
    uint64_t gamma;     // COUNT cost of one outer prefix beyond its runs
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src)
{
    uint32_t lo = __shfl_sync(kFull, (uint32_t)v, src);
    uint32_t hi = __shfl_sync(kFull, (uint32_t)(v >> 32), src);
    return ((uint64_t)hi << 32) | lo;
}

__device__ __forceinline__ uint64_t shfl_up_u64(uint64_t v, int o)
{
    uint32_t lo = __shfl_up_sync(kFull, (uint32_t)v, o);
    uint32_t hi = __shfl_up_sync(kFull, (uint32_t)(v >> 32), o);
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

// Block-wide exclusive scan of one u64 per thread (blockDim multiple of 32).
// Returns the exclusive prefix; *total gets the block sum.  Uses sm[33].
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *sm, uint64_t *total)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    uint64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t u = shfl_up_u64(inc, o);
        if (lane >= o) inc += u;
    }
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint64_t w = lane < nwarps ? sm[lane] : 0;
        uint64_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t u = shfl_up_u64(wi, o);
            if (lane >= o) wi += u;
        }
        if (lane < nwarps) sm[lane] = wi - w;
        if (lane == 31) sm[32] = wi;
    }
    __syncthreads();
    const uint64_t res = sm[warp] + inc - v;
    *total = sm[32];
    __syncthreads();
    return res;
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
            __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

// Inclusive scan down one residue column c of a level:
//   dst[x] = src(x) + dst[x - g]  for x = c, c+g, c+2g, ... < N.   One CTA.  src is a table in memory
// or a closed form evaluated on the fly (the scans whose source level is closed run in phase 0).
// One block barrier per round: warp w takes the contiguous rows [w S, (w+1) S) of the column
// (S = ceil(rows / warps)), each lane E consecutive rows of them; warp-level scan, warp totals through
// shared memory, and every warp adds the totals of the warps before it itself (no serial
// second-level scan).  Columns longer than warps x 32 x kE rows take several rounds.
template <class Src>
__device__ void block_column_scan_w(Src src, uint64_t *dst, uint64_t N, uint64_t g, uint64_t c, uint64_t *sm)
{
    constexpr int kE = 4;
    const uint64_t rows = (N - c + g - 1) / g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint64_t per_round = (uint64_t)nwarps * 32 * kE;
    uint64_t carry = 0;
    for (uint64_t r0 = 0; r0 < rows; r0 += per_round) {
        const uint64_t rr = (rows - r0 < per_round) ? rows - r0 : per_round;
        const uint64_t S = (rr + nwarps - 1) / nwarps;           // rows per warp this round
        const uint64_t ws = r0 + (uint64_t)warp * S;             // first row of this warp
        const uint64_t we = (ws + S < r0 + rr) ? ws + S : r0 + rr;
        const uint64_t kb = ws + (uint64_t)lane * kE;
        uint64_t v[kE];
        uint64_t s = 0;
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const uint64_t k = kb + e;
            v[e] = k < we ? src(c + k * g) : 0;
            s += v[e];
        }
        uint64_t inc = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t u = shfl_up_u64(inc, o);
            if (lane >= o) inc += u;
        }
        if (lane == 31) sm[warp] = inc;
        __syncthreads();
        uint64_t before = (lane < warp) ? sm[lane] : 0;   // totals of the warps before this one
        uint64_t all = (lane < nwarps) ? sm[lane] : 0;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            before += __shfl_xor_sync(kFull, before, o);
            all += __shfl_xor_sync(kFull, all, o);
        }
        uint64_t run = carry + before + inc - s;
#pragma unroll
        for (int e = 0; e < kE; ++e) {
            const uint64_t k = kb + e;
            run += v[e];
            if (k < we) dst[c + k * g] = run;
        }
        carry += all;
        __syncthreads();   // sm reused by the next round / the caller
    }
}

__device__ void block_column_scan(const uint64_t *src, uint64_t *dst, uint64_t N, uint64_t g, uint64_t c, uint64_t *sm)
{
    block_column_scan_w([=](uint64_t x) { return __ldcg(src + x); }, dst, N, g, c, sm);
}

template <int T>
__device__ __forceinline__ void incr_word(uint32_t (&w)[T], int i)
{
#pragma unroll
    for (int j = 0; j < T; ++j) w[j] += (j == i) ? 1u : 0u;
}

// ------------------------------------------------------------ PTX helpers
// Programmatic dependent launch: wait for the preceding kernel of the stream (no-op without PDL).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// ... and let the next kernel of the stream be scheduled now (it still waits for this one's completion).
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ uint32_t lds32(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a)
{
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx_arrive(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

// 1-D bulk copy global -> shared (TMA engine), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// ---------------------------------------------------------------------- K3
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t nthreads)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Progress flags between the ring-fill workers and its helper warp: shared-memory atomics with
// acquire / release ordering (atomics, so compute-sanitizer racecheck sees the synchronisation).
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t *p)
{
    uint32_t v;
    asm volatile("atom.acquire.cta.shared::cta.or.b32 %0, [%1], 0;" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(uint32_t *p, uint32_t v)
{
    asm volatile("{\n\t.reg .b32 old;\n\tatom.release.cta.shared::cta.exch.b32 old, [%0], %1;\n\t}" ::"r"(smem_addr(p)),
                 "r"(v)
                 : "memory");
}

// Fill mode 1: one CTA runs the elementwise batches in order;
// inside a batch every row is independent (factorizationwise).
// Worker warps compute rows only in shared memory: the live window sits in a
// ring indexed by (row & mask); a row is ring[src] with one coordinate
// incremented, src / index from the u32 link (ring index | tail index << 27).
// Workers prefetch the next batch's links into registers, so a batch's
// dependent chain is ring LDS -> increment -> ring STS -> named barrier.
// The last warp is a TMA helper that never joins the workers' barrier: it
// bulk-loads the links CHB batches at a time (double-buffered, mbarrier
// completion) and bulk-stores finished batches from the ring to the global CSR,
// following the workers through a release/acquire progress counter; workers only
// wait for it when the ring would overwrite rows not yet stored (Q batches back).
// Shared memory: boff[nb+1] u32 | ring[RING*T] u32 | lbuf[2][chunk_words] u32 |
//                mbar[2] | done, stored (u32).
template <int T>
__global__ void __launch_bounds__(1024) k3_fill_ring(const uint64_t *__restrict__ off,
                                                      const uint32_t *__restrict__ links, uint32_t *rows,
                                                      uint64_t top, uint32_t b, uint32_t nb, uint32_t ring_rows,
                                                      uint32_t chunk_words, uint32_t chb, uint32_t Q)
{
    constexpr int RPT = 4;
    extern __shared__ __align__(16) uint32_t sh[];
    const uint32_t ring_mask = ring_rows - 1;
    uint32_t *boff = sh;                                            // nb + 1 entries
    uint32_t *ring = sh + ((nb + 1 + 3) & ~3u);
    uint32_t *lbuf = ring + ring_rows * T;
    uint64_t *mbar = reinterpret_cast<uint64_t *>(lbuf + 2 * chunk_words);
    uint32_t *done = reinterpret_cast<uint32_t *>(mbar + 2);
    uint32_t *stored = done + 1;
    const uint32_t tid = threadIdx.x;
    const uint32_t nw = blockDim.x - 32;                           // worker threads
    const bool helper = tid >= nw;
    const uint32_t nchunks = (nb + chb - 1) / chb;
    const uint64_t ring_bytes = (uint64_t)ring_rows * T * 4;
    for (uint32_t k = tid; k <= nb; k += blockDim.x) {
        const uint64_t x = (uint64_t)k * b;
        boff[k] = (uint32_t)__ldg(off + (x < top ? x : top));
    }
    if (tid == 0) {
        mbar_init(mbar + 0, 1);
        mbar_init(mbar + 1, 1);
        *done = 0;
        *stored = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto chunk_base = [&](uint32_t c) { return boff[c * chb] & ~3u; };

    if (helper) {
        if ((tid & 31) != 0) return;
        auto load_chunk = [&](uint32_t c) {
            const uint32_t k1 = (c + 1) * chb < nb ? (c + 1) * chb : nb;
            const uint32_t a0 = chunk_base(c), a1 = (boff[k1] + 3u) & ~3u;
            const uint32_t bytes = (a1 - a0) * 4u;
            fence_proxy_async();
            mbar_expect_tx_arrive(mbar + (c & 1), bytes);
            if (bytes) bulk_g2s(lbuf + (c & 1) * chunk_words, links + a0, bytes, mbar + (c & 1));
        };
        // bytes [B0, B1) of the CSR rows <- ring bytes B0 mod ring_bytes (split at the wrap)
        auto store_bytes = [&](uint64_t B0, uint64_t B1) {
            while (B0 < B1) {
                const uint64_t rb = B0 % ring_bytes;
                uint64_t len = B1 - B0;
                if (rb + len > ring_bytes) len = ring_bytes - rb;
                bulk_s2g(reinterpret_cast<char *>(rows) + B0, reinterpret_cast<char *>(ring) + rb, (uint32_t)len);
                B0 += len;
            }
        };
        load_chunk(0);
        uint32_t next_chunk = 1, j = 0;
        while (j < nb) {
            const uint32_t d = ld_acquire_cta(done);
            if (next_chunk < nchunks && d >= (next_chunk - 1) * chb) {   // workers are in chunk next_chunk-1
                load_chunk(next_chunk);
                ++next_chunk;
            }
            if (d > j) {
                fence_proxy_async();
                const uint64_t B0 = ((uint64_t)boff[j] * T * 4) & ~15ull;
                uint64_t B1 = (uint64_t)boff[d] * T * 4;
                B1 = (d == nb) ? ((B1 + 15) & ~15ull) : (B1 & ~15ull);
                store_bytes(B0, B1);
                bulk_commit();
                bulk_wait_read<0>();
                st_release_cta(stored, d);
                j = d;
            } else {
                __nanosleep(20);
            }
        }
        bulk_wait_all();
        return;
    }

    // ------------------------------------------------------------- workers
    auto wait_chunk = [&](uint32_t c) { mbar_wait(mbar + (c & 1), (c >> 1) & 1); };
    wait_chunk(0);
    uint32_t lnk[RPT];
    uint32_t R0 = boff[0], R1 = boff[1];
    const uint32_t *lk = lbuf - chunk_base(0);
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const uint32_t r = R0 + tid + q * nw;
        lnk[q] = r < R1 ? lk[r] : 0u;
    }
    uint32_t c = 0, kk = 0;
    for (uint32_t k = 0; k < nb; ++k) {
        // ring-reuse guard: the ring holds batches k-Q-1..k (+ one 16-B granule), so batch k may only
        // overwrite rows once every batch before k-Q-1 has been read by its bulk store
        if (tid == 0 && k > Q + 1) {
            while (ld_acquire_cta(stored) + Q + 1 < k) __nanosleep(20);
        }
        if (k > 0) named_bar(1, nw);
        if (tid == 0 && k > 0) st_release_cta(done, k);
        // next batch's boundaries and links (independent of this batch's results)
        const uint32_t Rn = R1, Rn1 = (k + 1 < nb) ? boff[k + 2] : R1;
        uint32_t kk1 = kk + 1, c1 = c;
        if (kk1 == chb) {
            kk1 = 0;
            ++c1;
            if (c1 < nchunks) wait_chunk(c1);
        }
        const uint32_t *lk1 = (c1 == c) ? lk : lbuf + (c1 & 1) * chunk_words - chunk_base(c1 < nchunks ? c1 : 0);
        uint32_t nl[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t r = Rn + tid + q * nw;
            nl[q] = r < Rn1 ? lk1[r] : 0u;
        }
        auto row = [&](uint32_t r, uint32_t link) {
            uint32_t w[T];
            if (link == kZeroLink32) {
#pragma unroll
                for (int j = 0; j < T; ++j) w[j] = 0;
            } else {
                const uint32_t *s = ring + (link & ((1u << kRingIdxBits) - 1)) * T;
                if constexpr (T == 2) {
                    uint2 v = *reinterpret_cast<const uint2 *>(s);
                    w[0] = v.x; w[1] = v.y;
                } else if constexpr (T == 4) {
                    uint4 v = *reinterpret_cast<const uint4 *>(s);
                    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
                } else {
#pragma unroll
                    for (int j = 0; j < T; ++j) w[j] = s[j];
                }
                incr_word<T>(w, (int)(link >> kRingIdxBits));
            }
            uint32_t *dr = ring + (r & ring_mask) * T;
            if constexpr (T == 2) {
                *reinterpret_cast<uint2 *>(dr) = make_uint2(w[0], w[1]);
            } else if constexpr (T == 4) {
                *reinterpret_cast<uint4 *>(dr) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
#pragma unroll
                for (int j = 0; j < T; ++j) dr[j] = w[j];
            }
        };
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const uint32_t r = R0 + tid + q * nw;
            if (r < R1) row(r, lnk[q]);
        }
        for (uint32_t r = R0 + tid + RPT * nw; r < R1; r += nw) row(r, lk[r]);   // rare: oversized batch
        R0 = Rn;
        R1 = Rn1;
        kk = kk1;
        c = c1;
        lk = lk1;
#pragma unroll
        for (int q = 0; q < RPT; ++q) lnk[q] = nl[q];
    }
    named_bar(1, nw);
    if (tid == 0) st_release_cta(done, nb);
}

// ------------------------------------------------------------- K3 chains
// Fill mode 4 (default): the same copy-increment tasks as PAPER.md:171-192,
// scheduled one tail dimension at a time.  With tail index i (0-based) and
// h = h_i, block i of Z(x) is
//     incr_i( Z_{>=i}(x - h) ) = incr_i( block_i(Z(x - h)) ++ Z_{>=i+1}(x - h) )
// (PAPER.md:77-88 with PAPER.md:83-85), so once blocks i+1.. exist (earlier
// passes), block i only depends on block i of x - h: the x values of one
// residue class r mod h form an independent chain, and the elementwise batch of
// pass i is {one x per residue} (size h_i >= min h).  Each
// chain is one warp; the block state lives in registers (K slots of 32 rows) or in
// shared memory (K = 0), each step adds 1 to coordinate i of every row and appends
// the suffix Z_{>=i+1}(x - h) (incremented), then stores the block.  No CTA or
// grid barrier inside a pass.  Per 32-step group the lanes prefetch the step
// metadata from the count tables and stage the suffix rows in shared memory with
// cp.async.

// last tail dimension: block t-1 of Z(x) = [(0,..,0, x/h)] if h | x (x = 0 gives Memo[0] = [0])
template <int T>
__device__ __forceinline__ void last_level_body(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                                uint32_t *rows, uint64_t top, uint64_t ltop, int L, uint32_t h,
                                                uint64_t gt, uint64_t ng)
{
    const uint64_t *Sl = S + (uint64_t)(L + T - 1) * top;
    for (uint64_t x = gt; x < ltop; x += ng) {
        if (x % h) continue;
        const uint64_t dst = __ldcg(off + x + 1) - __ldcg(Sl + x);
        uint32_t *o = rows + dst * T;
#pragma unroll
        for (int j = 0; j < T - 1; ++j) o[j] = 0;
        o[T - 1] = (uint32_t)(x / h);
    }
}

template <int T>
__global__ void __launch_bounds__(256) k3_last_level(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                                      uint32_t *rows, uint64_t top, uint64_t ltop, int L, uint32_t h)
{
    const uint64_t *Sl = S + (uint64_t)(L + T - 1) * top;
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < ltop; x += (uint64_t)gridDim.x * blockDim.x) {
        if (x % h) continue;
        const uint64_t dst = __ldg(off + x + 1) - __ldg(Sl + x);
        uint32_t *o = rows + dst * T;
#pragma unroll
        for (int j = 0; j < T - 1; ++j) o[j] = 0;
        o[T - 1] = (uint32_t)(x / h);
    }
}

__device__ __forceinline__ void cp_async4(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

constexpr int kChainStage = 512;   // staged suffix rows per 32-position group
constexpr int kMetaSlots = 6;      // metadata ring (groups g-1 .. g+4 live)
constexpr int kStageSlots = 3;     // suffix staging ring (groups g .. g+2 live)

__device__ __forceinline__ void cp_async8(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// One CTA per residue chain r of tail level i (h = h_i), P = blockDim/32 warps.
// Chain position j: x_j = r + j h.  block_i(Z(x_{j+1})) = incr_i(block_i(Z(x_j)) ++ suffix(x_j)),
// suffix(x) = Z_{>=i+1}(x) (rows from earlier passes).  Unrolled, block_i(Z(x_{j+1})) is every
// suffix row appended at positions j' <= j, incremented (j + 1 - j') times, in append order.  The
// state is therefore an append-only list: a row appended at position j' is kept as row - j' e_i
// and read back as + (j + 1) e_i.  Warp 0 appends each 32-position group; after one CTA barrier
// every warp stores the blocks of its share of the group's positions (j = w mod P).  Warp 0 keeps
// a cp.async pipeline: per-position table values four groups ahead (shared ring), suffix rows two
// groups ahead (shared staging ring), so no step waits on global memory.
// Shared memory: buf[cap*T] | stage[3][kChainStage*T] | meta[6][4][32] u64 | desc dst[2][32] u64, rows[2][32] u32.
// Needs P >= 2 (warp 0 produces, warps 1.. store).
template <int T>
__global__ void __launch_bounds__(512) k3_chain(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                                 uint32_t *rows, uint64_t top, int L, int i, uint32_t h, uint32_t cap)
{
    extern __shared__ __align__(16) uint32_t csh[];
    uint32_t *buf = csh;
    uint32_t *stage = csh + (((uint64_t)cap * T + 3) & ~3ull);
    uint64_t *meta = reinterpret_cast<uint64_t *>(stage + kStageSlots * kChainStage * T);   // [slot][field][lane]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, P = blockDim.x >> 5;
    const uint64_t r = blockIdx.x;
    if (r + h >= top) return;
    const uint64_t *Si = S + (uint64_t)(L + i) * top;
    const uint64_t *Si1 = S + (uint64_t)(L + i + 1) * top;
    const uint64_t npos = (top - 1 - r) / h;            // positions j < npos have x_{j+1} < top
    const uint64_t ngroups = (npos + 31) / 32;
    uint32_t inc[T];
#pragma unroll
    for (int j = 0; j < T; ++j) inc[j] = (j == i) ? 1u : 0u;
    // field 0: ns = S_{i+1}[x]; 1: o1 = off[x+1]; 2: on = off[xn+1]; 3: sn = S_i[xn]
    auto M = [&](uint64_t g, int f) -> uint64_t * { return meta + ((g % kMetaSlots) * 4 + f) * 32; };
    auto meta_issue = [&](uint64_t g) {   // warp 0
        const uint64_t j = g * 32 + lane;
        if (j < npos) {
            const uint64_t x = r + j * h, xn = x + h;
            cp_async8(M(g, 0) + lane, Si1 + x);
            cp_async8(M(g, 1) + lane, off + x + 1);
            cp_async8(M(g, 2) + lane, off + xn + 1);
            cp_async8(M(g, 3) + lane, Si + xn);
        } else {
            M(g, 0)[lane] = 0;
            M(g, 1)[lane] = 0;
            M(g, 2)[lane] = 0;
            M(g, 3)[lane] = 0;
        }
    };
    auto scan = [&](uint32_t v) {
        uint32_t s2 = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t u = __shfl_up_sync(kFull, s2, o);
            if (lane >= o) s2 += u;
        }
        return s2 - v;
    };
    auto stage_issue = [&](uint64_t g) {   // warp 0; metadata of group g is complete
        uint32_t *sb = stage + (g % kStageSlots) * kChainStage * T;
        const uint32_t ns = (uint32_t)M(g, 0)[lane];
        const uint64_t so = M(g, 1)[lane] - ns;
        const uint32_t ex = scan(ns);
        for (unsigned msk = __ballot_sync(kFull, ns > 0); msk; msk &= msk - 1) {
            const int l = __ffs(msk) - 1;
            const uint32_t nl = __shfl_sync(kFull, ns, l);
            const uint32_t el = __shfl_sync(kFull, ex, l);
            const uint64_t sl = shfl_u64(so, l);
            for (uint32_t j = lane; j < nl && el + j < (uint32_t)kChainStage; j += 32)
#pragma unroll
                for (int w = 0; w < T; ++w) cp_async4(sb + (el + j) * T + w, rows + (sl + j) * T + w);
        }
    };
    // store descriptors of a group: block start (u64), rows, increment count, double-buffered
    uint64_t *ddst = meta + kMetaSlots * 4 * 32;                     // [2][32]
    uint32_t *dnr = reinterpret_cast<uint32_t *>(ddst + 2 * 32);     // [2][32]
    if (warp == 0) {   // prologue: metadata of groups 0..3, then suffix rows of groups 0, 1
        for (uint64_t g = 0; g < 4; ++g) meta_issue(g);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
        stage_issue(0);
        stage_issue(1);
        cp_async_commit();
        cp_async_wait<0>();
        __syncwarp();
    }
    uint32_t nbase = 0;                                  // rows appended before the producer's group
    // iteration g: warp 0 appends group g and publishes its store descriptors; warps 1..P-1 store
    // group g-1 (appended one iteration earlier; the list is append-only, so no conflict)
    for (uint64_t g = 0; g <= ngroups; ++g) {
        if (warp == 0) {
            if (g < ngroups) {
                cp_async_wait<1>();   // everything issued up to iteration g-2: meta(g+2), stage(g)
                __syncwarp();
                meta_issue(g + 4);
                stage_issue(g + 2);
                cp_async_commit();
                // append group g: a row appended at position j' is kept as row - j' e_i
                const uint32_t *sb = stage + (g % kStageSlots) * kChainStage * T;
                const uint32_t ns = (uint32_t)M(g, 0)[lane];
                const uint64_t so = M(g, 1)[lane] - ns;
                const uint32_t ex = scan(ns);
                for (unsigned msk = __ballot_sync(kFull, ns > 0); msk; msk &= msk - 1) {
                    const int l = __ffs(msk) - 1;
                    const uint32_t nl = __shfl_sync(kFull, ns, l);
                    const uint32_t el = __shfl_sync(kFull, ex, l);
                    const uint64_t sl = shfl_u64(so, l);
                    const uint32_t jabs = (uint32_t)(g * 32 + l);
                    for (uint32_t q = lane; q < nl; q += 32) {
#pragma unroll
                        for (int w = 0; w < T; ++w) {
                            const uint32_t v =
                                (el + q < (uint32_t)kChainStage) ? sb[(el + q) * T + w] : rows[(sl + q) * T + w];
                            buf[(nbase + el + q) * T + w] = v - jabs * inc[w];
                        }
                    }
                }
                // block_i(Z(x_{j+1})) = first nbase + ex + ns rows (+ (j + 1) e_i), stored at on - sn
                ddst[(g & 1) * 32 + lane] = M(g, 2)[lane] - M(g, 3)[lane];
                dnr[(g & 1) * 32 + lane] = nbase + ex + ns;
                nbase += __shfl_sync(kFull, ex + ns, 31);
            }
        } else if (g > 0) {
            const uint64_t gp = g - 1;
            const uint64_t *dd = ddst + (gp & 1) * 32;
            const uint32_t *dn = dnr + (gp & 1) * 32;
            const int Pc = P - 1;
            const uint32_t first = (uint32_t)((Pc - (int)((gp * 32) % Pc) + (warp - 1)) % Pc);
            for (uint32_t l = first; l < 32 && gp * 32 + l < npos; l += Pc) {
                const uint64_t d = dd[l];
                const uint32_t nr = dn[l];
                const uint32_t c = (uint32_t)(gp * 32 + l + 1);
                for (uint32_t q = lane; q < nr; q += 32) {
                    uint32_t v[T];
#pragma unroll
                    for (int w = 0; w < T; ++w) v[w] = buf[q * T + w] + c * inc[w];
                    uint32_t *o = rows + (d + q) * T;
                    if constexpr (T == 2) {
                        *reinterpret_cast<uint2 *>(o) = make_uint2(v[0], v[1]);
                    } else if constexpr (T == 4) {
                        *reinterpret_cast<uint4 *>(o) = make_uint4(v[0], v[1], v[2], v[3]);
                    } else {
#pragma unroll
                        for (int w = 0; w < T; ++w) o[w] = v[w];
                    }
                }
            }
        }
        __syncthreads();
    }
    if (warp == 0) cp_async_wait<0>();
}

// ------------------------------------------------------------- K3 scan
// Fill mode 5 (default): the chain recurrence of mode 4 evaluated in its unrolled form.
// For chain r of level i (h = h_i), the lazy list of the chain holds, at positions
// [S_i[x] - S_{i+1}[x], S_i[x]), the suffix Z_{>=i+1}(x) of x = r + j h, each row minus j e_i;
// its prefix of length S_i[x] is Z_{>=i}(x) (lazy).  Since S_i[x] - S_{i+1}[x] = S_i[x - h]
// (PAPER.md:163-166 bookkeeping, suffix-table recurrence) the segments tile the list, so
//   phase A: every x writes its suffix rows into its chain list       (parallel over x)
//   phase B: block_i(Z(x)) = list prefix of length S_i[x] - S_{i+1}[x], + (x div h) e_i
//            (= incr_i applied x div h - j' times to the row appended at position j')
// -- the same copy-and-increment results, with no dependency between x values inside a pass.
// Rows are copied by groups of G = 2^lg lanes (one group per x; lg chosen per level by the host from
// the level's mean rows per x, so the common few-row blocks do not idle a whole warp), U rows per lane
// loaded before any is stored (U loads in flight instead of one dependent round trip per row).
template <int T>
__device__ __forceinline__ void copy_incr(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst, uint32_t n,
                                          uint32_t lane, uint32_t G, int i, uint32_t delta)
{
    constexpr int U = 4;
    auto ld = [&](uint32_t k, uint32_t (&v)[T]) {
        if constexpr (T == 2) {
            const uint2 w = __ldcg(reinterpret_cast<const uint2 *>(src) + k);
            v[0] = w.x;
            v[1] = w.y;
        } else if constexpr (T == 4) {
            const uint4 w = __ldcg(reinterpret_cast<const uint4 *>(src) + k);
            v[0] = w.x;
            v[1] = w.y;
            v[2] = w.z;
            v[3] = w.w;
        } else {
#pragma unroll
            for (int w = 0; w < T; ++w) v[w] = __ldcg(src + (uint64_t)k * T + w);
        }
    };
    auto st = [&](uint32_t k, uint32_t (&v)[T]) {
#pragma unroll
        for (int w = 0; w < T; ++w) v[w] += (w == i) ? delta : 0u;
        if constexpr (T == 2) {
            reinterpret_cast<uint2 *>(dst)[k] = make_uint2(v[0], v[1]);
        } else if constexpr (T == 4) {
            reinterpret_cast<uint4 *>(dst)[k] = make_uint4(v[0], v[1], v[2], v[3]);
        } else {
#pragma unroll
            for (int w = 0; w < T; ++w) dst[(uint64_t)k * T + w] = v[w];
        }
    };
    for (uint32_t k = lane; k < n; k += U * G) {   // one batch: up to U rows per lane, loads before stores
        uint32_t v[U][T];
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u * G < n) ld(k + u * G, v[u]);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (k + u * G < n) st(k + u * G, v[u]);
    }
}

// gg / ng: this lane's group index and the number of groups; lane: index within the group of G lanes.
template <int T>
__device__ __forceinline__ void scan_a_body(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                            const uint32_t *rows, uint32_t *list, uint64_t cap_list, uint64_t top,
                                            uint64_t ltop, int L, int i, uint32_t h, uint64_t gg, uint64_t ng,
                                            uint32_t lane, uint32_t G)
{
    const uint64_t *Si = S + (uint64_t)(L + i) * top, *Si1 = Si + top;
    // rounds of ng consecutive x, assigned in alternating direction (block sizes grow with x)
    uint64_t k = 0, x = gg;
    if (x + h >= ltop) return;
    uint64_t ns = __ldg(Si1 + x), o1 = __ldg(off + x + 1), si = __ldg(Si + x);
    for (;;) {   // the next x's header is loaded before this x's rows are copied
        ++k;
        const uint64_t xn = k * ng + ((k & 1) ? ng - 1 - gg : gg);
        const bool more = xn + h < ltop;
        uint64_t nsn = 0, o1n = 0, sin = 0;
        if (more) {
            nsn = __ldg(Si1 + xn);
            o1n = __ldg(off + xn + 1);
            sin = __ldg(Si + xn);
        }
        if (ns) {
            const uint64_t so = o1 - ns, base = si - ns;
            const uint32_t j = (uint32_t)x / h, r = (uint32_t)x - j * h;   // x < top <= 2^28
            copy_incr<T>(rows + so * T, list + ((uint64_t)r * cap_list + base) * T, (uint32_t)ns, lane, G, i, 0u - j);
        }
        if (!more) break;
        x = xn;
        ns = nsn;
        o1 = o1n;
        si = sin;
    }
}

template <int T>
__device__ __forceinline__ void scan_b_body(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                            uint32_t *rows, const uint32_t *list, uint64_t cap_list, uint64_t top,
                                            uint64_t ltop, int L, int i, uint32_t h, uint64_t gg, uint64_t ng,
                                            uint32_t lane, uint32_t G)
{
    const uint64_t *Si = S + (uint64_t)(L + i) * top, *Si1 = Si + top;
    uint64_t k = 0, x = h + gg;
    if (x >= ltop) return;
    uint64_t si = __ldg(Si + x), s1 = __ldg(Si1 + x), o1 = __ldg(off + x + 1);
    for (;;) {   // the next x's header is loaded before this x's rows are copied
        ++k;
        const uint64_t xn = h + k * ng + ((k & 1) ? ng - 1 - gg : gg);
        const bool more = xn < ltop;
        uint64_t sin = 0, s1n = 0, o1n = 0;
        if (more) {
            sin = __ldg(Si + xn);
            s1n = __ldg(Si1 + xn);
            o1n = __ldg(off + xn + 1);
        }
        const uint64_t nb = si - s1;
        if (nb) {
            const uint32_t c = (uint32_t)x / h, r = (uint32_t)x - c * h;
            copy_incr<T>(list + (uint64_t)r * cap_list * T, rows + (o1 - si) * T, (uint32_t)nb, lane, G, i, c);
        }
        if (!more) break;
        x = xn;
        si = sin;
        s1 = s1n;
        o1 = o1n;
    }
}

template <int T>
__global__ void __launch_bounds__(256) k3_scan_a(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                                  const uint32_t *rows, uint32_t *list, uint64_t cap_list, uint64_t top,
                                                  uint64_t ltop, int L, int i, uint32_t h, int lg)
{
    scan_a_body<T>(S, off, rows, list, cap_list, top, ltop, L, i, h, (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> lg,
                   ((uint64_t)gridDim.x * blockDim.x) >> lg, threadIdx.x & ((1u << lg) - 1), 1u << lg);
}

template <int T>
__global__ void __launch_bounds__(256) k3_scan_b(const uint64_t *__restrict__ S, const uint64_t *__restrict__ off,
                                                  uint32_t *rows, const uint32_t *list, uint64_t cap_list, uint64_t top,
                                                  uint64_t ltop, int L, int i, uint32_t h, int lg)
{
    scan_b_body<T>(S, off, rows, list, cap_list, top, ltop, L, i, h, (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> lg,
                   ((uint64_t)gridDim.x * blockDim.x) >> lg, threadIdx.x & ((1u << lg) - 1), 1u << lg);
}

// ------------------------------------------------------------------ K1 + K2 (+ K3 mode 5)
// One cooperative launch (all CTAs co-resident), phases separated by grid barriers.  Phase 0 writes
// the closed forms: S_d[x] = [x = 0], S_{d-1}[x] = [g_{d-1} | x], S_{d-2}[x] = |Z(x; g_{d-2}, g_{d-1})|
// (prog_count), W_L[x] = 1, W_{L-1}[x] = floor(x / g_{L-1}) + 1.  Phase p >= 0 scans S_{d-3-p} and
// W_{L-2-p} (column scans, one CTA per residue class; in phase 0 their sources are the closed forms,
// evaluated on the fly).  The CSR scan of card = S_L (off, residue-major cardT / offT) takes two
// phases: chunk sums (stage A) as soon as card is final — phase 0 when t <= 2, since card is then a
// closed form — and the scan (stage B) one phase later, which also writes the last tail level of every
// memo block (the row (0,..,0, x / g_{d-1}) at off[x+1] - 1 when g_{d-1} | x).  With T >= 2 (fill
// mode 5 fused) the copy-increment passes follow, one tail level per two phases (chain lists, then
// blocks), overlapping the leading-level scans still in flight.  The column scans take the leading
// CTAs; stage A / B chunks, the fill passes and the elementwise closed forms go to the other CTAs
// when the scans leave at least half the grid free.
template <int T>
__device__ __forceinline__ void k1_body(const Gens &G, const Tables &tb, unsigned int *counter, unsigned int &target,
                                        uint64_t *sm, uint32_t *list = nullptr, uint64_t cap_list = 0)
{
    const uint64_t top = tb.top, ltop = tb.ltop;
    const int d = tb.d, L = tb.L, t = d - L;
    const uint32_t gd1 = G.g[d - 1];
    const uint64_t *card = tb.S + (uint64_t)L * top;
    auto closed_card = [&](uint64_t x) -> uint64_t {   // card = S_L when t <= 2
        if (L == d) return x == 0;
        if (L == d - 1) return x % gd1 == 0;
        return prog_count(tb.P, (uint32_t)x);
    };
    const bool card_closed = t <= 2;
    const int pa = card_closed ? 0 : t - 2;   // stage A: the phase after S_L (scanned in phase t-3) is final
    const int pb = pa + 1;                    // stage B (+ last tail level)
    const int lastS = d >= 3 ? d - 3 : -1, lastW = L >= 2 ? L - 2 : -1;
    const int nfill = (T >= 2) ? 2 * (T - 1) : 0;
    int last = pb + nfill;
    if (lastS > last) last = lastS;
    if (lastW > last) last = lastW;
    // column-scan CTAs of phase p (leading CTAs); the rest of the grid does the other work of p
    auto ncols = [&](int p) -> uint64_t {
        const int i = d - 3 - p, j = L - 2 - p, jc = L - 2 - p;
        uint64_t c = 0;
        if (p >= 0 && i >= 0) c += G.g[i] < top ? G.g[i] : top;
        if (p >= 0 && j >= 0) c += G.g[j] < top ? G.g[j] : top;
        if (tb.C && p >= 1 && jc >= 0) c += G.g[jc] < top ? G.g[jc] : top;
        return c;
    };
    auto free0 = [&](int p) -> uint32_t {   // first CTA free of column scans in phase p (0: share the grid)
        const uint64_t c = ncols(p);
        return 2 * c <= gridDim.x ? (uint32_t)c : 0u;
    };
    // stage A / B chunks over the CTAs free in phase pb
    const uint32_t b0 = free0(pb), nB = gridDim.x - b0;
    const bool has_chunk = blockIdx.x >= b0;
    const uint32_t cb = has_chunk ? blockIdx.x - b0 : 0;
    const uint64_t CH = (top + nB - 1) / nB;
    const uint64_t c0 = has_chunk ? (uint64_t)cb * CH : 0;
    const uint64_t c1 = has_chunk ? ((c0 + CH < top) ? c0 + CH : top) : 0;
    auto trace = [&](int p, int k) {   // diagnostics (FZ_K1_TRACE): per-CTA phase timestamps
        if (tb.trace && threadIdx.x == 0 && p < 16) {
            uint64_t t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            tb.trace[((uint64_t)blockIdx.x * 16 + p) * 2 + k] = t;
        }
    };
    for (int p = 0; p <= last; ++p) {
        if (p > 0) {
            trace(p - 1, 1);
            grid_barrier(counter, target);
        }
        trace(p, 0);
        if (p == last) griddep_launch();   // PDL: the planner may be scheduled during the last phase
        {   // column scans of S_{d-3-p} and W_{L-2-p}
            const int i = d - 3 - p, j = L - 2 - p;
            const uint64_t gi = i >= 0 ? G.g[i] : 1;
            const uint64_t ncolS = i >= 0 ? (gi < top ? gi : top) : 0;
            const uint64_t gj = j >= 0 ? G.g[j] : 1;
            const uint64_t ncolW = j >= 0 ? (gj < top ? gj : top) : 0;
            const uint64_t gw1 = L >= 1 ? G.g[L - 1] : 1;
            // COUNT cost tables (pair walk): C_{L-2}[x] = W_{L-2}[x] + beta (x / g_{L-2} + 1) + gamma
            // (each innermost run costs its lookups plus beta, each outer prefix gamma more), C_jc = column scan
            // of C_{jc+1} by g_jc,
            // one phase behind W (C_{L-3} in phase 1 reads the W_{L-2} of phase 0)
            const int jc = L - 2 - p;
            const uint64_t gc = (tb.C && p >= 1 && jc >= 0) ? G.g[jc] : 1;
            const uint64_t ncolC = (tb.C && p >= 1 && jc >= 0) ? (gc < top ? gc : top) : 0;
            for (uint64_t c = blockIdx.x; c < ncolS + ncolW + ncolC; c += gridDim.x) {
                if (c >= ncolS + ncolW) {
                    uint64_t *dst = tb.C + (uint64_t)jc * top;
                    if (jc + 1 == L - 2) {
                        const uint64_t *W2 = tb.W + (uint64_t)(L - 2) * top;
                        const uint64_t g2 = G.g[L - 2], beta = tb.beta, gamma = tb.gamma;
                        block_column_scan_w([=](uint64_t x) { return __ldcg(W2 + x) + beta * (x / g2 + 1) + gamma; },
                                            dst, top, gc, c - ncolS - ncolW, sm);
                    } else {
                        block_column_scan(tb.C + (uint64_t)(jc + 1) * top, dst, top, gc, c - ncolS - ncolW, sm);
                    }
                } else if (c < ncolS) {
                    uint64_t *dst = tb.S + (uint64_t)i * top;
                    if (p == 0)
                        block_column_scan_w([&](uint64_t x) { return prog_count(tb.P, (uint32_t)x); }, dst, top, gi,
                                            c, sm);
                    else
                        block_column_scan(tb.S + (uint64_t)(i + 1) * top, dst, top, gi, c, sm);
                } else {
                    uint64_t *dst = tb.W + (uint64_t)j * top;
                    if (p == 0)
                        block_column_scan_w([&](uint64_t x) { return x / gw1 + 1; }, dst, top, gj, c - ncolS, sm);
                    else
                        block_column_scan(tb.W + (uint64_t)(j + 1) * top, dst, top, gj, c - ncolS, sm);
                }
            }
        }
        if (p == 0) {   // elementwise closed forms, from the last CTA down (the leading CTAs scan columns)
            const uint64_t gl = L > 0 ? G.g[L - 1] : 1;
            const uint64_t gtr = (gridDim.x - 1 - blockIdx.x) * (uint64_t)blockDim.x + threadIdx.x;
            const uint64_t ng = (uint64_t)gridDim.x * blockDim.x;
            for (uint64_t x = gtr; x < top; x += ng) {
                tb.S[(uint64_t)d * top + x] = (x == 0) ? 1ull : 0ull;
                tb.S[(uint64_t)(d - 1) * top + x] = (x % gd1 == 0) ? 1ull : 0ull;
                if (d >= 2) tb.S[(uint64_t)(d - 2) * top + x] = prog_count(tb.P, (uint32_t)x);
                tb.W[(uint64_t)L * top + x] = 1ull;
                if (L > 0) tb.W[(uint64_t)(L - 1) * top + x] = x / gl + 1;
            }
        }
        if (p == pa && has_chunk) {   // K2 stage A: chunk sums of card (memo rows only: x < ltop)
            uint64_t s = 0;
            for (uint64_t x = c0 + threadIdx.x; x < c1 && x < ltop; x += blockDim.x)
                s += card_closed ? closed_card(x) : __ldcg(card + x);
            uint64_t tot;
            block_excl_scan(s, sm, &tot);
            if (threadIdx.x == 0) tb.chunk[cb] = tot;
        }
        if (p == pb && has_chunk) {   // K2 stage B: off = exclusive scan of card; cardT / offT; last tail level
            uint64_t pre = 0;
            for (unsigned b = threadIdx.x; b < cb; b += blockDim.x) pre += __ldcg(tb.chunk + b);
            uint64_t tot;
            block_excl_scan(pre, sm, &tot);
            pre = tot;
            const uint64_t m = tb.m;
            for (uint64_t xb = c0; xb < c1; xb += blockDim.x) {
                const uint64_t x = xb + threadIdx.x;
                const uint64_t c = x < c1 ? __ldcg(card + x) : 0;
                const uint64_t v = x < ltop ? c : 0;   // CSR over the memo's rows only (x < ltop)
                uint64_t t2;
                const uint64_t ex = pre + block_excl_scan(v, sm, &t2);
                if (x < c1) {
                    tb.off[x] = ex;
                    const uint64_t ti = (x % m) * tb.R + x / m;
                    tb.cardT[ti] = (uint32_t)c;
                    tb.offT[ti] = ex;
                    if (x + 1 == top) tb.off[top] = ex + v;
                    if (tb.rows && t >= 1 && x < ltop && x % gd1 == 0) {   // block t-1 of Z(x): [(0,..,0, x/h)]
                        uint32_t *o = tb.rows + (ex + v - 1) * (uint64_t)t;
                        for (int w = 0; w < t - 1; ++w) o[w] = 0;
                        o[t - 1] = (uint32_t)(x / gd1);
                    }
                }
                pre += t2;
            }
        }
        if constexpr (T >= 2) {   // fill mode 5: level i = T-2 .. 0, chain lists then blocks
            if (p > pb && p <= pb + nfill) {
                const int k = p - pb - 1, i = T - 2 - k / 2;
                const uint32_t h = G.g[L + i];
                const uint32_t f0 = free0(p);
                if (blockIdx.x >= f0) {
                    const uint64_t gt = (blockIdx.x - f0) * (uint64_t)blockDim.x + threadIdx.x;
                    const uint64_t ng = (uint64_t)(gridDim.x - f0) * blockDim.x;
                    const int lg = (k % 2 == 0) ? tb.lg_a[i] : tb.lg_b[i];
                    const uint32_t lane = (uint32_t)threadIdx.x & ((1u << lg) - 1);
                    if (k % 2 == 0)
                        scan_a_body<T>(tb.S, tb.off, tb.rows, list, cap_list, top, ltop, L, i, h, gt >> lg, ng >> lg,
                                       lane, 1u << lg);
                    else
                        scan_b_body<T>(tb.S, tb.off, tb.rows, list, cap_list, top, ltop, L, i, h, gt >> lg, ng >> lg,
                                       lane, 1u << lg);
                }
            }
        }
    }
    trace(last, 1);
}

__global__ void __launch_bounds__(1024) k1_tables(Gens G, Tables tb, unsigned int *counter)
{
    __shared__ uint64_t sm[40];
    unsigned int target = 0;
    k1_body<0>(G, tb, counter, target, sm);
    if (tb.link_mode == 0) return;
    grid_barrier(counter, target);
    const uint64_t top = tb.top;
    const int L = tb.L, t = tb.t;
    const uint64_t gt = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t ng = (uint64_t)gridDim.x * blockDim.x;
    // links: row q of Z(x; tail) lies in block i (0-based tail index) with start
    // card[x] - S_{L+i}[x] ("beginning index of Z_{>=i}"); it is
    // incr_i of row off[y+1] - S_{L+i}[y] + k of Z(y), y = x - g_{L+i}, k = q - start.
    const int lane = threadIdx.x & 31;
    const uint64_t gw = gt >> 5, nw = ng >> 5;
    if (gw == 0 && lane == 0) {
        if (tb.link_mode == 1) ((uint32_t *)tb.links)[0] = kZeroLink32;
        else ((uint64_t *)tb.links)[0] = ~0ull;
    }
    for (uint64_t x = 1 + gw; x < top; x += nw) {
        const uint64_t base = __ldcg(tb.off + x);
        const uint64_t c = __ldcg(tb.off + x + 1) - base;
        for (uint64_t q = lane; q < c; q += 32) {
            int i = 0;
            uint64_t st = 0;
            for (int jj = t - 1; jj >= 1; --jj) {
                uint64_t sj = c - __ldcg(tb.S + (uint64_t)(L + jj) * top + x);
                if (sj <= q) { i = jj; st = sj; break; }
            }
            const uint64_t y = x - G.g[L + i];
            const uint64_t src = __ldcg(tb.off + y + 1) - __ldcg(tb.S + (uint64_t)(L + i) * top + y) + (q - st);
            if (tb.link_mode == 1)
                ((uint32_t *)tb.links)[base + q] = (uint32_t)(src & tb.ring_mask) | ((uint32_t)i << kRingIdxBits);
            else
                ((uint64_t *)tb.links)[base + q] = src | ((uint64_t)i << 56);
        }
    }
}

// The whole default memo build in ONE cooperative launch: K1 (count pass + CSR + last tail level) and
// the fill-mode-5 passes of K3 (per tail level: chain lists, blocks), separated by grid barriers
// instead of kernel boundaries.
template <int T>
__global__ void __launch_bounds__(1024) k1_memo(Gens G, Tables tb, unsigned int *counter, uint32_t *list,
                                                 uint64_t cap_list)
{
    __shared__ uint64_t sm[40];
    unsigned int target = 0;
    k1_body<T>(G, tb, counter, target, sm, list, cap_list);
}

// Fill mode 2: one CTA, sources read back through L2 (window too large for the
// ring, few rows per batch).  u64 links, prefetched one batch ahead.
template <int T>
__global__ void __launch_bounds__(1024) k3_fill_l2(const uint64_t *__restrict__ off,
                                                    const uint64_t *__restrict__ links, uint32_t *rows,
                                                    uint64_t top, uint32_t b)
{
    constexpr int MAXR = 4;
    const uint64_t nt = blockDim.x, tid = threadIdx.x;
    auto bend = [&](uint64_t x0) -> uint64_t {
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
            const uint32_t *s = rows + (link & kLinkMask) * T;
#pragma unroll
            for (int j = 0; j < T; ++j) w[j] = s[j];
            incr_word<T>(w, (int)(link >> 56));
        }
        uint32_t *dg = rows + r * T;
#pragma unroll
        for (int j = 0; j < T; ++j) dg[j] = w[j];
    };
    for (uint64_t x0 = 0; x0 < top; x0 += b) {
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

// Fill mode 3: whole grid (memos with many rows per batch); the row ->
// (x, block, source) mapping is computed inline, sources are read through L2,
// a grid barrier separates batches.
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
                uint64_t lo = x0, hi = x1 - 1;   // x: largest x in [x0, x1) with off[x] <= r
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
// F0 (optional, shared memory): F0[a] = Tb_0[n - a g_0] for a <= n / g_0, the level-0 column of the
// search, so the first (widest) level costs shared-memory probes instead of L2 round trips.
__device__ uint64_t unrank(const uint64_t *__restrict__ Tb, uint64_t top, const Gens &G, int L, uint64_t n,
                           uint64_t R, uint32_t *a, const uint64_t *F0 = nullptr)
{
    const int lane = threadIdx.x & 31;
    uint64_t r = n;
    for (int j = 0; j < L; ++j) {
        const uint64_t *Tj = Tb + (uint64_t)j * top;
        const uint64_t gj = G.g[j];
        const uint64_t amax = r / gj;
        const bool cached = (j == 0) && F0 != nullptr;
        uint64_t lo = 0, hi = amax;
        while (lo < hi) {
            if (hi - lo <= 64) {   // <= 64 candidates left: two per lane, one round trip
                const uint64_t c1 = lo + lane + 1, c2 = lo + lane + 33;
                const bool p1 = c1 <= hi && (cached ? F0[c1] : __ldg(Tj + (r - c1 * gj))) > R;
                const bool p2 = c2 <= hi && (cached ? F0[c2] : __ldg(Tj + (r - c2 * gj))) > R;
                lo += __popc(__ballot_sync(kFull, p1)) + __popc(__ballot_sync(kFull, p2));
                break;
            }
            const uint64_t step = (hi - lo + 31) / 32;
            const uint64_t cand = lo + (uint64_t)(lane + 1) * step;
            const bool pred = cand <= hi && (cached ? F0[cand] : __ldg(Tj + (r - cand * gj))) > R;
            const unsigned bal = __ballot_sync(kFull, pred);
            const int m = __popc(bal);
            const uint64_t nlo = lo + (uint64_t)m * step;
            uint64_t nhi = lo + (uint64_t)(m + 1) * step - 1;
            if (nhi > hi) nhi = hi;
            lo = nlo;
            hi = nhi;
        }
        a[j] = (uint32_t)lo;
        const uint64_t fnext = (lo + 1 <= amax) ? (cached ? F0[lo + 1] : __ldg(Tj + (r - (lo + 1) * gj))) : 0;
        R -= fnext;
        r -= lo * gj;
    }
    return R;
}

// floor(U * a / b) without 128-bit arithmetic (a <= b)
__device__ __forceinline__ uint64_t mul_div(uint64_t U, uint64_t a, uint64_t b)
{
    return (U / b) * a + ((U % b) * a) / b;
}

// Global row index of the first row of leading prefix a (PAPER.md lex order):
//   rank(a) = sum_j S_j[ r_{j} - (a_j + 1) g_j ],   r_0 = n, r_{j+1} = r_j - a_j g_j.
__device__ uint64_t row_rank(const uint64_t *__restrict__ S, uint64_t top, const Gens &G, int L, uint64_t n,
                             const uint32_t *a)
{
    uint64_t r = n, R = 0;
    for (int j = 0; j < L; ++j) {
        const uint64_t nxt = ((uint64_t)a[j] + 1) * G.g[j];
        if (nxt <= r) R += __ldg(S + (uint64_t)j * top + (r - nxt));
        r -= (uint64_t)a[j] * G.g[j];
    }
    return R;
}

// Walk cost units (MATERIALIZE / HASH slices): every leading prefix a = (a_1..a_L) the walk visits costs beta
// units and then one unit per row of its memo block, in the walk's (descending lex) order.  The units of the
// subtrees with coordinate j >= c are C_j[r - c g_j], C_j = S_j + beta W_j (both satisfy X_j[y] =
// sum_a X_{j+1}[y - a g_j] for j < L), so the search is unrank's with C in place of T.  Returns the units left
// inside the leaf a (R' < beta + card: R' < beta = inside its visit, else row R' - beta of its block) and,
// in rows_before, the rows of Z(n) before a (the S part of the skipped subtrees).  F0: level 0 of C cached.
__device__ __forceinline__ uint64_t unrank_cost(const uint64_t *__restrict__ S, const uint64_t *__restrict__ Wt, uint64_t beta,
                                uint64_t top, const Gens &G, int L, uint64_t n, uint64_t R, uint32_t *a,
                                const uint64_t *F0, uint64_t &rows_before)
{
    const int lane = threadIdx.x & 31;
    uint64_t r = n, rb = 0;
    for (int j = 0; j < L; ++j) {
        const uint64_t *Sj = S + (uint64_t)j * top, *Wj = Wt + (uint64_t)j * top;
        const uint64_t gj = G.g[j];
        const uint64_t amax = r / gj;
        const bool cached = (j == 0) && F0 != nullptr;
        auto C = [&](uint64_t c) -> uint64_t {
            const uint64_t x = r - c * gj;
            return cached ? F0[c] : __ldg(Sj + x) + beta * __ldg(Wj + x);
        };
        uint64_t lo = 0, hi = amax;
        while (lo < hi) {
            if (hi - lo <= 64) {   // <= 64 candidates left: two per lane, one round trip
                const uint64_t c1 = lo + lane + 1, c2 = lo + lane + 33;
                const bool p1 = c1 <= hi && C(c1) > R;
                const bool p2 = c2 <= hi && C(c2) > R;
                lo += __popc(__ballot_sync(kFull, p1)) + __popc(__ballot_sync(kFull, p2));
                break;
            }
            const uint64_t step = (hi - lo + 31) / 32;
            const uint64_t cand = lo + (uint64_t)(lane + 1) * step;
            const bool pred = cand <= hi && C(cand) > R;
            const unsigned bal = __ballot_sync(kFull, pred);
            const int m = __popc(bal);
            const uint64_t nlo = lo + (uint64_t)m * step;
            uint64_t nhi = lo + (uint64_t)(m + 1) * step - 1;
            if (nhi > hi) nhi = hi;
            lo = nlo;
            hi = nhi;
        }
        a[j] = (uint32_t)lo;
        if (lo + 1 <= amax) {   // the later subtrees (a_j > lo came first): their units and rows
            const uint64_t x = r - (lo + 1) * gj;
            const uint64_t fS = __ldg(Sj + x);
            R -= cached ? F0[lo + 1] : fS + beta * __ldg(Wj + x);
            rb += fS;
        }
        r -= lo * gj;
    }
    rows_before = rb;
    return R;
}

// nextCandidate over the first nl coordinates: the rightmost nonzero a_i, i < nl,
// decrements and the later ones restart at their maximum r_j / g_j; false at the end of the stream.
__device__ __forceinline__ bool prefix_next(uint32_t *a, const Gens &G, int nl, uint64_t n)
{
    int i = -1;
    for (int j = 0; j < nl; ++j)
        if (a[j] > 0) i = j;
    if (i < 0) return false;
    uint64_t r = n;
    for (int j = 0; j < nl; ++j) {
        if (j == i) a[j] -= 1;
        if (j > i) a[j] = (uint32_t)(r / G.g[j]);
        r -= (uint64_t)a[j] * G.g[j];
    }
    return true;
}

// Pair walk (COUNT, L >= 3): the global row of the first outer prefix (a_1..a_{L-2}) whose first cost
// rank is >= u (an outer prefix belongs to the shard / slice holding its first cost rank); the C
// tables C_0..C_{L-3} rank outer prefixes by cost.  rows_total when there is none.
__device__ uint64_t pair_row_at(const uint64_t *__restrict__ C, const uint64_t *__restrict__ S, uint64_t top,
                                const Gens &G, int L, uint64_t n, uint64_t u, uint64_t U, uint64_t rows_total)
{
    if (u >= U) return rows_total;
    uint32_t a[kMaxD];
    for (int j = 0; j < kMaxD; ++j) a[j] = 0;
    const uint64_t rin = unrank(C, top, G, L - 2, n, u, a);
    if (rin > 0 && !prefix_next(a, G, L - 2, n)) return rows_total;
    return row_rank(S, top, G, L - 2, n, a);
}

// K4: shard geometry, entirely on the device (no host round trip).  One warp.
// MAT/HASH cut the rows of Z(n) evenly; COUNT cuts the leading-prefix walk evenly, or, for the pair
// walk, the cost ranks of the C tables (each outer prefix goes whole to the shard holding its first
// cost rank).  The slices themselves are unranked by the K5 warp that walks them.
__global__ void __launch_bounds__(32) k4_plan(Gens G, PlanArgs A, const uint64_t *__restrict__ S,
                                               const uint64_t *__restrict__ W, const uint64_t *__restrict__ C,
                                               PlanHdr *hdr)
{
    griddep_wait();   // PDL: the count tables of the memo build are complete and visible
    griddep_launch();
    const int lane = threadIdx.x & 31;
    const bool count_mode = (A.mode == FZ_COUNT) && A.L > 0;   // t = d (L = 0): rows in every mode
    const uint64_t *Tb = A.pairs ? C : (count_mode ? W : S);
    const uint64_t U = __ldg(Tb + A.n);
    const uint64_t ub = mul_div(U, A.shard, A.nshards);
    const uint64_t ue = mul_div(U, A.shard + 1, A.nshards);
    uint64_t len = ue - ub;
    // MATERIALIZE / HASH through k5_walk: the shard stays the row range [ub, ue); its slices cut the walk's cost
    // units (unrank_cost) between the units of its first and last rows, cost(x) = x + rbeta (leading prefixes
    // up to and including the one holding row x), so that sparse parts of the walk (many visited prefixes per
    // row) get as many slices as their work asks
    uint64_t cb = ub;
    const bool cost_slices = !A.pairs && !count_mode && A.rbeta && A.L > 0;
    if (cost_slices) {
        auto cost_of = [&](uint64_t x) -> uint64_t {
            if (x >= U) return U + A.rbeta * __ldg(W + A.n);
            uint32_t a[kMaxD];
            for (int j = 0; j < kMaxD; ++j) a[j] = 0;
            unrank(S, A.top, G, A.L, A.n, x, a);
            return x + A.rbeta * (row_rank(W, A.top, G, A.L, A.n, a) + 1);
        };
        cb = cost_of(ub);
        len = cost_of(ue) - cb;
    }
    uint64_t slice_len, nslices, gw = 0;
    if (A.pairs) {
        gw = A.wg;
        slice_len = len / (A.wg * A.gss_tail);
        if (slice_len < 1024) slice_len = 1024;
        nslices = gss_count(len, gw, slice_len);
    } else if (A.wg && !count_mode) {   // MATERIALIZE / HASH rows (k5_walk): guided slices as well
        gw = A.wg;
        slice_len = len / (A.wg * A.gss_tail);
        if (slice_len < A.floor_len) slice_len = A.floor_len;
        if (slice_len > (1ull << 26)) slice_len = 1ull << 26;
        nslices = gss_count(len, gw, slice_len);
    } else {
        slice_len = (len + A.max_slices - 1) / A.max_slices;
        if (slice_len < A.floor_len) slice_len = A.floor_len;
        if (slice_len > (1ull << 26)) slice_len = 1ull << 26;   // K5 sums 32 lanes' budgets in 32 bits
        nslices = (len + slice_len - 1) / slice_len;
    }
    uint64_t rb = ub, re = ue;
    if (A.pairs) {
        const uint64_t rows_total = __ldg(S + A.n);
        rb = pair_row_at(C, S, A.top, G, A.L, A.n, ub, U, rows_total);
        re = pair_row_at(C, S, A.top, G, A.L, A.n, ue, U, rows_total);
    } else if (count_mode) {
        const uint64_t rows_total = __ldg(S + A.n);
        uint32_t a[kMaxD];
        for (int j = 0; j < kMaxD; ++j) a[j] = 0;
        if (ub < U) {
            unrank(W, A.top, G, A.L, A.n, ub, a);
            rb = row_rank(S, A.top, G, A.L, A.n, a);
        } else {
            rb = rows_total;
        }
        if (ue < U) {
            unrank(W, A.top, G, A.L, A.n, ue, a);
            re = row_rank(S, A.top, G, A.L, A.n, a);
        } else {
            re = rows_total;
        }
    }
    if (lane == 0) {
        PlanHdr h;
        h.result[0] = 0;
        h.result[1] = 0;
        h.err = 0;
        h.total_units = U;
        h.shard_begin = cost_slices ? cb : ub;
        h.shard_len = len;
        h.rbeta = cost_slices ? A.rbeta : 0;
        h.slice_len = slice_len;
        h.nslices = nslices;
        h.row_begin = rb;
        h.rows = re - rb;
        h.next_slice = 0;
        h.gss_warps = gw;
        *hdr = h;
    }
}

// ----------------------------------------------------------------------- K5
// Order-sensitive row hash (reading R17), the product's own
// implementation.
constexpr uint64_t kHashK = 0x9E3779B97F4A7C15ull;   // R17: x = (k + 1) * kHashK

// x * M mod 2^64 for a constant M in three 32-bit multiply-adds (lo(x) lo(M) wide, then lo(x) hi(M) and
// hi(x) lo(M) into the high word); the compiler's own 64-bit multiply takes four instructions
__device__ __forceinline__ uint64_t mul64c(uint64_t x, uint64_t M)
{
    uint32_t lo, hi;
    asm("{\n\t.reg .u32 xl, xh;\n\t.reg .u64 w;\n\t"
        "mov.b64 {xl, xh}, %2;\n\t"
        "mul.wide.u32 w, xl, %3;\n\t"
        "mov.b64 {%0, %1}, w;\n\t"
        "mad.lo.u32 %1, xl, %4, %1;\n\t"
        "mad.lo.u32 %1, xh, %3, %1;\n\t}"
        : "=r"(lo), "=r"(hi)
        : "l"(x), "r"((uint32_t)M), "r"((uint32_t)(M >> 32)));
    return ((uint64_t)hi << 32) | lo;
}

// R17 from its first state x0 = (k + 1) * kHashK (callers form x0 by additions along consecutive rows)
template <int D>
__device__ __forceinline__ uint64_t row_hash_x0(uint64_t x, const uint32_t (&w)[D])
{
#pragma unroll
    for (int j = 0; j < D; ++j) {
        x = mul64c(x ^ (uint64_t)w[j], 0xBF58476D1CE4E5B9ull);
        x ^= x >> 29;
    }
    x ^= (uint64_t)D;
    x ^= x >> 33;
    x = mul64c(x, 0xFF51AFD7ED558CCDull);
    x ^= x >> 33;
    x = mul64c(x, 0xC4CEB9FE1A85EC53ull);
    x ^= x >> 33;
    return x;
}

template <int D>
__device__ __forceinline__ uint64_t row_hash(uint64_t k, const uint32_t (&w)[D])
{
    return row_hash_x0<D>((k + 1) * kHashK, w);
}

// Memo-row loads and output stores as volatile PTX: they keep program order, so a warp issues the
// loads of all its UNR chunks before the first store (UNR L2 loads in flight per lane).
template <int T>
__device__ __forceinline__ void load_tail(const uint32_t *__restrict__ p, uint32_t *w)
{
    if constexpr (T == 2) {
        asm volatile("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "l"(p));
    } else if constexpr (T == 4) {
        asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                     : "l"(p));
    } else {
#pragma unroll
        for (int j = 0; j < T; ++j) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(w[j]) : "l"(p + j));
    }
}

template <int T>
__device__ __forceinline__ void load_tail16(const uint16_t *__restrict__ p, uint32_t *w)
{
#pragma unroll
    for (int j = 0; j < T; ++j) asm volatile("ld.global.nc.u16 %0, [%1];" : "=r"(w[j]) : "l"(p + j));
}

// u16 copy of the memo rows (flat: every coordinate narrowed; the host checked they are < 2^16)
__global__ void __launch_bounds__(256) k3_pack16(const uint32_t *__restrict__ rows, uint16_t *__restrict__ out,
                                                  uint64_t words)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (uint16_t)__ldg(rows + i);
}

template <int D>
__device__ __forceinline__ void store_row(uint32_t *p, const uint32_t (&w)[D])
{
    if constexpr (D % 4 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 4)
            asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p + j), "r"(w[j]), "r"(w[j + 1]),
                         "r"(w[j + 2]), "r"(w[j + 3])
                         : "memory");
    } else if constexpr (D % 2 == 0) {
#pragma unroll
        for (int j = 0; j < D; j += 2)
            asm volatile("st.global.cs.v2.u32 [%0], {%1, %2};" ::"l"(p + j), "r"(w[j]), "r"(w[j + 1]) : "memory");
    } else {
#pragma unroll
        for (int j = 0; j < D; ++j) asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p + j), "r"(w[j]) : "memory");
    }
}

__device__ __forceinline__ void st_cs_u32(uint32_t *p, uint32_t v)
{
    asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void st_cs_v4(uint32_t *p, const uint4 &v)
{
    asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

struct BlockInfo {      // one non-empty memo block of the current warp round (16 B)
    uint64_t memo_row;  // first memo row to copy (off[p] + k offset)
    uint32_t start;     // first output row of the block, relative to the round
    uint32_t v;         // innermost leading coordinate a_L of the block
};

__device__ __forceinline__ BlockInfo lds_block_info(uint32_t a)
{
    uint32_t x, y, z, w;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(w) : "r"(a));
    BlockInfo b;
    b.memo_row = ((uint64_t)y << 32) | x;
    b.start = z;
    b.v = w;
    return b;
}

#ifndef FZ_SLICE_TRACE
#define FZ_SLICE_TRACE 0   // diagnostic builds: per-slice unrank / walk cycles of k5_walk (fz_debug_slice_trace)
#endif
#if FZ_SLICE_TRACE
__device__ uint4 g_slice_trace[1u << 20];
#endif
#ifndef FZ_HASH_MINB
#define FZ_HASH_MINB 4  // HASH walk, d <= 6: resident CTAs per SM the register budget is sized for
#endif
#ifndef FZ_WIDE_MINB
#define FZ_WIDE_MINB 2  // MATERIALIZE / HASH walk, d > 6 without the word stream: resident CTAs per SM
#endif
#ifndef FZ_HASH_UNR
#define FZ_HASH_UNR 2   // HASH / COUNT (L <= 2) walk: 32-row chunks in flight per warp
#endif
#ifndef FZ_WS_GROUP
#define FZ_WS_GROUP 1   // word stream: 32-row chunks whose memo loads are in flight together (4: more registers, spills)
#endif
constexpr int kWalkThreads = 256;
#ifndef FZ_COUNT_THREADS
#define FZ_COUNT_THREADS 1024
#endif
constexpr int kCountThreads = FZ_COUNT_THREADS;   // COUNT walk: one CTA per SM shares one staged card table
template <int MODE>
constexpr int walk_threads() { return MODE == FZ_COUNT ? kCountThreads : kWalkThreads; }

struct WalkTables {
    const uint32_t *cardT;   // residue-major card (w.r.t. m = g_L)
    const uint64_t *offT;    // residue-major CSR offsets
    const uint32_t *memo;    // CSR rows, t u32 each
    const uint16_t *memo16;  // the same rows as t u16 each (large memos with small coordinates), or nullptr
    const uint64_t *card64;  // card = S_L, natural layout
    const uint64_t *Wt;      // leading-prefix count tables W_0..W_L (cost slices: unrank_cost)
    uint64_t gmag[kMaxD];    // division magic of each generator: x / g_j = umulhi64(x, gmag[j]) (+x if g_j = 1)
    uint32_t m;              // g_L (residue modulus of cardT / offT)
    uint64_t R;              // rows per residue column
    int word_stream;         // MATERIALIZE, d not a multiple of 4: write rows as a 16-B word stream
};


template <int D, int T, int MODE, bool M16 = false, bool WS = false, bool CS = false>
__global__ void __launch_bounds__(walk_threads<MODE>(), (MODE == FZ_COUNT ? 1 : (MODE == FZ_HASH && D <= 6 ? FZ_HASH_MINB : (D <= 6 ? 4 : (WS ? 4 : FZ_WIDE_MINB)))))
k5_walk(Gens G, uint64_t n64, PlanHdr *hdr,
                                                         const uint64_t *__restrict__ Tb, uint64_t top, WalkTables wt,
                                                         uint32_t *out, uint64_t out_cap_rows, uint64_t row_base,
                                                         uint32_t f0n, uint32_t c16R)
{
    griddep_wait();   // PDL: the plan header (K4) and the memo tables are complete and visible
    extern __shared__ uint64_t f0s[];   // level-0 unrank column (f0n entries, 0 = not cached)
    // cost slices (MATERIALIZE / HASH): the walk's units are rows plus rbeta per visited leading prefix, and the
    // cached level-0 column holds C_0 = S_0 + rbeta W_0 (unrank_cost)
    const uint64_t rbeta = (MODE != FZ_COUNT && CS) ? hdr->rbeta : 0;   // CS: the cost-slice instantiation
    for (uint32_t q = threadIdx.x; q < f0n; q += blockDim.x) {
        const uint64_t x = n64 - (uint64_t)q * G.g[0];
        f0s[q] = __ldg(Tb + x) + (rbeta ? rbeta * __ldg(wt.Wt + x) : 0);
    }
    // COUNT, L = 2: card[x] = S_L[x], x <= n, as u16 in shared memory after f0s, residue-major w.r.t.
    // m = g_L with c16R entries per residue column (16-B aligned columns; c16R = 0: not staged)
    uint16_t *c16 = reinterpret_cast<uint16_t *>(f0s + ((f0n + 1) & ~1u));
    if (c16R) {
        const uint32_t mm = G.g[D - T - 1];
        for (uint32_t x = threadIdx.x; x <= (uint32_t)n64; x += blockDim.x)
            c16[(x % mm) * c16R + x / mm] = (uint16_t)__ldg(wt.card64 + x);
    }
    __syncthreads();
    constexpr int L = D - T;
    static_assert(L >= 1, "at least one leading coordinate");
    __shared__ BlockInfo binfo[MODE == FZ_COUNT ? 1 : kWalkThreads / 32][32];   // MAT/HASH block lists
    // MATERIALIZE with d not a multiple of 4 (the WS variant): per-warp staging of 128 rows as a word stream (+ 3 words of phase)
    constexpr bool kWordStream = WS && MODE == FZ_MATERIALIZE && (D % 4) != 0;
    constexpr int kUnr = (MODE == FZ_MATERIALIZE) ? 4 : FZ_HASH_UNR;   // 32-row chunks per group (MAT d >= 7 with 2: slower)
    __shared__ __align__(16) uint32_t wsb[kWordStream ? kWalkThreads / 32 : 1][kWordStream ? 32 * kUnr * D + 4 : 1];
    const int lane = threadIdx.x & 31, wib = (MODE == FZ_COUNT) ? 0 : threadIdx.x >> 5;
    const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint32_t n = (uint32_t)n64;
    const uint32_t m = G.g[L - 1];
    const uint64_t nslices = hdr->nslices, slice_len = hdr->slice_len, shard_begin = hdr->shard_begin,
                   shard_len = hdr->shard_len;
    const uint64_t gsw = hdr->gss_warps;   // guided slices (MATERIALIZE / HASH rows) when != 0
    if (MODE == FZ_MATERIALIZE && hdr->rows > out_cap_rows) {
        if (threadIdx.x == 0 && blockIdx.x == 0) hdr->err = 1;
        return;
    }
    if (row_base == ~0ull) row_base = hdr->row_begin;
    uint64_t *result = hdr->result;
    const uint32_t *__restrict__ cardT = wt.cardT;
    const uint64_t *__restrict__ offT = wt.offT;
    uint64_t acc_rows = 0, acc_hash = 0;
    // 32-bit shared address of this warp's block list, read back with ld.shared (keeps the compiler from
    // re-deriving the generic shared window -- S2R TID / CgaCtaId -- for every 32-row chunk)
    const uint64_t lane_k = (uint64_t)lane * kHashK;   // HASH: lane's share of the row-key multiply
    uint32_t bi_sa;   // (through a volatile move: the compiler keeps it in a register instead of recomputing it)
    asm volatile("mov.b32 %0, %1;" : "=r"(bi_sa) : "r"(smem_addr(binfo[wib])));
    uint32_t ws_sa = 0;   // the word-stream staging buffer of this warp, the same way
    if constexpr (kWordStream) asm volatile("mov.b32 %0, %1;" : "=r"(ws_sa) : "r"(smem_addr(wsb[wib])));
    (void)ws_sa;
    const uint32_t cgq = (L >= 2) ? G.g[L >= 2 ? L - 2 : 0] / m : 0, cgr = (L >= 2) ? G.g[L >= 2 ? L - 2 : 0] % m : 0;

    (void)gw;
    (void)nw;
    for (;;) {
        uint64_t s = 0;
        if (lane == 0) s = atomicAdd(&hdr->next_slice, 1ull);
        s = shfl_u64(s, 0);
        if (s >= nslices) break;
        // K4 slice: units [rel, rel + len) of the shard; unrank its first unit (rows: S, prefixes: W)
#if FZ_SLICE_TRACE
        const long long tr_t0 = clock64();
#endif
        Slice sl;
        if (gsw) {   // guided slices (K4): sizes halve round by round down to slice_len
            sl.begin = gss_begin(s, shard_len, gsw, slice_len);
            sl.len = gss_begin(s + 1, shard_len, gsw, slice_len) - sl.begin;
            if (sl.len == 0) continue;
        } else {
            sl.begin = s * slice_len;
            sl.len = (shard_len - sl.begin) < slice_len ? (shard_len - sl.begin) : slice_len;
        }
        // cost slices: visit units of the slice's first leading prefix still inside the slice (rbeta, or the
        // rest of them when the slice starts inside that visit; 0 when it starts inside its rows)
        uint64_t vfirst = rbeta;
        {
            uint32_t ua[kMaxD];
#pragma unroll
            for (int j = 0; j < kMaxD; ++j) ua[j] = 0;
            if (rbeta) {
                uint64_t rows_before;
                const uint64_t Rp = unrank_cost(Tb, wt.Wt, rbeta, top, G, L, n64, shard_begin + sl.begin, ua,
                                                f0n ? f0s : nullptr, rows_before);
                sl.k0 = Rp >= rbeta ? Rp - rbeta : 0;
                vfirst = Rp >= rbeta ? 0 : rbeta - Rp;
                sl.begin = rows_before + sl.k0 - hdr->row_begin;   // the slice's first row, shard-relative
            } else {
                const uint64_t k0 = unrank(Tb, top, G, L, n64, shard_begin + sl.begin, ua, f0n ? f0s : nullptr);
                sl.k0 = (MODE == FZ_COUNT) ? 0 : k0;
            }
#pragma unroll
            for (int j = 0; j < L; ++j) sl.a[j] = ua[j];
        }
        uint32_t a[L];
#pragma unroll
        for (int j = 0; j < L; ++j) a[j] = sl.a[j];
#if FZ_SLICE_TRACE
        const long long tr_t1 = clock64();
#endif
        uint32_t r_in = n;
#pragma unroll
        for (int j = 0; j < L - 1; ++j) r_in -= a[j] * G.g[j];
        int32_t v = (int32_t)a[L - 1];
        // residue-major index of p = r_in - v*m is colbase + (r_in/m - v): contiguous in v
        uint64_t colbase = (uint64_t)(r_in % m) * wt.R + r_in / m;
        uint64_t kfirst = sl.k0;
        uint64_t left = sl.len;
        uint64_t outpos = sl.begin;
        if constexpr (MODE == FZ_COUNT) {
            // COUNT walk: every leading prefix adds card[p], p = n - phi(prefix) (one card lookup per
            // leading prefix).  An innermost run v, v-1, .., 0 is the contiguous residue-major segment
            // [col R + q - v, col R + q]: a run is summed by the 32 lanes together (the slice's partial
            // first and last runs, and every run when the card table is not staged).  With the card
            // table staged in shared memory (u16, natural layout), whole runs go one per lane: lane l
            // takes sibling a_{L-2} - l and sums card[r_l - v m], v = 0..r_l / m, so the per-run
            // bookkeeping is shared by 32 runs.
            uint32_t q = r_in / m, col = r_in - q * m;
            uint32_t vv = (uint32_t)v;
            uint32_t left32 = (uint32_t)left;   // K4 keeps COUNT slices below 2^31 prefixes
            const uint32_t g2 = (L >= 2) ? G.g[L >= 2 ? L - 2 : 0] : 0u;
            const uint64_t mmag = wt.gmag[L - 1];
            // outer carry (rightmost nonzero a_i, i < L-2 ... L-1 excluded): false at end of stream
            auto carry = [&]() -> bool {
                if (a[L - 2] > 0) {
                    a[L - 2] -= 1;
                    col += cgr;
                    if (col >= m) {
                        col -= m;
                        ++q;
                    }
                    q += cgq;
                } else {
                    int i = -1;
#pragma unroll
                    for (int j = 0; j < L - 1; ++j)
                        if (a[j] > 0) i = j;
                    if (i < 0) return false;
                    uint32_t r = n;
#pragma unroll
                    for (int j = 0; j < L - 1; ++j) {
                        if (j == i) a[j] -= 1;
                        if (j > i) a[j] = fdiv(r, wt.gmag[j]);
                        r -= a[j] * G.g[j];
                    }
                    q = fdiv(r, mmag);
                    col = r - q * m;
                }
                vv = q;
                return true;
            };
            for (;;) {
                {   // one run, warp-cooperative: v = vv .. max(0, vv + 1 - left)
                    const uint32_t run = vv + 1;
                    const uint32_t take = left32 < run ? left32 : run;
                    const uint32_t *p = cardT + ((uint64_t)col * wt.R + (q - vv) + lane);
                    uint32_t rem = take;
                    // u64 sums: card values are unbounded in COUNT-only layouts
                    for (; rem >= 128; rem -= 128, p += 128)
                        acc_rows += (uint64_t)__ldg(p) + __ldg(p + 32) + __ldg(p + 64) + __ldg(p + 96);
                    uint64_t part = 0;
                    if ((uint32_t)lane < rem) part += __ldg(p);
                    if ((uint32_t)lane + 32 < rem) part += __ldg(p + 32);
                    if ((uint32_t)lane + 64 < rem) part += __ldg(p + 64);
                    if ((uint32_t)lane + 96 < rem) part += __ldg(p + 96);
                    acc_rows += part;
                    left32 -= take;
                }
                if (left32 == 0 || L == 1 || !carry()) break;
                if (L >= 2 && c16R) {
                    // whole runs, one per lane, while they fit the slice's budget
                    bool more = true;
                    for (;;) {
                        const uint32_t A = a[L - 2];
                        const uint32_t rin = q * m + col;
                        const uint32_t rl = rin + (uint32_t)lane * g2;
                        const uint32_t len = ((uint32_t)lane <= A) ? fdiv(rl, mmag) + 1 : 0u;
                        uint32_t incl = len;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const uint32_t u = __shfl_up_sync(kFull, incl, o);
                            if (lane >= o) incl += u;
                        }
                        const bool fit = len > 0 && incl <= left32;
                        const int nf = __popc(__ballot_sync(kFull, fit));
                        if (nf == 0) break;
                        if (fit) {   // entries 0..len-1 of residue column rl mod m: 16-B vectors, 2 cards per dp2a
                            const uint32_t cl = rl - (len - 1) * m;
                            const uint16_t *cp = c16 + cl * c16R;
                            const uint4 *vp = reinterpret_cast<const uint4 *>(cp);
                            const uint32_t nv = len >> 3;
                            uint32_t s0 = 0, s1 = 0;
                            uint32_t k = 0;
                            for (; k + 2 <= nv; k += 2) {
                                const uint4 w0 = vp[k], w1 = vp[k + 1];
                                s0 = __dp2a_lo(w0.x, 0x0101u, s0);
                                s1 = __dp2a_lo(w0.y, 0x0101u, s1);
                                s0 = __dp2a_lo(w0.z, 0x0101u, s0);
                                s1 = __dp2a_lo(w0.w, 0x0101u, s1);
                                s0 = __dp2a_lo(w1.x, 0x0101u, s0);
                                s1 = __dp2a_lo(w1.y, 0x0101u, s1);
                                s0 = __dp2a_lo(w1.z, 0x0101u, s0);
                                s1 = __dp2a_lo(w1.w, 0x0101u, s1);
                            }
                            if (k < nv) {
                                const uint4 w0 = vp[k];
                                s0 = __dp2a_lo(w0.x, 0x0101u, s0);
                                s1 = __dp2a_lo(w0.y, 0x0101u, s1);
                                s0 = __dp2a_lo(w0.z, 0x0101u, s0);
                                s1 = __dp2a_lo(w0.w, 0x0101u, s1);
                            }
                            const uint32_t tl = len & 7;   // last partial vector, masked
                            if (tl) {
                                const uint4 w0 = vp[nv];
                                auto mk = [&](uint32_t i) {
                                    return tl > 2 * i + 1 ? 0xffffffffu : (tl > 2 * i ? 0xffffu : 0u);
                                };
                                s0 = __dp2a_lo(w0.x & mk(0), 0x0101u, s0);
                                s1 = __dp2a_lo(w0.y & mk(1), 0x0101u, s1);
                                s0 = __dp2a_lo(w0.z & mk(2), 0x0101u, s0);
                                s1 = __dp2a_lo(w0.w & mk(3), 0x0101u, s1);
                            }
                            acc_rows += s0 + s1;
                        }
                        left32 -= __shfl_sync(kFull, incl, (nf - 1) & 31);
                        if (left32 == 0) {
                            more = false;
                            break;
                        }
                        if ((uint32_t)nf <= A) {   // siblings left at level L-2: a_{L-2} = A - nf
                            a[L - 2] = A - (uint32_t)nf;
                            const uint32_t r2 = rin + (uint32_t)nf * g2;
                            q = fdiv(r2, mmag);
                            col = r2 - q * m;
                            vv = q;
                        } else {                   // level L-2 exhausted: outer carry
                            a[L - 2] = 0;
                            if (!carry()) {
                                more = false;
                                break;
                            }
                        }
                    }
                    if (!more) break;
                }
            }
            left = left32;
        } else {
        while (left > 0) {
            {
                const int32_t vv = v - lane;
                const bool valid = vv >= 0;
                const uint64_t ti = colbase - (uint64_t)v + lane;
                uint32_t c = valid ? __ldg(cardT + ti) : 0u;
                uint64_t mrow = valid ? __ldg(offT + ti) : 0;
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
                uint32_t use;   // rows of this round inside the slice
                if (rbeta) {
                    // cost budget: lane l (a valid prefix, l <= v) costs its visit (vfirst for lane 0, rbeta for
                    // the others) plus its c rows; the valid lanes are 0..min(v, 31)
                    const uint64_t nvis = (uint64_t)((uint32_t)lane < (uint32_t)v ? lane : v);
                    const uint64_t cincl = incl + vfirst + rbeta * nvis;   // units of lanes 0..lane
                    const uint64_t ctot = shfl_u64(cincl, 31);
                    if (ctot <= left) {
                        use = total;
                        left -= ctot;
                    } else {   // the slice ends in lane j: its rows after the budget's end belong to the next slice
                        const unsigned over = __ballot_sync(kFull, cincl > left);
                        const int j = __ffs(over) - 1;
                        const uint64_t cex = shfl_u64(cincl, j) - __shfl_sync(kFull, c, j) -
                                             (j == 0 ? vfirst : rbeta);   // units before lane j
                        const uint64_t vis = (j == 0) ? vfirst : rbeta;
                        const uint32_t cj = __shfl_sync(kFull, c, j), exj = __shfl_sync(kFull, excl, j);
                        const uint64_t in_rows = left > cex + vis ? left - cex - vis : 0;   // < cj
                        use = exj + (uint32_t)(in_rows < cj ? in_rows : cj);
                        left = 0;
                    }
                    vfirst = rbeta;
                } else {
                    use = (uint64_t)total < left ? total : (uint32_t)left;
                }
                const uint32_t cc = excl >= use ? 0u : (c < use - excl ? c : use - excl);
                const unsigned nz = __ballot_sync(kFull, cc > 0);
                if (cc > 0) {
                    const int e = __popc(nz & ((1u << lane) - 1));
                    // byte address of the block's memo rows, pre-offset by its first output row (u64 wrap)
                    const uint64_t mr = M16 ? (uint64_t)(uintptr_t)wt.memo16 + (mrow - excl) * (uint64_t)(2 * (T > 0 ? T : 1))
                                            : (uint64_t)(uintptr_t)wt.memo + (mrow - excl) * (uint64_t)(4 * (T > 0 ? T : 1));
                    // {memo_row, start, v} as one 16-B store through the register-kept shared address
                    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(bi_sa + 16u * (uint32_t)e),
                                 "r"((uint32_t)mr), "r"((uint32_t)(mr >> 32)), "r"(excl), "r"((uint32_t)vv)
                                 : "memory");
                }
                __syncwarp();
                // flattened copy: rows q0 + lane of the round, owner block via block-start bitmask.
                // UNR chunks of 32 rows are resolved and their memo tails loaded before any store,
                // so each lane keeps UNR L2 loads in flight.
                constexpr int UNR = kUnr;
                const uint32_t rel = cc > 0 ? excl : 0xffffffffu;   // this lane's block start (none: ~0)
                uint32_t lm_le;                                       // lanes 0..lane
                asm("mov.u32 %0, %%lanemask_le;" : "=r"(lm_le));
                int before = -1;   // block starts before the chunk, minus one
                for (uint32_t q0 = 0; q0 < use; q0 += 32 * UNR) {
                    if constexpr (kWordStream) {
                        // d not a multiple of 4 (WS variant): the warp's rows [q0, q0 + nr) are one contiguous run
                        // of nr d words; each row goes to shared memory (at the 16-B phase of its global
                        // address) as soon as its memo tail is loaded, then the aligned middle leaves as 16-B
                        // vectors (scalar head and tail words)
                        const uint32_t nr = (use - q0 < 32u * UNR) ? use - q0 : 32u * UNR;
                        const uint64_t G0 = (outpos + q0) * (uint64_t)D;        // first word (shard-relative)
                        const uint32_t sft = (uint32_t)(((uintptr_t)(out + G0) >> 2) & 3);
                        const uint32_t sb = ws_sa + 4u * sft;   // 32-bit shared address of the staged run
                        // WSG 32-row chunks have their memo loads in flight before their rows go to shared memory
                        constexpr int WSG = (FZ_WS_GROUP < UNR) ? FZ_WS_GROUP : UNR;
#pragma unroll
                        for (int u0 = 0; u0 < UNR; u0 += WSG) {
                            uint32_t tw[WSG][T > 0 ? T : 1], vv[WSG];
                            bool okg[WSG];
#pragma unroll
                            for (int g = 0; g < WSG; ++g) {
                                const uint32_t qb = q0 + 32 * (u0 + g);
                                uint32_t bit;
                                asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"(rel - qb));
                                const unsigned M = __reduce_or_sync(kFull, bit);
                                const uint32_t q = qb + lane;
                                const int e = before + __popc(M & lm_le);
                                before += __popc(M);
                                okg[g] = q < use;
                                if (okg[g]) {
                                    const BlockInfo info = lds_block_info(bi_sa + 16u * (uint32_t)e);
                                    vv[g] = info.v;
                                    if constexpr (T > 0)
                                        load_tail<T>(reinterpret_cast<const uint32_t *>(info.memo_row + (uint64_t)q * (4 * T)),
                                                     tw[g]);
                                }
                            }
#pragma unroll
                            for (int g = 0; g < WSG; ++g) {
                                if (!okg[g]) continue;
                                const uint32_t rw = sb + 4u * (uint32_t)((32 * (u0 + g) + lane) * D);
#pragma unroll
                                for (int j = 0; j < L - 1; ++j) sts32(rw + 4u * j, a[j]);
                                sts32(rw + 4u * (L - 1), vv[g]);
#pragma unroll
                                for (int j = 0; j < T; ++j) sts32(rw + 4u * (L + j), tw[g][j]);
                            }
                        }
                        __syncwarp();
                        const uint32_t W = nr * D, head = ((4 - sft) & 3) < W ? ((4 - sft) & 3) : W;
                        const uint32_t nv = (W - head) >> 2, tail0 = head + 4 * nv;
                        uint32_t *og = out + G0;
                        if ((uint32_t)lane < head) st_cs_u32(og + lane, lds32(sb + 4u * lane));
                        {   // lane l stores vectors l, l + 32, ..: pointers advance by 512 B (no per-store 64-bit index math)
                            uint32_t sa = sb + 4u * head + 16u * (uint32_t)lane;
                            uint32_t *gp = og + head + 4 * lane;
                            for (uint32_t v = lane; v < nv; v += 32, sa += 512, gp += 128) st_cs_v4(gp, lds128(sa));
                        }
                        if ((uint32_t)lane < W - tail0) st_cs_u32(og + tail0 + lane, lds32(sb + 4u * (tail0 + lane)));
                        __syncwarp();
                        continue;
                    }
                    uint32_t wv[UNR][D];
                    bool ok[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const uint32_t qb = q0 + 32 * u;
                        uint32_t bit;   // 1 << (rel - qb), 0 unless the block starts inside this chunk
                        asm("shl.b32 %0, 1, %1;" : "=r"(bit) : "r"(rel - qb));   // PTX clamps shifts >= 32 to 0
                        const unsigned M = __reduce_or_sync(kFull, bit);
                        const uint32_t q = qb + lane;
                        ok[u] = q < use;
                        const int e = before + __popc(M & lm_le);   // owner: the last block starting at or before q
                        before += __popc(M);
                        if (ok[u]) {
                            const BlockInfo info = lds_block_info(bi_sa + 16u * (uint32_t)e);
#pragma unroll
                            for (int j = 0; j < L - 1; ++j) wv[u][j] = a[j];
                            wv[u][L - 1] = info.v;
                            if constexpr (T > 0) {
                                uint32_t tw[T];
                                if constexpr (M16)   // u16 copy: half the L2 / DRAM bytes per row
                                    load_tail16<T>(reinterpret_cast<const uint16_t *>(info.memo_row + (uint64_t)q * (2 * T)),
                                                   tw);
                                else
                                    load_tail<T>(reinterpret_cast<const uint32_t *>(info.memo_row + (uint64_t)q * (4 * T)),
                                                 tw);
#pragma unroll
                                for (int j = 0; j < T; ++j) wv[u][L + j] = tw[j];
                            }
                        }
                    }
                    {
                        uint32_t *ob = out + (outpos + q0 + lane) * (uint64_t)D;   // chunk u at ob + 32 u D
                        // HASH: the first state (k + 1) kHashK of row k = row_base + outpos + q0 + 32 u + lane by
                        // additions from one multiply per group (mod 2^64)
                        const uint64_t x0 = (row_base + outpos + q0 + 1) * kHashK + lane_k;
#pragma unroll
                        for (int u = 0; u < UNR; ++u) {
                            if (!ok[u]) continue;
                            if constexpr (MODE == FZ_MATERIALIZE) {
                                store_row<D>(ob + 32 * u * D, wv[u]);
                            } else {
                                acc_hash += row_hash_x0<D>(x0 + (uint64_t)(32 * u) * kHashK, wv[u]);
                            }
                        }
                    }
                }
                __syncwarp();
                acc_rows += (lane == 0) ? use : 0;
                outpos += use;
                if (!rbeta) left -= use;   // cost slices: the round's units were taken above
                if (left == 0) break;
                if (v >= 32) {
                    v -= 32;
                    continue;
                }
            }
            // carry: nextCandidate over the outer leading coordinates:
            // rightmost nonzero index i < L-1, a_i--, later coordinates restart at their maximum.
            int i = -1;
#pragma unroll
            for (int j = 0; j < L - 1; ++j)
                if (a[j] > 0) i = j;
            if (i < 0) break;   // end of stream
            if (i == L - 2) {   // common case: only a_{L-1} changes, r_in grows by g_{L-1}
                a[L - 2] -= 1;
                r_in += G.g[L - 2];
            } else {
                uint32_t r = n;
#pragma unroll
                for (int j = 0; j < L - 1; ++j) {
                    if (j == i) a[j] -= 1;
                    if (j > i) a[j] = r / G.g[j];
                    r -= a[j] * G.g[j];
                }
                r_in = r;
            }
            const uint32_t q = r_in / m;
            v = (int32_t)q;
            colbase = (uint64_t)(r_in - q * m) * wt.R + q;
        }
        }
#if FZ_SLICE_TRACE
        if (lane == 0 && s < (1u << 20)) {
            uint64_t gt;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
            uint32_t smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            g_slice_trace[s] = make_uint4((uint32_t)(tr_t1 - tr_t0), (uint32_t)(clock64() - tr_t1), (uint32_t)(gt / 64),
                                          smid);
        }
#endif
    }
    acc_rows = warp_sum_u64(acc_rows);
    if (lane == 0) atomicAdd((unsigned long long *)result, (unsigned long long)acc_rows);
    if constexpr (MODE == FZ_HASH) {
        acc_hash = warp_sum_u64(acc_hash);
        if (lane == 0) atomicAdd((unsigned long long *)(result + 1), (unsigned long long)acc_hash);
    }
}

// ------------------------------------------------------ K5, COUNT pair walk
// COUNT for L >= 3 (one card lookup per leading prefix).  The walk goes
// by OUTER prefixes o = (a_1..a_{L-2}) with remainder R (nextCandidate over the outer coordinates,
// PAPER.md:208-218).  An outer prefix holds the runs k = 0..A, A = R / g2 (g2 = g_{L-2}); run k has
// remainder r_k = rmin + k g2 (rmin = R - A g2) and sums card[r_k - v m], v = 0..r_k / m (m = g_{L-1}):
// entries 0..r_k / m of the residue column r_k mod m.  One lane takes the PAIR of runs (k, A - k)
// (k <= A / 2; k = A / 2 alone when A is even): X = run k, Y = run A - k, |X| <= |Y|, and every pass of a
// warp fills its 32 lanes with the next 32 pairs of the outer-prefix stream, from as many outer prefixes
// as that takes.
//
// Card table: staged once per CTA in shared memory as u16 (u8 when every card < 64), 16-B vectors,
// columns of R16 entries (R16 / entries-per-vector odd).  Column order follows the runs: run k + 1 lies
// in column (col_k + Delta) mod m, Delta = g2 mod m, so with e = gcd(Delta, m), m' = m / e the columns
// of coset s in [0, e) are stored as the orbit s + j Delta, j = 0..m'-1, followed by `dup` (31 or 0)
// repeated columns: the lanes of one outer prefix in a pass read consecutive stored columns (X runs
// ascending, Y runs descending), so the 16-B vectors of 8 lanes fall in 8 distinct bank groups.  Each
// lane reads vector j of Y and of X (while X has one) in the same iteration -- the same vector index in
// every lane, which keeps the loads conflict-free -- adding the packed u16 (u8) words with IADD3 into two
// packed accumulators that dp2a (dp4a) unpacks every F iterations (F = 65535 / (4 card_max), resp.
// 255 / (4 card_max), a multiple of 4); the last, partial vector of each run is read once and summed by
// dp2a / dp4a with 0/1 byte selectors for its first entries (no masking of the data).
//
// Slices: cost ranks of the C tables (C_{L-2}[R] = W_{L-2}[R] + beta (A + 1) + gamma: a run costs its
// lookups plus beta, an outer prefix gamma more), guided sizes (gss_begin).  A slice [b, e) takes the
// outer prefixes whose first cost rank lies in it: both ends are unranked through C_0..C_{L-3} (level 0
// cached in shared memory) and the walk stops at the end's outer prefix.
struct PairGeo {
    uint32_t m, dlt, e, mp, dup, inv;   // m = g_{L-1}, Delta = g2 mod m, e = gcd(Delta, m), m' = m/e, inverse
    uint32_t R16, ncolv, F;             // entries per stored column, stored columns e (m' + dup), flush period
    uint32_t ncolv8, vstride;           // k5_runs' transposed image: ncolv rounded up to 8, bytes between a column's vectors
    uint32_t Mm, Mg2, Me, Mmp;          // div32 magics of m, g2, e, m'
    uint32_t Mg[kMaxD];                 // div32 magics of the generators (outer carry)
    // the common outer step (a_{L-3} decrements: R += g3, g3 = Q3 g2 + S3): column steps (mod m) and,
    // when e = 1, orbit-position steps (mod m) for the two outcomes of rmin + S3 >= g2
    uint32_t Q3, S3, cs1, cs2, is1, is2;
    uint32_t QD, RD, Fr;                // k5_runs: 32 g2 = QD m + RD; flush period (vectors) of its packed sums
    uint32_t bstep, bwrap;              // k5_runs: orbit position - 32 mod m' = p - bstep (p >= bstep) or p + bwrap
    uint64_t one_thr;                   // k5_runs: R < one_thr <=> a run's full vectors ((R / m + 1) / VE) <= Fr
    uint64_t beta, gamma;               // the C tables' cost of a run / an outer prefix (k5_runs slice ends)
};

// x / d for any x < 2^32, d >= 1, from M = floor(2^32 / d) (d = 1: 2^32 - 1): umulhi underestimates the
// quotient by at most one, one compare corrects it
__device__ __forceinline__ uint32_t div32(uint32_t x, uint32_t d, uint32_t M)
{
    const uint32_t q = __umulhi(x, M);
    return (x - q * d >= d) ? q + 1 : q;
}

template <bool U8>
__device__ __forceinline__ uint32_t unpack_add(uint32_t p, uint32_t s)
{
    if constexpr (U8) return __dp4a(p, 0x01010101u, s);
    else return __dp2a_lo(p, 0x0101u, s);
}

// s + the first t entries of the 16-B vector w (t < entries per vector): byte selectors of dp2a / dp4a,
// 1 for the first t entries and 0 after (no masking of the data)
template <bool U8>
__device__ __forceinline__ uint32_t add_prefix(const uint4 &w, uint32_t t, uint32_t s)
{
    uint64_t lo, hi;
    const uint32_t tl = U8 ? (t < 8 ? t : 8) : t, th = (U8 && t > 8) ? t - 8 : 0;
    // bytes 0..tl-1 of 0x0101.. by one right shift (PTX clamps shifts >= 64 to 0: th = 0 gives no bytes)
    asm("shr.b64 %0, %1, %2;" : "=l"(lo) : "l"(0x0101010101010101ull), "r"(64u - 8u * tl));
    if constexpr (U8) {
        asm("shr.b64 %0, %1, %2;" : "=l"(hi) : "l"(0x0101010101010101ull), "r"(64u - 8u * th));
        s = __dp4a(w.x, (uint32_t)lo, s);
        s = __dp4a(w.y, (uint32_t)(lo >> 32), s);
        s = __dp4a(w.z, (uint32_t)hi, s);
        s = __dp4a(w.w, (uint32_t)(hi >> 32), s);
    } else {   // entry k of the vector <-> selector byte k: word i takes bytes 2i, 2i + 1
        (void)hi;
        s = __dp2a_lo(w.x, (uint32_t)lo, s);
        s = __dp2a_hi(w.y, (uint32_t)lo, s);
        s = __dp2a_lo(w.z, (uint32_t)(lo >> 32), s);
        s = __dp2a_hi(w.w, (uint32_t)(lo >> 32), s);
    }
    return s;
}

// the outer prefix (coordinates o, remainders rj) holding cost rank u of the C tables; with its first
// rank below u (it belongs to an earlier slice) the next one.  false: no such outer prefix.
template <int NO>
__device__ __forceinline__ bool pair_locate(const uint64_t *__restrict__ Ct, uint64_t top, const Gens &G,
                                            uint64_t n64, uint64_t u, const uint64_t *F0, const PairGeo &pg,
                                            uint32_t (&o)[NO], uint32_t (&rj)[NO + 1])
{
    uint32_t ua[kMaxD];
#pragma unroll
    for (int j = 0; j < kMaxD; ++j) ua[j] = 0;
    const uint64_t rin = unrank(Ct, top, G, NO, n64, u, ua, F0);
    rj[0] = (uint32_t)n64;
#pragma unroll
    for (int j = 0; j < NO; ++j) {
        o[j] = ua[j];
        rj[j + 1] = rj[j] - o[j] * G.g[j];
    }
    if (rin == 0) return true;
    int i = -1;
#pragma unroll
    for (int j = 0; j < NO; ++j)
        if (o[j] > 0) i = j;
    if (i < 0) return false;
#pragma unroll
    for (int j = 0; j < NO; ++j) {
        if (j == i) o[j] -= 1;
        if (j > i) o[j] = div32(rj[j], G.g[j], pg.Mg[j]);
        if (j >= i) rj[j + 1] = rj[j] - o[j] * G.g[j];
    }
    return true;
}

// the card image of the COUNT walks: stored column vp = coset s, orbit position j -> residue column
// (s + (j mod m') Delta) mod m, R16 entries each (card[col + v m] for col + v m <= n, else 0).
// Column-major (k5_pairs): column vp is R16 consecutive entries.  Transposed (TR, k5_runs): 16-B vector vv of
// every stored column in turn -- vector (vp, vv) at byte (vv ncolv8 + vp) 16, ncolv8 = ncolv rounded up to 8 --
// so the vectors of any 8 consecutive stored columns lie in 8 distinct bank groups whatever their vector
// indices (a round's tails and remainders are conflict-free, not only its common vector index).
template <bool U8, bool TR = false>
__device__ __forceinline__ void stage_card_image(uint8_t *img, const PairGeo &pg, const uint32_t *__restrict__ cardT,
                                                 uint64_t Rcol, uint64_t n64)
{
    const uint32_t m = pg.m;
    constexpr uint32_t VE = U8 ? 16 : 8;
    if constexpr (TR) {   // one 16-B vector (VE entries of one stored column) per thread and step
        const uint32_t nvec = pg.ncolv8 * (pg.R16 / VE), per = pg.mp + pg.dup;
        for (uint32_t w = threadIdx.x; w < nvec; w += blockDim.x) {
            const uint32_t vv = w / pg.ncolv8, vp = w - vv * pg.ncolv8;
            uint32_t e[VE];
#pragma unroll
            for (int k = 0; k < (int)VE; ++k) e[k] = 0;
            if (vp < pg.ncolv) {
                const uint32_t cs = vp / per, j = (vp - cs * per) % pg.mp;
                const uint32_t col = (cs + j * pg.dlt) % m;
                const uint32_t *src = cardT + (uint64_t)col * Rcol;
#pragma unroll
                for (int k = 0; k < (int)VE; ++k) {
                    const uint32_t v = vv * VE + k;
                    if ((uint64_t)col + (uint64_t)v * m <= n64) e[k] = __ldg(src + v);
                }
            }
            uint4 pk;
            if constexpr (U8) {
                pk.x = e[0] | (e[1] << 8) | (e[2] << 16) | (e[3] << 24);
                pk.y = e[4] | (e[5] << 8) | (e[6] << 16) | (e[7] << 24);
                pk.z = e[8 % VE] | (e[9 % VE] << 8) | (e[10 % VE] << 16) | (e[11 % VE] << 24);
                pk.w = e[12 % VE] | (e[13 % VE] << 8) | (e[14 % VE] << 16) | (e[15 % VE] << 24);
            } else {
                pk.x = e[0] | (e[1] << 16);
                pk.y = e[2] | (e[3] << 16);
                pk.z = e[4] | (e[5] << 16);
                pk.w = e[6] | (e[7] << 16);
            }
            reinterpret_cast<uint4 *>(img)[w] = pk;
        }
        return;
    }
    {
        const uint32_t tot = (TR ? pg.ncolv8 : pg.ncolv) * pg.R16, per = pg.mp + pg.dup;
        for (uint32_t i0 = threadIdx.x; i0 < tot; i0 += 8 * blockDim.x) {
            uint32_t val[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t i = i0 + k * blockDim.x;
                val[k] = 0;
                uint32_t vp, v;
                if constexpr (TR) {
                    const uint32_t vv = i / (pg.ncolv8 * VE), r = i - vv * (pg.ncolv8 * VE);
                    vp = r / VE;
                    v = vv * VE + (r - vp * VE);
                } else {
                    vp = i / pg.R16;
                    v = i - vp * pg.R16;
                }
                if (i < tot && vp < pg.ncolv) {
                    const uint32_t cs = vp / per, j = (vp - cs * per) % pg.mp;
                    const uint32_t col = (cs + j * pg.dlt) % m;
                    if ((uint64_t)col + (uint64_t)v * m <= n64) val[k] = __ldg(cardT + (uint64_t)col * Rcol + v);
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t i = i0 + k * blockDim.x;
                if (i < tot) {
                    if constexpr (U8) img[i] = (uint8_t)val[k];
                    else reinterpret_cast<uint16_t *>(img)[i] = (uint16_t)val[k];
                }
            }
        }
    }
}

template <int D, int T, bool U8>
__global__ void __launch_bounds__(kCountThreads, 1)
k5_pairs(Gens G, uint64_t n64, PlanHdr *hdr, const uint64_t *__restrict__ Ct, uint64_t top,
         const uint32_t *__restrict__ cardT, uint64_t Rcol, PairGeo pg, uint32_t f0n)
{
    constexpr int L = D - T;
    static_assert(L >= 3, "pair walk: at least one outer coordinate");
    constexpr int NO = L - 2;   // outer coordinates
    constexpr uint32_t VE = U8 ? 16 : 8, VSH = U8 ? 4 : 3;   // entries per vector, log2
    griddep_wait();   // PDL: the plan header (K4) and the count tables are complete and visible
    extern __shared__ uint64_t f0s[];   // level-0 unrank column C_0[n - q g_0] (f0n entries), then the card image
    for (uint32_t q = threadIdx.x; q < f0n; q += blockDim.x) f0s[q] = __ldg(Ct + (n64 - (uint64_t)q * G.g[0]));
    uint8_t *img = reinterpret_cast<uint8_t *>(f0s + ((f0n + 1) & ~1u));
    const uint32_t m = pg.m;
    stage_card_image<U8>(img, pg, cardT, Rcol, n64);
    __syncthreads();
    int lane;
    asm volatile("mov.b32 %0, %1;" : "=r"(lane) : "r"((int)(threadIdx.x & 31)));
    const uint32_t g2 = G.g[L - 2];
    const uint64_t shard_begin = hdr->shard_begin, shard_len = hdr->shard_len, nslices = hdr->nslices,
                   gw = hdr->gss_warps, fl = hdr->slice_len, total = hdr->total_units;
    const uint32_t per = pg.mp + pg.dup;
    const uint32_t colB = pg.R16 * (U8 ? 1u : 2u);   // bytes per stored column
    uint32_t img_a;   // kept in a register (a volatile move): no per-round S2R TID / CgaCtaId re-derivation
    asm volatile("mov.b32 %0, %1;" : "=r"(img_a) : "r"(smem_addr(img)));
    const uint64_t *F0 = f0n ? f0s : nullptr;
    const bool e1 = pg.e == 1;
    uint64_t acc = 0;

    for (;;) {
        uint64_t si = 0;
        if (lane == 0) si = atomicAdd(&hdr->next_slice, 1ull);
        si = shfl_u64(si, 0);
        if (si >= nslices) break;
        const uint64_t b = shard_begin + gss_begin(si, shard_len, gw, fl),
                       e = shard_begin + gss_begin(si + 1, shard_len, gw, fl);
        if (b >= e) continue;
        uint32_t o[NO], rj[NO + 1], oe[NO], re[NO + 1];
        if (!pair_locate<NO>(Ct, top, G, n64, b, F0, pg, o, rj)) continue;
        // the slice ends at the outer prefix holding rank e (exclusive), or at the end of the stream
        const bool to_stream_end = e >= total || !pair_locate<NO>(Ct, top, G, n64, e, F0, pg, oe, re);
        auto at_end = [&]() -> bool {
            if (to_stream_end) return false;
            bool eq = true;
#pragma unroll
            for (int j = 0; j < NO; ++j) eq = eq && (o[j] == oe[j]);
            return eq;
        };
        if (at_end()) continue;   // the slice holds no outer prefix start
        // the current outer prefix (uniform): remainder R, runs - 1 A, smallest run remainder rmin, column of
        // run 0 col, its coset base cb = s (m' + dup), orbit position idx0; c = its next pair
        uint32_t R = 0, A = 0, rmin = 0, col = 0, cb = 0, idx0 = 0, c = 0;
        auto orbit = [&]() {   // coset and orbit position of col (e > 1)
            const uint32_t s = col - div32(col, pg.e, pg.Me) * pg.e;
            const uint32_t cp = div32(col - s, pg.e, pg.Me) * pg.inv;   // < m'^2
            idx0 = cp - div32(cp, pg.mp, pg.Mmp) * pg.mp;
            cb = s * per;
        };
        auto load = [&]() {
            R = rj[NO];
            A = div32(R, g2, pg.Mg2);
            rmin = R - A * g2;
            col = rmin - div32(rmin, m, pg.Mm) * m;
            if (e1) {
                const uint32_t cp = col * pg.inv;   // < m^2
                idx0 = cp - div32(cp, m, pg.Mm) * m;
                cb = 0;
            } else {
                orbit();
            }
            c = 0;
        };
        // nextCandidate over the outer coordinates; false at the end of the stream or the
        // slice.  The common step (only a_{L-3} decrements, R += g3) updates R, A, rmin, col, idx0 without
        // division.
        auto advance = [&]() -> bool {
            if (o[NO - 1] > 0) {   // the common step: only a_{L-3} decrements
                o[NO - 1] -= 1;
                rj[NO] += G.g[NO - 1];
                if (at_end()) return false;
                R = rj[NO];
                rmin += pg.S3;
                A += pg.Q3;
                const bool cy = rmin >= g2;
                if (cy) {
                    rmin -= g2;
                    A += 1;
                }
                col += cy ? pg.cs2 : pg.cs1;
                if (col >= m) col -= m;
                if (e1) {
                    idx0 += cy ? pg.is2 : pg.is1;
                    if (idx0 >= m) idx0 -= m;
                } else {
                    orbit();
                }
                c = 0;
                return true;
            }
            int i = -1;
#pragma unroll
            for (int j = 0; j < NO - 1; ++j)
                if (o[j] > 0) i = j;
            if (i < 0) return false;
#pragma unroll
            for (int j = 0; j < NO; ++j) {
                if (j == i) o[j] -= 1;
                if (j > i) o[j] = div32(rj[j], G.g[j], pg.Mg[j]);
                if (j >= i) rj[j + 1] = rj[j] - o[j] * G.g[j];
            }
            if (at_end()) return false;
            load();
            return true;
        };
        load();
        bool live = true;
        while (live) {
            // fill the 32 lanes with the next pairs of the stream (as many outer prefixes as it takes)
            uint32_t mR = 0, mA = 0, mrmin = 0, mcb = 0, mbx = 0, mby = 0, mpp = 0, mf = 0;
            bool mine = false;
            uint32_t filled = 0;
            if (A / 2 + 1 - c >= 32) {   // common pass: all 32 lanes from the current outer prefix (uniform)
                uint32_t bx = idx0 + c, by = idx0 + A + 32 * pg.mp - c - 31;
                if (pg.dup) {
                    bx -= div32(bx, pg.mp, pg.Mmp) * pg.mp;
                    by -= div32(by, pg.mp, pg.Mmp) * pg.mp;
                }
                mine = true;
                mR = R;
                mA = A;
                mrmin = rmin;
                mcb = cb;
                mbx = bx;
                mby = by;
                mpp = c;
                filled = 32;
                c += 32;
                if (c == A / 2 + 1) live = advance();
            }
            while (filled < 32 && live) {
                const uint32_t P = A / 2 + 1;
                const uint32_t take = (P - c < 32 - filled) ? P - c : 32 - filled;
                // orbit positions of the group's first X run and (minus 31) its first Y run, mod m' (uniform);
                // without duplicate columns the lanes reduce their own positions
                uint32_t bx = idx0 + c, by = idx0 + A + 32 * pg.mp - c - 31;
                if (pg.dup) {
                    bx -= div32(bx, pg.mp, pg.Mmp) * pg.mp;
                    by -= div32(by, pg.mp, pg.Mmp) * pg.mp;
                }
                if ((uint32_t)lane >= filled && (uint32_t)lane < filled + take) {
                    mine = true;
                    mR = R;
                    mA = A;
                    mrmin = rmin;
                    mcb = cb;
                    mbx = bx;
                    mby = by;
                    mpp = c;
                    mf = filled;
                }
                filled += take;
                c += take;
                if (c == P) live = advance();
            }
            // this lane's pair: X = run pp (ascending stored columns), Y = run A - pp (descending, |Y| >= |X|)
            uint32_t lenX = 0, lenY = 0, jX = 0, jY = 0;
            if (mine) {
                const uint32_t li = (uint32_t)lane - mf, pp = mpp + li;
                lenX = (2 * pp == mA) ? 0u : div32(mrmin + pp * g2, m, pg.Mm) + 1;
                lenY = div32(mR - pp * g2, m, pg.Mm) + 1;
                if (pg.dup) {   // 32 consecutive stored columns per group, ascending / descending
                    jX = mbx + li;
                    jY = mby + 31 - li;
                } else {
                    const uint32_t x = mbx + li, y = mby + 31 - li;
                    jX = x - div32(x, pg.mp, pg.Mmp) * pg.mp;
                    jY = y - div32(y, pg.mp, pg.Mmp) * pg.mp;
                }
            }
            uint32_t xa = img_a + (mcb + jX) * colB, ya = img_a + (mcb + jY) * colB;
            const uint32_t NX = lenX >> VSH, NY = lenY >> VSH;
            // vector j of Y and of X (while X has one) in the same iteration: every lane reads vector index j
            // of its columns, so the 8 lanes of a quarter-warp stay in distinct bank groups
            uint32_t sum = 0, j = 0;
            while (j < NY) {   // chunks of F iterations (F a multiple of 4: the 1-step loop runs in the last only)
                const uint32_t je = (NY - j < pg.F) ? NY : j + pg.F;
                uint32_t a0 = 0, a1 = 0;   // packed: words 0-1, 2-3 of Y and X vectors
#pragma unroll 1
                for (; j + 4 <= je; j += 4) {
                    const uint4 y0 = lds128(ya), y1 = lds128(ya + 16), y2 = lds128(ya + 32), y3 = lds128(ya + 48);
                    a0 += y0.x + y0.y;
                    a1 += y0.z + y0.w;
                    a0 += y1.x + y1.y;
                    a1 += y1.z + y1.w;
                    a0 += y2.x + y2.y;
                    a1 += y2.z + y2.w;
                    a0 += y3.x + y3.y;
                    a1 += y3.z + y3.w;
                    if (j < NX) {
                        const uint4 x0 = lds128(xa);
                        a0 += x0.x + x0.y;
                        a1 += x0.z + x0.w;
                    }
                    if (j + 1 < NX) {
                        const uint4 x1 = lds128(xa + 16);
                        a0 += x1.x + x1.y;
                        a1 += x1.z + x1.w;
                    }
                    if (j + 2 < NX) {
                        const uint4 x2 = lds128(xa + 32);
                        a0 += x2.x + x2.y;
                        a1 += x2.z + x2.w;
                    }
                    if (j + 3 < NX) {
                        const uint4 x3 = lds128(xa + 48);
                        a0 += x3.x + x3.y;
                        a1 += x3.z + x3.w;
                    }
                    ya += 64;
                    xa += 64;
                }
#pragma unroll 1
                for (; j < je; ++j) {
                    const uint4 y0 = lds128(ya);
                    a0 += y0.x + y0.y;
                    a1 += y0.z + y0.w;
                    if (j < NX) {
                        const uint4 x0 = lds128(xa);
                        a0 += x0.x + x0.y;
                        a1 += x0.z + x0.w;
                    }
                    ya += 16;
                    xa += 16;
                }
                sum = unpack_add<U8>(a1, unpack_add<U8>(a0, sum));
            }
            // the last, partial vectors (each read once; ya points at Y's vector NY, xa at X's vector NY)
            const uint32_t tX = lenX & (VE - 1), tY = lenY & (VE - 1);
            if (tY) sum = add_prefix<U8>(lds128(ya), tY, sum);
            if (tX) sum = add_prefix<U8>(lds128(xa - 16 * (NY - NX)), tX, sum);
            acc += sum;
        }
    }
    acc = warp_sum_u64(acc);
    if (lane == 0) atomicAdd((unsigned long long *)hdr->result, (unsigned long long)acc);
}

// COUNT, lane-per-run variant of the same walk (k5_runs): inside an outer prefix the rounds go DOWN the
// runs -- round r gives lane l the run k = A - 31 - 32 r + l -- so the last, partially filled round holds the
// shortest runs; each lane steps its run's remainder by -32 g2 without division (q -= QD, residue -= RD,
// borrow); the 32 runs of a round sit in 32 consecutive stored columns (orbit order), each
// lane reads vectors 0.. of its own column (the same index in every lane: conflict-free) and drops out
// after its own length (divergent trip counts instead of k5_pairs' per-pass pair setup).  Same card image,
// packed IADD3 sums (two per vector, flushed every Fr vectors), dp2a / dp4a selector tails, cost-rank
// guided slices and slice ends as k5_pairs.
template <int D, int T, bool U8>
__global__ void __launch_bounds__(kCountThreads, 1)
k5_runs(Gens G, uint64_t n64, PlanHdr *hdr, const uint64_t *__restrict__ Ct, uint64_t top,
        const uint32_t *__restrict__ cardT, uint64_t Rcol, PairGeo pg, uint32_t f0n, const uint64_t *__restrict__ W2)
{
    constexpr int L = D - T;
    static_assert(L >= 3, "run walk: at least one outer coordinate");
    constexpr int NO = L - 2;   // outer coordinates
    constexpr uint32_t VE = U8 ? 16 : 8, VSH = U8 ? 4 : 3;   // entries per vector, log2
    griddep_wait();   // PDL: the plan header (K4) and the count tables are complete and visible
    extern __shared__ uint64_t f0s[];   // level-0 unrank column C_0[n - q g_0] (f0n entries), then the card image
    for (uint32_t q = threadIdx.x; q < f0n; q += blockDim.x) f0s[q] = __ldg(Ct + (n64 - (uint64_t)q * G.g[0]));
    uint8_t *img = reinterpret_cast<uint8_t *>(f0s + ((f0n + 1) & ~1u));
    stage_card_image<U8, true>(img, pg, cardT, Rcol, n64);   // transposed: conflict-free at any vector index
    __syncthreads();
    int lane;
    asm volatile("mov.b32 %0, %1;" : "=r"(lane) : "r"((int)(threadIdx.x & 31)));
    const uint32_t m = pg.m, g2 = G.g[L - 2];
    const uint64_t shard_begin = hdr->shard_begin, shard_len = hdr->shard_len, nslices = hdr->nslices,
                   gw = hdr->gss_warps, fl = hdr->slice_len;
    const uint32_t per = pg.mp + pg.dup;
    const uint32_t VS = pg.vstride;   // bytes between consecutive vectors of a stored column (transposed image)
    uint32_t img_a;   // kept in a register (a volatile move): no per-round S2R TID / CgaCtaId re-derivation
    asm volatile("mov.b32 %0, %1;" : "=r"(img_a) : "r"(smem_addr(img)));
    const uint64_t *F0 = f0n ? f0s : nullptr;
    const bool e1 = pg.e == 1;
    uint64_t acc = 0;

    for (;;) {
        uint64_t si = 0;
        if (lane == 0) si = atomicAdd(&hdr->next_slice, 1ull);
        si = shfl_u64(si, 0);
        if (si >= nslices) break;
        const uint64_t b = shard_begin + gss_begin(si, shard_len, gw, fl),
                       e = shard_begin + gss_begin(si + 1, shard_len, gw, fl);
        if (b >= e) continue;
        // the outer prefix holding cost rank b and its first rank ob; the slice takes the outer prefixes whose
        // first rank lies in [b, e): it ends when the running rank ob (+ each outer prefix's cost
        // C_{L-2}[R] = W_{L-2}[R] + beta (A + 1) + gamma, its W value prefetched when the outer prefix starts)
        // reaches e -- no second unrank
        uint32_t o[NO], rj[NO + 1];
        uint64_t ob;
        {
            uint32_t ua[kMaxD];
#pragma unroll
            for (int j = 0; j < kMaxD; ++j) ua[j] = 0;
            const uint64_t rin = unrank(Ct, top, G, NO, n64, b, ua, F0);
            rj[0] = (uint32_t)n64;
#pragma unroll
            for (int j = 0; j < NO; ++j) {
                o[j] = ua[j];
                rj[j + 1] = rj[j] - o[j] * G.g[j];
            }
            ob = b - rin;
            if (rin != 0) {   // o began in an earlier slice: the next outer prefix
                const uint32_t R0 = rj[NO];
                ob += __ldg(W2 + R0) + pg.beta * (uint64_t)(div32(R0, g2, pg.Mg2) + 1) + pg.gamma;
                if (ob >= e) continue;
                int i = -1;
#pragma unroll
                for (int j = 0; j < NO; ++j)
                    if (o[j] > 0) i = j;
                if (i < 0) continue;
#pragma unroll
                for (int j = 0; j < NO; ++j) {
                    if (j == i) o[j] -= 1;
                    if (j > i) o[j] = div32(rj[j], G.g[j], pg.Mg[j]);
                    if (j >= i) rj[j + 1] = rj[j] - o[j] * G.g[j];
                }
            }
        }
        uint32_t R = 0, A = 0, rmin = 0, col = 0, cb = 0, idx0 = 0;
        auto orbit = [&]() {
            const uint32_t s = col - div32(col, pg.e, pg.Me) * pg.e;
            const uint32_t cp = div32(col - s, pg.e, pg.Me) * pg.inv;
            idx0 = cp - div32(cp, pg.mp, pg.Mmp) * pg.mp;
            cb = s * per;
        };
        auto load = [&]() {
            R = rj[NO];
            A = div32(R, g2, pg.Mg2);
            rmin = R - A * g2;
            col = rmin - div32(rmin, m, pg.Mm) * m;
            if (e1) {
                const uint32_t cp = col * pg.inv;
                idx0 = cp - div32(cp, m, pg.Mm) * m;
                cb = 0;
            } else {
                orbit();
            }
        };
        auto advance = [&]() -> bool {
            if (o[NO - 1] > 0) {
                o[NO - 1] -= 1;
                rj[NO] += G.g[NO - 1];
                R = rj[NO];
                rmin += pg.S3;
                A += pg.Q3;
                const bool cy = rmin >= g2;
                if (cy) {
                    rmin -= g2;
                    A += 1;
                }
                col += cy ? pg.cs2 : pg.cs1;
                if (col >= m) col -= m;
                if (e1) {
                    idx0 += cy ? pg.is2 : pg.is1;
                    if (idx0 >= m) idx0 -= m;
                } else {
                    orbit();
                }
                return true;
            }
            int i = -1;
#pragma unroll
            for (int j = 0; j < NO - 1; ++j)
                if (o[j] > 0) i = j;
            if (i < 0) return false;
#pragma unroll
            for (int j = 0; j < NO; ++j) {
                if (j == i) o[j] -= 1;
                if (j > i) o[j] = div32(rj[j], G.g[j], pg.Mg[j]);
                if (j >= i) rj[j + 1] = rj[j] - o[j] * G.g[j];
            }
            load();
            return true;
        };
        load();
        for (;;) {
            const uint64_t wR = __ldg(W2 + R);   // this outer prefix's lookups (used after its rounds)
            // this outer prefix, in DESCENDING rounds: round r gives lane l the run k = A - 31 - 32 r + l (run k
            // has remainder rmin + k g2 = R - (A - k) g2: quotient q, residue rr mod m; it lies in stored column
            // cb + orbit position idx0 + k), so the last, partially filled round holds the shortest runs.
            // back = A - k in the first round; the lane's run exists while back <= rem (rem = A - 32 r).
            const uint32_t back = 31u - (uint32_t)lane;
            const uint32_t rk = (back <= A) ? R - back * g2 : 0u;
            uint32_t q = div32(rk, m, pg.Mm), rr = rk - q * m;
            // orbit position of the round's first run (k = A - 31 - 32 r) mod m': -31 = 31 (m' - 1) mod m'
            uint32_t base;
            {
                const uint32_t t0 = idx0 + A + 31u * (pg.mp - 1u);
                base = t0 - div32(t0, pg.mp, pg.Mmp) * pg.mp;
            }
            // the longest run of this outer prefix (run A) has (R / m + 1) / VE full vectors: one flush chunk of
            // the packed sums suffices when that is at most Fr (uniform; R < one_thr)
            const bool one_chunk = R < pg.one_thr;
            for (int32_t rem = (int32_t)A; rem >= 0; rem -= 32) {
                const uint32_t len = (back <= (uint32_t)rem) ? q + 1 : 0u;
                const uint32_t jp = base + lane;   // < m' + 31 with duplicates, reduced below without
                uint32_t a = img_a + 16u * (cb + (pg.dup ? jp : jp - div32(jp, pg.mp, pg.Mmp) * pg.mp));
                const uint32_t N = len >> VSH;
                uint32_t sum = 0;
                // vectors of this lane's run up to shared byte address ae into the packed sums (the loop bound is
                // the address itself: no separate vector counter); consecutive vectors are VS bytes apart
                auto span = [&](uint32_t ae) {
                    uint32_t a0 = 0, a1 = 0;
#pragma unroll 1
                    for (; a + 3 * VS < ae; a += 4 * VS) {
                        const uint4 w0 = lds128(a), w1 = lds128(a + VS), w2 = lds128(a + 2 * VS), w3 = lds128(a + 3 * VS);
                        a0 += w0.x + w0.y;
                        a1 += w0.z + w0.w;
                        a0 += w1.x + w1.y;
                        a1 += w1.z + w1.w;
                        a0 += w2.x + w2.y;
                        a1 += w2.z + w2.w;
                        a0 += w3.x + w3.y;
                        a1 += w3.z + w3.w;
                    }
                    // the remaining 0..3 vectors: predicated loads (no divergent 1-step loop)
                    if (a < ae) {
                        const uint4 w0 = lds128(a);
                        a0 += w0.x + w0.y;
                        a1 += w0.z + w0.w;
                    }
                    if (a + VS < ae) {
                        const uint4 w1 = lds128(a + VS);
                        a0 += w1.x + w1.y;
                        a1 += w1.z + w1.w;
                    }
                    if (a + 2 * VS < ae) {
                        const uint4 w2 = lds128(a + 2 * VS);
                        a0 += w2.x + w2.y;
                        a1 += w2.z + w2.w;
                    }
                    a = ae;
                    sum = unpack_add<U8>(a1, unpack_add<U8>(a0, sum));
                };
                const uint32_t aN = a + VS * N;   // the run's partial last vector
                if (one_chunk) {
                    span(aN);
                } else {
                    while (a < aN) span((aN - a < VS * pg.Fr) ? aN : a + VS * pg.Fr);
                }
                const uint32_t tl = len & (VE - 1);
                if (tl) sum = add_prefix<U8>(lds128(a), tl, sum);
                acc += sum;
                // next round: k -= 32 (32 g2 = QD m + RD)
                const bool bw = rr < pg.RD;
                q -= pg.QD + (bw ? 1u : 0u);
                rr += (bw ? m : 0u) - pg.RD;
                base = (base >= pg.bstep) ? base - pg.bstep : base + pg.bwrap;   // base - 32 mod m'
            }
            ob += wR + pg.beta * (uint64_t)(A + 1) + pg.gamma;
            if (ob >= e || !advance()) break;
        }
    }
    acc = warp_sum_u64(acc);
    if (lane == 0) atomicAdd((unsigned long long *)hdr->result, (unsigned long long)acc);
}

// ------------------------------------------------- K5, partial memo (f2)
// topOfMemo = ltop <= n: remainders p >= ltop have no memo
// block.  The paper's Else branch then walks the tail coordinates with plain nextCandidate steps;
// here the walk is a depth-first traversal of the prefix tree in descending lex order.  A node at
// depth k (a_0..a_k fixed, remainder x = n - phi(a_0..a_k)) is a LEAF BLOCK when
//   PROG:   k = d-3: its rows Z(x; g_{d-2}, g_{d-1}) are an arithmetic progression, in closed form
//           (a_{d-2} = w_0 - j h', a_{d-1} = l_0 + j g'; g' = g_{d-2}/e, h' = g_{d-1}/e, e = gcd);
//   DIRECT: k = d-2 (d = 2, or a walk started there): at most the row (.., x / g_{d-1});
//   MEMO:   k >= L-1 and x < ltop: the suffix Z_{>=k+1}(x) of Memo[x] (its last S_{k+1}[x] rows, whose
//           coordinates L..k are zero), with a_L..a_k written over them.
// Other nodes are descended; empty subtrees (S = 0) are skipped, and a node whose remaining children
// hold no rows is left at once.  Same rows in the same order as the full-memo walk and as Alg 5
// with topOfMemo (reading R19).  Per warp: the 32 lanes evaluate 32 consecutive children of the
// current node; the leaf blocks before the first child that must be descended are copied with the
// flattened block copy of k5_walk, then the walk descends into that child, moves to the next 32
// siblings, or backs up.
template <int N>
__device__ __forceinline__ uint64_t sel_u64(const uint64_t (&v)[N], int k)
{
    uint64_t x = 0;
#pragma unroll
    for (int j = 0; j < N; ++j)
        if (j == k) x = v[j];
    return x;
}

template <int N>
__device__ __forceinline__ uint32_t sel_u32(const uint32_t (&v)[N], int k)
{
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < N; ++j)
        if (j == k) x = v[j];
    return x;
}

// BlockInfo.memo_row of a computed leaf: flag bits, then two 30-bit coordinates
constexpr uint64_t kComputed = 1ull << 63, kProg = 1ull << 62;

template <int D, int T, int MODE>
__global__ void __launch_bounds__(kWalkThreads) k5_deep(Gens G, uint64_t n64, PlanHdr *hdr,
                                                        const uint64_t *__restrict__ S, uint64_t top, uint64_t ltop,
                                                        const uint64_t *__restrict__ off,
                                                        const uint32_t *__restrict__ memo, uint32_t *out,
                                                        uint64_t out_cap_rows, uint64_t row_base, ProgGens P,
                                                        uint32_t f0n)
{
    constexpr int L = D - T;
    static_assert(T >= 1 && MODE != FZ_COUNT, "partial walk: rows of a memo with t >= 1");
    extern __shared__ uint64_t f0s[];   // level-0 unrank column S_0[n - q g_0] (f0n entries, 0 = not cached)
    for (uint32_t q = threadIdx.x; q < f0n; q += blockDim.x) f0s[q] = __ldg(S + (n64 - (uint64_t)q * G.g[0]));
    if (f0n) __syncthreads();
    __shared__ BlockInfo binfo[kWalkThreads / 32][32];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint64_t nslices = hdr->nslices, slice_len = hdr->slice_len, shard_begin = hdr->shard_begin,
                   shard_len = hdr->shard_len;
    const uint64_t gsw = hdr->gss_warps;
    if (MODE == FZ_MATERIALIZE && hdr->rows > out_cap_rows) {
        if (threadIdx.x == 0 && blockIdx.x == 0) hdr->err = 1;
        return;
    }
    if (row_base == ~0ull) row_base = hdr->row_begin;
    uint64_t acc_rows = 0, acc_hash = 0;
    BlockInfo *bi = binfo[wib];
    const uint32_t hl = G.g[D - 1];
    for (;;) {
        uint64_t s = 0;
        if (lane == 0) s = atomicAdd(&hdr->next_slice, 1ull);
        s = shfl_u64(s, 0);
        if (s >= nslices) break;
        const uint64_t begin = gsw ? gss_begin(s, shard_len, gsw, slice_len) : s * slice_len;
        uint64_t left = gsw ? gss_begin(s + 1, shard_len, gsw, slice_len) - begin
                            : ((shard_len - begin) < slice_len ? (shard_len - begin) : slice_len);
        if (left == 0) continue;
        uint64_t outpos = begin;
        // unrank the slice's first row level by level (the S tables cover every x <= n) down to the
        // leaf that holds it (same rules as the walk below); kfirst = its offset inside that leaf
        uint32_t a[D];
        uint64_t r[D + 1];
        int k = 0;
        uint64_t kfirst = shard_begin + begin;
        r[0] = n64;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            a[j] = 0;
            r[j + 1] = 0;
        }
#pragma unroll
        for (int j = 0; j < D; ++j) {
            if (j > k) continue;
            const uint64_t rj = r[j], gj = G.g[j], amax = rj / gj;
            const uint64_t *Tj = S + (uint64_t)j * top;
            const bool cached = (j == 0) && f0n != 0;
            uint64_t lo = 0, hi = amax;   // a_j = max{a : S_j[r_j - a g_j] > kfirst}
            while (lo < hi) {
                const uint64_t step = (hi - lo + 31) / 32;
                const uint64_t cand = lo + (uint64_t)(lane + 1) * step;
                const bool pred = cand <= hi && (cached ? f0s[cand] : __ldg(Tj + (rj - cand * gj))) > kfirst;
                const int m = __popc(__ballot_sync(kFull, pred));
                const uint64_t nlo = lo + (uint64_t)m * step;
                uint64_t nhi = lo + (uint64_t)(m + 1) * step - 1;
                hi = nhi > hi ? hi : nhi;
                lo = nlo;
            }
            a[j] = (uint32_t)lo;
            if (lo + 1 <= amax) kfirst -= cached ? f0s[lo + 1] : __ldg(Tj + (rj - (lo + 1) * gj));
            r[j + 1] = rj - lo * gj;
            if (!(j + 3 == D || j + 2 == D || (j + 1 >= L && r[j + 1] < ltop))) ++k;
        }
        while (left > 0) {
            const uint64_t rk = sel_u64(r, k);
            const uint64_t gk = G.g[k];
            const uint32_t v = sel_u32(a, k);
            const int32_t vv = (int32_t)v - lane;
            const bool valid = vv >= 0;
            const uint64_t p = valid ? rk - (uint64_t)vv * gk : 0;
            // child leaf type and rows
            uint64_t cnt = 0, mrow = 0;
            bool leaf = false;
            if (k + 3 == D) {   // PROG
                uint32_t w0 = 0, l0 = 0;
                cnt = valid ? prog_block(P, (uint32_t)p, w0, l0) : 0;
                if (lane == 0 && kfirst) {
                    w0 -= (uint32_t)kfirst * P.h1;
                    l0 += (uint32_t)kfirst * P.g1;
                }
                mrow = kComputed | kProg | ((uint64_t)l0 << 30) | w0;
                leaf = true;
            } else if (k + 2 == D) {   // DIRECT
                cnt = (valid && p % hl == 0) ? 1 : 0;
                mrow = kComputed | ((p / hl) << 30);
                leaf = true;
            } else {
                cnt = valid ? __ldg(S + (uint64_t)(k + 1) * top + p) : 0;
                leaf = (k + 1 >= L) && p < ltop;
                if (leaf && cnt) mrow = __ldg(off + p + 1) - cnt + (lane == 0 ? kfirst : 0);
            }
            const unsigned dball = __ballot_sync(kFull, !leaf && cnt > 0);
            const int dl = dball ? __ffs(dball) - 1 : 32;
            // rows this lane's leaf offers, clamped to the slice's budget (K4 keeps slices <= 2^26 rows), so
            // the 32-lane u32 scan cannot overflow on closed-form leaves (|Z(x; g, h)| is not bounded by the
            // memo-block guard)
            uint64_t c64 = (leaf && lane < dl) ? cnt : 0ull;
            if (lane == 0) c64 -= kfirst;
            uint32_t c = (uint32_t)(c64 < left ? c64 : left);
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
            constexpr int UNR = 1;   // (UNR = 4 measured slower here: the computed rows need no loads)
            int e0 = 0;
            for (uint32_t q0 = 0; q0 < use; q0 += 32 * UNR) {
                uint32_t wv[UNR][D];
                bool ok[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const uint32_t qb = q0 + 32 * u;
                    const unsigned bit = (cc > 0 && excl >= qb && excl - qb < 32) ? (1u << (excl - qb)) : 0u;
                    const unsigned M = __reduce_or_sync(kFull, bit);
                    if (qb != 0) e0 += (int)(M & 1u);
                    const uint32_t q = qb + lane;
                    const int e = e0 + __popc(M & ((2u << lane) - 2u));
                    e0 += __popc(M & 0xfffffffeu);
                    ok[u] = q < use;
                    if (ok[u]) {
                        const BlockInfo info = bi[e];
                        const uint32_t jq = q - info.start;
                        const uint64_t mr = info.memo_row;
                        uint32_t tw[T];
#pragma unroll
                        for (int j = 0; j < T; ++j) tw[j] = 0;
                        uint32_t c2 = 0, c1 = 0;   // computed a_{d-2}, a_{d-1}
                        if (mr & kComputed) {
                            c2 = (uint32_t)(mr & 0x3fffffffu) - jq * P.h1;
                            c1 = (uint32_t)((mr >> 30) & 0x3fffffffu) + jq * P.g1;
                        } else {
                            load_tail<T>(memo + (mr + jq) * T, tw);
                        }
#pragma unroll
                        for (int j = 0; j < D; ++j) {
                            // j < k: the walk's prefix; j == k: the child; j > k: the leaf's rows
                            uint32_t x = (j >= L) ? tw[j >= L ? j - L : 0] : 0u;
                            if (mr & kComputed) {
                                if (j == D - 2) x = c2;
                                if (j == D - 1) x = c1;
                            }
                            if (j < k) x = a[j];
                            if (j == k) x = info.v;
                            wv[u][j] = x;
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    if (!ok[u]) continue;
                    const uint32_t q = q0 + 32 * u + lane;
                    if constexpr (MODE == FZ_MATERIALIZE) {
                        store_row<D>(out + (outpos + q) * (uint64_t)D, wv[u]);
                    } else {
                        acc_hash += row_hash<D>(row_base + outpos + q, wv[u]);
                    }
                }
            }
            __syncwarp();
            acc_rows += (lane == 0) ? use : 0;
            outpos += use;
            left -= use;
            if (left == 0) break;
            if (dl < 32) {   // descend into child v - dl
                const uint32_t av = v - (uint32_t)dl;
                const uint64_t rn = rk - (uint64_t)av * gk;
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    if (j == k) a[j] = av;
                    if (j == k + 1) a[j] = (uint32_t)(rn / G.g[j]);
                    if (j == k + 1) r[j] = rn;
                }
                ++k;
                continue;
            }
            // rows left under the current prefix with a_k <= w: S_k[r_k] - S_k[r_k - (w + 1) g_k]
            auto rows_left = [&](int kk, uint32_t w) {
                const uint64_t rr = sel_u64(r, kk), nx = ((uint64_t)w + 1) * G.g[kk];
                const uint64_t *Sk = S + (uint64_t)kk * top;
                return __ldg(Sk + rr) > (nx <= rr ? __ldg(Sk + (rr - nx)) : 0ull);
            };
            if (v >= 32 && (k + 3 >= D || rows_left(k, v - 32))) {   // next 32 siblings (PROG: no test)
#pragma unroll
                for (int j = 0; j < D; ++j)
                    if (j == k) a[j] = v - 32;
                continue;
            }
            // no rows among the remaining children: back up to the nearest ancestor with a next sibling
            // that still has rows (nextCandidate)
            bool more = false;
            while (k > 0) {
                --k;
                const uint32_t ak = sel_u32(a, k);
                if (ak > 0 && rows_left(k, ak - 1)) {
#pragma unroll
                    for (int j = 0; j < D; ++j)
                        if (j == k) a[j] = ak - 1;
                    more = true;
                    break;
                }
            }
            if (!more) break;   // end of stream
        }
    }
    acc_rows = warp_sum_u64(acc_rows);
    if (lane == 0) atomicAdd((unsigned long long *)hdr->result, (unsigned long long)acc_rows);
    if constexpr (MODE == FZ_HASH) {
        acc_hash = warp_sum_u64(acc_hash);
        if (lane == 0) atomicAdd((unsigned long long *)(hdr->result + 1), (unsigned long long)acc_hash);
    }
}

// ------------------------------------------------------- end-to-end ring
// fz_run_host: fold a finished chunk's {rows, hash, err} into the run's accumulator (stream-ordered after
// the chunk's K5, before the next chunk's K4 reuses the plan header).
__global__ void __launch_bounds__(32) k_run_acc(const PlanHdr *h, uint64_t *acc)
{
    if (threadIdx.x == 0) {
        acc[0] += h->result[0];
        acc[1] += h->result[1];
        acc[2] |= h->err;
    }
}

// ------------------------------------------------------------ K5, t = d
// Full DP table (t = d; Alg 2/3's product): Z(n) is the memo
// block Memo[n] itself; the shard's rows are copied (MATERIALIZE), counted, or hashed.
template <int D, int MODE>
__global__ void __launch_bounds__(256) k5_table(PlanHdr *hdr, const uint64_t *__restrict__ off, uint64_t n,
                                                 const uint32_t *__restrict__ memo, uint32_t *out, uint64_t out_cap_rows,
                                                 uint64_t row_base)
{
    const uint64_t rows = hdr->rows, rb = hdr->row_begin;
    if (MODE == FZ_MATERIALIZE && rows > out_cap_rows) {
        if (threadIdx.x == 0 && blockIdx.x == 0) hdr->err = 1;
        return;
    }
    if (row_base == ~0ull) row_base = rb;
    const uint64_t base = __ldg(off + n) + rb;
    uint64_t acc_h = 0;
    for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t w[D];
        load_tail<D>(memo + (base + r) * D, w);
        if constexpr (MODE == FZ_MATERIALIZE) store_row<D>(out + r * D, w);
        if constexpr (MODE == FZ_HASH) acc_h += row_hash<D>(row_base + r, w);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd((unsigned long long *)hdr->result, (unsigned long long)rows);
    if constexpr (MODE == FZ_HASH) {
        acc_h = warp_sum_u64(acc_h);
        if ((threadIdx.x & 31) == 0) atomicAdd((unsigned long long *)(hdr->result + 1), (unsigned long long)acc_h);
    }
}

}  // namespace fzk
