// fz.cu -- host side of the C ABI declared in include/fz.h.
//
// A1 validation and sizing run on the host (uint64 arithmetic with overflow
// checks); everything on the data path (A2-A9) is a kernel in fz_kernels.cuh
// launched on the caller's stream into caller-owned device memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/fz.h"
#include "fz_kernels.cuh"

using fzk::Gens;
using fzk::PlanParams;
using fzk::Slice;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;
uint64_t g_memo_cap = 8000000000ull;

fz_status fail(fz_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

fz_status cuda_check(const char *what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(FZ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return FZ_OK;
}

#define FZ_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) return fail(FZ_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

int device_sms()
{
    static thread_local int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    }
    return sms;
}

// ------------------------------------------------------------ host tables (A1)
// The host recomputes the count tables only to size workspaces and to cut
// shard boundaries before any device work (no device round trip).  The device
// count pass (K1) is what the kernels use.
struct HostTables {
    std::vector<uint64_t> S;   // (d+1) * top
    std::vector<uint64_t> W;   // (L+1) * top
};

fz_status host_tables(const uint32_t *g, int d, int L, uint64_t top, HostTables &H)
{
    try {
        H.S.assign((size_t)(d + 1) * top, 0);
        H.W.assign((size_t)(L + 1) * top, 0);
    } catch (const std::bad_alloc &) {
        return fail(FZ_ECAP, "host tables for top=%llu do not fit host memory", (unsigned long long)top);
    }
    uint64_t *S = H.S.data(), *W = H.W.data();
    S[(size_t)d * top] = 1;
    for (int i = d - 1; i >= 0; --i) {
        const uint64_t *nx = S + (size_t)(i + 1) * top;
        uint64_t *cu = S + (size_t)i * top;
        for (uint64_t x = 0; x < top; ++x) {
            uint64_t v = nx[x];
            if (x >= g[i] && __builtin_add_overflow(v, cu[x - g[i]], &v))
                return fail(FZ_ERANGE, "|Z(%llu; g_%d..g_d)| exceeds 2^64", (unsigned long long)x, i + 1);
            cu[x] = v;
        }
    }
    for (uint64_t x = 0; x < top; ++x) W[(size_t)L * top + x] = 1;
    for (int j = L - 1; j >= 0; --j) {
        const uint64_t *nx = W + (size_t)(j + 1) * top;
        uint64_t *cu = W + (size_t)j * top;
        for (uint64_t x = 0; x < top; ++x) {
            uint64_t v = nx[x];
            if (x >= g[j] && __builtin_add_overflow(v, cu[x - g[j]], &v))
                return fail(FZ_ERANGE, "leading-prefix count at x=%llu exceeds 2^64", (unsigned long long)x);
            cu[x] = v;
        }
    }
    return FZ_OK;
}

struct Layout {
    uint64_t S, W, card, off, links, rows, counter, total;
};

struct Sizing {
    int d, t, L;
    uint64_t top;
    uint64_t entries = 0, max_card = 0, window = 0, ring_rows = 0, batches = 0;
    uint32_t batch = 0;
    int fill_mode = 0;
    Layout lay{};
};

constexpr uint64_t kRingBytesMax = 160 * 1024;

fz_status validate(const uint32_t *g, int d, int t, uint64_t top)
{
    if (!g) return fail(FZ_EINVAL, "gens is NULL");
    if (d < 1 || d > FZ_MAX_D) return fail(FZ_EINVAL, "d=%d outside [1, %d]", d, FZ_MAX_D);
    if (t < 0 || t > d - 1) return fail(FZ_EINVAL, "t=%d outside [0, d-1=%d]", t, d - 1);
    for (int i = 0; i < d; ++i)
        if (g[i] == 0) return fail(FZ_EINVAL, "g_%d = 0 (generators must be positive)", i + 1);
    if (top == 0) return fail(FZ_EINVAL, "top must be >= 1");
    if (top > (1ull << 28)) return fail(FZ_ERANGE, "top=%llu above 2^28", (unsigned long long)top);
    return FZ_OK;
}

fz_status size_memo(const uint32_t *g, int d, int t, uint64_t top, int with_entries, const HostTables &H, Sizing &z)
{
    z.d = d;
    z.t = t;
    z.L = d - t;
    z.top = top;
    const int L = z.L;
    const uint64_t *card = H.S.data() + (size_t)L * top;
    uint64_t entries = 0, mx = 0;
    for (uint64_t x = 0; x < top; ++x) {
        if (__builtin_add_overflow(entries, card[x], &entries)) return fail(FZ_ERANGE, "memo entries exceed 2^64");
        mx = std::max(mx, card[x]);
    }
    if (mx >= (1ull << 26)) return fail(FZ_ERANGE, "a memo block has %llu >= 2^26 rows", (unsigned long long)mx);
    z.entries = entries;
    z.max_card = mx;
    uint32_t b = 0xffffffffu, hmax = 0;
    for (int i = L; i < d; ++i) {
        b = std::min(b, g[i]);
        hmax = std::max(hmax, g[i]);
    }
    if (t == 0) b = 1;
    z.batch = b;
    z.batches = (top + b - 1) / b;
    // live window of the recurrence: rows of [x0 - hmax, x0 + b) for every batch start x0
    std::vector<uint64_t> off(top + 1, 0);
    for (uint64_t x = 0; x < top; ++x) off[x + 1] = off[x] + card[x];
    uint64_t win = 0;
    for (uint64_t x0 = 0; x0 < top; x0 += b) {
        uint64_t lo = x0 > hmax ? x0 - hmax : 0, hi = std::min<uint64_t>(x0 + b, top);
        win = std::max(win, off[hi] - off[lo]);
    }
    z.window = win;
    uint64_t rows_bytes = 0;
    if (with_entries && t > 0) {
        if (entries > (g_memo_cap / (4ull * t)))
            return fail(FZ_ECAP, "memo of %llu rows x %d coords exceeds the cap of %llu bytes",
                        (unsigned long long)entries, t, (unsigned long long)g_memo_cap);
        rows_bytes = entries * 4ull * t;
        uint64_t ring = 1;
        while (ring < win) ring <<= 1;
        z.ring_rows = ring;
        if (entries >= (1ull << 25) || entries / z.batches > 16384)
            z.fill_mode = 3;
        else if (ring * 4ull * t <= kRingBytesMax)
            z.fill_mode = 1;
        else
            z.fill_mode = 2;
    } else {
        z.fill_mode = 0;
    }
    Layout &l = z.lay;
    uint64_t p = 256;                                   // header
    l.S = p;       p = align_up(p + 8ull * (d + 1) * top, 256);
    l.W = p;       p = align_up(p + 8ull * (L + 1) * top, 256);
    l.card = p;    p = align_up(p + 4ull * top, 256);
    l.off = p;     p = align_up(p + 8ull * (top + 1), 256);
    l.counter = p; p = align_up(p + 256, 256);
    l.links = p;   if (z.fill_mode == 1 || z.fill_mode == 2) p = align_up(p + 8ull * entries, 256);
    l.rows = p;    p = align_up(p + rows_bytes, 256);
    l.total = p;
    return FZ_OK;
}

}  // namespace

struct fz_memo {
    Sizing z;
    uint32_t g[FZ_MAX_D];
    int with_entries;
    HostTables H;
    char *ws;
    uint64_t *S, *W, *off;
    uint32_t *card, *rows;
    uint64_t *links;
    unsigned int *counter;
};

struct fz_plan {
    const fz_memo *m;
    PlanParams P;
    fz_mode mode;
    int shard, nshards;
    uint64_t shard_row_begin, shard_rows;
    char *d_plan;
};

// ------------------------------------------------------------ launch helpers
namespace {

Gens make_gens(const uint32_t *g, int d)
{
    Gens G;
    for (int i = 0; i < FZ_MAX_D; ++i) G.g[i] = i < d ? g[i] : 1u;
    return G;
}

template <int T>
fz_status launch_fill_t(const fz_memo *m, cudaStream_t s)
{
    const Sizing &z = m->z;
    if (z.fill_mode == 1 || z.fill_mode == 2) {
        const int threads = 1024;
        const bool ring = z.fill_mode == 1;
        const size_t smem = ring ? (size_t)(z.ring_rows * 4ull * T) : 0;
        if (ring) {
            FZ_CUDA(cudaFuncSetAttribute(fzk::k3_fill_single<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
            fzk::k3_fill_single<T, true><<<1, threads, smem, s>>>(m->off, m->links, m->rows, z.top, z.batch,
                                                                  z.ring_rows - 1);
        } else {
            fzk::k3_fill_single<T, false><<<1, threads, 0, s>>>(m->off, m->links, m->rows, z.top, z.batch, 0);
        }
        ++g_launches;
        return cuda_check("k3_fill_single");
    }
    if (z.fill_mode == 3) {
        int per_sm = 0;
        FZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fzk::k3_fill_grid<T>, 256, 0));
        if (per_sm < 1) return fail(FZ_ECUDA, "k3_fill_grid cannot be resident");
        int blocks = device_sms() * std::min(per_sm, 4);
        FZ_CUDA(cudaMemsetAsync(m->counter, 0, 256, s));
        Gens G = make_gens(m->g, z.d);
        int L = z.L;
        uint64_t top = z.top;
        uint32_t b = z.batch;
        const uint64_t *S = m->S, *off = m->off;
        uint32_t *rows = m->rows;
        unsigned int *counter = m->counter;
        void *args[] = {&G, &L, &top, &b, &S, &off, &rows, &counter};
        FZ_CUDA(cudaLaunchCooperativeKernel((const void *)fzk::k3_fill_grid<T>, blocks, 256, args, 0, s));
        ++g_launches;
        return cuda_check("k3_fill_grid");
    }
    return FZ_OK;
}

template <int T = 1>
fz_status launch_fill(const fz_memo *m, cudaStream_t s)
{
    if constexpr (T < FZ_MAX_D) {
        if (m->z.t == T) return launch_fill_t<T>(m, s);
        return launch_fill<T + 1>(m, s);
    } else {
        return fail(FZ_EINVAL, "t=%d not instantiated", m->z.t);
    }
}

struct WalkArgs {
    Gens G;
    PlanParams P;
    const Slice *slices;
    const uint32_t *card;
    const uint64_t *off;
    const uint32_t *memo;
    uint32_t *out;
    uint64_t row_base;
    uint64_t *result;
};

template <int D, int T, int MODE>
fz_status launch_walk_dtm(const WalkArgs &a, cudaStream_t s)
{
    const int threads = fzk::kWalkThreads;
    uint64_t want = (a.P.nslices * 32 + threads - 1) / threads;
    int per_sm = 8;
    uint64_t blocks = std::min<uint64_t>(want, (uint64_t)device_sms() * per_sm);
    if (blocks == 0) blocks = 1;
    fzk::k5_walk<D, T, MODE><<<(unsigned)blocks, threads, 0, s>>>(a.G, a.P, a.slices, a.card, a.off, a.memo, a.out,
                                                                   a.row_base, a.result);
    ++g_launches;
    return cuda_check("k5_walk");
}

template <int D, int T = 0>
fz_status launch_walk_d(int t, int mode, const WalkArgs &a, cudaStream_t s)
{
    if constexpr (T < D) {
        if (t == T) {
            switch (mode) {
            case FZ_MATERIALIZE: return launch_walk_dtm<D, T, FZ_MATERIALIZE>(a, s);
            case FZ_COUNT: return launch_walk_dtm<D, T, FZ_COUNT>(a, s);
            default: return launch_walk_dtm<D, T, FZ_HASH>(a, s);
            }
        }
        return launch_walk_d<D, T + 1>(t, mode, a, s);
    } else {
        return fail(FZ_EINVAL, "t=%d not instantiated for d=%d", t, D);
    }
}

template <int D = 1>
fz_status launch_walk(int d, int t, int mode, const WalkArgs &a, cudaStream_t s)
{
    if constexpr (D <= FZ_MAX_D) {
        if (d == D) return launch_walk_d<D>(t, mode, a, s);
        return launch_walk<D + 1>(d, t, mode, a, s);
    } else {
        return fail(FZ_EINVAL, "d=%d not instantiated", d);
    }
}

// host-side rank / unrank over the host tables (shard boundaries for COUNT)
uint64_t host_row_rank(const fz_memo *m, uint64_t n, const uint32_t *a)
{
    const uint64_t top = m->z.top;
    uint64_t r = n, R = 0;
    for (int j = 0; j < m->z.L; ++j) {
        const uint64_t nxt = (uint64_t)(a[j] + 1ull) * m->g[j];
        if (nxt <= r) R += m->H.S[(size_t)j * top + (r - nxt)];
        r -= (uint64_t)a[j] * m->g[j];
    }
    return R;
}

void host_unrank_prefix(const fz_memo *m, uint64_t n, uint64_t R, uint32_t *a)
{
    const uint64_t top = m->z.top;
    uint64_t r = n;
    for (int j = 0; j < m->z.L; ++j) {
        const uint64_t *Tj = m->H.W.data() + (size_t)j * top;
        const uint64_t gj = m->g[j], amax = r / gj;
        uint64_t lo = 0, hi = amax;   // largest a with Tj[r - a gj] > R
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo + 1) / 2;
            if (Tj[r - mid * gj] > R) lo = mid; else hi = mid - 1;
        }
        a[j] = (uint32_t)lo;
        R -= (lo + 1 <= amax) ? Tj[r - (lo + 1) * gj] : 0;
        r -= lo * gj;
    }
}

fz_status shard_units(const fz_memo *m, uint64_t n, fz_mode mode, int nshards, int s, uint64_t &ub, uint64_t &ul,
                      uint64_t &rb, uint64_t &rl)
{
    const uint64_t top = m->z.top;
    const uint64_t rows_total = m->H.S[n];
    if (mode == FZ_COUNT) {
        const uint64_t P = m->H.W[n];
        auto cut = [&](int k) { return (uint64_t)((unsigned __int128)P * (unsigned)k / (unsigned)nshards); };
        ub = cut(s);
        ul = cut(s + 1) - ub;
        auto rowat = [&](uint64_t pidx) -> uint64_t {
            if (pidx >= P) return rows_total;
            uint32_t a[FZ_MAX_D] = {0};
            host_unrank_prefix(m, n, pidx, a);
            return host_row_rank(m, n, a);
        };
        rb = rowat(ub);
        rl = rowat(ub + ul) - rb;
    } else {
        auto cut = [&](int k) { return (uint64_t)((unsigned __int128)rows_total * (unsigned)k / (unsigned)nshards); };
        ub = cut(s);
        ul = cut(s + 1) - ub;
        rb = ub;
        rl = ul;
    }
    (void)top;
    return FZ_OK;
}

uint64_t slice_len_for(fz_mode mode, uint64_t units)
{
    const uint64_t target = (uint64_t)device_sms() * 8 * (fzk::kWalkThreads / 32) * 4;
    uint64_t len = (units + target - 1) / std::max<uint64_t>(target, 1);
    const uint64_t floor_len = (mode == FZ_COUNT) ? 1024 : 256;
    return std::max(len, floor_len);
}

constexpr uint64_t kPlanHeader = 256;

// plan workspace for a shard of `units` units (shards differ by at most one unit)
uint64_t plan_bytes_for(fz_mode mode, uint64_t units)
{
    const uint64_t len = slice_len_for(mode, units + 1);
    const uint64_t ns = (units + 1 + len - 1) / len;
    return kPlanHeader + align_up(ns * sizeof(Slice), 256);
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char *fz_last_error(void) { return g_err.c_str(); }
uint64_t fz_launch_count(void) { return g_launches; }
void fz_set_memo_cap(uint64_t bytes) { g_memo_cap = bytes ? bytes : 8000000000ull; }

fz_status fz_memo_workspace_bytes(const uint32_t *gens, int d, int t, uint64_t top, int with_entries,
                                  uint64_t *bytes)
{
    if (!bytes) return fail(FZ_EINVAL, "bytes is NULL");
    fz_status st = validate(gens, d, t, top);
    if (st) return st;
    HostTables H;
    if ((st = host_tables(gens, d, d - t, top, H))) return st;
    Sizing z;
    if ((st = size_memo(gens, d, t, top, with_entries, H, z))) return st;
    *bytes = z.lay.total;
    return FZ_OK;
}

fz_status fz_memo_build(const uint32_t *gens, int d, int t, uint64_t top, int with_entries, void *d_ws,
                        uint64_t ws_bytes, void *stream, fz_memo **out)
{
    if (!out) return fail(FZ_EINVAL, "out is NULL");
    *out = nullptr;
    fz_status st = validate(gens, d, t, top);
    if (st) return st;
    if (!d_ws || ((uintptr_t)d_ws & 255)) return fail(FZ_EINVAL, "workspace NULL or not 256-byte aligned");
    fz_memo *m = new (std::nothrow) fz_memo();
    if (!m) return fail(FZ_ECAP, "host allocation failed");
    for (int i = 0; i < d; ++i) m->g[i] = gens[i];
    m->with_entries = with_entries ? 1 : 0;
    if ((st = host_tables(gens, d, d - t, top, m->H)) || (st = size_memo(gens, d, t, top, with_entries, m->H, m->z))) {
        delete m;
        return st;
    }
    const Sizing &z = m->z;
    if (ws_bytes < z.lay.total) {
        delete m;
        return fail(FZ_ENOSPC, "workspace %llu B < required %llu B", (unsigned long long)ws_bytes,
                    (unsigned long long)z.lay.total);
    }
    char *w = (char *)d_ws;
    m->ws = w;
    m->S = (uint64_t *)(w + z.lay.S);
    m->W = (uint64_t *)(w + z.lay.W);
    m->card = (uint32_t *)(w + z.lay.card);
    m->off = (uint64_t *)(w + z.lay.off);
    m->counter = (unsigned int *)(w + z.lay.counter);
    m->links = (uint64_t *)(w + z.lay.links);
    m->rows = (uint32_t *)(w + z.lay.rows);
    cudaStream_t s = (cudaStream_t)stream;
    Gens G = make_gens(m->g, d);
    fzk::k1_tables<<<1, 1024, 0, s>>>(G, d, z.L, top, m->S, m->W, m->card, m->off);
    ++g_launches;
    if ((st = cuda_check("k1_tables"))) { delete m; return st; }
    if (z.fill_mode == 1 || z.fill_mode == 2) {
        uint64_t blocks = std::min<uint64_t>((top * 32 + 255) / 256, (uint64_t)device_sms() * 16);
        fzk::k3_links<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, s>>>(G, z.L, t, top, m->S, m->off, m->links);
        ++g_launches;
        if ((st = cuda_check("k3_links"))) { delete m; return st; }
    }
    if ((st = launch_fill(m, s))) { delete m; return st; }
    *out = m;
    return FZ_OK;
}

fz_status fz_memo_get_info(const fz_memo *m, fz_memo_info *info)
{
    if (!m || !info) return fail(FZ_EINVAL, "NULL argument");
    const Sizing &z = m->z;
    info->d = z.d;
    info->t = z.t;
    info->top = z.top;
    info->entries = z.entries;
    info->max_card = z.max_card;
    info->batches = z.batches;
    info->batch = z.batch;
    info->fill_mode = z.fill_mode;
    info->window_rows = z.window;
    return FZ_OK;
}

fz_status fz_memo_device_views(const fz_memo *m, const uint32_t **rows, const uint64_t **off, const uint64_t **S)
{
    if (!m) return fail(FZ_EINVAL, "NULL memo");
    if (rows) *rows = m->rows;
    if (off) *off = m->off;
    if (S) *S = m->S;
    return FZ_OK;
}

fz_status fz_count(const fz_memo *m, uint64_t n, void *stream, uint64_t *count)
{
    if (!m || !count) return fail(FZ_EINVAL, "NULL argument");
    if (n >= m->z.top) return fail(FZ_EINVAL, "n=%llu >= top=%llu", (unsigned long long)n, (unsigned long long)m->z.top);
    cudaStream_t s = (cudaStream_t)stream;
    FZ_CUDA(cudaMemcpyAsync(count, m->S + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    FZ_CUDA(cudaStreamSynchronize(s));
    return FZ_OK;
}

fz_status fz_shard_rows(const fz_memo *m, uint64_t n, fz_mode mode, int nshards, uint64_t *row_begin, uint64_t *rows)
{
    if (!m || nshards < 1) return fail(FZ_EINVAL, "NULL memo or nshards < 1");
    if (n >= m->z.top) return fail(FZ_EINVAL, "n >= top");
    for (int s = 0; s < nshards; ++s) {
        uint64_t ub, ul, rb, rl;
        shard_units(m, n, mode, nshards, s, ub, ul, rb, rl);
        if (row_begin) row_begin[s] = rb;
        if (rows) rows[s] = rl;
    }
    return FZ_OK;
}

static fz_status plan_params(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, PlanParams &P,
                             uint64_t &rb, uint64_t &rl)
{
    if (!m) return fail(FZ_EINVAL, "NULL memo");
    if (mode != FZ_MATERIALIZE && mode != FZ_COUNT && mode != FZ_HASH) return fail(FZ_EINVAL, "bad mode %d", (int)mode);
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(FZ_EINVAL, "shard %d of %d", shard, nshards);
    if (n >= m->z.top) return fail(FZ_EINVAL, "n=%llu >= top=%llu (full memo required)", (unsigned long long)n,
                                   (unsigned long long)m->z.top);
    if (mode != FZ_COUNT && m->z.t > 0 && !m->with_entries)
        return fail(FZ_EINVAL, "memo built without entries; only FZ_COUNT is possible");
    uint64_t ub, ul;
    shard_units(m, n, mode, nshards, shard, ub, ul, rb, rl);
    P.n = n;
    P.top = m->z.top;
    P.shard_begin = ub;
    P.shard_len = ul;
    P.slice_len = slice_len_for(mode, ul);
    P.nslices = (ul + P.slice_len - 1) / P.slice_len;
    P.d = m->z.d;
    P.t = m->z.t;
    P.L = m->z.L;
    P.mode = (int)mode;
    return FZ_OK;
}

fz_status fz_plan_workspace_bytes(const fz_memo *m, uint64_t n, fz_mode mode, int nshards, uint64_t *bytes)
{
    if (!bytes) return fail(FZ_EINVAL, "bytes is NULL");
    uint64_t mx = 0;
    for (int s = 0; s < std::max(nshards, 1); ++s) {
        PlanParams P;
        uint64_t rb, rl;
        fz_status st = plan_params(m, n, mode, s, nshards, P, rb, rl);
        if (st) return st;
        mx = std::max(mx, P.nslices);
    }
    *bytes = kPlanHeader + align_up(mx * sizeof(Slice), 256);
    return FZ_OK;
}

fz_status fz_plan_create(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, void *d_plan,
                         uint64_t plan_bytes, void *stream, fz_plan **out)
{
    if (!out) return fail(FZ_EINVAL, "out is NULL");
    *out = nullptr;
    if (!d_plan || ((uintptr_t)d_plan & 255)) return fail(FZ_EINVAL, "plan workspace NULL or misaligned");
    PlanParams P;
    uint64_t rb, rl;
    fz_status st = plan_params(m, n, mode, shard, nshards, P, rb, rl);
    if (st) return st;
    const uint64_t need = kPlanHeader + align_up(P.nslices * sizeof(Slice), 256);
    if (plan_bytes < need)
        return fail(FZ_ENOSPC, "plan workspace %llu B < required %llu B", (unsigned long long)plan_bytes,
                    (unsigned long long)need);
    fz_plan *p = new (std::nothrow) fz_plan();
    if (!p) return fail(FZ_ECAP, "host allocation failed");
    p->m = m;
    p->P = P;
    p->mode = mode;
    p->shard = shard;
    p->nshards = nshards;
    p->shard_row_begin = rb;
    p->shard_rows = rl;
    p->d_plan = (char *)d_plan;
    cudaStream_t s = (cudaStream_t)stream;
    uint64_t *result = (uint64_t *)p->d_plan;
    Slice *slices = (Slice *)(p->d_plan + kPlanHeader);
    Gens G = make_gens(m->g, m->z.d);
    uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>((P.nslices * 32 + 255) / 256, 4096));
    fzk::k4_plan<<<(unsigned)blocks, 256, 0, s>>>(G, P, m->S, m->W, slices, result);
    ++g_launches;
    if ((st = cuda_check("k4_plan"))) {
        delete p;
        return st;
    }
    *out = p;
    return FZ_OK;
}

void fz_plan_free(fz_plan *p) { delete p; }

fz_status fz_plan_get_shard(const fz_plan *p, uint64_t *row_begin, uint64_t *rows, uint64_t *nslices)
{
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    if (row_begin) *row_begin = p->shard_row_begin;
    if (rows) *rows = p->shard_rows;
    if (nslices) *nslices = p->P.nslices;
    return FZ_OK;
}

fz_status fz_enumerate_launch(const fz_plan *p, uint32_t *d_out, uint64_t out_capacity_rows, uint64_t row_base,
                              void *stream)
{
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    const fz_memo *m = p->m;
    if (p->mode == FZ_MATERIALIZE) {
        if (!d_out && p->shard_rows) return fail(FZ_EINVAL, "d_out is NULL");
        if (((uintptr_t)d_out & 15)) return fail(FZ_EINVAL, "d_out not 16-byte aligned");
        if (out_capacity_rows < p->shard_rows)
            return fail(FZ_ENOSPC, "output holds %llu rows, shard has %llu", (unsigned long long)out_capacity_rows,
                        (unsigned long long)p->shard_rows);
    }
    if (p->P.nslices == 0) return FZ_OK;
    WalkArgs a;
    a.G = make_gens(m->g, m->z.d);
    a.P = p->P;
    a.slices = (const Slice *)(p->d_plan + kPlanHeader);
    a.card = m->card;
    a.off = m->off;
    a.memo = m->rows;
    a.out = d_out;
    a.row_base = row_base;
    a.result = (uint64_t *)p->d_plan;
    return launch_walk(m->z.d, m->z.t, (int)p->mode, a, (cudaStream_t)stream);
}

fz_status fz_plan_result(const fz_plan *p, void *stream, uint64_t *rows, uint64_t *hash)
{
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    uint64_t h[2] = {0, 0};
    cudaStream_t s = (cudaStream_t)stream;
    FZ_CUDA(cudaMemcpyAsync(h, p->d_plan, sizeof h, cudaMemcpyDeviceToHost, s));
    FZ_CUDA(cudaStreamSynchronize(s));
    if (rows) *rows = h[0];
    if (hash) *hash = h[1];
    return FZ_OK;
}

fz_status fz_plan_result_ptr(const fz_plan *p, uint64_t **d_result)
{
    if (!p || !d_result) return fail(FZ_EINVAL, "NULL argument");
    *d_result = (uint64_t *)p->d_plan;
    return FZ_OK;
}

fz_status fz_enumerate(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, uint64_t row_base,
                       uint32_t *d_out, uint64_t out_capacity_rows, void *d_plan, uint64_t plan_bytes, void *stream,
                       uint64_t *rows_out, uint64_t *hash_out)
{
    fz_plan *p = nullptr;
    fz_status st = fz_plan_create(m, n, mode, shard, nshards, d_plan, plan_bytes, stream, &p);
    if (st) return st;
    st = fz_enumerate_launch(p, d_out, out_capacity_rows, row_base, stream);
    if (!st) st = fz_plan_result(p, stream, rows_out, hash_out);
    fz_plan_free(p);
    return st;
}

// ------------------------------------------------------------- end to end
static constexpr int kRunChunks = 8;

fz_status fz_run_workspace_bytes(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, uint64_t *bytes)
{
    if (!bytes) return fail(FZ_EINVAL, "bytes is NULL");
    uint64_t memo_b = 0;
    fz_status st = fz_memo_workspace_bytes(gens, d, t, n + 1, mode != FZ_COUNT, &memo_b);
    if (st) return st;
    HostTables H;
    if ((st = host_tables(gens, d, d - t, n + 1, H))) return st;
    const uint64_t rows = H.S[n];
    const int chunks = (mode == FZ_MATERIALIZE) ? kRunChunks : 1;
    const uint64_t units = (mode == FZ_COUNT) ? H.W[n] : rows;
    const uint64_t plan_b = align_up(plan_bytes_for(mode, (units + chunks - 1) / chunks), 256);
    uint64_t out_b = 0;
    if (mode == FZ_MATERIALIZE) out_b = align_up(rows * 4ull * d, 256);
    *bytes = align_up(memo_b, 256) + plan_b * chunks + out_b;
    return FZ_OK;
}

fz_status fz_run_host(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, void *d_ws, uint64_t ws_bytes,
                      uint32_t *h_out, uint64_t h_out_capacity_rows, void *stream, uint64_t *rows_out,
                      uint64_t *hash_out)
{
    uint64_t need = 0;
    fz_status st = fz_run_workspace_bytes(gens, d, t, n, mode, &need);
    if (st) return st;
    if (ws_bytes < need) return fail(FZ_ENOSPC, "workspace %llu B < %llu B", (unsigned long long)ws_bytes,
                                     (unsigned long long)need);
    uint64_t memo_b = 0;
    if ((st = fz_memo_workspace_bytes(gens, d, t, n + 1, mode != FZ_COUNT, &memo_b))) return st;
    char *w = (char *)d_ws;
    cudaStream_t s = (cudaStream_t)stream;
    fz_memo *m = nullptr;
    if ((st = fz_memo_build(gens, d, t, n + 1, mode != FZ_COUNT, w, memo_b, stream, &m))) return st;
    const uint64_t rows_total = m->H.S[n];
    if (mode == FZ_MATERIALIZE && (!h_out || h_out_capacity_rows < rows_total)) {
        fz_free(m);
        return fail(FZ_ENOSPC, "host output holds %llu rows, |Z(n)| = %llu", (unsigned long long)h_out_capacity_rows,
                    (unsigned long long)rows_total);
    }
    char *plan_area = w + align_up(memo_b, 256);
    const int chunks = (mode == FZ_MATERIALIZE) ? kRunChunks : 1;
    uint64_t plan_b = 0;
    if ((st = fz_plan_workspace_bytes(m, n, mode, chunks, &plan_b))) { fz_free(m); return st; }
    plan_b = align_up(plan_b, 256);
    uint32_t *d_out = (uint32_t *)(plan_area + plan_b * chunks);
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> ev(chunks, nullptr);
    if (mode == FZ_MATERIALIZE) {
        FZ_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (auto &e : ev) FZ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    uint64_t tot_rows = 0, tot_hash = 0;
    std::vector<fz_plan *> plans(chunks, nullptr);
    for (int c = 0; c < chunks && !st; ++c) {
        st = fz_plan_create(m, n, mode, c, chunks, plan_area + plan_b * c, plan_b, stream, &plans[c]);
        if (st) break;
        const uint64_t rb = plans[c]->shard_row_begin;
        st = fz_enumerate_launch(plans[c], d_out + rb * (uint64_t)d, rows_total - rb, rb, stream);
        if (st) break;
        if (mode == FZ_MATERIALIZE && plans[c]->shard_rows) {
            if (cudaEventRecord(ev[c], s) != cudaSuccess || cudaStreamWaitEvent(cs, ev[c], 0) != cudaSuccess ||
                cudaMemcpyAsync(h_out + rb * (uint64_t)d, d_out + rb * (uint64_t)d,
                                plans[c]->shard_rows * 4ull * d, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
                st = cuda_check("chunk D2H");
        }
    }
    for (int c = 0; c < chunks && !st; ++c) {
        uint64_t r = 0, h = 0;
        st = fz_plan_result(plans[c], stream, &r, &h);
        tot_rows += r;
        tot_hash += h;
    }
    if (cs) {
        cudaError_t e = cudaStreamSynchronize(cs);
        if (!st && e != cudaSuccess) st = fail(FZ_ECUDA, "D2H stream: %s", cudaGetErrorString(e));
        cudaStreamDestroy(cs);
    }
    for (auto &e : ev)
        if (e) cudaEventDestroy(e);
    for (auto *p : plans) fz_plan_free(p);
    fz_free(m);
    if (st) return st;
    if (rows_out) *rows_out = tot_rows;
    if (hash_out) *hash_out = tot_hash;
    return FZ_OK;
}

void fz_free(fz_memo *m) { delete m; }

}  // extern "C"
