// fz.cu -- host side of the C ABI declared in include/fz.h.
//
// A1 validation and sizing run on the host (uint64 arithmetic with overflow
// checks); everything on the data path (A2-A9) is a kernel in fz_kernels.cuh
// launched on the caller's stream into caller-owned device memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "../../include/fz.h"
#include "fz_kernels.cuh"
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges per C-ABI phase (free without an attached tool)

using fzk::Gens;
using fzk::PlanArgs;
using fzk::PlanHdr;
using fzk::Slice;

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;
std::atomic<uint64_t> g_memo_cap{8000000000ull};   // SPEC.md:237 (process-wide setting, read at layout creation)
std::atomic<int> g_fill_override{0};               // 0 = automatic fill-mode choice (process-wide, ditto)
bool g_fuse_memo = true;               // fill mode 5 inside K1's cooperative launch (FZ_FUSE_MEMO=0 to split)

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

// Programmatic dependent launch (PDL): the kernel may be scheduled while the previous kernel of the
// stream drains; it calls griddepcontrol.wait before reading anything that kernel wrote.
// FZ_PDL=0 launches plainly (A/B comparisons).
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args)
{
    static const bool on = [] {
        const char *e = getenv("FZ_PDL");
        return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define FZ_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) return fail(FZ_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// SM count of the current device (cached per device id; 148 when no device is visible, e.g. host-only
// shard queries on a machine without a GPU)
int device_sms()
{
    static std::atomic<int> cache[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0) {
        cudaGetLastError();
        return 148;
    }
    if (dev < 64) {
        const int c = cache[dev].load(std::memory_order_relaxed);
        if (c > 0) return c;
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) {
        cudaGetLastError();
        sms = 148;
    }
    if (dev < 64) cache[dev].store(sms, std::memory_order_relaxed);
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
    uint64_t S, W, C, cardT, off, offT, chunk, links, rows, rows16, counter, list, total;
};

struct Sizing {
    int d, t, L;
    uint64_t top;
    uint64_t ltop = 0;   // memo rows cover x < ltop <= top (topOfMemo); tables cover x < top
    uint64_t card_max_all = 0;   // max_x<top |Z(x; tail)| (the COUNT walk reads card up to n)
    uint64_t entries = 0, max_card = 0, window = 0, ring_rows = 0, batches = 0;
    uint32_t batch = 0;
    uint32_t stage_words = 0;   // fill mode 1: words per TMA link chunk buffer
    uint32_t chb = 0;           // fill mode 1: batches per link chunk
    uint32_t Q = 1;             // fill mode 1: batches the bulk stores may lag behind
    uint64_t max_batch_rows = 0;
    uint64_t level_block[FZ_MAX_D] = {0};   // fill mode 4: largest block i of any Z(x), per tail level
    uint64_t list_cap = 0;                   // fill mode 5: rows per chain list (max_x S_{L+i}[x] over levels)
    uint64_t list_bytes = 0;
    uint8_t lg_a[FZ_MAX_D] = {0}, lg_b[FZ_MAX_D] = {0};   // fill mode 5: log2 lanes per x, per level and pass
    uint64_t smem_bytes = 0;    // fill mode 1: dynamic shared memory
    int fill_mode = 0;
    uint64_t beta = 32;         // COUNT pair walk: cost of a run beyond its lookups (C tables)
    uint64_t gamma = 0;         // COUNT pair walk: cost of an outer prefix beyond its runs (C tables)
    Layout lay{};
};

constexpr uint64_t kCountRunCost = 48;     // COUNT cost model (card lookups, u16 image; x2 for u8; measured, tools/count_tune.py,
constexpr uint64_t kCountOuterCost = 1536;  // profiles/r02_shard_balance.md): per innermost run and per outer prefix
constexpr uint64_t kWordStreamRowsPerPrefix = 8;    // MATERIALIZE word stream from this many rows per prefix
constexpr uint64_t kRows16MinBytes = 64ull << 20;   // u16 row copy: u32 rows above this (half the 126 MB L2)
constexpr uint64_t kRows16MaxBytes = 96ull << 20;   //   ... and the copy below this
constexpr uint64_t kSmemMax = 220 * 1024;   // dynamic shared memory budget of the ring fill
constexpr int kMaxGrid = 1024;              // chunk scratch entries of the K1 grid

fz_status validate(const uint32_t *g, int d, int t, uint64_t top)
{
    if (!g) return fail(FZ_EINVAL, "gens is NULL");
    if (d < 1 || d > FZ_MAX_D) return fail(FZ_EINVAL, "d=%d outside [1, %d]", d, FZ_MAX_D);
    if (t < 0 || t > d) return fail(FZ_EINVAL, "t=%d outside [0, d=%d]", t, d);
    for (int i = 0; i < d; ++i)
        if (g[i] == 0) return fail(FZ_EINVAL, "g_%d = 0 (generators must be positive)", i + 1);
    if (top == 0) return fail(FZ_EINVAL, "top must be >= 1");
    if (top > (1ull << 28)) return fail(FZ_ERANGE, "top=%llu above 2^28", (unsigned long long)top);
    return FZ_OK;
}

// memo_top: FZ_MEMO_TOP_FULL (= top), FZ_MEMO_TOP_AUTO (the largest that fits the cap), or 1..top.
fz_status size_memo(const uint32_t *g, int d, int t, uint64_t top, uint64_t memo_top, int with_entries,
                    const HostTables &H, Sizing &z)
{
    z.d = d;
    z.t = t;
    z.L = d - t;
    z.top = top;
    const int L = z.L;
    const uint64_t *card = H.S.data() + (size_t)L * top;
    const uint64_t g_cap = g_memo_cap.load();   // one snapshot of the process-wide cap per layout
    if (!with_entries || t == 0 || memo_top == FZ_MEMO_TOP_FULL) {
        memo_top = top;
    } else if (memo_top == FZ_MEMO_TOP_AUTO) {   // partial memo: longest prefix of x whose rows fit the cap
        const uint64_t cap_rows = g_cap / (4ull * t);
        uint64_t e = 0, x = 0;
        while (x < top && e + card[x] <= cap_rows) e += card[x++];
        if (x == 0) return fail(FZ_ECAP, "even Memo[0] exceeds the memo cap");
        memo_top = x;
    } else if (memo_top > top) {
        return fail(FZ_EINVAL, "memo_top=%llu > top=%llu", (unsigned long long)memo_top, (unsigned long long)top);
    }
    z.ltop = memo_top;
    for (uint64_t x = 0; x < top; ++x) z.card_max_all = std::max(z.card_max_all, card[x]);
    {   // cost model of the COUNT walk's cut (in card lookups): FZ_COUNT_RUN_COST per innermost run,
        // FZ_COUNT_OUTER_COST per outer prefix, beyond the lookups; a u8 card image (every card < 64) reads
        // twice the lookups per vector, so its runs and outer prefixes weigh twice as many lookups
        const bool u8 = z.card_max_all <= 63;
        const char *e = getenv("FZ_COUNT_RUN_COST");
        z.beta = (e && *e) ? (uint64_t)strtoull(e, nullptr, 10) : (u8 ? 2 : 1) * kCountRunCost;
        const char *e2 = getenv("FZ_COUNT_OUTER_COST");
        z.gamma = (e2 && *e2) ? (uint64_t)strtoull(e2, nullptr, 10) : (u8 ? 2 : 1) * kCountOuterCost;
    }
    const uint64_t ltop = memo_top;
    uint64_t entries = 0, mx = 0;
    for (uint64_t x = 0; x < ltop; ++x) {
        if (__builtin_add_overflow(entries, card[x], &entries)) return fail(FZ_ERANGE, "memo entries exceed 2^64");
        mx = std::max(mx, card[x]);
    }
    // memo blocks are copied and indexed with 32-bit row counts per warp round (< 2^26); a count-only layout
    // holds no blocks (its COUNT walk reads the u32 card table: fz_plan_create checks < 2^32)
    if (with_entries && t > 0 && mx >= (1ull << 26))
        return fail(FZ_ERANGE, "a memo block has %llu >= 2^26 rows", (unsigned long long)mx);
    z.entries = entries;
    z.max_card = mx;
    uint32_t b = 0xffffffffu, hmax = 0;
    for (int i = L; i < d; ++i) {
        b = std::min(b, g[i]);
        hmax = std::max(hmax, g[i]);
    }
    if (t == 0) b = 1;
    z.batch = b;
    z.batches = (ltop + b - 1) / b;
    // live window of the recurrence: rows of [x0 - hmax, x0 + b) for every batch start x0
    std::vector<uint64_t> off(ltop + 1, 0);
    for (uint64_t x = 0; x < ltop; ++x) off[x + 1] = off[x] + card[x];
    uint64_t win = 0;
    for (uint64_t x0 = 0; x0 < ltop; x0 += b) {
        uint64_t lo = x0 > hmax ? x0 - hmax : 0, hi = std::min<uint64_t>(x0 + b, ltop);
        win = std::max(win, off[hi] - off[lo]);
    }
    z.window = win;
    uint64_t rows_bytes = 0;
    if (with_entries && t > 0) {
        if (entries > (g_cap / (4ull * t)))
            return fail(FZ_ECAP, "memo of %llu rows x %d coords exceeds the cap of %llu bytes",
                        (unsigned long long)entries, t, (unsigned long long)g_cap);
        rows_bytes = entries * 4ull * t;
        // fill mode 1 (k3_fill_ring): ring over the rows of [x0 - max(hmax, 2b), x0 + b) for every batch
        // (look-back window + the batch whose bulk store may still be reading), links in chunks of chb batches
        // ring: rows of [x0 - max(hmax, (Q+1) b), x0 + b) for every batch (look-back window + batches whose
        // bulk store may still be pending); links in chunks of chb batches.  Largest Q, chb that fit.
        auto boffv = [&](uint64_t k) { return off[std::min<uint64_t>(k * b, ltop)]; };
        auto ring_for = [&](uint64_t Q) {
            uint64_t win2 = 0;
            const uint64_t back = std::max<uint64_t>((uint64_t)hmax, (Q + 1) * b);
            for (uint64_t x0 = 0; x0 < ltop; x0 += b) {
                uint64_t lo = x0 > back ? x0 - back : 0, hi = std::min<uint64_t>(x0 + b, ltop);
                win2 = std::max<uint64_t>(win2, off[hi] - off[lo]);
            }
            uint64_t ring = 4;
            while (ring < win2 + 4) ring <<= 1;   // + the rows sharing the first 16-B granule of a bulk store
            return ring;
        };
        auto chunk_for = [&](uint64_t chb) {
            uint64_t cw = 0;
            for (uint64_t k0 = 0; k0 < z.batches; k0 += chb) {
                uint64_t k1 = std::min<uint64_t>(k0 + chb, z.batches);
                cw = std::max<uint64_t>(cw, ((boffv(k1) + 3) & ~3ull) - (boffv(k0) & ~3ull));
            }
            return cw;
        };
        uint64_t smem = ~0ull, chb = 2, cw = 0, ring = 0, Q = 1;
        bool fit = false;
        for (uint64_t q : {8ull, 4ull, 2ull, 1ull}) {
            ring = ring_for(q);
            for (uint64_t cb : {32ull, 16ull, 8ull, 4ull, 2ull}) {
                cw = chunk_for(cb);
                smem = 4 * ((z.batches + 1 + 3) & ~3ull) + ring * 4ull * t + 2 * 4ull * cw + 32;
                if (smem <= kSmemMax) { chb = cb; Q = q; fit = true; break; }
            }
            if (fit) break;
        }
        z.ring_rows = ring;
        z.Q = (uint32_t)Q;
        for (uint64_t k = 0; k < z.batches; ++k) z.max_batch_rows = std::max<uint64_t>(z.max_batch_rows, boffv(k + 1) - boffv(k));
        z.chb = (uint32_t)std::max<uint64_t>(chb, 1);
        z.stage_words = (uint32_t)std::min<uint64_t>(cw, 0xffffffffu);
        z.smem_bytes = smem;
        bool chains_fit = true;
        for (int i = 0; i + 1 < t; ++i) {
            const uint64_t *Si = H.S.data() + (size_t)(L + i) * top, *Si1 = Si + top;
            uint64_t mb = 0;
            for (uint64_t x = 0; x < ltop; ++x) mb = std::max<uint64_t>(mb, Si[x] - Si1[x]);
            z.level_block[i] = mb;
            if (3ull * 512 * 4 * t + mb * 4ull * t + 6 * 1024 + 16 > kSmemMax) chains_fit = false;
        }
        // mode 5: one lazy list per residue chain and level, list_cap rows each
        uint64_t chains_max = 0;
        for (int i = 0; i + 1 < t; ++i) {
            const uint64_t *Si = H.S.data() + (size_t)(L + i) * top;
            uint64_t mx = 0;
            for (uint64_t x = 0; x < ltop; ++x) mx = std::max<uint64_t>(mx, Si[x]);
            z.list_cap = std::max<uint64_t>(z.list_cap, mx);
            chains_max = std::max<uint64_t>(chains_max, std::min<uint64_t>(g[L + i], ltop));
        }
        z.list_bytes = chains_max * z.list_cap * 4ull * t;
        // lanes per x of the two passes of level i: a whole warp per x (coalesced row copies), except
        // a single lane per x for chain-list passes averaging at most one row per x (measured with
        // tools/k1_trace.py: smaller groups lose coalescing on the block passes)
        auto pick_lg = [&](double rows_per_x, bool chain_pass) -> uint8_t {
            return (chain_pass && rows_per_x <= 1.0) ? 0 : 5;
        };
        for (int i = 0; i + 1 < t; ++i) {
            const uint64_t *Si = H.S.data() + (size_t)(L + i) * top, *Si1 = Si + top;
            double sa = 0, sb = 0;
            for (uint64_t x = 0; x < ltop; ++x) {
                sa += double(Si1[x]);
                sb += double(Si[x] - Si1[x]);
            }
            z.lg_a[i] = pick_lg(sa / double(std::max<uint64_t>(ltop, 1)), true);
            z.lg_b[i] = pick_lg(sb / double(std::max<uint64_t>(ltop, 1)), false);
            const char *fl = getenv("FZ_SCAN_LG");   // tuning override: log2 lanes per x in both passes
            if (fl && *fl && atoi(fl) >= 0 && atoi(fl) <= 5) z.lg_a[i] = z.lg_b[i] = (uint8_t)atoi(fl);
        }
        const int forced = g_fill_override;
        // modes 1-4 fill the whole table range; a partial memo (ltop < top) takes mode 5
        if (forced >= 1 && forced <= 5 && !(forced == 1 && !fit) && !(forced == 4 && !chains_fit) &&
            (ltop == top || forced == 5))
            z.fill_mode = forced;
        else if (t >= 5 && chains_fit && ltop == top)
            z.fill_mode = 4;   // deep tails: chains stepped in order beat the scan form (measured, tools/fill_modes.py)
        else
            z.fill_mode = 5;
    } else {
        z.fill_mode = 0;
    }
    const uint64_t m = L > 0 ? g[L - 1] : 1;
    Layout &l = z.lay;
    uint64_t p = 256;                                   // header
    l.S = p;       p = align_up(p + 8ull * (d + 1) * top, 256);
    l.W = p;       p = align_up(p + 8ull * (L + 1) * top, 256);
    l.C = p;       if (L >= 3) p = align_up(p + 8ull * (L - 2) * top, 256);   // COUNT cost tables C_0..C_{L-3}
    l.off = p;     p = align_up(p + 8ull * (top + 1), 256);
    l.cardT = p;   p = align_up(p + 4ull * (top + m), 256);
    l.offT = p;    p = align_up(p + 8ull * (top + m), 256);
    l.chunk = p;   p = align_up(p + 8ull * kMaxGrid, 256);
    l.counter = p; p = align_up(p + 256, 256);
    l.links = p;
    if (z.fill_mode == 1) p = align_up(p + 4ull * entries + 64, 256);
    if (z.fill_mode == 2) p = align_up(p + 8ull * entries, 256);
    l.rows = p;    p = align_up(p + rows_bytes + 64, 256);
    // u16 copy of the rows for the walks (k3_pack16) when the u32 rows overflow L2 but the u16 copy does not
    // and every coordinate is below 2^16 (C3 t = 3: 162 MB -> 81 MB)
    l.rows16 = 0;
    const char *r16e = getenv("FZ_ROWS16");   // 0: never build the u16 copy (A/B switch)
    if (!(r16e && r16e[0] == '0') && z.fill_mode && rows_bytes > kRows16MinBytes &&
        entries * 2ull * t <= kRows16MaxBytes) {
        uint32_t gmin = 0xffffffffu;
        for (int i = L; i < d; ++i) gmin = std::min(gmin, g[i]);
        if ((ltop - 1) / gmin < 65536) {
            l.rows16 = p;
            p = align_up(p + entries * 2ull * t + 64, 256);
        }
    }
    l.list = p;    if (z.fill_mode == 5) p = align_up(p + z.list_bytes, 256);
    l.total = p;
    return FZ_OK;
}

}  // namespace

// A1 result: validated generators + sizing + host tables (kept for host-side
// shard queries and the end-to-end host API).  Immutable; reusable for many builds.
struct fz_layout {
    Sizing z;
    uint32_t g[FZ_MAX_D];
    int with_entries;
    HostTables H;
};

struct fz_memo {
    const fz_layout *lay;
    fz_layout *owned;      // layout created by fz_memo_build (freed with the memo)
    char *ws;
    uint64_t *S, *W, *C, *off, *offT, *chunk;
    uint32_t *cardT, *rows;
    uint16_t *rows16;      // u16 copy of the rows, or nullptr
    void *links;
    unsigned int *counter;
};

namespace {
// COUNT pair walk (k5_pairs, L >= 3): geometry of the staged card image, or on = false when the walk
// cannot stage it (cards too large, image above the shared-memory budget) or FZ_COUNT_SMEM=0.
struct PairPlan {
    bool on = false, u8 = false;
    fzk::PairGeo pg{};
    uint32_t f0n = 0;
    size_t smem = 0;
};
}  // namespace

struct fz_plan {
    const fz_memo *m;
    uint64_t n;
    fz_mode mode;
    int shard, nshards;
    char *d_plan;
    PairPlan pp;
    uint64_t rbeta = 0;   // K4 cut the slices in walk cost units (k5_walk's cost-slice instantiation)
};

// ------------------------------------------------------------ launch helpers
namespace {

// NVTX range over one C-ABI call (memo build, count, plan, enumerate, run_host): the phases of a step on the
// profiler's host timeline (SURVEY §5 tracing)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

Gens make_gens(const uint32_t *g, int d)
{
    Gens G;
    for (int i = 0; i < FZ_MAX_D; ++i) G.g[i] = i < d ? g[i] : 1u;
    return G;
}

// closed form of Z(x; g, h) for the last two generators g = g_{d-2}, h = g_{d-1} (d >= 2):
// e = gcd(g, h), g1 = g/e, h1 = h/e, inv = g1^{-1} mod h1 (extended Euclid; 0 when h1 = 1)
fzk::ProgGens make_prog(const uint32_t *g, int d)
{
    fzk::ProgGens P{1, 1, 1, 1, 1, 0, 0, 0, 0, 0};
    if (d < 2) return P;
    const uint32_t a = g[d - 2], h = g[d - 1];
    uint32_t x = a, y = h;
    while (y) {
        const uint32_t t = x % y;
        x = y;
        y = t;
    }
    P.g = a;
    P.h = h;
    P.e = x;
    P.g1 = a / x;
    P.h1 = h / x;
    int64_t r0 = P.h1, r1 = P.g1 % P.h1, s0 = 0, s1 = 1;
    while (r1) {
        const int64_t q = r0 / r1, r2 = r0 - q * r1, s2 = s0 - q * s1;
        r0 = r1;
        r1 = r2;
        s0 = s1;
        s1 = s2;
    }
    P.inv = P.h1 == 1 ? 0u : (uint32_t)(((s0 % (int64_t)P.h1) + P.h1) % P.h1);
    auto magic = [](uint32_t v) -> uint64_t { return v == 1 ? 0ull : ~0ull / v + 1; };   // ceil(2^64 / v)
    P.mg = magic(P.g);
    P.mh = magic(P.h);
    P.me = magic(P.e);
    P.mh1 = magic(P.h1);
    return P;
}


constexpr uint64_t kPairSmemMax = 220 * 1024;   // dynamic shared memory of one k5_pairs CTA (one per SM)

// the COUNT kernel of the staged walk: k5_runs (default) or k5_pairs (FZ_COUNT_WALK=pairs)
bool count_walk_pairs()
{
    const char *wk = getenv("FZ_COUNT_WALK");
    return wk && wk[0] == 'p';
}

PairPlan pair_plan(const fz_layout *lay, uint64_t n)
{
    PairPlan P;
    const Sizing &z = lay->z;
    const int L = z.L;
    if (L < 3) return P;
    const char *env = getenv("FZ_COUNT_SMEM");
    if (env && env[0] == '0') return P;
    const uint64_t cmax = z.card_max_all;
    const uint32_t m = lay->g[L - 1], g2 = lay->g[L - 2];
    if (m >= 65536) return P;
    // packed accumulators: a byte (u8) / half (u16) takes 4 cards of the two masked last vectors
    const bool u8 = cmax <= 63;
    if (!u8 && cmax > 16383) return P;
    const uint64_t q = n / m + 1;                    // longest column prefix of a run
    if (2 * q * cmax >= (1ull << 32)) return P;      // per-pair u32 sum
    const uint64_t VE = u8 ? 16 : 8, eb = u8 ? 1 : 2;
    // > q entries per column (a run's pointer never leaves its column: k5_pairs' merged loop), rounded to
    // whole vectors, an odd number of them (the 16-B vectors of 8 consecutive columns: 8 bank groups)
    uint64_t R16 = (q + 1 + VE - 1) / VE * VE;
    if ((R16 / VE) % 2 == 0) R16 += VE;
    const uint32_t dlt = g2 % m;
    uint32_t e = m, y = dlt;                         // e = gcd(Delta, m) (gcd(0, m) = m)
    while (y) {
        const uint32_t r = e % y;
        e = y;
        y = r;
    }
    const uint32_t mp = m / e;
    const uint64_t f0 = n / lay->g[0] + 1;
    const uint32_t f0n = (f0 <= 4096) ? (uint32_t)f0 : 0u;
    const uint64_t f0b = (uint64_t)(f0n + 1) / 2 * 16;
    // k5_runs stages the transposed image (stored columns padded to a multiple of 8), k5_pairs the column-major one
    const bool tr = !count_walk_pairs();
    auto ncols = [&](uint64_t dd) { const uint64_t c = (uint64_t)e * (mp + dd); return tr ? (c + 7) / 8 * 8 : c; };
    auto bytes = [&](uint64_t dd) { return f0b + ncols(dd) * R16 * eb; };
    uint32_t dup = 31;
    if (bytes(31) > kPairSmemMax) dup = 0;
    if (bytes(dup) > kPairSmemMax) return P;
    // inverse of Delta / e modulo m' (extended Euclid; 0 when m' = 1)
    uint32_t inv = 0;
    if (mp > 1) {
        int64_t r0 = mp, r1 = (dlt / e) % mp, s0 = 0, s1 = 1;
        while (r1) {
            const int64_t qq = r0 / r1, r2 = r0 - qq * r1, s2 = s0 - qq * s1;
            r0 = r1;
            r1 = r2;
            s0 = s1;
            s1 = s2;
        }
        inv = (uint32_t)(((s0 % (int64_t)mp) + mp) % mp);
    }
    fzk::PairGeo &g = P.pg;
    g.m = m;
    g.dlt = dlt;
    g.e = e;
    g.mp = mp;
    g.dup = dup;
    g.inv = inv;
    g.R16 = (uint32_t)R16;
    g.ncolv = e * (mp + dup);
    g.ncolv8 = (uint32_t)ncols(dup);
    g.vstride = g.ncolv8 * 16;
    // flush period (iterations of 4 cards per packed lane: a Y and an X word pair)
    // flush period of the packed accumulators (iterations; each adds 4 cards per packed lane: two Y words, two
    // X words), a multiple of 4 (the unrolled step) when at least 4
    g.F = cmax == 0 ? (1u << 30) : (uint32_t)((u8 ? 255ull : 65535ull) / (4 * cmax));
    if (g.F >= 4) g.F &= ~3u;
    auto m32 = [](uint64_t v) -> uint32_t { return v == 1 ? 0xffffffffu : (uint32_t)((1ull << 32) / v); };
    g.Mm = m32(m);
    g.Mg2 = m32(g2);
    g.Me = m32(e);
    g.Mmp = m32(mp);
    for (int j = 0; j < FZ_MAX_D; ++j) g.Mg[j] = m32(j < z.d ? lay->g[j] : 1);
    // the common outer step R += g3 (k5_pairs advance): g3 = Q3 g2 + S3; column steps mod m for the two
    // outcomes of rmin + S3 >= g2, and their orbit-position steps when e = 1
    const uint32_t g3 = lay->g[L - 3];
    g.Q3 = g3 / g2;
    g.S3 = g3 % g2;
    g.cs1 = g.S3 % m;
    g.cs2 = (uint32_t)(((uint64_t)g.S3 % m + m - g2 % m) % m);
    g.is1 = e == 1 ? (uint32_t)((uint64_t)g.cs1 * inv % m) : 0;
    g.is2 = e == 1 ? (uint32_t)((uint64_t)g.cs2 * inv % m) : 0;
    g.QD = (uint32_t)(32ull * g2 / m);
    g.RD = (uint32_t)(32ull * g2 % m);
    g.Fr = cmax == 0 ? (1u << 30) : (uint32_t)((u8 ? 255ull : 65535ull) / (2 * cmax));   // 2 cards per packed lane
    g.beta = z.beta;
    g.gamma = z.gamma;
    if (g.Fr >= 4) g.Fr &= ~3u;
    g.bstep = 32u % mp;
    g.bwrap = mp - g.bstep;
    g.one_thr = ((((uint64_t)g.Fr + 1) * VE) - 1) * m;
    P.on = true;
    P.u8 = u8;
    P.f0n = f0n;
    P.smem = (size_t)bytes(dup);
    return P;
}

// host copy of the device cost tables C_0..C_{L-3} (same integer arithmetic as K1)
std::vector<uint64_t> host_cost_tables(const fz_layout *lay)
{
    const int L = lay->z.L;
    const uint64_t top = lay->z.top, beta = lay->z.beta, gamma = lay->z.gamma;
    std::vector<uint64_t> C((size_t)(L - 2) * top, 0);
    const uint64_t *W2 = lay->H.W.data() + (size_t)(L - 2) * top;
    const uint64_t g2 = lay->g[L - 2];
    for (int jc = L - 3; jc >= 0; --jc) {
        const uint64_t gj = lay->g[jc];
        uint64_t *Cj = C.data() + (size_t)jc * top;
        const uint64_t *Cn = (jc + 1 <= L - 3) ? C.data() + (size_t)(jc + 1) * top : nullptr;
        for (uint64_t x = 0; x < top; ++x) {
            const uint64_t src = Cn ? Cn[x] : W2[x] + beta * (x / g2 + 1) + gamma;
            Cj[x] = src + (x >= gj ? Cj[x - gj] : 0);
        }
    }
    return C;
}

constexpr uint64_t kPlanHeader = 256;
// cost slices of the MATERIALIZE / HASH walk (measured on Table 1 rows, C2, C3: profiles/r02_cost_slices.md)
constexpr uint64_t kRowBeta = 16;            // walk cost of a visited leading prefix, in rows (FZ_ROW_BETA)
constexpr uint64_t kLongSliceRows = 65536;   // row slices longer than this: 4x the slices (profiles/r02_hash.md)
constexpr uint64_t kCostSlicesPerWarp = 4;   // slices per resident warp with cost slices
constexpr double kCostRho = 64.0;            // cost slices when n / (L g_L) < kCostRho (short rounds)

// K5 queue granularity: slices per resident warp (measured optimum: 16 for MATERIALIZE / HASH, whose
// slices are row ranges; 64 for COUNT, whose outer prefixes vary more in work)
uint64_t max_slices(fz_mode mode)
{
    static const char *e = getenv("FZ_SLICES_PER_WARP");
    const uint64_t per_warp = (e && atoi(e) > 0) ? (uint64_t)atoi(e) : (mode == FZ_COUNT ? 64 : 16);
    return (uint64_t)device_sms() * 4 * (fzk::kWalkThreads / 32) * per_warp;
}

uint64_t plan_bytes() { return kPlanHeader; }   // the header; slices are unranked inside K5


template <int T>
fz_status launch_fill_t(const fz_memo *m, cudaStream_t s)
{
    const Sizing &z = m->lay->z;
    if (z.fill_mode == 1) {
        const size_t smem = (size_t)z.smem_bytes;
        FZ_CUDA(cudaFuncSetAttribute(fzk::k3_fill_ring<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        // workers: enough that the largest batch needs <= 4 rows per thread (prefetched in registers)
        const unsigned workers =
            (unsigned)std::min<uint64_t>(992, std::max<uint64_t>(64, align_up((z.max_batch_rows + 3) / 4, 32)));
        fzk::k3_fill_ring<T><<<1, workers + 32, smem, s>>>(m->off, (const uint32_t *)m->links, m->rows, z.top, z.batch,
                                                   (uint32_t)z.batches, (uint32_t)z.ring_rows, z.stage_words, z.chb, z.Q);
        ++g_launches;
        return cuda_check("k3_fill_ring");
    }
    if (z.fill_mode == 5) {   // the last tail level was written by K2 stage B
        fz_status st = FZ_OK;
        const unsigned wblocks = (unsigned)std::min<uint64_t>((z.top * 32 + 255) / 256, (uint64_t)device_sms() * 16);
        uint32_t *list = (uint32_t *)(m->ws + z.lay.list);
        for (int i = T - 2; i >= 0 && !st; --i) {
            const uint32_t h = m->lay->g[z.L + i];
            fzk::k3_scan_a<T><<<wblocks, 256, 0, s>>>(m->S, m->off, m->rows, list, z.list_cap, z.top, z.ltop, z.L, i, h,
                                                      z.lg_a[i]);
            fzk::k3_scan_b<T><<<wblocks, 256, 0, s>>>(m->S, m->off, m->rows, list, z.list_cap, z.top, z.ltop, z.L, i, h,
                                                      z.lg_b[i]);
            g_launches += 2;
            st = cuda_check("k3_scan");
        }
        return st;
    }
    if (z.fill_mode == 4) {   // the last tail level was written by K2 stage B
        fz_status st = FZ_OK;
        for (int i = T - 2; i >= 0 && !st; --i) {
            const uint32_t h = m->lay->g[z.L + i];
            const uint64_t cap = std::max<uint64_t>(z.level_block[i], 1);
            const unsigned chains = (unsigned)std::min<uint64_t>(h, z.top);
            // warps per chain: enough to fill the GPU, at most 16
            static const char *pe = getenv("FZ_CHAIN_P");
            const unsigned pmax = (pe && atoi(pe) > 1) ? (unsigned)atoi(pe) : 8;
            const unsigned P = (unsigned)std::max<uint64_t>(2, std::min<uint64_t>(pmax, (uint64_t)device_sms() * 8 / chains));
            const size_t smem = (((cap * T + 3) & ~3ull) + (size_t)fzk::kStageSlots * fzk::kChainStage * T) * 4 +
                                (size_t)fzk::kMetaSlots * 4 * 32 * 8 + 2 * 32 * 8 + 2 * 32 * 4;
            FZ_CUDA(cudaFuncSetAttribute(fzk::k3_chain<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            fzk::k3_chain<T><<<chains, 32 * P, smem, s>>>(m->S, m->off, m->rows, z.top, z.L, i, h, (uint32_t)cap);
            ++g_launches;
            st = cuda_check("k3_chain");
        }
        return st;
    }
    if (z.fill_mode == 2) {
        fzk::k3_fill_l2<T><<<1, 1024, 0, s>>>(m->off, (const uint64_t *)m->links, m->rows, z.top, z.batch);
        ++g_launches;
        return cuda_check("k3_fill_l2");
    }
    if (z.fill_mode == 3) {
        int per_sm = 0;
        FZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fzk::k3_fill_grid<T>, 256, 0));
        if (per_sm < 1) return fail(FZ_ECUDA, "k3_fill_grid cannot be resident");
        int blocks = device_sms() * std::min(per_sm, 4);
        FZ_CUDA(cudaMemsetAsync(m->counter, 0, 256, s));
        Gens G = make_gens(m->lay->g, z.d);
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
const void *memo_kernel(int t)
{
    if constexpr (T <= FZ_MAX_D) {
        if (t == T) return (const void *)fzk::k1_memo<T>;
        return memo_kernel<T + 1>(t);
    } else {
        return nullptr;
    }
}

template <int T = 1>
fz_status launch_fill(const fz_memo *m, cudaStream_t s)
{
    if (m->lay->z.fill_mode == 0) return FZ_OK;
    if constexpr (T <= FZ_MAX_D) {
        if (m->lay->z.t == T) return launch_fill_t<T>(m, s);
        return launch_fill<T + 1>(m, s);
    } else {
        return fail(FZ_EINVAL, "t=%d not instantiated", m->lay->z.t);
    }
}

constexpr uint64_t kCountSmemMax = 100 * 1024;   // COUNT u16 card table in shared memory (2 CTAs / SM)

struct WalkArgs {
    uint64_t card_max = ~0ull;   // max card over every x < top (COUNT smem staging needs < 2^16)
    uint64_t prefixes = 0;       // leading prefixes of the whole walk (W_0[n])
    Gens G;
    uint64_t n;
    PlanHdr *hdr;
    const uint64_t *Tb;
    uint64_t top;
    fzk::WalkTables wt;
    uint32_t *out;
    uint64_t cap;
    uint64_t row_base;
    bool cs = false;             // the plan's K5 slices are walk cost units (PlanHdr::rbeta != 0)
};

template <int D, int T, int MODE>
fz_status launch_walk_dtm(const WalkArgs &a, cudaStream_t s)
{
    // level-0 unrank column in shared memory when it is short (<= 4096 entries, 32 KB)
    const uint64_t f0 = a.n / a.G.g[0] + 1;
    const uint32_t f0n = (f0 <= 4096) ? (uint32_t)f0 : 0u;
    // COUNT with L = 2: the residue-major card table as u16 in shared memory (x <= n, R16 entries per
    // column: a multiple of 8 with R16 / 8 odd, so the 16-B vector loads of 8 lanes in different columns hit
    // distinct banks) when its values and size allow and the walk has enough prefixes per CTA to repay
    // the staging.  FZ_COUNT_SMEM=0 never stages the table, =2 stages it whatever the walk size (tests).
    const char *c16e = getenv("FZ_COUNT_SMEM");
    const bool c16_env = !(c16e && c16e[0] == '0'), c16_force = c16e && c16e[0] == '2';
    uint64_t R16 = (a.n / a.wt.m + 1 + 7) / 8 * 8;
    if ((R16 / 8) % 2 == 0) R16 += 8;
    const uint64_t cbytes = R16 * a.wt.m * 2;
    const uint32_t c16R = (MODE == FZ_COUNT && D - T == 2 && c16_env && a.card_max < 65536 &&
                           a.card_max * (a.n / a.wt.m + 1) < (1ull << 32) &&   // per-lane u32 run sums
                           cbytes + f0n * 8 + 8 <= kCountSmemMax &&
                           (c16_force || a.prefixes >= (a.n + 1) * 64 * (uint64_t)device_sms()))
                              ? (uint32_t)R16
                              : 0u;
    const size_t smem = (size_t)(f0n + 1) / 2 * 16 + (c16R ? cbytes : 0);
    // persistent grid: exactly the resident CTAs (the walk is a grid-stride loop over slices)
    int per_sm = 0;
    // grid sized for the largest dynamic part any n can ask (the 32 KB level-0 cache), so the residency does
    // not depend on n (measured: the residency the smaller dynamic part allows is slower on Table 1 rows); the
    // attribute must allow that size for the occupancy query (static shared memory -- the MATERIALIZE
    // word-stream staging -- plus the dynamic part may pass 48 KB)
    const size_t smem_q = std::max<size_t>(smem, 4096 * 8);
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_q);
        if (e != cudaSuccess) return e;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fzk::walk_threads<MODE>(), smem_q) !=
                cudaSuccess ||
            per_sm < 1) {
            cudaGetLastError();
            per_sm = 1;
        }
        per_sm = std::min(per_sm, 8);
        return launch_pdl(kern, dim3((unsigned)(device_sms() * per_sm)), dim3(fzk::walk_threads<MODE>()), smem, s,
                          a.G, (uint64_t)a.n, a.hdr, a.Tb, (uint64_t)a.top, a.wt, a.out, (uint64_t)a.cap,
                          (uint64_t)a.row_base, f0n, c16R);
    };
    // cost slices (a.cs) run their own instantiation, so the row-slice kernels carry none of their code
    if constexpr (MODE == FZ_HASH) {
        if (a.wt.memo16)   // the u16 copy of the rows
            FZ_CUDA(a.cs ? go(fzk::k5_walk<D, T, MODE, true, false, true>) : go(fzk::k5_walk<D, T, MODE, true>));
        else
            FZ_CUDA(a.cs ? go(fzk::k5_walk<D, T, MODE, false, false, true>) : go(fzk::k5_walk<D, T, MODE>));
    } else if constexpr (MODE == FZ_MATERIALIZE && (D % 4) != 0) {
        if (a.wt.word_stream)   // the word-stream variant
            FZ_CUDA(a.cs ? go(fzk::k5_walk<D, T, MODE, false, true, true>) : go(fzk::k5_walk<D, T, MODE, false, true>));
        else
            FZ_CUDA(a.cs ? go(fzk::k5_walk<D, T, MODE, false, false, true>) : go(fzk::k5_walk<D, T, MODE>));
    } else if constexpr (MODE == FZ_MATERIALIZE) {
        FZ_CUDA(a.cs ? go(fzk::k5_walk<D, T, MODE, false, false, true>) : go(fzk::k5_walk<D, T, MODE>));
    } else {
        FZ_CUDA(go(fzk::k5_walk<D, T, MODE>));
    }
    ++g_launches;
    return cuda_check("k5_walk");
}

// COUNT staged walk (L >= 3: k5_runs, or k5_pairs with FZ_COUNT_WALK=pairs): one 1024-thread CTA per SM (the K4
// guided slices assume exactly that grid)
template <int D, int T = 0>
fz_status launch_pairs_d(int t, const PairPlan &pp, const WalkArgs &a, const uint64_t *C, const uint64_t *W,
                         const uint32_t *cardT, uint64_t Rcol, cudaStream_t s)
{
    if constexpr (T + 3 <= D) {
        if (t != T) return launch_pairs_d<D, T + 1>(t, pp, a, C, W, cardT, Rcol, s);
        auto go = [&](auto kern, auto... extra) -> cudaError_t {
            cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pp.smem);
            if (e != cudaSuccess) return e;
            return launch_pdl(kern, dim3((unsigned)device_sms()), dim3(fzk::kCountThreads), pp.smem, s, a.G,
                              (uint64_t)a.n, a.hdr, C, (uint64_t)a.top, cardT, Rcol, pp.pg, pp.f0n, extra...);
        };
        const uint64_t *W2 = W + (uint64_t)(D - T - 2) * a.top;   // W_{L-2}: an outer prefix's lookups
        if (count_walk_pairs())
            FZ_CUDA(pp.u8 ? go(fzk::k5_pairs<D, T, true>) : go(fzk::k5_pairs<D, T, false>));
        else
            FZ_CUDA(pp.u8 ? go(fzk::k5_runs<D, T, true>, W2) : go(fzk::k5_runs<D, T, false>, W2));
        ++g_launches;
        return cuda_check("k5_pairs / k5_runs");
    } else {
        return fail(FZ_EINVAL, "pair walk: t=%d not instantiated for d=%d", t, D);
    }
}

template <int D = 3>
fz_status launch_pairs(int d, int t, const PairPlan &pp, const WalkArgs &a, const uint64_t *C, const uint64_t *W,
                       const uint32_t *cardT, uint64_t Rcol, cudaStream_t s)
{
    if constexpr (D <= FZ_MAX_D) {
        if (d == D) return launch_pairs_d<D>(t, pp, a, C, W, cardT, Rcol, s);
        return launch_pairs<D + 1>(d, t, pp, a, C, W, cardT, Rcol, s);
    } else {
        return fail(FZ_EINVAL, "d=%d not instantiated", d);
    }
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

template <int D = 1>
fz_status launch_table(int d, int mode, const WalkArgs &a, const uint64_t *off, cudaStream_t s)
{
    if constexpr (D <= FZ_MAX_D) {
        if (d != D) return launch_table<D + 1>(d, mode, a, off, s);
        const unsigned blocks = (unsigned)device_sms() * 4;
        if (mode == FZ_MATERIALIZE)
            fzk::k5_table<D, FZ_MATERIALIZE><<<blocks, 256, 0, s>>>(a.hdr, off, a.n, a.wt.memo, a.out, a.cap, a.row_base);
        else if (mode == FZ_COUNT)
            fzk::k5_table<D, FZ_COUNT><<<blocks, 256, 0, s>>>(a.hdr, off, a.n, a.wt.memo, a.out, a.cap, a.row_base);
        else
            fzk::k5_table<D, FZ_HASH><<<blocks, 256, 0, s>>>(a.hdr, off, a.n, a.wt.memo, a.out, a.cap, a.row_base);
        ++g_launches;
        return cuda_check("k5_table");
    } else {
        return fail(FZ_EINVAL, "d=%d not instantiated", d);
    }
}

template <int D, int T>
fz_status launch_deep_dt(int mode, const WalkArgs &a, const uint64_t *S, uint64_t ltop, const uint64_t *off,
                         cudaStream_t s)
{
    auto kern = (mode == FZ_MATERIALIZE) ? fzk::k5_deep<D, T, FZ_MATERIALIZE> : fzk::k5_deep<D, T, FZ_HASH>;
    int ps = 0;   // resident CTAs per SM (queried per launch: no per-thread cache that could outlive a device switch)
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kern, fzk::kWalkThreads, 4096 * 8) != cudaSuccess || ps < 1)
        ps = 2;
    ps = std::min(ps, 8);
    // closed form of the last two coordinates (PROG leaves): Z(x; g, h), g = g_{d-2}, h = g_{d-1}
    uint32_t gg[D];
    for (int j = 0; j < D; ++j) gg[j] = a.G.g[j];
    const fzk::ProgGens P = make_prog(gg, D);
    const uint64_t f0 = a.n / a.G.g[0] + 1;
    const uint32_t f0n = (f0 <= 4096) ? (uint32_t)f0 : 0u;
    kern<<<(unsigned)(device_sms() * ps), fzk::kWalkThreads, (size_t)f0n * 8, s>>>(
        a.G, a.n, a.hdr, S, a.top, ltop, off, a.wt.memo, a.out, a.cap, a.row_base, P, f0n);
    ++g_launches;
    return cuda_check("k5_deep");
}

template <int D, int T = 1>
fz_status launch_deep_d(int t, int mode, const WalkArgs &a, const uint64_t *S, uint64_t ltop, const uint64_t *off,
                        cudaStream_t s)
{
    if constexpr (T <= D) {
        if (t == T) return launch_deep_dt<D, T>(mode, a, S, ltop, off, s);
        return launch_deep_d<D, T + 1>(t, mode, a, S, ltop, off, s);
    } else {
        return fail(FZ_EINVAL, "t=%d not instantiated for d=%d", t, D);
    }
}

template <int D = 1>
fz_status launch_deep(int d, int t, int mode, const WalkArgs &a, const uint64_t *S, uint64_t ltop,
                      const uint64_t *off, cudaStream_t s)
{
    if constexpr (D <= FZ_MAX_D) {
        if (d == D) return launch_deep_d<D>(t, mode, a, S, ltop, off, s);
        return launch_deep<D + 1>(d, t, mode, a, S, ltop, off, s);
    } else {
        return fail(FZ_EINVAL, "d=%d not instantiated", d);
    }
}

// host-side rank / unrank over the layout's host tables (fz_shard_rows, fz_run_host)
// global row of the first row of prefix a_1..a_levels: sum_j S_j[r_j - (a_j + 1) g_j]
uint64_t host_row_rank(const fz_layout *lay, uint64_t n, const uint32_t *a, int levels)
{
    const uint64_t top = lay->z.top;
    uint64_t r = n, R = 0;
    for (int j = 0; j < levels; ++j) {
        const uint64_t nxt = (uint64_t)(a[j] + 1ull) * lay->g[j];
        if (nxt <= r) R += lay->H.S[(size_t)j * top + (r - nxt)];
        r -= (uint64_t)a[j] * lay->g[j];
    }
    return R;
}

// unrank R over `levels` levels of a unit table T (level j: T[j][r - a g_j] = units with a'_j >= a);
// returns the rank left inside the prefix reached (same search as the device unrank)
uint64_t host_unrank(const fz_layout *lay, const uint64_t *T, uint64_t n, int levels, uint64_t R, uint32_t *a)
{
    const uint64_t top = lay->z.top;
    uint64_t r = n;
    for (int j = 0; j < levels; ++j) {
        const uint64_t *Tj = T + (size_t)j * top;
        const uint64_t gj = lay->g[j], amax = r / gj;
        uint64_t lo = 0, hi = amax;   // largest a with Tj[r - a gj] > R
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo + 1) / 2;
            if (Tj[r - mid * gj] > R) lo = mid; else hi = mid - 1;
        }
        a[j] = (uint32_t)lo;
        R -= (lo + 1 <= amax) ? Tj[r - (lo + 1) * gj] : 0;
        r -= lo * gj;
    }
    return R;
}

// nextCandidate over the first nl coordinates (host twin of fzk::prefix_next)
bool host_prefix_next(const fz_layout *lay, uint32_t *a, int nl, uint64_t n)
{
    int i = -1;
    for (int j = 0; j < nl; ++j)
        if (a[j] > 0) i = j;
    if (i < 0) return false;
    uint64_t r = n;
    for (int j = 0; j < nl; ++j) {
        if (j == i) a[j] -= 1;
        if (j > i) a[j] = (uint32_t)(r / lay->g[j]);
        r -= (uint64_t)a[j] * lay->g[j];
    }
    return true;
}

uint64_t mul_div_h(uint64_t U, uint64_t a, uint64_t b) { return (U / b) * a + ((U % b) * a) / b; }

// same shard cut as k4_plan, on the host tables.  C: host_cost_tables when the COUNT pair walk runs.
void host_shard(const fz_layout *lay, uint64_t n, fz_mode mode, int nshards, int s, uint64_t &rb, uint64_t &rl,
                const std::vector<uint64_t> *C)
{
    const uint64_t rows_total = lay->H.S[n];
    const int L = lay->z.L;
    if (mode == FZ_COUNT && C) {   // pair walk: cost ranks, whole outer prefixes
        const uint64_t U = (*C)[n];
        auto rowat = [&](uint64_t u) -> uint64_t {
            if (u >= U) return rows_total;
            uint32_t a[FZ_MAX_D] = {0};
            if (host_unrank(lay, C->data(), n, L - 2, u, a) != 0 && !host_prefix_next(lay, a, L - 2, n))
                return rows_total;
            return host_row_rank(lay, n, a, L - 2);
        };
        rb = rowat(mul_div_h(U, s, nshards));
        rl = rowat(mul_div_h(U, s + 1, nshards)) - rb;
    } else if (mode == FZ_COUNT && L > 0) {   // leading prefixes
        const uint64_t P = lay->H.W[n];
        auto rowat = [&](uint64_t pidx) -> uint64_t {
            if (pidx >= P) return rows_total;
            uint32_t a[FZ_MAX_D] = {0};
            host_unrank(lay, lay->H.W.data(), n, L, pidx, a);
            return host_row_rank(lay, n, a, L);
        };
        rb = rowat(mul_div_h(P, s, nshards));
        rl = rowat(mul_div_h(P, s + 1, nshards)) - rb;
    } else {
        rb = mul_div_h(rows_total, s, nshards);
        rl = mul_div_h(rows_total, s + 1, nshards) - rb;
    }
}

// host shard cut of every shard (fz_shard_rows, fz_layout_shard_rows)
fz_status host_shards(const fz_layout *lay, uint64_t n, fz_mode mode, int nshards, uint64_t *row_begin,
                      uint64_t *rows)
{
    try {
        std::vector<uint64_t> C;
        const bool pairs = mode == FZ_COUNT && pair_plan(lay, n).on;
        if (pairs) C = host_cost_tables(lay);
        for (int s = 0; s < nshards; ++s) {
            uint64_t rb, rl;
            host_shard(lay, n, mode, nshards, s, rb, rl, pairs ? &C : nullptr);
            if (row_begin) row_begin[s] = rb;
            if (rows) rows[s] = rl;
        }
    } catch (const std::bad_alloc &) {
        return fail(FZ_ECAP, "host cost tables do not fit host memory");
    }
    return FZ_OK;
}

fz_status make_layout(const uint32_t *gens, int d, int t, uint64_t top, int with_entries, fz_layout **out,
                      uint64_t memo_top = FZ_MEMO_TOP_FULL)
{
    *out = nullptr;
    fz_status st = validate(gens, d, t, top);
    if (st) return st;
    fz_layout *lay = new (std::nothrow) fz_layout();
    if (!lay) return fail(FZ_ECAP, "host allocation failed");
    for (int i = 0; i < d; ++i) lay->g[i] = gens[i];
    lay->with_entries = with_entries ? 1 : 0;
    try {   // (host vectors: a failed allocation is FZ_ECAP, never an exception through the C ABI)
        if ((st = host_tables(gens, d, d - t, top, lay->H)) ||
            (st = size_memo(gens, d, t, top, memo_top, with_entries, lay->H, lay->z))) {
            delete lay;
            return st;
        }
    } catch (const std::bad_alloc &) {
        delete lay;
        return fail(FZ_ECAP, "host sizing tables for top=%llu do not fit host memory", (unsigned long long)top);
    }
    *out = lay;
    return FZ_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char *fz_last_error(void) { return g_err.c_str(); }
uint64_t fz_launch_count(void) { return g_launches; }
void fz_set_memo_cap(uint64_t bytes) { g_memo_cap = bytes ? bytes : 8000000000ull; }
void fz_set_fill_mode(int mode) { g_fill_override = (mode >= 1 && mode <= 5) ? mode : 0; }

fz_status fz_layout_create(const uint32_t *gens, int d, int t, uint64_t top, int with_entries, fz_layout **out)
{
    if (!out) return fail(FZ_EINVAL, "out is NULL");
    return make_layout(gens, d, t, top, with_entries, out);
}

fz_status fz_layout_create_partial(const uint32_t *gens, int d, int t, uint64_t top, uint64_t memo_top,
                                   int with_entries, fz_layout **out)
{
    if (!out) return fail(FZ_EINVAL, "out is NULL");
    if (memo_top == FZ_MEMO_TOP_FULL) memo_top = top;
    return make_layout(gens, d, t, top, with_entries, out, memo_top);
}

void fz_layout_free(fz_layout *lay) { delete lay; }

fz_status fz_layout_workspace_bytes(const fz_layout *lay, uint64_t *bytes)
{
    if (!lay || !bytes) return fail(FZ_EINVAL, "NULL argument");
    *bytes = lay->z.lay.total;
    return FZ_OK;
}

fz_status fz_layout_get_info(const fz_layout *lay, fz_memo_info *info)
{
    if (!lay || !info) return fail(FZ_EINVAL, "NULL argument");
    const Sizing &z = lay->z;
    info->d = z.d;
    info->t = z.t;
    info->top = z.top;
    info->entries = z.entries;
    info->max_card = z.max_card;
    info->batches = z.batches;
    info->batch = z.batch;
    info->fill_mode = z.fill_mode;
    info->window_rows = z.window;
    info->memo_top = z.ltop;
    return FZ_OK;
}

fz_status fz_memo_workspace_bytes(const uint32_t *gens, int d, int t, uint64_t top, int with_entries,
                                  uint64_t *bytes)
{
    if (!bytes) return fail(FZ_EINVAL, "bytes is NULL");
    fz_layout *lay = nullptr;
    fz_status st = make_layout(gens, d, t, top, with_entries, &lay);
    if (st) return st;
    *bytes = lay->z.lay.total;
    delete lay;
    return FZ_OK;
}

fz_status fz_memo_build_layout(const fz_layout *lay, void *d_ws, uint64_t ws_bytes, void *stream, fz_memo **out)
{
    NvtxRange nvtx("fz_memo_build");
    static const bool fuse_env = [] {
        const char *e = getenv("FZ_FUSE_MEMO");
        return !(e && e[0] == '0');
    }();
    g_fuse_memo = fuse_env;
    if (!out || !lay) return fail(FZ_EINVAL, "NULL argument");
    *out = nullptr;
    if (!d_ws || ((uintptr_t)d_ws & 255)) return fail(FZ_EINVAL, "workspace NULL or not 256-byte aligned");
    const Sizing &z = lay->z;
    if (ws_bytes < z.lay.total)
        return fail(FZ_ENOSPC, "workspace %llu B < required %llu B", (unsigned long long)ws_bytes,
                    (unsigned long long)z.lay.total);
    fz_memo *m = new (std::nothrow) fz_memo();
    if (!m) return fail(FZ_ECAP, "host allocation failed");
    m->lay = lay;
    char *w = (char *)d_ws;
    m->ws = w;
    m->S = (uint64_t *)(w + z.lay.S);
    m->W = (uint64_t *)(w + z.lay.W);
    m->C = z.L >= 3 ? (uint64_t *)(w + z.lay.C) : nullptr;
    m->off = (uint64_t *)(w + z.lay.off);
    m->cardT = (uint32_t *)(w + z.lay.cardT);
    m->offT = (uint64_t *)(w + z.lay.offT);
    m->chunk = (uint64_t *)(w + z.lay.chunk);
    m->counter = (unsigned int *)(w + z.lay.counter);
    m->links = (void *)(w + z.lay.links);
    m->rows = (uint32_t *)(w + z.lay.rows);
    m->rows16 = z.lay.rows16 ? (uint16_t *)(w + z.lay.rows16) : nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    Gens G = make_gens(lay->g, z.d);
    fzk::Tables tb;
    tb.S = m->S;
    tb.W = m->W;
    tb.C = m->C;
    tb.beta = z.beta;
    tb.gamma = z.gamma;
    tb.off = m->off;
    tb.cardT = m->cardT;
    tb.offT = m->offT;
    tb.chunk = m->chunk;
    tb.links = m->links;
    tb.top = z.top;
    tb.ltop = z.ltop;
    tb.m = z.L > 0 ? lay->g[z.L - 1] : 1;
    tb.R = (z.top + tb.m - 1) / tb.m;
    tb.d = z.d;
    tb.L = z.L;
    tb.t = z.t;
    tb.link_mode = (z.fill_mode == 1) ? 1 : (z.fill_mode == 2 ? 2 : 0);
    tb.ring_mask = z.ring_rows ? z.ring_rows - 1 : 0;
    tb.P = make_prog(lay->g, z.d);
    tb.rows = z.fill_mode ? m->rows : nullptr;
    {   // diagnostics: FZ_K1_TRACE = device address of a u64[grid * 32] buffer for phase timestamps
        const char *tr = getenv("FZ_K1_TRACE");
        tb.trace = (tr && *tr) ? (uint64_t *)(uintptr_t)strtoull(tr, nullptr, 0) : nullptr;
    }
    for (int i = 0; i < FZ_MAX_D; ++i) {
        tb.lg_a[i] = z.lg_a[i];
        tb.lg_b[i] = z.lg_b[i];
    }
    fz_status st = [&]() -> fz_status {
        FZ_CUDA(cudaMemsetAsync(m->counter, 0, 256, s));
        unsigned int *counter = m->counter;
        void *args[] = {&G, &tb, &counter};
        static const char *ge = getenv("FZ_K1_GRID");
        const int want = (ge && atoi(ge) > 0) ? atoi(ge) : device_sms();
        const int blocks = std::min(std::min(device_sms(), kMaxGrid), want);
        if (z.fill_mode == 5 && g_fuse_memo) {   // count pass + CSR + default fill in one launch
            uint32_t *list = (uint32_t *)(m->ws + z.lay.list);
            uint64_t cap_list = z.list_cap;
            void *args5[] = {&G, &tb, &counter, &list, &cap_list};
            const void *fn = memo_kernel(z.t);
            if (!fn) return fail(FZ_EINVAL, "t=%d not instantiated", z.t);
            FZ_CUDA(cudaLaunchCooperativeKernel(fn, blocks, 1024, args5, 0, s));
            ++g_launches;
            return cuda_check("k1_memo");
        }
        FZ_CUDA(cudaLaunchCooperativeKernel((const void *)fzk::k1_tables, blocks, 1024, args, 0, s));
        ++g_launches;
        return cuda_check("k1_tables");
    }();
    if (!st && !(z.fill_mode == 5 && g_fuse_memo)) st = launch_fill(m, s);
    if (!st && m->rows16) {   // the u16 copy of the rows for the walks
        const uint64_t words = z.entries * (uint64_t)z.t;
        fzk::k3_pack16<<<(unsigned)std::min<uint64_t>((words + 255) / 256, (uint64_t)device_sms() * 16), 256, 0, s>>>(
            m->rows, m->rows16, words);
        ++g_launches;
        st = cuda_check("k3_pack16");
    }
    if (st) {
        delete m;
        return st;
    }
    *out = m;
    return FZ_OK;
}

fz_status fz_memo_build(const uint32_t *gens, int d, int t, uint64_t top, int with_entries, void *d_ws,
                        uint64_t ws_bytes, void *stream, fz_memo **out)
{
    if (!out) return fail(FZ_EINVAL, "out is NULL");
    *out = nullptr;
    fz_layout *lay = nullptr;
    fz_status st = make_layout(gens, d, t, top, with_entries, &lay);
    if (st) return st;
    st = fz_memo_build_layout(lay, d_ws, ws_bytes, stream, out);
    if (st) {
        delete lay;
        return st;
    }
    (*out)->owned = lay;
    return FZ_OK;
}

fz_status fz_memo_get_info(const fz_memo *m, fz_memo_info *info)
{
    if (!m) return fail(FZ_EINVAL, "NULL memo");
    return fz_layout_get_info(m->lay, info);
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
    NvtxRange nvtx("fz_count");
    if (!m || !count) return fail(FZ_EINVAL, "NULL argument");
    if (n >= m->lay->z.top)
        return fail(FZ_EINVAL, "n=%llu >= top=%llu", (unsigned long long)n, (unsigned long long)m->lay->z.top);
    cudaStream_t s = (cudaStream_t)stream;
    FZ_CUDA(cudaMemcpyAsync(count, m->S + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    FZ_CUDA(cudaStreamSynchronize(s));
    return FZ_OK;
}

fz_status fz_shard_rows(const fz_memo *m, uint64_t n, fz_mode mode, int nshards, uint64_t *row_begin, uint64_t *rows)
{
    if (!m || nshards < 1) return fail(FZ_EINVAL, "NULL memo or nshards < 1");
    if (n >= m->lay->z.top) return fail(FZ_EINVAL, "n >= top");
    if (mode != FZ_MATERIALIZE && mode != FZ_COUNT && mode != FZ_HASH) return fail(FZ_EINVAL, "bad mode");
    return host_shards(m->lay, n, mode, nshards, row_begin, rows);
}

// SURVEY §8(f) f4 (the best memo dimension depends on the instance).  Predicted seconds
// of a whole step (memo build + plan + walk) for memo dimension t, from the host count tables:
//   R = |Z(n)|, P = leading prefixes (a_1..a_L, phi <= n), E = memo rows sum_{x<=n} |Z(x; tail)|, L = d - t;
//   MATERIALIZE: 9.04e-5 + 2.66e-13 (4 d R) + 1.045e-11 P + 9.964e-13 (4 t E)
//   HASH:        3.273e-12 R + 7.424e-12 P + 4.144e-13 (4 t E)
//   COUNT:       8.74e-5 + c_P P, c_P = 9.4e-14 with the staged pair walk (L >= 3, cards < 2^14, image fits
//                shared memory), else 9.2e-13 (the u32 card table from L2)
// The constants are a non-negative least-squares fit (relative error) of B200 step times over every t of
// Table 1's 31 rows, C2, C3 and C4 (tools/f4_fit.py on profiles/r02x_f4_study.jsonl -- the kernels with cost slices -- from
// `bench.py --study f4`).  Memos above the memory cap, and COUNT with a tail block >= 2^32, are infeasible.
fz_status fz_recommend_t(const uint32_t *gens, int d, uint64_t n, fz_mode mode, int *t_best, double *cost)
{
    if (!t_best) return fail(FZ_EINVAL, "t_best is NULL");
    fz_status st = validate(gens, d, d > 1 ? 1 : 0, n + 1);
    if (st) return st;
    const uint64_t top = n + 1;
    double best = 1e300;
    int bt = d > 1 ? 1 : 0;
    try {
        HostTables H;
        if ((st = host_tables(gens, d, 0, top, H))) return st;   // S levels (suffix counts) only
        // cumulative prefix counts over the first nl generators: sum_{y<=n} |Z(y; g_1..g_nl)|
        auto cum = [&](int nl) -> double {
            std::vector<double> c2(top, 0.0);
            c2[0] = 1;
            for (int i = 0; i < nl; ++i)
                for (uint64_t x = gens[i]; x < top; ++x) c2[x] += c2[x - gens[i]];
            double sum = 0;
            for (uint64_t x = 0; x < top; ++x) sum += c2[x];
            return sum;
        };
        const double R = (double)H.S[n];
        const uint64_t cap = g_memo_cap.load();
        for (int t = 0; t <= d; ++t) {
            double c = 1e300;
            const int L = d - t;
            if (t >= 1 && t <= d - 1) {
                const double P = cum(L);
                double E = 0;
                uint64_t cmax = 0;
                const uint64_t *card = H.S.data() + (size_t)L * top;
                for (uint64_t x = 0; x < top; ++x) {
                    E += (double)card[x];
                    cmax = std::max(cmax, card[x]);
                }
                const bool fits = E * 4.0 * t <= (double)cap;
                if (mode == FZ_MATERIALIZE && fits)
                    c = 9.04e-5 + 2.66e-13 * (4.0 * d * R) + 1.045e-11 * P + 9.964e-13 * (4.0 * t * E);
                if (mode == FZ_HASH && fits) c = 3.273e-12 * R + 7.424e-12 * P + 4.144e-13 * (4.0 * t * E);
                if (mode == FZ_COUNT && cmax < (1ull << 32)) {
                    const uint64_t m = gens[L - 1];
                    const double img = double(n + 1 + 32 * (n / m + 1)) * (cmax <= 63 ? 1.0 : 2.0);
                    const bool pairs = L >= 3 && cmax <= 16383 && img <= (double)kPairSmemMax;
                    c = 8.74e-5 + (pairs ? 9.4e-14 : 9.2e-13) * P;
                }
            }
            if (cost) cost[t] = c;
            if (c < best) {
                best = c;
                bt = t;
            }
        }
    } catch (const std::bad_alloc &) {
        return fail(FZ_ECAP, "host tables for n=%llu do not fit host memory", (unsigned long long)n);
    }
    *t_best = bt;
    return FZ_OK;
}

fz_status fz_layout_shard_rows(const fz_layout *lay, uint64_t n, fz_mode mode, int nshards, uint64_t *row_begin,
                               uint64_t *rows)
{
    if (!lay || nshards < 1) return fail(FZ_EINVAL, "NULL layout or nshards < 1");
    if (n >= lay->z.top) return fail(FZ_EINVAL, "n >= top");
    if (mode != FZ_MATERIALIZE && mode != FZ_COUNT && mode != FZ_HASH) return fail(FZ_EINVAL, "bad mode");
    return host_shards(lay, n, mode, nshards, row_begin, rows);
}

fz_status fz_plan_workspace_bytes(const fz_memo *m, uint64_t *bytes)
{
    if (!bytes) return fail(FZ_EINVAL, "bytes is NULL");
    (void)m;
    *bytes = plan_bytes();
    return FZ_OK;
}

fz_status fz_plan_create(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, void *d_plan,
                         uint64_t plan_ws_bytes, void *stream, fz_plan **out)
{
    NvtxRange nvtx("fz_plan_create");
    if (!out) return fail(FZ_EINVAL, "out is NULL");
    *out = nullptr;
    if (!m) return fail(FZ_EINVAL, "NULL memo");
    if (mode != FZ_MATERIALIZE && mode != FZ_COUNT && mode != FZ_HASH) return fail(FZ_EINVAL, "bad mode %d", (int)mode);
    if (nshards < 1 || shard < 0 || shard >= nshards) return fail(FZ_EINVAL, "shard %d of %d", shard, nshards);
    const Sizing &z = m->lay->z;
    if (n >= z.top)
        return fail(FZ_EINVAL, "n=%llu >= top=%llu (full memo required)", (unsigned long long)n,
                    (unsigned long long)z.top);
    if (mode != FZ_COUNT && z.t > 0 && z.fill_mode == 0)
        return fail(FZ_EINVAL, "memo built without entries; only FZ_COUNT is possible");
    if (mode == FZ_COUNT && z.card_max_all >= (1ull << 32))   // the walk reads the u32 card table (K2 cardT)
        return fail(FZ_ERANGE, "a tail block has %llu >= 2^32 rows (COUNT walk reads u32 cards)",
                    (unsigned long long)z.card_max_all);
    if (!d_plan || ((uintptr_t)d_plan & 255)) return fail(FZ_EINVAL, "plan workspace NULL or misaligned");
    if (plan_ws_bytes < plan_bytes())
        return fail(FZ_ENOSPC, "plan workspace %llu B < required %llu B", (unsigned long long)plan_ws_bytes,
                    (unsigned long long)plan_bytes());
    fz_plan *p = new (std::nothrow) fz_plan();
    if (!p) return fail(FZ_ECAP, "host allocation failed");
    p->m = m;
    p->n = n;
    p->mode = mode;
    p->shard = shard;
    p->nshards = nshards;
    p->d_plan = (char *)d_plan;
    PlanArgs A;
    A.n = n;
    A.top = z.top;
    A.max_slices = max_slices(mode);
    if (mode != FZ_COUNT && !getenv("FZ_SLICES_PER_WARP")) {
        // long row walks: when the default slices would hold more than kLongSliceRows rows each, 4x as many
        // (measured: C3 hash t = 3 33.4 -> 32.9 ms, t = 2 69.9 -> 67.2 ms; C2's 1e8 rows keep the default)
        const uint64_t rows = m->lay->H.S.empty() ? 0 : m->lay->H.S[n] / (uint64_t)nshards;
        if (rows / A.max_slices > kLongSliceRows) A.max_slices *= 4;
    }
    A.floor_len = (mode == FZ_COUNT) ? 1024 : 32;
    A.mode = (int)mode;
    A.shard = shard;
    A.nshards = nshards;
    A.L = z.L;
    p->pp = (mode == FZ_COUNT) ? pair_plan(m->lay, n) : PairPlan{};
    A.pairs = p->pp.on ? 1 : 0;
    // guided slices for the COUNT cost ranks (k5_pairs / k5_runs: one 1024-thread CTA per SM).  Row slices
    // (MATERIALIZE / HASH) stay uniform: with half-share first slices the per-row cost variance along the walk
    // leaves warps idle (measured: C3 t=2 hash 83 -> 134 ms); FZ_ROW_GSS=1 turns them on for experiments
    A.wg = (uint64_t)device_sms() * (fzk::kCountThreads / 32);
    {
        const char *e = getenv("FZ_ROW_GSS");
        if (mode != FZ_COUNT && !(e && e[0] == '1')) A.wg = 0;
    }
    {
        const char *e = getenv("FZ_GSS_TAIL");                    // last slices ~ 1/tail of a warp's share
        A.gss_tail = (e && atoi(e) > 0) ? (uint64_t)atoi(e) : 128;
    }
    {   // MATERIALIZE / HASH through k5_walk (full memo, L >= 1, uniform slices): when the walk's rounds are
        // short -- rho = n / (L g_L) innermost values per outer prefix on average, below kCostRho -- the time per
        // row varies along the walk with the round structure, and the slices are cut in walk cost units (one per
        // row plus kRowBeta per visited leading prefix), kCostSlicesPerWarp per warp; dense walks keep row
        // slices.  FZ_ROW_BETA (0: row slices) and FZ_SLICES_PER_WARP override.
        const bool walk = mode != FZ_COUNT && z.L > 0 && !(z.t > 0 && n >= z.ltop) && A.wg == 0;
        const double rho = z.L > 0 ? (double)n / ((double)z.L * m->lay->g[z.L - 1]) : 0.0;
        const char *e = getenv("FZ_ROW_BETA");
        const uint64_t beta = (e && *e) ? (uint64_t)atoll(e) : (rho < kCostRho ? kRowBeta : 0);
        A.rbeta = walk ? beta : 0;
        p->rbeta = A.rbeta;
        if (A.rbeta) {
            static const char *se = getenv("FZ_SLICES_PER_WARP");
            const uint64_t per_warp = (se && atoi(se) > 0) ? (uint64_t)atoi(se) : kCostSlicesPerWarp;
            A.max_slices = (uint64_t)device_sms() * 4 * (fzk::kWalkThreads / 32) * per_warp;
        }
    }
    Gens G = make_gens(m->lay->g, z.d);
    const cudaError_t le = launch_pdl(fzk::k4_plan, dim3(1), dim3(32), 0, (cudaStream_t)stream, G, A,
                                      (const uint64_t *)m->S, (const uint64_t *)m->W, (const uint64_t *)m->C,
                                      (PlanHdr *)p->d_plan);
    if (le != cudaSuccess) {
        delete p;
        return fail(FZ_ECUDA, "k4_plan launch: %s", cudaGetErrorString(le));
    }
    ++g_launches;
    fz_status st = cuda_check("k4_plan");
    if (st) {
        delete p;
        return st;
    }
    *out = p;
    return FZ_OK;
}

void fz_plan_free(fz_plan *p) { delete p; }

fz_status fz_plan_walk(const fz_plan *p, int *kind, int *card_bytes)
{
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    const Sizing &z = p->m->lay->z;
    int k = FZ_WALK_ROWS, cb = 0;
    if (p->mode == FZ_COUNT && z.L > 0) {
        if (p->pp.on) {
            k = count_walk_pairs() ? FZ_WALK_COUNT_PAIRS : FZ_WALK_COUNT_STAGED;
            cb = p->pp.u8 ? 1 : 2;
        } else {
            k = FZ_WALK_COUNT_RUNS;
            cb = 4;
        }
    } else if (p->mode != FZ_COUNT && z.t > 0 && p->n >= z.ltop) {
        k = FZ_WALK_DEEP;
    } else if (z.L == 0) {
        k = FZ_WALK_TABLE;
    }
    if (kind) *kind = k;
    if (card_bytes) *card_bytes = cb;
    return FZ_OK;
}

fz_status fz_plan_shard(const fz_plan *p, void *stream, uint64_t *row_begin, uint64_t *rows, uint64_t *nslices)
{
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    PlanHdr h;
    cudaStream_t s = (cudaStream_t)stream;
    FZ_CUDA(cudaMemcpyAsync(&h, p->d_plan, sizeof h, cudaMemcpyDeviceToHost, s));
    FZ_CUDA(cudaStreamSynchronize(s));
    if (row_begin) *row_begin = h.row_begin;
    if (rows) *rows = h.rows;
    if (nslices) *nslices = h.nslices;
    return FZ_OK;
}

fz_status fz_enumerate_launch(const fz_plan *p, uint32_t *d_out, uint64_t out_capacity_rows, uint64_t row_base,
                              void *stream)
{
    NvtxRange nvtx("fz_enumerate_launch");
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    const fz_memo *m = p->m;
    const Sizing &z = m->lay->z;
    if (p->mode == FZ_MATERIALIZE) {
        const uintptr_t align = (z.d % 4 == 0) ? 16 : (z.d % 2 == 0 ? 8 : 4);
        if (!d_out && out_capacity_rows) return fail(FZ_EINVAL, "d_out is NULL");
        if (((uintptr_t)d_out & (align - 1))) return fail(FZ_EINVAL, "d_out not %d-byte aligned", (int)align);
    }
    WalkArgs a;
    a.G = make_gens(m->lay->g, z.d);
    a.n = p->n;
    a.hdr = (PlanHdr *)p->d_plan;
    a.Tb = (p->mode == FZ_COUNT) ? m->W : m->S;
    a.top = z.top;
    a.wt.cardT = m->cardT;
    a.wt.offT = m->offT;
    a.wt.memo = m->rows;
    a.wt.memo16 = (p->mode == FZ_HASH) ? m->rows16 : nullptr;   // MATERIALIZE is bound by its stores
    const uint64_t gl = z.L > 0 ? m->lay->g[z.L - 1] : 1;
    a.wt.R = (z.top + gl - 1) / gl;
    a.wt.m = (uint32_t)gl;
    for (int j = 0; j < FZ_MAX_D; ++j) {
        const uint64_t g = j < z.d ? m->lay->g[j] : 1;
        a.wt.gmag[j] = (g == 1) ? 0 : (~0ull / g + 1);   // ceil(2^64 / g)
    }
    a.wt.card64 = m->S + (uint64_t)z.L * z.top;
    a.wt.Wt = m->W;
    a.cs = p->rbeta != 0;
    {   // d not a multiple of 4: rows leave as a 16-B word stream when the warp rounds are long (measured on
        // Table 1 rows: it pays from ~8 rows per leading prefix); FZ_WORD_STREAM=0/1 forces
        const char *e = getenv("FZ_WORD_STREAM");
        const uint64_t P = m->lay->H.W.empty() ? 0 : m->lay->H.W[p->n];
        const bool long_rounds = P && m->lay->H.S[p->n] >= kWordStreamRowsPerPrefix * P;
        a.wt.word_stream = (e && *e) ? (e[0] != '0') : long_rounds;
    }
    a.card_max = z.card_max_all;
    a.prefixes = m->lay->H.W.empty() ? 0 : m->lay->H.W[p->n];
    a.out = d_out;
    a.cap = (p->mode == FZ_MATERIALIZE) ? out_capacity_rows : ~0ull;
    a.row_base = row_base;
    if (p->mode != FZ_COUNT && z.t > 0 && p->n >= z.ltop)   // partial memo: Memo[p] missing for p >= ltop
        return launch_deep(z.d, z.t, (int)p->mode, a, m->S, z.ltop, m->off, (cudaStream_t)stream);
    if (z.L == 0) return launch_table(z.d, (int)p->mode, a, m->off, (cudaStream_t)stream);
    if (p->mode == FZ_COUNT && p->pp.on)
        return launch_pairs(z.d, z.t, p->pp, a, m->C, m->W, m->cardT, a.wt.R, (cudaStream_t)stream);
    return launch_walk(z.d, z.t, (int)p->mode, a, (cudaStream_t)stream);
}

fz_status fz_plan_result(const fz_plan *p, void *stream, uint64_t *rows, uint64_t *hash)
{
    if (!p) return fail(FZ_EINVAL, "NULL plan");
    PlanHdr h;
    cudaStream_t s = (cudaStream_t)stream;
    FZ_CUDA(cudaMemcpyAsync(&h, p->d_plan, sizeof h, cudaMemcpyDeviceToHost, s));
    FZ_CUDA(cudaStreamSynchronize(s));
    if (h.err)
        return fail(FZ_ENOSPC, "output buffer smaller than the shard's %llu rows (nothing written)",
                    (unsigned long long)h.rows);
    if (rows) *rows = h.result[0];
    if (hash) *hash = h.result[1];
    return FZ_OK;
}

fz_status fz_plan_result_ptr(const fz_plan *p, uint64_t **d_result)
{
    if (!p || !d_result) return fail(FZ_EINVAL, "NULL argument");
    *d_result = (uint64_t *)p->d_plan;
    return FZ_OK;
}

fz_status fz_enumerate(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, uint64_t row_base,
                       uint32_t *d_out, uint64_t out_capacity_rows, void *d_plan, uint64_t plan_ws_bytes, void *stream,
                       uint64_t *rows_out, uint64_t *hash_out)
{
    fz_plan *p = nullptr;
    fz_status st = fz_plan_create(m, n, mode, shard, nshards, d_plan, plan_ws_bytes, stream, &p);
    if (st) return st;
    st = fz_enumerate_launch(p, d_out, out_capacity_rows, row_base, stream);
    if (!st) st = fz_plan_result(p, stream, rows_out, hash_out);
    fz_plan_free(p);
    return st;
}

// ------------------------------------------------------------- end to end
// fz_run_host (Outputs -> Buffer -> copyDeviceBufferToHostAndClear,
// flushed whenever a buffer is full and once at the end).  The device holds the memo and a RING of
// kRingSlots output slots; MATERIALIZE output of any size is cut into chunks of at most one slot (the
// K4 shard cut with nshards = chunks), each chunk enumerated into its slot and copied to the host on a
// copy stream while the next chunks are enumerated; a slot is reused once its copy has drained (events).
// Device memory is bounded by the workspace the caller passes, not by |Z(n)|.
}  // extern "C"

namespace {
constexpr int kRingSlots = 4;
constexpr uint64_t kRunRingDefault = 64ull << 20;   // default output ring of fz_run_workspace_bytes (4 x 16 MB)

struct RunCtx {   // per-thread copy stream and ring events, created once per device (never destroyed:
                  // a thread-exit destructor could run after the CUDA runtime's own teardown)
    int dev = -1;
    cudaStream_t cs = nullptr;
    cudaEvent_t ready[kRingSlots] = {}, drained[kRingSlots] = {};
};
thread_local RunCtx g_run;

fz_status run_ctx(RunCtx *&out)
{
    int dev = 0;
    FZ_CUDA(cudaGetDevice(&dev));
    if (g_run.dev != dev) {
        RunCtx c;
        c.dev = dev;
        FZ_CUDA(cudaStreamCreateWithFlags(&c.cs, cudaStreamNonBlocking));
        for (int i = 0; i < kRingSlots; ++i) {
            FZ_CUDA(cudaEventCreateWithFlags(&c.ready[i], cudaEventDisableTiming));
            FZ_CUDA(cudaEventCreateWithFlags(&c.drained[i], cudaEventDisableTiming));
        }
        g_run = c;   // (a context of an earlier device is left alive: its device may be used again)
    }
    out = &g_run;
    return FZ_OK;
}

// the layout of the last fz_run_host call of this thread (A1 host tables reused across identical calls)
struct RunLayoutCache {
    uint32_t g[FZ_MAX_D] = {0};
    int d = -1, t = -1, with_entries = -1;
    uint64_t n = 0, cap = 0;
    int fill = 0;
    fz_layout *lay = nullptr;
};
thread_local RunLayoutCache g_run_lay;

fz_status run_layout(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, const fz_layout *&out)
{
    if (!gens || d < 1 || d > FZ_MAX_D) return fail(FZ_EINVAL, "gens NULL or d=%d outside [1, %d]", d, FZ_MAX_D);
    RunLayoutCache &c = g_run_lay;
    const int we = mode != FZ_COUNT;
    bool hit = c.lay && c.d == d && c.t == t && c.n == n && c.with_entries == we && c.cap == g_memo_cap.load() &&
               c.fill == g_fill_override.load();
    for (int i = 0; hit && i < d; ++i) hit = c.g[i] == gens[i];
    if (!hit) {
        fz_layout *lay = nullptr;
        fz_status st = make_layout(gens, d, t, n + 1, we, &lay, FZ_MEMO_TOP_AUTO);
        if (st) return st;
        delete c.lay;
        c.lay = lay;
        for (int i = 0; i < d; ++i) c.g[i] = gens[i];
        c.d = d;
        c.t = t;
        c.n = n;
        c.with_entries = we;
        c.cap = g_memo_cap.load();
        c.fill = g_fill_override.load();
    }
    out = c.lay;
    return FZ_OK;
}

constexpr uint64_t kRunFixed = kPlanHeader * kRingSlots + 256;   // plan headers + the run accumulator
}  // namespace

extern "C" {

fz_status fz_run_workspace_bytes(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, uint64_t ring_bytes,
                                 uint64_t *bytes)
{
    if (!bytes) return fail(FZ_EINVAL, "bytes is NULL");
    if (mode != FZ_MATERIALIZE && mode != FZ_COUNT && mode != FZ_HASH) return fail(FZ_EINVAL, "bad mode");
    const fz_layout *lay = nullptr;
    fz_status st = run_layout(gens, d, t, n, mode, lay);
    if (st) return st;
    uint64_t ring = 0;
    if (mode == FZ_MATERIALIZE) {   // the ring asked for, else what the output needs, at most kRunRingDefault
        const uint64_t out_b = lay->H.S[n] * 4ull * d;
        ring = ring_bytes ? ring_bytes
                          : std::min<uint64_t>(kRunRingDefault, align_up(out_b, 256) + kRingSlots * 256ull);
        ring = std::max<uint64_t>(ring, kRingSlots * align_up(32ull * 4 * d, 256));   // >= 32 rows per slot
    }
    *bytes = align_up(lay->z.lay.total, 256) + kRunFixed + ring;
    return FZ_OK;
}

fz_status fz_run_host(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, void *d_ws, uint64_t ws_bytes,
                      uint32_t *h_out, uint64_t h_out_capacity_rows, void *stream, uint64_t *rows_out,
                      uint64_t *hash_out)
{
    NvtxRange nvtx("fz_run_host");
    if (mode != FZ_MATERIALIZE && mode != FZ_COUNT && mode != FZ_HASH) return fail(FZ_EINVAL, "bad mode");
    if (!d_ws || ((uintptr_t)d_ws & 255)) return fail(FZ_EINVAL, "workspace NULL or not 256-byte aligned");
    const fz_layout *lay = nullptr;
    fz_status st = run_layout(gens, d, t, n, mode, lay);
    if (st) return st;
    const uint64_t rows_total = lay->H.S[n];
    const uint64_t memo_b = align_up(lay->z.lay.total, 256);
    if (ws_bytes < memo_b + kRunFixed)
        return fail(FZ_ENOSPC, "workspace %llu B < %llu B (memo + plan headers)", (unsigned long long)ws_bytes,
                    (unsigned long long)(memo_b + kRunFixed));
    // output ring: whatever the workspace holds beyond the memo and the headers, in kRingSlots slots
    const uint64_t slot_b = ((ws_bytes - memo_b - kRunFixed) / kRingSlots) & ~255ull;
    const uint64_t slot_rows = slot_b / (4ull * d);
    if (mode == FZ_MATERIALIZE) {
        if (rows_total && slot_rows == 0)
            return fail(FZ_ENOSPC, "workspace leaves no room for an output ring (%llu B per slot)",
                        (unsigned long long)slot_b);
        if (rows_total && (!h_out || h_out_capacity_rows < rows_total))
            return fail(FZ_ENOSPC, "host output holds %llu rows, |Z(n)| = %llu",
                        (unsigned long long)h_out_capacity_rows, (unsigned long long)rows_total);
    }
    RunCtx *rc = nullptr;
    if ((st = run_ctx(rc))) return st;
    char *w = (char *)d_ws;
    cudaStream_t s = (cudaStream_t)stream;
    char *plan_area = w + memo_b;
    uint64_t *acc = (uint64_t *)(plan_area + kPlanHeader * kRingSlots);
    char *ring = plan_area + kRunFixed;
    FZ_CUDA(cudaMemsetAsync(acc, 0, 3 * sizeof(uint64_t), s));
    fz_memo *m = nullptr;
    if ((st = fz_memo_build_layout(lay, w, memo_b, stream, &m))) return st;
    const uint64_t nch = (mode == FZ_MATERIALIZE && rows_total) ? (rows_total + slot_rows - 1) / slot_rows : 1;
    for (uint64_t c = 0; c < nch && !st; ++c) {
        const int slot = (int)(c % kRingSlots);
        if (mode == FZ_MATERIALIZE && c >= (uint64_t)kRingSlots &&
            cudaStreamWaitEvent(s, rc->drained[slot], 0) != cudaSuccess) {   // the slot's last copy drained
            st = cuda_check("ring slot wait");
            break;
        }
        fz_plan *p = nullptr;
        st = fz_plan_create(m, n, mode, (int)c, (int)nch, plan_area + kPlanHeader * slot, kPlanHeader, stream, &p);
        if (st) break;
        uint32_t *d_slot = (uint32_t *)(ring + (uint64_t)slot * slot_b);
        st = fz_enumerate_launch(p, mode == FZ_MATERIALIZE ? d_slot : nullptr,
                                 mode == FZ_MATERIALIZE ? slot_rows : 0, ~0ull, stream);
        fz_plan_free(p);
        if (st) break;
        fzk::k_run_acc<<<1, 32, 0, s>>>((const PlanHdr *)(plan_area + kPlanHeader * slot), acc);
        ++g_launches;
        if ((st = cuda_check("k_run_acc"))) break;
        if (mode == FZ_MATERIALIZE) {   // chunk c = rows [rb, rb + rl) of the K4 cut (the host twin of it)
            uint64_t rb = 0, rl = 0;
            host_shard(lay, n, mode, (int)nch, (int)c, rb, rl, nullptr);
            if (rl && (cudaEventRecord(rc->ready[slot], s) != cudaSuccess ||
                       cudaStreamWaitEvent(rc->cs, rc->ready[slot], 0) != cudaSuccess ||
                       cudaMemcpyAsync(h_out + rb * (uint64_t)d, d_slot, rl * 4ull * d, cudaMemcpyDeviceToHost,
                                       rc->cs) != cudaSuccess ||
                       cudaEventRecord(rc->drained[slot], rc->cs) != cudaSuccess))
                st = cuda_check("chunk D2H");
        }
    }
    uint64_t res[3] = {0, 0, 0};
    {   // drain both streams whatever happened (nothing may still reference the workspace), then read
        const cudaError_t e1 = cudaStreamSynchronize(rc->cs), e0 = cudaStreamSynchronize(s);
        if (!st && (e0 != cudaSuccess || e1 != cudaSuccess))
            st = fail(FZ_ECUDA, "run streams: %s", cudaGetErrorString(e0 != cudaSuccess ? e0 : e1));
        if (!st && cudaMemcpy(res, acc, sizeof res, cudaMemcpyDeviceToHost) != cudaSuccess)
            st = cuda_check("result read");
    }
    fz_free(m);
    if (st) return st;
    if (res[2]) return fail(FZ_ENOSPC, "an output chunk overflowed its ring slot");
    if (rows_out) *rows_out = res[0];
    if (hash_out) *hash_out = res[1];
    return FZ_OK;
}

void fz_free(fz_memo *m)
{
    if (!m) return;
    delete m->owned;
    delete m;
}

}  // extern "C"

#if FZ_SLICE_TRACE
// diagnostic builds only: copy the per-slice trace of the last k5_walk launches ({unrank cycles, walk cycles,
// end globaltimer / 64, SM id} per slice index) into host memory
extern "C" int fz_debug_slice_trace(void *host, uint64_t n)
{
    if (n > (1u << 20)) n = 1u << 20;
    return (int)cudaMemcpyFromSymbol(host, fzk::g_slice_trace, n * sizeof(uint4));
}
#endif
