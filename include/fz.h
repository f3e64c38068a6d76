/*
 * fz.h -- C ABI of the B200 (sm_100a) factorization-set engine.
 *
 * The library enumerates the factorization set (§1)
 *     Z(n, (g_1..g_d)) = { a in N^d : sum_i a_i g_i = n }
 * in strictly DESCENDING lexicographic order (Lemma
 * "respects lexicographic order" and its Corollary; reading R1),
 * with the paper's low-dimension tabulation (§3.1): the
 * memo of tail factorization sets Z(x, (g_{L+1}..g_d)), L = d - t, for every
 * x < top, built on the GPU by the disjoint dimensionwise recurrence
 *     Z(x) = disjoint-union_i incr_i( Z_{>=i}(x - g_i) )
 * in elementwise batches of b <= min(tail g), and then a
 * bounded lexicographic walk over the L leading coordinates (nextCandidate,
 * PAPER.md:203-222; nextCandidateDynamic) that copies whole
 * memo blocks.
 *
 * Conventions for every entry point:
 *   - All functions are extern "C", never throw, and return fz_status.
 *     On any non-FZ_OK status a thread-local message is available from
 *     fz_last_error(); output arguments are then unspecified.
 *   - Generators are a HOST array uint32_t[d] of positive values in the given
 *     order (never sorted: the order defines the lex order, reading R2).
 *     Duplicates, gcd > 1 and g_i = 1 are legal.  1 <= d <= FZ_MAX_D.
 *   - All DEVICE memory is caller-owned (e.g. torch tensors): the memo
 *     workspace, the plan workspace and the output buffer.  The library never
 *     allocates device memory.  Device pointers must be 256-byte aligned.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Calls that return host scalars synchronise that stream; all
 *     others are asynchronous on it.
 *   - Coordinates are uint32; n, phi, counts, offsets and hashes are uint64.  Limits the kernels
 *     enforce (FZ_ERANGE beyond them): top <= 2^28 (so n < 2^28), memo blocks < 2^26 rows, COUNT
 *     tail blocks < 2^32 rows, every count < 2^64 (reading R15).
 */
#ifndef FZ_H
#define FZ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FZ_MAX_D 10   /* largest dimension d the kernels are instantiated for */

typedef enum {
    FZ_OK = 0,
    FZ_EINVAL = 1,  /* contract violation: d, t, gens, n >= top, null or misaligned pointer */
    FZ_ERANGE = 2,  /* top > 2^28 (n < 2^28), a count >= 2^64, a memo block >= 2^26 rows, or (COUNT)
                       a tail block >= 2^32 rows */
    FZ_ECAP = 3,    /* memo bytes exceed the memory cap (default 8e9 B; fz_set_memo_cap) */
    FZ_ENOSPC = 4,  /* caller workspace or output buffer too small */
    FZ_ECUDA = 5    /* CUDA runtime error (message in fz_last_error) */
} fz_status;

typedef enum {
    FZ_MATERIALIZE = 0, /* write every row of Z(n) (u32[d] row-major) to the caller buffer */
    FZ_COUNT = 1,       /* walk the leading prefixes and sum memo block sizes (no rows touched) */
    FZ_HASH = 2         /* walk + read every row; order-sensitive hash (reading R17) */
} fz_mode;

typedef struct fz_memo fz_memo; /* opaque host handle; references the caller's workspace */

typedef struct {
    int d;                  /* dimension */
    int t;                  /* memo dimension (tail generators tabulated), 0 <= t <= d */
    uint64_t top;           /* memo covers every x in [0, top) */
    uint64_t entries;       /* total memo rows = sum_{x<top} |Z(x; tail)| */
    uint64_t max_card;      /* max_x |Z(x; tail)| */
    uint64_t batches;       /* elementwise batches of the copy-increment pass */
    uint32_t batch;         /* batch size b = min(tail g) */
    int fill_mode;          /* 0 = no rows; 1 = one CTA, batches of min(tail g), shared-memory ring;
                               2 = same through L2; 3 = whole grid, batches of min(tail g);
                               4 = one pass per tail dimension, residue chains stepped in order;
                               5 = one pass per tail dimension, chains in unrolled (scan) form */
    uint64_t window_rows;   /* max rows a batch and its look-back window span (ring size needed) */
    uint64_t memo_top;      /* memo ROWS cover x < memo_top <= top (topOfMemo); the count
                               tables cover x < top.  memo_top < top is a partial memo */
} fz_memo_info;

#define FZ_MEMO_TOP_AUTO 0ull           /* fz_layout_create_partial: largest memo_top whose rows fit the cap */
#define FZ_MEMO_TOP_FULL UINT64_MAX     /* fz_layout_create_partial: memo_top = top (full memo) */

/* ---------------------------------------------------------------- A1 -- */
/* Validate (gens, d, t, top) and return the device workspace bytes
 * fz_memo_build needs.  with_entries = 0 sizes the count tables only (enough
 * for FZ_COUNT and fz_count).  t = 0 means no memo (plain bounded walk, the
 * prior-work nextCandidate); t = d builds the full DP table
 * (Alg 2/3's product F[m] for every m < top),
 * in which Z(n) is the block Memo[n].
 * Errors: FZ_EINVAL (d, t, gens, top = 0), FZ_ERANGE (a table entry >= 2^64,
 * top > 2^28, a memo block >= 2^26 rows), FZ_ECAP (memo rows * t * 4 B above the cap). */
fz_status fz_memo_workspace_bytes(const uint32_t *gens, int d, int t, uint64_t top, int with_entries,
                                  uint64_t *bytes);

/* Memory cap for memo rows (bytes); 0 restores the default 8e9. */
void fz_set_memo_cap(uint64_t bytes);

/* Force the copy-increment schedule of later layouts (1..5, see fz_memo_info.fill_mode;
 * a mode that does not fit falls back to the automatic choice); 0 = automatic. */
void fz_set_fill_mode(int mode);

/* A1 as a reusable host object (like an FFT plan): validation, sizing and the
 * host copy of the count tables for (gens, d, t, top, with_entries).  Building
 * a memo from a layout (fz_memo_build_layout) launches kernels only, with no
 * host-side loops.  Same errors as fz_memo_workspace_bytes.  Immutable; must
 * outlive every memo built from it. */
typedef struct fz_layout fz_layout;
fz_status fz_layout_create(const uint32_t *gens, int d, int t, uint64_t top, int with_entries, fz_layout **out);
fz_status fz_layout_workspace_bytes(const fz_layout *lay, uint64_t *bytes);

/* Partial memo (topOfMemo; "excepting dimension 3"):
 * count tables for every x < top (so any n < top can be planned and counted), memo ROWS only for
 * x < memo_top (1 <= memo_top <= top; FZ_MEMO_TOP_AUTO = the largest memo_top whose rows fit the memo
 * cap; FZ_MEMO_TOP_FULL = top).  Enumerating n >= memo_top (MATERIALIZE / HASH) walks into the tail
 * coordinates wherever the remainder has no memo block and copies the memo suffix blocks
 * Z_{>=k}(x), x < memo_top, below it (k5_deep; reading R19): the same rows in the same order
 * as the full memo.  COUNT needs the count tables only.  memo_top is forced to top when t = 0 or
 * with_entries = 0.  Errors as fz_layout_create, plus FZ_EINVAL for memo_top > top (other than FULL). */
fz_status fz_layout_create_partial(const uint32_t *gens, int d, int t, uint64_t top, uint64_t memo_top,
                                   int with_entries, fz_layout **out);
void fz_layout_free(fz_layout *lay);

/* Memo-dimension recommendation (PAPER.md:301 observes that the best memoDim
 * depends on the instance): predicted seconds per t in 0..d written to cost[0..d] (optional,
 * +inf-like 1e300 when infeasible: t = 0 or d, or a memo above the cap), best t in *t_best.
 * Host only (count tables of gens up to n); model constants in fz.cu. */
fz_status fz_recommend_t(const uint32_t *gens, int d, uint64_t n, fz_mode mode, int *t_best, double *cost);

/* ------------------------------------------------------------- A2-A4 -- */
/* Build the memo on the GPU (asynchronous on `stream`):
 *   K1 count pass: suffix tables S_i[x] = |Z(x; g_i..g_d)| = |Z_{>=i}(x)|
 *      (PAPER.md:83-85, 163-166), S_{d+1}[x] = [x = 0],
 *      S_i[x] = S_{i+1}[x] + S_i[x - g_i]  (strided scans over residues of g_i);
 *      card[x] = S_{L+1}[x] = |Z(x; tail)|; prefix tables W_i for the planner;
 *   K2 CSR offsets off[x] = sum_{y<x} card[y]  ("pre-assigned output location");
 *   K3 copy-increment (PAPER.md:171-192 semantics): for elementwise batches of
 *      b = min(tail g) consecutive x, every row of block i of
 *      Z(x) is incr_i of the matching row of Z_{>=i}(x - g_i), which is the
 *      suffix of Z(x - g_i) of length S_i[x - g_i]; block i of Z(x) starts at
 *      card[x] - S_i[x].  Memo[0] = [0].
 * d_ws (>= the fz_memo_workspace_bytes value, 256-B aligned) becomes owned by the
 * returned handle until fz_free.  top must exceed every n later enumerated
 * (full memo).  The handle is immutable and may be used from
 * several streams once the build's stream work has completed. */
fz_status fz_memo_build(const uint32_t *gens, int d, int t, uint64_t top, int with_entries, void *d_ws,
                        uint64_t ws_bytes, void *stream, fz_memo **out);

/* Same, from a layout (no host work beyond the launches). */
fz_status fz_memo_build_layout(const fz_layout *lay, void *d_ws, uint64_t ws_bytes, void *stream, fz_memo **out);

fz_status fz_memo_get_info(const fz_memo *m, fz_memo_info *info);
fz_status fz_layout_get_info(const fz_layout *lay, fz_memo_info *info);

/* Device pointers into the memo workspace (read-only views for tests):
 * rows = u32[entries * t] (CSR, x-major, each block descending lex),
 * off = u64[top + 1], S = u64[(d + 1) * top] (row i = S_{i+1} in 1-based paper indexing). */
fz_status fz_memo_device_views(const fz_memo *m, const uint32_t **rows, const uint64_t **off, const uint64_t **S);

/* |Z(n)| = S_1[n] read back from the device count tables (synchronises `stream`).
 * Requires n < top. */
fz_status fz_count(const fz_memo *m, uint64_t n, void *stream, uint64_t *count);

/* ---------------------------------------------------------------- A5 -- */
/* Shard plan of the lexicographic space of Z(n) over `nshards` ranks (host
 * copy of the same cut K4 makes on the device).  MATERIALIZE/HASH split the
 * output rows into nshards contiguous ranges, floor(|Z| s / nshards) ..;
 * COUNT splits the leading-prefix walk evenly.  Returns, per shard s, the
 * first global row and the row count (host arrays of nshards entries; NULL to
 * skip).  No device work. */
fz_status fz_shard_rows(const fz_memo *m, uint64_t n, fz_mode mode, int nshards, uint64_t *row_begin,
                        uint64_t *rows);

/* Same cut from a layout alone (host only, no device memory or GPU needed). */
fz_status fz_layout_shard_rows(const fz_layout *lay, uint64_t n, fz_mode mode, int nshards, uint64_t *row_begin,
                               uint64_t *rows);

/* Device plan-workspace bytes: the 256-B plan header (accumulators, shard geometry, slice queue); K5 unranks
 * its slices itself, so no slice table is stored. */
fz_status fz_plan_workspace_bytes(const fz_memo *m, uint64_t *bytes);

/* K4 planner (asynchronous, entirely on the device): read |Z(n)| (or the
 * leading-prefix count) from the device tables and cut shard `shard` of
 * `nshards` -- equal rows (MATERIALIZE, HASH) or equal modelled cost (COUNT:
 * the C tables' cost ranks of whole outer prefixes) -- and its geometry of K5
 * slices: equal rows, or, for MATERIALIZE / HASH walks with short rounds, equal
 * walk cost (one unit per row plus a weight per visited leading prefix;
 * DESIGN.md §6), or COUNT cost ranks in guided sizes.  K5 unranks each slice
 * start to its leading prefix (a_1..a_L) and offset in the memo block from the
 * S / W (/ C) tables:
 *   rank(a_1..a_L) = sum_j S_j[ r_{j-1} - (a_j + 1) g_j ],  r_j = n - sum_{i<=j} a_i g_i.
 * Writes the plan header and zeroes the result accumulators in d_plan
 * (>= fz_plan_workspace_bytes, 256-B aligned, caller-owned) and returns a host
 * handle (free with fz_plan_free; the memo must outlive it).
 * Errors: FZ_EINVAL (n >= top, shard range, COUNT-only memo used for rows),
 * FZ_ENOSPC (plan workspace too small). */
typedef struct fz_plan fz_plan;
fz_status fz_plan_create(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, void *d_plan,
                         uint64_t plan_bytes, void *stream, fz_plan **out);
void fz_plan_free(fz_plan *p);

/* Which K5 kernel an enumeration of this plan runs (diagnostics, roofline bookkeeping):
 *   FZ_WALK_ROWS         k5_walk over memo blocks (MATERIALIZE / HASH, full memo)
 *   FZ_WALK_DEEP         k5_deep (partial memo, n >= memo_top)
 *   FZ_WALK_TABLE        k5_table (t = d: Z(n) is the block Memo[n])
 *   FZ_WALK_COUNT_STAGED k5_runs (COUNT, L >= 3: staged card image, one innermost run per lane; default)
 *   FZ_WALK_COUNT_PAIRS  k5_pairs (the same walk with a pair of runs per lane; FZ_COUNT_WALK=pairs)
 *   FZ_WALK_COUNT_RUNS   k5_walk COUNT (L <= 2, or a card table that cannot be staged)
 * card_bytes: bytes per card lookup of the COUNT walk (1 = u8 image, 2 = u16 image, 4 = u32 table; 0 otherwise). */
enum { FZ_WALK_ROWS = 0, FZ_WALK_DEEP = 1, FZ_WALK_TABLE = 2, FZ_WALK_COUNT_PAIRS = 3, FZ_WALK_COUNT_RUNS = 4,
       FZ_WALK_COUNT_STAGED = 5 };
fz_status fz_plan_walk(const fz_plan *p, int *kind, int *card_bytes);

/* This plan's shard as computed on the device: first global row, row count,
 * number of slices (synchronises `stream`). */
fz_status fz_plan_shard(const fz_plan *p, void *stream, uint64_t *row_begin, uint64_t *rows, uint64_t *nslices);

/* ------------------------------------------------------------- A6-A9 -- */
/* K5 enumerator (asynchronous) over a plan: every warp walks its slices'
 * leading prefixes in descending lex order (the innermost leading coordinate
 * vectorised over the 32 lanes, outer coordinates carried as in nextCandidate),
 * looks up Memo[p], p = n - phi(prefix), and
 *   MATERIALIZE: writes prefix ++ Memo[p][k] for each row to
 *                d_out[(row - shard_row_begin) * d ...] (rows of this shard only;
 *                aligned to 16 B if 4 | d, 8 B if 2 | d, else 4 B).  If
 *                out_capacity_rows is below the shard's rows the kernel writes
 *                nothing and fz_plan_result returns FZ_ENOSPC;
 *   COUNT:       accumulates |Memo[p]| (no memo rows read);
 *   HASH:        accumulates h(row_base + row - shard_row_begin, row) (R17).
 * row_base is the global index the hash uses for this shard's first row;
 * UINT64_MAX (~0) takes the shard's row_begin from the device plan.
 * d_out may be NULL unless MATERIALIZE. */
fz_status fz_enumerate_launch(const fz_plan *p, uint32_t *d_out, uint64_t out_capacity_rows, uint64_t row_base,
                              void *stream);

/* Read the plan's accumulators after its enumeration (synchronises `stream`):
 * rows = rows this shard produced / counted, hash = sum of row hashes mod 2^64. */
fz_status fz_plan_result(const fz_plan *p, void *stream, uint64_t *rows, uint64_t *hash);

/* Device address of the plan's two u64 accumulators {rows, hash} (for
 * collectives without a host round trip). */
fz_status fz_plan_result_ptr(const fz_plan *p, uint64_t **d_result);

/* Convenience: fz_plan_create + fz_enumerate_launch + fz_plan_result + fz_plan_free (synchronises). */
fz_status fz_enumerate(const fz_memo *m, uint64_t n, fz_mode mode, int shard, int nshards, uint64_t row_base,
                       uint32_t *d_out, uint64_t out_capacity_rows, void *d_plan, uint64_t plan_bytes, void *stream,
                       uint64_t *rows_out, uint64_t *hash_out);

/* ------------------------------------------------------- end to end -- */
/* Whole path from HOST buffers (Alg 5 as one call): build the memo (top = n + 1, full
 * memo; partial, memo_top = FZ_MEMO_TOP_AUTO, when the full one exceeds the memo cap),
 * plan, enumerate, and for MATERIALIZE stream the rows into the HOST buffer h_out (u32[rows * d]; pinned
 * memory recommended) through a bounded DEVICE OUTPUT RING (PAPER.md:267, 281-285:
 * Outputs -> Buffer -> copyDeviceBufferToHostAndClear, flushed whenever a buffer is full): the output is
 * cut into chunks of at most one ring slot (the K4 shard cut with one shard per chunk); each chunk is
 * enumerated into its slot and copied to the host on a copy stream while later chunks are enumerated,
 * and a slot is reused once its copy has drained (CUDA events).  Output larger than the GPU's memory
 * streams through any ring size.
 *
 * d_ws (256-B aligned, caller-owned) is laid out as [memo | 4 plan headers + accumulator | output ring]:
 * everything beyond the memo and the headers is the ring, split into 4 slots.
 * fz_run_workspace_bytes returns the memo + headers + `ring_bytes` of ring (0 = default: what the output
 * needs, at most 64 MB; COUNT/HASH need no ring); the result does not grow with |Z(n)| beyond that.
 * The copy stream and ring events are created once per thread and device and reused; so is the host
 * layout of the last (gens, t, n, mode) of the thread.  Synchronises `stream`.
 * Errors: FZ_EINVAL (mode, gens, d, misaligned workspace), FZ_ENOSPC (workspace below memo + headers,
 * no room for one row per slot, h_out smaller than |Z(n)|), and the errors of the steps. */
fz_status fz_run_workspace_bytes(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, uint64_t ring_bytes,
                                 uint64_t *bytes);
fz_status fz_run_host(const uint32_t *gens, int d, int t, uint64_t n, fz_mode mode, void *d_ws, uint64_t ws_bytes,
                      uint32_t *h_out, uint64_t h_out_capacity_rows, void *stream, uint64_t *rows_out,
                      uint64_t *hash_out);

/* Frees the host handle only; the caller frees the workspace. NULL is ignored. */
void fz_free(fz_memo *m);

/* Thread-local message for the last non-FZ_OK status on this thread. */
const char *fz_last_error(void);

/* Number of kernel launches this thread issued through the library so far. */
uint64_t fz_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FZ_H */
