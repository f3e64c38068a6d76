/*
 * fz_oracle.c -- CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
 * `--impl reference`) may load this library.  The product path
 * (paper_2407_20474_b200/) never links, imports or calls it, and this file
 * shares no code, header, table or constant generator with the CUDA path.
 *
 * What it computes is the plain definition of the paper's object,
 *     Z(n, (g_1..g_d)) = { a in N^d : sum_i a_i g_i = n }          PAPER.md:30-37 (§1)
 * as a list in strictly DESCENDING lexicographic order (reading E1,
 * PAPER.md:120-134 Lemma "respects lexicographic order" + Corollary;
 * SPEC.md:3), plus:
 *   - orc_enum_o1      : O1, the nested-loop definition.  Every
 *                        a_k runs floor(rem/g_k) down to 0, the last
 *                        coordinate is solved by divisibility.  Descending
 *                        loops give descending lex order with no sort.
 *   - orc_count_hash   : O1 (or O2: last two coordinates by the d=2 closed-form
 *                        list) with the E17 order-sensitive hash, optionally
 *                        OpenMP-parallel over a_1.  Global row indices of each
 *                        a_1 chunk come from the GF count of (g_2..g_d); the
 *                        per-chunk emitted count is checked against it.
 *   - orc_gf_count     : |Z(n)| as the coefficient of x^n in prod 1/(1-x^{g_i})
 *                        (coin-change DP, unsigned 128-bit), independent of
 *                        any enumeration.
 *   - orc_memo_alg2    : PAPER.md:139-153, Algorithm
 *                        LexicographicFactorizationListsUpToElement, literally
 *                        (list concatenation of incr_i over
 *                        isAllZeroesLeftOfIndex-filtered F[m-g_i]); used as the
 *                        memo oracle (memo = Alg 2 over the tail generators,
 *                        PAPER.md:233).
 *   - orc_hash_row     : E17 (reading R17): the build's own
 *                        order-sensitive row hash (not in the paper).
 *
 * Pins (tests/test_oracle_pins.py, -m "not gpu"): SPEC worked examples,
 * Table 1 num_results (erratum at :318), brute force O0 on
 * tiny inputs, GF count, d=2 closed form, hash KATs.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- E17 hash */
/* Reading R17: x=(k+1)*0x9E3779B97F4A7C15;
 * for j: x=(x^a_j)*0xBF58476D1CE4E5B9; x^=x>>29;  h = fmix64(x^d). */
static uint64_t orc_fmix64(uint64_t x)
{
    x ^= x >> 33;
    x *= 0xFF51AFD7ED558CCDULL;
    x ^= x >> 33;
    x *= 0xC4CEB9FE1A85EC53ULL;
    x ^= x >> 33;
    return x;
}

uint64_t orc_hash_row(uint64_t k, const uint32_t *a, int d)
{
    uint64_t x = (k + 1) * 0x9E3779B97F4A7C15ULL;
    for (int j = 0; j < d; ++j) {
        x = (x ^ (uint64_t)a[j]) * 0xBF58476D1CE4E5B9ULL;
        x ^= x >> 29;
    }
    return orc_fmix64(x ^ (uint64_t)d);
}

/* ------------------------------------------------------- generating function */
/* Coin-change DP: c[0]=1; for each g: for x=g..n: c[x] += c[x-g].
 * c[n] = coefficient of x^n in prod_i 1/(1-x^{g_i}) = |Z(n)|. */
int orc_gf_count(const uint32_t *g, int d, uint64_t n, uint64_t *lo, uint64_t *hi)
{
    if (d < 1 || n > (1ULL << 34)) return 1;
    u128 *c = (u128 *)calloc(n + 1, sizeof(u128));
    if (!c) return 2;
    c[0] = 1;
    for (int i = 0; i < d; ++i) {
        if (g[i] == 0) { free(c); return 1; }
        for (uint64_t x = g[i]; x <= n; ++x) c[x] += c[x - g[i]];
    }
    *lo = (uint64_t)c[n];
    *hi = (uint64_t)(c[n] >> 64);
    free(c);
    return 0;
}

/* Same DP, every coefficient c[0..N] (must fit 64 bits; returns 3 if not). */
int orc_gf_table(const uint32_t *g, int d, uint64_t N, uint64_t *out)
{
    u128 *c = (u128 *)calloc(N + 1, sizeof(u128));
    if (!c) return 2;
    c[0] = 1;
    for (int i = 0; i < d; ++i)
        for (uint64_t x = g[i]; x <= N; ++x) c[x] += c[x - g[i]];
    int rc = 0;
    for (uint64_t x = 0; x <= N; ++x) {
        if (c[x] >> 64) rc = 3;
        out[x] = (uint64_t)c[x];
    }
    free(c);
    return rc;
}

/* ---------------------------------------------------------------- O1 / O2 */
typedef struct {
    const uint32_t *g;
    int d;
    int use_o2;        /* solve the last two coordinates by the d=2 closed form */
    uint32_t *out;     /* optional row sink, row-major u32[d] */
    uint64_t cap;      /* rows the sink holds */
    uint64_t k;        /* next global row index */
    uint64_t hash;     /* sum of E17 row hashes mod 2^64 */
    int want_hash;
    uint32_t a[64];    /* current prefix */
} orc_ctx;

static void orc_emit(orc_ctx *c)
{
    if (c->out && c->k < c->cap) memcpy(c->out + c->k * (uint64_t)c->d, c->a, sizeof(uint32_t) * c->d);
    if (c->want_hash) c->hash += orc_hash_row(c->k, c->a, c->d);
    c->k += 1;
}

static uint64_t orc_gcd(uint64_t a, uint64_t b)
{
    while (b) { uint64_t t = a % b; a = b; b = t; }
    return a;
}

/* inverse of a modulo m (gcd(a,m)=1, m>=2), extended Euclid */
static uint64_t orc_inv(uint64_t a, uint64_t m)
{
    int64_t t = 0, nt = 1;
    int64_t r = (int64_t)m, nr = (int64_t)(a % m);
    while (nr) {
        int64_t q = r / nr, tmp;
        tmp = t - q * nt; t = nt; nt = tmp;
        tmp = r - q * nr; r = nr; nr = tmp;
    }
    if (t < 0) t += (int64_t)m;
    return (uint64_t)t;
}

/* d=2 closed-form list: all (x, y) with ga*x + gb*y = rem,
 * x descending.  c = gcd; A=ga/c, B=gb/c, R=rem/c; x0 = R*A^{-1} mod B;
 * x_max = x0 + floor((R - A x0)/(A B)) * B; x = x_max, x_max-B, ..., >= 0. */
static void orc_last_two(orc_ctx *c, int k, uint64_t rem)
{
    uint64_t ga = c->g[k], gb = c->g[k + 1];
    uint64_t cc = orc_gcd(ga, gb);
    if (rem % cc) return;
    uint64_t A = ga / cc, B = gb / cc, R = rem / cc;
    uint64_t x0 = (B == 1) ? 0 : ((R % B) * orc_inv(A % B, B)) % B;
    if (A * x0 > R) return;
    uint64_t xmax = x0 + ((R - A * x0) / (A * B)) * B;
    for (uint64_t x = xmax;; x -= B) {
        c->a[k] = (uint32_t)x;
        c->a[k + 1] = (uint32_t)((rem - ga * x) / gb);
        orc_emit(c);
        if (x < B) break;
    }
}

/* O1:
 *   rec(k, rem): if k == d-1: if rem % g[d-1] == 0: emit(prefix ++ [rem/g[d-1]])
 *                else for a = floor(rem/g[k]) down to 0: rec(k+1, rem - a*g[k]) */
static void orc_rec(orc_ctx *c, int k, uint64_t rem)
{
    if (k == c->d - 1) {
        if (rem % c->g[k] == 0) {
            c->a[k] = (uint32_t)(rem / c->g[k]);
            orc_emit(c);
        }
        return;
    }
    if (c->use_o2 && k == c->d - 2) {
        orc_last_two(c, k, rem);
        return;
    }
    for (uint64_t a = rem / c->g[k];; --a) {
        c->a[k] = (uint32_t)a;
        orc_rec(c, k + 1, rem - a * c->g[k]);
        if (a == 0) break;
    }
}

static int orc_check(const uint32_t *g, int d, uint64_t n)
{
    if (d < 1 || d > 64 || !g) return 1;
    for (int i = 0; i < d; ++i) if (g[i] == 0) return 1;
    if (n >= (1ULL << 32)) return 1;
    return 0;
}

/* Enumerate Z(n) single-threaded, descending lex.  Rows go to out[0..cap) when
 * out != NULL; count and E17 hash (row index k from 0) are always returned. */
int orc_enum_o1(const uint32_t *g, int d, uint64_t n, int use_o2, uint32_t *out, uint64_t cap,
                uint64_t *count, uint64_t *hash)
{
    if (orc_check(g, d, n)) return 1;
    orc_ctx c;
    memset(&c, 0, sizeof c);
    c.g = g; c.d = d; c.use_o2 = (use_o2 && d >= 2); c.out = out; c.cap = cap; c.want_hash = 1;
    orc_rec(&c, 0, n);
    *count = c.k;
    *hash = c.hash;
    return 0;
}

/* Count + hash of Z(n) with rows indexed from row_base, parallel over a_1.
 * a1_hi/a1_lo restrict a_1 to [a1_lo, a1_hi] (inclusive; pass a1_hi = UINT64_MAX
 * for the full range) -- used for the bounded cpu_baseline sample.
 * The global index of the first row with a_1 = v is
 *   start(v) = sum_{v' > v} |Z(n - v' g_1; g_2..g_d)|    (GF count table). */
int orc_count_hash(const uint32_t *g, int d, uint64_t n, int use_o2, int nthreads,
                   uint64_t a1_lo, uint64_t a1_hi, uint64_t *count, uint64_t *hash)
{
    if (orc_check(g, d, n)) return 1;
    if (d == 1) {
        uint32_t a = (uint32_t)(n / g[0]);
        int ok = (n % g[0] == 0) && a >= a1_lo && a <= a1_hi;
        *count = ok ? 1 : 0;
        *hash = ok ? orc_hash_row(0, &a, 1) : 0;
        return 0;
    }
    uint64_t top = n / g[0];
    uint64_t *c2 = (uint64_t *)malloc(sizeof(uint64_t) * (n + 1));
    if (!c2) return 2;
    if (orc_gf_table(g + 1, d - 1, n, c2)) { free(c2); return 3; }
    uint64_t *start = (uint64_t *)malloc(sizeof(uint64_t) * (top + 2));
    if (!start) { free(c2); return 2; }
    uint64_t run = 0;
    for (uint64_t v = top;; --v) {   /* descending a_1: rows of larger a_1 come first */
        start[v] = run;
        run += c2[n - v * g[0]];
        if (v == 0) break;
    }
    uint64_t lo = a1_lo, hi = (a1_hi > top) ? top : a1_hi;
    uint64_t tot_count = 0, tot_hash = 0;
    int bad = 0;
    if (lo <= hi) {
#ifdef _OPENMP
        if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : tot_count, tot_hash) reduction(| : bad)
#endif
        for (int64_t vv = (int64_t)hi; vv >= (int64_t)lo; --vv) {
            uint64_t v = (uint64_t)vv;
            orc_ctx c;
            memset(&c, 0, sizeof c);
            c.g = g; c.d = d; c.use_o2 = use_o2; c.want_hash = 1;
            c.k = start[v];
            c.a[0] = (uint32_t)v;
            orc_rec(&c, 1, n - v * g[0]);
            uint64_t emitted = c.k - start[v];
            if (emitted != c2[n - v * g[0]]) bad |= 1;
            tot_count += emitted;
            tot_hash += c.hash;
        }
    }
    free(start);
    free(c2);
    *count = tot_count;
    *hash = tot_hash;
    return bad ? 4 : 0;
}

int orc_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ Alg 2 */
/* PAPER.md:139-153, LexicographicFactorizationListsUpToElement(n, (g_1..g_d)):
 *   F[0] <- [0]
 *   for m in [0, n]:                (m = 0 is the base case, reading R3b)
 *     Z <- []
 *     for i = 1..d with m - g_i >= 0:
 *       Z <- Z ++ [ incr_i(a) : a in F[m - g_i] if isAllZeroesLeftOfIndex(a, i) ]
 *     F[m] <- Z
 * Here run for m in [0, top) (top exclusive, the memo's topOfMemo).
 * Output: CSR.  off[m] = first row of F[m], off[top] = total rows.  rows holds
 * up to cap rows of d u32; returns 0, or 5 if cap is too small (off still
 * filled up to the failure point is unspecified). */
static int orc_all_zero_left(const uint32_t *a, int i)
{
    for (int j = 0; j < i; ++j) if (a[j] != 0) return 0;   /* 0-based i: a_j = 0 for j < i */
    return 1;
}

int orc_memo_alg2(const uint32_t *g, int d, uint64_t top, uint32_t *rows, uint64_t cap, uint64_t *off)
{
    if (d < 1 || top < 1) return 1;
    for (int i = 0; i < d; ++i) if (g[i] == 0) return 1;
    uint64_t used = 0;
    /* F[0] <- [0] */
    if (cap < 1) return 5;
    memset(rows, 0, sizeof(uint32_t) * d);
    off[0] = 0;
    used = 1;
    for (uint64_t m = 1; m < top; ++m) {
        off[m] = used;
        for (int i = 0; i < d; ++i) {
            if (m < g[i]) continue;
            uint64_t src = m - g[i];
            for (uint64_t r = off[src]; r < off[src + 1]; ++r) {
                const uint32_t *a = rows + r * (uint64_t)d;
                if (!orc_all_zero_left(a, i)) continue;
                if (used >= cap) return 5;
                uint32_t *z = rows + used * (uint64_t)d;
                memcpy(z, a, sizeof(uint32_t) * d);
                z[i] += 1;                                       /* incr_i */
                used += 1;
            }
        }
    }
    off[top] = used;
    return 0;
}

/* Sum of E17 row hashes of rows[0..count) (row-major u32[d]) keyed from row_base. */
uint64_t orc_hash_rows(const uint32_t *rows, uint64_t count, int d, uint64_t row_base)
{
    uint64_t h = 0;
    for (uint64_t k = 0; k < count; ++k) h += orc_hash_row(row_base + k, rows + k * (uint64_t)d, d);
    return h;
}
