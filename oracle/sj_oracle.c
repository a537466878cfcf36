/*
 * sj_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU epsilon self-join.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load this library.  It shares NO code, header, constant or helper with the CUDA path
 * (paper_1803_04120_b200/csrc); it is compiled separately with
 *     gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC -pthread
 * so that every -, * and + below is one IEEE-754 binary64 round-to-nearest operation.
 *
 * What it computes (§3 "Problem Statement"; readings R1-R5):
 *     S = { (i,k) in [0,N)^2 : s(p_i,p_k) <= E },  E = fl(eps*eps),
 *     s(a,b) = (((a_0-b_0)^2 + (a_1-b_1)^2) + ...) + (a_{d-1}-b_{d-1})^2, left to right, no FMA.
 * Pairs are ordered (key = query i, value = neighbour k), both
 * orientations, self pairs included unless include_self == 0 (reading R3),
 * 0-based ids, packed as (uint64)i << 32 | k and returned sorted ascending.
 *
 * Three entry points, all following that one definition:
 *   orc_brute_force  -- the O(N^2) nested-loop join ("brute force nested loop
 *                       join"), literally the definition above.
 *   orc_grid_join    -- a hash grid with its OWN robust cell width w_o (not the GPU's) and a
 *                       FULL 3^d neighbourhood scan (no unicomp, no masks, no binary search).
 *                       The grid is only a filter: completeness follows from w_o > max accepted
 *                       |x_j-y_j| + coordinate rounding (DESIGN.md "Oracle" section).
 *   orc_rows         -- for sampled query ids, the full neighbour row by brute force over all N
 *                       points (used for parity at full size, one query at a time).
 *   orc_grid_digest  -- the grid join of orc_grid_join, but instead of storing S it returns
 *                       |S|, per-query counts and order-independent fingerprints of the multiset S
 *                       and of the count vector (full-size parity of results too large to hold:
 *                       tens of GB of pairs).  Fingerprint definition:
 *                         F_a(S) = sum over pairs x of mix_a(x)  (mod 2^64)
 *                         F_b(S) = sum over pairs x of mix_b(x)  (mod 2^64)
 *                         F_c(cnt) = sum over queries i of mix_a((uint64)i << 32 | cnt_i)
 *                       mix_a = SplitMix64 output function of x + 0x9E3779B97F4A7C15,
 *                       mix_b = MurmurHash3 fmix64 of x ^ 0xC2B2AE3D27D4EB4F.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- the predicate (PAPER.md:130 squared form; R1, R2) ---------------------- */
static int orc_within(const double *a, const double *b, int d, double E)
{
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        double t = a[j] - b[j];
        double t2 = t * t;
        s = s + t2;
    }
    return s <= E;
}

/* exported so tests can probe the predicate on hand-picked knife-edge values */
int orc_pair_within(const double *a, const double *b, int d, double eps)
{
    double E = eps * eps;
    return orc_within(a, b, d, E);
}

/* ---- brute force ----------------------------------------------------------------------- */
/* Writes up to cap pairs into out (may be NULL); returns |S| (or -1 on bad arguments). */
int64_t orc_brute_force(const double *pts, int64_t n, int d, double eps, int include_self,
                        uint64_t *out, int64_t cap)
{
    if (n < 0 || d < 1 || !(eps > 0.0)) return -1;
    double E = eps * eps;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t k = 0; k < n; ++k) {
            if (i == k && !include_self) continue;
            if (orc_within(pts + i * d, pts + k * d, d, E)) {
                if (out && cnt < cap) out[cnt] = ((uint64_t)i << 32) | (uint64_t)k;
                ++cnt;
            }
        }
    }
    return cnt;
}

/* ---- per-query rows by brute force, threaded over queries -------------------------------- */
typedef struct {
    const double *pts; int64_t n; int d; double E; int include_self;
    const int64_t *qids; int64_t nq; int64_t t0, t1;
    int64_t *counts;          /* [nq] */
    uint64_t **rows;          /* [nq] malloc'd, sorted by k */
} rows_job;

static void *rows_worker(void *arg)
{
    rows_job *J = (rows_job *)arg;
    for (int64_t t = J->t0; t < J->t1; ++t) {
        int64_t i = J->qids[t];
        int64_t cap = 64, cnt = 0;
        uint64_t *r = (uint64_t *)malloc((size_t)cap * sizeof(uint64_t));
        for (int64_t k = 0; k < J->n; ++k) {
            if (i == k && !J->include_self) continue;
            if (orc_within(J->pts + i * J->d, J->pts + k * J->d, J->d, J->E)) {
                if (cnt == cap) { cap *= 2; r = (uint64_t *)realloc(r, (size_t)cap * sizeof(uint64_t)); }
                r[cnt++] = ((uint64_t)i << 32) | (uint64_t)k;
            }
        }
        J->counts[t] = cnt;
        J->rows[t] = r;
    }
    return NULL;
}

/* Two-call protocol: call with out == NULL to get counts[nq] (returns total); then call again
 * with out sized >= total to receive the concatenated rows (query order as given). */
int64_t orc_rows(const double *pts, int64_t n, int d, double eps, int include_self,
                 const int64_t *qids, int64_t nq, int nthreads, int64_t *counts, uint64_t *out)
{
    if (n < 0 || d < 1 || !(eps > 0.0) || nq < 0) return -1;
    if (nthreads < 1) nthreads = 1;
    uint64_t **rows = (uint64_t **)calloc((size_t)(nq > 0 ? nq : 1), sizeof(uint64_t *));
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    rows_job *jobs = (rows_job *)malloc(sizeof(rows_job) * (size_t)nthreads);
    for (int t = 0; t < nthreads; ++t) {
        rows_job j = {pts, n, d, eps * eps, include_self, qids, nq,
                      nq * t / nthreads, nq * (t + 1) / nthreads, counts, rows};
        jobs[t] = j;
        pthread_create(&th[t], NULL, rows_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    int64_t total = 0;
    for (int64_t t = 0; t < nq; ++t) {
        if (out) memcpy(out + total, rows[t], (size_t)counts[t] * sizeof(uint64_t));
        total += counts[t];
        free(rows[t]);
    }
    free(rows); free(th); free(jobs);
    return total;
}

/* ---- hash-grid join, full 3^d neighbourhood ------------------------------------------------ */
#define ORC_MAXD 8

typedef struct {
    int64_t c[ORC_MAXD];   /* integer cell tuple floor(x_j / w_o) */
    int64_t start;         /* first position in the cell-sorted order */
    int64_t count;
    int used;
} orc_cell;

typedef struct {
    const double *pts; int64_t n; int d; double w;
    int64_t *cellc;        /* [n*d] cell tuple per point */
    int64_t *order;        /* point ids sorted by (tuple, id) */
    orc_cell *table; uint64_t mask;
} orc_grid;

static orc_grid *G_sort_ctx; /* qsort has no context argument */

static int cmp_tuple(const int64_t *a, const int64_t *b, int d)
{
    for (int j = 0; j < d; ++j) {
        if (a[j] < b[j]) return -1;
        if (a[j] > b[j]) return 1;
    }
    return 0;
}

static int cmp_point(const void *pa, const void *pb)
{
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    const orc_grid *g = G_sort_ctx;
    int c = cmp_tuple(g->cellc + a * g->d, g->cellc + b * g->d, g->d);
    if (c) return c;
    return (a < b) ? -1 : (a > b);
}

static uint64_t hash_tuple(const int64_t *c, int d)
{
    uint64_t h = 1469598103934665603ULL;
    for (int j = 0; j < d; ++j) {
        uint64_t v = (uint64_t)c[j];
        h ^= v + 0x9e3779b97f4a7c15ULL + (h << 6) + (h >> 2);
        h *= 1099511628211ULL;
    }
    h ^= h >> 33; h *= 0xff51afd7ed558ccdULL; h ^= h >> 33;
    return h;
}

static const orc_cell *grid_find(const orc_grid *g, const int64_t *c)
{
    uint64_t s = hash_tuple(c, g->d) & g->mask;
    for (;;) {
        const orc_cell *e = &g->table[s];
        if (!e->used) return NULL;
        if (cmp_tuple(e->c, c, g->d) == 0) return e;
        s = (s + 1) & g->mask;
    }
}

static int grid_build(orc_grid *g, const double *pts, int64_t n, int d, double eps)
{
    double maxabs = 0.0;
    for (int64_t i = 0; i < n * d; ++i) {
        double a = fabs(pts[i]);
        if (a > maxabs) maxabs = a;
    }
    /* own robust width: > eps*(1+2^-51) + 2 * 2^-53 * maxabs with a wide margin */
    g->w = eps * (1.0 + ldexp(1.0, -30)) + ldexp(maxabs, -40);
    g->pts = pts; g->n = n; g->d = d;
    g->cellc = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * d > 0 ? n * d : 1));
    g->order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t i = 0; i < n; ++i) {
        g->order[i] = i;
        for (int j = 0; j < d; ++j) {
            double q = floor(pts[i * d + j] / g->w);
            if (!(fabs(q) < 4.0e18)) return -2; /* cell tuple would not fit int64 */
            g->cellc[i * d + j] = (int64_t)q;
        }
    }
    G_sort_ctx = g;
    qsort(g->order, (size_t)n, sizeof(int64_t), cmp_point);
    uint64_t cap = 16;
    while (cap < (uint64_t)(2 * n + 2)) cap <<= 1;
    g->table = (orc_cell *)calloc(cap, sizeof(orc_cell));
    g->mask = cap - 1;
    int64_t i = 0;
    while (i < n) {
        int64_t j = i + 1;
        const int64_t *ci = g->cellc + g->order[i] * d;
        while (j < n && cmp_tuple(g->cellc + g->order[j] * d, ci, d) == 0) ++j;
        uint64_t s = hash_tuple(ci, d) & g->mask;
        while (g->table[s].used) s = (s + 1) & g->mask;
        orc_cell *e = &g->table[s];
        e->used = 1; e->start = i; e->count = j - i;
        memcpy(e->c, ci, sizeof(int64_t) * (size_t)d);
        i = j;
    }
    return 0;
}

static void grid_free(orc_grid *g)
{
    free(g->cellc); free(g->order); free(g->table);
}

typedef struct {
    const orc_grid *g; double E; int include_self;
    int64_t q0, q1;
    int64_t *counts;            /* [q1-q0] per query, relative to the job's global q0 (may be NULL) */
    int64_t counts_base;
    uint64_t *buf; int64_t len, cap; int store;
} grid_job;

static int cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x < y) ? -1 : (x > y);
}

static void *grid_worker(void *arg)
{
    grid_job *J = (grid_job *)arg;
    const orc_grid *g = J->g;
    int d = g->d;
    int64_t noff = 1;
    for (int j = 0; j < d; ++j) noff *= 3;
    int64_t nb[ORC_MAXD];
    for (int64_t i = J->q0; i < J->q1; ++i) {
        const int64_t *ci = g->cellc + i * d;
        int64_t before = J->len, cnt = 0;
        for (int64_t o = 0; o < noff; ++o) {          /* every cell of the 3^d neighbourhood */
            int64_t r = o;
            for (int j = 0; j < d; ++j) { nb[j] = ci[j] + (r % 3) - 1; r /= 3; }
            const orc_cell *e = grid_find(g, nb);
            if (!e) continue;
            for (int64_t m = e->start; m < e->start + e->count; ++m) {
                int64_t k = g->order[m];
                if (k == i && !J->include_self) continue;
                if (orc_within(g->pts + i * d, g->pts + k * d, d, J->E)) {
                    ++cnt;
                    if (J->store) {
                        if (J->len == J->cap) {
                            J->cap = J->cap ? 2 * J->cap : 1024;
                            J->buf = (uint64_t *)realloc(J->buf, (size_t)J->cap * sizeof(uint64_t));
                        }
                        J->buf[J->len++] = ((uint64_t)i << 32) | (uint64_t)k;
                    }
                }
            }
        }
        if (J->store) qsort(J->buf + before, (size_t)(J->len - before), sizeof(uint64_t), cmp_u64);
        if (J->counts) J->counts[i - J->counts_base] = cnt;
        if (!J->store) J->len += cnt;
    }
    return NULL;
}

/* Join of queries [q0,q1) against all N points.  Two-call protocol as orc_rows: with
 * out == NULL returns the total (and fills counts[q1-q0] if non-NULL); with out != NULL
 * (capacity cap) also writes the sorted pairs.  Returns -1/-2 on bad input. */
int64_t orc_grid_join(const double *pts, int64_t n, int d, double eps, int include_self,
                      int64_t q0, int64_t q1, int nthreads, int64_t *counts,
                      uint64_t *out, int64_t cap)
{
    if (n < 0 || d < 1 || d > ORC_MAXD || !(eps > 0.0)) return -1;
    if (q0 < 0 || q1 > n || q0 > q1) return -1;
    if (nthreads < 1) nthreads = 1;
    orc_grid g;
    memset(&g, 0, sizeof g);
    if (grid_build(&g, pts, n, d, eps) != 0) { grid_free(&g); return -2; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    grid_job *jobs = (grid_job *)calloc((size_t)nthreads, sizeof(grid_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].g = &g; jobs[t].E = eps * eps; jobs[t].include_self = include_self;
        jobs[t].q0 = q0 + (q1 - q0) * t / nthreads;
        jobs[t].q1 = q0 + (q1 - q0) * (t + 1) / nthreads;
        jobs[t].counts = counts; jobs[t].counts_base = q0;
        jobs[t].store = (out != NULL);
        pthread_create(&th[t], NULL, grid_worker, &jobs[t]);
    }
    int64_t total = 0;
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; ++t) {
        if (out) {
            int64_t m = jobs[t].len;
            if (total + m > cap) m = cap - total > 0 ? cap - total : 0;
            if (m > 0) memcpy(out + total, jobs[t].buf, (size_t)m * sizeof(uint64_t));
        }
        total += jobs[t].len;
        free(jobs[t].buf);
    }
    free(th); free(jobs);
    grid_free(&g);
    return total;
}

/* ---- order-independent fingerprints of S (full-size parity without storing S) ------------ */
static uint64_t orc_mix_a(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;               /* SplitMix64 (Steele, Lea, Flood 2014) */
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t orc_mix_b(uint64_t x)
{
    uint64_t k = x ^ 0xC2B2AE3D27D4EB4FULL;                /* MurmurHash3 fmix64 */
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDULL;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ULL;
    k ^= k >> 33;
    return k;
}

/* exported so tests can pin the mixers against their published reference values */
uint64_t orc_mix(int which, uint64_t x) { return which == 0 ? orc_mix_a(x) : orc_mix_b(x); }

typedef struct {
    const orc_grid *g; double E; int include_self;
    int64_t q0, q1;
    int64_t *counts; int64_t counts_base;
    int64_t total; uint64_t fa, fb, fc;
} digest_job;

static void *digest_worker(void *arg)
{
    digest_job *J = (digest_job *)arg;
    const orc_grid *g = J->g;
    int d = g->d;
    int64_t noff = 1;
    for (int j = 0; j < d; ++j) noff *= 3;
    int64_t nb[ORC_MAXD];
    for (int64_t i = J->q0; i < J->q1; ++i) {
        const int64_t *ci = g->cellc + i * d;
        int64_t cnt = 0;
        for (int64_t o = 0; o < noff; ++o) {          /* every cell of the 3^d neighbourhood */
            int64_t r = o;
            for (int j = 0; j < d; ++j) { nb[j] = ci[j] + (r % 3) - 1; r /= 3; }
            const orc_cell *e = grid_find(g, nb);
            if (!e) continue;
            for (int64_t m = e->start; m < e->start + e->count; ++m) {
                int64_t k = g->order[m];
                if (k == i && !J->include_self) continue;
                if (orc_within(g->pts + i * d, g->pts + k * d, d, J->E)) {
                    uint64_t x = ((uint64_t)i << 32) | (uint64_t)k;
                    J->fa += orc_mix_a(x);
                    J->fb += orc_mix_b(x);
                    ++cnt;
                }
            }
        }
        J->fc += orc_mix_a(((uint64_t)i << 32) | (uint64_t)cnt);
        J->total += cnt;
        if (J->counts) J->counts[i - J->counts_base] = cnt;
    }
    return NULL;
}

/* Fingerprints of the pairs of queries [q0,q1) against all N points (full 3^d grid scan, the
 * same filter and predicate as orc_grid_join).  fp[0..2] = F_a, F_b, F_c over those queries;
 * counts[q1-q0] (may be NULL) = per-query counts.  Returns the number of pairs, or -1/-2. */
int64_t orc_grid_digest(const double *pts, int64_t n, int d, double eps, int include_self,
                        int64_t q0, int64_t q1, int nthreads, int64_t *counts, uint64_t *fp)
{
    if (n < 0 || d < 1 || d > ORC_MAXD || !(eps > 0.0) || !fp) return -1;
    if (q0 < 0 || q1 > n || q0 > q1) return -1;
    if (nthreads < 1) nthreads = 1;
    orc_grid g;
    memset(&g, 0, sizeof g);
    if (grid_build(&g, pts, n, d, eps) != 0) { grid_free(&g); return -2; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    digest_job *jobs = (digest_job *)calloc((size_t)nthreads, sizeof(digest_job));
    /* many more chunks than threads would balance skewed inputs better; static chunks keep it plain */
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].g = &g; jobs[t].E = eps * eps; jobs[t].include_self = include_self;
        jobs[t].q0 = q0 + (q1 - q0) * t / nthreads;
        jobs[t].q1 = q0 + (q1 - q0) * (t + 1) / nthreads;
        jobs[t].counts = counts; jobs[t].counts_base = q0;
        pthread_create(&th[t], NULL, digest_worker, &jobs[t]);
    }
    int64_t total = 0;
    fp[0] = fp[1] = fp[2] = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        total += jobs[t].total;
        fp[0] += jobs[t].fa; fp[1] += jobs[t].fb; fp[2] += jobs[t].fc;
    }
    free(th); free(jobs);
    grid_free(&g);
    return total;
}
