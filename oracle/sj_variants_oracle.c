/*
 * sj_variants_oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain CPU definitions of the SURVEY.md §8(f)
 * rank-4 variants built on the self-join's predicate: the two-set similarity join and the k-nearest-
 * neighbour self-join.  Same rules as sj_oracle.c (compiled into the same libsj_oracle.so with
 * gcc -O2 -ffp-contract=off -fno-fast-math): no code, header or constant shared with the CUDA path,
 * only tests/, smoke() and bench.py's baseline legs load it.
 *
 * The predicate and distance are the self-join's (§3; R1-R2):
 *     s(a,b) = (((a_0-b_0)^2 + (a_1-b_1)^2) + ...) + (a_{d-1}-b_{d-1})^2   left to right, no FMA,
 *     a within eps of b  <=>  s(a,b) <= fl(eps*eps).
 *
 * Two-set join ("Self-joins and the related similarity join"; reading R19):
 *     J(Q,P) = { (i,k) : s(q_i, p_k) <= fl(eps^2) },  packed (uint64)i << 32 | k, sorted ascending.
 *   orc_join_sets_brute -- the definition written out (nested loops).
 *   orc_join_sets_grid  -- P sorted by an integer cell tuple floor(x_j / w_o) with its own robust
 *                          width w_o (as sj_oracle.c's grid: a filter only), each query scanning the
 *                          3^d tuples around its own by binary search in that sorted order.
 *
 * kNN self-join ("applying this work to other spatial searches, such as kNN"; reading
 * R20): for each query point i, the k points k != i (ids of P) with the smallest (s(q_i,p_k), k),
 * lexicographically -- ties in s broken by the smaller id, so the answer is unique.
 *   orc_knn -- brute force over all of P per query with a sorted insertion list of length k.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static double vo_dist(const double *a, const double *b, int d)
{
    double s = 0.0;
    for (int j = 0; j < d; ++j) {
        double t = a[j] - b[j];
        double t2 = t * t;
        s = s + t2;
    }
    return s;
}

/* ---- two-set join, brute force ------------------------------------------------------------ */
/* Writes up to cap pairs (may be NULL); returns |J| or -1. */
int64_t orc_join_sets_brute(const double *Q, int64_t nq, const double *P, int64_t n, int d, double eps,
                            uint64_t *out, int64_t cap)
{
    if (nq < 0 || n < 0 || d < 1 || !(eps > 0.0)) return -1;
    double E = eps * eps;
    int64_t cnt = 0;
    for (int64_t i = 0; i < nq; ++i)
        for (int64_t k = 0; k < n; ++k)
            if (vo_dist(Q + i * d, P + k * d, d) <= E) {
                if (out && cnt < cap) out[cnt] = ((uint64_t)i << 32) | (uint64_t)k;
                ++cnt;
            }
    return cnt;
}

/* ---- two-set join, sorted-tuple grid over P, full 3^d scan ------------------------------- */
#define VO_MAXD 8

typedef struct {
    int d; int64_t n;
    const double *P;
    double w;
    int64_t *tup;        /* [n*d] cell tuple of each point of P */
    int64_t *order;      /* ids of P sorted by (tuple, id) */
} vo_grid;

static vo_grid *VO_CTX;

static int vo_cmp_tuple(const int64_t *a, const int64_t *b, int d)
{
    for (int j = 0; j < d; ++j) {
        if (a[j] < b[j]) return -1;
        if (a[j] > b[j]) return 1;
    }
    return 0;
}

static int vo_cmp_point(const void *pa, const void *pb)
{
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    int c = vo_cmp_tuple(VO_CTX->tup + a * VO_CTX->d, VO_CTX->tup + b * VO_CTX->d, VO_CTX->d);
    if (c) return c;
    return (a < b) ? -1 : (a > b);
}

/* first position in `order` whose tuple is >= c */
static int64_t vo_lower(const vo_grid *g, const int64_t *c)
{
    int64_t lo = 0, hi = g->n;
    while (lo < hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (vo_cmp_tuple(g->tup + g->order[mid] * g->d, c, g->d) < 0) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

/* cell tuple of a coordinate vector; returns 0 if some |x_j / w| is too large for int64 */
static int vo_tuple(const double *x, int d, double w, int64_t *c)
{
    for (int j = 0; j < d; ++j) {
        double q = floor(x[j] / w);
        if (!(fabs(q) < 4.0e18)) return 0;
        c[j] = (int64_t)q;
    }
    return 1;
}

typedef struct {
    const vo_grid *g; const double *Q; double E;
    int64_t q0, q1;
    int64_t *counts;
    uint64_t *buf; int64_t len, cap; int store;
} vo_job;

static int vo_cmp_u64(const void *a, const void *b)
{
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x < y) ? -1 : (x > y);
}

static void *vo_sets_worker(void *arg)
{
    vo_job *J = (vo_job *)arg;
    const vo_grid *g = J->g;
    int d = g->d;
    int64_t noff = 1;
    for (int j = 0; j < d; ++j) noff *= 3;
    int64_t ci[VO_MAXD], nb[VO_MAXD];
    for (int64_t i = J->q0; i < J->q1; ++i) {
        const double *q = J->Q + i * d;
        int64_t before = J->len, cnt = 0;
        if (vo_tuple(q, d, g->w, ci)) {
            for (int64_t o = 0; o < noff; ++o) {          /* every tuple of the 3^d neighbourhood */
                int64_t r = o;
                for (int j = 0; j < d; ++j) { nb[j] = ci[j] + (r % 3) - 1; r /= 3; }
                for (int64_t m = vo_lower(g, nb); m < g->n; ++m) {
                    int64_t k = g->order[m];
                    if (vo_cmp_tuple(g->tup + k * d, nb, d) != 0) break;
                    if (vo_dist(q, g->P + k * d, d) <= J->E) {
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
        }
        if (J->store) qsort(J->buf + before, (size_t)(J->len - before), sizeof(uint64_t), vo_cmp_u64);
        if (J->counts) J->counts[i] = cnt;
        if (!J->store) J->len += cnt;
    }
    return NULL;
}

/* J(Q,P) through the grid.  Two-call protocol: out == NULL returns |J| (and fills counts[nq] if
 * non-NULL); out != NULL (capacity cap) also writes the pairs sorted.  -1 bad input, -2 a point of P
 * too large for the grid's integer tuples. */
int64_t orc_join_sets_grid(const double *Q, int64_t nq, const double *P, int64_t n, int d, double eps,
                           int nthreads, int64_t *counts, uint64_t *out, int64_t cap)
{
    if (nq < 0 || n < 0 || d < 1 || d > VO_MAXD || !(eps > 0.0)) return -1;
    if (nthreads < 1) nthreads = 1;
    double maxabs = 0.0;
    for (int64_t i = 0; i < n * d; ++i) if (fabs(P[i]) > maxabs) maxabs = fabs(P[i]);
    for (int64_t i = 0; i < nq * d; ++i) if (fabs(Q[i]) > maxabs) maxabs = fabs(Q[i]);
    vo_grid g;
    g.d = d; g.n = n; g.P = P;
    /* robust width (as sj_oracle.c): > eps*(1+2^-51) + the rounding of x/w over |x| <= maxabs */
    g.w = eps * (1.0 + ldexp(1.0, -30)) + ldexp(maxabs, -40);
    g.tup = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * d > 0 ? n * d : 1));
    g.order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t k = 0; k < n; ++k) {
        g.order[k] = k;
        if (!vo_tuple(P + k * d, d, g.w, g.tup + k * d)) { free(g.tup); free(g.order); return -2; }
    }
    VO_CTX = &g;
    qsort(g.order, (size_t)n, sizeof(int64_t), vo_cmp_point);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    vo_job *jobs = (vo_job *)calloc((size_t)nthreads, sizeof(vo_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].g = &g; jobs[t].Q = Q; jobs[t].E = eps * eps;
        jobs[t].q0 = nq * t / nthreads;
        jobs[t].q1 = nq * (t + 1) / nthreads;
        jobs[t].counts = counts;
        jobs[t].store = (out != NULL);
        pthread_create(&th[t], NULL, vo_sets_worker, &jobs[t]);
    }
    int64_t total = 0;
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    for (int t = 0; t < nthreads; ++t) {       /* threads hold ascending query ranges: concatenation is sorted */
        if (out) {
            int64_t m = jobs[t].len;
            if (total + m > cap) m = cap - total > 0 ? cap - total : 0;
            if (m > 0) memcpy(out + total, jobs[t].buf, (size_t)m * sizeof(uint64_t));
        }
        total += jobs[t].len;
        free(jobs[t].buf);
    }
    free(th); free(jobs);
    free(g.tup); free(g.order);
    return total;
}

/* ---- kNN by brute force --------------------------------------------------------------------- */
typedef struct {
    const double *Q; const int64_t *qself; const double *P; int64_t n; int d; int k;
    int64_t q0, q1;
    int64_t *ids; double *s;
} vo_knn_job;

static void *vo_knn_worker(void *arg)
{
    vo_knn_job *J = (vo_knn_job *)arg;
    int d = J->d, K = J->k;
    for (int64_t i = J->q0; i < J->q1; ++i) {
        int64_t *bid = J->ids + i * K;
        double *bs = J->s + i * K;
        int64_t have = 0;
        int64_t self = J->qself ? J->qself[i] : -1;
        for (int64_t k = 0; k < J->n; ++k) {
            if (k == self) continue;
            double s = vo_dist(J->Q + i * d, J->P + k * d, d);
            /* k ascends, so an equal s never displaces an earlier (smaller) id */
            if (have == K && !(s < bs[K - 1])) continue;
            int64_t pos = have < K ? have : K - 1;
            while (pos > 0 && s < bs[pos - 1]) {
                bs[pos] = bs[pos - 1];
                bid[pos] = bid[pos - 1];
                --pos;
            }
            bs[pos] = s;
            bid[pos] = k;
            if (have < K) ++have;
        }
        for (int64_t t = have; t < K; ++t) { bid[t] = -1; bs[t] = INFINITY; }
    }
    return NULL;
}

/* For queries Q[0..nq) against P[0..n): ids[nq*k] (int64, -1 if fewer than k candidates) and
 * s[nq*k] (the distances s, +inf for missing), each row ascending in (s, id).  qself: NULL, or per
 * query the id of P to exclude (the query itself in a self kNN join; -1 = none).  Returns 0 / -1. */
int orc_knn(const double *Q, int64_t nq, const int64_t *qself, const double *P, int64_t n, int d, int k,
            int nthreads, int64_t *ids, double *s)
{
    if (nq < 0 || n < 0 || d < 1 || k < 1 || !ids || !s) return -1;
    if (nthreads < 1) nthreads = 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    vo_knn_job *jobs = (vo_knn_job *)calloc((size_t)nthreads, sizeof(vo_knn_job));
    for (int t = 0; t < nthreads; ++t) {
        vo_knn_job j = {Q, qself, P, n, d, k, nq * t / nthreads, nq * (t + 1) / nthreads, ids, s};
        jobs[t] = j;
        pthread_create(&th[t], NULL, vo_knn_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th); free(jobs);
    return 0;
}

/* ---- FP32 self-join, brute force (SURVEY.md §8(f) rank 4 "FP32 coordinates (SuperEGO's precision)";
 *      PAPER.md:393 "We execute the algorithm using 32-bit floats"; reading R21) ------------
 * The self-join's definition with every coordinate, difference, square and sum a binary32 value:
 *     s32(a,b) = (((a_0-b_0)^2 + (a_1-b_1)^2) + ...) in float, left to right, no FMA,
 *     (i,k) in S32  <=>  s32(p_i,p_k) <= fl32(eps*eps),   eps itself a float.
 * Writes up to cap pairs (may be NULL), sorted (loop order); returns |S32| or -1. */
static float vo_dist_f32(const float *a, const float *b, int d)
{
    float s = 0.0f;
    for (int j = 0; j < d; ++j) {
        float t = a[j] - b[j];
        float t2 = t * t;
        s = s + t2;
    }
    return s;
}

int64_t orc_brute_force_f32(const float *pts, int64_t n, int d, float eps, int include_self,
                            uint64_t *out, int64_t cap)
{
    if (n < 0 || d < 1 || !(eps > 0.0f)) return -1;
    float E = eps * eps;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = 0; k < n; ++k) {
            if (i == k && !include_self) continue;
            if (vo_dist_f32(pts + i * d, pts + k * d, d) <= E) {
                if (out && cnt < cap) out[cnt] = ((uint64_t)i << 32) | (uint64_t)k;
                ++cnt;
            }
        }
    return cnt;
}

/* ---- J(Q,P) fingerprints (full-size parity of two-set results too large to hold) ------------------
 * The grid join above, accumulating instead of storing: |J|, F_a = sum of mix_a(pair), F_b = sum of
 * mix_b(pair) (mod 2^64; the mixers of sj_oracle.c, orc_mix), per-query counts optional. */
uint64_t orc_mix(int which, uint64_t x);

typedef struct {
    const vo_grid *g; const double *Q; double E;
    int64_t q0, q1;
    int64_t *counts;
    int64_t total; uint64_t fa, fb;
} vo_dig_job;

static void *vo_digest_worker(void *arg)
{
    vo_dig_job *J = (vo_dig_job *)arg;
    const vo_grid *g = J->g;
    int d = g->d;
    int64_t noff = 1;
    for (int j = 0; j < d; ++j) noff *= 3;
    int64_t ci[VO_MAXD], nb[VO_MAXD];
    for (int64_t i = J->q0; i < J->q1; ++i) {
        const double *q = J->Q + i * d;
        int64_t cnt = 0;
        if (vo_tuple(q, d, g->w, ci)) {
            for (int64_t o = 0; o < noff; ++o) {
                int64_t r = o;
                for (int j = 0; j < d; ++j) { nb[j] = ci[j] + (r % 3) - 1; r /= 3; }
                for (int64_t m = vo_lower(g, nb); m < g->n; ++m) {
                    int64_t k = g->order[m];
                    if (vo_cmp_tuple(g->tup + k * d, nb, d) != 0) break;
                    if (vo_dist(q, g->P + k * d, d) <= J->E) {
                        uint64_t x = ((uint64_t)i << 32) | (uint64_t)k;
                        J->fa += orc_mix(0, x);
                        J->fb += orc_mix(1, x);
                        ++cnt;
                    }
                }
            }
        }
        if (J->counts) J->counts[i] = cnt;
        J->total += cnt;
    }
    return NULL;
}

int64_t orc_join_sets_digest(const double *Q, int64_t nq, const double *P, int64_t n, int d, double eps,
                             int nthreads, int64_t *counts, uint64_t *fp)
{
    if (nq < 0 || n < 0 || d < 1 || d > VO_MAXD || !(eps > 0.0) || !fp) return -1;
    if (nthreads < 1) nthreads = 1;
    double maxabs = 0.0;
    for (int64_t i = 0; i < n * d; ++i) if (fabs(P[i]) > maxabs) maxabs = fabs(P[i]);
    for (int64_t i = 0; i < nq * d; ++i) if (fabs(Q[i]) > maxabs) maxabs = fabs(Q[i]);
    vo_grid g;
    g.d = d; g.n = n; g.P = P;
    g.w = eps * (1.0 + ldexp(1.0, -30)) + ldexp(maxabs, -40);
    g.tup = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n * d > 0 ? n * d : 1));
    g.order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t k = 0; k < n; ++k) {
        g.order[k] = k;
        if (!vo_tuple(P + k * d, d, g.w, g.tup + k * d)) { free(g.tup); free(g.order); return -2; }
    }
    VO_CTX = &g;
    qsort(g.order, (size_t)n, sizeof(int64_t), vo_cmp_point);
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    vo_dig_job *jobs = (vo_dig_job *)calloc((size_t)nthreads, sizeof(vo_dig_job));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].g = &g; jobs[t].Q = Q; jobs[t].E = eps * eps;
        jobs[t].q0 = nq * t / nthreads;
        jobs[t].q1 = nq * (t + 1) / nthreads;
        jobs[t].counts = counts;
        pthread_create(&th[t], NULL, vo_digest_worker, &jobs[t]);
    }
    int64_t total = 0;
    fp[0] = fp[1] = 0;
    for (int t = 0; t < nthreads; ++t) {
        pthread_join(th[t], NULL);
        total += jobs[t].total;
        fp[0] += jobs[t].fa; fp[1] += jobs[t].fb;
    }
    free(th); free(jobs);
    free(g.tup); free(g.order);
    return total;
}
