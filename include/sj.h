/*
 * sj.h -- C ABI of the B200-native epsilon-distance self-join (arXiv 1803.04120, "GPU
 * Accelerated Self-join for the Distance Similarity Metric", Gowanlock & Karsin).
 *
 * Library: paper_1803_04120_b200/libsj.so (hand-written CUDA for sm_100a, no CPU fallback).
 * Conventions for every entry point:
 *   - returns sj_status; out-parameters are written only when SJ_OK is returned;
 *   - no C++ exception crosses the ABI; on failure sj_last_error() returns a thread-local,
 *     human-readable message (valid until the next failing call on the same thread);
 *   - argument errors are detected on the host BEFORE any allocation or CUDA call;
 *   - CUDA failures return SJ_ERR_CUDA with cudaGetErrorString() in sj_last_error().
 *
 * The problem (§3 "Problem Statement"): for points D = (p_0..p_{N-1}) in d
 * dimensions (2 <= d <= 6) and eps > 0, return every ORDERED pair (i,k) with
 *     s(p_i,p_k) <= fl(eps*eps),  s(a,b) = (((a_0-b_0)^2 + (a_1-b_1)^2) + ...) + (a_{d-1}-b_{d-1})^2,
 * every -, *, + one IEEE-754 binary64 round-to-nearest operation, left to right, no FMA
 * (readings R1-R2: the squared form of PAPER.md:130's sqrt(...) <= eps; ties kept).
 * Both orientations are returned ("add both (p,q) and (q,p)"); (p,p) is
 * returned unless include_self == 0 (reading R3).  A pair is packed as one uint64
 * (key << 32) | value with key = query id, value = neighbour id ("key/value
 * pair"), ids = 0-based input row positions (reading R5), so integer order == (key,value)
 * order.  The SET of pairs is deterministic; their order inside a batch is not (atomic
 * emission); compare after a canonical sort.
 */
#ifndef SJ_H
#define SJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SJ_ABI_VERSION 5   /* 5: sj_join_sets, sj_knn_self, sj_knn_join, sj_self_join_f32; 4: drain_csr, CSR batches, sj_dbscan, sj_result_counters */
#define SJ_MAX_DIM 6

typedef enum {
    SJ_OK = 0,
    SJ_ERR_ARG = 1,           /* bad pointer/size/eps/option (eps<=0, non-finite, fl(eps^2) not
                                 normal, N==0, N>=2^32, query range outside [0,N), ...)        */
    SJ_ERR_NONFINITE = 2,     /* a coordinate is NaN or +-inf                                   */
    SJ_ERR_DIM = 3,           /* d not in [2, 6] ("we only focus on dimensions 2--6") */
    SJ_ERR_KEY_OVERFLOW = 4,  /* prod_j |g_j| >= 2^64: linear cell ids would not fit a uint64;
                                 use a larger eps (SPEC S.132)                                  */
    SJ_ERR_NOMEM = 5,         /* device or pinned-host allocation failed                        */
    SJ_ERR_CUDA = 6,          /* any other CUDA runtime error                                    */
    SJ_ERR_EPS_MISMATCH = 7,  /* reserved (S.233); the index carries eps, so not raised today  */
    SJ_ERR_STATE = 8          /* NULL handle / handle used on the wrong device / no GPU          */
} sj_status;

typedef struct sj_index sj_index;    /* opaque; immutable after build; device-resident; may be
                                        shared read-only by concurrent joins                      */
typedef struct sj_result sj_result;  /* opaque; owns its batches (device or pinned host memory);
                                        independent of the index (either may be freed first)      */

/* ---- options ------------------------------------------------------------------------------ */
typedef struct {
    int device;            /* CUDA device ordinal                                                */
    int points_on_device;  /* 1: `points` is a device pointer on `device`; 0: host memory (copied
                              H2D inside the call; pinned memory gives full PCIe bandwidth)       */
    void *stream;          /* cudaStream_t to order the build on (NULL = library stream); the call
                              returns after the build completed                                   */
    int build_masks;       /* 1 (default): build the per-dimension masks M_j       */
    int speculative_estimate; /* 1 (default): run the a5 result-size estimate of the DEFAULT join
                              (full range, unicomp, self pairs, masks) on the device before the
                              build's final sync; sj_self_join with those options then skips its
                              own estimate launch and host round trip (same sample, same counts) */
} sj_build_opts;

typedef struct {
    int unicomp;                   /* 1 (default): duplicate-search removal, Alg. 2;
                                      0: full 3^d search, Alg. 1              */
    int include_self;              /* 1 (default): emit (p,p)                                      */
    uint64_t batch_capacity_pairs; /* C: pairs per result batch buffer (default 2^28)             */
    int min_batches;               /* minimum number of batches (default 3)         */
    int n_streams;                 /* concurrent CUDA streams for the batch pipeline (default 3)  */
    int result_on_host;            /* 0 (default): batches stay in device memory; 1: each batch is
                                      drained into pinned host memory while later batches compute */
    uint64_t query_begin;          /* queries = A-order positions [query_begin, query_end)       */
    uint64_t query_end;            /*   (0,0 = all N).  A-order is the cell-sorted order of the
                                      index; ranges of it are the multi-GPU shard unit.  With
                                      unicomp, a shard emits both orientations of the pairs its
                                      queries decide, so the union over a partition of [0,N) is
                                      exactly S with no duplicates.                               */
    int use_masks;                 /* 1 (default): filter adjacent coordinates by M_j (Alg. 1 l.6) */
    int lanes_per_query;           /* 0 (default): chosen per index; else 1,2,4,8,16 or 32 GPU lanes
                                      cooperate on one query (a tuning / testing knob; S is
                                      independent of it)                                         */
    int dense_cells;               /* 1 (default): queries of populous cells (>= 16 points) run one
                                      warp per 32 queries with warp-buffered emission; 0: off     */
    int sort_pairs;                /* 0 (default); 1: each batch is sorted by (key, value) on the
                                      device before it is returned / drained       */
    int drain_csr;                 /* 0 (default); 1 (requires result_on_host): each batch crosses
                                      PCIe as CSR neighbour lists -- uint32 row offsets over all N
                                      keys + one uint32 neighbour per pair, 4 B/pair instead of 8
                                      (PAPER.md:209 sorted key/value pairs; the D2H drain is the
                                      bottleneck PAPER.md:262/601 names).  Rows are in arbitrary
                                      order unless sort_pairs = 1 (then ascending).  Read with
                                      sj_result_batch_csr; sj_result_copy_to_host expands them.  */
} sj_join_opts;

typedef struct {
    uint64_t pairs;              /* pairs emitted (sum over batches)                              */
    uint64_t cells_probed;       /* binary searches of B performed (work counter)                  */
    uint64_t candidates_tested;  /* distance evaluations (work counter)                            */
    uint64_t estimated_pairs;    /* the sampled estimate used to plan the batches                  */
    uint32_t batches;            /* batches delivered                                              */
    uint32_t retries;            /* batches re-run after a buffer overflow                         */
    float estimate_ms;           /* device time of the estimator kernel (CUDA events)             */
    float refine_ms;             /* sum of device times of the refine kernels (CUDA events)       */
    float refine_max_ms;         /* longest single refine launch                                   */
    float total_ms;              /* host wall time of sj_self_join                                 */
    uint32_t refine_launches;    /* refine kernel launches (incl. retries)                         */
    float refine_span_ms;        /* device time from the first refine launch's start to the last
                                    one's end (batches on different streams overlap)              */
} sj_stats;

typedef struct {
    int d, device;
    uint64_t n;                  /* |D|                                                            */
    uint64_t n_cells;            /* |G| = |B|                                       */
    double eps, eps2, w;         /* eps, fl(eps*eps), cell width (reading R6)                      */
    double mins[SJ_MAX_DIM];     /* per-dimension minima (exact)                                   */
    uint64_t cpd[SJ_MAX_DIM];    /* |g_j| = cells per dimension incl. one pad cell each side (R7) */
    uint64_t strides[SJ_MAX_DIM];/* linearisation strides, dimension 1 fastest (R8)               */
    int key_bits;                /* ceil(log2(prod |g_j|)): bits sorted by the radix sort          */
    uint64_t mask_offsets[SJ_MAX_DIM + 1]; /* bit offsets of M_j inside `masks`; [d] = total bits   */
    /* device pointers (owned by the index; valid while it lives):                                 */
    const uint64_t *B;           /* [n_cells] sorted linear ids of the non-empty cells             */
    const uint32_t *G;           /* [n_cells+1] cell h holds A-positions [G[h], G[h+1])            */
    const uint32_t *A;           /* [n] original point id at each A-position                       */
    const uint32_t *pcell;       /* [n] cell h of each A-position                                  */
    const double *X;             /* [d][n] SoA coordinates in A-order: X[j*n+k] = D[A[k]][j]      */
    const uint32_t *masks;       /* bitmap of the M_j: bit mask_offsets[j]+c set iff coordinate c of
                                    dimension j is occupied (little-endian words), or NULL          */
    int dir_k;                   /* prefix directory over the dir_k slowest dimensions (bounds every
                                    binary search of B; rebuilt from B on import)                  */
    uint64_t dir_entries;        /* entries of dir (= number of prefixes + 1)                     */
    const uint32_t *dir;         /* [dir_entries] dir[p] = first cell with top-dir_k prefix >= p   */
    /* build timings (CUDA events, ms).  t_geometry_ms covers the min/max pass, the geometry AND the
       key pass: the key pass is a programmatic dependent launch that overlaps the geometry tail, so
       there is no event between them (t_keys_ms = 0) */
    float t_h2d_ms, t_geometry_ms, t_keys_ms, t_sort_ms, t_compact_ms, t_total_ms;
    /* the index's arrays as ONE contiguous device buffer (multi-GPU broadcast):
       packed_bytes bytes at `packed`; X, A, pcell, G, masks and B sit at the off_* byte offsets in it
       (off_masks = UINT64_MAX when the masks live outside it, at `masks`).  NULL for an index whose
       arrays are not contiguous (sj_index_import with copies).                                    */
    const void *packed;
    uint64_t packed_bytes;
    uint64_t off_X, off_A, off_pcell, off_G, off_masks, off_B;
} sj_index_view;

/* Fill *o with the defaults above. */
void sj_build_opts_default(sj_build_opts *o);
void sj_join_opts_default(sj_join_opts *o);

/* ---- REQUIRED entry points (north_star) ---------------------------------------------------- */

/* Build the sparse eps-grid index (§4.2-4.4): geometry (per-dimension
 * min/max, cell width w, |g_j|), per-point linear cell ids, stable radix sort on device,
 * compaction into the non-empty-cell list B / ranges G / point list A, SoA coordinate gather
 * and masks M_j.
 *   points : row-major N x d float64 (AoS), host or device per opts->points_on_device; borrowed
 *            for the duration of the call only (copied).
 *   n      : N, 1 <= N < 2^32.     d: 2..6.     eps: finite, > 0, fl(eps*eps) normal.
 *   opts   : NULL = defaults.      *out: receives the new index (free with sj_free_index).
 * Errors: SJ_ERR_ARG, SJ_ERR_DIM, SJ_ERR_NONFINITE, SJ_ERR_KEY_OVERFLOW, SJ_ERR_NOMEM,
 *         SJ_ERR_CUDA, SJ_ERR_STATE (no device). */
sj_status sj_build_index(const double *points, uint64_t n, int d, double eps,
                         const sj_build_opts *opts, sj_index **out);

/* Run the self-join over the index (Alg. 1-2, §5.1 batching): estimate the result size
 * on a deterministic sample (count-only kernel), cut the A-order queries into k >= min_batches
 * contiguous batches, run the refine kernel per batch on n_streams streams with warp-aggregated
 * emission into batch buffers, drain to pinned host memory if result_on_host, re-run any batch
 * whose buffer overflowed.  Returns after all batches completed.
 *   idx : an index built or imported on the current process.   opts: NULL = defaults.
 *   *out: receives the result (free with sj_free_result).
 * Errors: SJ_ERR_ARG (bad options / query range), SJ_ERR_STATE (NULL index), SJ_ERR_NOMEM,
 *         SJ_ERR_CUDA. */
sj_status sj_self_join(const sj_index *idx, const sj_join_opts *opts, sj_result **out);

/* Build + join in ONE call (the common path of a user holding points): sj_build_index followed by
 * sj_self_join on the same device, with no return to the caller in between.  *out_index receives
 * the index (free with sj_free_index) unless out_index is NULL, in which case it is freed here
 * (after the join completed).  Errors: those of sj_build_index and sj_self_join. */
sj_status sj_self_join_points(const double *points, uint64_t n, int d, double eps, const sj_build_opts *bopts,
                              const sj_join_opts *jopts, sj_index **out_index, sj_result **out);

/* Release a result and every batch buffer it owns.  NULL-safe.  Device batch buffers go to a
 * per-device cache reused by later joins; they are reused only after the work queued before this
 * call on the legacy default stream (and every blocking stream) completed. */
void sj_free_result(sj_result *r);

/* Same, ordered after the work queued on `stream` (cudaStream_t; NULL = legacy default stream):
 * use it when the caller read zero-copy batch views on a non-blocking stream. */
void sj_free_result_async(sj_result *r, void *stream);

/* ---- supporting entry points ---------------------------------------------------------------- */

void sj_free_index(sj_index *idx);   /* NULL-safe */

/* Totals and work counters of a result. Any out pointer may be NULL.  The device timings in
 * *stats are computed from the join's CUDA events on the first call that asks for stats. */
sj_status sj_result_info(const sj_result *r, uint64_t *n_pairs, uint32_t *n_batches, sj_stats *stats);

/* The work counters alone -- [pairs, cells_probed, candidates_tested, retries] -- without the lazy
 * event-timing evaluation sj_result_info(stats) performs (the multi-GPU step all-reduces them).
 * Errors: SJ_ERR_STATE (NULL result), SJ_ERR_ARG (NULL counters). */
sj_status sj_result_counters(const sj_result *r, uint64_t counters[4]);

/* N of the point set the result's ids refer to (the joined index's N).  Errors: SJ_ERR_STATE (NULL). */
sj_status sj_result_n_points(const sj_result *r, uint64_t *n_points);

/* Batch b of a result: *pairs points to *n packed uint64 pairs in device memory (*on_device=1,
 * on the index's device) or pinned host memory (*on_device=0); owned by the result. */
sj_status sj_result_batch(const sj_result *r, uint32_t b, const uint64_t **pairs, uint64_t *n,
                          int *on_device);

/* Batch b of a drain_csr result: row_offsets[i] .. row_offsets[i+1] index the neighbours (original
 * ids) that batch b holds for key i in `neighbors`; *n_rows = N of the joined index (row_offsets has
 * N + 1 entries), *n = pairs in the batch.  Pinned host memory owned by the result.  Errors:
 * SJ_ERR_STATE if the batch is not in CSR form (sj_result_batch then returns its pairs; for a CSR
 * batch sj_result_batch fails with SJ_ERR_STATE), SJ_ERR_ARG for a bad index. */
sj_status sj_result_batch_csr(const sj_result *r, uint32_t b, const uint32_t **row_offsets,
                              const uint32_t **neighbors, uint64_t *n_rows, uint64_t *n);

/* DBSCAN (Ester et al. 1996) read off a whole self-join result -- the epsilon-
 * neighbourhood table N_eps(p) = {q : (p,q) in S}.  core(p) <=> |N_eps(p)| >= min_pts (p counts
 * itself); clusters = connected components of the core points under S, labelled by their
 * smallest core id; a non-core point with core neighbours takes the smallest of their labels
 * (border), else -1 (noise) -- DESIGN.md reading R17.  labels: int32[N] in DEVICE memory on the
 * result's device (caller-owned), indexed by original id.  Optional outputs: number of clusters,
 * core points, noise points.  The result must cover the full query range, in pair batches (not
 * drain_csr); device or pinned-host batches.  Blocks until written.  Errors: SJ_ERR_ARG (NULL
 * labels, min_pts < 1, partial result, N >= 2^31), SJ_ERR_STATE (CSR batches), SJ_ERR_CUDA. */
sj_status sj_dbscan(const sj_result *r, uint32_t min_pts, int32_t *labels, uint64_t *n_clusters,
                    uint64_t *n_core, uint64_t *n_noise);

/* Copy all pairs of a result, batch after batch, into host memory dst (capacity cap pairs).
 * Errors: SJ_ERR_ARG if cap < total. */
sj_status sj_result_copy_to_host(const sj_result *r, uint64_t *dst, uint64_t cap);

/* The whole result as CSR neighbour lists (the sorted key/value pairs of
 * PAPER.md:209): row_offsets[i] .. row_offsets[i+1] (n_points + 1 uint64, DEVICE memory on the
 * result's device) index the neighbours of point i (original ids) in `neighbors` (n_pairs uint32,
 * DEVICE memory), ascending within a row.  4 bytes per pair instead of 8.  Both arrays are owned by
 * the caller.  Blocks until written.  Errors: SJ_ERR_ARG (n_points out of range, NULL arrays,
 * >= 2^32 pairs), SJ_ERR_NOMEM (scratch of 16 B per pair), SJ_ERR_CUDA. */
sj_status sj_result_to_csr(const sj_result *r, uint64_t n_points, uint64_t *row_offsets, uint32_t *neighbors);

/* Order-independent fingerprints of the result's pair multiset (full-size parity of results too
 * large to hold twice): fp[0] = sum over pairs x of mix_a(x),
 * fp[1] = sum of mix_b(x), both mod 2^64, with mix_a = SplitMix64's output function of
 * x + 0x9E3779B97F4A7C15 and mix_b = MurmurHash3's fmix64 of x ^ 0xC2B2AE3D27D4EB4F.  The
 * fingerprints add over disjoint results (e.g. query shards).  counts: NULL, or DEVICE memory for
 * n_points uint32 (the N of the joined point set) receiving cnt[i] = pairs with key i in this
 * result (zeroed by the call).  Reads device batches in place and pinned host batches through
 * their UVA mapping.  Blocks until done.  Errors: SJ_ERR_STATE (NULL result, or a key >= N),
 * SJ_ERR_ARG (fp NULL), SJ_ERR_CUDA. */
sj_status sj_result_fingerprint(const sj_result *r, uint64_t fp[2], uint32_t *counts);

/* Per-point neighbour counts cnt[i] = |{k : (i,k) in S}| without materialising
 * pairs.  cnt: device pointer to N uint32 on the index's device (zeroed by the call), or NULL.
 * *total receives |S| (restricted to the pairs decided by queries of opts' query range). */
sj_status sj_neighbor_counts(const sj_index *idx, const sj_join_opts *opts, uint32_t *cnt,
                             uint64_t *total);

/* GPU brute-force nested-loop join: every query compared with
 * every point with the same predicate; one batch.  points/n/d/eps/bopts as sj_build_index; from
 * jopts only include_self, sort_pairs and result_on_host are used.  O(N^2): for cross-checks and
 * the paper's brute-force comparison, not for large N. */
sj_status sj_brute_force_join(const double *points, uint64_t n, int d, double eps, const sj_build_opts *bopts,
                              const sj_join_opts *jopts, sj_result **out);

/* ---- SURVEY §8(f) rank 4 variants on the same index and predicate --------------------------- */

/* Two-set similarity join J(Q,P) ("the related similarity join"; R19): every
 * ordered pair (i,k), i a row of `queries`, k an original id of the index's points P, with
 * s(q_i,p_k) <= fl(eps^2) (the self-join's predicate and eps -- the index's), packed (i << 32) | k.
 * Each query probes the 3^d cells around its own cell in P's grid (R7 against P's geometry; no
 * unicomp, no self rule); the queries are processed sorted by that cell (a warp of one populous cell
 * shares candidate tiles).  Batches are contiguous ranges of the sorted queries (>= min_batches when
 * there is output): with >= 65536 queries planned from a sampled count (the self-join's estimate-
 * then-batch scheme; buffers of 1.75x the estimate, an overflowed batch re-filled at its exact size),
 * else from exact per-query counts (a count pass, then exact sizes).
 *   queries : row-major nq x d float64, device memory on the index's device (queries_on_device = 1;
 *             read after the work queued on the legacy default stream) or host memory (copied).
 *   opts    : NULL = defaults; batch_capacity_pairs, min_batches, result_on_host and sort_pairs are
 *             used; drain_csr must be 0; the query range / unicomp / include_self / masks / lanes /
 *             dense options do not apply and are ignored.
 *   *out    : a result like sj_self_join's (sj_result_* accessors, copy, CSR, fingerprints); its
 *             n_points is max(nq, N).  sj_dbscan rejects it.  Blocks until complete.
 * Errors: SJ_ERR_STATE (NULL index), SJ_ERR_ARG (nq >= 2^32, NULL queries with nq > 0, drain_csr,
 *         capacity 0), SJ_ERR_NONFINITE (a query coordinate NaN / inf), SJ_ERR_NOMEM, SJ_ERR_CUDA. */
sj_status sj_join_sets(const sj_index *idx, const double *queries, uint64_t nq, int queries_on_device,
                       const sj_join_opts *opts, sj_result **out);

/* FP32 self-join (SURVEY §8(f) rank 4 "FP32 coordinates (SuperEGO's precision)"; PAPER.md:393 runs
 * SuperEGO "using 32-bit floats"; R21): the self-join of float points with every coordinate
 * difference, square and sum a binary32 round-to-nearest operation, left to right, no FMA:
 *     (i,k) in S32  <=>  (((p_i0-p_k0)^2 + (p_i1-p_k1)^2) + ...) <= fl32(eps*eps)   (all in float).
 * Pairs / ids / result and every join option as sj_self_join (unicomp holds: the float distance is
 * symmetric).  The grid index is built from the points widened exactly to binary64 for radius
 * eps * (1 + 2^-16), so every pair the float predicate accepts lies in adjacent cells; the self-join's
 * path then runs with the predicate in binary32 (estimate, batches, sparse / dense refine, drains).
 *   points : row-major n x d float32, host or device per bopts->points_on_device.   eps: float > 0,
 *            fl32(eps*eps) normal.   jopts: NULL = defaults.
 * Errors: as sj_build_index / sj_self_join. */
sj_status sj_self_join_f32(const float *points, uint64_t n, int d, float eps, const sj_build_opts *bopts,
                           const sj_join_opts *jopts, sj_result **out);

typedef struct {
    uint32_t rounds;             /* radius steps + 1 (index builds)                                  */
    double eps_final;            /* radius of the last round                                        */
    uint64_t cells_probed;       /* cell lookups over all rounds                                    */
    uint64_t candidates_tested;  /* distance evaluations over all rounds                            */
} sj_knn_stats;

/* kNN self-join ("other spatial searches, such as kNN"; R20): for every point
 * i the k points j != i with the smallest (s(p_i,p_j), j) -- s the self-join's rounded distance, ties
 * to the smaller id -- written as row i of ids[n*k] (original ids) and dist2[n*k] (s), ascending.
 * The ε-grid does it: an index with radius eps0; each point's k best among the points of its 3^d
 * neighbour cells within eps are final when there are k of them (every other point fails the
 * predicate); the rest are re-run on an index for eps * 4^(1/d) (the neighbourhood volume x 4), until
 * none is left.
 *   points : row-major n x d float64, host or device per bopts->points_on_device.
 *   k      : 1..32, k + 1 <= n < 2^32.       eps0: the first radius, finite, > 0 (about the k-th
 *            neighbour distance is cheapest; too small costs rounds, too large costs candidates).
 *   ids, dist2 : DEVICE memory on bopts->device, n*k uint32 / float64, caller-owned.
 *   stats  : NULL or receives the rounds / final radius / work counters.
 * Blocks until written.  Errors: SJ_ERR_ARG, SJ_ERR_DIM, SJ_ERR_NONFINITE (from the index build),
 *         SJ_ERR_KEY_OVERFLOW (eps0 too small for the range), SJ_ERR_NOMEM, SJ_ERR_CUDA. */
sj_status sj_knn_self(const double *points, uint64_t n, int d, uint32_t k, double eps0, const sj_build_opts *bopts,
                      uint32_t *ids, double *dist2, sj_knn_stats *stats);

/* kNN join of query rows against points (the two-set form of sj_knn_self; DESIGN.md
 * R20): row i of ids[nq*k] / dist2[nq*k] = the k points j of `points` with the smallest
 * (s(q_i,p_j), j), ascending; nothing is excluded (a query equal to a point gets it at s = 0).  Same
 * growing-radius grid certificate (R19's cells for queries outside the points' box).
 *   points (n x d) and queries (nq x d): row-major float64, both host or both device per
 *   bopts->points_on_device.  k: 1..32, k <= n < 2^32, nq < 2^32.  ids / dist2: DEVICE memory.
 * Errors: as sj_knn_self, and SJ_ERR_NONFINITE for a NaN / inf query. */
sj_status sj_knn_join(const double *points, uint64_t n, const double *queries, uint64_t nq, int d, uint32_t k,
                      double eps0, const sj_build_opts *bopts, uint32_t *ids, double *dist2, sj_knn_stats *stats);

/* Multi-GPU shard plan: cut the A-order queries [0, N) into `world` contiguous
 * ranges cuts[r] .. cuts[r+1] (cuts: world + 1 host uint64) of about equal estimated work, using
 * the a5 sampled estimate (the build's own estimate of the default join when it
 * has one, else a count-only run of the sample now): per query, its estimated emitted pairs plus a
 * constant search cost.  Joining every range (sj_join_opts.query_begin/end) on its own GPU gives
 * shards whose union is exactly S.  Errors: SJ_ERR_STATE, SJ_ERR_ARG (world < 1), SJ_ERR_CUDA. */
sj_status sj_plan_shards(const sj_index *idx, uint32_t world, uint64_t *cuts);

/* Geometry, sizes, timings and device pointers of an index (for tests and NCCL broadcast). */
sj_status sj_index_export(const sj_index *idx, sj_index_view *view);

/* Same as sj_index_export, with the build-phase timings t_*_ms filled in (device time from CUDA
 * events recorded during sj_build_index; computed on this first request so the build itself never
 * waits on event queries -- sj_index_export leaves them 0 until then).  Blocks until the build's
 * events completed. */
sj_status sj_index_timings(const sj_index *idx, sj_index_view *view);

/* Build an index on `device` from a view whose array pointers are device memory on that device
 * (e.g. buffers received by an NCCL broadcast); the arrays are copied.  Only the geometry fields
 * (d, n, n_cells, eps, eps2, w, mins, cpd, strides, key_bits, mask_offsets) and the array pointers
 * B, G, A, pcell, X, masks are read; the prefix directory, occupancy bitmaps and dense-cell tasks
 * are rebuilt from B and G on the device. */
sj_status sj_index_import(const sj_index_view *view, int device, sj_index **out);

/* Same, but the arrays are BORROWED, not copied: the index reads B, G, A, pcell, X, masks in place,
 * and the caller keeps that memory alive (and unmodified) until sj_free_index.  For a rank that
 * received the packed buffer of sj_index_view.packed, this makes the import cost only the rebuild
 * of the small derived tables. */
sj_status sj_index_import_borrowed(const sj_index_view *view, int device, sj_index **out);

/* Optional allocator hook for device memory (index arrays, result batches, scratch).
 * alloc(bytes, device, stream, ctx) returns a device pointer or NULL; release(ptr, ctx).
 * Pass NULLs to restore the default (cudaMallocAsync from the device's default pool). */
void sj_set_allocator(void *(*alloc)(size_t, int, void *, void *), void (*release)(void *, void *),
                      void *ctx);

/* Upper bound on the device memory the freed-result-batch cache may hold per device (default
 * 48 GB, or env SJ_RESULT_CACHE_BYTES); lowering it releases cached buffers above the new bound. */
void sj_set_result_cache_limit(uint64_t bytes);

/* Release every cache the library keeps on `device` (-1: all devices): freed result batches, the
 * index-build scratch buffer, pooled pinned host blocks, and memory held by the device's default
 * stream-ordered pool beyond what live objects use.  Live indexes and results are untouched.
 * Synchronises the device.  Errors: SJ_ERR_CUDA. */
sj_status sj_trim(int device);

/* Batch planner (host-only, no GPU needed): given per-sample emission counts of a strided sample
 * (sample s stands for `step` consecutive queries starting at q_begin + s*step), cut
 * [q_begin, q_end) into k >= min_batches ranges whose estimated pairs stay below
 * capacity/(1+margin).  cuts[0..k] receives the boundaries (cuts capacity max_cuts+1).
 * Returns k in *k.  (§5.1; reading R13.) */
sj_status sj_plan_batches(const uint32_t *sample_counts, uint64_t n_samples, uint64_t step,
                          uint64_t q_begin, uint64_t q_end, uint64_t capacity, int min_batches,
                          double margin, uint64_t *cuts, uint32_t max_cuts, uint32_t *k,
                          uint64_t *estimated_total);

/* Measurement helper (bench.py roofline): throughput of the FP64 pipe for single DADD and DMUL
 * instructions on `device`, in operations per second (a saturating microbenchmark, best of 3
 * timed runs).  The predicate issues no FMA (reading R1), so this -- not the datasheet's
 * FMA-counted FP64 figure -- is the refine's FP64 roofline.  Errors: SJ_ERR_CUDA. */
sj_status sj_diag_fp64_peak(int device, double *dadd_ops_per_s, double *dmul_ops_per_s);

/* Number of CUDA kernels this library has launched in the process (monotone counter). */
uint64_t sj_kernel_launches(void);

/* Thread-local message of the last failure ("" if none). */
const char *sj_last_error(void);

/* SJ_ABI_VERSION. */
int sj_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SJ_H */
