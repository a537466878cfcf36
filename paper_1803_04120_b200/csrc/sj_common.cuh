// sj_common.cuh -- internal declarations of libsj (B200 / sm_100a epsilon self-join).
// Nothing here is shared with oracle/ (task rule ③).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <string>
#include <vector>

#include "sj.h"

namespace sj {

// ---------------------------------------------------------------- errors
struct Error {
    sj_status status;
    std::string msg;
};

[[noreturn]] void fail(sj_status st, const std::string &msg);
void cuda_check(cudaError_t e, const char *what, const char *file, int line);
#define SJ_CUDA(x) ::sj::cuda_check((x), #x, __FILE__, __LINE__)

// ---------------------------------------------------------------- launch accounting
extern std::atomic<uint64_t> g_kernel_launches;
inline void count_launch(uint64_t k = 1) { g_kernel_launches.fetch_add(k, std::memory_order_relaxed); }
// Checks the launch configuration error right after a <<<>>> launch.
#define SJ_LAUNCHED() do { ::sj::count_launch(); SJ_CUDA(cudaGetLastError()); } while (0)

// ---------------------------------------------------------------- programmatic dependent launch
// A kernel launched with launch_pdl may start while the previous kernel on its stream is still
// running (its CTAs fill the SM slots the predecessor leaves free); it must call pdl_wait() before
// it touches anything the predecessor writes -- the wait returns once the predecessor grid has
// completed and its memory is visible.  A predecessor calls pdl_trigger() to let the dependent
// launch early.  Both are no-ops when the launch did not ask for it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args &&...args)
{
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    static const bool off = [] { const char *e = std::getenv("SJ_NO_PDL"); return e && *e && *e != '0'; }();
    cfg.attrs = at;
    cfg.numAttrs = off ? 0 : 1;
    SJ_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// ---------------------------------------------------------------- host tracing (SJ_TRACE=1..2)
// SJ_TRACE=1: host marks printed as they happen.  SJ_TRACE=2: one step's timeline (from the start of
// a build to the end of the following join): every mark() with its host time and every dev() with
// its host enqueue time AND the GPU time its stream reached that point (pooled events), printed
// together when the join's trace ends -- a GPU time well after the host time means the GPU was busy,
// one just after it means the GPU waited for the host.
struct HostTrace {
    bool on;
    const char *what;
    double t0, last;
    explicit HostTrace(const char *w);
    ~HostTrace();
    void mark(const char *stage);
    void dev(const char *stage, cudaStream_t s);
};

// ---------------------------------------------------------------- device memory
void *dev_alloc(size_t bytes, cudaStream_t s);
void dev_free(void *p, cudaStream_t s);
void *host_pinned_alloc(size_t bytes, size_t *granted);   // pooled pinned memory
void host_pinned_free(void *p);
void host_pinned_trim();              // release every cached pinned block

template <class T>
T *dalloc(size_t count, cudaStream_t s) { return static_cast<T *>(dev_alloc(count * sizeof(T), s)); }

// RAII scratch buffer freed stream-ordered.
template <class T>
struct Scratch {
    T *p = nullptr;
    cudaStream_t s = nullptr;
    Scratch() = default;
    Scratch(size_t n, cudaStream_t st) : p(dalloc<T>(n ? n : 1, st)), s(st) {}
    ~Scratch() { if (p) dev_free(p, s); }
    Scratch(const Scratch &) = delete;
    Scratch &operator=(const Scratch &) = delete;
    T *release() { T *q = p; p = nullptr; return q; }
};

// ---------------------------------------------------------------- the index as kernels see it
// Layout in HBM:
//   B[nG]   uint64  sorted linear ids of non-empty cells
//   G[nG+1] uint32  CSR starts: cell h = A-positions [G[h],G[h+1])
//   A[N]    uint32  original point id per A-position            (|A| = |D|)
//   pcell[N] uint32 cell of each A-position
//   X[d][N] double  SoA coordinates in A-order
//   masks   uint32  M_j bitmaps, concatenated (bits mask_off[j] .. mask_off[j+1])
struct DevIndex {
    int d;
    uint32_t n;
    uint32_t nG;
    double w;
    double eps2;                 // fl(eps*eps)
    double mins[SJ_MAX_DIM];
    uint64_t cpd[SJ_MAX_DIM];
    uint64_t strides[SJ_MAX_DIM];
    const uint64_t *B;
    const uint32_t *G;
    const uint32_t *A;
    const uint32_t *pcell;
    const double *X;
    const uint32_t *masks;       // bitmap, bit mask_off[j] + c = M_j contains c; nullptr if not built
    uint64_t mask_off[SJ_MAX_DIM + 1];
    // prefix directory over the top dir_k (slowest) dimensions:
    // dir[p] = first cell whose top-k coordinate prefix is >= p, p in [0, dir_P]; the cells of
    // prefix p are B[dir[p], dir[p+1]).  dir_k == d makes it a dense table of all cells.
    const uint32_t *dir;
    int dir_k;
    uint64_t dir_P;              // number of prefixes (entries = dir_P + 1)
    uint64_t dir_div;            // stride of dimension d - dir_k (key / dir_div = prefix)
    uint64_t pstride[SJ_MAX_DIM];// prefix strides: stride_j / dir_div for j >= d-k, else 0
    // search mode of the refine (uniform per index, chosen at directory build):
    //   kSearchDenseRows : dir_k == d, a row of 3 cells is [dir[p-1], dir[p+2])
    //   kSearchCellScan  : prefix ranges hold a few cells: scan them, test the low coordinates
    //   kSearchRows      : prefix ranges are large: bounded binary search per row of 3 cells
    int search_mode;
    uint32_t dir_ntop;           // 3^dir_k top-prefix offsets
    double inv_cpd[SJ_MAX_DIM];  // 1/|g_j| (fast exact divmod of low key parts, see refine.cuh)
    int64_t lowR[SJ_MAX_DIM + 1];// lowR[i] = sum_{m<i} stride_m: largest |key offset| of dims < i
    // occupancy bitmap over the top-(k+1) coordinate prefixes (cell-scan mode): bit q set iff some
    // cell has prefix q = key / occ_div; lets a prefix range be skipped by one bit test
    const uint32_t *occ;
    uint64_t occ_div;            // stride of dimension d-k-1
    uint64_t occ_cpd;            // |g_{d-k-1}|
    // second occupancy bitmap over (top-k prefix, c_{d-k-2}) -- the next low dimension -- for the
    // survivors of the first (both stored dilated by +-1 along their low dimension)
    const uint32_t *occ2;
    uint64_t occ2_cpd;           // |g_{d-k-2}|
    uint64_t occ_mul[SJ_MAX_DIM];   // bitmap index = sum_j c_j * occ_mul[j]: pstride_j * |g_{d-k-1}| for top
    uint64_t occ2_mul[SJ_MAX_DIM];  // dims, 1 for dim d-k-1 (occ) / d-k-2 (occ2), else 0
    // per non-empty cell, precomputed at build time: packed coordinates (c_j at bit cshift[j],
    // width cbits[j]; nullptr when sum of widths > 64) and the Alg. 1 line-6 mask word (bit i: move
    // -1 in dim i leaves M_i; bit 8+i: move +1 leaves M_i)
    const uint64_t *ccoord;
    const uint32_t *cmask;
    int key_fastdiv;             // key -> coordinates by double reciprocals (see index_build.cu)
    double inv_stride[SJ_MAX_DIM];
    uint32_t cshift[SJ_MAX_DIM];
    uint32_t cbits[SJ_MAX_DIM];
    // dense-cell tasks: every cell with >= dense_T points is cut into tasks of <= 32 consecutive
    // queries (start A-positions), processed one warp per task by k_refine_dense
    const uint32_t *dense_tasks;
    uint32_t n_dense_tasks;
    uint32_t dense_T;
    // FP32 self-join (R21; sj_self_join_f32 sets these on its private index): the refine
    // evaluates the predicate in binary32, s32 <= eps2f, instead of R1's binary64 s <= eps2
    int f32;
    float eps2f;
};

enum SearchMode { kSearchDenseRows = 0, kSearchCellScan = 1, kSearchRows = 2 };

// shape of the a5 sample: sample slots (runs of 32 queries every 32*step), buckets of `group` slots
struct EstimateShape {
    uint64_t step = 1, ns = 0, group = 32, nbk = 0;
};

// Cell coordinates from a linear id: c_j = (key / stride_j) mod |g_j|, taken from the slowest
// dimension down (each quotient < |g_j|).  Fast path: the quotient from a double reciprocal,
// corrected by +-1 in exact integer arithmetic (valid while quotients < 2^50 and keys < 2^63, which
// the host checks -> ix.key_fastdiv); otherwise exact 64-bit division.
template <int D>
__device__ __forceinline__ void key_to_coords(const DevIndex &ix, uint64_t key, uint64_t (&c)[D])
{
    uint64_t rem = key;
#pragma unroll
    for (int j = D - 1; j >= 1; --j) {
        const uint64_t st = ix.strides[j];
        uint64_t q;
        if (ix.key_fastdiv) {
            q = (uint64_t)((double)rem * ix.inv_stride[j]);
            if (q * st > rem) --q;
            else if ((q + 1) * st <= rem) ++q;
        } else {
            q = rem / st;
        }
        c[j] = q;
        rem -= q * st;
    }
    c[0] = rem;
}


}  // namespace sj

// The opaque handle.
struct sj_index {
    int device = 0;
    // build phase events (pooled); the t_*_ms timings are computed from them on first request
    // (sj_index_timings), so the build itself never waits on event queries
    cudaEvent_t tev[7] = {nullptr};
    bool timed = false;
    // the a5 estimate for the default join (full range, unicomp, self pairs, masks), run by the
    // build on the device before its final sync (join.cu spec_estimate_applies)
    bool spec_est_valid = false;
    sj::EstimateShape spec_shape{};
    std::vector<unsigned long long> spec_buckets;
    sj_index_view view{};        // geometry + device pointers (exported as is)
    sj::DevIndex dev{};          // same, in kernel form
    void *bufs[16] = {nullptr};  // owned device allocations
    int nbufs = 0;
    void *zbufs[2] = {nullptr, nullptr};   // the occupancy bitmaps: from / back to the zeroed-buffer cache
    size_t zbytes[2] = {0, 0};
    char *arena = nullptr;       // the build's contiguous arena (sj_index_view.packed), if any
};

struct sj_batch {
    uint64_t *pairs = nullptr;   // device or pinned host
    uint64_t n = 0;
    uint64_t cap = 0;
    int on_device = 1;
    // drain_csr: the batch is held in pinned host memory as CSR, one block [row offsets (rows + 1
    // uint32) | neighbours (n uint32)] at `pairs` (reinterpreted); rows = N of the joined index
    int csr = 0;
    uint64_t rows = 0;
};

struct sj_result {
    int device = 0;
    // pooled events: estimate start/end, first refine launch start, one (start, end) per batch run;
    // refine/estimate timings are computed on first request (sj_result_info with stats)
    cudaEvent_t est_ev[2] = {nullptr, nullptr};
    cudaEvent_t span0 = nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> runs;
    bool timed = false;
    std::vector<sj_batch> batches;
    sj_stats stats{};
    uint64_t total = 0;
    uint64_t n_points = 0;       // N of the index / point set the pairs' ids refer to
    // what the pairs cover (sj_dbscan needs the whole self-join): the A-order query range and the
    // predicate options of the join that produced them
    uint64_t q0 = 0, q1 = 0;
    int include_self = 1, unicomp = 1;
    int two_set = 0;             // a two-set join J(Q,P) (variants.cu): keys are query rows, not a self-join
};

namespace sj {
// context.cu -- reusable per-device streams / events / slot buffers
struct DevCtx {
    int dev = 0;
    std::vector<cudaStream_t> streams;
    std::vector<cudaEvent_t> events;
    void *d_slots = nullptr;     // device scratch for cursors / counters
    void *h_slots = nullptr;     // pinned mirror (mapped: kernels may write it directly)
    size_t slot_bytes = 0;
    uint32_t doorbell = 0;       // epoch of the last device -> host doorbell written into h_slots
    // the join's per-stream counter blocks (only joins touch them): device + pinned mirror, and whether
    // the previous join left them zero (it re-zeroes them on each stream right after reading them back)
    void *jb_d = nullptr;
    void *jb_h = nullptr;        // mapped pinned mirror (kernels publish into it)
    void *jb_hd = nullptr;       // its device address
    size_t jb_bytes = 0;
    bool jb_clean = false;
};
// spin until a device-written doorbell shows `epoch` (the stream is queried now and then so a failed
// kernel is reported, not waited for); returns false if the stream drained without ringing
bool wait_doorbell(const volatile unsigned int *bell, unsigned int epoch, cudaStream_t s);
// Zeroed device buffers (the occupancy bitmaps): a released bitmap is zeroed at release time (the
// index's free, off any build's critical path) and handed to the next build that asks for one at least
// as large, so the build needs no memset.  zbuf_get returns nullptr when none is cached.
void *zbuf_get(int dev, size_t bytes, size_t *granted);
void zbuf_put(int dev, void *p, size_t bytes);     // caller: p is no longer in use; zeroes + caches
void zbuf_trim(int dev);
// grow the join blocks to `bytes` (a fresh allocation is not clean)
void ensure_join_blocks(DevCtx *c, size_t bytes);
DevCtx *acquire_ctx(int dev, int nstreams, int nevents, size_t slot_bytes);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device): the call costs
// tens of microseconds of host time, on the build's / join's critical path if repeated.
void set_max_dyn_smem(const void *func, int bytes);
int device_count();                            // cached cudaGetDeviceCount (0 on error)
bool alloc_hook_set();                         // api.cu: a user allocator hook is installed
// device batch buffers, cached per device up to a limit (sj_set_result_cache_limit).  put() records
// an event on the freeing stream (cudaStreamLegacy when none is given, which orders after the
// caller's work on blocking streams such as torch's default stream); get() makes the new owner's
// stream wait for it, so a reused buffer is never written while the old owner still reads it.
void *result_buffer_get(int dev, size_t bytes, cudaStream_t s);
void result_buffer_put(int dev, void *p, cudaStream_t s);
void result_cache_trim(int dev);                 // free every cached buffer of dev (-1: all devices)
void set_result_cache_limit(size_t bytes);
void scratch_trim(int dev);
int device_sm_count(int dev);                  // cached multiprocessor count
// L2 persisting window over the build's input (context.cu): begin/stop on a stream, end after a sync
size_t l2_persist_limit(int dev);
void l2_persist_begin(int dev, cudaStream_t s, const void *base, size_t bytes);
void l2_persist_stop(int dev, cudaStream_t s);
void l2_persist_end(int dev);
// the build's scratch buffer (nullptr if busy: use the pool instead); *zero_prefix = leading bytes known
// to be zero; the releasing build states how many leading bytes it leaves zero
void *scratch_acquire(int dev, size_t bytes, size_t *zero_prefix);
void scratch_release(int dev, void *p, size_t zero_prefix);
// pooled timing events (cudaEventCreate / elapsed-time queries stay off the critical path)
cudaEvent_t event_get(int dev);
void event_put(int dev, cudaEvent_t e);
void result_finalize_timing(sj_result *r);
void result_release_events(sj_result *r);
void index_finalize_timing(sj_index *idx);
void release_ctx(DevCtx *c);
struct CtxGuard {
    DevCtx *c;
    bool idle = false;           // the owner already synchronised every stream it used
    ~CtxGuard()
    {
        if (!c) return;
        if (!idle)
            for (auto s : c->streams) cudaStreamSynchronize(s);
        release_ctx(c);
    }
};

// index_build.cu
sj_index *build_index_impl(const double *points, uint64_t n, int d, double eps, const sj_build_opts &o);
sj_index *import_index_impl(const sj_index_view &v, int device, bool borrow);
void free_index_impl(sj_index *idx);

// radix_sort.cu
void radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp,
                      uint32_t n, int key_bits, cudaStream_t s, bool *result_in_tmp);

void bucket_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp, uint32_t n,
                       uint64_t div, uint64_t P, uint32_t *hist, uint32_t *overflow, uint32_t *local,
                       uint32_t *cellcnt, cudaStream_t s);
void exclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s);
void exclusive_scan_u32_consume(uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s);   // zeroes in
void exclusive_scan_u32_dup(const uint32_t *in, uint32_t *out, uint32_t *out2, uint64_t n, cudaStream_t s);
void inclusive_scan_u32(const uint32_t *in, uint32_t *out, uint64_t n, cudaStream_t s);

// extras.cu
void sort_pairs_device(uint64_t *pairs, uint64_t n, uint64_t n_points, cudaStream_t s);
void result_to_csr_impl(const sj_result *r, uint64_t n_points, uint64_t *row_offsets, uint32_t *neighbors);
void dbscan_impl(const sj_result *r, uint32_t min_pts, int32_t *labels, uint64_t *n_clusters, uint64_t *n_core,
                 uint64_t *n_noise);
void batch_to_csr_device(const uint64_t *pairs, uint64_t n, uint64_t rows, bool sorted, uint32_t *counts,
                         uint32_t *cursor, uint32_t *dst_offs, uint32_t *dst_nbrs, cudaStream_t s, int nsm);
void result_fingerprint_impl(const sj_result *r, uint64_t *fp, uint32_t *counts);
sj_result *brute_force_impl(const double *points, uint64_t n, int d, double eps, const sj_build_opts &bo,
                            const sj_join_opts &jo);

// variants.cu
sj_result *join_sets_impl(const sj_index *idx, const double *queries, uint64_t nq, int queries_on_device,
                          const sj_join_opts &o);
sj_result *self_join_f32_impl(const float *points, uint64_t n, int d, float eps, const sj_build_opts &bo,
                              const sj_join_opts &o);
void knn_impl(const double *points, uint64_t n, const double *queries, uint64_t nq, int d, uint32_t k, double eps0,
              const sj_build_opts &bo, uint32_t *ids, double *dist2, sj_knn_stats *st);
void knn_self_impl(const double *points, uint64_t n, int d, uint32_t k, double eps0, const sj_build_opts &bo,
                   uint32_t *ids, double *dist2, sj_knn_stats *st);

// join.cu
sj_result *self_join_impl(const sj_index *idx, const sj_join_opts &o);
void neighbor_counts_impl(const sj_index *idx, const sj_join_opts &o, uint32_t *cnt, uint64_t *total);
void plan_shards_impl(const sj_index *idx, uint32_t world, uint64_t *cuts);
EstimateShape estimate_shape(uint64_t nq);
// Completion publish: a one-CTA kernel (k_publish) launched right behind the work it reports, on the
// same stream (a stream's last batch, or the build's estimate), copies `words` 8-byte words from
// device memory into mapped pinned memory, optionally zeroes the source, optionally computes the
// masks-trivial flag into the source first, and rings a doorbell the host polls -- instead of a D2H
// copy + stream sync (each ~5-10 us of latency).  (An epilogue inside the refine kernels raised their
// register spills: 6-D eps=8 join 4.1 -> 6.0 ms.)
struct Publish {
    unsigned long long *src;       // device words (nullptr: no publish)
    unsigned long long *dst;       // mapped host words (device address)
    uint32_t words;
    int zero_src;                  // zero src after copying (the join's counter blocks)
    volatile unsigned int *bell;   // mapped host doorbell
    unsigned int epoch;
    // join counter blocks: instead of the raw block, publish [sum of the work slots (4 words) | the
    // first nslots cursor slots (2 words each)] -- 8 KB less over PCIe
    uint32_t reduce_slots;         // work slots to sum (0: plain copy of `words`)
    uint32_t nslots;
    uint32_t *masks_flag;          // build: aux word for "every coordinate occupied" (or nullptr)
    const uint32_t *masks;         //   the masks and, per dimension, the bit range [lo, hi] of the
    int d;                         //   coordinates 1 .. |g_j|-2 that must all be set
    uint64_t mask_lo[SJ_MAX_DIM], mask_hi[SJ_MAX_DIM];
};
void launch_publish(const Publish &p, cudaStream_t s);

void launch_estimate(const DevIndex &ix, int device, const sj_join_opts &o, uint64_t q0, uint64_t q1,
                     const EstimateShape &es, unsigned long long *dbk, cudaStream_t s, const Publish *pub = nullptr);
void plan_from_buckets(const double *bucket_est, uint64_t nbk, uint64_t width, uint64_t q0, uint64_t q1,
                       uint64_t capacity, int min_batches, double margin, std::vector<uint64_t> &cuts,
                       std::vector<uint64_t> &est, uint64_t *estimated_total);
void plan_batches(const uint32_t *sample_counts, uint64_t n_samples, uint64_t step, uint64_t q_begin,
                  uint64_t q_end, uint64_t capacity, int min_batches, double margin,
                  std::vector<uint64_t> &cuts, std::vector<uint64_t> &est, uint64_t *estimated_total);
}  // namespace sj
