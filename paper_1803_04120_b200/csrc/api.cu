// api.cu -- the C ABI of libsj (include/sj.h): argument marshalling, error translation,
// device / pinned-host memory management.  No compute happens here.
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <set>

#include "sj_common.cuh"

namespace sj {

std::atomic<uint64_t> g_kernel_launches{0};

namespace {
thread_local std::string t_last_error;

struct AllocHook {
    void *(*alloc)(size_t, int, void *, void *) = nullptr;
    void (*release)(void *, void *) = nullptr;
    void *ctx = nullptr;
};
AllocHook g_hook;
std::mutex g_hook_mu;
// provenance of hooked allocations: a pointer is released by the hook that produced it, whatever
// hook is installed when it is freed (sj_set_allocator may change in between)
std::map<void *, AllocHook> g_hooked;
std::set<int> g_pool_configured;
std::mutex g_pool_mu;

void configure_pool(int dev)
{
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_pool_configured.count(dev)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;  // keep freed memory cached in the pool (no OS round trips)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // let blocks freed on one stream (e.g. result batches freed on the legacy stream) serve
        // allocations on another once the free completed, instead of mapping fresh memory
        int on = 1;
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowOpportunistic, &on);
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &on);
        cudaMemPoolSetAttribute(pool, cudaMemPoolReuseFollowEventDependencies, &on);
    }
    g_pool_configured.insert(dev);
}

// ---- pinned host pool (result batches drained to the host; reused across joins)
std::mutex g_pin_mu;
std::multimap<size_t, void *> g_pin_free;     // size -> block
std::map<void *, size_t> g_pin_size;          // block -> size
}  // namespace

void fail(sj_status st, const std::string &msg) { throw Error{st, msg}; }

void cuda_check(cudaError_t e, const char *what, const char *file, int line)
{
    if (e == cudaSuccess) return;
    char buf[512];
    std::snprintf(buf, sizeof buf, "%s: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
    cudaGetLastError();  // clear sticky-free errors
    if (e == cudaErrorMemoryAllocation) throw Error{SJ_ERR_NOMEM, buf};
    throw Error{SJ_ERR_CUDA, buf};
}

bool alloc_hook_set()
{
    std::lock_guard<std::mutex> lk(g_hook_mu);
    return g_hook.alloc != nullptr;
}

void *dev_alloc(size_t bytes, cudaStream_t s)
{
    if (bytes == 0) bytes = 1;
    int dev = 0;
    SJ_CUDA(cudaGetDevice(&dev));
    {
        std::lock_guard<std::mutex> lk(g_hook_mu);
        if (g_hook.alloc) {
            void *p = g_hook.alloc(bytes, dev, s, g_hook.ctx);
            if (!p) fail(SJ_ERR_NOMEM, "allocator hook returned NULL");
            g_hooked[p] = g_hook;
            return p;
        }
    }
    configure_pool(dev);
    void *p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bytes, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        char buf[160];
        std::snprintf(buf, sizeof buf, "device allocation of %zu bytes failed: %s", bytes, cudaGetErrorString(e));
        fail(SJ_ERR_NOMEM, buf);
    }
    return p;
}

void dev_free(void *p, cudaStream_t s)
{
    if (!p) return;
    AllocHook h;
    {
        std::lock_guard<std::mutex> lk(g_hook_mu);
        auto it = g_hooked.find(p);
        if (it != g_hooked.end()) {
            h = it->second;
            g_hooked.erase(it);
        }
    }
    if (h.alloc) {
        // hooked memory is released stream-unordered: make prior work complete first
        if (s) cudaStreamSynchronize(s);
        else cudaDeviceSynchronize();
        if (h.release) h.release(p, h.ctx);
        return;
    }
    cudaFreeAsync(p, s);
}

void *host_pinned_alloc(size_t bytes, size_t *granted)
{
    if (bytes == 0) bytes = 1;
    {
        std::lock_guard<std::mutex> lk(g_pin_mu);
        auto it = g_pin_free.lower_bound(bytes);
        if (it != g_pin_free.end() && it->first <= 2 * bytes + (64u << 20)) {
            void *p = it->second;
            if (granted) *granted = it->first;
            g_pin_free.erase(it);
            return p;
        }
    }
    const size_t gran = 2u << 20;
    const size_t sz = (bytes + gran - 1) / gran * gran;
    void *p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, sz, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        // trim the pool once and retry
        {
            std::lock_guard<std::mutex> lk(g_pin_mu);
            for (auto &kv : g_pin_free) { cudaFreeHost(kv.second); g_pin_size.erase(kv.second); }
            g_pin_free.clear();
        }
        e = cudaHostAlloc(&p, sz, cudaHostAllocPortable);
        if (e != cudaSuccess) { cudaGetLastError(); fail(SJ_ERR_NOMEM, "pinned host allocation failed"); }
    }
    std::lock_guard<std::mutex> lk(g_pin_mu);
    g_pin_size[p] = sz;
    if (granted) *granted = sz;
    return p;
}

void host_pinned_trim()
{
    std::lock_guard<std::mutex> lk(g_pin_mu);
    for (auto &kv : g_pin_free) {
        cudaFreeHost(kv.second);
        g_pin_size.erase(kv.second);
    }
    g_pin_free.clear();
}

void host_pinned_free(void *p)
{
    if (!p) return;
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_size.find(p);
    if (it == g_pin_size.end()) return;
    g_pin_free.emplace(it->second, p);
}

}  // namespace sj

using sj::Error;

#define SJ_API_BEGIN try {
#define SJ_API_END                                                                    \
    }                                                                                 \
    catch (const Error &e) {                                                          \
        sj::t_last_error = e.msg;                                                     \
        return e.status;                                                              \
    }                                                                                 \
    catch (const std::bad_alloc &) {                                                  \
        sj::t_last_error = "host allocation failed";                                  \
        return SJ_ERR_NOMEM;                                                          \
    }                                                                                 \
    catch (...) {                                                                     \
        sj::t_last_error = "unexpected internal error";                               \
        return SJ_ERR_CUDA;                                                           \
    }

extern "C" {

int sj_abi_version(void) { return SJ_ABI_VERSION; }

const char *sj_last_error(void) { return sj::t_last_error.c_str(); }

uint64_t sj_kernel_launches(void) { return sj::g_kernel_launches.load(); }

void sj_build_opts_default(sj_build_opts *o)
{
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->device = 0;
    o->points_on_device = 0;
    o->stream = nullptr;
    o->build_masks = 1;
    o->speculative_estimate = 1;
}

void sj_join_opts_default(sj_join_opts *o)
{
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->unicomp = 1;
    o->include_self = 1;
    o->batch_capacity_pairs = 1ull << 28;
    o->min_batches = 3;
    o->n_streams = 3;
    o->result_on_host = 0;
    o->query_begin = 0;
    o->query_end = 0;
    o->use_masks = 1;
    o->lanes_per_query = 0;
    o->dense_cells = 1;
    o->sort_pairs = 0;
}

sj_status sj_build_index(const double *points, uint64_t n, int d, double eps, const sj_build_opts *opts,
                         sj_index **out)
{
    SJ_API_BEGIN
    if (!out) sj::fail(SJ_ERR_ARG, "out is NULL");
    sj_build_opts o;
    if (opts) o = *opts;
    else sj_build_opts_default(&o);
    *out = sj::build_index_impl(points, n, d, eps, o);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_self_join(const sj_index *idx, const sj_join_opts *opts, sj_result **out)
{
    SJ_API_BEGIN
    if (!out) sj::fail(SJ_ERR_ARG, "out is NULL");
    if (!idx) sj::fail(SJ_ERR_STATE, "index is NULL");
    sj_join_opts o;
    if (opts) o = *opts;
    else sj_join_opts_default(&o);
    *out = sj::self_join_impl(idx, o);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_self_join_points(const double *points, uint64_t n, int d, double eps, const sj_build_opts *bopts,
                              const sj_join_opts *jopts, sj_index **out_index, sj_result **out)
{
    SJ_API_BEGIN
    if (!out) sj::fail(SJ_ERR_ARG, "out is NULL");
    sj_build_opts bo;
    if (bopts) bo = *bopts;
    else sj_build_opts_default(&bo);
    sj_join_opts jo;
    if (jopts) jo = *jopts;
    else sj_join_opts_default(&jo);
    sj_index *idx = sj::build_index_impl(points, n, d, eps, bo);
    try {
        *out = sj::self_join_impl(idx, jo);
    } catch (...) {
        sj::free_index_impl(idx);
        throw;
    }
    if (out_index) *out_index = idx;
    else sj::free_index_impl(idx);
    return SJ_OK;
    SJ_API_END
}

void sj_free_result_async(sj_result *r, void *stream)
{
    if (!r) return;
    cudaSetDevice(r->device);
    sj::result_release_events(r);
    for (auto &b : r->batches) {
        if (!b.pairs) continue;
        if (b.on_device) sj::result_buffer_put(r->device, b.pairs, static_cast<cudaStream_t>(stream));
        else sj::host_pinned_free(b.pairs);
    }
    delete r;
}

void sj_free_result(sj_result *r) { sj_free_result_async(r, nullptr); }

void sj_set_result_cache_limit(uint64_t bytes) { sj::set_result_cache_limit((size_t)bytes); }

sj_status sj_trim(int device)
{
    SJ_API_BEGIN
    sj::result_cache_trim(device);
    sj::scratch_trim(device);
    sj::zbuf_trim(device);
    sj::host_pinned_trim();
    const int n = sj::device_count();
    for (int dv = 0; dv < n; ++dv) {
        if (device >= 0 && dv != device) continue;
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dv) == cudaSuccess) {
            SJ_CUDA(cudaSetDevice(dv));
            SJ_CUDA(cudaDeviceSynchronize());
            SJ_CUDA(cudaMemPoolTrimTo(pool, 0));
        } else {
            cudaGetLastError();
        }
    }
    return SJ_OK;
    SJ_API_END
}

void sj_free_index(sj_index *idx) { sj::free_index_impl(idx); }

sj_status sj_result_info(const sj_result *r, uint64_t *n_pairs, uint32_t *n_batches, sj_stats *stats)
{
    SJ_API_BEGIN
    if (!r) sj::fail(SJ_ERR_STATE, "result is NULL");
    if (n_pairs) *n_pairs = r->total;
    if (n_batches) *n_batches = (uint32_t)r->batches.size();
    if (stats) {
        sj::result_finalize_timing(const_cast<sj_result *>(r));   // lazy: event queries on request
        *stats = r->stats;
    }
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_counters(const sj_result *r, uint64_t counters[4])
{
    SJ_API_BEGIN
    if (!r) sj::fail(SJ_ERR_STATE, "result is NULL");
    if (!counters) sj::fail(SJ_ERR_ARG, "counters is NULL");
    counters[0] = r->total;
    counters[1] = r->stats.cells_probed;
    counters[2] = r->stats.candidates_tested;
    counters[3] = r->stats.retries;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_batch(const sj_result *r, uint32_t b, const uint64_t **pairs, uint64_t *n, int *on_device)
{
    SJ_API_BEGIN
    if (!r) sj::fail(SJ_ERR_STATE, "result is NULL");
    if (b >= r->batches.size()) sj::fail(SJ_ERR_ARG, "batch index out of range");
    const sj_batch &bt = r->batches[b];
    if (bt.csr) sj::fail(SJ_ERR_STATE, "batch is in CSR form (drain_csr): use sj_result_batch_csr");
    if (pairs) *pairs = bt.pairs;
    if (n) *n = bt.n;
    if (on_device) *on_device = bt.on_device;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_batch_csr(const sj_result *r, uint32_t b, const uint32_t **row_offsets, const uint32_t **neighbors,
                              uint64_t *n_rows, uint64_t *n)
{
    SJ_API_BEGIN
    if (!r) sj::fail(SJ_ERR_STATE, "result is NULL");
    if (b >= r->batches.size()) sj::fail(SJ_ERR_ARG, "batch index out of range");
    const sj_batch &bt = r->batches[b];
    if (!bt.csr) sj::fail(SJ_ERR_STATE, "batch is not in CSR form: use sj_result_batch");
    const uint32_t *blk = reinterpret_cast<const uint32_t *>(bt.pairs);
    if (row_offsets) *row_offsets = blk;
    if (neighbors) *neighbors = blk ? blk + bt.rows + 1 : nullptr;
    if (n_rows) *n_rows = bt.rows;
    if (n) *n = bt.n;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_copy_to_host(const sj_result *r, uint64_t *dst, uint64_t cap)
{
    SJ_API_BEGIN
    if (!r) sj::fail(SJ_ERR_STATE, "result is NULL");
    if (!dst && r->total) sj::fail(SJ_ERR_ARG, "dst is NULL");
    if (cap < r->total) sj::fail(SJ_ERR_ARG, "dst capacity smaller than the result");
    SJ_CUDA(cudaSetDevice(r->device));
    uint64_t off = 0;
    for (const auto &b : r->batches) {
        if (!b.n) continue;
        if (b.csr) {                       // expand the CSR block: (row << 32) | neighbour
            const uint32_t *offs = reinterpret_cast<const uint32_t *>(b.pairs), *nb = offs + b.rows + 1;
            for (uint64_t i = 0; i < b.rows; ++i)
                for (uint32_t e = offs[i]; e < offs[i + 1]; ++e) dst[off + e] = (i << 32) | nb[e];
        } else if (b.on_device) {
            SJ_CUDA(cudaMemcpy(dst + off, b.pairs, b.n * 8, cudaMemcpyDeviceToHost));
        } else {
            std::memcpy(dst + off, b.pairs, b.n * 8);
        }
        off += b.n;
    }
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_n_points(const sj_result *r, uint64_t *n_points)
{
    SJ_API_BEGIN
    if (!r) sj::fail(SJ_ERR_STATE, "result is NULL");
    if (n_points) *n_points = r->n_points;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_dbscan(const sj_result *r, uint32_t min_pts, int32_t *labels, uint64_t *n_clusters, uint64_t *n_core,
                    uint64_t *n_noise)
{
    SJ_API_BEGIN
    sj::dbscan_impl(r, min_pts, labels, n_clusters, n_core, n_noise);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_to_csr(const sj_result *r, uint64_t n_points, uint64_t *row_offsets, uint32_t *neighbors)
{
    SJ_API_BEGIN
    sj::result_to_csr_impl(r, n_points, row_offsets, neighbors);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_plan_shards(const sj_index *idx, uint32_t world, uint64_t *cuts)
{
    SJ_API_BEGIN
    sj::plan_shards_impl(idx, world, cuts);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_result_fingerprint(const sj_result *r, uint64_t fp[2], uint32_t *counts)
{
    SJ_API_BEGIN
    sj::result_fingerprint_impl(r, fp, counts);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_neighbor_counts(const sj_index *idx, const sj_join_opts *opts, uint32_t *cnt, uint64_t *total)
{
    SJ_API_BEGIN
    if (!idx) sj::fail(SJ_ERR_STATE, "index is NULL");
    sj_join_opts o;
    if (opts) o = *opts;
    else sj_join_opts_default(&o);
    sj::neighbor_counts_impl(idx, o, cnt, total);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_brute_force_join(const double *points, uint64_t n, int d, double eps, const sj_build_opts *bopts,
                              const sj_join_opts *jopts, sj_result **out)
{
    SJ_API_BEGIN
    if (!out) sj::fail(SJ_ERR_ARG, "out is NULL");
    sj_build_opts bo;
    if (bopts) bo = *bopts;
    else sj_build_opts_default(&bo);
    sj_join_opts jo;
    if (jopts) jo = *jopts;
    else sj_join_opts_default(&jo);
    *out = sj::brute_force_impl(points, n, d, eps, bo, jo);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_join_sets(const sj_index *idx, const double *queries, uint64_t nq, int queries_on_device,
                       const sj_join_opts *opts, sj_result **out)
{
    SJ_API_BEGIN
    if (!out) sj::fail(SJ_ERR_ARG, "out is NULL");
    sj_join_opts jo;
    if (opts) jo = *opts;
    else sj_join_opts_default(&jo);
    *out = sj::join_sets_impl(idx, queries, nq, queries_on_device, jo);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_self_join_f32(const float *points, uint64_t n, int d, float eps, const sj_build_opts *bopts,
                           const sj_join_opts *jopts, sj_result **out)
{
    SJ_API_BEGIN
    if (!out) sj::fail(SJ_ERR_ARG, "out is NULL");
    sj_build_opts bo;
    if (bopts) bo = *bopts;
    else sj_build_opts_default(&bo);
    sj_join_opts jo;
    if (jopts) jo = *jopts;
    else sj_join_opts_default(&jo);
    *out = sj::self_join_f32_impl(points, n, d, eps, bo, jo);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_knn_join(const double *points, uint64_t n, const double *queries, uint64_t nq, int d, uint32_t k,
                      double eps0, const sj_build_opts *bopts, uint32_t *ids, double *dist2, sj_knn_stats *stats)
{
    SJ_API_BEGIN
    if (nq && !queries) sj::fail(SJ_ERR_ARG, "queries is NULL");
    sj_build_opts bo;
    if (bopts) bo = *bopts;
    else sj_build_opts_default(&bo);
    sj_knn_stats st{};
    static const double kNoQueries = 0.0;       // nq == 0: a non-NULL marker for the two-set form
    sj::knn_impl(points, n, nq ? queries : &kNoQueries, nq, d, k, eps0, bo, ids, dist2, &st);
    if (stats) *stats = st;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_knn_self(const double *points, uint64_t n, int d, uint32_t k, double eps0, const sj_build_opts *bopts,
                      uint32_t *ids, double *dist2, sj_knn_stats *stats)
{
    SJ_API_BEGIN
    sj_build_opts bo;
    if (bopts) bo = *bopts;
    else sj_build_opts_default(&bo);
    sj_knn_stats st{};
    sj::knn_self_impl(points, n, d, k, eps0, bo, ids, dist2, &st);
    if (stats) *stats = st;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_index_timings(const sj_index *idx, sj_index_view *view)
{
    SJ_API_BEGIN
    if (!idx) sj::fail(SJ_ERR_STATE, "index is NULL");
    if (!view) sj::fail(SJ_ERR_ARG, "view is NULL");
    sj::index_finalize_timing(const_cast<sj_index *>(idx));
    *view = idx->view;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_index_export(const sj_index *idx, sj_index_view *view)
{
    SJ_API_BEGIN
    if (!idx) sj::fail(SJ_ERR_STATE, "index is NULL");
    if (!view) sj::fail(SJ_ERR_ARG, "view is NULL");
    *view = idx->view;
    return SJ_OK;
    SJ_API_END
}

sj_status sj_index_import(const sj_index_view *view, int device, sj_index **out)
{
    SJ_API_BEGIN
    if (!view || !out) sj::fail(SJ_ERR_ARG, "NULL argument");
    *out = sj::import_index_impl(*view, device, false);
    return SJ_OK;
    SJ_API_END
}

sj_status sj_index_import_borrowed(const sj_index_view *view, int device, sj_index **out)
{
    SJ_API_BEGIN
    if (!view || !out) sj::fail(SJ_ERR_ARG, "NULL argument");
    *out = sj::import_index_impl(*view, device, true);
    return SJ_OK;
    SJ_API_END
}

void sj_set_allocator(void *(*alloc)(size_t, int, void *, void *), void (*release)(void *, void *), void *ctx)
{
    std::lock_guard<std::mutex> lk(sj::g_hook_mu);
    sj::g_hook.alloc = alloc;
    sj::g_hook.release = release;
    sj::g_hook.ctx = ctx;
}

sj_status sj_plan_batches(const uint32_t *sample_counts, uint64_t n_samples, uint64_t step, uint64_t q_begin,
                          uint64_t q_end, uint64_t capacity, int min_batches, double margin, uint64_t *cuts,
                          uint32_t max_cuts, uint32_t *k, uint64_t *estimated_total)
{
    SJ_API_BEGIN
    if ((!sample_counts && n_samples) || !cuts || !k) sj::fail(SJ_ERR_ARG, "NULL argument");
    if (q_end < q_begin || step == 0 || capacity == 0 || min_batches < 1 || margin < 0)
        sj::fail(SJ_ERR_ARG, "bad planner arguments");
    std::vector<uint64_t> c, e;
    uint64_t tot = 0;
    sj::plan_batches(sample_counts, n_samples, step, q_begin, q_end, capacity, min_batches, margin, c, e, &tot);
    if (c.size() > (size_t)max_cuts + 1) sj::fail(SJ_ERR_ARG, "cuts buffer too small");
    std::memcpy(cuts, c.data(), c.size() * sizeof(uint64_t));
    *k = (uint32_t)(c.size() - 1);
    if (estimated_total) *estimated_total = tot;
    return SJ_OK;
    SJ_API_END
}

}  // extern "C"
