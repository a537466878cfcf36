// context.cu -- per-device execution contexts reused across calls (streams, timing events,
// counter / cursor slots in device + pinned memory), so a build or a join does not create and
// destroy CUDA objects on every call.  A context is owned by one call at a time (pool + mutex);
// concurrent calls on one device simply get different contexts.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "sj_common.cuh"

namespace sj {

namespace {
std::mutex g_ctx_mu;
std::vector<DevCtx *> g_ctx_free;
}  // namespace

static void ensure(DevCtx *c, int nstreams, int nevents, size_t slot_bytes)
{
    while ((int)c->streams.size() < nstreams) {
        cudaStream_t s;
        SJ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        c->streams.push_back(s);
    }
    while ((int)c->events.size() < nevents) {
        cudaEvent_t e;
        SJ_CUDA(cudaEventCreate(&e));
        c->events.push_back(e);
    }
    if (slot_bytes > c->slot_bytes) {
        if (c->d_slots) cudaFree(c->d_slots);
        if (c->h_slots) cudaFreeHost(c->h_slots);
        c->d_slots = nullptr;
        c->h_slots = nullptr;
        c->slot_bytes = 0;
        size_t b = 4096;
        while (b < slot_bytes) b <<= 1;
        SJ_CUDA(cudaMalloc(&c->d_slots, b));
        SJ_CUDA(cudaMemset(c->d_slots, 0, b));       // (the build's last-CTA counter starts at 0)
        SJ_CUDA(cudaHostAlloc(&c->h_slots, b, cudaHostAllocPortable | cudaHostAllocMapped));
        c->slot_bytes = b;
    }
}

void ensure_join_blocks(DevCtx *c, size_t bytes)
{
    if (bytes <= c->jb_bytes) return;
    if (c->jb_d) cudaFree(c->jb_d);
    if (c->jb_h) cudaFreeHost(c->jb_h);
    c->jb_d = c->jb_h = nullptr;
    c->jb_bytes = 0;
    c->jb_clean = false;
    size_t b = 4096;
    while (b < bytes) b <<= 1;
    SJ_CUDA(cudaMalloc(&c->jb_d, b));
    SJ_CUDA(cudaMemset(c->jb_d, 0, b));               // (the publish CTA counters start at 0)
    SJ_CUDA(cudaHostAlloc(&c->jb_h, b, cudaHostAllocPortable | cudaHostAllocMapped));
    SJ_CUDA(cudaHostGetDevicePointer(&c->jb_hd, c->jb_h, 0));
    std::memset(c->jb_h, 0, b);
    c->jb_bytes = b;
}

namespace {
__global__ void __launch_bounds__(256) k_publish(const Publish p)
{
    if (p.masks_flag) {                           // masks M_j trivial? (the build's estimate only)
        __shared__ int s_bad;
        if (threadIdx.x == 0) s_bad = 0;
        __syncthreads();
        for (int j = 0; j < p.d; ++j)
            for (uint64_t b = p.mask_lo[j] + threadIdx.x; b <= p.mask_hi[j]; b += blockDim.x)
                if (!((__ldcg(p.masks + (b >> 5)) >> (b & 31)) & 1u)) s_bad = 1;
        __syncthreads();
        if (threadIdx.x == 0) *p.masks_flag = s_bad ? 0u : 1u;
        __syncthreads();
    }
    if (p.reduce_slots) {
        // work counters: 4 sums over reduce_slots slots of 4 words, then the cursor slots
        __shared__ unsigned long long s_sum[4][8];
        unsigned long long a[4] = {0, 0, 0, 0};
        for (uint32_t sl = threadIdx.x; sl < p.reduce_slots; sl += blockDim.x)
            for (int c = 0; c < 4; ++c) a[c] += __ldcg(p.src + 4 * sl + c);
        for (int c = 0; c < 4; ++c) {
            for (int o = 16; o; o >>= 1) a[c] += __shfl_xor_sync(0xffffffffu, a[c], o);
            if ((threadIdx.x & 31) == 0) s_sum[c][threadIdx.x >> 5] = a[c];
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            unsigned long long t = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_sum[threadIdx.x][w];
            p.dst[threadIdx.x] = t;
        }
        const unsigned long long *slots = p.src + 4 * p.reduce_slots;
        for (uint32_t i = threadIdx.x; i < 2 * p.nslots; i += blockDim.x) p.dst[4 + i] = __ldcg(slots + i);
        __syncthreads();
        if (p.zero_src)
            for (uint32_t i = threadIdx.x; i < p.words; i += blockDim.x) p.src[i] = 0ull;
    } else {
        for (uint32_t i = threadIdx.x; i < p.words; i += blockDim.x) {
            p.dst[i] = __ldcg(p.src + i);
            if (p.zero_src) p.src[i] = 0ull;
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) *p.bell = p.epoch;
}
}  // namespace

void launch_publish(const Publish &p, cudaStream_t s)
{
    k_publish<<<1, 256, 0, s>>>(p);
    SJ_LAUNCHED();
}

bool wait_doorbell(const volatile unsigned int *bell, unsigned int epoch, cudaStream_t s)
{
    uint64_t spins = 0;
    while (*bell != epoch) {
        if ((++spins & 255u) == 0) {
            const cudaError_t e = cudaStreamQuery(s);
            if (e == cudaSuccess) return *bell == epoch;
            if (e != cudaErrorNotReady) SJ_CUDA(e);
        }
    }
    return true;
}

DevCtx *acquire_ctx(int dev, int nstreams, int nevents, size_t slot_bytes)
{
    DevCtx *c = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_ctx_mu);
        for (size_t i = 0; i < g_ctx_free.size(); ++i) {
            if (g_ctx_free[i]->dev == dev) {
                c = g_ctx_free[i];
                g_ctx_free.erase(g_ctx_free.begin() + (long)i);
                break;
            }
        }
    }
    if (!c) {
        c = new DevCtx();
        c->dev = dev;
    }
    try {
        ensure(c, nstreams, nevents, slot_bytes);
    } catch (...) {
        release_ctx(c);
        throw;
    }
    return c;
}

void release_ctx(DevCtx *c)
{
    if (!c) return;
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    g_ctx_free.push_back(c);
}

namespace {
std::mutex g_ev_mu;
std::vector<std::pair<int, cudaEvent_t>> g_ev_free;
}  // namespace

cudaEvent_t event_get(int dev)
{
    {
        std::lock_guard<std::mutex> lk(g_ev_mu);
        for (size_t i = g_ev_free.size(); i-- > 0;) {
            if (g_ev_free[i].first == dev) {
                cudaEvent_t e = g_ev_free[i].second;
                g_ev_free.erase(g_ev_free.begin() + (long)i);
                return e;
            }
        }
    }
    cudaEvent_t e;
    SJ_CUDA(cudaEventCreate(&e));
    return e;
}

void event_put(int dev, cudaEvent_t e)
{
    if (!e) return;
    std::lock_guard<std::mutex> lk(g_ev_mu);
    g_ev_free.emplace_back(dev, e);
}

// One grow-only scratch buffer per device for the index build's N-sized temporaries (keys, sort
// buffers, prefix histogram): the stream-ordered pool re-maps memory when a previous join freed
// gigabytes of result batches on another stream (measured 0.36 ms per build on 2-D eps=1).  A build
// holds it from allocation to its final stream sync; a concurrent build falls back to the pool.
namespace {
struct ScratchSlot { void *p = nullptr; size_t bytes = 0; bool busy = false; size_t zero = 0; };
std::mutex g_scr_mu;
std::map<int, ScratchSlot> g_scr;
}  // namespace

// Device-resident result batches: a bounded per-device cache of freed batch buffers.  Joins with
// results of tens of GB otherwise had the stream-ordered pool map fresh memory again (C4 2-D
// eps=0.02: joins of 0.08 vs 0.8 s).  Each cached buffer carries an event recorded on the stream
// that freed it; the next owner's stream waits on it, so a buffer still read by the previous owner's
// pending work (e.g. an async torch op on a zero-copy batch view) is never overwritten early.
// Holds at most the limit (default 48 GB, env SJ_RESULT_CACHE_BYTES, sj_set_result_cache_limit);
// sj_trim() empties it.  The allocator hook bypasses it.
namespace {
struct CachedBuf { void *p; cudaEvent_t ev; };
std::mutex g_rc_mu;
std::map<int, std::multimap<size_t, CachedBuf>> g_rc;    // device -> (bytes -> buffer)
std::map<void *, size_t> g_rc_size;                      // buffer -> bytes (cached or handed out)
std::map<int, size_t> g_rc_held;
size_t g_rc_limit = [] {
    const char *e = std::getenv("SJ_RESULT_CACHE_BYTES");
    return (e && *e) ? (size_t)std::strtoull(e, nullptr, 10) : (size_t)(48ull << 30);
}();
}  // namespace

void set_result_cache_limit(size_t bytes)
{
    {
        std::lock_guard<std::mutex> lk(g_rc_mu);
        g_rc_limit = bytes;
    }
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
        std::vector<CachedBuf> drop;
        {
            std::lock_guard<std::mutex> lk(g_rc_mu);
            for (auto &kv : g_rc) {
                auto &m = kv.second;
                while (g_rc_held[kv.first] > g_rc_limit && !m.empty()) {
                    auto it = std::prev(m.end());          // largest first
                    g_rc_held[kv.first] -= it->first;
                    g_rc_size.erase(it->second.p);
                    drop.push_back(it->second);
                    m.erase(it);
                }
            }
        }
        for (auto &c : drop) {
            cudaEventSynchronize(c.ev);
            cudaFree(c.p);
            cudaEventDestroy(c.ev);
        }
    } else {
        cudaGetLastError();
    }
}

void *result_buffer_get(int dev, size_t bytes, cudaStream_t s)
{
    if (alloc_hook_set()) return dev_alloc(bytes, s);
    {
        std::lock_guard<std::mutex> lk(g_rc_mu);
        auto &m = g_rc[dev];
        auto it = m.lower_bound(bytes);
        if (it != m.end() && it->first <= 2 * bytes + (64u << 20)) {
            const CachedBuf c = it->second;
            g_rc_held[dev] -= it->first;
            m.erase(it);
            SJ_CUDA(cudaStreamWaitEvent(s, c.ev, 0));       // the previous owner's reads are done
            event_put(dev, c.ev);
            return c.p;
        }
    }
    void *p = dev_alloc(bytes, s);
    std::lock_guard<std::mutex> lk(g_rc_mu);
    g_rc_size[p] = bytes;
    return p;
}

void result_buffer_put(int dev, void *p, cudaStream_t s)
{
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_rc_mu);
        auto it = g_rc_size.find(p);
        if (it != g_rc_size.end() && g_rc_held[dev] + it->second <= g_rc_limit) {
            cudaEvent_t ev = event_get(dev);
            if (cudaEventRecord(ev, s ? s : cudaStreamLegacy) == cudaSuccess) {
                g_rc[dev].emplace(it->second, CachedBuf{p, ev});
                g_rc_held[dev] += it->second;
                return;
            }
            cudaGetLastError();
            event_put(dev, ev);
        }
        if (it != g_rc_size.end()) g_rc_size.erase(it);
    }
    dev_free(p, s ? s : cudaStreamLegacy);
}

void result_cache_trim(int dev)
{
    std::vector<CachedBuf> drop;
    {
        std::lock_guard<std::mutex> lk(g_rc_mu);
        for (auto &kv : g_rc) {
            if (dev >= 0 && kv.first != dev) continue;
            for (auto &e : kv.second) {
                g_rc_size.erase(e.second.p);
                drop.push_back(e.second);
            }
            kv.second.clear();
            g_rc_held[kv.first] = 0;
        }
    }
    for (auto &c : drop) {
        cudaEventSynchronize(c.ev);
        cudaFree(c.p);             // pool memory: cudaFree of a cudaMallocAsync block is synchronous and valid
        cudaEventDestroy(c.ev);
    }
}

int device_count()
{
    static const int n = [] {
        int c = 0;
        if (cudaGetDeviceCount(&c) != cudaSuccess) {
            cudaGetLastError();
            c = 0;
        }
        return c;
    }();
    return n;
}

int device_sm_count(int dev)
{
    static std::mutex mu;
    static std::map<int, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int nsm = 148;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
        cudaGetLastError();
        nsm = 148;
    }
    cache[dev] = nsm;
    return nsm;
}

// L2 set-aside for persisting accesses (per device, once): the build marks its input points as
// persisting while its three passes over them run (min/max, keys, the random row gather), then
// demotes them (l2_persist_end).  The set-aside is usable by normal accesses while no persisting
// lines occupy it.  SJ_L2_PERSIST=0 turns this off.  Returns the window size usable (0 = off).
size_t l2_persist_limit(int dev)
{
    static std::mutex mu;
    static std::map<int, size_t> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    size_t lim = 0;
    const char *e = std::getenv("SJ_L2_PERSIST");
    const bool on = e && *e && *e != '0';        // off by default: measured slower (below)
    int maxp = 0, maxw = 0;
    if (on && cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev) == cudaSuccess && maxp > 0 &&
        maxw > 0) {
        int cur = -1;
        cudaGetDevice(&cur);
        cudaSetDevice(dev);
        if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp) == cudaSuccess)
            lim = std::min<size_t>((size_t)maxp, (size_t)maxw);
        if (cur >= 0) cudaSetDevice(cur);
    }
    cudaGetLastError();
    cache[dev] = lim;
    return lim;
}

void l2_persist_begin(int dev, cudaStream_t s, const void *base, size_t bytes)
{
    const size_t lim = l2_persist_limit(dev);
    if (!lim || !bytes) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.base_ptr = const_cast<void *>(base);
    a.accessPolicyWindow.num_bytes = std::min(bytes, lim);
    a.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)lim / (double)a.accessPolicyWindow.num_bytes));
    a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess) cudaGetLastError();
}

// stop marking (kernels launched on s after this call) ...
void l2_persist_stop(int dev, cudaStream_t s)
{
    if (!l2_persist_limit(dev)) return;
    cudaStreamAttrValue a{};
    a.accessPolicyWindow.num_bytes = 0;
    if (cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a) != cudaSuccess) cudaGetLastError();
}

// ... and, once those kernels have completed (after a sync), demote the persisting lines
void l2_persist_end(int dev)
{
    if (!l2_persist_limit(dev)) return;
    if (cudaCtxResetPersistingL2Cache() != cudaSuccess) cudaGetLastError();
}

void *scratch_acquire(int dev, size_t bytes, size_t *zero_prefix)
{
    *zero_prefix = 0;
    if (alloc_hook_set()) return nullptr;      // scratch goes through the hook (dev_alloc) too
    std::lock_guard<std::mutex> lk(g_scr_mu);
    ScratchSlot &sl = g_scr[dev];
    if (sl.busy) return nullptr;
    if (sl.bytes < bytes) {
        if (sl.p) cudaFree(sl.p);
        sl.p = nullptr;
        sl.bytes = 0;
        sl.zero = 0;
        const size_t b = bytes + bytes / 4;
        if (cudaMalloc(&sl.p, b) != cudaSuccess) {
            cudaGetLastError();
            sl.p = nullptr;
            return nullptr;
        }
        sl.bytes = b;
    }
    sl.busy = true;
    *zero_prefix = sl.zero;
    sl.zero = 0;                               // unknown while the build runs
    return sl.p;
}

void scratch_release(int dev, void *p, size_t zero_prefix)
{
    std::lock_guard<std::mutex> lk(g_scr_mu);
    ScratchSlot &sl = g_scr[dev];
    if (sl.p == p) {
        sl.busy = false;
        sl.zero = zero_prefix;
    }
}

namespace {
std::mutex g_zb_mu;
std::map<int, std::multimap<size_t, void *>> g_zb;     // device -> (bytes -> zeroed buffer)
std::map<int, size_t> g_zb_held;
constexpr size_t kZbLimit = 1ull << 30;                  // per device
}  // namespace

void *zbuf_get(int dev, size_t bytes, size_t *granted)
{
    if (alloc_hook_set()) return nullptr;
    std::lock_guard<std::mutex> lk(g_zb_mu);
    auto &m = g_zb[dev];
    auto it = m.lower_bound(bytes);
    if (it == m.end() || it->first > 2 * bytes + (1u << 20)) return nullptr;
    void *p = it->second;
    *granted = it->first;
    g_zb_held[dev] -= it->first;
    m.erase(it);
    return p;
}

void zbuf_put(int dev, void *p, size_t bytes)
{
    if (!p) return;
    {
        std::lock_guard<std::mutex> lk(g_zb_mu);
        if (g_zb_held[dev] + bytes <= kZbLimit && cudaMemset(p, 0, bytes) == cudaSuccess) {
            g_zb[dev].emplace(bytes, p);
            g_zb_held[dev] += bytes;
            return;
        }
    }
    cudaGetLastError();
    cudaFree(p);
}

void zbuf_trim(int dev)
{
    std::lock_guard<std::mutex> lk(g_zb_mu);
    for (auto &kv : g_zb) {
        if (dev >= 0 && kv.first != dev) continue;
        for (auto &e : kv.second) cudaFree(e.second);
        kv.second.clear();
        g_zb_held[kv.first] = 0;
    }
}

void scratch_trim(int dev)
{
    std::lock_guard<std::mutex> lk(g_scr_mu);
    for (auto &kv : g_scr) {
        if (dev >= 0 && kv.first != dev) continue;
        ScratchSlot &sl = kv.second;
        if (sl.busy || !sl.p) continue;
        cudaFree(sl.p);
        sl.p = nullptr;
        sl.bytes = 0;
    }
}

void set_max_dyn_smem(const void *func, int bytes)
{
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> done;   // (kernel, device) -> bytes set
    int dev = 0;
    SJ_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto &b = done[{func, dev}];
    if (b >= bytes) return;
    SJ_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    // the largest shared-memory carve-out: the occupancy the launch bounds ask for needs it (the
    // default configuration left k_refine_dense at 2 CTAs per SM)
    SJ_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    b = bytes;
}

static float elapsed(cudaEvent_t a, cudaEvent_t b)
{
    float t = 0;
    if (a && b && cudaEventElapsedTime(&t, a, b) != cudaSuccess) {
        cudaGetLastError();
        t = 0;
    }
    return t;
}

void result_finalize_timing(sj_result *r)
{
    if (r->timed) return;
    cudaSetDevice(r->device);
    r->stats.estimate_ms = elapsed(r->est_ev[0], r->est_ev[1]);
    float sum = 0, mx = 0, span = 0;
    for (auto &pr : r->runs) {
        cudaEventSynchronize(pr.second);
        const float ms = elapsed(pr.first, pr.second);
        sum += ms;
        mx = std::max(mx, ms);
        span = std::max(span, elapsed(r->span0, pr.second));
    }
    r->stats.refine_ms = sum;
    r->stats.refine_max_ms = mx;
    r->stats.refine_span_ms = span;
    r->timed = true;
    result_release_events(r);
}

void result_release_events(sj_result *r)
{
    for (auto &pr : r->runs) {
        event_put(r->device, pr.first);
        event_put(r->device, pr.second);
    }
    r->runs.clear();
    event_put(r->device, r->est_ev[0]);
    event_put(r->device, r->est_ev[1]);
    event_put(r->device, r->span0);
    r->est_ev[0] = r->est_ev[1] = r->span0 = nullptr;
}

void index_finalize_timing(sj_index *idx)
{
    if (idx->timed || !idx->tev[0]) return;
    cudaSetDevice(idx->device);
    cudaEventSynchronize(idx->tev[6]);
    sj_index_view &v = idx->view;
    v.t_h2d_ms = elapsed(idx->tev[0], idx->tev[1]);
    v.t_geometry_ms = elapsed(idx->tev[1], idx->tev[2]);
    v.t_keys_ms = elapsed(idx->tev[2], idx->tev[3]);
    v.t_sort_ms = elapsed(idx->tev[3], idx->tev[4]);
    v.t_compact_ms = elapsed(idx->tev[4], idx->tev[6]);
    v.t_total_ms = elapsed(idx->tev[0], idx->tev[6]);
    idx->timed = true;
    for (auto &e : idx->tev) {
        event_put(idx->device, e);
        e = nullptr;
    }
}

static double now_us()
{
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static int trace_level()
{
    static const int lvl = [] { const char *e = std::getenv("SJ_TRACE"); return (e && *e) ? std::atoi(e) : 0; }();
    return lvl;
}

namespace {
struct TraceEntry {
    const char *what, *stage;
    double host_us;
    cudaEvent_t ev;
};
std::mutex g_tr_mu;
std::vector<TraceEntry> g_tr;
double g_tr_h0 = 0;
cudaEvent_t g_tr_e0 = nullptr;
int g_tr_dev = 0;

void trace_dump()
{
    std::vector<TraceEntry> v;
    cudaEvent_t e0;
    double h0;
    {
        std::lock_guard<std::mutex> lk(g_tr_mu);
        v.swap(g_tr);
        e0 = g_tr_e0;
        h0 = g_tr_h0;
        g_tr_e0 = nullptr;
    }
    if (v.empty()) return;
    for (auto &e : v)
        if (e.ev) cudaEventSynchronize(e.ev);
    std::fprintf(stderr, "[sj-timeline] %-7s %-34s %10s %10s\n", "", "stage", "host us", "gpu us");
    for (auto &e : v) {
        float ms = 0;
        if (e.ev && e0) cudaEventElapsedTime(&ms, e0, e.ev);
        if (e.ev)
            std::fprintf(stderr, "[sj-timeline] %-7s %-34s %10.1f %10.1f\n", e.what, e.stage, e.host_us - h0,
                         1000.0 * ms);
        else
            std::fprintf(stderr, "[sj-timeline] %-7s %-34s %10.1f %10s\n", e.what, e.stage, e.host_us - h0, "");
    }
    for (auto &e : v)
        if (e.ev) event_put(g_tr_dev, e.ev);
}
}  // namespace

HostTrace::HostTrace(const char *w) : what(w)
{
    on = trace_level() > 0;
    t0 = last = on ? now_us() : 0.0;
    if (trace_level() >= 2 && std::strcmp(w, "build") == 0) {
        std::lock_guard<std::mutex> lk(g_tr_mu);
        for (auto &e : g_tr)
            if (e.ev) event_put(g_tr_dev, e.ev);
        g_tr.clear();
        g_tr_e0 = nullptr;
    }
}

void HostTrace::dev(const char *stage, cudaStream_t s)
{
    if (trace_level() < 2) return;
    int d = 0;
    cudaGetDevice(&d);
    cudaEvent_t e = event_get(d);       // pooled: recording costs ~1 us of host time, no creation
    const double h = now_us();
    cudaEventRecord(e, s);
    std::lock_guard<std::mutex> lk(g_tr_mu);
    if (!g_tr_e0) {
        g_tr_e0 = e;
        g_tr_h0 = h;
        g_tr_dev = d;
    }
    g_tr.push_back({what, stage, h, e});
}

HostTrace::~HostTrace()
{
    if (trace_level() >= 2 && std::strcmp(what, "join") == 0) trace_dump();
}

void HostTrace::mark(const char *stage)
{
    if (!on) return;
    const double t = now_us();
    if (trace_level() >= 2) {
        std::lock_guard<std::mutex> lk(g_tr_mu);
        if (g_tr_e0) g_tr.push_back({what, stage, t, nullptr});
    } else {
        std::fprintf(stderr, "[sj-trace] %-10s %-28s +%8.1f us  (t=%8.1f us)\n", what, stage, t - last, t - t0);
    }
    last = t;
}

}  // namespace sj
