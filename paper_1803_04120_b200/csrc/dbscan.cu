// dbscan.cu -- SURVEY §8(f) rank 4: DBSCAN read off the epsilon self-join ("the DBSCAN
// clustering algorithm requires range queries that search the neighborhood of all data points").
// The join's pairs ARE the epsilon-neighbourhood table N_eps(p) = {q : (p, q) in S}; on it
// (Ester et al. 1996, reading R17 of DESIGN.md for the choices the definition leaves open):
//   core(p)  <=> |N_eps(p)| >= min_pts (p counts itself);
//   clusters  = connected components of the core points under (p, q) in S, labelled by their
//               smallest core id;
//   border p  = non-core with a core neighbour: the smallest label among its core neighbours;
//   noise     = -1.
// Device passes over the result's batches (device memory, or pinned host memory through its UVA
// mapping): neighbour counts (warp-aggregated per key), lock-free union-find over the core-core
// pairs (each unordered pair once: p < q; the larger root is hooked under the smaller with one
// atomicCAS, path halving in find), one flattening pass, then the border labels (atomicMin).
#include <algorithm>

#include "sj_common.cuh"

namespace sj {

namespace {

__global__ void __launch_bounds__(256)
k_db_count(const uint64_t *__restrict__ pairs, uint64_t n, uint32_t *__restrict__ cnt)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const uint64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        const uint32_t key = ok ? (uint32_t)(pairs[i] >> 32) : 0xffffffffu;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        if (ok && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) atomicAdd(cnt + key, (uint32_t)__popc(grp));
    }
}

__global__ void __launch_bounds__(256)
k_db_init(const uint32_t *__restrict__ cnt, uint32_t n, uint32_t min_pts, uint32_t self_extra,
          uint32_t *__restrict__ parent, int32_t *__restrict__ border)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    parent[i] = (cnt[i] + self_extra >= min_pts) ? i : 0xffffffffu;    // 0xffffffff: not core
    border[i] = 0x7fffffff;
}

// parent[] is read through L2 (__ldcg: other SMs hook roots concurrently; the atomicCAS is the
// authority, a stale read only costs a retry)
__device__ __forceinline__ uint32_t db_find(uint32_t *parent, uint32_t x)
{
    uint32_t p = __ldcg(parent + x);
    while (p != x) {
        const uint32_t g = __ldcg(parent + p);
        if (g != p) parent[x] = g;                    // path halving (benign race: g is an ancestor)
        x = p;
        p = __ldcg(parent + x);
    }
    return x;
}

__global__ void __launch_bounds__(256)
k_db_union(const uint64_t *__restrict__ pairs, uint64_t n, uint32_t *parent)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t x = pairs[i];
        const uint32_t a = (uint32_t)(x >> 32), b = (uint32_t)x;
        if (a >= b) continue;                                  // each unordered pair once
        if (__ldcg(parent + a) == 0xffffffffu || __ldcg(parent + b) == 0xffffffffu) continue;   // both core
        uint32_t ra = db_find(parent, a), rb = db_find(parent, b);
        while (ra != rb) {
            if (ra < rb) { const uint32_t t = ra; ra = rb; rb = t; }   // hook the larger root
            const uint32_t old = atomicCAS(parent + ra, ra, rb);
            if (old == ra) break;
            ra = db_find(parent, old);
            rb = db_find(parent, rb);
        }
    }
}

// Every core point's entry becomes its root.  The walk is read-only: the only write to parent[i]
// is thread i's own (a path-halving write by another thread could store a non-root ancestor over
// it after thread i wrote the root).
__global__ void __launch_bounds__(256)
k_db_flatten(uint32_t *parent, uint32_t n)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t x = __ldcg(parent + i);
    if (x == 0xffffffffu) return;
    uint32_t p = __ldcg(parent + x);
    while (p != x) {
        x = p;
        p = __ldcg(parent + x);
    }
    parent[i] = x;
}

__global__ void __launch_bounds__(256)
k_db_border(const uint64_t *__restrict__ pairs, uint64_t n, const uint32_t *__restrict__ parent,
            int32_t *__restrict__ border)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint64_t x = pairs[i];
        const uint32_t a = (uint32_t)(x >> 32), b = (uint32_t)x;
        if (parent[a] != 0xffffffffu) continue;                // a is core: not a border candidate
        const uint32_t lb = parent[b];
        if (lb != 0xffffffffu) atomicMin(border + a, (int32_t)lb);
    }
}

// labels, and the counts of clusters (roots), core points and noise points
__global__ void __launch_bounds__(256)
k_db_label(const uint32_t *__restrict__ parent, const int32_t *__restrict__ border, uint32_t n,
           int32_t *__restrict__ labels, unsigned long long *__restrict__ tally)
{
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t root = 0, core = 0, noise = 0;
    if (i < n) {
        const uint32_t p = parent[i];
        if (p != 0xffffffffu) {
            labels[i] = (int32_t)p;
            core = 1;
            root = p == i;
        } else {
            const int32_t b = border[i];
            labels[i] = b == 0x7fffffff ? -1 : b;
            noise = b == 0x7fffffff;
        }
    }
    root = __reduce_add_sync(0xffffffffu, root);
    core = __reduce_add_sync(0xffffffffu, core);
    noise = __reduce_add_sync(0xffffffffu, noise);
    if ((threadIdx.x & 31) == 0) {
        if (root) atomicAdd(tally + 0, root);
        if (core) atomicAdd(tally + 1, core);
        if (noise) atomicAdd(tally + 2, noise);
    }
}

}  // namespace

void dbscan_impl(const sj_result *r, uint32_t min_pts, int32_t *labels, uint64_t *n_clusters, uint64_t *n_core,
                 uint64_t *n_noise)
{
    if (!r) fail(SJ_ERR_STATE, "result is NULL");
    if (!labels) fail(SJ_ERR_ARG, "labels is NULL");
    if (min_pts < 1) fail(SJ_ERR_ARG, "min_pts must be >= 1");
    if (r->two_set) fail(SJ_ERR_ARG, "DBSCAN needs a self-join result, not a two-set join");
    if (r->q0 != 0 || r->q1 != r->n_points)
        fail(SJ_ERR_ARG, "DBSCAN needs the whole self-join (the result covers only a query range)");
    for (const auto &b : r->batches)
        if (b.csr) fail(SJ_ERR_STATE, "DBSCAN reads pair batches; this result was drained as CSR");
    const uint64_t n64 = r->n_points;
    if (n64 == 0 || n64 >= (1ull << 31)) fail(SJ_ERR_ARG, "DBSCAN labels are int32: N must be < 2^31");
    const uint32_t n = (uint32_t)n64;
    SJ_CUDA(cudaSetDevice(r->device));
    CtxGuard cg{acquire_ctx(r->device, 1, 0, 64)};
    cudaStream_t s = cg.c->streams[0];
    unsigned long long *dt = static_cast<unsigned long long *>(cg.c->d_slots);
    unsigned long long *ht = static_cast<unsigned long long *>(cg.c->h_slots);
    SJ_CUDA(cudaMemsetAsync(dt, 0, 3 * sizeof(unsigned long long), s));
    Scratch<uint32_t> cnt(n, s), parent(n, s);
    Scratch<int32_t> border(n, s);
    SJ_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(uint32_t) * n, s));
    const int nsm = device_sm_count(r->device);
    std::vector<const uint64_t *> src;
    for (const auto &b : r->batches) {
        if (!b.n) {
            src.push_back(nullptr);
            continue;
        }
        const uint64_t *p = b.pairs;
        if (!b.on_device) {
            void *dp = nullptr;
            SJ_CUDA(cudaHostGetDevicePointer(&dp, const_cast<uint64_t *>(b.pairs), 0));
            p = static_cast<const uint64_t *>(dp);
        }
        src.push_back(p);
    }
    auto grid_for = [&](uint64_t m) {
        return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((m + 255) / 256, (uint64_t)nsm * 16));
    };
    for (size_t i = 0; i < src.size(); ++i)
        if (src[i]) {
            k_db_count<<<grid_for(r->batches[i].n), 256, 0, s>>>(src[i], r->batches[i].n, cnt.p);
            SJ_LAUNCHED();
        }
    const unsigned gn = (n + 255) / 256;
    k_db_init<<<gn, 256, 0, s>>>(cnt.p, n, min_pts, r->include_self ? 0u : 1u, parent.p, border.p);
    SJ_LAUNCHED();
    for (size_t i = 0; i < src.size(); ++i)
        if (src[i]) {
            k_db_union<<<grid_for(r->batches[i].n), 256, 0, s>>>(src[i], r->batches[i].n, parent.p);
            SJ_LAUNCHED();
        }
    k_db_flatten<<<gn, 256, 0, s>>>(parent.p, n);
    SJ_LAUNCHED();
    for (size_t i = 0; i < src.size(); ++i)
        if (src[i]) {
            k_db_border<<<grid_for(r->batches[i].n), 256, 0, s>>>(src[i], r->batches[i].n, parent.p, border.p);
            SJ_LAUNCHED();
        }
    k_db_label<<<gn, 256, 0, s>>>(parent.p, border.p, n, labels, dt);
    SJ_LAUNCHED();
    SJ_CUDA(cudaMemcpyAsync(ht, dt, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    if (n_clusters) *n_clusters = ht[0];
    if (n_core) *n_core = ht[1];
    if (n_noise) *n_noise = ht[2];
}

}  // namespace sj
