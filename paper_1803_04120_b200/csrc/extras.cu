// extras.cu -- the SURVEY §8(f) "NEXT" rows built on the same primitives:
//   f2: on-device sort of a result batch by (key, value) ("After the kernel's
//       execution, we sort the key/value pairs, and transfer the result to the host").
//   f3: the GPU brute-force nested-loop join: every query compared with every
//       point, the paper's epsilon-independent control and a cross-check of the grid join.
#include <algorithm>

#include "sj_common.cuh"

namespace sj {

// ------------------------------------------------------------------ f2: batch sort
// Packed pairs (key << 32 | value) sort as plain uint64 (integer order == (key, value) order);
// only the bits below 32 + ceil(log2 N) are used.
void sort_pairs_device(uint64_t *pairs, uint64_t n, uint64_t n_points, cudaStream_t s)
{
    if (n <= 1) return;
    if (n >= (1ull << 32)) fail(SJ_ERR_ARG, "sort_pairs: a batch of >= 2^32 pairs cannot be sorted in one pass");
    int id_bits = 1;
    while (id_bits < 32 && (1ull << id_bits) < n_points) ++id_bits;
    Scratch<uint64_t> tmp(n, s);
    bool in_tmp = false;
    radix_sort_pairs(pairs, nullptr, tmp.p, nullptr, (uint32_t)n, 32 + id_bits, s, &in_tmp);
    if (in_tmp) SJ_CUDA(cudaMemcpyAsync(pairs, tmp.p, n * sizeof(uint64_t), cudaMemcpyDeviceToDevice, s));
}

// ------------------------------------------------------------------ f2: CSR neighbour lists
// The whole result as compressed rows: row_offsets[i] .. row_offsets[i+1] index the neighbours of
// point i (original ids) in `neighbors`, ascending -- 4 B per pair instead of 8 (SURVEY §8(f) rank
// 2).  All batches are gathered, sorted as packed uint64 (the radix sort above: integer order ==
// (key, value) order, so rows come out sorted), rows counted, scanned, values extracted.
namespace {
__global__ void k_csr_hist(const uint64_t *__restrict__ pairs, uint64_t n, uint32_t *__restrict__ counts)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(counts + (pairs[i] >> 32), 1u);
}

__global__ void k_csr_values(const uint64_t *__restrict__ pairs, uint64_t n, uint32_t *__restrict__ nbrs)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        nbrs[i] = (uint32_t)pairs[i];
}

__global__ void k_widen_u32(const uint32_t *__restrict__ in, uint64_t n, uint64_t *__restrict__ out)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}
}  // namespace

void result_to_csr_impl(const sj_result *r, uint64_t n_points, uint64_t *row_offsets, uint32_t *neighbors)
{
    if (!r) fail(SJ_ERR_STATE, "result is NULL");
    if (n_points == 0 || n_points >= (1ull << 32)) fail(SJ_ERR_ARG, "n_points must satisfy 1 <= n < 2^32");
    if (n_points < r->n_points) fail(SJ_ERR_ARG, "n_points is smaller than the N of the joined point set");
    if (!row_offsets || (!neighbors && r->total)) fail(SJ_ERR_ARG, "NULL output array");
    if (r->total >= (1ull << 32)) fail(SJ_ERR_ARG, "CSR of >= 2^32 pairs is not supported");
    SJ_CUDA(cudaSetDevice(r->device));
    CtxGuard cg{acquire_ctx(r->device, 1, 0, 64)};
    cudaStream_t s = cg.c->streams[0];
    const uint64_t n = r->total;
    const int nsm = device_sm_count(r->device);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)nsm * 8));
    for (const auto &b : r->batches)
        if (b.csr) fail(SJ_ERR_STATE, "the result's batches are already CSR (drain_csr): read them with sj_result_batch_csr");
    Scratch<uint64_t> all(n ? n : 1, s);
    uint64_t off = 0;
    for (const auto &b : r->batches) {
        if (!b.n) continue;
        SJ_CUDA(cudaMemcpyAsync(all.p + off, b.pairs, b.n * sizeof(uint64_t),
                                b.on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s));
        off += b.n;
    }
    sort_pairs_device(all.p, n, n_points, s);
    Scratch<uint32_t> counts(n_points + 1, s), offs(n_points + 1, s);
    SJ_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(uint32_t) * (n_points + 1), s));
    if (n) {
        k_csr_hist<<<grid, 256, 0, s>>>(all.p, n, counts.p);
        SJ_LAUNCHED();
    }
    exclusive_scan_u32(counts.p, offs.p, n_points + 1, s);
    const unsigned gridN =
        (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n_points + 256) / 256, (uint64_t)nsm * 8));
    k_widen_u32<<<gridN, 256, 0, s>>>(offs.p, n_points + 1, row_offsets);
    SJ_LAUNCHED();
    if (n) {
        k_csr_values<<<grid, 256, 0, s>>>(all.p, n, neighbors);
        SJ_LAUNCHED();
    }
    SJ_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ a8 + f2: CSR drain of a batch
// One finished batch (device pairs) -> CSR over all N keys in device memory: counts by key (one
// atomic per distinct key per warp: __match_any_sync groups a warp's equal keys -- a query's
// pairs sit together in the batch), exclusive scan, then every pair's value is placed at its row's
// running cursor (rows in arbitrary order), or -- for a batch sorted by (key, value) -- at its own
// index (rows ascending, no atomics).  The caller copies [offsets | neighbours] to the host.
namespace {
__global__ void __launch_bounds__(256)
k_drain_hist(const uint64_t *__restrict__ pairs, uint64_t n, uint32_t *__restrict__ counts)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {   // warp-uniform trips
        const uint64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        const uint32_t key = ok ? (uint32_t)(pairs[i] >> 32) : 0xffffffffu;
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        if (ok && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1)) atomicAdd(counts + key, (uint32_t)__popc(grp));
    }
}

__global__ void __launch_bounds__(256)
k_drain_scatter(const uint64_t *__restrict__ pairs, uint64_t n, uint32_t *__restrict__ cursor,
                uint32_t *__restrict__ nbrs)
{
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    const unsigned lane = threadIdx.x & 31;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const uint64_t i = i0 + threadIdx.x;
        const bool ok = i < n;
        const uint64_t x = ok ? pairs[i] : ~0ull;
        const uint32_t key = (uint32_t)(x >> 32);
        const unsigned grp = __match_any_sync(0xffffffffu, key);
        const int leader = __ffs(grp) - 1;
        uint32_t base = 0;
        if (ok && lane == (unsigned)leader) base = atomicAdd(cursor + key, (uint32_t)__popc(grp));
        base = __shfl_sync(0xffffffffu, base, leader);
        if (ok) nbrs[base + __popc(grp & ((1u << lane) - 1u))] = (uint32_t)x;
    }
}
}  // namespace

// pairs (device, n) -> dst_offs[rows + 1] and dst_nbrs[n] (device); counts / cursor: rows + 1 uint32
// scratch (device).  sorted: the batch is in (key, value) order.
void batch_to_csr_device(const uint64_t *pairs, uint64_t n, uint64_t rows, bool sorted, uint32_t *counts,
                         uint32_t *cursor, uint32_t *dst_offs, uint32_t *dst_nbrs, cudaStream_t s, int nsm)
{
    SJ_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * (rows + 1), s));
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, (uint64_t)nsm * 16));
    if (n) {
        k_drain_hist<<<grid, 256, 0, s>>>(pairs, n, counts);
        SJ_LAUNCHED();
    }
    exclusive_scan_u32_dup(counts, dst_offs, cursor, rows + 1, s);
    if (!n) return;
    if (sorted) {
        k_csr_values<<<grid, 256, 0, s>>>(pairs, n, dst_nbrs);
    } else {
        k_drain_scatter<<<grid, 256, 0, s>>>(pairs, n, cursor, dst_nbrs);
    }
    SJ_LAUNCHED();
}

// ------------------------------------------------------------------ result fingerprints
// Order-independent fingerprints of the pair multiset:
//   F_a = sum_x mix_a(x), F_b = sum_x mix_b(x) (mod 2^64), mix_a = SplitMix64 output function of
//   x + 0x9E3779B97F4A7C15, mix_b = MurmurHash3 fmix64 of x ^ 0xC2B2AE3D27D4EB4F;
// optionally the per-key counts cnt[x >> 32].  One pass over every batch (device memory, or pinned
// host memory read in place over PCIe through its UVA mapping).  The oracle computes the same
// fingerprints from its own join (oracle/sj_oracle.c orc_grid_digest), so results of tens of GB
// are compared without being held twice.
namespace {
__device__ __forceinline__ uint64_t fp_mix_a(uint64_t x)
{
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t fp_mix_b(uint64_t x)
{
    uint64_t k = x ^ 0xC2B2AE3D27D4EB4Full;
    k ^= k >> 33;
    k *= 0xFF51AFD7ED558CCDull;
    k ^= k >> 33;
    k *= 0xC4CEB9FE1A85EC53ull;
    k ^= k >> 33;
    return k;
}

__global__ void __launch_bounds__(256)
k_fingerprint(const uint64_t *__restrict__ pairs, uint64_t n, unsigned long long *__restrict__ acc,
              uint32_t *__restrict__ counts, uint64_t n_points, uint32_t *__restrict__ bad)
{
    uint64_t fa = 0, fb = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t x = pairs[i];
        fa += fp_mix_a(x);
        fb += fp_mix_b(x);
        if (counts) {
            const uint64_t key = x >> 32;
            if (key < n_points) atomicAdd(counts + key, 1u);
            else atomicOr(bad, 1u);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        fa += __shfl_xor_sync(0xffffffffu, fa, o);
        fb += __shfl_xor_sync(0xffffffffu, fb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc + 0, (unsigned long long)fa);       // wraps mod 2^64: the definition
        atomicAdd(acc + 1, (unsigned long long)fb);
    }
}

// the same fingerprints over a CSR batch (drain_csr): one thread per row, x = (row << 32) | neighbour
__global__ void __launch_bounds__(256)
k_fingerprint_csr(const uint32_t *__restrict__ offs, const uint32_t *__restrict__ nbrs, uint64_t rows,
                  unsigned long long *__restrict__ acc, uint32_t *__restrict__ counts, uint64_t n_points,
                  uint32_t *__restrict__ bad)
{
    uint64_t fa = 0, fb = 0;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t a = offs[i], b = offs[i + 1];
        for (uint32_t e = a; e < b; ++e) {
            const uint64_t x = (i << 32) | nbrs[e];
            fa += fp_mix_a(x);
            fb += fp_mix_b(x);
        }
        if (counts && b > a) {
            if (i < n_points) atomicAdd(counts + i, b - a);
            else atomicOr(bad, 1u);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        fa += __shfl_xor_sync(0xffffffffu, fa, o);
        fb += __shfl_xor_sync(0xffffffffu, fb, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc + 0, (unsigned long long)fa);
        atomicAdd(acc + 1, (unsigned long long)fb);
    }
}
}  // namespace

void result_fingerprint_impl(const sj_result *r, uint64_t *fp, uint32_t *counts)
{
    if (!r) fail(SJ_ERR_STATE, "result is NULL");
    if (!fp) fail(SJ_ERR_ARG, "fp is NULL");
    SJ_CUDA(cudaSetDevice(r->device));
    CtxGuard cg{acquire_ctx(r->device, 1, 0, 64)};
    cudaStream_t s = cg.c->streams[0];
    unsigned long long *dacc = static_cast<unsigned long long *>(cg.c->d_slots);
    unsigned long long *hacc = static_cast<unsigned long long *>(cg.c->h_slots);
    SJ_CUDA(cudaMemsetAsync(dacc, 0, 4 * sizeof(unsigned long long), s));
    if (counts) SJ_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * r->n_points, s));
    const int nsm = device_sm_count(r->device);
    uint32_t *bad = reinterpret_cast<uint32_t *>(dacc + 2);
    for (const auto &b : r->batches) {
        if (!b.n) continue;
        if (b.csr) {
            void *dp = nullptr;
            SJ_CUDA(cudaHostGetDevicePointer(&dp, const_cast<uint64_t *>(b.pairs), 0));
            const uint32_t *offs = static_cast<const uint32_t *>(dp);
            const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((b.rows + 255) / 256, (uint64_t)nsm * 8));
            k_fingerprint_csr<<<grid, 256, 0, s>>>(offs, offs + b.rows + 1, b.rows, dacc, counts, r->n_points, bad);
            SJ_LAUNCHED();
            continue;
        }
        const uint64_t *src = b.pairs;
        if (!b.on_device) {
            void *dp = nullptr;
            SJ_CUDA(cudaHostGetDevicePointer(&dp, const_cast<uint64_t *>(b.pairs), 0));
            src = static_cast<const uint64_t *>(dp);
        }
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((b.n + 255) / 256, (uint64_t)nsm * 8));
        k_fingerprint<<<grid, 256, 0, s>>>(src, b.n, dacc, counts, r->n_points, bad);
        SJ_LAUNCHED();
    }
    SJ_CUDA(cudaMemcpyAsync(hacc, dacc, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    if (hacc[2] & 0xffffffffull) fail(SJ_ERR_STATE, "a pair's key is >= the result's n_points (corrupt result)");
    fp[0] = hacc[0];
    fp[1] = hacc[1];
}

// ------------------------------------------------------------------ f3: brute force
namespace {
constexpr int kBfThreads = 256;
constexpr int kBfTile = 256;           // candidates staged per round (SoA in shared memory)
constexpr int kBfBuf = 512;            // per-warp output buffer (pairs)

template <int D>
__global__ void __launch_bounds__(kBfThreads)
k_brute_force(const double *__restrict__ pts, uint32_t n, double eps2, int include_self, uint64_t *out,
              unsigned long long *cursor, uint64_t cap, uint32_t *overflow)
{
    __shared__ double s_x[D][kBfTile];
    __shared__ uint64_t s_buf[kBfThreads / 32][kBfBuf];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t i = blockIdx.x * kBfThreads + threadIdx.x;
    const bool active = i < n;
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = active ? pts[(uint64_t)i * D + j] : 0.0;
    uint32_t cnt = 0;                  // warp-uniform fill of s_buf[warp]
    auto flush = [&]() {
        unsigned long long base = 0;
        if (lane == 0) base = atomicAdd(cursor, (unsigned long long)cnt);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (uint32_t e = lane; e < cnt; e += 32) {
            if (base + e < cap) out[base + e] = s_buf[warp][e];
            else atomicOr(overflow, 1u);
        }
        __syncwarp();
        cnt = 0;
    };
    for (uint32_t t0 = 0; t0 < n; t0 += kBfTile) {
        __syncthreads();
        for (int e = threadIdx.x; e < kBfTile; e += kBfThreads) {
            const uint32_t m = t0 + e;
#pragma unroll
            for (int j = 0; j < D; ++j) s_x[j][e] = m < n ? pts[(uint64_t)m * D + j] : 0.0;
        }
        __syncthreads();
        const uint32_t lim = min((uint32_t)kBfTile, n - t0);
        for (uint32_t e = 0; e < lim; ++e) {
            const uint32_t m = t0 + e;
            double s;
            {
                const double t = __dsub_rn(x[0], s_x[0][e]);
                s = __dmul_rn(t, t);
            }
#pragma unroll
            for (int j = 1; j < D; ++j) {
                const double t = __dsub_rn(x[j], s_x[j][e]);
                s = __dadd_rn(s, __dmul_rn(t, t));
            }
            const bool hit = active && s <= eps2 && (include_self || m != i);
            const unsigned hits = __ballot_sync(0xffffffffu, hit);
            if (!hits) continue;
            if (cnt + 32u > (uint32_t)kBfBuf) flush();
            if (hit) s_buf[warp][cnt + __popc(hits & ((1u << lane) - 1u))] = ((uint64_t)i << 32) | m;
            __syncwarp();
            cnt += __popc(hits);
        }
    }
    flush();
}

template <int D>
void launch_bf(uint32_t n, cudaStream_t s, const double *pts, double eps2, int inc, uint64_t *out,
               unsigned long long *cur, uint64_t cap, uint32_t *ovf)
{
    k_brute_force<D><<<(n + kBfThreads - 1) / kBfThreads, kBfThreads, 0, s>>>(pts, n, eps2, inc, out, cur, cap, ovf);
    SJ_LAUNCHED();
}
}  // namespace

sj_result *brute_force_impl(const double *points, uint64_t n, int d, double eps, const sj_build_opts &bo,
                            const sj_join_opts &jo)
{
    if (d < 2 || d > SJ_MAX_DIM) fail(SJ_ERR_DIM, "d must be in [2,6]");
    if (!points) fail(SJ_ERR_ARG, "points is NULL");
    if (n == 0 || n >= (1ull << 32)) fail(SJ_ERR_ARG, "N must satisfy 1 <= N < 2^32");
    if (!(eps > 0.0) || eps != eps || eps > 1e308) fail(SJ_ERR_ARG, "eps must be finite and > 0");
    SJ_CUDA(cudaSetDevice(bo.device));
    CtxGuard cg{acquire_ctx(bo.device, 1, 0, 64)};
    cudaStream_t s = cg.c->streams[0];
    const double *pts = points;
    Scratch<double> dp;
    if (!bo.points_on_device) {
        dp.p = dalloc<double>(n * d, s);
        dp.s = s;
        SJ_CUDA(cudaMemcpyAsync(dp.p, points, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
        pts = dp.p;
    }
    volatile double e2v = eps * eps;
    const double eps2 = e2v;
    struct Slot { unsigned long long cursor; uint32_t overflow; uint32_t pad; };
    Slot *dslot = static_cast<Slot *>(cg.c->d_slots), *hslot = static_cast<Slot *>(cg.c->h_slots);
    sj_result *res = new sj_result();
    res->device = bo.device;
    res->n_points = n;
    res->q0 = 0;
    res->q1 = n;
    res->include_self = jo.include_self;
    res->unicomp = 0;
    try {
        uint64_t cap = std::max<uint64_t>(n * 8, 1024);
        for (int attempt = 0; attempt < 2; ++attempt) {
            sj_batch bt;
            bt.pairs = dalloc<uint64_t>(cap, s);
            bt.cap = cap;
            bt.on_device = 1;
            SJ_CUDA(cudaMemsetAsync(dslot, 0, sizeof(Slot), s));
            switch (d) {
            case 2: launch_bf<2>((uint32_t)n, s, pts, eps2, jo.include_self, bt.pairs, &dslot->cursor, cap, &dslot->overflow); break;
            case 3: launch_bf<3>((uint32_t)n, s, pts, eps2, jo.include_self, bt.pairs, &dslot->cursor, cap, &dslot->overflow); break;
            case 4: launch_bf<4>((uint32_t)n, s, pts, eps2, jo.include_self, bt.pairs, &dslot->cursor, cap, &dslot->overflow); break;
            case 5: launch_bf<5>((uint32_t)n, s, pts, eps2, jo.include_self, bt.pairs, &dslot->cursor, cap, &dslot->overflow); break;
            default: launch_bf<6>((uint32_t)n, s, pts, eps2, jo.include_self, bt.pairs, &dslot->cursor, cap, &dslot->overflow); break;
            }
            SJ_CUDA(cudaMemcpyAsync(hslot, dslot, sizeof(Slot), cudaMemcpyDeviceToHost, s));
            SJ_CUDA(cudaStreamSynchronize(s));
            const uint64_t got = hslot->cursor;
            if (got > cap) {                   // exact re-allocation and re-run
                dev_free(bt.pairs, s);
                cap = got;
                continue;
            }
            bt.n = got;
            if (jo.sort_pairs) sort_pairs_device(bt.pairs, bt.n, n, s);
            if (jo.result_on_host) {
                uint64_t *h = static_cast<uint64_t *>(host_pinned_alloc(std::max<uint64_t>(1, got) * 8, nullptr));
                if (got) SJ_CUDA(cudaMemcpyAsync(h, bt.pairs, got * 8, cudaMemcpyDeviceToHost, s));
                SJ_CUDA(cudaStreamSynchronize(s));
                dev_free(bt.pairs, s);
                bt.pairs = h;
                bt.on_device = 0;
                bt.cap = got;
            }
            res->batches.push_back(bt);
            res->total = got;
            break;
        }
        SJ_CUDA(cudaStreamSynchronize(s));
        res->stats.pairs = res->total;
        res->stats.batches = (uint32_t)res->batches.size();
        res->stats.candidates_tested = n * n;
    } catch (...) {
        cudaStreamSynchronize(s);
        for (auto &b : res->batches) {
            if (b.on_device) dev_free(b.pairs, nullptr);
            else host_pinned_free(b.pairs);
        }
        delete res;
        throw;
    }
    return res;
}

}  // namespace sj
