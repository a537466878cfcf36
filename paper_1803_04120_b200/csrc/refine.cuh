// refine.cuh -- the per-point refine kernel (steps a5-a7 of the hot path).
//
// PAPER.md §4.5 Alg. 1 (lines 216-251, GPUSelfJoinGlobal): one thread per query point, in
// A-order (the cell-sorted order, so a warp's queries share cells and index prefixes).  The
// thread holds its point in registers (Alg. 1 l.4), finds its home cell, enumerates the
// adjacent cells (l.5-10), looks each up in B (l.11) and tests the points of every non-empty
// one (l.12-16).  With unicomp (§5.2, Alg. 2, readings R10-R13) only the
// cells whose highest differing dimension j has c_j odd are searched, and every hit is
// emitted in both orientations; the home cell emits (p,p) once plus, for
// every q after p in A-order, both (p,q) and (q,p).
//
// B200-specific choices:
//  * bounded, hierarchical binary search: the linear id is dimension-1-fastest, so the cells
//    sharing coordinates of dims >= L form ONE contiguous range of B.  The search descends
//    from the slowest dimension, narrowing the B range level by level ("bounded binary
//    search"); an empty range prunes the whole sub-tree of adjacent cells below it.  At
//    dimension 1 the three cells c_1-1..c_1+1 are consecutive ids, hence consecutive in B and
//    their points one contiguous A-range: one search per row of 3 cells, not per cell.
//  * the distance is s = (((x_0-y_0)^2 + (x_1-y_1)^2) + ...) with __dsub_rn/__dmul_rn/__dadd_rn
//    (no FMA contraction possible) compared with fl(eps^2): bit-identical decisions to the
//    oracle (readings R1, R2).
//  * warp-aggregated emission: __ballot_sync of the hits, __popc, ONE atomicAdd per warp on the
//    batch cursor, __shfl_sync of the base, each hitting lane writes its 1 or 2 packed pairs.
//    Writes past the batch capacity are dropped and flag an overflow; the cursor keeps counting
//    so the host learns the exact size and re-runs the batch (split-retry / exact realloc).
#pragma once

#include "sj_common.cuh"

namespace sj {

enum RefineMode { kEmit = 0, kCountQuery = 1, kCountPoint = 2 };

struct JoinArgs {
    uint64_t *out;                 // kEmit: batch pair buffer
    unsigned long long *cursor;    // kEmit: pairs emitted (exact even on overflow)
    uint64_t cap;                  // kEmit: capacity of out
    uint32_t *overflow;            // kEmit: set when a write was dropped
    uint32_t *qcount;              // kCountQuery: emissions of sample t
    uint32_t *pcount;              // kCountPoint: cnt[original id]
    unsigned long long *work;      // [0] B searches, [1] distance tests, [2] emissions
    uint32_t q0, q1;               // A-position range of the queries
    uint32_t step, nsamples;       // kCountQuery: sample t is query q0 + t*step
    int include_self;
    int use_masks;
};

constexpr int kRefineThreads = 256;

__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t *__restrict__ B, uint32_t lo, uint32_t hi,
                                                    uint64_t key)
{
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(B + mid) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

template <int D>
struct QueryState {
    double x[D];
    uint64_t c[D];
    uint32_t k;        // A-position of the query
    uint32_t pid;      // original id A[k]
    uint32_t emitted;  // pairs emitted by this thread
    uint32_t probes;   // binary searches
    uint32_t tests;    // distance evaluations
};

template <int MODE, bool BOTH>
__device__ __forceinline__ void emit(const JoinArgs &ja, bool hit, uint32_t pid, uint32_t qid, uint32_t &emitted)
{
    if constexpr (MODE == kCountQuery) {
        if (hit) emitted += BOTH ? 2u : 1u;
        return;
    } else if constexpr (MODE == kCountPoint) {
        if (hit) {
            emitted += BOTH ? 2u : 1u;
            atomicAdd(ja.pcount + pid, 1u);
            if (BOTH) atomicAdd(ja.pcount + qid, 1u);
        }
        return;
    } else {
        const unsigned mask = __activemask();
        const unsigned hits = __ballot_sync(mask, hit);
        if (hits == 0u) return;
        const int lane = threadIdx.x & 31;
        const int leader = __ffs(hits) - 1;
        constexpr unsigned per = BOTH ? 2u : 1u;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(ja.cursor, (unsigned long long)(__popc(hits) * per));
        base = __shfl_sync(mask, base, leader);
        if (hit) {
            emitted += per;
            const unsigned long long pos = base + (unsigned long long)(__popc(hits & ((1u << lane) - 1u)) * per);
            if (pos + per <= ja.cap) {
                ja.out[pos] = ((uint64_t)pid << 32) | qid;
                if (BOTH) ja.out[pos + 1] = ((uint64_t)qid << 32) | pid;
            } else {
                atomicOr(ja.overflow, 1u);
            }
        }
    }
}

// Test the points at A-positions [m0, m1) against the query.
template <int D, int MODE, bool BOTH>
__device__ __forceinline__ void scan_range(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q, uint32_t m0,
                                           uint32_t m1)
{
    const uint32_t n = ix.n;
    for (uint32_t m = m0; m < m1; ++m) {
        double s;
        {
            const double t = __dsub_rn(q.x[0], __ldg(ix.X + m));
            s = __dmul_rn(t, t);
        }
#pragma unroll
        for (int j = 1; j < D; ++j) {
            const double t = __dsub_rn(q.x[j], __ldg(ix.X + (uint64_t)j * n + m));
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        ++q.tests;
        const bool hit = s <= ix.eps2;
        uint32_t qid = 0;
        if (MODE != kCountQuery && hit) qid = __ldg(ix.A + m);
        emit<MODE, BOTH>(ja, hit, q.pid, qid, q.emitted);
    }
}

// Cells whose coordinates in dims > L are fixed (prefix contribution pk) occupy B[lo, hi).
// Visit every adjacent combination of dims 0..L (each in c-1..c+1).
template <int D, int MODE, bool BOTH, int L>
__device__ void descend(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q, uint32_t lo, uint32_t hi,
                        uint64_t pk)
{
    if constexpr (L == 0) {
        const uint64_t a = pk + q.c[0] - 1ull;            // row: ids a, a+1, a+2 (dim 1 fastest)
        const uint32_t s = lower_bound_u64(ix.B, lo, hi, a);
        ++q.probes;
        uint32_t e = s;
        while (e < hi && __ldg(ix.B + e) <= a + 2ull) ++e;
        if (s < e) scan_range<D, MODE, BOTH>(ix, ja, q, __ldg(ix.G + s), __ldg(ix.G + e));
    } else {
        const uint64_t st = ix.strides[L];
        const uint64_t base = pk + (q.c[L] - 1ull) * st;
        uint32_t b = lower_bound_u64(ix.B, lo, hi, base);
        ++q.probes;
#pragma unroll 1
        for (int v = 0; v < 3; ++v) {
            if (b >= hi) break;
            const uint32_t e = lower_bound_u64(ix.B, b, hi, base + (uint64_t)(v + 1) * st);
            ++q.probes;
            if (b < e) descend<D, MODE, BOTH, L - 1>(ix, ja, q, b, e, base + (uint64_t)v * st);
            b = e;
        }
    }
}

template <int D, int MODE, bool UNICOMP>
__device__ __forceinline__ void refine_query(const DevIndex &ix, const JoinArgs &ja, uint32_t k,
                                            QueryState<D> &q)
{
    q.k = k;
    q.pid = __ldg(ix.A + k);
    q.emitted = q.probes = q.tests = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        q.x[j] = __ldg(ix.X + (uint64_t)j * ix.n + k);
        // same IEEE operations as the build (reading R7): identical coordinates
        q.c[j] = 1ull + (uint64_t)floor(__ddiv_rn(__dsub_rn(q.x[j], ix.mins[j]), ix.w));
    }
    const uint32_t h = __ldg(ix.pcell + k);
    const uint64_t key = __ldg(ix.B + h);
    const uint32_t cs = __ldg(ix.G + h), ce = __ldg(ix.G + h + 1);

    // ---- home cell: (p,p) once; unicomp: q after p in A-order, both orientations
    emit<MODE, false>(ja, ja.include_self != 0, q.pid, q.pid, q.emitted);
    if constexpr (UNICOMP) {
        scan_range<D, MODE, true>(ix, ja, q, k + 1, ce);
    } else {
        scan_range<D, MODE, false>(ix, ja, q, cs, k);
        scan_range<D, MODE, false>(ix, ja, q, k + 1, ce);
    }
    // ---- home row: cells key-1 / key+1 (dims >= 2 equal); unicomp: only when c_1 is odd
    if (!UNICOMP || (q.c[0] & 1ull)) {
        if (h > 0 && __ldg(ix.B + h - 1) == key - 1ull)
            scan_range<D, MODE, UNICOMP>(ix, ja, q, __ldg(ix.G + h - 1), cs);
        if (h + 1 < ix.nG && __ldg(ix.B + h + 1) == key + 1ull)
            scan_range<D, MODE, UNICOMP>(ix, ja, q, ce, __ldg(ix.G + h + 2));
    }
    // ---- dims L = D-1 .. 1 as the highest differing dimension
    uint32_t lo = 0, hi = ix.nG;
    uint64_t pk = 0;  // contribution of dims > L (all equal to the home cell)
#pragma unroll
    for (int L = D - 1; L >= 1; --L) {
        const uint64_t st = ix.strides[L];
        if (!UNICOMP || (q.c[L] & 1ull)) {
#pragma unroll
            for (int sgn = 0; sgn < 2; ++sgn) {
                const uint64_t v = sgn ? q.c[L] + 1ull : q.c[L] - 1ull;
                if (ja.use_masks && ix.masks && !__ldg(ix.masks + ix.mask_off[L] + v)) continue;
                const uint64_t a = pk + v * st;
                const uint32_t s = lower_bound_u64(ix.B, lo, hi, a);
                const uint32_t e = lower_bound_u64(ix.B, s, hi, a + st);
                q.probes += 2;
                if (s < e) {
                    switch (L) {  // compile-time level dispatch (L is unrolled)
                    case 5: if constexpr (D > 5) descend<D, MODE, UNICOMP, 4>(ix, ja, q, s, e, a); break;
                    case 4: if constexpr (D > 4) descend<D, MODE, UNICOMP, 3>(ix, ja, q, s, e, a); break;
                    case 3: if constexpr (D > 3) descend<D, MODE, UNICOMP, 2>(ix, ja, q, s, e, a); break;
                    case 2: if constexpr (D > 2) descend<D, MODE, UNICOMP, 1>(ix, ja, q, s, e, a); break;
                    case 1: descend<D, MODE, UNICOMP, 0>(ix, ja, q, s, e, a); break;
                    }
                }
            }
        }
        // narrow to the home coordinate of dim L
        const uint64_t a = pk + q.c[L] * st;
        const uint32_t s = lower_bound_u64(ix.B, lo, hi, a);
        const uint32_t e = lower_bound_u64(ix.B, s, hi, a + st);
        q.probes += 2;
        lo = s;
        hi = e;
        pk = a;
    }
}

template <int D, int MODE, bool UNICOMP>
__global__ void __launch_bounds__(kRefineThreads)
k_refine(const DevIndex ix, const JoinArgs ja)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t k;
    bool active;
    if constexpr (MODE == kCountQuery) {
        active = t < ja.nsamples;
        k = ja.q0 + t * ja.step;
    } else {
        k = ja.q0 + t;
        active = k < ja.q1;
    }
    QueryState<D> q;
    q.emitted = q.probes = q.tests = 0;
    if (active) {
        refine_query<D, MODE, UNICOMP>(ix, ja, k, q);
        if constexpr (MODE == kCountQuery) ja.qcount[t] = q.emitted;
    }
    // work counters: warp reduce, one atomic per warp
    unsigned long long p = q.probes, c = q.tests, em = q.emitted;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        p += __shfl_xor_sync(0xffffffffu, p, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
        em += __shfl_xor_sync(0xffffffffu, em, o);
    }
    if ((threadIdx.x & 31) == 0 && ja.work) {
        atomicAdd(ja.work + 0, p);
        atomicAdd(ja.work + 1, c);
        atomicAdd(ja.work + 2, em);
    }
}

}  // namespace sj
