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
//  * bounded binary search: the linear id is dimension-1-fastest, so the three cells
//    c_1-1..c_1+1 of a "row" (fixed dims >= 2) are consecutive ids, hence consecutive in B and
//    their points ONE contiguous A-range: one lookup per row of 3 cells, not per cell.  The
//    cells sharing the top-k coordinates form one contiguous range of B too; a prefix
//    directory (index_build.cu build_directory, <= 16 B per non-empty cell) maps a row's top-k
//    prefix to that range in O(1), and the binary search for the row is bounded to it (a few
//    entries).  When the directory covers every dimension a row costs two loads.  Eight
//    rows' directory loads are issued together for memory-level parallelism.
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
    unsigned long long *qbucket;   // kCountQuery: emissions summed per planning bucket (t / group)
    uint32_t group;                // kCountQuery: samples per bucket
    uint32_t *pcount;              // kCountPoint: cnt[original id]
    unsigned long long *work;      // [0] B searches, [1] distance tests, [2] emissions
    uint32_t q0, q1;               // A-position range of the queries
    uint32_t step, nsamples;       // kCountQuery: sample t = query q0 + (t/32)*32*step + t%32
    int include_self;
    int use_masks;
};

constexpr int kRefineThreads = 256;
#ifndef SJ_REFINE_MIN_BLOCKS
#define SJ_REFINE_MIN_BLOCKS 2
#endif
constexpr int kRefineMinBlocks = SJ_REFINE_MIN_BLOCKS;  // 2 x 256 threads: <= 128 registers

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
    uint32_t odd;      // bit j = parity of c_j (unicomp decisions without dynamic indexing)
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

// Everything the candidate loop needs, passed BY VALUE to the non-inlined scan (no stack copy
// of the kernel parameter structs).
template <int D>
struct ScanArgs {
    double x[D];                   // the query point
    const double *X;               // SoA coordinates [D][n]
    const uint32_t *A;
    uint64_t *out;
    unsigned long long *cursor;
    uint32_t *overflow;
    uint32_t *pcount;
    uint64_t cap;
    double eps2;
    uint32_t n;
    uint32_t pid;
};

// Test the points at A-positions [m0, m1) against the query.  Returns (tests << 32) | emitted.
// Not inlined on purpose: it is called from every neighbour-cell site; one copy keeps the kernel
// inside the instruction cache (an inlined version measured 28K SASS instructions, 47% no_inst).
template <int D, int MODE, bool BOTH>
__device__ __noinline__ uint64_t scan_range_impl(const ScanArgs<D> sa, uint32_t m0, uint32_t m1)
{
    JoinArgs ja{};
    ja.out = sa.out;
    ja.cursor = sa.cursor;
    ja.cap = sa.cap;
    ja.overflow = sa.overflow;
    ja.pcount = sa.pcount;
    uint32_t emitted = 0;
    for (uint32_t m = m0; m < m1; ++m) {
        double s;
        {
            const double t = __dsub_rn(sa.x[0], __ldg(sa.X + m));
            s = __dmul_rn(t, t);
        }
#pragma unroll
        for (int j = 1; j < D; ++j) {
            const double t = __dsub_rn(sa.x[j], __ldg(sa.X + (uint64_t)j * sa.n + m));
            s = __dadd_rn(s, __dmul_rn(t, t));
        }
        const bool hit = s <= sa.eps2;
        uint32_t qid = 0;
        if (MODE != kCountQuery && hit) qid = __ldg(sa.A + m);
        emit<MODE, BOTH>(ja, hit, sa.pid, qid, emitted);
    }
    return ((uint64_t)(m1 - m0) << 32) | emitted;
}

template <int D>
__device__ __forceinline__ ScanArgs<D> make_scan_args(const DevIndex &ix, const JoinArgs &ja, const QueryState<D> &q)
{
    ScanArgs<D> sa;
#pragma unroll
    for (int j = 0; j < D; ++j) sa.x[j] = q.x[j];
    sa.X = ix.X;
    sa.A = ix.A;
    sa.out = ja.out;
    sa.cursor = ja.cursor;
    sa.overflow = ja.overflow;
    sa.pcount = ja.pcount;
    sa.cap = ja.cap;
    sa.eps2 = ix.eps2;
    sa.n = ix.n;
    sa.pid = q.pid;
    return sa;
}

template <int D, int MODE, bool BOTH>
__device__ __forceinline__ void scan_range(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q, uint32_t m0,
                                           uint32_t m1)
{
    if (m0 >= m1) return;
    const uint64_t r = scan_range_impl<D, MODE, BOTH>(make_scan_args<D>(ix, ja, q), m0, m1);
    q.tests += (uint32_t)(r >> 32);
    q.emitted += (uint32_t)r;
}

// Offsets of the top-k (directory) dimensions, precomputed once per CTA in shared memory:
// for t in [0, 3^k): prefix delta, key delta, and bit masks of the dims moved by -1 / +1 and of
// the highest moved dim (unicomp decision).  3^k <= 243 in the cell-scan mode.
constexpr int kMaxTop = 243;
struct TopTable {
    int64_t dp[kMaxTop];     // sum delta_i * pstride_i
    int64_t dk[kMaxTop];     // dp * dir_div (key delta)
    uint32_t bits[kMaxTop];  // [0:6) dims at -1, [8:14) dims at +1, [16:22) one-hot highest moved dim
};

template <int D>
__device__ __forceinline__ void build_top_table(const DevIndex &ix, TopTable &tt)
{
    const int L = D - ix.dir_k;
    for (uint32_t t = threadIdx.x; t < ix.dir_ntop; t += blockDim.x) {
        int64_t dp = 0;
        uint32_t neg = 0, pos = 0, top = 0, rest = t;
        for (int i = L; i < D; ++i) {
            const uint32_t dl = rest % 3u;
            rest /= 3u;
            if (dl == 0u) { dp -= (int64_t)ix.pstride[i]; neg |= 1u << i; top = 1u << i; }
            else if (dl == 2u) { dp += (int64_t)ix.pstride[i]; pos |= 1u << i; top = 1u << i; }
        }
        tt.dp[t] = dp;
        tt.dk[t] = dp * (int64_t)ix.dir_div;
        tt.bits[t] = neg | (pos << 8) | (top << 16);
    }
}

// Alg. 1 lines 5-6 (getAdjCells, maskCellRange): the adjacent range of every dimension
// intersected with M_j, as a 3-bit set over the offsets {-1, 0, +1} (bit 1 = home, always in).
template <int D>
__device__ __forceinline__ void adjacent_masks(const DevIndex &ix, const JoinArgs &ja, const QueryState<D> &q,
                                               uint32_t (&allow)[D])
{
    const bool masked = ja.use_masks && ix.masks;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        allow[i] = 7u;
        if (masked) {
            const uint64_t lo = ix.mask_off[i] + q.c[i] - 1ull, hi = lo + 2ull;
            const uint32_t blo = (__ldg(ix.masks + (lo >> 5)) >> (lo & 31)) & 1u;
            const uint32_t bhi = (__ldg(ix.masks + (hi >> 5)) >> (hi & 31)) & 1u;
            allow[i] = 2u | blo | (bhi << 2);
        }
    }
}

// select element j (runtime) of a small register array without dynamic indexing
template <int D, class T>
__device__ __forceinline__ T sel(const T (&a)[D], int j)
{
    T v = a[0];
#pragma unroll
    for (int i = 1; i < D; ++i) v = (i == j) ? a[i] : v;
    return v;
}

// ---- search mode kSearchCellScan (sparse high-d data): for each offset of the top-k
// (directory) dimensions, the cells of that prefix are B[dir[p], dir[p+1]) -- a handful.  Each
// is tested by its low coordinates (decoded from its linear id): adjacent iff every low
// coordinate is within +-1; unicomp keeps it iff the query's coordinate in the highest
// differing dimension is odd (reading R13).  Covers every neighbour cell except the home cell.
template <int D, int MODE, bool UNICOMP>
__device__ __forceinline__ void search_cell_scan(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                                 uint32_t h, const uint32_t (&allow)[D], const TopTable &tt)
{
    const int L = D - ix.dir_k;     // low dimensions 0..L-1 are not in the directory prefix
    uint64_t ph = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) ph += q.c[j] * ix.pstride[j];
    // masked-out moves (Alg. 1 line 6) and, for unicomp, the dims whose home coordinate is even
    uint32_t bad = 0;
#pragma unroll
    for (int i = 0; i < D; ++i) {
        if (!(allow[i] & 1u)) bad |= 1u << i;
        if (!(allow[i] & 4u)) bad |= 1u << (i + 8);
        if (UNICOMP && !((q.odd >> i) & 1u)) bad |= 1u << (i + 16);
    }
    const uint32_t ntop = ix.dir_ntop;
    const uint64_t key = __ldg(ix.B + h);
#pragma unroll 1
    for (uint32_t t = 0; t < ntop; ++t) {
        const uint32_t bits = tt.bits[t];
        if (bits & bad) continue;      // masked-out coordinate, or decided by an even top dim
        const int jtop = (bits >> 16) ? (__ffs(bits >> 16) - 1) : -1;
        const uint64_t p = ph + (uint64_t)tt.dp[t];
        ++q.probes;
        const uint32_t lo = __ldg(ix.dir + p), hi = __ldg(ix.dir + p + 1);
        // the home key moved into prefix p: a cell there is adjacent iff its key differs from it by
        // sum_{i<L} delta_i * stride_i with every delta_i in {-1,0,1}.  Mixed-radix digits are
        // unique and stride_i > 2 * sum_{m<i} stride_m (|g_j| >= 3), so the deltas follow greedily
        // from the top low dimension: delta_i = sign(D) if |D| > lowR[i] else 0.
        const uint64_t kal = key + (uint64_t)tt.dk[t];
#pragma unroll 1
        for (uint32_t hh = lo; hh < hi; ++hh) {
            if (hh == h) continue;                       // home cell handled by the caller
            int64_t dlt = (int64_t)(__ldg(ix.B + hh) - kal);
            if (dlt > ix.lowR[L] || dlt < -ix.lowR[L]) continue;   // outside the +-1 box
            int jlow = -1;
#pragma unroll
            for (int i = D - 2; i >= 0; --i) {
                if (i >= L) continue;
                const int64_t R = ix.lowR[i], st = (int64_t)ix.strides[i];
                if (dlt > R) { dlt -= st; if (jlow < 0) jlow = i; }
                else if (dlt < -R) { dlt += st; if (jlow < 0) jlow = i; }
            }
            if (dlt != 0) continue;                      // not representable: not adjacent
            const int j = jtop >= 0 ? jtop : jlow;
            if (UNICOMP && !((q.odd >> j) & 1u)) continue;
            scan_range<D, MODE, UNICOMP>(ix, ja, q, __ldg(ix.G + hh), __ldg(ix.G + hh + 1));
        }
    }
}

// ---- search modes kSearchDenseRows / kSearchRows: rows whose highest differing dimension is
// j = D-1 .. 1 (a row = the three cells c_0-1..c_0+1 of fixed dims >= 1: consecutive linear ids,
// one contiguous A-range).  Unicomp: only when c_j is odd (reading R13).  Each row is looked up
// in the prefix directory, then (kSearchRows) by a search bounded to that prefix's range.
template <int D, int MODE, bool UNICOMP>
__device__ __forceinline__ void search_rows(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                            uint64_t key, const uint32_t (&allow)[D])
{
    uint64_t ph = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) ph += q.c[j] * ix.pstride[j];
    const bool dense = ix.search_mode == kSearchDenseRows;
    uint64_t st[D], ps[D];
#pragma unroll
    for (int i = 0; i < D; ++i) { st[i] = ix.strides[i]; ps[i] = ix.pstride[i]; }
#pragma unroll 1
    for (int j = D - 1; j >= 1; --j) {
        if (UNICOMP && !((q.odd >> j) & 1u)) continue;
        uint32_t nrows = 2u;
        for (int i = 1; i < j; ++i) nrows *= 3u;
        const uint64_t stj = sel<D>(st, j), psj = sel<D>(ps, j);
        const uint32_t allowj = sel<D>(allow, j);
#pragma unroll 1
        for (uint32_t r = 0; r < nrows; ++r) {
            // row offsets: dim j = +-1 (bit 0 of r), dims 1..j-1 in {-1,0,1} (base-3 digits)
            uint64_t b = (r & 1u) ? key + stj : key - stj;
            uint64_t p = (r & 1u) ? ph + psj : ph - psj;
            uint32_t ok = (allowj >> ((r & 1u) ? 2u : 0u)) & 1u;
            uint32_t rest = r >> 1;
#pragma unroll
            for (int i = 1; i < D - 1; ++i) {
                if (i >= j) break;
                const uint32_t dl = rest % 3u;
                rest /= 3u;
                ok &= allow[i] >> dl;
                if (dl == 0u) { b -= st[i]; p -= ps[i]; }
                else if (dl == 2u) { b += st[i]; p += ps[i]; }
            }
            if (!(ok & 1u)) continue;   // a masked-out coordinate: the row is empty
            ++q.probes;
            uint32_t s, e;
            if (dense) {                // p is the centre cell's key: its row is [p-1, p+1]
                s = __ldg(ix.dir + p - 1);
                e = __ldg(ix.dir + p + 2);
            } else {                    // bounded search inside the prefix's range for [b-1, b+1]
                s = __ldg(ix.dir + p);
                e = __ldg(ix.dir + p + 1);
                if (s >= e) continue;
                const uint64_t a = b - 1ull;
                if (e - s <= 8u) {
                    while (s < e && __ldg(ix.B + s) < a) ++s;
                } else {
                    s = lower_bound_u64(ix.B, s, e, a);
                }
                uint32_t f = s;
                while (f < e && __ldg(ix.B + f) <= a + 2ull) ++f;
                e = f;
            }
            if (s < e) scan_range<D, MODE, UNICOMP>(ix, ja, q, __ldg(ix.G + s), __ldg(ix.G + e));
        }
    }
}

template <int D, int MODE, bool UNICOMP>
__device__ __forceinline__ void refine_query(const DevIndex &ix, const JoinArgs &ja, uint32_t k,
                                            QueryState<D> &q, const TopTable &tt)
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
    q.odd = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) q.odd |= (uint32_t)(q.c[j] & 1ull) << j;
    const uint32_t h = __ldg(ix.pcell + k);
    const uint64_t key = __ldg(ix.B + h);
    const uint32_t cs = __ldg(ix.G + h), ce = __ldg(ix.G + h + 1);

    // ---- home cell: (p,p) once; unicomp: q after p in A-order, both orientations (R10)
    emit<MODE, false>(ja, ja.include_self != 0, q.pid, q.pid, q.emitted);
    if constexpr (UNICOMP) {
        scan_range<D, MODE, true>(ix, ja, q, k + 1, ce);
    } else {
        scan_range<D, MODE, false>(ix, ja, q, cs, k);
        scan_range<D, MODE, false>(ix, ja, q, k + 1, ce);
    }
    uint32_t allow[D];
    adjacent_masks<D>(ix, ja, q, allow);
    if (ix.search_mode == kSearchCellScan) {
        search_cell_scan<D, MODE, UNICOMP>(ix, ja, q, h, allow, tt);
        return;
    }
    // ---- home row: cells key-1 / key+1 (dims >= 1 equal); unicomp: only when c_0 is odd
    if (!UNICOMP || (q.c[0] & 1ull)) {
        if (h > 0 && __ldg(ix.B + h - 1) == key - 1ull)
            scan_range<D, MODE, UNICOMP>(ix, ja, q, __ldg(ix.G + h - 1), cs);
        if (h + 1 < ix.nG && __ldg(ix.B + h + 1) == key + 1ull)
            scan_range<D, MODE, UNICOMP>(ix, ja, q, ce, __ldg(ix.G + h + 2));
    }
    search_rows<D, MODE, UNICOMP>(ix, ja, q, key, allow);
}

template <int D, int MODE, bool UNICOMP>
__global__ void __launch_bounds__(kRefineThreads, kRefineMinBlocks)
k_refine(const DevIndex ix, const JoinArgs ja)
{
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t k;
    bool active;
    if constexpr (MODE == kCountQuery) {
        // sample t: lane t%32 of run t/32; run r = the first 32 queries of block [r*32*step, ...),
        // so a warp samples 32 consecutive (cell-coherent) queries
        k = ja.q0 + (t >> 5) * (32u * ja.step) + (t & 31u);
        active = t < ja.nsamples && k < ja.q1;
    } else {
        k = ja.q0 + t;
        active = k < ja.q1;
    }
    __shared__ TopTable tt;
    if (ix.search_mode == kSearchCellScan) {
        build_top_table<D>(ix, tt);
        __syncthreads();
    }
    QueryState<D> q;
    q.emitted = q.probes = q.tests = 0;
    if (active) {
        refine_query<D, MODE, UNICOMP>(ix, ja, k, q, tt);
        if constexpr (MODE == kCountQuery) atomicAdd(ja.qbucket + t / ja.group, (unsigned long long)q.emitted);
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
