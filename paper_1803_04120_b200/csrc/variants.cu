// variants.cu -- SURVEY.md §8(f) rank 4: queries from outside the index's own A-order over the same
// grid index and predicate.
//
//   * two-set similarity join J(Q,P) ("the related similarity join"; R19): every
//     query of Q probes the 3^d cells around its own cell in P's grid, full search (no unicomp: Q != P).
//   * kNN self-join ("other spatial searches, such as kNN"; R20): every point's k
//     best (s, id) among the points of its 3^d neighbour cells that satisfy the join predicate; certified
//     when there are k of them, otherwise re-run on an index with a larger eps (x 4^(1/d)).
//
// One kernel, k_probe<D, MODE>, ONE WARP PER QUERY:
//   1. the query's coordinates are warp-uniform; per dimension the <= 3 neighbour coordinates that lie in
//      [1, |g_j|-2] and are occupied (M_j, Alg. 1 l.6) form a 3-bit set, so boundary and masked queries
//      enumerate only the product of what can exist;
//   2. the lanes look up 32 of those cells at a time: linear id (R8), prefix p = sum c_j * pstride_j, the
//      directory range [dir[p], dir[p+1]) of B, one bounded binary search (PAPER.md:173 B, G); on
//      cell-scan indexes (sparse: a few cells per top-k prefix) the lanes enumerate the 3^k top prefixes
//      instead (occupancy bitmaps drop the empty ones) and the warp scans their cells' low coordinates;
//   3. the cells' point ranges are concatenated by a warp prefix sum and swept 32 candidates per step,
//      each lane finding its candidate's cell by a 5-step shuffle search -- the warp stays converged and
//      every lane tests a candidate even when the cells hold one point each (sparse 6-D);
//   4. the predicate is the self-join's (R1: __dsub_rn/__dmul_rn/__dadd_rn left to right, <= fl(eps^2));
//      (the FP32 self-join, R21, is the self-join's own path with a binary32 predicate: refine.cuh kF32)
//   5. count: hits per query; fill: warp-aggregated emission (one atomic per 32 candidates);
//      kNN: a warp-wide sorted top-k list (lane i holds the i-th best (s, id)), each surviving candidate
//      inserted by one ballot + one shuffle-up.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "sj_common.cuh"

namespace sj {
namespace {

constexpr int kProbeThreads = 256;
constexpr int kMaxK = 32;
enum ProbeMode { kPCount = 0, kPFill = 1, kPKnn = 2 };

struct ProbeArgs {
    const double *q;              // AoS query coordinates [rows][D] (unused with q_index)
    const uint32_t *qlist;        // optional: query rows to process (kNN re-runs: original ids)
    uint32_t q_begin, nq;         // queries q_begin .. q_begin+nq-1 (rows, or qlist entries)
    int q_index;                  // 1: the queries are the index's own points in A-order (X, A)
    int self;                     // skip the candidate whose id is the query's (kNN)
    int tiled;                    // count / fill through k_probe_tiled (qlist sorted by cell)
    uint32_t *counts;             // count: per query (index t - q_begin)
    unsigned long long *buckets;  // count: per 1024 queries
    uint32_t *nonfinite;          // count: set when a query coordinate is NaN / inf
    uint64_t *out;                // fill: pair buffer, cursor, capacity, overflow flag
    unsigned long long *cursor;
    uint64_t cap;
    uint32_t *overflow;
    uint32_t k;                   // kNN: neighbours per query (1..32)
    uint32_t *ids;                // kNN: [N][k] rows by original id
    double *dist2;
    uint32_t *unres;              // kNN: ids of uncertified queries, count in *n_unres
    uint32_t *n_unres;
    unsigned long long *work;     // [0] cells probed, [1] candidates tested, [2] pairs / hits
};

__device__ __forceinline__ bool kv_less(uint64_t as, uint32_t ai, uint64_t bs, uint32_t bi)
{
    return as < bs || (as == bs && ai < bi);
}

// Per-query state of the warp (every lane holds the same query; kNN: lane i < k holds the i-th best).
struct ProbeState {
    uint32_t found;                 // hits so far (all lanes agree)
    uint64_t bs;                    // kNN: this lane's entry (s bits, id); sentinels sort last
    uint32_t bi;
    uint64_t kth_s;                 // kNN: the k-th entry (warp-uniform)
    uint32_t kth_i;
    unsigned long long tests;       // this lane's distance evaluations
};

// Lane-level flattening: given one range [lo, hi) per lane, returns (via the shuffle search) for
// position f of the concatenation the owner lane's lo and exclusive prefix.  inc = inclusive prefix of
// the lengths across lanes.
__device__ __forceinline__ uint32_t owner_of(uint32_t inc, uint32_t f)
{
    uint32_t pos = 0;                                   // lanes whose range ends at or before f
#pragma unroll
    for (uint32_t s = 16; s; s >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, inc, pos + s - 1u);
        if (v <= f) pos += s;
    }
    return pos & 31u;
}

__device__ __forceinline__ uint32_t warp_inclusive(uint32_t v, uint32_t lane)
{
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, v, s);
        if (lane >= (uint32_t)s) v += t;
    }
    return v;
}

// Test every point of the lanes' A-ranges [lo, hi) against the query, 32 candidates per step over the
// concatenation (Alg. 1 l.12-16 with R1's predicate), and hand the hits to the mode.
template <int D, int MODE>
__device__ __forceinline__ void sweep(const DevIndex &ix, const ProbeArgs &pa, const double (&x)[D], uint32_t qid,
                                      uint32_t lo, uint32_t hi, uint32_t lane, ProbeState &st)
{
    const uint32_t n = ix.n;
    const uint32_t len = hi - lo;
    const uint32_t inc = warp_inclusive(len, lane);
    const uint32_t total = __shfl_sync(0xffffffffu, inc, 31);
    const uint32_t exc = inc - len;
    for (uint32_t f0 = 0; f0 < total; f0 += 32u) {
        const uint32_t f = f0 + lane;
        const uint32_t own = owner_of(inc, f);
        const uint32_t olo = __shfl_sync(0xffffffffu, lo, own);
        const uint32_t oexc = __shfl_sync(0xffffffffu, exc, own);
        const bool act = f < total;
        const uint32_t m = olo + (f - oexc);
        bool hit = false;
        double s = 0.0;
        uint32_t pid = 0;
        if (act) {
            {
                const double d0 = __dsub_rn(x[0], __ldg(ix.X + m));
                s = __dmul_rn(d0, d0);
            }
#pragma unroll
            for (int j = 1; j < D; ++j) {
                const double dj = __dsub_rn(x[j], __ldg(ix.X + (uint64_t)j * n + m));
                s = __dadd_rn(s, __dmul_rn(dj, dj));
            }
            ++st.tests;
            hit = s <= ix.eps2;
        }
        if (hit) {
            pid = __ldg(ix.A + m);
            if (pa.self && pid == qid) hit = false;
        }
        const unsigned hb = __ballot_sync(0xffffffffu, hit);
        st.found += (uint32_t)__popc(hb);
        if constexpr (MODE == kPFill) {
            if (hb) {
                unsigned long long b0 = 0;
                if (lane == 0) b0 = atomicAdd(pa.cursor, (unsigned long long)__popc(hb));
                b0 = __shfl_sync(0xffffffffu, b0, 0);
                if (hit) {
                    const unsigned long long at = b0 + (unsigned long long)__popc(hb & ((1u << lane) - 1u));
                    if (at < pa.cap) pa.out[at] = ((uint64_t)qid << 32) | pid;
                    else atomicOr(pa.overflow, 1u);
                }
            }
        } else if constexpr (MODE == kPKnn) {
            const uint64_t sb = (uint64_t)__double_as_longlong(s);
            unsigned surv = __ballot_sync(0xffffffffu, hit && kv_less(sb, pid, st.kth_s, st.kth_i));
            while (surv) {
                const int src = __ffs(surv) - 1;
                surv &= surv - 1u;
                const uint64_t cs = __shfl_sync(0xffffffffu, sb, src);
                const uint32_t ci = __shfl_sync(0xffffffffu, pid, src);
                if (!kv_less(cs, ci, st.kth_s, st.kth_i)) continue;          // warp-uniform
                const bool gt = lane < pa.k && kv_less(cs, ci, st.bs, st.bi);
                const uint32_t ins = pa.k - (uint32_t)__popc(__ballot_sync(0xffffffffu, gt));
                const uint64_t us = __shfl_up_sync(0xffffffffu, st.bs, 1);
                const uint32_t ui = __shfl_up_sync(0xffffffffu, st.bi, 1);
                if (lane == ins) { st.bs = cs; st.bi = ci; }
                else if (lane > ins && lane < pa.k) { st.bs = us; st.bi = ui; }
                st.kth_s = __shfl_sync(0xffffffffu, st.bs, pa.k - 1u);
                st.kth_i = __shfl_sync(0xffffffffu, st.bi, pa.k - 1u);
            }
        }
    }
}

// Decode the r-th member (mixed radix over the dims' valid sets) of the neighbour enumeration: the
// e-th set bit of sel_j is the coordinate (c_j - 1) + e.
__device__ __forceinline__ uint64_t pick(uint32_t sel, uint32_t rj, uint64_t c0)
{
    uint32_t m = sel;
    if (rj >= 1u) m &= m - 1u;
    if (rj >= 2u) m &= m - 1u;
    return c0 - 1u + (uint64_t)(__ffs(m) - 1);
}

// One query (warp-uniform qid and point): its neighbour cells, their candidates, the mode's epilogue.
// t = the query's position in this launch (count: index of counts[]).
template <int D, int MODE>
__device__ __forceinline__ void probe_query(const DevIndex &ix, const ProbeArgs &pa, uint32_t t, uint32_t qid,
                                            const double (&x)[D], uint32_t lane, unsigned long long &probes,
                                            unsigned long long &tests, unsigned long long &hits_all)
{
    // cell-scan indexes (few cells per top-k prefix): enumerate the 3^k top prefixes and scan their
    // cells, instead of one bounded binary search per neighbour cell (3^d of them)
    const bool prefix_scan = ix.search_mode == kSearchCellScan && ix.dir_k < D;
    const int L = D - ix.dir_k;
    // ---- 1. per dimension: c_j (R7 against the index's geometry) and the valid neighbour set
    uint64_t c0[D];
    uint32_t sel[D];
    uint32_t ncell = 1, ntop = 1;
    bool finite = true;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        finite = finite && isfinite(x[j]);
        const double tq = floor(__ddiv_rn(__dsub_rn(x[j], ix.mins[j]), ix.w));   // = c_j - 1
        uint32_t m = 0;
        c0[j] = 0;
        if (tq >= -1.0 && tq <= (double)ix.cpd[j]) {       // some of tq .. tq+2 may be in [1, |g_j|-2]
            const int64_t b = (int64_t)tq;
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const int64_t cc = b + e;
                bool ok = cc >= 1 && cc <= (int64_t)ix.cpd[j] - 2;
                if (ok && ix.masks) {
                    const uint64_t bit = ix.mask_off[j] + (uint64_t)cc;
                    ok = (__ldg(ix.masks + (bit >> 5)) >> (bit & 31u)) & 1u;
                }
                if (ok) m |= 1u << e;
            }
            c0[j] = (uint64_t)(b + 1);                      // as unsigned: b >= -1
        }
        sel[j] = m;
        ncell *= (uint32_t)__popc(m);
        if (j >= L) ntop *= (uint32_t)__popc(m);
    }
    if (MODE == kPCount && !finite && lane == 0) atomicOr(pa.nonfinite, 1u);
    ProbeState st{0u, ~0ull, 0xffffffffu, ~0ull, 0xffffffffu, 0ull};
    if (ncell == 0u) {
        // nothing adjacent exists
    } else if (prefix_scan) {
        // ---- 2a. top prefixes, 32 per round; the occupancy bitmap (dilated +-1 along dimension
        //      L-1) drops prefixes with no cell near the query's c_{L-1}
        uint64_t qh = 0, qh2 = 0;
#pragma unroll
        for (int j = 0; j < D; ++j)
            if (j < L) { qh += c0[j] * ix.occ_mul[j]; qh2 += c0[j] * ix.occ2_mul[j]; }
        for (uint32_t base = 0; base < ntop; base += 32u) {
            uint32_t clo = 0, chi = 0;
            const uint32_t o = base + lane;
            if (o < ntop) {
                uint32_t r = o;
                uint64_t p = 0, ob = qh, ob2 = qh2;
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    if (j < L) continue;
                    const uint32_t nj = (uint32_t)__popc(sel[j]);
                    const uint32_t rj = r % nj;
                    r /= nj;
                    const uint64_t cj = pick(sel[j], rj, c0[j]);
                    p += cj * ix.pstride[j];
                    ob += cj * ix.occ_mul[j];
                    ob2 += cj * ix.occ2_mul[j];
                }
                bool live = true;
                if (ix.occ) {
                    live = (__ldg(ix.occ + (ob >> 5)) >> (ob & 31u)) & 1u;
                    if (live && ix.occ2) live = (__ldg(ix.occ2 + (ob2 >> 5)) >> (ob2 & 31u)) & 1u;
                }
                ++probes;
                if (live) {
                    clo = __ldg(ix.dir + p);
                    chi = __ldg(ix.dir + p + 1);
                }
            }
            // ---- 2b. the prefixes' cells, 32 per step: keep those whose low coordinates are
            //      adjacent (and valid) -> their point ranges
            const uint32_t clen = chi - clo;
            const uint32_t cinc = warp_inclusive(clen, lane);
            const uint32_t ctotal = __shfl_sync(0xffffffffu, cinc, 31);
            const uint32_t cexc = cinc - clen;
            for (uint32_t g0 = 0; g0 < ctotal; g0 += 32u) {
                const uint32_t g = g0 + lane;
                const uint32_t own = owner_of(cinc, g);
                const uint32_t olo = __shfl_sync(0xffffffffu, clo, own);
                const uint32_t oexc = __shfl_sync(0xffffffffu, cexc, own);
                uint32_t lo = 0, hi = 0;
                if (g < ctotal) {
                    const uint32_t h = olo + (g - oexc);
                    uint64_t c[D];
                    key_to_coords<D>(ix, __ldg(ix.B + h), c);
                    bool ok = true;
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        if (j >= L) continue;
                        const uint64_t e = c[j] - (c0[j] - 1u);    // 0..2 when adjacent
                        ok = ok && e < 3u && ((sel[j] >> e) & 1u);
                    }
                    if (ok) {
                        lo = __ldg(ix.G + h);
                        hi = __ldg(ix.G + h + 1);
                    }
                }
                sweep<D, MODE>(ix, pa, x, qid, lo, hi, lane, st);
            }
        }
    } else {
        // ---- 2. 32 neighbour cells per round, each looked up by one lane: linear id (R8), prefix
        //      p = sum c_j * pstride_j, one binary search of B bounded to [dir[p], dir[p+1])
        for (uint32_t base = 0; base < ncell; base += 32u) {
            uint32_t lo = 0, hi = 0;
            const uint32_t o = base + lane;
            if (o < ncell) {
                uint32_t r = o;
                uint64_t key = 0, p = 0;
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    const uint32_t nj = (uint32_t)__popc(sel[j]);
                    const uint32_t rj = r % nj;
                    r /= nj;
                    const uint64_t cj = pick(sel[j], rj, c0[j]);
                    key += cj * ix.strides[j];
                    p += cj * ix.pstride[j];
                }
                ++probes;
                uint32_t h = __ldg(ix.dir + p);
                uint32_t h1 = __ldg(ix.dir + p + 1);
                while (h < h1) {
                    const uint32_t mid = (h + h1) >> 1;
                    if (__ldg(ix.B + mid) < key) h = mid + 1;
                    else h1 = mid;
                }
                if (h < ix.nG && __ldg(ix.B + h) == key) {
                    lo = __ldg(ix.G + h);
                    hi = __ldg(ix.G + h + 1);
                }
            }
            // ---- 3. the cells' points, swept by the whole warp
            sweep<D, MODE>(ix, pa, x, qid, lo, hi, lane, st);
        }
    }
    tests += st.tests;
    const uint32_t found = st.found;
    hits_all += found;
    if constexpr (MODE == kPCount) {
        if (lane == 0) {
            pa.counts[t] = found;
            atomicAdd(pa.buckets + (t >> 10), (unsigned long long)found);
        }
    } else if constexpr (MODE == kPKnn) {
        if (found >= pa.k) {
            if (lane < pa.k) {
                pa.ids[(uint64_t)qid * pa.k + lane] = st.bi;
                pa.dist2[(uint64_t)qid * pa.k + lane] = __longlong_as_double((long long)st.bs);
            }
        } else if (lane == 0) {
            pa.unres[atomicAdd(pa.n_unres, 1u)] = qid;
        }
    }
}

#ifndef SJ_PROBE_MINB
#define SJ_PROBE_MINB 4   // 4 x 256 threads per SM (<= 64 registers): 6-D eps=8 two-set 82 -> 68 ms, kNN 6-D 74 -> 68 ms (2: slower)
#endif
template <int D, int MODE>
__global__ void __launch_bounds__(kProbeThreads, SJ_PROBE_MINB) k_probe(const DevIndex ix, const ProbeArgs pa)
{
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n = ix.n;
    unsigned long long probes = 0, tests = 0, hits_all = 0;
    for (uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < pa.nq; t += warps) {
        const uint32_t row = pa.q_begin + t;
        uint32_t qid;
        double x[D];
        if (pa.q_index) {
            qid = __ldg(ix.A + row);
#pragma unroll
            for (int j = 0; j < D; ++j) x[j] = __ldg(ix.X + (uint64_t)j * n + row);
        } else {
            qid = pa.qlist ? __ldg(pa.qlist + row) : row;
#pragma unroll
            for (int j = 0; j < D; ++j) x[j] = __ldg(pa.q + (uint64_t)qid * D + j);
        }
        probe_query<D, MODE>(ix, pa, t, qid, x, lane, probes, tests, hits_all);
    }
    // per-lane counters: one atomic per warp and counter
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        probes += __shfl_xor_sync(0xffffffffu, probes, s);
        tests += __shfl_xor_sync(0xffffffffu, tests, s);
    }
    if (lane == 0 && pa.work) {
        atomicAdd(pa.work + 0, probes);
        atomicAdd(pa.work + 1, tests);
        atomicAdd(pa.work + 2, hits_all);
    }
}

// ---- two-set join, dense regimes: queries sorted by their cell in P's grid, 32 per warp.  A warp
// whose 32 queries share one cell (populous cells) shares the candidates too: each 32-candidate tile
// of the neighbour cells is staged once in shared memory (SoA) and every lane tests it against its own
// query (32 x 32 tests per tile instead of 32 per tile); other warps take their queries one by one
// (probe_query).  Count / fill only.
constexpr int kTileWarps = kProbeThreads / 32;
#ifndef SJ_TILE_RUNS
#define SJ_TILE_RUNS 4    // a warp with more cell runs than this takes its queries one by one (8: 3-D
                          // about equal, 16 / 32: 3-D 5.2 -> 8.7 / 9.4 ms)
#endif

// cell key of every query in P's grid (R7, R8), or 2^key_bits when no neighbour cell can exist
// (a coordinate outside the pad cells 0 .. |g_j|-1, or non-finite): the sort key of the tiled join
template <int D>
__global__ void __launch_bounds__(256) k_qkeys(const DevIndex ix, const double *__restrict__ q, uint32_t nq,
                                               uint64_t sentinel, uint64_t *__restrict__ keys,
                                               uint32_t *__restrict__ vals, uint32_t *__restrict__ nonfinite)
{
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nq; t += gridDim.x * blockDim.x) {
        uint64_t key = 0;
        bool ok = true;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const double xj = __ldg(q + (uint64_t)t * D + j);
            if (!isfinite(xj)) atomicOr(nonfinite, 1u);
            const double tq = floor(__ddiv_rn(__dsub_rn(xj, ix.mins[j]), ix.w));
            ok = ok && tq >= -1.0 && tq <= (double)ix.cpd[j] - 2.0;    // c_j = tq + 1 in [0, |g_j| - 1]
            if (ok) key += (uint64_t)(tq + 1.0) * ix.strides[j];
        }
        keys[t] = ok ? key : sentinel;
        vals[t] = t;
    }
}

template <int D, int MODE>
__global__ void __launch_bounds__(kProbeThreads, SJ_PROBE_MINB) k_probe_tiled(const DevIndex ix, const ProbeArgs pa)
{
    __shared__ __align__(16) double s_tx[kTileWarps][D * 32];
    __shared__ uint32_t s_tid[kTileWarps][32];
    const uint32_t lane = threadIdx.x & 31u, wib = threadIdx.x >> 5;
    const uint32_t groups = (pa.nq + 31u) >> 5;
    const uint32_t n = ix.n;
    double *tx = s_tx[wib];
    uint32_t *tid = s_tid[wib];
    unsigned long long probes = 0, tests = 0, hits_all = 0;
    for (uint32_t grp = blockIdx.x * kTileWarps + wib; grp < groups; grp += gridDim.x * kTileWarps) {
        const uint32_t t = grp * 32u + lane;             // this lane's query position in the launch
        const bool have = t < pa.nq;
        uint32_t qid = 0;
        double x[D];
        double tq[D];
        bool ok = have;
        if (have) {
            qid = __ldg(pa.qlist + pa.q_begin + t);
#pragma unroll
            for (int j = 0; j < D; ++j) x[j] = __ldg(pa.q + (uint64_t)qid * D + j);
        } else {
#pragma unroll
            for (int j = 0; j < D; ++j) x[j] = 0.0;
        }
        uint64_t mykey = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            tq[j] = floor(__ddiv_rn(__dsub_rn(x[j], ix.mins[j]), ix.w));   // c_j - 1
            ok = ok && tq[j] >= -1.0 && tq[j] <= (double)ix.cpd[j] - 2.0;  // some neighbour can exist
            if (ok) mykey += (uint64_t)(tq[j] + 1.0) * ix.strides[j];
        }
        // the group's runs of queries sharing a cell (sorted: runs are contiguous lanes); lanes whose
        // query has no possible neighbour take a key of their own and no run
        const unsigned peers = __match_any_sync(0xffffffffu, ok ? mykey : (0x8000000000000000ull | lane));
        const unsigned leaders = __ballot_sync(0xffffffffu, ok && (uint32_t)(__ffs(peers) - 1) == lane);
        uint32_t found = 0;
        if constexpr (MODE == kPCount) {
            bool finite = true;
#pragma unroll
            for (int j = 0; j < D; ++j) finite = finite && isfinite(x[j]);
            if (have && !finite) atomicOr(pa.nonfinite, 1u);
        }
        if (__popc(leaders) > SJ_TILE_RUNS) {
            // many cells (sparse regime): the queries one by one, each over a flattened sweep
            for (uint32_t i = 0; i < 32u; ++i) {
                const uint32_t ti = grp * 32u + i;
                if (ti >= pa.nq) break;                  // warp-uniform
                const uint32_t qi = __shfl_sync(0xffffffffu, qid, i);
                double xi[D];
#pragma unroll
                for (int j = 0; j < D; ++j) xi[j] = __shfl_sync(0xffffffffu, x[j], i);
                probe_query<D, MODE>(ix, pa, ti, qi, xi, lane, probes, tests, hits_all);
            }
            continue;
        }
        for (unsigned lead = leaders; lead; lead &= lead - 1u) {
        const int ld = __ffs(lead) - 1;
        const bool mine = (__shfl_sync(0xffffffffu, peers, ld) >> lane) & 1u;   // this lane's query is in the run
        // ---- the run's cell: its neighbour coordinates (valid, occupied), as in probe_query
        uint64_t c0[D];
        uint32_t sel[D];
        uint32_t ncell = 1;
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const int64_t b = (int64_t)__shfl_sync(0xffffffffu, tq[j], ld);
            uint32_t m = 0;
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const int64_t cc = b + e;
                bool v = cc >= 1 && cc <= (int64_t)ix.cpd[j] - 2;
                if (v && ix.masks) {
                    const uint64_t bit = ix.mask_off[j] + (uint64_t)cc;
                    v = (__ldg(ix.masks + (bit >> 5)) >> (bit & 31u)) & 1u;
                }
                if (v) m |= 1u << e;
            }
            c0[j] = (uint64_t)(b + 1);
            sel[j] = m;
            ncell *= (uint32_t)__popc(m);
        }
        for (uint32_t base = 0; base < ncell; base += 32u) {
            uint32_t lo = 0, hi = 0;
            const uint32_t o = base + lane;
            if (o < ncell) {
                uint32_t r = o;
                uint64_t key = 0, p = 0;
#pragma unroll
                for (int j = 0; j < D; ++j) {
                    const uint32_t nj = (uint32_t)__popc(sel[j]);
                    const uint32_t rj = r % nj;
                    r /= nj;
                    const uint64_t cj = pick(sel[j], rj, c0[j]);
                    key += cj * ix.strides[j];
                    p += cj * ix.pstride[j];
                }
                ++probes;
                uint32_t h = __ldg(ix.dir + p);
                uint32_t h1 = __ldg(ix.dir + p + 1);
                while (h < h1) {
                    const uint32_t mid = (h + h1) >> 1;
                    if (__ldg(ix.B + mid) < key) h = mid + 1;
                    else h1 = mid;
                }
                if (h < ix.nG && __ldg(ix.B + h) == key) {
                    lo = __ldg(ix.G + h);
                    hi = __ldg(ix.G + h + 1);
                }
            }
            unsigned pend = __ballot_sync(0xffffffffu, lo < hi);
            while (pend) {
                const int src = __ffs(pend) - 1;
                pend &= pend - 1u;
                const uint32_t rlo = __shfl_sync(0xffffffffu, lo, src), rhi = __shfl_sync(0xffffffffu, hi, src);
                for (uint32_t m0 = rlo; m0 < rhi; m0 += 32u) {
                    const uint32_t lim = min(32u, rhi - m0);
                    __syncwarp();
                    if (lane < lim) {
#pragma unroll
                        for (int j = 0; j < D; ++j) tx[j * 32 + lane] = __ldg(ix.X + (uint64_t)j * n + m0 + lane);
                        tid[lane] = __ldg(ix.A + m0 + lane);
                    }
                    __syncwarp();
                    // two candidates per 16-byte broadcast load per dimension; fully unrolled (constant bit
                    // positions), the ragged last tile leaves by a uniform branch
                    uint32_t hm = 0;
                    const double2 *t2 = reinterpret_cast<const double2 *>(tx);
                    const uint32_t npair = (lim + 1u) >> 1;
#pragma unroll
                    for (uint32_t e2 = 0; e2 < 16u; ++e2) {
                        if (e2 >= npair) break;
                        double2 c = t2[e2];
                        double ta = __dsub_rn(x[0], c.x), tb = __dsub_rn(x[0], c.y);
                        double sa = __dmul_rn(ta, ta), sb = __dmul_rn(tb, tb);
#pragma unroll
                        for (int j = 1; j < D; ++j) {
                            c = t2[j * 16 + e2];
                            ta = __dsub_rn(x[j], c.x);
                            tb = __dsub_rn(x[j], c.y);
                            sa = __dadd_rn(sa, __dmul_rn(ta, ta));
                            sb = __dadd_rn(sb, __dmul_rn(tb, tb));
                        }
                        if (sa <= ix.eps2) hm |= 1u << (2u * e2);
                        if (sb <= ix.eps2) hm |= 2u << (2u * e2);
                    }
                    hm &= lim == 32u ? 0xffffffffu : ((1u << lim) - 1u);   // (the odd tail's partner is stale)
                    if (!mine) hm = 0u;
                    tests += lim;
                    const uint32_t cnt = (uint32_t)__popc(hm);
                    found += cnt;
                    if constexpr (MODE == kPFill) {
                        const uint32_t inc = warp_inclusive(cnt, lane);
                        const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
                        if (tot) {
                            unsigned long long b0 = 0;
                            if (lane == 31) b0 = atomicAdd(pa.cursor, (unsigned long long)tot);
                            b0 = __shfl_sync(0xffffffffu, b0, 31);
                            // the tile's pairs written cooperatively: output slot k (lane k mod 32) is hit
                            // k - excl(L) of the owner lane L -- consecutive slots, coalesced stores
                            // (per-lane loops over their own hits stored 32 scattered runs per instruction)
                            for (uint32_t k0 = 0; k0 < tot; k0 += 32u) {
                                const uint32_t k = k0 + lane;
                                const uint32_t own = owner_of(inc, k);
                                const uint32_t ohm = __shfl_sync(0xffffffffu, hm, own);
                                const uint32_t oex = __shfl_sync(0xffffffffu, inc - cnt, own);
                                const uint32_t oqid = __shfl_sync(0xffffffffu, qid, own);
                                if (k < tot) {
                                    const uint32_t e = __fns(ohm, 0u, (int)(k - oex) + 1);
                                    const unsigned long long at = b0 + k;
                                    if (at < pa.cap) pa.out[at] = ((uint64_t)oqid << 32) | tid[e];
                                    else atomicOr(pa.overflow, 1u);
                                }
                            }
                        }
                    }
                }
            }
        }
        }   // runs
        hits_all += found;
        if constexpr (MODE == kPCount) {
            pa.counts[t] = found;
            unsigned long long sum = found;
#pragma unroll
            for (int o2 = 16; o2; o2 >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o2);
            if (lane == 0) atomicAdd(pa.buckets + (t >> 10), sum);      // a group never straddles a bucket
        }
    }
#pragma unroll
    for (int o2 = 16; o2; o2 >>= 1) {
        probes += __shfl_xor_sync(0xffffffffu, probes, o2);
        tests += __shfl_xor_sync(0xffffffffu, tests, o2);
        hits_all += __shfl_xor_sync(0xffffffffu, hits_all, o2);
    }
    if (lane == 0 && pa.work) {
        atomicAdd(pa.work + 0, probes);
        atomicAdd(pa.work + 1, tests);
        atomicAdd(pa.work + 2, hits_all);
    }
}

template <int D>
void launch_probe_d(int mode, const DevIndex &ix, const ProbeArgs &pa, dim3 grid, cudaStream_t s)
{
    if (pa.tiled && mode != kPKnn) {
        const uint64_t groups = ((uint64_t)pa.nq + 31) / 32;
        const dim3 g2((uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((groups + kTileWarps - 1) / kTileWarps, grid.x)));
        if (mode == kPCount) k_probe_tiled<D, kPCount><<<g2, kProbeThreads, 0, s>>>(ix, pa);
        else k_probe_tiled<D, kPFill><<<g2, kProbeThreads, 0, s>>>(ix, pa);
        return;
    }
    switch (mode) {
    case kPCount: k_probe<D, kPCount><<<grid, kProbeThreads, 0, s>>>(ix, pa); break;
    case kPFill: k_probe<D, kPFill><<<grid, kProbeThreads, 0, s>>>(ix, pa); break;
    default: k_probe<D, kPKnn><<<grid, kProbeThreads, 0, s>>>(ix, pa); break;
    }
}

void launch_probe(int mode, const DevIndex &ix, const ProbeArgs &pa, int dev, cudaStream_t s)
{
    if (pa.nq == 0) return;
    // one warp per query, grid-strided; 8 CTAs of 256 per SM fill it
    const uint64_t want = ((uint64_t)pa.nq + (kProbeThreads / 32) - 1) / (kProbeThreads / 32);
    const dim3 grid((uint32_t)std::min<uint64_t>(want, (uint64_t)device_sm_count(dev) * 8));
    switch (ix.d) {
    case 2: launch_probe_d<2>(mode, ix, pa, grid, s); break;
    case 3: launch_probe_d<3>(mode, ix, pa, grid, s); break;
    case 4: launch_probe_d<4>(mode, ix, pa, grid, s); break;
    case 5: launch_probe_d<5>(mode, ix, pa, grid, s); break;
    case 6: launch_probe_d<6>(mode, ix, pa, grid, s); break;
    default: fail(SJ_ERR_DIM, "bad d");
    }
    SJ_LAUNCHED();
}

void free_batches(sj_result *res)
{
    for (auto &b : res->batches) {
        if (b.on_device) dev_free(b.pairs, nullptr);
        else host_pinned_free(b.pairs);
    }
    res->batches.clear();
}

}  // namespace

// ------------------------------------------------------------------ count -> plan -> fill
namespace {
// Runs the exact two-pass join of the queries described by `q` (q.q / q.qlist / q.q_index / q.self /
// q.f32 set by the caller) over ix into res: per-query counts, a batch plan of contiguous query ranges
// of <= target pairs, one fill launch per batch.  Throws SJ_ERR_NONFINITE for a non-finite query.
void probe_join(const DevIndex &ix, int dev, const ProbeArgs &q, uint64_t nq, const sj_join_opts &o,
                cudaStream_t s, sj_result *res)
{
    const uint64_t nbk = (nq + 1023) / 1024;
    // device words: [0..3) work, [3] nonfinite flag, [4] cursor, [5] overflow; then the bucket sums
    Scratch<unsigned long long> words(8 + nbk, s);
    Scratch<uint32_t> counts(nq, s);
    SJ_CUDA(cudaMemsetAsync(words.p, 0, sizeof(unsigned long long) * (8 + nbk), s));
    ProbeArgs pa = q;
    pa.q_begin = 0;
    pa.nq = (uint32_t)nq;
    pa.counts = counts.p;
    pa.buckets = words.p + 8;
    pa.nonfinite = reinterpret_cast<uint32_t *>(words.p + 3);
    pa.work = words.p;
    launch_probe(kPCount, ix, pa, dev, s);
    std::vector<unsigned long long> hw(8 + nbk);
    SJ_CUDA(cudaMemcpyAsync(hw.data(), words.p, sizeof(unsigned long long) * hw.size(), cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    if (hw[3]) fail(SJ_ERR_NONFINITE, "a query coordinate is NaN or inf");
    uint64_t total = 0;
    for (uint64_t b = 0; b < nbk; ++b) total += hw[8 + b];

    // ---- batch plan: contiguous query ranges of <= target pairs (exact counts: no overflow re-runs);
    //      at least min_batches when there is output (the paper's pipeline shape)
    uint64_t target = o.batch_capacity_pairs;
    if (o.min_batches > 1 && total) target = std::min<uint64_t>(target, (total + o.min_batches - 1) / o.min_batches);
    target = std::max<uint64_t>(target, 1);
    std::vector<uint64_t> cuts{0};
    std::vector<uint64_t> sizes;
    {
        std::vector<uint32_t> qc;     // per-query counts of a bucket larger than the target (fetched lazily)
        uint64_t acc = 0;
        for (uint64_t b = 0; b < nbk; ++b) {
            const uint64_t bq0 = b * 1024, bq1 = std::min<uint64_t>(nq, bq0 + 1024);
            if (hw[8 + b] <= target) {
                if (acc && acc + hw[8 + b] > target) { cuts.push_back(bq0); sizes.push_back(acc); acc = 0; }
                acc += hw[8 + b];
                continue;
            }
            qc.resize(bq1 - bq0);
            SJ_CUDA(cudaMemcpy(qc.data(), counts.p + bq0, sizeof(uint32_t) * qc.size(), cudaMemcpyDeviceToHost));
            for (uint64_t i = bq0; i < bq1; ++i) {
                const uint64_t c = qc[i - bq0];
                if (acc && acc + c > target) { cuts.push_back(i); sizes.push_back(acc); acc = 0; }
                acc += c;
            }
        }
        cuts.push_back(nq);
        sizes.push_back(acc);
    }

    const uint64_t w0 = hw[0], w1 = hw[1];
    SJ_CUDA(cudaMemsetAsync(words.p, 0, sizeof(unsigned long long) * 8, s));
    for (size_t b = 0; b + 1 < cuts.size(); ++b) {
        if (total && sizes[b] == 0) continue;     // an empty range between two non-empty ones
        sj_batch bt;
        bt.cap = std::max<uint64_t>(sizes[b], 1);
        bt.pairs = dalloc<uint64_t>(bt.cap, s);
        bt.on_device = 1;
        bt.n = sizes[b];
        res->batches.push_back(bt);               // owned by res from here (freed on failure)
        SJ_CUDA(cudaMemsetAsync(words.p + 4, 0, 16, s));
        ProbeArgs pf = q;
        pf.q_begin = (uint32_t)cuts[b];
        pf.nq = (uint32_t)(cuts[b + 1] - cuts[b]);
        pf.out = bt.pairs;
        pf.cursor = words.p + 4;
        pf.cap = bt.cap;
        pf.overflow = reinterpret_cast<uint32_t *>(words.p + 5);
        pf.work = nullptr;
        if (sizes[b]) launch_probe(kPFill, ix, pf, dev, s);
        if (o.sort_pairs) sort_pairs_device(bt.pairs, bt.n, res->n_points, s);
        if (o.result_on_host) {
            uint64_t *h = static_cast<uint64_t *>(host_pinned_alloc(bt.cap * 8, nullptr));
            if (bt.n) SJ_CUDA(cudaMemcpyAsync(h, bt.pairs, bt.n * 8, cudaMemcpyDeviceToHost, s));
            SJ_CUDA(cudaStreamSynchronize(s));
            dev_free(bt.pairs, s);
            res->batches.back().pairs = h;
            res->batches.back().on_device = 0;
        }
    }
    unsigned long long tail[2];
    SJ_CUDA(cudaMemcpyAsync(tail, words.p + 4, 16, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    if (tail[1]) fail(SJ_ERR_STATE, "probe join: fill pass exceeded its exact count (internal error)");
    res->total = total;
    res->stats.pairs = total;
    res->stats.estimated_pairs = total;
    res->stats.cells_probed = 2 * w0;
    res->stats.candidates_tested = 2 * w1;
    res->stats.batches = (uint32_t)res->batches.size();
    res->stats.refine_launches = (uint32_t)res->batches.size() + 1;
}

// the sampled two-set plan (the paper's estimate-then-batch scheme, PAPER.md:262 / reading R15, for
// J(Q,P)): runs of 32 consecutive sorted queries every R positions (~1.5 %, >= 4096 queries) are
// counted; each run stands for its R positions; batches of <= capacity / 1.75 estimated pairs are filled
// into buffers of 1.75x their estimate, and a batch whose cursor overflowed is counted exactly and
// filled again.  One pass over the queries instead of the exact plan's count + fill.
__global__ void k_sample_list(const uint32_t *__restrict__ qlist, uint32_t nq, uint32_t R, uint32_t nruns,
                              uint32_t *__restrict__ out)
{
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nruns * 32u; i += gridDim.x * blockDim.x) {
        const uint64_t pos = (uint64_t)(i >> 5) * R + (i & 31u);
        out[i] = qlist[pos < nq ? pos : nq - 1];
    }
}

void probe_join_sampled(const DevIndex &ix, int dev, const ProbeArgs &q, uint64_t nq, const sj_join_opts &o,
                        cudaStream_t s, sj_result *res, const uint32_t *d_nonfinite)
{
    constexpr double kMargin = 0.75;
    const uint64_t want = std::max<uint64_t>(4096, nq / 64);
    const uint64_t runs = (want + 31) / 32;
    const uint64_t R = std::max<uint64_t>(32, (nq / runs) & ~31ull);
    const uint64_t nruns = (nq + R - 1) / R;
    const uint32_t ns = (uint32_t)(nruns * 32);
    Scratch<uint32_t> slist(ns, s), scnt(ns, s);
    const uint64_t nbk = (ns + 1023) / 1024;
    Scratch<unsigned long long> words(8 + nbk, s);
    SJ_CUDA(cudaMemsetAsync(words.p, 0, sizeof(unsigned long long) * (8 + nbk), s));
    k_sample_list<<<(unsigned)std::min<uint64_t>((ns + 255) / 256, 1024), 256, 0, s>>>(q.qlist, (uint32_t)nq, (uint32_t)R,
                                                                                       (uint32_t)nruns, slist.p);
    SJ_LAUNCHED();
    ProbeArgs pa = q;
    pa.qlist = slist.p;
    pa.q_begin = 0;
    pa.nq = ns;
    pa.counts = scnt.p;
    pa.buckets = words.p + 8;
    pa.nonfinite = reinterpret_cast<uint32_t *>(words.p + 3);
    pa.work = words.p;
    launch_probe(kPCount, ix, pa, dev, s);
    std::vector<uint32_t> hc(ns);
    unsigned long long hw[8];
    uint32_t hbad = 0;
    SJ_CUDA(cudaMemcpyAsync(hc.data(), scnt.p, sizeof(uint32_t) * ns, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaMemcpyAsync(hw, words.p, sizeof hw, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaMemcpyAsync(&hbad, d_nonfinite, sizeof hbad, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    if (hbad) fail(SJ_ERR_NONFINITE, "a query coordinate is NaN or inf");
    std::vector<double> be(nruns, 0.0);
    for (uint64_t r = 0; r < nruns; ++r) {
        double c = 0;
        uint32_t v = 0;
        for (uint32_t l = 0; l < 32; ++l)
            if (r * R + l < nq) { c += hc[r * 32 + l]; ++v; }
        const uint64_t span = std::min<uint64_t>(R, nq - r * R);
        be[r] = v ? c * (double)span / (double)v : 0.0;
    }
    std::vector<uint64_t> cuts, est;
    uint64_t est_total = 0;
    plan_from_buckets(be.data(), nruns, R, 0, nq, o.batch_capacity_pairs, std::max(1, o.min_batches), kMargin, cuts,
                      est, &est_total);
    const size_t nb = cuts.size() - 1;
    // fill every batch (per-batch cursor slots), read the cursors back once, re-fill the overflowed
    Scratch<unsigned long long> cur(2 * nb + 8, s);
    SJ_CUDA(cudaMemsetAsync(cur.p, 0, sizeof(unsigned long long) * (2 * nb + 8), s));
    unsigned long long *work = cur.p + 2 * nb;
    auto fill = [&](size_t b, uint64_t cap) {
        sj_batch &bt = res->batches[b];
        bt.cap = cap;
        bt.pairs = dalloc<uint64_t>(cap, s);
        bt.on_device = 1;
        ProbeArgs pf = q;
        pf.q_begin = (uint32_t)cuts[b];
        pf.nq = (uint32_t)(cuts[b + 1] - cuts[b]);
        pf.out = bt.pairs;
        pf.cursor = cur.p + 2 * b;
        pf.cap = cap;
        pf.overflow = reinterpret_cast<uint32_t *>(cur.p + 2 * b + 1);
        pf.work = work;
        launch_probe(kPFill, ix, pf, dev, s);
    };
    res->batches.resize(nb);
    for (size_t b = 0; b < nb; ++b) {
        const uint64_t cap = std::min<uint64_t>(o.batch_capacity_pairs, (uint64_t)((double)est[b] * (1.0 + kMargin))) + 4096;
        fill(b, cap);
    }
    std::vector<unsigned long long> hcur(2 * nb);
    SJ_CUDA(cudaMemcpyAsync(hcur.data(), cur.p, sizeof(unsigned long long) * 2 * nb, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    uint32_t retries = 0;
    for (size_t b = 0; b < nb; ++b) {
        if (hcur[2 * b] > res->batches[b].cap) {          // overflowed: the cursor kept the exact count
            const uint64_t exact = hcur[2 * b];
            dev_free(res->batches[b].pairs, s);
            res->batches[b].pairs = nullptr;
            SJ_CUDA(cudaMemsetAsync(cur.p + 2 * b, 0, 16, s));
            fill(b, exact);
            ++retries;
        }
        res->batches[b].n = hcur[2 * b];
    }
    if (retries) {
        std::vector<unsigned long long> h2(2 * nb);
        SJ_CUDA(cudaMemcpyAsync(h2.data(), cur.p, sizeof(unsigned long long) * 2 * nb, cudaMemcpyDeviceToHost, s));
        SJ_CUDA(cudaStreamSynchronize(s));
        for (size_t b = 0; b < nb; ++b)
            if (h2[2 * b] > res->batches[b].cap) fail(SJ_ERR_STATE, "two-set join: exact re-fill overflowed (internal error)");
    }
    uint64_t total = 0;
    for (size_t b = 0; b < nb; ++b) {
        sj_batch &bt = res->batches[b];
        total += bt.n;
        if (o.sort_pairs) sort_pairs_device(bt.pairs, bt.n, res->n_points, s);
        if (o.result_on_host) {
            uint64_t *h = static_cast<uint64_t *>(host_pinned_alloc(std::max<uint64_t>(bt.n, 1) * 8, nullptr));
            if (bt.n) SJ_CUDA(cudaMemcpyAsync(h, bt.pairs, bt.n * 8, cudaMemcpyDeviceToHost, s));
            SJ_CUDA(cudaStreamSynchronize(s));
            dev_free(bt.pairs, s);
            bt.pairs = h;
            bt.on_device = 0;
            bt.cap = std::max<uint64_t>(bt.n, 1);
        }
    }
    unsigned long long hwk[3];
    SJ_CUDA(cudaMemcpyAsync(hwk, work, sizeof hwk, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    res->total = total;
    res->stats.pairs = total;
    res->stats.estimated_pairs = est_total;
    res->stats.cells_probed = hw[0] + hwk[0];
    res->stats.candidates_tested = hw[1] + hwk[1];
    res->stats.batches = (uint32_t)nb;
    res->stats.retries = retries;
    res->stats.refine_launches = (uint32_t)(nb + retries + 1);
}
}  // namespace

// ------------------------------------------------------------------ two-set join
sj_result *join_sets_impl(const sj_index *idx, const double *queries, uint64_t nq, int queries_on_device,
                          const sj_join_opts &o)
{
    if (!idx) fail(SJ_ERR_STATE, "index is NULL");
    if (nq >= (1ull << 32)) fail(SJ_ERR_ARG, "the number of queries must be < 2^32");
    if (nq && !queries) fail(SJ_ERR_ARG, "queries is NULL");
    if (o.batch_capacity_pairs == 0) fail(SJ_ERR_ARG, "batch_capacity_pairs must be > 0");
    if (o.drain_csr) fail(SJ_ERR_ARG, "drain_csr is not supported by the two-set join");
    const DevIndex &ix = idx->dev;
    const int dev = idx->device;
    SJ_CUDA(cudaSetDevice(dev));
    CtxGuard cg{acquire_ctx(dev, 1, 2, 64)};
    cudaStream_t s = cg.c->streams[0];
    // ordered after the caller's work on the legacy default stream (e.g. torch producing Q)
    SJ_CUDA(cudaEventRecord(cg.c->events[1], cudaStreamLegacy));
    SJ_CUDA(cudaStreamWaitEvent(s, cg.c->events[1], 0));
    const int D = ix.d;
    const double *qd = queries;
    Scratch<double> qcopy;
    if (nq && !queries_on_device) {
        qcopy.p = dalloc<double>(nq * D, s);
        qcopy.s = s;
        SJ_CUDA(cudaMemcpyAsync(qcopy.p, queries, sizeof(double) * nq * D, cudaMemcpyHostToDevice, s));
        qd = qcopy.p;
    }
    sj_result *res = new sj_result();
    res->device = dev;
    res->n_points = std::max<uint64_t>(nq, ix.n);
    res->q0 = 0;
    res->q1 = nq;
    res->include_self = 1;
    res->unicomp = 0;
    res->two_set = 1;
    try {
        ProbeArgs q{};
        q.q = qd;
        // queries sorted by their cell in P's grid (LSD radix sort of (key, row)): neighbouring queries
        // share neighbour cells (L2 reuse) and a warp of one populous cell shares candidate tiles
        Scratch<uint64_t> qk(nq, s), qk2(nq, s);
        Scratch<uint32_t> qv(nq, s), qv2(nq, s), bad(1, s);
        SJ_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(uint32_t), s));
        if (nq) {
            // keys < prod |g_j| <= 2^key_bits; the sentinel 2^key_bits (all ones at 64 bits) sorts last
            const int kb = std::min(64, idx->view.key_bits + 1);
            const uint64_t sentinel = idx->view.key_bits >= 64 ? ~0ull : (1ull << idx->view.key_bits);
            const unsigned g = (unsigned)std::min<uint64_t>((nq + 255) / 256, (uint64_t)device_sm_count(dev) * 8);
            switch (D) {
            case 2: k_qkeys<2><<<g, 256, 0, s>>>(ix, qd, (uint32_t)nq, sentinel, qk.p, qv.p, bad.p); break;
            case 3: k_qkeys<3><<<g, 256, 0, s>>>(ix, qd, (uint32_t)nq, sentinel, qk.p, qv.p, bad.p); break;
            case 4: k_qkeys<4><<<g, 256, 0, s>>>(ix, qd, (uint32_t)nq, sentinel, qk.p, qv.p, bad.p); break;
            case 5: k_qkeys<5><<<g, 256, 0, s>>>(ix, qd, (uint32_t)nq, sentinel, qk.p, qv.p, bad.p); break;
            default: k_qkeys<6><<<g, 256, 0, s>>>(ix, qd, (uint32_t)nq, sentinel, qk.p, qv.p, bad.p); break;
            }
            SJ_LAUNCHED();
            bool in_tmp = false;
            radix_sort_pairs(qk.p, qv.p, qk2.p, qv2.p, (uint32_t)nq, kb, s, &in_tmp);
            q.qlist = in_tmp ? qv2.p : qv.p;
            q.tiled = 1;
        }
        // large query sets: the sampled plan (one pass); small ones: exact counts (cheap, no re-runs)
#ifndef SJ_SETS_SAMPLE_MIN
#define SJ_SETS_SAMPLE_MIN 65536
#endif
        if (nq >= SJ_SETS_SAMPLE_MIN) probe_join_sampled(ix, dev, q, nq, o, s, res, bad.p);
        else probe_join(ix, dev, q, nq, o, s, res);
    } catch (...) {
        cudaStreamSynchronize(s);
        free_batches(res);
        delete res;
        throw;
    }
    return res;
}

// ------------------------------------------------------------------ FP32 self-join
namespace {
__global__ void k_f32_to_f64(const float *__restrict__ in, double *__restrict__ out, uint64_t m)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = (double)in[i];
}
}  // namespace

sj_result *self_join_f32_impl(const float *points, uint64_t n, int d, float eps, const sj_build_opts &bo,
                              const sj_join_opts &o)
{
    if (d < 2 || d > SJ_MAX_DIM) fail(SJ_ERR_DIM, "d must be in [2,6]");
    if (!points) fail(SJ_ERR_ARG, "points is NULL");
    if (n == 0 || n >= (1ull << 32)) fail(SJ_ERR_ARG, "N must satisfy 1 <= N < 2^32");
    if (!std::isfinite(eps) || !(eps > 0.0f)) fail(SJ_ERR_ARG, "eps must be finite and > 0");
    volatile float e2v = eps * eps;              // fl32(eps*eps)
    const float eps2f = e2v;
    if (!std::isnormal(eps2f)) fail(SJ_ERR_ARG, "fl32(eps*eps) must be a normal float");
    if (bo.device < 0 || bo.device >= device_count()) fail(SJ_ERR_ARG, "bad device ordinal");
    SJ_CUDA(cudaSetDevice(bo.device));
    CtxGuard cg{acquire_ctx(bo.device, 1, 2, 64)};
    cudaStream_t s = cg.c->streams[0];
    SJ_CUDA(cudaEventRecord(cg.c->events[1], cudaStreamLegacy));
    SJ_CUDA(cudaStreamWaitEvent(s, cg.c->events[1], 0));
    // the points widened to binary64 (exact) for the grid index
    const uint64_t m = n * (uint64_t)d;
    Scratch<float> fcopy;
    const float *fp = points;
    if (!bo.points_on_device) {
        fcopy.p = dalloc<float>(m, s);
        fcopy.s = s;
        SJ_CUDA(cudaMemcpyAsync(fcopy.p, points, sizeof(float) * m, cudaMemcpyHostToDevice, s));
        fp = fcopy.p;
    }
    Scratch<double> wide(m, s);
    k_f32_to_f64<<<(unsigned)std::min<uint64_t>((m + 255) / 256, (uint64_t)device_sm_count(bo.device) * 8), 256, 0, s>>>(
        fp, wide.p, m);
    SJ_LAUNCHED();
    // R21: the float predicate can accept a pair whose exact distance exceeds eps by a relative
    // (d + 3) * 2^-24 at most; a grid for eps * (1 + 2^-16) keeps every such pair in adjacent cells
    sj_build_opts b2 = bo;
    b2.points_on_device = 1;
    b2.stream = s;
    b2.speculative_estimate = 0;
    sj_index *idx = build_index_impl(wide.p, n, d, (double)eps * (1.0 + std::ldexp(1.0, -16)), b2);
    // the self-join's whole path (estimate, plan, batches, unicomp -- the binary32 distance is symmetric
    // too --, sparse / dense / queued refine kernels, host drain, CSR) with the predicate in binary32
    idx->dev.f32 = 1;
    idx->dev.eps2f = eps2f;
    sj_result *res = nullptr;
    try {
        SJ_CUDA(cudaStreamSynchronize(s));      // the widened copy is read by the build only
        res = self_join_impl(idx, o);
    } catch (...) {
        free_index_impl(idx);
        throw;
    }
    free_index_impl(idx);
    return res;
}

// ------------------------------------------------------------------ kNN self-join
namespace {
__global__ void k_nonfinite(const double *__restrict__ a, uint64_t m, uint32_t *__restrict__ flag)
{
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        if (!isfinite(a[i])) atomicOr(flag, 1u);
}
}  // namespace

// kNN over the growing-radius grid (R20): queries == nullptr is the self join (queries = the points,
// each excluding itself); otherwise nq query rows against the n points, nothing excluded.
void knn_impl(const double *points, uint64_t n, const double *queries, uint64_t nq, int d, uint32_t k, double eps0,
              const sj_build_opts &bo, uint32_t *ids, double *dist2, sj_knn_stats *st)
{
    const bool self = queries == nullptr;
    if (self) nq = n;
    if (d < 2 || d > SJ_MAX_DIM) fail(SJ_ERR_DIM, "d must be in [2,6]");
    if (!points || (nq && (!ids || !dist2))) fail(SJ_ERR_ARG, "points / ids / dist2 is NULL");
    if (k < 1 || k > (uint32_t)kMaxK) fail(SJ_ERR_ARG, "k must be in [1, 32]");
    if (n < (uint64_t)k + (self ? 1 : 0) || n >= (1ull << 32))
        fail(SJ_ERR_ARG, self ? "N must satisfy k + 1 <= N < 2^32" : "N must satisfy k <= N < 2^32");
    if (nq >= (1ull << 32)) fail(SJ_ERR_ARG, "the number of queries must be < 2^32");
    if (!std::isfinite(eps0) || !(eps0 > 0.0)) fail(SJ_ERR_ARG, "eps0 must be finite and > 0");
    if (bo.device < 0 || bo.device >= device_count()) fail(SJ_ERR_ARG, "bad device ordinal");
    SJ_CUDA(cudaSetDevice(bo.device));
    CtxGuard cg{acquire_ctx(bo.device, 1, 2, 64)};
    cudaStream_t s = cg.c->streams[0];
    SJ_CUDA(cudaEventRecord(cg.c->events[1], cudaStreamLegacy));
    SJ_CUDA(cudaStreamWaitEvent(s, cg.c->events[1], 0));
    const double *pd = points;
    Scratch<double> pcopy;
    if (!bo.points_on_device) {
        pcopy.p = dalloc<double>(n * d, s);
        pcopy.s = s;
        SJ_CUDA(cudaMemcpyAsync(pcopy.p, points, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
        pd = pcopy.p;
    }
    const double *qd = pd;
    Scratch<double> qcopy;
    Scratch<unsigned long long> words(8, s);
    if (!self) {
        qd = queries;
        if (nq && !bo.points_on_device) {
            qcopy.p = dalloc<double>(nq * d, s);
            qcopy.s = s;
            SJ_CUDA(cudaMemcpyAsync(qcopy.p, queries, sizeof(double) * nq * d, cudaMemcpyHostToDevice, s));
            qd = qcopy.p;
        }
        // a non-finite query would never be certified: rejected up front
        SJ_CUDA(cudaMemsetAsync(words.p, 0, 8, s));
        if (nq) {
            k_nonfinite<<<(unsigned)std::min<uint64_t>((nq * d + 255) / 256, 4096), 256, 0, s>>>(
                qd, nq * d, reinterpret_cast<uint32_t *>(words.p));
            SJ_LAUNCHED();
        }
        uint32_t bad = 0;
        SJ_CUDA(cudaMemcpyAsync(&bad, words.p, sizeof bad, cudaMemcpyDeviceToHost, s));
        SJ_CUDA(cudaStreamSynchronize(s));
        if (bad) fail(SJ_ERR_NONFINITE, "a query coordinate is NaN or inf");
    }
    Scratch<uint32_t> unres[2] = {Scratch<uint32_t>(nq, s), Scratch<uint32_t>(nq, s)};
    sj_build_opts b2 = bo;
    b2.points_on_device = 1;
    b2.stream = s;
    b2.speculative_estimate = 0;
    double eps = eps0;
    // radius growth per round: the 3^d neighbourhood's volume x SJ_KNN_GROW_VOL (a doubling of eps
    // multiplies a 6-D neighbourhood's candidates by 64 for the few uncertified -- mostly boundary --
    // queries); the certificate does not depend on the schedule
#ifndef SJ_KNN_GROW_VOL
#define SJ_KNN_GROW_VOL 4.0
#endif
    const double grow = std::max(1.1, std::pow(SJ_KNN_GROW_VOL, 1.0 / d));
    uint64_t pending = nq, probes = 0, tests = 0;
    uint32_t rounds = 0;
    int cur = 0;
    while (pending) {
        if (++rounds > 400) fail(SJ_ERR_STATE, "kNN: not certified after 400 radius steps");
        sj_index *idx = build_index_impl(pd, n, d, eps, b2);
        try {
            SJ_CUDA(cudaMemsetAsync(words.p, 0, sizeof(unsigned long long) * 8, s));
            ProbeArgs pa{};
            pa.q = qd;
            // first self round: every point, in the index's A-order (coalesced, cell-sorted)
            pa.q_index = self && rounds == 1;
            pa.qlist = rounds == 1 ? nullptr : unres[cur].p;
            pa.q_begin = 0;
            pa.nq = (uint32_t)pending;
            pa.self = self ? 1 : 0;
            pa.k = k;
            pa.ids = ids;
            pa.dist2 = dist2;
            pa.unres = unres[cur ^ 1].p;
            pa.n_unres = reinterpret_cast<uint32_t *>(words.p + 4);
            pa.work = words.p;
            launch_probe(kPKnn, idx->dev, pa, bo.device, s);
            unsigned long long hw[5];
            SJ_CUDA(cudaMemcpyAsync(hw, words.p, sizeof hw, cudaMemcpyDeviceToHost, s));
            SJ_CUDA(cudaStreamSynchronize(s));
            probes += hw[0];
            tests += hw[1];
            pending = (uint32_t)hw[4];
        } catch (...) {
            free_index_impl(idx);
            throw;
        }
        free_index_impl(idx);
        cur ^= 1;
        if (pending) eps *= grow;
    }
    if (st) {
        st->rounds = rounds;
        st->eps_final = eps;
        st->cells_probed = probes;
        st->candidates_tested = tests;
    }
}

void knn_self_impl(const double *points, uint64_t n, int d, uint32_t k, double eps0, const sj_build_opts &bo,
                   uint32_t *ids, double *dist2, sj_knn_stats *st)
{
    knn_impl(points, n, nullptr, 0, d, k, eps0, bo, ids, dist2, st);
}

}  // namespace sj
