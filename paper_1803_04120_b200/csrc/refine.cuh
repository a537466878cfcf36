// refine.cuh -- the refine kernel (steps a5-a7 of the hot path).
//
// PAPER.md §4.5 Alg. 1 (lines 216-251, GPUSelfJoinGlobal): queries in A-order (the cell-sorted
// order, so neighbouring queries share cells and index prefixes); each query holds its point in
// registers (Alg. 1 l.4), finds its home cell, enumerates the adjacent cells (l.5-10), looks each
// up in B (l.11) and tests the points of every non-empty one (l.12-16).  With unicomp (PAPER.md
// §5.2, Alg. 2, readings R10-R13) a neighbour cell is searched only when the query's
// coordinate in the highest differing dimension is odd, and every hit is emitted in both
// orientations; the home cell emits (p,p) once plus, for every q after p in
// A-order, both (p,q) and (q,p).
//
// B200-specific design:
//  * G lanes per query (G = 1..32, power of two, chosen per index from the expected work): the
//    lanes of a group split the query's top-prefix offsets (cell-scan mode), rows (row modes) and
//    home-cell points, so a warp stays converged even when per-query work varies (a 6-D eps=8
//    join ran with 7 of 32 lanes active at G=1).
//  * bounded search through the prefix directory: the cells sharing their top-k coordinates form
//    one contiguous range of B, dir[p] gives it in O(1), and every search is bounded to it.
//    Three modes (index_build.cu): dense rows (k = d), cell scan (few cells per prefix: test the
//    low coordinates greedily on the key difference) and rows (bounded binary search per row of
//    three consecutive ids = one contiguous A-range).
//  * per-CTA shared-memory table of the top-prefix offsets: unicomp / mask decisions per offset
//    are two bit tests.
//  * the distance s = (((x_0-y_0)^2 + (x_1-y_1)^2) + ...) with __dsub_rn/__dmul_rn/__dadd_rn (no FMA
//    contraction possible) compared with fl(eps^2): bit-identical decisions to the oracle (R1, R2).
//  * warp-aggregated emission: __ballot_sync of the hits, __popc, ONE atomicAdd per warp on the
//    batch cursor, __shfl_sync of the base; each hitting lane writes its 1 or 2 packed pairs.
//    Writes past the batch capacity are dropped and flag an overflow; the cursor keeps counting
//    so the host learns the exact size and re-runs the batch.
//  * every search loop is rolled and the candidate loop is inlined at four call sites only,
//    keeping the kernel ~3 K SASS (an unrolled version measured 28 K SASS, 47% no_inst stalls).
#pragma once

#include "sj_common.cuh"

namespace sj {

enum RefineMode { kEmit = 0, kCountQuery = 1, kCountPoint = 2 };
// mode flag: the predicate in binary32 (FP32 self-join, R21: coordinates are floats widened
// exactly, s32 = (((x0-y0)^2 + (x1-y1)^2) + ...) in float with __fsub_rn/__fmul_rn/__fadd_rn, <= eps2f)
constexpr int kModeMask = 3;
constexpr int kF32 = 8;

struct JoinArgs {
    uint64_t *out;                 // kEmit: batch pair buffer
    unsigned long long *cursor;    // kEmit: pairs emitted (exact even on overflow)
    uint64_t cap;                  // kEmit: capacity of out
    uint32_t *overflow;            // kEmit: set when a write was dropped
    unsigned long long *qbucket;   // kCountQuery: emissions summed per planning bucket (t / group)
    uint32_t group;                // kCountQuery: samples per bucket
    uint32_t *pcount;              // kCountPoint: cnt[original id]
    unsigned long long *work;      // [0] directory/row lookups, [1] distance tests, [2] emissions
    uint32_t q0, q1;               // A-position range of the queries
    uint32_t step, nsamples;       // kCountQuery: sample t = query q0 + (t/32)*32*step + t%32
    uint32_t lanes_log2;           // G = 1 << lanes_log2 lanes cooperate on one query
    uint32_t dense_T;              // kEmit: queries of cells with >= dense_T points go to the
                                   // warp-per-task dense kernel (0 = off)
    const uint32_t *dense_tasks;   // start A-position of each dense task (<= 32 queries of a cell)
    uint32_t n_dense_tasks;
    int include_self;
    int use_masks;
    uint32_t nself;                // kEmit: self pairs of the batch (q1 - q0 if include_self, else 0):
                                   // query k's (p,p) sits at out[k - q0], every other pair after them
};

// Per-warp shared memory of the dense kernel: the emission ring (hits are appended once per
// 32-candidate tile) and the candidate tile (the coordinates of 32 consecutive A-positions in SoA
// form, tx[j*32 + e], and their original ids), loaded coalesced by the warp and read back as
// broadcasts by every query lane.
// The ring holds kWarpBufPairs pairs between the counters head <= tail (ring slot = counter mod
// kWarpBufPairs).  Output space is reserved AHEAD: once half the ring is filled, the leader issues
// the atomicAdd on the batch cursor for [head, tail) and the warp goes on testing candidates; the
// reserved pairs are written out only when the ring needs the room (usually one tile later), so
// the round trip of that atomic -- contended by every warp of the launch -- is off the warp's
// critical path (ncu: 23% of the dense kernel's stall samples sat on the flush's shuffle of the
// returned base).  Every reservation covers exactly the pairs it is for, so the batch stays dense.
#ifndef SJ_RING
#define SJ_RING 1024
#endif
constexpr int kWarpBufPairs = SJ_RING;   // power of two >= 512
struct WarpBuf {
    uint64_t *buf;        // [kWarpBufPairs] ring in shared memory
    double *tx;           // [D][32] candidate tile (SoA)
    uint32_t *tid;        // [32] original ids of the tile's candidates
    uint32_t head, tail;  // warp-uniform ring counters
    uint32_t pend;        // pairs [head, head + pend) are reserved, their base in `base` (leader)
    unsigned long long base;
};
// dynamic shared memory of k_refine_dense<D>: per warp the pair buffer, the SoA tile and the ids
template <int D>
__host__ __device__ constexpr size_t dense_smem_per_warp() { return sizeof(uint64_t) * kWarpBufPairs + sizeof(double) * 32 * D + 4 * 32; }

constexpr int kRefineThreads = 256;
#ifndef SJ_REFINE_MIN_BLOCKS
#define SJ_REFINE_MIN_BLOCKS 5
#endif
constexpr int kRefineMinBlocks = SJ_REFINE_MIN_BLOCKS;  // 5 x 256 threads: <= 51 registers (measured best once the query state left the stack: 6-D eps=1 span 0.192 -> 0.180 ms)

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
    uint32_t sub, G;   // this lane's rank in the query's group, group size
    bool valid;        // dense kernel: false for helper lanes past the task's end (never emit)
    uint32_t emitted;  // pairs emitted by this lane
    uint32_t probes;   // directory / row lookups
    uint32_t tests;    // distance evaluations
};

template <int MODE, bool BOTH>
__device__ __forceinline__ void emit(const JoinArgs &ja, bool hit, uint32_t pid, uint32_t qid, uint32_t &emitted)
{
    if constexpr ((MODE & kModeMask) == kCountQuery) {
        if (hit) emitted += BOTH ? 2u : 1u;
        return;
    } else if constexpr ((MODE & kModeMask) == kCountPoint) {
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
            const unsigned long long pos = ja.nself + base + (unsigned long long)(__popc(hits & ((1u << lane) - 1u)) * per);
            if (pos + per <= ja.cap) {
                ja.out[pos] = ((uint64_t)pid << 32) | qid;
                if (BOTH) ja.out[pos + 1] = ((uint64_t)qid << 32) | pid;
            } else {
                atomicOr(ja.overflow, 1u);
            }
        }
    }
}

// The self pair (p,p) of query k (reading R3): in kEmit mode its slot is fixed, out[k - q0], so it
// needs no cursor atomic (one same-address atomic per warp serialised in L2 on sparse data).
template <int MODE>
__device__ __forceinline__ void emit_self(const JoinArgs &ja, uint32_t k, uint32_t pid, uint32_t &emitted)
{
    if constexpr ((MODE & kModeMask) == kEmit) {
        const uint64_t pos = (uint64_t)(k - ja.q0);
        if (pos < ja.cap) ja.out[pos] = ((uint64_t)pid << 32) | pid;
        else atomicOr(ja.overflow, 1u);
        ++emitted;
    } else {
        emit<MODE, false>(ja, true, pid, pid, emitted);
    }
}

// Write the ring's pairs [head, head + len) to the batch at p0 (all 32 lanes).  16-byte streaming
// stores when both ends are even (the pairs are not read again by the join; the index stays in L2),
// as (at most) two contiguous runs of the ring.
__device__ __forceinline__ void ring_write(const JoinArgs &ja, const WarpBuf &wb, uint32_t head, uint32_t len,
                                           unsigned long long p0)
{
    constexpr uint32_t R = (uint32_t)kWarpBufPairs;
    const uint32_t lane = threadIdx.x & 31u;
    if (p0 + len <= ja.cap && !((p0 | len | head) & 1ull)) {
        const uint32_t h2 = (head & (R - 1)) >> 1, n2 = len >> 1;
        const uint32_t first = min(n2, R / 2 - h2);              // 16-byte units before the wrap
        const ulonglong2 *src = reinterpret_cast<const ulonglong2 *>(wb.buf);
        ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(ja.out + p0);
        for (uint32_t i = lane; i < first; i += 32u) __stcs(dst + i, src[h2 + i]);
        for (uint32_t i = lane; i < n2 - first; i += 32u) __stcs(dst + first + i, src[i]);
    } else {
        for (uint32_t i = lane; i < len; i += 32u) {
            const unsigned long long pos = p0 + i;
            if (pos < ja.cap) __stcs(reinterpret_cast<unsigned long long *>(ja.out + pos), wb.buf[(head + i) & (R - 1)]);
            else atomicOr(ja.overflow, 1u);
        }
    }
}

// Write out the reserved pairs (waits for the reservation's atomic only now).
__device__ __forceinline__ void ring_retire(const JoinArgs &ja, WarpBuf &wb)
{
    if (!wb.pend) return;
    const unsigned long long base = __shfl_sync(0xffffffffu, wb.base, 0);
    ring_write(ja, wb, wb.head, wb.pend, ja.nself + base);
    wb.head += wb.pend;
    wb.pend = 0;
}

// Reserve output space for everything not yet reserved (asynchronous: the result is consumed by
// ring_retire).  ATOM issued by lane 0.
__device__ __forceinline__ void ring_reserve(const JoinArgs &ja, WarpBuf &wb)
{
    const uint32_t len = wb.tail - wb.head;
    if (wb.pend || !len) return;
    if ((threadIdx.x & 31u) == 0) wb.base = atomicAdd(ja.cursor, (unsigned long long)len);
    wb.pend = len;
}

// Empty the ring (end of the kernel, or a unit that needs more room than retiring frees).
__device__ __forceinline__ void ring_drain(const JoinArgs &ja, WarpBuf &wb)
{
    ring_retire(ja, wb);
    ring_reserve(ja, wb);
    ring_retire(ja, wb);
    __syncwarp();
}

// Emission of one 32-candidate tile of the dense kernel: lane = query, bit e of hm = candidate e of
// the tile (id wb.tid[e]) is a hit.  One warp prefix sum places every lane's pairs in the ring (no
// per-candidate ballot); each lane then writes its hits, (p,q) and (q,p) as one 16-byte store when
// BOTH.  A tile yields at most 32*32*per pairs; one that does not fit the ring (> kWarpBufPairs, only
// with BOTH and > 50% hits) is emitted in two halves of 16 candidates.
template <bool BOTH>
__device__ __forceinline__ void emit_tile(const JoinArgs &ja, WarpBuf &wb, uint32_t hm, uint32_t pid,
                                          uint32_t &emitted)
{
    constexpr uint32_t per = BOTH ? 2u : 1u;
    constexpr uint32_t R = (uint32_t)kWarpBufPairs;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(wb.buf);
    // chunks of cw candidates, each fitting the ring: 32, else 16 if both halves fit, else 8 (a chunk
    // of 8 yields <= 32 * 8 * per <= 512 pairs)
    uint32_t cw = 32;
    {
        const uint32_t t = __reduce_add_sync(0xffffffffu, __popc(hm) * per);
        if (t == 0u) return;
        if (t > R) {
            const uint32_t tlo = __reduce_add_sync(0xffffffffu, __popc(hm & 0xFFFFu) * per);
            cw = (tlo <= R && t - tlo <= R) ? 16u : 8u;
        }
    }
#pragma unroll 1
    for (uint32_t c = 0; c < 32u; c += cw) {
        uint32_t m = cw == 32u ? hm : hm & (((1u << cw) - 1u) << c);
        const uint32_t n = __popc(m) * per;
        const uint32_t total = __reduce_add_sync(0xffffffffu, n);
        if (total == 0u) continue;
        uint32_t inc = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += t;
        }
        if (wb.tail - wb.head + total > R) {             // make room: the reserved part first
            ring_retire(ja, wb);
            if (wb.tail - wb.head + total > R) ring_drain(ja, wb);
            __syncwarp();
        }
        // byte offset into the ring (wraps with one AND: the ring is 8 KB); two hits per iteration
        uint32_t pb = (wb.tail + inc - n) << 3;
        const uint32_t stid = (uint32_t)__cvta_generic_to_shared(wb.tid);
        emitted += n;
        constexpr uint32_t kStep = per * 8u;
        while (m) {
            uint32_t e1, e2;
            asm("bfind.u32 %0, %1;" : "=r"(e1) : "r"(m));
            m ^= 1u << e1;
            const bool two = m != 0u;
            asm("bfind.u32 %0, %1;" : "=r"(e2) : "r"(m));   // 0xffffffff when m == 0 (unused then)
            if (two) m ^= 1u << e2;
            uint32_t q1, q2;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(q1) : "r"(stid + 4u * e1));
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(q2) : "r"(stid + 4u * (e2 & 31u)));
            const uint32_t a1 = sbuf + (pb & (R * 8u - 1u)), a2 = sbuf + ((pb + kStep) & (R * 8u - 1u));
            if constexpr (BOTH) {
                // (p,q) = {q, p} and (q,p) = {p, q} as little-endian 32-bit words
                asm volatile("st.shared.v4.u32 [%0], {%1, %2, %2, %1};" ::"r"(a1), "r"(q1), "r"(pid) : "memory");
                if (two) asm volatile("st.shared.v4.u32 [%0], {%1, %2, %2, %1};" ::"r"(a2), "r"(q2), "r"(pid) : "memory");
            } else {
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a1), "r"(q1), "r"(pid) : "memory");
                if (two) asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a2), "r"(q2), "r"(pid) : "memory");
            }
            pb += two ? 2u * kStep : kStep;
        }
        __syncwarp();
        wb.tail += total;
        if (wb.tail - wb.head >= R / 2) ring_reserve(ja, wb);
    }
}

// Test the points at A-positions m0, m0+stride, ... < m1 against the query.
// DENSE (dense kernel): the loop bounds are warp-uniform; HOME selects the home-cell predicate
// (unicomp: m > k; full: m != k) and hits go to the per-warp buffer.
template <int D, int MODE, bool BOTH, bool DENSE = false, bool HOME = false>
__device__ __forceinline__ void scan_range(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q, uint32_t m0,
                                           uint32_t m1, uint32_t stride, WarpBuf *wb = nullptr,
                                           unsigned wmask = 0u)
{
    const uint32_t n = ix.n;
    if constexpr (DENSE) {
        // all 32 lanes are active here (helper lanes included).  Tiles of 32 candidates: lane e loads
        // candidate g+e (coalesced SoA reads of X) into the warp's shared-memory tile; every query
        // lane then tests the whole tile reading two candidates per 16-byte broadcast load per
        // dimension, collects a 32-bit hit mask, and the tile is emitted at once (emit_tile).
        // The next tile's loads are issued before the current tile is tested (software pipelining:
        // their L2/DRAM latency hides behind the tile's FP64 work).
        const uint32_t lane = threadIdx.x & 31u;
        double nx[D];
        uint32_t nid = 0;
        if (m0 + lane < m1) {
#pragma unroll
            for (int j = 0; j < D; ++j) nx[j] = __ldg(ix.X + (uint64_t)j * n + m0 + lane);
            nid = __ldg(ix.A + m0 + lane);
        }
#pragma unroll 1
        for (uint32_t g = m0; g < m1; g += 32u) {
            __syncwarp();                                   // the previous tile is consumed
            if (g + lane < m1) {
#pragma unroll
                for (int j = 0; j < D; ++j) wb->tx[j * 32 + lane] = nx[j];
                wb->tid[lane] = nid;
            }
            const uint32_t nxt = g + 32u + lane;
            if (nxt < m1) {
#pragma unroll
                for (int j = 0; j < D; ++j) nx[j] = __ldg(ix.X + (uint64_t)j * n + nxt);
                nid = __ldg(ix.A + nxt);
            }
            __syncwarp();
            const uint32_t lim = min(32u, m1 - g);
            // candidates this lane must test: e < lim, a real query, and the home-cell rule
            uint32_t vm = lim == 32u ? 0xffffffffu : ((1u << lim) - 1u);
            if (!q.valid) vm = 0u;
            if (HOME && q.k >= g) {
                const uint32_t r = q.k - g;                 // the query's own position in the tile
                if (BOTH) vm &= r >= 31u ? 0u : ~((2u << r) - 1u);   // unicomp: only m > k
                else if (r < 32u) vm &= ~(1u << r);                  // full: every m != k
            }
            q.tests += __popc(vm);
            uint32_t hm = 0u;
            const double2 *t2 = reinterpret_cast<const double2 *>(wb->tx);
            const uint32_t npair = (lim + 1u) >> 1;         // warp-uniform
            // fully unrolled (constant bit positions: the hit bit is one predicated OR); the
            // ragged last tile of a range leaves early by a uniform branch
            if constexpr ((MODE & kF32) != 0) {
#pragma unroll
                for (uint32_t e2 = 0; e2 < 16u; ++e2) {
                    if (e2 >= npair) break;
                    double2 c = t2[e2];
                    float ta = __fsub_rn((float)q.x[0], (float)c.x), tb = __fsub_rn((float)q.x[0], (float)c.y);
                    float sa = __fmul_rn(ta, ta), sb = __fmul_rn(tb, tb);
#pragma unroll
                    for (int j = 1; j < D; ++j) {
                        c = t2[j * 16 + e2];
                        ta = __fsub_rn((float)q.x[j], (float)c.x);
                        tb = __fsub_rn((float)q.x[j], (float)c.y);
                        sa = __fadd_rn(sa, __fmul_rn(ta, ta));
                        sb = __fadd_rn(sb, __fmul_rn(tb, tb));
                    }
                    if (sa <= ix.eps2f) hm |= 1u << (2u * e2);
                    if (sb <= ix.eps2f) hm |= 2u << (2u * e2);
                }
                emit_tile<BOTH>(ja, *wb, hm & vm, q.pid, q.emitted);
                continue;
            }
#pragma unroll
            for (uint32_t e2 = 0; e2 < 16u; ++e2) {
                if (e2 >= npair) break;
                double2 c = t2[e2];                         // dim 0 of candidates 2e2, 2e2+1
                double ta = __dsub_rn(q.x[0], c.x), tb = __dsub_rn(q.x[0], c.y);
                double sa = __dmul_rn(ta, ta), sb = __dmul_rn(tb, tb);
#pragma unroll
                for (int j = 1; j < D; ++j) {
                    c = t2[j * 16 + e2];
                    ta = __dsub_rn(q.x[j], c.x);
                    tb = __dsub_rn(q.x[j], c.y);
                    sa = __dadd_rn(sa, __dmul_rn(ta, ta));
                    sb = __dadd_rn(sb, __dmul_rn(tb, tb));
                }
                if (sa <= ix.eps2) hm |= 1u << (2u * e2);
                if (sb <= ix.eps2) hm |= 2u << (2u * e2);
            }
            emit_tile<BOTH>(ja, *wb, hm & vm, q.pid, q.emitted);
        }
        return;
    }
    for (uint32_t m = m0; m < m1; m += stride) {
        bool hit;
        if constexpr ((MODE & kF32) != 0) {
            float s;
            {
                const float t = __fsub_rn((float)q.x[0], (float)__ldg(ix.X + m));
                s = __fmul_rn(t, t);
            }
#pragma unroll
            for (int j = 1; j < D; ++j) {
                const float t = __fsub_rn((float)q.x[j], (float)__ldg(ix.X + (uint64_t)j * n + m));
                s = __fadd_rn(s, __fmul_rn(t, t));
            }
            hit = s <= ix.eps2f;
        } else {
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
            hit = s <= ix.eps2;
        }
        ++q.tests;
        uint32_t qid = 0;
        if ((MODE & kModeMask) != kCountQuery && hit) qid = __ldg(ix.A + m);
        emit<MODE, BOTH>(ja, hit, q.pid, qid, q.emitted);
    }
}

// Offsets of the top-k (directory) dimensions, precomputed once per CTA in shared memory:
// for t in [0, 3^k): prefix delta, key delta, and bit masks of the dims moved by -1 / +1 and of
// the highest moved dim (unicomp decision).  3^k <= 243 in the cell-scan mode.
constexpr int kMaxTop = 243;
struct TopTable {
    int64_t dp[kMaxTop];     // sum delta_i * pstride_i
    int64_t dk[kMaxTop];     // dp * dir_div (key delta)
    int64_t dq[kMaxTop];     // dp * occ_cpd (occupancy-bitmap index delta)
    int64_t dq2[kMaxTop];    // dp * occ2_cpd (second bitmap)
    uint32_t bits[kMaxTop];  // [0:6) dims at -1, [8:14) dims at +1, [16:22) one-hot highest moved dim
};

__device__ __forceinline__ uint32_t kPow3i(int e)
{
    uint32_t r = 1;
    for (int i = 0; i < e; ++i) r *= 3u;
    return r;
}

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
        // bitmap index deltas in the grouped layout (apply_dir_geometry): the lowest top dim moves
        // the index by 1, the others by pstride_i * |g_lo|
        int64_t dq = 0, dq2 = 0;
        for (int i = L; i < D; ++i) {
            const int dl = (int)((t / kPow3i(i - L)) % 3u) - 1;
            dq += dl * (int64_t)ix.occ_mul[i];
            dq2 += dl * (int64_t)ix.occ2_mul[i];
        }
        tt.dq[t] = dq;
        tt.dq2[t] = dq2;
        tt.bits[t] = neg | (pos << 8) | (top << 16);
    }
}

// Alg. 1 lines 5-6 (getAdjCells, maskCellRange): which moves of each dimension stay inside M_j,
// as a "bad" bit set: bit i = move -1 in dim i leaves M_i, bit 8+i = move +1 leaves M_i;
// unicomp adds bit 16+i when the query's c_i is even (cells decided by dim i are not searched).
template <int D, bool UNICOMP>
__device__ __forceinline__ uint32_t bad_moves(const DevIndex &ix, const JoinArgs &ja, const QueryState<D> &q,
                                              uint32_t h)
{
    uint32_t bad = 0;
    if (ja.use_masks && ix.masks) {
        if (ix.cmask) {
            bad = __ldg(ix.cmask + h);                          // precomputed per cell at build time
        } else {
#pragma unroll
            for (int i = 0; i < D; ++i) {
                const uint64_t lo = ix.mask_off[i] + q.c[i] - 1ull, hi = lo + 2ull;
                if (!((__ldg(ix.masks + (lo >> 5)) >> (lo & 31)) & 1u)) bad |= 1u << i;
                if (!((__ldg(ix.masks + (hi >> 5)) >> (hi & 31)) & 1u)) bad |= 1u << (i + 8);
            }
        }
    }
    if (UNICOMP) bad |= ((~q.odd) & ((1u << D) - 1u)) << 16;
    return bad;
}

// A cell hh of the prefix range whose key differs from the (offset-moved) home key by dlt, with
// |dlt| <= lowR[L]: adjacent iff dlt = sum_{i<L} delta_i * stride_i with every delta_i in {-1,0,1}
// (greedy from the top low dimension; mixed-radix digits are unique and stride_i > 2 sum_{m<i}
// stride_m).  The deciding dimension of unicomp is the highest moved one: jtop (a top dim) if
// the offset moved one, else the highest moved low dim.
template <int D, int MODE, bool UNICOMP, bool DENSE>
__device__ __forceinline__ void test_low_cell(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                              uint32_t hh, int64_t dlt, int jtop, int L, unsigned wmask,
                                              WarpBuf *wb)
{
    int jlow = -1;
#pragma unroll
    for (int i = D - 2; i >= 0; --i) {
        if (i >= L) continue;
        const int64_t R = ix.lowR[i], st = (int64_t)ix.strides[i];
        if (dlt > R) { dlt -= st; if (jlow < 0) jlow = i; }
        else if (dlt < -R) { dlt += st; if (jlow < 0) jlow = i; }
    }
    if (dlt != 0) return;                            // not representable: not adjacent
    const int j = jtop >= 0 ? jtop : jlow;
    if (UNICOMP && !((q.odd >> j) & 1u)) return;
    scan_range<D, MODE, UNICOMP, DENSE>(ix, ja, q, __ldg(ix.G + hh), __ldg(ix.G + hh + 1), 1u, wb, wmask);
}

// Sparse regime with k <= 3 top dimensions (the occupancy bitmap is built): the top offsets are
// visited in blocks by their highest moved top dimension, so a block that unicomp rejects (that
// dimension's coordinate even -- warp-uniform for the slow dimensions of A-ordered queries) is
// skipped with one branch; the bitmap loads of a block are issued together; the home top offset
// needs no directory lookup: its adjacent cells are the run of B within +-lowR[L] of the home
// key around h (B is sorted and |key difference| <= lowR[L] < stride_L keeps the run inside
// the prefix).
// One block of search_cell_scan_sparse: the 2 * 3^JT top offsets whose highest moved top dimension is
// L + JT (that dimension moved by -1 or +1, the top dimensions below it by -1/0/+1, the ones above
// it unmoved).  JT is a compile-time constant so the filter loop has exactly the block's offsets.
// Three bits of a bitmap starting at bit index b0 (the window c_L - 1 .. c_L + 1 of the grouped
// layout): one 64-bit load (a second only when the three straddle a 64-bit word, 3 in 64)
__device__ __forceinline__ uint32_t bits3(const uint32_t *bm, uint64_t b0)
{
    const uint64_t *w = reinterpret_cast<const uint64_t *>(bm) + (b0 >> 6);
    const uint32_t sh = (uint32_t)(b0 & 63u);
    uint64_t v = __ldg(w) >> sh;
    if (sh > 61) v |= __ldg(w + 1) << (64u - sh);
    return (uint32_t)v & 7u;
}

template <int D, int MODE, bool UNICOMP, int JT>
__device__ __forceinline__ void sparse_block(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q, uint64_t key,
                                             uint32_t bad, const TopTable &tt, uint64_t ph, uint64_t qc,
                                             uint64_t qc2, int64_t Rl, uint32_t pow3k, int L)
{
    constexpr uint32_t p3 = JT == 2 ? 9u : (JT == 1 ? 3u : 1u);   // 3^JT
    constexpr uint32_t nb = 2u * p3;
    const uint32_t tbase = (pow3k - 3u * p3) / 2u;               // digits above JT = "0 move"
    // bit i of live <-> offset t(i) = tbase + (i >> 1) + (i & 1 ? 2 p3 : 0).  The offsets come in
    // groups of three consecutive t (the lowest top dim at -1, 0, +1: adjacent bits of both bitmaps
    // in the grouped layout), so each group costs ONE window load per bitmap instead of three.
    uint32_t live = 0;
    if constexpr (JT == 0) {
        // the pair c_L - 1, c_L + 1 (t = tbase, tbase + 2): one window of the home group
        const uint32_t tm = tbase + 1u;                          // the home offset (all top dims 0)
        uint32_t w = bits3(ix.occ, qc + (uint64_t)tt.dq[tm] - 1ull);
        if (ix.occ2) w &= bits3(ix.occ2, qc2 + (uint64_t)tt.dq2[tm] - 1ull);
        if ((w & 1u) && !(tt.bits[tbase] & bad)) live |= 1u;
        if ((w & 4u) && !(tt.bits[tbase + 2u] & bad)) live |= 2u;
    } else {
#pragma unroll
        for (uint32_t g = 0; g < nb / 3u; ++g) {
            // group g: members i = 3g .. 3g+2 are consecutive t (i>>1 and the +2p3 half alternate, so
            // enumerate groups in t order instead): t0 = first t of the group
            const uint32_t half = g / (p3 / 3u), gi = g % (p3 / 3u);
            const uint32_t t0 = tbase + half * 2u * p3 + 3u * gi;
            const uint32_t tm = t0 + 1u;
            uint32_t ok3 = 0;
#pragma unroll
            for (uint32_t m = 0; m < 3u; ++m) ok3 |= (tt.bits[t0 + m] & bad) ? 0u : (1u << m);
            if (!ok3) continue;
            uint32_t w = bits3(ix.occ, qc + (uint64_t)tt.dq[tm] - 1ull);
            if (ix.occ2) w &= bits3(ix.occ2, qc2 + (uint64_t)tt.dq2[tm] - 1ull);
            w &= ok3;
            // member m of the group is offset t0 + m -> live bit index i with t(i) = t0 + m
#pragma unroll
            for (uint32_t m = 0; m < 3u; ++m) {
                const uint32_t t = t0 + m - tbase;               // position in the block
                const uint32_t i = t < p3 ? 2u * t : 2u * (t - 2u * p3) + 1u;
                if ((w >> m) & 1u) live |= 1u << i;
            }
        }
    }
    const int dim = L + JT;
#pragma unroll 1
    while (live) {
        const uint32_t i = __ffs(live) - 1;
        live &= live - 1u;
        const uint32_t t = tbase + (i >> 1) + ((i & 1u) ? 2u * p3 : 0u);
        const uint64_t p = ph + (uint64_t)tt.dp[t];
        ++q.probes;
        const uint32_t lo = __ldg(ix.dir + p), hi = __ldg(ix.dir + p + 1);
        const uint64_t kal = key + (uint64_t)tt.dk[t];
#pragma unroll 1
        for (uint32_t hh = lo; hh < hi; ++hh) {
            const int64_t dlt = (int64_t)(__ldg(ix.B + hh) - kal);
            if (dlt > Rl || dlt < -Rl) continue;
            test_low_cell<D, MODE, UNICOMP, false>(ix, ja, q, hh, dlt, dim, L, 0u, nullptr);
        }
    }
}

// Sparse regime with k <= 3 top dimensions (the occupancy bitmap is built): the top offsets are
// visited in blocks by their highest moved top dimension, so a block that unicomp rejects (that
// dimension's coordinate even -- warp-uniform for the slow dimensions of A-ordered queries) is
// skipped with one branch; the bitmap loads of a block are issued together; the home top offset
// needs no directory lookup: its adjacent cells are the run of B within +-lowR[L] of the home
// key around h (B is sorted and |key difference| <= lowR[L] < stride_L keeps the run inside
// the prefix).
template <int D, int MODE, bool UNICOMP>
__device__ __forceinline__ void search_cell_scan_sparse(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                                        uint32_t h, uint64_t key, uint32_t bad, const TopTable &tt,
                                                        unsigned wmask)
{
    const int k = ix.dir_k;
    const int L = D - k;
    uint64_t ph = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) ph += q.c[j] * ix.pstride[j];
    // bitmap indices as sums with static per-dimension multipliers (a runtime-selected q.c[L-1]
    // made the compiler keep q in local memory)
    uint64_t qc = 0, qc2 = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) {
        qc += q.c[j] * ix.occ_mul[j];
        qc2 += q.c[j] * ix.occ2_mul[j];
    }
    const int64_t Rl = ix.lowR[L];
    const uint32_t pow3k = k == 3 ? 27u : (k == 2 ? 9u : 3u);
    if (k >= 3 && (!UNICOMP || ((q.odd >> (L + 2)) & 1u)))
        sparse_block<D, MODE, UNICOMP, 2>(ix, ja, q, key, bad, tt, ph, qc, qc2, Rl, pow3k, L);
    __syncwarp(wmask);
    if (k >= 2 && (!UNICOMP || ((q.odd >> (L + 1)) & 1u)))
        sparse_block<D, MODE, UNICOMP, 1>(ix, ja, q, key, bad, tt, ph, qc, qc2, Rl, pow3k, L);
    __syncwarp(wmask);
    if (!UNICOMP || ((q.odd >> L) & 1u))
        sparse_block<D, MODE, UNICOMP, 0>(ix, ja, q, key, bad, tt, ph, qc, qc2, Rl, pow3k, L);
    // home top offset: outward from h while |B[hh] - key| <= lowR[L]
    __syncwarp(wmask);
    ++q.probes;
#pragma unroll 1
    for (uint32_t hh = h; hh-- > 0;) {
        const int64_t dlt = (int64_t)(__ldg(ix.B + hh) - key);
        if (dlt < -Rl) break;
        test_low_cell<D, MODE, UNICOMP, false>(ix, ja, q, hh, dlt, -1, L, wmask, nullptr);
    }
#pragma unroll 1
    for (uint32_t hh = h + 1; hh < ix.nG; ++hh) {
        const int64_t dlt = (int64_t)(__ldg(ix.B + hh) - key);
        if (dlt > Rl) break;
        test_low_cell<D, MODE, UNICOMP, false>(ix, ja, q, hh, dlt, -1, L, wmask, nullptr);
    }
}

// ---- search mode kSearchCellScan (sparse high-d data): for each offset of the top-k
// (directory) dimensions, the cells of that prefix are B[dir[p], dir[p+1]) -- a handful.  Each
// is tested by its low coordinates: it is adjacent iff its key differs from the home key moved
// into prefix p by sum_{i<L} delta_i * stride_i with every delta_i in {-1,0,1}.  Mixed-radix
// digits are unique and stride_i > 2 * sum_{m<i} stride_m (|g_j| >= 3), so the deltas follow
// greedily from the top low dimension (delta_i = sign(D) if |D| > lowR[i], else 0) -- no division.
// Lanes of a query's group take offsets t = sub, sub+G, ...  Covers every neighbour cell except
// the home cell.
template <int D, int MODE, bool UNICOMP, bool DENSE = false>
__device__ __forceinline__ void search_cell_scan(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                                 uint32_t h, uint64_t key, uint32_t bad, const TopTable &tt,
                                                 unsigned wmask, WarpBuf *wb = nullptr)
{
    const int L = D - ix.dir_k;     // low dimensions 0..L-1 are not in the directory prefix
    uint64_t ph = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) ph += q.c[j] * ix.pstride[j];
    const int64_t Rl = ix.lowR[L];
    // Uniform trip count for every lane of the warp and an explicit __syncwarp per chunk: without
    // it the lanes drift apart (independent thread scheduling) and their divergent cell loops
    // serialise -- measured 2.4 of 32 lanes active on 6-D eps=8.
    // Offsets are taken in chunks of kChunk: phase 1 (unrolled) issues the occupancy-bitmap loads
    // of the whole chunk together (memory-level parallelism), phase 2 scans the survivors.
    uint64_t qh = 0, qh2 = 0;                    // bitmap indices of the home top-(k+1) prefixes
#pragma unroll
    for (int j = 0; j < D; ++j) {
        qh += q.c[j] * ix.occ_mul[j];
        qh2 += q.c[j] * ix.occ2_mul[j];
    }
#ifndef SJ_CHUNK
#define SJ_CHUNK 27
#endif
    constexpr int kChunk = SJ_CHUNK;
    const uint32_t ntop = ix.dir_ntop;
    const uint32_t step = q.G * kChunk;
#pragma unroll 1
    for (uint32_t t0 = 0; t0 < ntop; t0 += step) {
        __syncwarp(wmask);
        uint32_t live = 0;                       // bit u: offset t0 + sub + u*G survives the filters
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            const uint32_t t = t0 + q.sub + (uint32_t)u * q.G;
            if (t >= ntop) continue;
            const uint32_t bits = tt.bits[t];
            if (bits & bad) continue;            // masked-out coordinate, or decided by an even top dim
            if (ix.occ) {
                // joint-occupancy filter: is any (k+1)-prefix p*|g_{L-1}| + c_{L-1} + {-1,0,1}
                // occupied?  (the top low dimension's window, one bit of the dilated bitmap;
                // PAPER.md:173 masks, generalised)
                const uint64_t qb = qh + (uint64_t)tt.dq[t];
                if (!((__ldg(ix.occ + (qb >> 5)) >> (qb & 31)) & 1u)) continue;
                if (ix.occ2) {
                    const uint64_t qb2 = qh2 + (uint64_t)tt.dq2[t];
                    if (!((__ldg(ix.occ2 + (qb2 >> 5)) >> (qb2 & 31)) & 1u)) continue;
                }
            }
            live |= 1u << u;
        }
        // phase 2.  With the occupancy bitmap (sparse regime) survivors are rare and each lane walks
        // its own (measured 0.54 vs 0.71 ms on 6-D eps=1).  Without it (denser regime) survivors are
        // common and the warp visits the offsets live in ANY lane together, re-converging at each
        // (lanes' cell loops differ; drifting apart serialises the warp: 14 vs 26 ms on eps=8).
        const bool sparse = ix.occ != nullptr;
        uint32_t any = sparse ? live : __reduce_or_sync(wmask, live);
#pragma unroll 1
        while (any) {
            const int u = __ffs(any) - 1;
            any &= any - 1u;
            if (!sparse) {
                __syncwarp(wmask);
                if (!((live >> u) & 1u)) continue;
            }
            const uint32_t t = t0 + q.sub + (uint32_t)u * q.G;
            const uint32_t bits = tt.bits[t];
            const int jtop = (bits >> 16) ? (__ffs(bits >> 16) - 1) : -1;
            const uint64_t p = ph + (uint64_t)tt.dp[t];
            ++q.probes;
            const uint32_t lo = __ldg(ix.dir + p), hi = __ldg(ix.dir + p + 1);
            const uint64_t kal = key + (uint64_t)tt.dk[t];
#pragma unroll 1
            for (uint32_t hh = lo; hh < hi; ++hh) {
                if (hh == h) continue;                       // home cell handled separately
                const int64_t dlt = (int64_t)(__ldg(ix.B + hh) - kal);
                if (dlt > Rl || dlt < -Rl) continue;         // outside the +-1 box
                test_low_cell<D, MODE, UNICOMP, DENSE>(ix, ja, q, hh, dlt, jtop, L, wmask, wb);
            }
        }
    }
}

// ---- search modes kSearchDenseRows / kSearchRows: rows whose highest differing dimension is
// j = D-1 .. 1 (a row = the three cells c_0-1..c_0+1 of fixed dims >= 1: consecutive linear ids,
// one contiguous A-range).  Unicomp: only when c_j is odd (reading R13).  Each row is looked up
// in the prefix directory, then (kSearchRows) by a search bounded to that prefix's range.  The
// rows of all j are numbered 0..3^(D-1)-2 (j = D-1 first) and dealt to the group's lanes.
template <int D, int MODE, bool UNICOMP, bool DENSE = false>
__device__ __forceinline__ void search_rows(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                            uint64_t key, uint32_t bad, unsigned wmask, WarpBuf *wb = nullptr)
{
    uint64_t ph = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) ph += q.c[j] * ix.pstride[j];
    const bool dense = ix.search_mode == kSearchDenseRows;
    constexpr uint32_t kPow3[7] = {1, 3, 9, 27, 81, 243, 729};
    constexpr uint32_t nrows_all = kPow3[D - 1] - 1;
#pragma unroll 1
    for (uint32_t R0 = 0; R0 < nrows_all; R0 += q.G) {
        __syncwarp(wmask);                    // re-converge the warp every row (see cell scan)
        const uint32_t R = R0 + q.sub;
        if (R >= nrows_all) continue;
        // decode (j, r): rows of top dim j are 2*3^(j-1), j = D-1 first
        int j = D - 1;
        uint32_t r = R;
#pragma unroll
        for (int jj = D - 1; jj >= 1; --jj) {
            const uint32_t cnt = 2u * kPow3[jj - 1];
            if (j == jj && r >= cnt) { r -= cnt; j = jj - 1; }
        }
        if (UNICOMP && !((q.odd >> j) & 1u)) continue;
        // row offsets: dim j = +-1 (bit 0 of r), dims 1..j-1 in {-1,0,1} (base-3 digits of r>>1)
        uint64_t b = key, p = ph;
        uint32_t moves = (r & 1u) ? (1u << (j + 8)) : (1u << j);
#pragma unroll
        for (int i = 1; i < D; ++i) {
            if (i == j) {
                if (r & 1u) { b += ix.strides[i]; p += ix.pstride[i]; }
                else { b -= ix.strides[i]; p -= ix.pstride[i]; }
            }
        }
        uint32_t rest = r >> 1;
#pragma unroll
        for (int i = 1; i < D - 1; ++i) {
            if (i >= j) break;
            const uint32_t dl = rest % 3u;
            rest /= 3u;
            if (dl == 0u) { b -= ix.strides[i]; p -= ix.pstride[i]; moves |= 1u << i; }
            else if (dl == 2u) { b += ix.strides[i]; p += ix.pstride[i]; moves |= 1u << (i + 8); }
        }
        if (moves & bad & 0xFFFFu) continue;   // a masked-out coordinate: the row is empty
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
        if (s < e) scan_range<D, MODE, UNICOMP, DENSE>(ix, ja, q, __ldg(ix.G + s), __ldg(ix.G + e), 1u, wb, wmask);
    }
}

// wmask: the lanes of the warp that run refine_query together (a full-warp ballot taken by the
// caller before any divergence); every __syncwarp below is over exactly these lanes.
template <int D, int MODE, bool UNICOMP, bool DENSE = false>
__device__ __forceinline__ void refine_query(const DevIndex &ix, const JoinArgs &ja, uint32_t k, uint32_t h,
                                            uint32_t cs, uint32_t ce, unsigned wmask, QueryState<D> &q,
                                            const TopTable &tt, WarpBuf *wb = nullptr)
{
    q.k = k;
    q.pid = __ldg(ix.A + k);
#pragma unroll
    for (int j = 0; j < D; ++j) q.x[j] = __ldg(ix.X + (uint64_t)j * ix.n + k);
    // the home cell's coordinates, decoded from its linear id (double-reciprocal quotients)
    const uint64_t key = __ldg(ix.B + h);
    key_to_coords<D>(ix, key, q.c);
    q.odd = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) q.odd |= (uint32_t)(q.c[j] & 1ull) << j;

    // ---- home cell: (p,p) once; unicomp: q after p in A-order, both orientations (R10)
    if constexpr (DENSE) {
        if (q.valid && ja.include_self) emit_self<MODE>(ja, q.k, q.pid, q.emitted);
        scan_range<D, MODE, UNICOMP, true, true>(ix, ja, q, cs, ce, 1u, wb, wmask);
    } else {
        if (q.sub == 0 && ja.include_self) emit_self<MODE>(ja, q.k, q.pid, q.emitted);
        if constexpr (UNICOMP) {
            scan_range<D, MODE, true>(ix, ja, q, k + 1 + q.sub, ce, q.G);
        } else {
#pragma unroll 1
            for (int part = 0; part < 2; ++part)
                scan_range<D, MODE, false>(ix, ja, q, (part ? k + 1 : cs) + q.sub, part ? ce : k, q.G);
        }
    }
    const uint32_t bad = bad_moves<D, UNICOMP>(ix, ja, q, h);
    __syncwarp(wmask);
    if (ix.search_mode == kSearchCellScan) {
        if constexpr (!DENSE) {
            if (ix.occ && ix.dir_k <= 3 && q.G == 1u) {
                search_cell_scan_sparse<D, MODE, UNICOMP>(ix, ja, q, h, key, bad, tt, wmask);
                return;
            }
        }
        search_cell_scan<D, MODE, UNICOMP, DENSE>(ix, ja, q, h, key, bad, tt, wmask, wb);
        return;
    }
    // ---- home row: cells key-1 / key+1 (dims >= 1 equal); unicomp: only when c_0 is odd
    if (!UNICOMP || (q.c[0] & 1ull)) {
#pragma unroll 1
        for (uint32_t side = q.sub; side < 2u; side += q.G) {
            uint32_t m0 = 0, m1 = 0;
            if (side == 0 && h > 0 && __ldg(ix.B + h - 1) == key - 1ull) { m0 = __ldg(ix.G + h - 1); m1 = cs; }
            if (side == 1 && h + 1 < ix.nG && __ldg(ix.B + h + 1) == key + 1ull) { m0 = ce; m1 = __ldg(ix.G + h + 2); }
            scan_range<D, MODE, UNICOMP, DENSE>(ix, ja, q, m0, m1, 1u, wb, wmask);
        }
    }
    __syncwarp(wmask);
    search_rows<D, MODE, UNICOMP, DENSE>(ix, ja, q, key, bad, wmask, wb);
}

// Work counters (directory/row lookups, distance tests, emissions): warp shuffle-reduce, then one
// set of fire-and-forget atomics per warp into one of kWorkSlots slots (warp id modulo; the host
// sums the slots).  Per-warp atomics on three shared addresses serialised in L2 and cost as much
// as the whole sparse 6-D refine; a CTA-wide reduction instead made every warp wait at a barrier
// for the CTA's slowest warp (19% of the stall samples).
constexpr int kWorkSlots = 256;
// Sum of a 64-bit per-lane counter over the full warp with two REDUX.SUM (32-bit warp reductions):
// the low 27 bits of 32 lanes sum below 2^32, the high parts below 2^32 for any counter < 2^59.  (Five
// rounds of 64-bit shuffles were 7 % of the sparse refine's instructions, for statistics only.)
__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v)
{
    const unsigned lo = __reduce_add_sync(0xffffffffu, (unsigned)(v & 0x7FFFFFFull));
    const unsigned hi = __reduce_add_sync(0xffffffffu, (unsigned)(v >> 27));
    return (unsigned long long)lo + ((unsigned long long)hi << 27);
}

__device__ __forceinline__ void flush_work(const JoinArgs &ja, unsigned long long p, unsigned long long c,
                                           unsigned long long em)
{
    p = warp_sum_u64(p);
    c = warp_sum_u64(c);
    em = warp_sum_u64(em);
    if ((threadIdx.x & 31) == 0 && ja.work) {
        const uint32_t gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        unsigned long long *w = ja.work + 4 * (gw % kWorkSlots);
        atomicAdd(w + 0, p);
        atomicAdd(w + 1, c);
        atomicAdd(w + 2, em);
    }
}

// Dense kernel (kEmit): one warp per task = up to 32 consecutive queries of one populous cell
// (>= dense_T points).  All lanes share the home cell, so the whole neighbour enumeration and every
// candidate loop are warp-uniform: candidates are broadcast loads, hits go through the per-warp
// shared-memory buffer (one cursor atomic per flush instead of one per candidate step).
constexpr int kDenseWarps = 8;
template <int D, bool UNICOMP, bool F32 = false>
#ifndef SJ_DENSE_MINB
#define SJ_DENSE_MINB 3
#endif
__global__ void __launch_bounds__(32 * kDenseWarps, D <= 3 ? SJ_DENSE_MINB : 2)   // 3 CTAs/SM: smem fits up to d = 4, registers (80) up to d = 3
k_refine_dense(const DevIndex ix, const JoinArgs ja)
{
    // dynamic shared memory: [rings | tiles | ids] (dense_smem_per_warp each warp) and, in the
    // cell-scan mode only, the top-offset table after them -- a static table (9.8 KB) kept the
    // kernel at 2 CTAs per SM
    extern __shared__ __align__(16) uint64_t s_buf[];
    TopTable &tt = *reinterpret_cast<TopTable *>(reinterpret_cast<char *>(s_buf) + kDenseWarps * dense_smem_per_warp<D>());
    if (ix.search_mode == kSearchCellScan) build_top_table<D>(ix, tt);
    // the batch's tasks are the contiguous range of the A-ordered task list whose real end
    // min(start + 32, end of its cell) lies after q0 and whose start lies before q1.  Task ends are
    // monotone in the task index (tasks of a cell are consecutive, cells are in A-order), so t_lo
    // is one search per CTA; the warps then stride over the tasks until start >= q1, so the
    // launch size is only a hint (tails of cells make tasks shorter than dense_T queries).  The search
    // is 32-ary by the first warp (each probe is 3 dependent loads: task start, its cell, the cell's
    // end): ~4 rounds instead of ~17 for 10^5 tasks -- a thread-serial binary search held every CTA's
    // warps at the barrier for ~8% of the 2-D kernel's stall samples.
    __shared__ uint32_t s_tlo;
    if (threadIdx.x < 32) {
        const uint32_t l = threadIdx.x;
        uint32_t lo = 0, hi = ja.n_dense_tasks;        // the answer lies in [lo, hi]
        while (lo < hi) {                              // warp-uniform
            const uint32_t step = (hi - lo + 31u) >> 5;
            const uint32_t p = lo + (l + 1u) * step - 1u;
            bool before = false;                       // task p ends at or before q0
            if (p < hi) {
                const uint32_t st = __ldg(ja.dense_tasks + p);
                before = min(st + 32u, __ldg(ix.G + __ldg(ix.pcell + st) + 1)) <= ja.q0;
            }
            const uint32_t c = (uint32_t)__popc(__ballot_sync(0xffffffffu, before));   // lanes 0..c-1 (monotone)
            const uint32_t nlo = lo + c * step;
            if (c < 32u && lo + (c + 1u) * step - 1u < hi) hi = lo + (c + 1u) * step - 1u;
            lo = nlo;
        }
        if (l == 0) s_tlo = lo;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    QueryState<D> q;
    q.G = 1u;
    q.sub = 0u;
    q.emitted = q.probes = q.tests = 0;
    double *s_tx = reinterpret_cast<double *>(s_buf + (size_t)kDenseWarps * kWarpBufPairs);
    uint32_t *s_tid = reinterpret_cast<uint32_t *>(s_tx + (size_t)kDenseWarps * 32 * D);
    WarpBuf wb{s_buf + (size_t)warp * kWarpBufPairs, s_tx + (size_t)warp * 32 * D, s_tid + warp * 32, 0u, 0u, 0u, 0ull};
#pragma unroll 1
    for (uint32_t task = s_tlo + blockIdx.x * kDenseWarps + warp; task < ja.n_dense_tasks;
         task += gridDim.x * kDenseWarps) {            // warp-uniform
        const uint32_t start = __ldg(ja.dense_tasks + task);
        if (start >= ja.q1) break;
        const uint32_t h = __ldg(ix.pcell + start);
        const uint32_t end = min(start + 32u, __ldg(ix.G + h + 1));
        const uint32_t a = max(start, ja.q0), b = min(end, ja.q1);
        if (a < b) {                                   // task inside this batch
            // every lane runs the (cell-uniform) enumeration; lanes past the task's end are helpers
            // that load and broadcast candidates but never emit (they take the first query's point)
            const uint32_t k = a + lane;
            q.valid = k < b;
            refine_query<D, F32 ? (kEmit | kF32) : kEmit, UNICOMP, true>(ix, ja, q.valid ? k : a, h, __ldg(ix.G + h), __ldg(ix.G + h + 1),
                                                  0xffffffffu, q, tt, &wb);
        }
    }
    ring_drain(ja, wb);                                // the ring lives across the warp's tasks
    flush_work(ja, q.probes, q.tests, q.emitted);
}

// MINB: CTAs per SM the register budget is sized for -- kRefineMinBlocks (5) in general; 6 for the
// many-offset cell scan without bitmaps (6-D eps=8: 9.4 -> 9.1 ms), where more warps hide more of
// the directory/B lookup latency
template <int D, int MODE, bool UNICOMP, int MINB = kRefineMinBlocks>
__global__ void __launch_bounds__(kRefineThreads, MINB)
k_refine(const DevIndex ix, const JoinArgs ja)
{
    __shared__ TopTable tt;
    if (ix.search_mode == kSearchCellScan) {
        build_top_table<D>(ix, tt);
        __syncthreads();
    }
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t qi = t >> ja.lanes_log2;            // query slot of this lane's group
    QueryState<D> q;
    q.valid = true;
    q.G = 1u << ja.lanes_log2;
    q.sub = t & (q.G - 1u);
    q.emitted = q.probes = q.tests = 0;
    uint32_t k;
    bool active;
    if constexpr ((MODE & kModeMask) == kCountQuery) {
        // sample qi: lane qi%32 of run qi/32; run r = the first 32 queries of block [r*32*step, ...)
        k = ja.q0 + (qi >> 5) * (32u * ja.step) + (qi & 31u);
        active = qi < ja.nsamples && k < ja.q1;
    } else {
        k = ja.q0 + qi;
        active = k < ja.q1;
    }
    uint32_t h = 0, cs = 0, ce = 0;
    if (active) {
        h = __ldg(ix.pcell + k);
        cs = __ldg(ix.G + h);
        ce = __ldg(ix.G + h + 1);
        // queries of populous cells are handled by the warp-per-task dense kernel
        if ((MODE & kModeMask) == kEmit && ja.dense_T && ce - cs >= ja.dense_T) active = false;
    }
    const unsigned wmask = __ballot_sync(0xffffffffu, active);   // before any divergence
    if (active) refine_query<D, MODE, UNICOMP>(ix, ja, k, h, cs, ce, wmask, q, tt);
    if constexpr ((MODE & kModeMask) == kCountQuery) {
        // sum the group's partial counts (all lanes of a group share `active`)
        uint32_t e = q.emitted;
        for (uint32_t o = 1; o < q.G; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (active && q.sub == 0) atomicAdd(ja.qbucket + qi / ja.group, (unsigned long long)e);
    }
    flush_work(ja, q.probes, q.tests, q.emitted);
}

// ---------------------------------------------------------------- queued cell scan (many offsets)
// The cell-scan search without occupancy bitmaps (6-D eps = 8: 243 top offsets per query) spent about
// half its issue slots in the candidate loop and the low-coordinate adjacency test with 4-5 of 32
// lanes active (every lane walks its own query's cells; ncu: 9.4 active threads per warp).  Here the
// search only FINDS the adjacent cells: each lane pushes the point range of every adjacent cell its
// query must test into a per-warp queue in shared memory, and the warp drains the queue with all 32
// lanes -- candidate t of the flattened ranges goes to lane t mod 32 (owner range by a binary search
// over the ranges' prefix sums held in registers), the query's coordinates come from shared memory,
// and hits are emitted warp-aggregated (ballot/popc, one cursor atomic per warp round).  The set of
// (query, candidate) tests is exactly the inline path's, so S is unchanged.
constexpr int kQCap = 192;             // queue entries per warp (1.5 KB)
constexpr int kQDrainAt = 96;           // drain once this many are queued (one round pushes <= 32 * 3^L)
constexpr int kQWarps = kRefineThreads / 32;

struct QEntry {
    uint32_t start;                     // first A-position of the range
    uint32_t len_lane;                  // length (< 2^24) | pushing lane << 24
};

template <int D>
struct WarpQueue {
    QEntry *e;                          // [kQCap]
    uint32_t *cnt;                      // entries queued
    double *qx;                         // [32][D] the lanes' query coordinates
    uint32_t *qid;                      // [32] the lanes' query ids (original)
    uint32_t *qem;                      // [32] pairs emitted for each lane's query (count modes)
};

template <int D>
struct QueueSmem {
    QEntry e[kQWarps][kQCap];
    uint32_t cnt[kQWarps];
    double qx[kQWarps][32 * D];
    uint32_t qid[kQWarps][32];
    uint32_t qem[kQWarps][32];
};

// Push a candidate range for the calling lane's query; false when the queue is full (the caller
// then tests the range inline).
template <int D>
__device__ __forceinline__ bool q_push(const WarpQueue<D> &w, uint32_t start, uint32_t len)
{
    if (len == 0) return true;
    if (len >= (1u << 24)) return false;
    const uint32_t slot = atomicAdd(w.cnt, 1u);
    if (slot >= (uint32_t)kQCap) {
        atomicSub(w.cnt, 1u);
        return false;
    }
    w.e[slot] = QEntry{start, len | ((uint32_t)(threadIdx.x & 31) << 24)};
    return true;
}

// Drain the queue (all 32 lanes, converged): while >= 32 entries are queued, or until empty when
// `final`.  Entries are taken from the top, 32 at a time.
template <int D, int MODE, bool BOTH>
__device__ __forceinline__ void q_drain(const DevIndex &ix, const JoinArgs &ja, const WarpQueue<D> &w, bool final,
                                     uint32_t &tests, uint32_t &emitted)
{
    const int lane = threadIdx.x & 31;
    __syncwarp();
    uint32_t cnt = *(volatile uint32_t *)w.cnt;
    const uint32_t n = ix.n;
    while (cnt >= 32u || (final && cnt > 0u)) {
        const uint32_t nb = min(32u, cnt);
        QEntry en{0u, 0u};
        if ((uint32_t)lane < nb) en = w.e[cnt - nb + lane];
        const uint32_t len = en.len_lane & 0xFFFFFFu;
        uint32_t incl = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t T = __shfl_sync(0xffffffffu, incl, 31);
        for (uint32_t t0 = 0; t0 < T; t0 += 32u) {
            const uint32_t t = t0 + lane;
            // owner range: the number of ranges whose inclusive end is <= t
            uint32_t l = 0;
#pragma unroll
            for (uint32_t step = 16; step; step >>= 1) {
                const uint32_t v = __shfl_sync(0xffffffffu, incl, l + step - 1);
                if (v <= t) l += step;
            }
            l = min(l, 31u);
            const uint32_t ex = __shfl_sync(0xffffffffu, incl - len, l);
            const uint32_t st = __shfl_sync(0xffffffffu, en.start, l);
            const uint32_t ql = __shfl_sync(0xffffffffu, en.len_lane, l) >> 24;
            const bool valid = t < T;
            bool hit = false;
            uint32_t cid = 0;
            if (valid) {
                const uint32_t m = st + (t - ex);
                const double *qx = w.qx + ql * D;
                if constexpr ((MODE & kF32) != 0) {
                    float s;
                    {
                        const float d0 = __fsub_rn((float)qx[0], (float)__ldg(ix.X + m));
                        s = __fmul_rn(d0, d0);
                    }
#pragma unroll
                    for (int j = 1; j < D; ++j) {
                        const float dj = __fsub_rn((float)qx[j], (float)__ldg(ix.X + (uint64_t)j * n + m));
                        s = __fadd_rn(s, __fmul_rn(dj, dj));
                    }
                    hit = s <= ix.eps2f;
                } else {
                    double s;
                    {
                        const double d0 = __dsub_rn(qx[0], __ldg(ix.X + m));
                        s = __dmul_rn(d0, d0);
                    }
#pragma unroll
                    for (int j = 1; j < D; ++j) {
                        const double dj = __dsub_rn(qx[j], __ldg(ix.X + (uint64_t)j * n + m));
                        s = __dadd_rn(s, __dmul_rn(dj, dj));
                    }
                    hit = s <= ix.eps2;
                }
                ++tests;
                if ((MODE & kModeMask) != kCountQuery && hit) cid = __ldg(ix.A + m);
            }
            const uint32_t pid = w.qid[ql];
            if constexpr ((MODE & kModeMask) == kCountQuery) {
                if (hit) atomicAdd(w.qem + ql, BOTH ? 2u : 1u);
            } else {
                uint32_t dummy = 0;
                emit<MODE, BOTH>(ja, hit, pid, cid, dummy);
                emitted += dummy;
            }
        }
        cnt -= nb;
        __syncwarp();
        if (lane == 0) *w.cnt = cnt;
        __syncwarp();
    }
}

template <int D, bool UNICOMP>
__device__ __forceinline__ bool low_cell_adjacent_odd(const DevIndex &ix, uint32_t odd, int64_t dlt, int jtop, int L)
{
    int jlow = -1;
#pragma unroll
    for (int i = D - 2; i >= 0; --i) {
        if (i >= L) continue;
        const int64_t R = ix.lowR[i], st = (int64_t)ix.strides[i];
        if (dlt > R) { dlt -= st; if (jlow < 0) jlow = i; }
        else if (dlt < -R) { dlt += st; if (jlow < 0) jlow = i; }
    }
    if (dlt != 0) return false;
    const int j = jtop >= 0 ? jtop : jlow;
    return !(UNICOMP && !((odd >> j) & 1u));
}

// kSearchCellScan without the bitmap filter, queued.  Every lane of the warp runs this (lanes without
// a query have `bad` = all ones: no live offsets) so the drains see a converged warp.  A lane whose
// push finds the queue full stops its cell walk there and resumes it after the warp drained, so no
// range is ever tested inline (the query's coordinates live only in the queue's shared memory).
// (Dealing the warp's live (query, offset) pairs out to all lanes instead of iterating the union of
// the lanes' live offsets measured slower: 11.5 vs 8.6 ms on 6-D eps = 8.)
template <int D, int MODE, bool UNICOMP>
__device__ __forceinline__ void search_cell_scan_q(const DevIndex &ix, const JoinArgs &ja, QueryState<D> &q,
                                                   bool active, uint32_t h, uint64_t key, uint32_t bad,
                                                   const TopTable &tt, const WarpQueue<D> &w)
{
    const int L = D - ix.dir_k;
    uint64_t ph = 0;
#pragma unroll
    for (int j = 0; j < D; ++j) ph += q.c[j] * ix.pstride[j];
    const int64_t Rl = ix.lowR[L];
    constexpr int kChunk = 27;
    const uint32_t ntop = ix.dir_ntop;
    const uint32_t step = q.G * kChunk;
#pragma unroll 1
    for (uint32_t t0 = 0; t0 < ntop; t0 += step) {
        uint32_t live = 0;
        if (active) {
#pragma unroll
            for (int u = 0; u < kChunk; ++u) {
                const uint32_t t = t0 + q.sub + (uint32_t)u * q.G;
                if (t < ntop && !(tt.bits[t] & bad)) live |= 1u << u;
            }
        }
        uint32_t any = __reduce_or_sync(0xffffffffu, live);
#pragma unroll 1
        while (any) {
            const int u = __ffs(any) - 1;
            any &= any - 1u;
            bool pending = (live >> u) & 1u;
            uint32_t hh = 0, hi = 0;
            uint64_t kal = 0;
            int jtop = -1;
            if (pending) {
                const uint32_t t = t0 + q.sub + (uint32_t)u * q.G;
                const uint32_t bits = tt.bits[t];
                jtop = (bits >> 16) ? (__ffs(bits >> 16) - 1) : -1;
                const uint64_t p = ph + (uint64_t)tt.dp[t];
                ++q.probes;
                hh = __ldg(ix.dir + p);
                hi = __ldg(ix.dir + p + 1);
                kal = key + (uint64_t)tt.dk[t];
            }
#pragma unroll 1
            while (true) {
                if (pending) {
#pragma unroll 1
                    for (; hh < hi; ++hh) {
                        if (hh == h) continue;                   // home cell handled separately
                        const int64_t dlt = (int64_t)(__ldg(ix.B + hh) - kal);
                        if (dlt > Rl || dlt < -Rl) continue;     // outside the +-1 box
                        if (!low_cell_adjacent_odd<D, UNICOMP>(ix, q.odd, dlt, jtop, L)) continue;
                        const uint32_t a = __ldg(ix.G + hh), b = __ldg(ix.G + hh + 1);
                        if (!q_push<D>(w, a, b - a)) break;      // queue full: resume at hh
                    }
                    pending = hh < hi;
                }
                const bool again = __any_sync(0xffffffffu, pending);
                if (again || *(volatile uint32_t *)w.cnt >= (uint32_t)kQDrainAt)
                    q_drain<D, MODE, UNICOMP>(ix, ja, w, false, q.tests, q.emitted);
                if (!again) break;
            }
        }
    }
    q_drain<D, MODE, UNICOMP>(ix, ja, w, true, q.tests, q.emitted);
}

// The refine for kSearchCellScan indexes without occupancy bitmaps (launch_refine picks it), queued.
template <int D, int MODE, bool UNICOMP, int MINB = kRefineMinBlocks>
__global__ void __launch_bounds__(kRefineThreads, MINB)
k_refine_q(const DevIndex ix, const JoinArgs ja)
{
    __shared__ TopTable tt;
    __shared__ QueueSmem<D> qs;
    build_top_table<D>(ix, tt);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) qs.cnt[warp] = 0;
    __syncthreads();
    WarpQueue<D> w{qs.e[warp], qs.cnt + warp, qs.qx[warp], qs.qid[warp], qs.qem[warp]};
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t qi = t >> ja.lanes_log2;            // G lanes split a query's top offsets
    QueryState<D> q;
    q.valid = true;
    q.G = 1u << ja.lanes_log2;
    q.sub = t & (q.G - 1u);
    q.emitted = q.probes = q.tests = 0;
    uint32_t k;
    bool active;
    if constexpr ((MODE & kModeMask) == kCountQuery) {
        k = ja.q0 + (qi >> 5) * (32u * ja.step) + (qi & 31u);
        active = qi < ja.nsamples && k < ja.q1;
    } else {
        k = ja.q0 + qi;
        active = k < ja.q1;
    }
    uint32_t h = 0, cs = 0, ce = 0;
    if (active) {
        h = __ldg(ix.pcell + k);
        cs = __ldg(ix.G + h);
        ce = __ldg(ix.G + h + 1);
        if ((MODE & kModeMask) == kEmit && ja.dense_T && ce - cs >= ja.dense_T) active = false;
    }
    uint64_t key = 0;
    uint32_t bad = 0xFFFFFFFFu;
    if (active) {
        q.k = k;
        q.pid = __ldg(ix.A + k);
#pragma unroll
        for (int j = 0; j < D; ++j) q.x[j] = __ldg(ix.X + (uint64_t)j * ix.n + k);
        key = __ldg(ix.B + h);
        key_to_coords<D>(ix, key, q.c);
        q.odd = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) q.odd |= (uint32_t)(q.c[j] & 1ull) << j;
#pragma unroll
        for (int j = 0; j < D; ++j) w.qx[lane * D + j] = q.x[j];
        w.qid[lane] = q.pid;
    } else {
        q.pid = 0;
#pragma unroll
        for (int j = 0; j < D; ++j) { q.x[j] = 0.0; q.c[j] = 0; }
        q.odd = 0;
    }
    w.qem[lane] = 0;
    __syncwarp();
    if (active && q.sub == 0) {
        // home cell: (p,p) once; unicomp: q after p in A-order, both orientations (R10); full: all others.
        // (The queue is empty here and a lane pushes <= 2 ranges; ranges of >= 2^24 points -- only with
        // dense_cells = 0 -- go in pieces.)
        if (ja.include_self) emit_self<MODE>(ja, q.k, q.pid, q.emitted);
        for (uint32_t a = k + 1; a < ce; a += (1u << 24) - 1u) q_push<D>(w, a, min(ce - a, (1u << 24) - 1u));
        if (!UNICOMP)
            for (uint32_t a = cs; a < k; a += (1u << 24) - 1u) q_push<D>(w, a, min(k - a, (1u << 24) - 1u));
    }
    if (active) bad = bad_moves<D, UNICOMP>(ix, ja, q, h);
    search_cell_scan_q<D, MODE, UNICOMP>(ix, ja, q, active, h, key, bad, tt, w);
    if constexpr ((MODE & kModeMask) == kCountQuery) {
        __syncwarp();
        q.emitted += w.qem[lane];                    // hits of the ranges this lane queued
        uint32_t e = q.emitted;
        for (uint32_t o = 1; o < q.G; o <<= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
        if (active && q.sub == 0) atomicAdd(ja.qbucket + qi / ja.group, (unsigned long long)e);
    }
    flush_work(ja, q.probes, q.tests, q.emitted);
}

}  // namespace sj
