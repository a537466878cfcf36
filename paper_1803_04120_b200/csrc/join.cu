// join.cu -- host orchestration of the self-join (steps a5, a8 of the hot path).
//
// PAPER.md §5.1 "Batching the Result Set" (line 262): the result may exceed GPU memory, so it is
// produced in incremental batches (minimum 3) whose transfers overlap the computation of later
// batches.  The result-size estimate is inherited from prior work and not described in the
// paper; reading R13: a count-only run of the refine kernel over a deterministic
// strided sample of the queries (>= 1% and >= 1000 points), scaled up; batches are contiguous
// A-order query ranges cut where the sampled prefix crosses multiples of C/(1+margin).  A
// batch whose buffer still overflows is re-run (device mode: exact re-allocation; host mode:
// split in two) -- the result set is invariant to batching.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <atomic>
#include <deque>

#include "refine_launch.cuh"

namespace sj {

namespace {

void launch_dense(const DevIndex &ix, const JoinArgs &ja, bool unicomp, cudaStream_t s)
{
    if (!ja.dense_T || ix.n_dense_tasks == 0) return;
    // tasks intersecting [q0, q1): a whole cell of m >= dense_T points has ceil(m/32) <= m/dense_T
    // tasks, and the two cells cut by the batch ends add at most 2 more each; the kernel strides
    // over its task range anyway (k_refine_dense), so this only sizes the launch
    const uint64_t max_tasks =
        std::min<uint64_t>(ix.n_dense_tasks, (uint64_t)(ja.q1 - ja.q0 + ix.dense_T - 1) / ix.dense_T + 4);
    const dim3 grid((uint32_t)((max_tasks + kDenseWarps - 1) / kDenseWarps));
    switch (ix.d) {
    case 2: launch_dense_d<2>(ix, ja, unicomp, ix.f32 != 0, grid, s); break;
    case 3: launch_dense_d<3>(ix, ja, unicomp, ix.f32 != 0, grid, s); break;
    case 4: launch_dense_d<4>(ix, ja, unicomp, ix.f32 != 0, grid, s); break;
    case 5: launch_dense_d<5>(ix, ja, unicomp, ix.f32 != 0, grid, s); break;
    case 6: launch_dense_d<6>(ix, ja, unicomp, ix.f32 != 0, grid, s); break;
    default: fail(SJ_ERR_DIM, "bad d");
    }
    SJ_LAUNCHED();
}

template <int MODE>
void launch_refine(const DevIndex &ix, const JoinArgs &ja, bool unicomp, uint32_t nqueries, cudaStream_t s)
{
    if (nqueries == 0) return;
    // cell scan without occupancy bitmaps: the queued kernel (candidate ranges tested by converged warps)
    static const bool no_queue = getenv_flag("SJ_NO_QUEUE");
    const bool queued = ix.search_mode == kSearchCellScan && !ix.occ && !no_queue;
    const uint64_t nthreads64 = (uint64_t)nqueries << ja.lanes_log2;
    if (nthreads64 >= (1ull << 32)) fail(SJ_ERR_ARG, "too many queries x lanes for one launch");
    const uint32_t nthreads = (uint32_t)nthreads64;
    const dim3 grid((nthreads + kRefineThreads - 1) / kRefineThreads);
    const bool occ6 = MODE == kEmit && ix.search_mode == kSearchCellScan && !ix.occ && ix.dir_ntop >= 81;
    const int mode = MODE | (ix.f32 ? kF32 : 0);      // the FP32 join's index: binary32 predicate (R21)
    switch (ix.d) {
    case 2: launch_refine_d<2>(mode, ix, ja, unicomp, occ6, queued, grid, s); break;
    case 3: launch_refine_d<3>(mode, ix, ja, unicomp, occ6, queued, grid, s); break;
    case 4: launch_refine_d<4>(mode, ix, ja, unicomp, occ6, queued, grid, s); break;
    case 5: launch_refine_d<5>(mode, ix, ja, unicomp, occ6, queued, grid, s); break;
    case 6: launch_refine_d<6>(mode, ix, ja, unicomp, occ6, queued, grid, s); break;
    default: fail(SJ_ERR_DIM, "bad d");
    }
    SJ_LAUNCHED();
}

void validate(const sj_index *idx, const sj_join_opts &o, uint64_t *qb, uint64_t *qe)
{
    if (o.lanes_per_query != 0 && (o.lanes_per_query < 1 || o.lanes_per_query > 32 ||
                                   (o.lanes_per_query & (o.lanes_per_query - 1))))
        fail(SJ_ERR_ARG, "lanes_per_query must be 0 (auto) or a power of two <= 32");
    if (!idx) fail(SJ_ERR_STATE, "index is NULL");
    if (o.min_batches < 1 || o.min_batches > 1 << 20) fail(SJ_ERR_ARG, "min_batches must be >= 1");
    if (o.n_streams < 1 || o.n_streams > 32) fail(SJ_ERR_ARG, "n_streams must be in [1,32]");
    if (o.batch_capacity_pairs < 1) fail(SJ_ERR_ARG, "batch_capacity_pairs must be >= 1");
    if (o.drain_csr && !o.result_on_host) fail(SJ_ERR_ARG, "drain_csr requires result_on_host = 1");
    const uint64_t n = idx->view.n;
    uint64_t b = o.query_begin, e = o.query_end;
    if (b == 0 && e == 0) e = n;
    if (b > e || e > n) fail(SJ_ERR_ARG, "query range outside [0, N)");
    *qb = b;
    *qe = e;
}

}  // namespace

// ------------------------------------------------------------------ batch planner (host only)
// Bucket i stands for queries [q0 + i*width, min(q1, q0 + (i+1)*width)) with estimated output
// bucket_est[i].  Cut points are placed at bucket boundaries where the running estimate crosses
// multiples of total/k, k = max(min_batches, ceil(total / (capacity/(1+margin)))); a bucket whose
// estimate alone exceeds the target is split evenly (it is not sampled any finer).
#ifndef SJ_PLAN_MARGIN
#define SJ_PLAN_MARGIN 0.75   // batches target C / 1.75: the sampled per-batch estimates of skewed data miss by up
                              // to ~50 % (C4 2-D eps=0.02: margin 0.25 -> 3 overflow re-runs in 14 batches,
                              // 31.2 ms; 0.5 -> 2 in 17, 27.0 ms; 0.75 -> none in 20, 24.7 ms; C3 eps=24
                              // 198 -> 188 ms; C2 2-D unchanged)
#endif
void plan_from_buckets(const double *bucket_est, uint64_t nbk, uint64_t width, uint64_t q0, uint64_t q1,
                       uint64_t capacity, int min_batches, double margin, std::vector<uint64_t> &cuts,
                       std::vector<uint64_t> &est, uint64_t *estimated_total)
{
    cuts.clear();
    est.clear();
    const uint64_t nq = q1 - q0;
    {
        // fast path (the join's common case, on its critical path): no bucket needs splitting and the
        // estimate cuts already give >= min_batches ranges -- then every bucket lies in one range and
        // the general walk below reduces to one pass (same cuts, same estimates)
        const double target = std::max(1.0, (double)capacity / (1.0 + margin));
        double total = 0, mx = 0;
        uint64_t nu = 0;
        for (uint64_t s = 0; s < nbk && q0 + s * width < q1; ++s, ++nu) {
            total += bucket_est[s];
            mx = std::max(mx, bucket_est[s]);
        }
        if (nq > 0 && total > 0 && nu > 0 && !(mx > target)) {
            uint64_t k = std::max<uint64_t>((uint64_t)min_batches, (uint64_t)std::ceil(total / target));
            k = std::min<uint64_t>(k, nq);
            const double per = total / (double)k;
            cuts.push_back(q0);
            double acc = 0;
            for (uint64_t u = 0; u + 1 < nu; ++u) {
                acc += bucket_est[u];
                const uint64_t b = std::min(q1, q0 + (u + 1) * width);
                if (acc >= per * (double)cuts.size() && b > cuts.back()) cuts.push_back(b);
            }
            if (q1 > cuts.back() || cuts.size() == 1) cuts.push_back(q1);
            if (cuts.size() - 1 >= (size_t)min_batches) {
                std::vector<double> e(cuts.size() - 1, 0.0);
                size_t r = 0;
                for (uint64_t u = 0; u < nu; ++u) {
                    const uint64_t a = q0 + u * width;
                    while (r + 2 < cuts.size() && cuts[r + 1] <= a) ++r;
                    e[r] += bucket_est[u];
                }
                est.resize(e.size());
                for (size_t i = 0; i < e.size(); ++i) est[i] = (uint64_t)std::ceil(e[i]);
                *estimated_total = (uint64_t)std::llround(total);
                return;
            }
            cuts.clear();
        }
    }
    struct Unit { uint64_t a, b; double e; };
    std::vector<Unit> units;
    units.reserve(nbk);
    const double target = std::max(1.0, (double)capacity / (1.0 + margin));
    double total = 0;
    for (uint64_t s = 0; s < nbk; ++s) {
        const uint64_t a = q0 + s * width, b = std::min(q1, a + width);
        if (a >= b) break;
        const double bv = bucket_est[s];
        total += bv;
        if (!(bv > target) || b - a < 2) {
            units.push_back({a, b, bv});
            continue;
        }
        const uint64_t parts = std::min<uint64_t>(b - a, (uint64_t)std::ceil(bv / target));
        for (uint64_t p = 0; p < parts; ++p) {
            const uint64_t ua = a + (b - a) * p / parts, ub = a + (b - a) * (p + 1) / parts;
            units.push_back({ua, ub, bv * (double)(ub - ua) / (double)(b - a)});
        }
    }
    *estimated_total = (uint64_t)std::llround(total);
    cuts.push_back(q0);
    if (nq > 0) {
        uint64_t k = std::max<uint64_t>((uint64_t)min_batches, (uint64_t)std::ceil(total / target));
        k = std::min<uint64_t>(k, nq);
        if (total > 0 && !units.empty()) {
            const double per = total / (double)k;
            double acc = 0;
            for (size_t u = 0; u + 1 < units.size(); ++u) {
                acc += units[u].e;
                if (acc >= per * (double)cuts.size() && units[u].b > cuts.back()) cuts.push_back(units[u].b);
            }
        }
    }
    if (q1 > cuts.back() || cuts.size() == 1) cuts.push_back(q1);
    // enforce the minimum number of batches: split the longest ranges
    while (cuts.size() - 1 < (size_t)min_batches) {
        size_t best = 0;
        uint64_t bl = 0;
        for (size_t i = 0; i + 1 < cuts.size(); ++i)
            if (cuts[i + 1] - cuts[i] > bl) { bl = cuts[i + 1] - cuts[i]; best = i; }
        if (bl < 2) break;
        cuts.insert(cuts.begin() + best + 1, cuts[best] + bl / 2);
    }
    // per-range estimates: one merge walk over units and ranges (units only straddle a cut made by
    // the min-batches split; their estimate is then shared by query count)
    est.assign(cuts.size() - 1, 0);
    std::vector<double> e(cuts.size() - 1, 0.0);
    size_t r = 0;
    for (const Unit &u : units) {
        uint64_t a = u.a;
        while (a < u.b) {
            while (r + 1 < cuts.size() - 1 && cuts[r + 1] <= a) ++r;
            const uint64_t b = std::min(u.b, cuts[r + 1]);
            e[r] += (b - a == u.b - u.a) ? u.e : u.e * (double)(b - a) / (double)(u.b - u.a);
            a = b;
            if (r + 1 >= cuts.size() - 1) {     // last range takes the rest
                if (a < u.b) e[r] += u.e * (double)(u.b - a) / (double)(u.b - u.a);
                break;
            }
        }
    }
    for (size_t i = 0; i < e.size(); ++i) est[i] = (uint64_t)std::ceil(e[i]);
}

// Counts of a strided sample (sample s = query q0 + s*step, standing for `step` queries).
void plan_batches(const uint32_t *cnt, uint64_t ns, uint64_t step, uint64_t q0, uint64_t q1, uint64_t capacity,
                  int min_batches, double margin, std::vector<uint64_t> &cuts, std::vector<uint64_t> &est,
                  uint64_t *estimated_total)
{
    // at most ~1024 planning buckets: merge g consecutive samples (cuts need no finer grain)
    const uint64_t g = std::max<uint64_t>(1, (ns + 1023) / 1024);
    const uint64_t nbk = (ns + g - 1) / g;
    std::vector<double> be(nbk, 0.0);
    for (uint64_t s = 0; s < ns; ++s) {
        const uint64_t a = q0 + s * step, b = std::min(q1, a + step);
        if (a < b) be[s / g] += (double)cnt[s] * (double)(b - a);
    }
    plan_from_buckets(be.data(), nbk, step * g, q0, q1, capacity, min_batches, margin, cuts, est, estimated_total);
}

namespace {

struct Sample {
    uint64_t step = 1, ns = 0;
};

// Deterministic sample of >= 1% and >= 1000 queries (SPEC S.260), taken as runs of 32
// consecutive A-order queries every 32*step queries (warp-coherent); each sample stands for
// `step` queries.  ns counts sample slots (multiple of 32; the ragged last run is masked).
Sample make_sample(uint64_t nq)
{
    Sample sm;
    if (nq == 0) return sm;
    const uint64_t target = std::min<uint64_t>(nq, std::max<uint64_t>(1000, (nq + 99) / 100));
    sm.step = std::max<uint64_t>(1, nq / target);
    const uint64_t runs = (nq + 32 * sm.step - 1) / (32 * sm.step);
    sm.ns = runs * 32;
    return sm;
}

// Lanes per query (G): the largest power of two with G * 64 <= per-query work units (top-prefix
// offsets in cell-scan mode, rows otherwise).  Measured on 6-D 2 M: eps=1 (27 offsets) is best at
// G=1 (0.59 ms vs 0.70 at G=2); eps=8 (243 offsets) at G=2-4 (14.8 ms vs 17.0 at G=1).
uint32_t lanes_log2_for(const DevIndex &ix, const sj_join_opts &o)
{
    uint32_t G = (uint32_t)o.lanes_per_query;
    if (G == 0) {
        uint32_t units;
        if (ix.search_mode == kSearchCellScan) {
            units = ix.dir_ntop;
        } else {
            units = 1;
            for (int j = 1; j < ix.d; ++j) units *= 3;
            units -= 1;
        }
        G = 1;
        while (G < 32 && G * 2 * 64 <= units) G *= 2;
    }
    uint32_t l = 0;
    while ((1u << l) < G) ++l;
    return l;
}

JoinArgs base_args(const sj_index *idx, const sj_join_opts &o, unsigned long long *work)
{
    JoinArgs ja{};
    ja.include_self = o.include_self;
    ja.use_masks = o.use_masks;
    ja.work = work;
    ja.lanes_log2 = lanes_log2_for(idx->dev, o);
    return ja;
}

}  // namespace

EstimateShape estimate_shape(uint64_t nq)
{
    const Sample sm = make_sample(nq);
    EstimateShape es;
    es.step = sm.step;
    es.ns = sm.ns;
    es.group = 32 * std::max<uint64_t>(1, (sm.ns / 32 + 1023) / 1024);   // whole runs per bucket
    es.nbk = sm.ns ? (sm.ns + es.group - 1) / es.group : 0;
    return es;
}

// a5: count-only refine over the strided sample of [q0, q1), summed per planning bucket into dbk
// (zeroed by the caller).  A small sample is one partial wave of long per-query chains: each query
// is spread over more lanes (the counts do not depend on the lane split) until the GPU is covered.
void launch_estimate(const DevIndex &ix, int device, const sj_join_opts &o, uint64_t q0, uint64_t q1,
                     const EstimateShape &es, unsigned long long *dbk, cudaStream_t s, const Publish *pub)
{
    if (!es.ns) return;
    JoinArgs ja{};
    ja.include_self = o.include_self;
    ja.use_masks = o.use_masks;
    ja.lanes_log2 = lanes_log2_for(ix, o);
    ja.q0 = (uint32_t)q0;
    ja.q1 = (uint32_t)q1;
    ja.step = (uint32_t)es.step;
    ja.nsamples = (uint32_t)es.ns;
    ja.qbucket = dbk;
    ja.group = (uint32_t)es.group;
    // (many top offsets per query, e.g. 6-D eps=8's 243: up to 16 lanes and 4 K threads per SM --
    //  its estimate 0.45 -> 0.23 ms; few offsets: up to 8 lanes within one wave of 1 K per SM)
    const bool heavy = ix.search_mode == kSearchCellScan && ix.dir_ntop >= 81;
    const uint32_t lanes_max = heavy ? 4u : 3u;
    const uint64_t threads_per_sm = heavy ? 4096 : 1024;
    // (the sparse bitmap search runs G = 1 in the join; for the sample -- a partial wave of long
    // per-query chains -- the lanes' share of the general offset scan, which tests the same bitmaps,
    // is shorter: 6-D eps=1 build 0.347 -> 0.340 ms)
    if (o.lanes_per_query == 0) {
        const int nsm = device_sm_count(device);
        while (ja.lanes_log2 < lanes_max && (es.ns << (ja.lanes_log2 + 1)) <= (uint64_t)nsm * threads_per_sm)
            ++ja.lanes_log2;
    }
    launch_refine<kCountQuery>(ix, ja, o.unicomp != 0, (uint32_t)es.ns, s);
    if (pub) launch_publish(*pub, s);
}

// The build's speculative estimate is valid for a join with the default predicate options over
// the full query range (sj_join_opts_default: unicomp, self pairs, masks, automatic lanes).
static bool spec_estimate_applies(const sj_index *idx, const sj_join_opts &o, uint64_t q0, uint64_t q1)
{
    return idx->spec_est_valid && o.unicomp == 1 && o.include_self == 1 && o.use_masks == 1 &&
           o.lanes_per_query == 0 && q0 == 0 && q1 == idx->view.n;
}

sj_result *self_join_impl(const sj_index *idx, const sj_join_opts &o)
{
    uint64_t q0, q1;
    validate(idx, o, &q0, &q1);
    const auto t_begin = std::chrono::steady_clock::now();
    HostTrace tr("join");
    SJ_CUDA(cudaSetDevice(idx->device));
    const DevIndex &ix = idx->dev;
    const int S = o.n_streams;

    // per-call execution context (pooled): S streams, events, slot buffers
    struct Slot { unsigned long long cursor; uint32_t overflow; uint32_t pad; };
    constexpr size_t kWorkBytes = sizeof(unsigned long long) * 4 * kWorkSlots;   // work counter slots
    const uint64_t nq = q1 - q0;
    const bool spec = spec_estimate_applies(idx, o, q0, q1);   // estimate already done by the build
    const EstimateShape es = spec ? idx->spec_shape : estimate_shape(nq);
    const uint64_t nbk = es.nbk;
    const size_t kSlotsBytes = sizeof(Slot) * 64;
    // per stream ONE block [work counters | 64 batch slots], mirrored in pinned memory: each stream
    // zeroes its own block before its first batch and copies it back after its last one, so no
    // stream waits for another (no event hops on the GPU between the batches and the read-back)
    const size_t kBlock = kWorkBytes + kSlotsBytes;
    const size_t slot_need = 8 * (size_t)(nbk + 1);
    // host drain: S more streams, one copy stream per compute stream (the drain of a batch overlaps the
    // next batch's refine on the same compute stream: double-buffered staging)
    CtxGuard cg{acquire_ctx(idx->device, o.result_on_host ? 2 * S : S, S + 2, slot_need)};
    DevCtx &cx = *cg.c;
    cudaStream_t s0 = cx.streams[0];
    ensure_join_blocks(&cx, kBlock * (size_t)S + 64 * (size_t)S);   // + per stream a CTA counter / doorbell
    const unsigned int bell_epoch = ++cx.doorbell;
    char *dbase = static_cast<char *>(cx.jb_d), *hbase = static_cast<char *>(cx.jb_h);
    auto dwork = [&](int si) { return reinterpret_cast<unsigned long long *>(dbase + kBlock * si); };
    auto hwork = [&](int si) { return reinterpret_cast<const unsigned long long *>(hbase + kBlock * si); };
    auto dslot = [&](int si, size_t j) { return reinterpret_cast<Slot *>(dbase + kBlock * si + kWorkBytes) + j; };
    auto hslot = [&](int si, size_t j) { return reinterpret_cast<Slot *>(hbase + kBlock * si + kWorkBytes) + j; };
    unsigned long long *dbk = static_cast<unsigned long long *>(cx.d_slots);
    unsigned long long *hbk = static_cast<unsigned long long *>(cx.h_slots);
    tr.mark("acquire ctx");
    sj_result *res = new sj_result();
    res->device = idx->device;
    res->n_points = idx->view.n;
    res->q0 = q0;
    res->q1 = q1;
    res->include_self = o.include_self;
    res->unicomp = o.unicomp;
    sj_stats &stats = res->stats;
    // self pairs of a batch [a, b): written at fixed slots, counted on the host (see JoinArgs::nself)
    auto nself_of = [&](uint64_t a, uint64_t b) -> uint64_t { return o.include_self ? b - a : 0; };
    try {
        // the blocks are zero when the previous join on this context re-zeroed them after reading them
        if (!cx.jb_clean)
            for (int i = 0; i < S; ++i) SJ_CUDA(cudaMemsetAsync(dwork(i), 0, kBlock, cx.streams[i]));
        cx.jb_clean = false;
        if (!spec && es.ns) SJ_CUDA(cudaMemsetAsync(dbk, 0, 8 * nbk, s0));
        // ---- a5: estimate on a strided sample (count-only refine), summed per planning bucket
        // (an index built for the default join already carries it: no launch, no round trip)
        const unsigned long long *bk = hbk;
        if (spec) {
            bk = idx->spec_buckets.data();          // the build's counts: no copy
        } else if (es.ns) {
            res->est_ev[0] = event_get(idx->device);
            res->est_ev[1] = event_get(idx->device);
            tr.dev("start", s0);
            SJ_CUDA(cudaEventRecord(res->est_ev[0], s0));
            launch_estimate(ix, idx->device, o, q0, q1, es, dbk, s0);
            tr.dev("estimate", s0);
            SJ_CUDA(cudaEventRecord(res->est_ev[1], s0));
            SJ_CUDA(cudaMemcpyAsync(hbk, dbk, nbk * 8, cudaMemcpyDeviceToHost, s0));
            SJ_CUDA(cudaStreamSynchronize(s0));
        }
        tr.dev("join start", s0);
        tr.mark("estimate (synced)");

        // ---- plan (k >= min_batches contiguous A-order ranges)
        std::vector<uint64_t> cuts, est;
        uint64_t est_total = 0;
        {
            std::vector<double> be(nbk);
            for (uint64_t i = 0; i < nbk; ++i) be[i] = (double)bk[i] * (double)es.step;
            plan_from_buckets(be.data(), nbk, es.step * es.group, q0, q1, o.batch_capacity_pairs, o.min_batches, SJ_PLAN_MARGIN,
                              cuts, est, &est_total);
        }
        stats.estimated_pairs = est_total;
        const size_t nb = cuts.size() - 1;
        tr.mark("plan");

        bool work_read = false;
        uint32_t launches = 0;
        unsigned long long wsum[3] = {0, 0, 0};
        auto add_work = [&]() {
            for (int si = 0; si < S; ++si)
                for (int sl = 0; sl < kWorkSlots; ++sl)
                    for (int i = 0; i < 3; ++i) wsum[i] += hwork(si)[4 * sl + i];
        };
        // every batch run records a (start, end) event pair; timings are computed on request
        auto run_batch = [&](uint64_t a, uint64_t b, uint64_t *buf, uint64_t cap, Slot *dslot, int si,
                             bool clear_slot, const Publish *pub = nullptr) {
            cudaStream_t s = cx.streams[si];
            cudaEvent_t e0 = event_get(idx->device), e1 = event_get(idx->device);
            res->runs.emplace_back(e0, e1);
            if (clear_slot) SJ_CUDA(cudaMemsetAsync(dslot, 0, sizeof(Slot), s));
            JoinArgs ja = base_args(idx, o, dwork(si));
            ja.out = buf;
            ja.cap = cap;
            ja.cursor = &dslot->cursor;
            ja.overflow = &dslot->overflow;
            ja.q0 = (uint32_t)a;
            ja.q1 = (uint32_t)b;
            ja.nself = o.include_self ? (uint32_t)(b - a) : 0u;
            if (!res->span0) {
                res->span0 = event_get(idx->device);
                SJ_CUDA(cudaEventRecord(res->span0, s));
            }
            if (o.dense_cells && ix.n_dense_tasks) {
                ja.dense_T = ix.dense_T;
                ja.dense_tasks = ix.dense_tasks;
                ja.n_dense_tasks = ix.n_dense_tasks;
            }
            SJ_CUDA(cudaEventRecord(e0, s));
            tr.dev("refine launch", s);
            launch_refine<kEmit>(ix, ja, o.unicomp != 0, (uint32_t)(b - a), s);
            launch_dense(ix, ja, o.unicomp != 0, s);
            if (pub) launch_publish(*pub, s);      // the stream's counters to the host behind the batch
            SJ_CUDA(cudaEventRecord(e1, s));
            tr.dev("refine done", s);
            ++launches;
        };

        if (!o.result_on_host) {
            // ---- device-resident batches: every batch owns its buffer; streams run them
            //      concurrently.  Batch b runs on stream b % S; up to 64 batches per stream own a
            //      cursor slot each in that stream's block (zeroed by its memset), read back with the
            //      stream's work counters by ONE copy after its last batch; beyond that slot 0 of the
            //      stream is reused in order and read back per batch.
            res->batches.resize(nb);
            std::vector<uint64_t> counts(nb, 0);
            const bool own_slots = nb <= (size_t)64 * S;
            static const bool no_pub = getenv_flag("SJ_NO_PUB");
            // the batches' buffers first (host bookkeeping), so the launches then go out back to back
            if (own_slots) {
                for (size_t b = 0; b < nb; ++b) {
                    const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(
                        o.batch_capacity_pairs, est[b] + est[b] / 4 + 65536));
                    sj_batch &bt = res->batches[b];
                    bt.pairs = static_cast<uint64_t *>(
                        result_buffer_get(idx->device, cap * sizeof(uint64_t), cx.streams[b % S]));
                    bt.cap = cap;
                    bt.on_device = 1;
                }
            }
            for (size_t b = 0; b < nb; ++b) {
                const int si = (int)(b % S);
                cudaStream_t s = cx.streams[si];
                const size_t slot = own_slots ? b / S : 0;
                if (own_slots) {
                    sj_batch &bt = res->batches[b];
                    if (b + S >= nb && !no_pub) {
                        // the stream's last batch: its last CTA publishes the stream's block into the
                        // mapped mirror, zeroes it for the next join and rings the stream's doorbell
                        Publish pb{};
                        pb.src = reinterpret_cast<unsigned long long *>(dbase + kBlock * si);
                        pb.dst = reinterpret_cast<unsigned long long *>(static_cast<char *>(cx.jb_hd) + kBlock * si);
                        pb.words = (uint32_t)(kBlock / 8);
                        pb.zero_src = 1;
                        pb.reduce_slots = kWorkSlots;
                        pb.nslots = (uint32_t)((nb - 1 - si) / S + 1);     // this stream's batches
                        pb.bell = reinterpret_cast<volatile unsigned int *>(static_cast<char *>(cx.jb_hd) + kBlock * S) + 16 * si;
                        pb.epoch = bell_epoch;
                        run_batch(cuts[b], cuts[b + 1], bt.pairs, bt.cap, dslot(si, slot), si, false, &pb);
                    } else {
                        run_batch(cuts[b], cuts[b + 1], bt.pairs, bt.cap, dslot(si, slot), si, false);
                        if (b + S >= nb) {            // (SJ_NO_PUB: copy + event + zeroing instead)
                            SJ_CUDA(cudaMemcpyAsync(hbase + kBlock * si, dbase + kBlock * si, kBlock,
                                                    cudaMemcpyDeviceToHost, s));
                            SJ_CUDA(cudaEventRecord(cx.events[2 + si], s));
                            SJ_CUDA(cudaMemsetAsync(dbase + kBlock * si, 0, kBlock, s));
                        }
                    }
                    continue;
                }
                if (!own_slots && b >= (size_t)S) {   // stream si's previous batch must have published its cursor
                    SJ_CUDA(cudaStreamSynchronize(s));
                    counts[b - S] = hslot(si, 0)->cursor;   // (+ the batch's self pairs below)
                }
                const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(
                    o.batch_capacity_pairs, est[b] + est[b] / 4 + 65536));
                sj_batch &bt = res->batches[b];
                bt.pairs = static_cast<uint64_t *>(result_buffer_get(idx->device, cap * sizeof(uint64_t), s));
                bt.cap = cap;
                bt.on_device = 1;
                run_batch(cuts[b], cuts[b + 1], bt.pairs, cap, dslot(si, slot), si, !own_slots);
                if (!own_slots)
                    SJ_CUDA(cudaMemcpyAsync(hslot(si, 0), dslot(si, 0), sizeof(Slot), cudaMemcpyDeviceToHost, s));
                if (b + S >= nb) {                    // the stream's last batch: its block back to the host,
                    SJ_CUDA(cudaMemcpyAsync(hbase + kBlock * si, dbase + kBlock * si, kBlock, cudaMemcpyDeviceToHost, s));
                    // then zeroed for the next join on this context (off the critical path)
                    SJ_CUDA(cudaMemsetAsync(dbase + kBlock * si, 0, kBlock, s));
                }
            }
            tr.mark("batches launched");
            // wait for the streams' doorbells (own slots) or the streams
            for (int i = 0; i < S && i < (int)nb; ++i) {
                if (own_slots && no_pub) {
                    SJ_CUDA(cudaEventSynchronize(cx.events[2 + i]));
                } else if (own_slots) {
                    const volatile unsigned int *bell =
                        reinterpret_cast<const volatile unsigned int *>(hbase + kBlock * S) + 16 * i;
                    if (!wait_doorbell(bell, bell_epoch, cx.streams[i]))
                        fail(SJ_ERR_CUDA, "a batch finished without publishing its counters (internal error)");
                } else {
                    SJ_CUDA(cudaStreamSynchronize(cx.streams[i]));
                }
            }
            std::atomic_thread_fence(std::memory_order_acquire);
            tr.mark("batches done (synced)");
            const bool published = own_slots && !no_pub;
            if (published) {
                // each stream's published [work sums | cursor slots]
                for (int i = 0; i < S && i < (int)nb; ++i) {
                    const unsigned long long *pw = reinterpret_cast<const unsigned long long *>(hbase + kBlock * i);
                    for (int c = 0; c < 3; ++c) wsum[c] += pw[c];
                }
            } else {
                add_work();                       // (the device blocks are being zeroed behind the copies)
            }
            work_read = true;
            cudaStream_t st_sort = s0;
            if (published) {
                for (size_t b = 0; b < nb; ++b)
                    counts[b] = reinterpret_cast<const unsigned long long *>(hbase + kBlock * (b % S))[4 + 2 * (b / S)];
            } else if (own_slots) {
                for (size_t b = 0; b < nb; ++b) counts[b] = hslot((int)(b % S), b / S)->cursor;
            } else {
                for (size_t b = (nb > (size_t)S ? nb - S : 0); b < nb; ++b) counts[b] = hslot((int)(b % S), 0)->cursor;
            }
            for (size_t b = 0; b < nb; ++b) counts[b] += nself_of(cuts[b], cuts[b + 1]);
            // overflowed batches (estimate too low): exact re-allocation, all re-runs launched
            // together across the streams (slot 0 of every stream is free again), one sync per round
            std::vector<size_t> redo;
            for (size_t b = 0; b < nb; ++b)
                if (counts[b] > res->batches[b].cap) redo.push_back(b);
            for (size_t r0 = 0; r0 < redo.size(); r0 += (size_t)S) {
                const size_t r1 = std::min(redo.size(), r0 + (size_t)S);
                for (size_t r = r0; r < r1; ++r) {
                    const size_t b = redo[r];
                    const int si = (int)(r - r0);
                    cudaStream_t st = cx.streams[si];
                    sj_batch &bt = res->batches[b];
                    result_buffer_put(idx->device, bt.pairs, st);
                    bt.pairs = static_cast<uint64_t *>(result_buffer_get(idx->device, counts[b] * sizeof(uint64_t), st));
                    bt.cap = counts[b];
                    run_batch(cuts[b], cuts[b + 1], bt.pairs, bt.cap, dslot(si, 0), si, true);
                    SJ_CUDA(cudaMemcpyAsync(hslot(si, 0), dslot(si, 0), sizeof(Slot), cudaMemcpyDeviceToHost, st));
                    ++stats.retries;
                }
                for (size_t r = r0; r < r1; ++r) SJ_CUDA(cudaStreamSynchronize(cx.streams[r - r0]));
                for (size_t r = r0; r < r1; ++r) {
                    const size_t b = redo[r];
                    const uint64_t n = hslot((int)(r - r0), 0)->cursor + nself_of(cuts[b], cuts[b + 1]);
                    if (n != counts[b]) fail(SJ_ERR_CUDA, "batch re-run produced a different count");
                }
            }
            for (size_t b = 0; b < nb; ++b) {
                sj_batch &bt = res->batches[b];
                bt.n = counts[b];
                res->total += bt.n;
                if (o.sort_pairs) sort_pairs_device(bt.pairs, bt.n, ix.n, st_sort);
            }
            tr.mark("batch loop");
        } else {
            // ---- host-drained batches: S device staging buffers; batch b+S on a stream runs after
            //      the D2H of batch b (stream order), while other streams compute.
            uint64_t maxest = 0;
            for (auto e : est) maxest = std::max(maxest, e);
            uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(o.batch_capacity_pairs,
                                                                    maxest + maxest / 4 + 65536));
            if (o.drain_csr) cap = std::min<uint64_t>(cap, 0xffffffffull);   // uint32 row offsets
            // two staging buffers per compute stream i (parity p): batch k+1 on stream i refines into
            // buffer p^1 while the copy stream S+i converts / drains buffer p; stream i waits for the
            // copy stream's event on a buffer before it overwrites it
            const int S2 = 2 * S;
            std::vector<uint64_t *> staging(S2, nullptr);
            std::vector<uint64_t> scap(S2, cap);          // per-buffer staging capacity
            std::vector<int> parity(S, 0);
            std::vector<cudaEvent_t> copied(S2, nullptr), computed(S, nullptr);
            struct StagingGuard {
                std::vector<uint64_t *> &v; std::vector<cudaEvent_t> &e1, &e2; DevCtx &cx; int dev;
                ~StagingGuard() {
                    for (size_t i = 0; i < v.size(); ++i) if (v[i]) dev_free(v[i], cx.streams[i / 2]);   // buffer 2s+p: stream s
                    for (auto e : e1) event_put(dev, e);
                    for (auto e : e2) event_put(dev, e);
                }
            } sg{staging, copied, computed, cx, idx->device};
            for (int i = 0; i < S2; ++i) staging[i] = dalloc<uint64_t>(cap, cx.streams[i / 2]);
            for (int i = 0; i < S; ++i) computed[i] = event_get(idx->device);
            // drain_csr: per buffer the CSR of the finished batch is built in device memory
            // ([offsets | neighbours] contiguous, one D2H copy) with two N+1 scratch arrays per copy stream
            const uint64_t rows = ix.n;
            std::vector<uint32_t *> csr_blk(S2, nullptr), csr_tmp(S, nullptr);
            struct CsrGuard {
                std::vector<uint32_t *> &a, &b; DevCtx &cx;
                ~CsrGuard() {
                    for (size_t i = 0; i < a.size(); ++i) if (a[i]) dev_free(a[i], cx.streams[i / 2]);
                    for (size_t i = 0; i < b.size(); ++i) if (b[i]) dev_free(b[i], cx.streams[i]);
                }
            } cgd{csr_blk, csr_tmp, cx};
            if (o.drain_csr) {
                for (int i = 0; i < S2; ++i) csr_blk[i] = dalloc<uint32_t>(rows + 1 + cap, cx.streams[i / 2]);
                for (int i = 0; i < S; ++i) csr_tmp[i] = dalloc<uint32_t>(2 * (rows + 1), cx.streams[i]);
            }
            const int nsm = device_sm_count(idx->device);
            std::deque<std::pair<uint64_t, uint64_t>> pending;
            for (size_t b = 0; b < nb; ++b) pending.emplace_back(cuts[b], cuts[b + 1]);
            std::vector<std::pair<uint64_t, uint64_t>> inflight(S, {0, 0});
            std::deque<int> order;  // streams in launch order
            auto launch_on = [&](int i) {
                auto r = pending.front();
                pending.pop_front();
                inflight[i] = r;
                const int bi = 2 * i + parity[i];
                if (copied[bi]) SJ_CUDA(cudaStreamWaitEvent(cx.streams[i], copied[bi], 0));   // its last drain
                run_batch(r.first, r.second, staging[bi], scap[bi], dslot(i, 0), i, true);
                SJ_CUDA(cudaMemcpyAsync(hslot(i, 0), dslot(i, 0), sizeof(Slot), cudaMemcpyDeviceToHost,
                                        cx.streams[i]));
                order.push_back(i);
            };
            for (int i = 0; i < S && !pending.empty(); ++i) launch_on(i);
            while (!order.empty()) {
                const int i = order.front();
                order.pop_front();
                // the cursor copy follows the kernel on stream i: a stream sync waits for exactly that
                // batch (its drain, on the copy stream, is not on stream i)
                SJ_CUDA(cudaStreamSynchronize(cx.streams[i]));
                const auto r = inflight[i];
                const int bi = 2 * i + parity[i];
                cudaStream_t cs = cx.streams[S + i];
                const uint64_t n = hslot(i, 0)->cursor + nself_of(r.first, r.second);
                if (n > scap[bi]) {
                    ++stats.retries;
                    if (r.second - r.first < 2) {
                        // one query emits more than the staging buffer holds: grow it to fit
                        if (o.drain_csr && n > 0xffffffffull)
                            fail(SJ_ERR_ARG, "drain_csr: one query emits >= 2^32 pairs");
                        if (copied[bi]) SJ_CUDA(cudaStreamWaitEvent(cx.streams[i], copied[bi], 0));
                        dev_free(staging[bi], cx.streams[i]);
                        staging[bi] = dalloc<uint64_t>(n, cx.streams[i]);
                        scap[bi] = n;
                        if (o.drain_csr) {
                            dev_free(csr_blk[bi], cx.streams[i]);
                            csr_blk[bi] = dalloc<uint32_t>(rows + 1 + n, cx.streams[i]);
                        }
                        pending.emplace_front(r);
                    } else {
                        // overflow: split the query range and re-run both halves first
                        const uint64_t mid = r.first + (r.second - r.first) / 2;
                        pending.emplace_front(mid, r.second);
                        pending.emplace_front(r.first, mid);
                    }
                } else {
                    sj_batch bt;
                    bt.on_device = 0;
                    bt.n = n;
                    bt.cap = n;
                    // the drain on the copy stream, behind the batch's kernels
                    SJ_CUDA(cudaEventRecord(computed[i], cx.streams[i]));
                    SJ_CUDA(cudaStreamWaitEvent(cs, computed[i], 0));
                    if (o.drain_csr) {
                        // 4 B per pair + 4 B per row cross PCIe instead of 8 B per pair
                        if (n && o.sort_pairs) sort_pairs_device(staging[bi], n, ix.n, cs);
                        batch_to_csr_device(staging[bi], n, rows, o.sort_pairs != 0, csr_tmp[i], csr_tmp[i] + rows + 1,
                                            csr_blk[bi], csr_blk[bi] + rows + 1, cs, nsm);
                        const size_t bytes = sizeof(uint32_t) * (rows + 1 + n);
                        bt.pairs = static_cast<uint64_t *>(host_pinned_alloc(bytes, nullptr));
                        bt.csr = 1;
                        bt.rows = rows;
                        SJ_CUDA(cudaMemcpyAsync(bt.pairs, csr_blk[bi], bytes, cudaMemcpyDeviceToHost, cs));
                    } else if (n) {
                        if (o.sort_pairs) sort_pairs_device(staging[bi], n, ix.n, cs);
                        bt.pairs = static_cast<uint64_t *>(host_pinned_alloc(n * sizeof(uint64_t), nullptr));
                        SJ_CUDA(cudaMemcpyAsync(bt.pairs, staging[bi], n * sizeof(uint64_t), cudaMemcpyDeviceToHost, cs));
                    }
                    if (!copied[bi]) copied[bi] = event_get(idx->device);
                    SJ_CUDA(cudaEventRecord(copied[bi], cs));
                    parity[i] ^= 1;
                    res->batches.push_back(bt);
                    res->total += n;
                }
                if (!pending.empty()) launch_on(i);
            }
            for (int i = 0; i < S2; ++i) SJ_CUDA(cudaStreamSynchronize(cx.streams[i]));
        }

        // ---- work counters: the device path read them with its first round; re-runs (which counted
        //      into the re-zeroed blocks) and the host path are read here (every stream is synced)
        if (!work_read || stats.retries) {
            SJ_CUDA(cudaMemcpyAsync(hbase, dbase, kBlock * S, cudaMemcpyDeviceToHost, s0));
            SJ_CUDA(cudaStreamSynchronize(s0));
            add_work();
        }
        cx.jb_clean = work_read && !stats.retries;   // zeroed behind the device path's read-back copies
        stats.cells_probed = wsum[0];
        stats.candidates_tested = wsum[1];
        stats.pairs = res->total;
        stats.batches = (uint32_t)res->batches.size();
        stats.refine_launches = launches;
        tr.mark("stats");
    } catch (...) {
        for (auto s : cx.streams) cudaStreamSynchronize(s);
        result_release_events(res);
        for (auto &b : res->batches) {
            if (!b.pairs) continue;
            if (b.on_device) result_buffer_put(res->device, b.pairs, nullptr);
            else host_pinned_free(b.pairs);
        }
        delete res;
        throw;
    }
    cg.idle = true;                          // every stream was synchronised above
    stats.total_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
    return res;
}

// Multi-GPU shard plan (north_star "Partitioning"): contiguous A-order query ranges
// balanced by the a5 sampled estimate -- per planning bucket, estimated pairs plus kQueryWeight per
// query (the per-query search cost, in units of emitted pairs) -- cut where the cumulative weight
// crosses multiples of total/world, interpolated by query count inside a bucket.  Uses the build's
// estimate of the default join when it carries one, else runs the estimate now.
void plan_shards_impl(const sj_index *idx, uint32_t world, uint64_t *cuts)
{
    if (!idx) fail(SJ_ERR_STATE, "index is NULL");
    if (world < 1 || !cuts) fail(SJ_ERR_ARG, "world must be >= 1 and cuts non-NULL");
    const uint64_t n = idx->view.n;
    constexpr double kQueryWeight = 4.0;
    EstimateShape es;
    std::vector<unsigned long long> bk;
    if (idx->spec_est_valid) {
        es = idx->spec_shape;
        bk = idx->spec_buckets;
    } else {
        SJ_CUDA(cudaSetDevice(idx->device));
        es = estimate_shape(n);
        const size_t bytes = 8 * (size_t)(es.nbk + 1);
        CtxGuard cg{acquire_ctx(idx->device, 1, 0, bytes)};
        cudaStream_t s = cg.c->streams[0];
        auto *dbk = static_cast<unsigned long long *>(cg.c->d_slots);
        SJ_CUDA(cudaMemsetAsync(dbk, 0, bytes, s));
        sj_join_opts o;
        sj_join_opts_default(&o);
        launch_estimate(idx->dev, idx->device, o, 0, n, es, dbk, s);
        SJ_CUDA(cudaMemcpyAsync(cg.c->h_slots, dbk, 8 * es.nbk, cudaMemcpyDeviceToHost, s));
        SJ_CUDA(cudaStreamSynchronize(s));
        const auto *h = static_cast<const unsigned long long *>(cg.c->h_slots);
        bk.assign(h, h + es.nbk);
    }
    const uint64_t width = std::max<uint64_t>(1, es.step * es.group);
    const uint64_t nbk = (n + width - 1) / width;
    std::vector<double> cum(nbk + 1, 0.0);
    for (uint64_t i = 0; i < nbk; ++i) {
        const uint64_t a = i * width, b = std::min(n, a + width);
        const double est = i < bk.size() ? (double)bk[i] * (double)es.step : 0.0;
        cum[i + 1] = cum[i] + est + kQueryWeight * (double)(b - a);
    }
    const double W = cum[nbk];
    cuts[0] = 0;
    uint64_t i = 0;
    for (uint32_t r = 1; r < world; ++r) {
        const double t = W * (double)r / (double)world;
        while (i < nbk && cum[i + 1] < t) ++i;
        uint64_t c = n;
        if (i < nbk) {
            const uint64_t a = i * width, b = std::min(n, a + width);
            const double f = cum[i + 1] > cum[i] ? (t - cum[i]) / (cum[i + 1] - cum[i]) : 0.0;
            c = a + (uint64_t)std::llround(f * (double)(b - a));
        }
        cuts[r] = std::max(cuts[r - 1], std::min(c, n));
    }
    cuts[world] = n;
}

void neighbor_counts_impl(const sj_index *idx, const sj_join_opts &o, uint32_t *cnt, uint64_t *total)
{
    uint64_t q0, q1;
    validate(idx, o, &q0, &q1);
    SJ_CUDA(cudaSetDevice(idx->device));
    constexpr size_t kWorkBytes = sizeof(unsigned long long) * 4 * kWorkSlots;
    CtxGuard cg{acquire_ctx(idx->device, 1, 2, kWorkBytes)};
    DevCtx &cx = *cg.c;
    cudaStream_t s = cx.streams[0];
    unsigned long long *work = static_cast<unsigned long long *>(cx.d_slots);
    unsigned long long *hwork = static_cast<unsigned long long *>(cx.h_slots);
    SJ_CUDA(cudaMemsetAsync(work, 0, kWorkBytes, s));
    Scratch<uint32_t> own_cnt;
    uint32_t *c = cnt;
    if (!c) {
        own_cnt.p = dalloc<uint32_t>(idx->view.n, s);
        own_cnt.s = s;
        c = own_cnt.p;
    }
    SJ_CUDA(cudaMemsetAsync(c, 0, sizeof(uint32_t) * idx->view.n, s));
    JoinArgs ja = base_args(idx, o, work);
    ja.pcount = c;
    ja.q0 = (uint32_t)q0;
    ja.q1 = (uint32_t)q1;
    launch_refine<kCountPoint>(idx->dev, ja, o.unicomp != 0, (uint32_t)(q1 - q0), s);
    SJ_CUDA(cudaMemcpyAsync(hwork, work, kWorkBytes, cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    unsigned long long em = 0;
    for (int sl = 0; sl < kWorkSlots; ++sl) em += hwork[4 * sl + 2];
    if (total) *total = em;
}

}  // namespace sj
