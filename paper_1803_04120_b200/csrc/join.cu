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
#include <deque>

#include "refine.cuh"

namespace sj {

namespace {

template <int MODE>
void launch_refine(const DevIndex &ix, const JoinArgs &ja, bool unicomp, uint32_t nthreads, cudaStream_t s)
{
    if (nthreads == 0) return;
    const dim3 grid((nthreads + kRefineThreads - 1) / kRefineThreads), block(kRefineThreads);
#define SJ_REFINE_CASE(DD)                                                                       \
    case DD:                                                                                     \
        if (unicomp) k_refine<DD, MODE, true><<<grid, block, 0, s>>>(ix, ja);                   \
        else k_refine<DD, MODE, false><<<grid, block, 0, s>>>(ix, ja);                          \
        break;
    switch (ix.d) {
        SJ_REFINE_CASE(2)
        SJ_REFINE_CASE(3)
        SJ_REFINE_CASE(4)
        SJ_REFINE_CASE(5)
        SJ_REFINE_CASE(6)
    default: fail(SJ_ERR_DIM, "bad d");
    }
#undef SJ_REFINE_CASE
    SJ_LAUNCHED();
}

struct Streams {
    std::vector<cudaStream_t> s;
    explicit Streams(int n)
    {
        s.resize(n);
        for (auto &x : s) SJ_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
    }
    ~Streams()
    {
        for (auto x : s) { cudaStreamSynchronize(x); cudaStreamDestroy(x); }
    }
};

struct Ev {
    cudaEvent_t e{};
    Ev() { SJ_CUDA(cudaEventCreate(&e)); }
    ~Ev() { cudaEventDestroy(e); }
    Ev(const Ev &) = delete;
    Ev &operator=(const Ev &) = delete;
};

void validate(const sj_index *idx, const sj_join_opts &o, uint64_t *qb, uint64_t *qe)
{
    if (!idx) fail(SJ_ERR_STATE, "index is NULL");
    if (o.min_batches < 1 || o.min_batches > 1 << 20) fail(SJ_ERR_ARG, "min_batches must be >= 1");
    if (o.n_streams < 1 || o.n_streams > 32) fail(SJ_ERR_ARG, "n_streams must be in [1,32]");
    if (o.batch_capacity_pairs < 1) fail(SJ_ERR_ARG, "batch_capacity_pairs must be >= 1");
    const uint64_t n = idx->view.n;
    uint64_t b = o.query_begin, e = o.query_end;
    if (b == 0 && e == 0) e = n;
    if (b > e || e > n) fail(SJ_ERR_ARG, "query range outside [0, N)");
    *qb = b;
    *qe = e;
}

}  // namespace

// ------------------------------------------------------------------ batch planner (host only)
void plan_batches(const uint32_t *cnt, uint64_t ns, uint64_t step, uint64_t q0, uint64_t q1, uint64_t capacity,
                  int min_batches, double margin, std::vector<uint64_t> &cuts, std::vector<uint64_t> &est,
                  uint64_t *estimated_total)
{
    cuts.clear();
    est.clear();
    const uint64_t nq = q1 - q0;
    struct Unit { uint64_t a, b; double e; };
    std::vector<Unit> units;
    const double target = std::max(1.0, (double)capacity / (1.0 + margin));
    double total = 0;
    // sample s stands for queries [q0 + s*step, min(q1, q0 + (s+1)*step)); a unit whose estimate
    // alone exceeds the target is split evenly (it is not sampled any finer)
    for (uint64_t s = 0; s < ns; ++s) {
        const uint64_t a = q0 + s * step, b = std::min(q1, a + step);
        if (a >= b) break;
        const double bv = (double)cnt[s] * (double)(b - a);
        total += bv;
        uint64_t parts = 1;
        if (bv > target) parts = std::min<uint64_t>(b - a, (uint64_t)std::ceil(bv / target));
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
    for (size_t i = 0; i + 1 < cuts.size(); ++i) {
        double e = 0;
        for (const Unit &u : units) {
            const uint64_t lo = std::max(u.a, cuts[i]), hi = std::min(u.b, cuts[i + 1]);
            if (hi > lo) e += u.e * (double)(hi - lo) / (double)(u.b - u.a);
        }
        est.push_back((uint64_t)std::ceil(e));
    }
}

namespace {

struct Sample {
    uint64_t step = 1, ns = 0;
};

Sample make_sample(uint64_t nq)
{
    Sample sm;
    if (nq == 0) return sm;
    const uint64_t target = std::min<uint64_t>(nq, std::max<uint64_t>(1000, (nq + 99) / 100));
    sm.step = std::max<uint64_t>(1, nq / target);
    sm.ns = (nq + sm.step - 1) / sm.step;
    return sm;
}

JoinArgs base_args(const sj_join_opts &o, unsigned long long *work)
{
    JoinArgs ja{};
    ja.include_self = o.include_self;
    ja.use_masks = o.use_masks;
    ja.work = work;
    return ja;
}

}  // namespace

sj_result *self_join_impl(const sj_index *idx, const sj_join_opts &o)
{
    uint64_t q0, q1;
    validate(idx, o, &q0, &q1);
    const auto t_begin = std::chrono::steady_clock::now();
    SJ_CUDA(cudaSetDevice(idx->device));
    const DevIndex &ix = idx->dev;
    const int S = o.n_streams;
    Streams st(S);
    cudaStream_t s0 = st.s[0];

    sj_result *res = new sj_result();
    res->device = idx->device;
    sj_stats &stats = res->stats;
    try {
        Scratch<unsigned long long> work(4, s0);
        SJ_CUDA(cudaMemsetAsync(work.p, 0, 4 * sizeof(unsigned long long), s0));

        // ---- a5: estimate on a strided sample (count-only refine)
        const uint64_t nq = q1 - q0;
        const Sample sm = make_sample(nq);
        std::vector<uint32_t> hcnt(sm.ns ? sm.ns : 1, 0);
        float est_ms = 0;
        if (sm.ns) {
            Scratch<uint32_t> qcount(sm.ns, s0);
            JoinArgs ja = base_args(o, nullptr);
            ja.q0 = (uint32_t)q0;
            ja.q1 = (uint32_t)q1;
            ja.step = (uint32_t)sm.step;
            ja.nsamples = (uint32_t)sm.ns;
            ja.qcount = qcount.p;
            Ev a, b;
            SJ_CUDA(cudaEventRecord(a.e, s0));
            launch_refine<kCountQuery>(ix, ja, o.unicomp != 0, (uint32_t)sm.ns, s0);
            SJ_CUDA(cudaEventRecord(b.e, s0));
            SJ_CUDA(cudaMemcpyAsync(hcnt.data(), qcount.p, sm.ns * sizeof(uint32_t), cudaMemcpyDeviceToHost, s0));
            SJ_CUDA(cudaStreamSynchronize(s0));
            SJ_CUDA(cudaEventElapsedTime(&est_ms, a.e, b.e));
        }
        stats.estimate_ms = est_ms;

        // ---- plan
        std::vector<uint64_t> cuts, est;
        uint64_t est_total = 0;
        plan_batches(hcnt.data(), sm.ns, sm.step, q0, q1, o.batch_capacity_pairs, o.min_batches, 0.25, cuts, est,
                     &est_total);
        stats.estimated_pairs = est_total;
        const size_t nb = cuts.size() - 1;

        // per-batch cursor/overflow slots, pinned host mirror of the cursors
        struct Slot { unsigned long long cursor; uint32_t overflow; uint32_t pad; };
        float refine_ms = 0, refine_max = 0;
        uint32_t launches = 0;

        auto run_batch = [&](uint64_t a, uint64_t b, uint64_t *buf, uint64_t cap, Slot *dslot, cudaStream_t s,
                             cudaEvent_t e0, cudaEvent_t e1) {
            SJ_CUDA(cudaMemsetAsync(dslot, 0, sizeof(Slot), s));
            JoinArgs ja = base_args(o, work.p);
            ja.out = buf;
            ja.cap = cap;
            ja.cursor = &dslot->cursor;
            ja.overflow = &dslot->overflow;
            ja.q0 = (uint32_t)a;
            ja.q1 = (uint32_t)b;
            SJ_CUDA(cudaEventRecord(e0, s));
            launch_refine<kEmit>(ix, ja, o.unicomp != 0, (uint32_t)(b - a), s);
            SJ_CUDA(cudaEventRecord(e1, s));
            ++launches;
        };
        auto add_time = [&](cudaEvent_t e0, cudaEvent_t e1) {
            float ms = 0;
            SJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            refine_ms += ms;
            refine_max = std::max(refine_max, ms);
        };

        if (!o.result_on_host) {
            // ---- device-resident batches: every batch owns its buffer; all run concurrently
            Scratch<Slot> slots(nb, s0);
            SJ_CUDA(cudaStreamSynchronize(s0));
            Slot *hslots = static_cast<Slot *>(host_pinned_alloc(sizeof(Slot) * nb, nullptr));
            std::vector<Ev> e0(nb), e1(nb);
            res->batches.resize(nb);
            for (size_t b = 0; b < nb; ++b) {
                cudaStream_t s = st.s[b % S];
                const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(
                    o.batch_capacity_pairs, est[b] + est[b] / 4 + 65536));
                sj_batch &bt = res->batches[b];
                bt.pairs = dalloc<uint64_t>(cap, s);
                bt.cap = cap;
                bt.on_device = 1;
                run_batch(cuts[b], cuts[b + 1], bt.pairs, cap, slots.p + b, s, e0[b].e, e1[b].e);
                SJ_CUDA(cudaMemcpyAsync(hslots + b, slots.p + b, sizeof(Slot), cudaMemcpyDeviceToHost, s));
            }
            for (int i = 0; i < S; ++i) SJ_CUDA(cudaStreamSynchronize(st.s[i]));
            for (size_t b = 0; b < nb; ++b) {
                add_time(e0[b].e, e1[b].e);
                sj_batch &bt = res->batches[b];
                uint64_t n = hslots[b].cursor;
                if (n > bt.cap) {  // overflow: exact re-allocation and re-run
                    cudaStream_t s = st.s[0];
                    dev_free(bt.pairs, s);
                    bt.pairs = dalloc<uint64_t>(n, s);
                    bt.cap = n;
                    run_batch(cuts[b], cuts[b + 1], bt.pairs, n, slots.p + b, s, e0[b].e, e1[b].e);
                    SJ_CUDA(cudaMemcpyAsync(hslots + b, slots.p + b, sizeof(Slot), cudaMemcpyDeviceToHost, s));
                    SJ_CUDA(cudaStreamSynchronize(s));
                    add_time(e0[b].e, e1[b].e);
                    ++stats.retries;
                    n = hslots[b].cursor;
                    if (n > bt.cap) { host_pinned_free(hslots); fail(SJ_ERR_CUDA, "batch re-run overflowed"); }
                }
                bt.n = n;
                res->total += n;
            }
            host_pinned_free(hslots);
        } else {
            // ---- host-drained batches: S device staging buffers; batch b+S on a stream runs after
            //      the D2H of batch b (stream order), while other streams compute.
            uint64_t maxest = 0;
            for (auto e : est) maxest = std::max(maxest, e);
            const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(o.batch_capacity_pairs,
                                                                          maxest + maxest / 4 + 65536));
            std::vector<uint64_t *> staging(S);
            for (int i = 0; i < S; ++i) staging[i] = dalloc<uint64_t>(cap, st.s[i]);
            Scratch<Slot> slots(S, s0);
            SJ_CUDA(cudaStreamSynchronize(s0));
            Slot *hslots = static_cast<Slot *>(host_pinned_alloc(sizeof(Slot) * S, nullptr));
            std::vector<Ev> e0(S), e1(S), edone(S);
            std::deque<std::pair<uint64_t, uint64_t>> pending;
            for (size_t b = 0; b < nb; ++b) pending.emplace_back(cuts[b], cuts[b + 1]);
            std::vector<std::pair<uint64_t, uint64_t>> inflight(S, {0, 0});
            std::deque<int> order;  // streams in launch order
            auto launch_on = [&](int i) {
                auto r = pending.front();
                pending.pop_front();
                inflight[i] = r;
                run_batch(r.first, r.second, staging[i], cap, slots.p + i, st.s[i], e0[i].e, e1[i].e);
                SJ_CUDA(cudaMemcpyAsync(hslots + i, slots.p + i, sizeof(Slot), cudaMemcpyDeviceToHost, st.s[i]));
                SJ_CUDA(cudaEventRecord(edone[i].e, st.s[i]));
                order.push_back(i);
            };
            for (int i = 0; i < S && !pending.empty(); ++i) launch_on(i);
            try {
                while (!order.empty()) {
                    const int i = order.front();
                    order.pop_front();
                    SJ_CUDA(cudaEventSynchronize(edone[i].e));
                    add_time(e0[i].e, e1[i].e);
                    const uint64_t n = hslots[i].cursor;
                    const auto r = inflight[i];
                    if (n > cap) {
                        // overflow: split the query range and re-run both halves first
                        ++stats.retries;
                        if (r.second - r.first < 2) fail(SJ_ERR_NOMEM, "a single query exceeds the batch capacity");
                        const uint64_t mid = r.first + (r.second - r.first) / 2;
                        pending.emplace_front(mid, r.second);
                        pending.emplace_front(r.first, mid);
                    } else {
                        sj_batch bt;
                        bt.on_device = 0;
                        bt.n = n;
                        bt.cap = n;
                        if (n) {
                            bt.pairs = static_cast<uint64_t *>(host_pinned_alloc(n * sizeof(uint64_t), nullptr));
                            SJ_CUDA(cudaMemcpyAsync(bt.pairs, staging[i], n * sizeof(uint64_t),
                                                    cudaMemcpyDeviceToHost, st.s[i]));
                        }
                        res->batches.push_back(bt);
                        res->total += n;
                    }
                    if (!pending.empty()) launch_on(i);
                }
            } catch (...) {
                for (int i = 0; i < S; ++i) cudaStreamSynchronize(st.s[i]);
                host_pinned_free(hslots);
                for (int i = 0; i < S; ++i) dev_free(staging[i], st.s[i]);
                throw;
            }
            for (int i = 0; i < S; ++i) SJ_CUDA(cudaStreamSynchronize(st.s[i]));
            host_pinned_free(hslots);
            for (int i = 0; i < S; ++i) dev_free(staging[i], st.s[i]);
        }

        // ---- work counters
        unsigned long long hw[4] = {0, 0, 0, 0};
        SJ_CUDA(cudaMemcpy(hw, work.p, sizeof(hw), cudaMemcpyDeviceToHost));
        stats.cells_probed = hw[0];
        stats.candidates_tested = hw[1];
        stats.pairs = res->total;
        stats.batches = (uint32_t)res->batches.size();
        stats.refine_ms = refine_ms;
        stats.refine_max_ms = refine_max;
        stats.refine_launches = launches;
        for (int i = 0; i < S; ++i) SJ_CUDA(cudaStreamSynchronize(st.s[i]));
    } catch (...) {
        for (int i = 0; i < S; ++i) cudaStreamSynchronize(st.s[i]);
        for (auto &b : res->batches) {
            if (!b.pairs) continue;
            if (b.on_device) dev_free(b.pairs, nullptr);
            else host_pinned_free(b.pairs);
        }
        delete res;
        throw;
    }
    stats.total_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t_begin).count();
    return res;
}

void neighbor_counts_impl(const sj_index *idx, const sj_join_opts &o, uint32_t *cnt, uint64_t *total)
{
    uint64_t q0, q1;
    validate(idx, o, &q0, &q1);
    SJ_CUDA(cudaSetDevice(idx->device));
    Streams st(1);
    cudaStream_t s = st.s[0];
    Scratch<unsigned long long> work(4, s);
    SJ_CUDA(cudaMemsetAsync(work.p, 0, 4 * sizeof(unsigned long long), s));
    Scratch<uint32_t> own_cnt;
    uint32_t *c = cnt;
    if (!c) {
        own_cnt.p = dalloc<uint32_t>(idx->view.n, s);
        own_cnt.s = s;
        c = own_cnt.p;
    }
    SJ_CUDA(cudaMemsetAsync(c, 0, sizeof(uint32_t) * idx->view.n, s));
    JoinArgs ja = base_args(o, work.p);
    ja.pcount = c;
    ja.q0 = (uint32_t)q0;
    ja.q1 = (uint32_t)q1;
    launch_refine<kCountPoint>(idx->dev, ja, o.unicomp != 0, (uint32_t)(q1 - q0), s);
    unsigned long long hw[4];
    SJ_CUDA(cudaMemcpyAsync(hw, work.p, sizeof(hw), cudaMemcpyDeviceToHost, s));
    SJ_CUDA(cudaStreamSynchronize(s));
    if (total) *total = hw[2];
}

}  // namespace sj
