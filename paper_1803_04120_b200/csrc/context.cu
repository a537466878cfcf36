// context.cu -- per-device execution contexts reused across calls (streams, timing events,
// counter / cursor slots in device + pinned memory), so a build or a join does not create and
// destroy CUDA objects on every call.  A context is owned by one call at a time (pool + mutex);
// concurrent calls on one device simply get different contexts.
#include <chrono>
#include <cstdio>
#include <cstdlib>
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
        SJ_CUDA(cudaHostAlloc(&c->h_slots, b, cudaHostAllocPortable));
        c->slot_bytes = b;
    }
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

static double now_us()
{
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

HostTrace::HostTrace(const char *w) : what(w)
{
    static const bool enabled = [] { const char *e = std::getenv("SJ_TRACE"); return e && *e && *e != '0'; }();
    on = enabled;
    t0 = last = on ? now_us() : 0.0;
}

void HostTrace::mark(const char *stage)
{
    if (!on) return;
    const double t = now_us();
    std::fprintf(stderr, "[sj-trace] %-10s %-28s +%8.1f us  (t=%8.1f us)\n", what, stage, t - last, t - t0);
    last = t;
}

}  // namespace sj
