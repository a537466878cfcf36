// context.cu -- per-device execution contexts reused across calls (streams, timing events,
// counter / cursor slots in device + pinned memory), so a build or a join does not create and
// destroy CUDA objects on every call.  A context is owned by one call at a time (pool + mutex);
// concurrent calls on one device simply get different contexts.
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

}  // namespace sj
