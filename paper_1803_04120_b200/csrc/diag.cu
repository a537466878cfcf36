// diag.cu -- measurement helpers for the roofline report (bench.py), not part of the join.
//
// sj_diag_fp64_peak: the FP64 pipe's throughput for the two operation kinds of the predicate
// (DADD/DSUB and DMUL; PAPER.md:130 distance, no FMA): a grid of 8 x SMs CTAs whose threads run 8
// independent dependency chains each (enough ILP x warps to saturate the pipe), timed with CUDA
// events.  B200's datasheet FP64 figure counts an FMA as 2 flops; the refine never issues FMA, so
// its roofline is this measured ops/s peak of single DADD / DMUL instructions.
#include <algorithm>

#include "sj_common.cuh"

namespace sj {
namespace {
constexpr int kDiagIters = 4096;
constexpr int kChains = 8;

template <bool MUL>
__global__ void __launch_bounds__(256) k_fp64_peak(double seed, double *out)
{
    double a[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) a[c] = seed + (double)(threadIdx.x + c);
    const double y = MUL ? 0.9999999999999999 : 1.0e-300;
#pragma unroll 4
    for (int i = 0; i < kDiagIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) a[c] = MUL ? __dmul_rn(a[c], y) : __dadd_rn(a[c], y);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s = __dadd_rn(s, a[c]);
    if (s == 12345.678) out[0] = s;     // never true; keeps the chains live
}
}  // namespace

double fp64_peak_impl(int device, bool mul)
{
    SJ_CUDA(cudaSetDevice(device));
    const int nsm = device_sm_count(device);
    cudaStream_t s;
    SJ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaEvent_t e0, e1;
    SJ_CUDA(cudaEventCreate(&e0));
    SJ_CUDA(cudaEventCreate(&e1));
    double *out = nullptr;
    SJ_CUDA(cudaMalloc(&out, sizeof(double)));
    const dim3 grid(nsm * 8), block(256);
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        SJ_CUDA(cudaEventRecord(e0, s));
        if (mul) k_fp64_peak<true><<<grid, block, 0, s>>>(1.0, out);
        else k_fp64_peak<false><<<grid, block, 0, s>>>(1.0, out);
        SJ_LAUNCHED();
        SJ_CUDA(cudaEventRecord(e1, s));
        SJ_CUDA(cudaEventSynchronize(e1));
        float ms = 0;
        SJ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0) best = std::min(best, ms);       // rep 0 warms up
    }
    cudaFree(out);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaStreamDestroy(s);
    const double ops = (double)grid.x * block.x * kChains * kDiagIters;
    return ops / (best * 1e-3);
}

}  // namespace sj

extern "C" sj_status sj_diag_fp64_peak(int device, double *dadd_ops_per_s, double *dmul_ops_per_s)
{
    try {
        if (dadd_ops_per_s) *dadd_ops_per_s = sj::fp64_peak_impl(device, false);
        if (dmul_ops_per_s) *dmul_ops_per_s = sj::fp64_peak_impl(device, true);
        return SJ_OK;
    } catch (const sj::Error &e) {
        return e.status;
    } catch (...) {
        return SJ_ERR_CUDA;
    }
}
