// refine_launch.cuh -- host-side launchers of the refine kernels, one explicit instantiation per
// dimension (refine_d2.cu .. refine_d6.cu), so the kernels of different d compile in parallel.
#pragma once

#include "refine.cuh"

#include <cstdlib>

namespace sj {

// experiment switches (read once): SJ_NO_QUEUE=1 falls back to the inline cell scan
inline bool getenv_flag(const char *name)
{
    const char *e = std::getenv(name);
    return e && *e && *e != '0';
}

// mode: kEmit / kCountQuery / kCountPoint, optionally | kF32 (kEmit, kCountQuery: the FP32 join);
// occ6: the 6-CTA/SM variant of the many-offset cell scan
template <int D>
void launch_refine_d(int mode, const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool occ6, bool queued,
                     dim3 grid, cudaStream_t s);
template <int D>
void launch_dense_d(const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool f32, dim3 grid, cudaStream_t s);

// ---- shared bodies of the per-dimension launchers (instantiated once each, in refine_d<D>.cu)
template <int D, int M>
inline void launch_refine_mode(const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool occ6, bool queued,
                               dim3 grid, cudaStream_t s)
{
    const dim3 block(kRefineThreads);
    if (queued) {
        if (unicomp) k_refine_q<D, M, true><<<grid, block, 0, s>>>(ix, ja);
        else k_refine_q<D, M, false><<<grid, block, 0, s>>>(ix, ja);
        return;
    }
    if constexpr ((M & kModeMask) == kEmit) {
        if (occ6) {
            if (unicomp) k_refine<D, M, true, 6><<<grid, block, 0, s>>>(ix, ja);
            else k_refine<D, M, false, 6><<<grid, block, 0, s>>>(ix, ja);
            return;
        }
    }
    if (unicomp) k_refine<D, M, true><<<grid, block, 0, s>>>(ix, ja);
    else k_refine<D, M, false><<<grid, block, 0, s>>>(ix, ja);
}

template <int D>
inline void launch_refine_body(int mode, const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool occ6,
                               bool queued, dim3 grid, cudaStream_t s)
{
    switch (mode) {
    case kEmit: launch_refine_mode<D, kEmit>(ix, ja, unicomp, occ6, queued, grid, s); break;
    case kCountQuery: launch_refine_mode<D, kCountQuery>(ix, ja, unicomp, occ6, queued, grid, s); break;
    case kCountPoint: launch_refine_mode<D, kCountPoint>(ix, ja, unicomp, occ6, queued, grid, s); break;
    case kEmit | kF32: launch_refine_mode<D, kEmit | kF32>(ix, ja, unicomp, occ6, queued, grid, s); break;
    case kCountQuery | kF32: launch_refine_mode<D, kCountQuery | kF32>(ix, ja, unicomp, occ6, queued, grid, s); break;
    default: fail(SJ_ERR_ARG, "bad refine mode");
    }
}

template <int D, bool F32>
inline void launch_dense_body(const DevIndex &ix, const JoinArgs &ja, bool unicomp, dim3 grid, cudaStream_t s)
{
    const dim3 block(32 * kDenseWarps);
    const size_t smem = kDenseWarps * dense_smem_per_warp<D>() + (ix.search_mode == kSearchCellScan ? sizeof(TopTable) : 0);
    if (unicomp) {
        set_max_dyn_smem(reinterpret_cast<const void *>(k_refine_dense<D, true, F32>), (int)smem);
        k_refine_dense<D, true, F32><<<grid, block, smem, s>>>(ix, ja);
    } else {
        set_max_dyn_smem(reinterpret_cast<const void *>(k_refine_dense<D, false, F32>), (int)smem);
        k_refine_dense<D, false, F32><<<grid, block, smem, s>>>(ix, ja);
    }
}

}  // namespace sj
