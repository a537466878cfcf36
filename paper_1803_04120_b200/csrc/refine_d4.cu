// refine_d4.cu -- the refine kernels for d = 4 (see refine.cuh; launch dispatch in join.cu).
#include "refine_launch.cuh"

namespace sj {

template <>
void launch_refine_d<4>(int mode, const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool occ6, bool queued,
                        dim3 grid, cudaStream_t s)
{
    const dim3 block(kRefineThreads);
#define SJ_MODE_CASE(M)                                                                          \
    case M:                                                                                      \
        if (queued) {                                                                            \
            if (unicomp) k_refine_q<4, M, true><<<grid, block, 0, s>>>(ix, ja);                  \
            else k_refine_q<4, M, false><<<grid, block, 0, s>>>(ix, ja);                         \
            break;                                                                               \
        }                                                                                        \
        if constexpr (M == kEmit) {                                                              \
            if (occ6) {                                                                          \
                if (unicomp) k_refine<4, M, true, 6><<<grid, block, 0, s>>>(ix, ja);             \
                else k_refine<4, M, false, 6><<<grid, block, 0, s>>>(ix, ja);                    \
                break;                                                                           \
            }                                                                                    \
        }                                                                                        \
        if (unicomp) k_refine<4, M, true><<<grid, block, 0, s>>>(ix, ja);                        \
        else k_refine<4, M, false><<<grid, block, 0, s>>>(ix, ja);                               \
        break;
    switch (mode) {
        SJ_MODE_CASE(kEmit)
        SJ_MODE_CASE(kCountQuery)
        SJ_MODE_CASE(kCountPoint)
    default: fail(SJ_ERR_ARG, "bad refine mode");
    }
#undef SJ_MODE_CASE
}

template <>
void launch_dense_d<4>(const DevIndex &ix, const JoinArgs &ja, bool unicomp, dim3 grid, cudaStream_t s)
{
    const dim3 block(32 * kDenseWarps);
    const size_t smem = kDenseWarps * dense_smem_per_warp<4>() + (ix.search_mode == kSearchCellScan ? sizeof(TopTable) : 0);
    if (unicomp) {
        set_max_dyn_smem(reinterpret_cast<const void *>(k_refine_dense<4, true>), (int)smem);
        k_refine_dense<4, true><<<grid, block, smem, s>>>(ix, ja);
    } else {
        set_max_dyn_smem(reinterpret_cast<const void *>(k_refine_dense<4, false>), (int)smem);
        k_refine_dense<4, false><<<grid, block, smem, s>>>(ix, ja);
    }
}

}  // namespace sj
