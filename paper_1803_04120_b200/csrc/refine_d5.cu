// refine_d5.cu -- the refine kernels for d = 5 (see refine.cuh; launch dispatch in join.cu).
#include "refine_launch.cuh"

namespace sj {

template <>
void launch_refine_d<5>(int mode, const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool occ6, bool queued,
                        dim3 grid, cudaStream_t s)
{
    launch_refine_body<5>(mode, ix, ja, unicomp, occ6, queued, grid, s);
}

template <>
void launch_dense_d<5>(const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool f32, dim3 grid, cudaStream_t s)
{
    if (f32) launch_dense_body<5, true>(ix, ja, unicomp, grid, s);
    else launch_dense_body<5, false>(ix, ja, unicomp, grid, s);
}

}  // namespace sj
