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

// MODE: kEmit / kCountQuery / kCountPoint; occ6: the 6-CTA/SM variant of the many-offset cell scan
template <int D>
void launch_refine_d(int mode, const DevIndex &ix, const JoinArgs &ja, bool unicomp, bool occ6, bool queued,
                     dim3 grid, cudaStream_t s);
template <int D>
void launch_dense_d(const DevIndex &ix, const JoinArgs &ja, bool unicomp, dim3 grid, cudaStream_t s);

}  // namespace sj
