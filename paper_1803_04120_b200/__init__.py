"""B200-native (sm_100a) epsilon-distance self-join -- arXiv 1803.04120 (GPU-SJ) hot path.

The work runs in ``libsj.so`` (hand-written CUDA behind the C ABI of ``include/sj.h``); this
package is its thin ctypes binding plus the multi-GPU glue.  There is no CPU fallback.
"""
from .sj import (  # noqa: F401
    Index, Result, SJError, build_index, self_join, join_points, neighbor_counts, import_index, plan_batches, plan_shards,
    brute_force_join, kernel_launches, load_library, trim, set_result_cache_limit, fp64_peak, LIB_PATH,
    use_torch_allocator, join_sets, knn_self, knn_join, self_join_f32,
)

__all__ = ["Index", "Result", "SJError", "build_index", "self_join", "join_points", "neighbor_counts", "import_index",
           "plan_batches", "plan_shards", "brute_force_join", "kernel_launches", "load_library", "trim",
           "set_result_cache_limit", "fp64_peak", "LIB_PATH", "use_torch_allocator", "join_sets", "knn_self", "knn_join", "self_join_f32"]
