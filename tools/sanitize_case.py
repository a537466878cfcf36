"""One small build + join workload for compute-sanitizer (no torch: numpy + the C ABI only, so
the sanitizer instruments only libsj's kernels).  Exits non-zero on a parity mismatch.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py c1
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import datagen  # noqa: E402
import oracle  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
if case == "c1":                      # BASELINE.json configs[0]: Syn-2D 10K, eps 2.5 (dense cells too)
    pts, eps = datagen.uniform_config("C1", 2), 2.5
elif case == "clustered6":            # small clustered 6-D cloud: cell scan, dense cells, masks
    pts, eps = datagen.clustered_small(4000, 6, seed=6, sigma=0.3), 0.6
elif case == "sparse6":               # sparse 6-D: prefix-bucket sort, occupancy bitmaps
    pts, eps = datagen.uniform(20000, 6, seed=66), 8.0
else:
    raise SystemExit(f"unknown case {case}")
want = oracle.brute_force(pts, eps)
idx = sj.build_index(pts, eps)
for kw in (dict(), dict(unicomp=False), dict(result_on_host=True, batch_capacity_pairs=4096),
           dict(sort_pairs=True, min_batches=5)):
    res = sj.self_join(idx, **kw)
    got = res.to_numpy(sort=True)
    if not np.array_equal(got, want):
        raise SystemExit(f"MISMATCH {case} {kw}: {len(got)} vs {len(want)}")
    res.free()
idx.free()
bf = sj.brute_force_join(pts, eps, result_on_host=True)
assert np.array_equal(bf.to_numpy(sort=True), want)
print(f"sanitize case {case}: OK ({len(want)} pairs)")
