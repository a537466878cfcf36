"""SJ_TRACE=2 timeline of the bench step (build + join) for a chosen workload: host enqueue times
vs GPU times per stage (see sj_common.cuh HostTrace).  Run on the GPU box:
    SJ_TRACE=2 python tools/timeline.py --d 6 --eps 1 [--points]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=6)
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--eps", type=float, default=1.0)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--points", action="store_true", help="use sj_self_join_points (one call)")
a = ap.parse_args()
P = torch.from_numpy(datagen.uniform(a.n, a.d, datagen.seed_for(a.d, "C2"))).cuda()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for i in range(a.steps):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    if a.points:
        res, idx = sj.join_points(P, a.eps)
    else:
        idx = sj.build_index(P, a.eps)
        res = sj.self_join(idx)
    e1.record()
    torch.cuda.synchronize()
    print(f"step {i}: wall {1e3 * (time.perf_counter() - t0):.3f} ms  dev {e0.elapsed_time(e1):.3f} ms  "
          f"pairs {res.n_pairs}", file=sys.stderr, flush=True)
    res.free()
    idx.free()
