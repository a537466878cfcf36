"""Profiling driver: one index build + one self-join of a chosen workload (for ncu -k ...)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=6)
ap.add_argument("--n", type=int, default=2_000_000)
ap.add_argument("--eps", type=float, default=1.0)
ap.add_argument("--config", default="C2")
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--host", action="store_true")
ap.add_argument("--full", action="store_true", help="unicomp off")
ap.add_argument("--lanes", type=int, default=0)
ap.add_argument("--quiet", action="store_true")
a = ap.parse_args()
pts = datagen.uniform(a.n, a.d, datagen.seed_for(a.d, a.config))
P = torch.from_numpy(pts).cuda()
for _ in range(a.reps):
    idx = sj.build_index(P, a.eps)
    res = sj.self_join(idx, result_on_host=a.host, unicomp=not a.full, lanes_per_query=a.lanes)
    if a.quiet:
        st = res.stats
        print(f"d={a.d} eps={a.eps} G={a.lanes} pairs={res.n_pairs} join_ms={st['total_ms']:.3f} "
              f"refine_ms={st['refine_ms']:.3f} span={st['refine_span_ms']:.3f} probes={st['cells_probed']} cand={st['candidates_tested']} est_ms={st['estimate_ms']:.3f} build_ms={idx.timings()['total_ms']:.3f}",
              flush=True)
    else:
        print(res.n_pairs, res.stats, idx.timings(), idx.geometry()["dir_k"], flush=True)
    res.free()
    idx.free()
