"""Timing sweep over the BASELINE.json configs (device-resident results): build + join per workload."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--set", default="c2,c3,c4,c5")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--host", action="store_true")
a = ap.parse_args()
work = []
sets = a.set.split(",")
if "c1" in sets:
    work.append(("C1", 2, 2.5, lambda: datagen.uniform_config("C1", 2)))
if "c2" in sets:
    for d in (2, 3, 4, 5, 6):
        work.append(("C2", d, 1.0, (lambda d=d: datagen.uniform_config("C2", d))))
if "c3" in sets:
    for e in (2.0, 4.0, 8.0, 12.0, 16.0):
        work.append(("C3", 6, e, lambda: datagen.uniform_config("C3", 6)))
if "c4" in sets:
    work.append(("C4", 2, 0.005, lambda: datagen.skewed(15_228_633, 2)))
    work.append(("C4", 2, 0.02, lambda: datagen.skewed(15_228_633, 2)))
    work.append(("C4", 3, 0.1, lambda: datagen.skewed(15_228_633, 3)))
if "c5" in sets:
    work.append(("C5", 4, 2.0, lambda: datagen.uniform_config("C5", 4)))
    work.append(("C5", 6, 8.0, lambda: datagen.uniform_config("C5", 6)))
cache = {}
for name, d, eps, gen in work:
    key = (name, d)
    if key not in cache:
        cache.clear()
        cache[key] = torch.from_numpy(gen()).cuda()
    P = cache[key]
    best = None
    first = None
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        idx = sj.build_index(P, eps)
        res = sj.self_join(idx, result_on_host=a.host)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        st, bt, g = res.stats, idx.timings(), idx.geometry()
        row = (dt, res.n_pairs, st, bt, g)
        if first is None:
            first = dt
        if best is None or dt < best[0]:
            best = row
        res.free()
        idx.free()
    dt, pairs, st, bt, g = best
    mode = {0: "dense", 1: "cellscan", 2: "rows"}
    print(f"{name} d={d} eps={eps:<6} N={len(P):>9} pairs={pairs:>11} total={dt*1e3:8.2f}ms "
          f"build={bt['total_ms']:6.2f} (sort {bt['sort_ms']:5.2f}) join={st['total_ms']:8.2f} "
          f"(est {st['estimate_ms']:.2f}, refine_sum {st['refine_ms']:.2f}, batches {st['batches']}, "
          f"retries {st['retries']}, est/pairs {st['estimated_pairs'] / max(pairs, 1):.3f}) "
          f"nG={g['n_cells']} k={g['dir_k']} cand={st['candidates_tested']:.3e} Gpairs/s={pairs/dt/1e9:.3f} "
          f"first_call={first*1e3:.2f}ms",
          flush=True)
