"""f1 ablation (Fig. 9 / Table 2 analogue on B200): join time and work counters with and
without unicomp on the same index.  Prints one line per workload."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

WORK = [("C2", 2, 1.0), ("C2", 3, 1.0), ("C2", 4, 1.0), ("C2", 5, 1.0), ("C2", 6, 1.0),
        ("C3", 6, 4.0), ("C3", 6, 8.0), ("C3", 6, 12.0)]
for cfg, d, eps in WORK:
    P = torch.from_numpy(datagen.uniform_config(cfg, d)).cuda()
    idx = sj.build_index(P, eps)
    out = {}
    for uni in (True, False):
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = sj.self_join(idx, unicomp=uni)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if best is None or dt < best[0]:
                best = (dt, r.stats, r.n_pairs)
            r.free()
        out[uni] = best
    (tu, su, pu), (tf, sf, pf) = out[True], out[False]
    assert pu == pf
    print(f"{cfg} d={d} eps={eps:<5} pairs={pu:>11} full={tf*1e3:8.2f}ms unicomp={tu*1e3:8.2f}ms "
          f"time_ratio(full/uni)={tf/tu:5.2f} cand_ratio(uni/full)={su['candidates_tested']/max(1,sf['candidates_tested']):.3f} "
          f"probe_ratio(uni/full)={su['cells_probed']/max(1,sf['cells_probed']):.3f}", flush=True)
