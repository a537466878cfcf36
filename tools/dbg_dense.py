import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import datagen, oracle, paper_1803_04120_b200 as sj
import math
n, d, m = 100, 2, 100
pts = datagen.uniform(n, d, seed=1000 * d + n + m)
vol = m / n * 100.0 ** d
eps = (vol * math.gamma(1 + d / 2) / math.pi ** (d / 2)) ** (1.0 / d)
want = oracle.brute_force(pts, eps)
idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
print("eps", eps, "cells", idx.n_cells, idx.geometry()["cpd"])
for dense in (False, True):
    for unicomp in (True, False):
        for mb in (1, 3):
            r = sj.self_join(idx, dense_cells=dense, unicomp=unicomp, min_batches=mb)
            got = r.to_numpy()
            extra = np.setdiff1d(got, want); miss = np.setdiff1d(want, got)
            dup = len(got) - len(np.unique(got))
            print(f"dense={dense} unicomp={unicomp} mb={mb} got={len(got)} want={len(want)} extra={len(extra)} miss={len(miss)} dup={dup} stats={r.stats['candidates_tested']}")
            if len(extra) or len(miss):
                print("  extra", [(int(x)>>32, int(x)&0xffffffff) for x in extra[:6]], " miss", [(int(x)>>32, int(x)&0xffffffff) for x in miss[:6]])
