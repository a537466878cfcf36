import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import paper_1803_04120_b200 as sj
from oracle import index_ref as ir
rng = np.random.default_rng(7000)
n, m = 20000, 7000
pts = rng.uniform(0, 100, (n, 6))
pts[:m, 4:] = 50.25 + rng.uniform(0, 0.5, (m, 2))
pts[:m, :4] = rng.uniform(40, 60, (m, 4))
rng.shuffle(pts)
idx = sj.build_index(torch.from_numpy(pts).cuda(), 1.0)
print("n_cells", idx.n_cells, idx.geometry()["dir_k"])
ref = ir.build_index(pts, 1.0)
print("ref cells", len(ref.B))
