"""Reproduction helper (debug): a variant call, then the error builds of test_errors, then C1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

mode = sys.argv[1]
P = datagen.uniform(5000, int(os.environ.get("RD", "3")), seed=3)
if mode == "knn":
    sj.knn_self(torch.from_numpy(P).cuda(), 8, 1.0)
elif mode == "build":
    sj.build_index(torch.from_numpy(P).cuda(), 4.0, speculative_estimate=False)
elif mode == "buildspec":
    sj.build_index(torch.from_numpy(P).cuda(), 4.0)
elif mode == "f32":
    sj.self_join_f32(torch.from_numpy(P.astype(np.float32)).cuda(), 4.0)
torch.cuda.synchronize()
if "nan" in sys.argv[2:]:
    bad = datagen.uniform(100, 3, seed=1)
    bad[17, 2] = np.nan
    try:
        sj.build_index(torch.from_numpy(bad).cuda(), 1.0)
    except sj.SJError as e:
        print("nonfinite:", e.name)
if "ovf" in sys.argv[2:]:
    try:
        sj.build_index(torch.from_numpy(datagen.uniform(100, 6, seed=2, hi=1e6)).cuda(), 1e-3)
    except sj.SJError as e:
        print("overflow:", e.name)
if "small" in sys.argv[2:]:
    idx = sj.build_index(torch.from_numpy(datagen.uniform(100, 3, seed=1)).cuda(), 1.0)
    del idx
pts = datagen.uniform_config("C1", 2)
idx = sj.build_index(torch.from_numpy(pts).cuda(), 2.5)
r = sj.self_join(idx)
print(mode, sys.argv[2:], "C1 OK", r.n_pairs)
