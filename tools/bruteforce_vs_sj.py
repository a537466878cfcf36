"""f3 vs the grid ("the GPU brute force ... GPU-SJ is faster in every experiment"):
sj_brute_force_join (all pairs, same FP64 predicate) against build + join of GPU-SJ on the same points,
device-resident results, best of 3 (CUDA-synchronised wall time).  Pair counts must agree."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402

WORK = [("C1 Syn-2D 10K", datagen.uniform_config("C1", 2), 2.5),
        ("Syn-6D 200K", datagen.uniform(200_000, 6, seed=7), 8.0),
        ("Syn-3D 300K", datagen.uniform(300_000, 3, seed=8), 2.0)]


def best(fn, reps=3):
    b = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        n = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        b = (dt, n) if b is None or dt < b[0] else b
    return b


for name, pts, eps in WORK:
    P = torch.from_numpy(pts).cuda()

    def grid():
        r, i = sj.join_points(P, eps)
        n = r.n_pairs
        r.free()
        i.free()
        return n

    def brute():
        r = sj.brute_force_join(P, eps)
        n = r.n_pairs
        r.free()
        return n

    tg, ng = best(grid)
    tb, nb = best(brute)
    assert ng == nb, (name, ng, nb)
    print(f"| {name} | {eps} | {ng} | {tb * 1e3:.2f} | {tg * 1e3:.3f} | {tb / tg:.1f}x |", flush=True)
