"""C4 2-D eps=0.02 build/join host trace (SJ_TRACE=1) over a few reps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen, paper_1803_04120_b200 as sj
eps = float(sys.argv[1]) if len(sys.argv) > 1 else 0.02
P = torch.from_numpy(datagen.skewed(15_228_633, 2)).cuda()
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    idx = sj.build_index(P, eps)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    res = sj.self_join(idx)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    st = res.stats
    print(f"rep {r}: build {1e3*(t1-t0):.2f} ms join {1e3*(t2-t1):.2f} ms pairs {res.n_pairs} batches {res.n_batches} retries {st["retries"]} est {st["estimated_pairs"]}", file=sys.stderr, flush=True)
    res.free(); idx.free()
