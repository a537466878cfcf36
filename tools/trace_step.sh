cd $GRAFT_REPO_ROOT
SJ_TRACE=${SJ_TRACE:-1} python - <<'PY' 2>&1 | tail -30
import os, sys, time
sys.path.insert(0, '.')
import torch, datagen, paper_1803_04120_b200 as sj
from paper_1803_04120_b200 import distributed as sjd
pts = datagen.uniform(2_000_000, 6, datagen.seed_for(6, "C2"))
P = torch.from_numpy(pts).cuda()
for i in range(8):
    pass
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    res, tot, idx = sjd.sharded_self_join(P, 1.0, 0)
    e1.record(); torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"step {i}: wall {1e3*(t1-t0):.3f} ms  dev {e0.elapsed_time(e1):.3f} ms", file=sys.stderr)
    res.free(); del idx
PY
