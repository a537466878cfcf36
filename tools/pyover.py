import os, sys, time, ctypes
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, datagen
from paper_1803_04120_b200 import sj
from paper_1803_04120_b200 import distributed as sjd
P = torch.from_numpy(datagen.uniform(2_000_000, 6, datagen.seed_for(6, "C2"))).cuda()
L = sj.load_library()
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    o = sj.BuildOpts(); L.sj_build_opts_default(ctypes.byref(o))
    t1 = time.perf_counter()
    idx = sj.build_index(P, 1.0)
    t2 = time.perf_counter()
    jo = sj.join_opts(); 
    t3 = time.perf_counter()
    res = sj.self_join(idx)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    st = idx.timings()
    print(f"opts {1e6*(t1-t0):.1f} build_py {1e6*(t2-t1):.1f} (C build {1e3*st['total_ms']:.1f}) joinopts {1e6*(t3-t2):.1f} join_py {1e6*(t4-t3):.1f} sync {1e6*(t5-t4):.1f}")
    res.free(); idx.free()
# pure python overhead of wrappers
t0=time.perf_counter()
for _ in range(1000): sj.join_opts()
t1=time.perf_counter()
for _ in range(1000): torch.cuda.current_stream(P.device).cuda_stream
t2=time.perf_counter()
for _ in range(1000): P.contiguous()
t3=time.perf_counter()
print(f"join_opts {1e3*(t1-t0):.1f} us, current_stream {1e3*(t2-t1):.1f} us, contiguous {1e3*(t3-t2):.1f} us (per call)")
