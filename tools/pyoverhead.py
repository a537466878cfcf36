"""Host-side cost of one headline step outside the library (Python marshalling): times each part of
sj.join_points + counters with perf_counter after a device sync.  Run on the GPU box."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402
from paper_1803_04120_b200 import sj as m  # noqa: E402

P = torch.from_numpy(datagen.uniform(2_000_000, 6, datagen.seed_for(6, "C2"))).cuda()
L = m.load_library()
acc = {}
for it in range(30):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    o, ptr, n, d, keep = m._points_arg(P, None, None)
    t.append(time.perf_counter())
    jo = m.join_opts()
    t.append(time.perf_counter())
    hi, hr = ctypes.c_void_p(), ctypes.c_void_p()
    L.sj_self_join_points(ctypes.c_void_p(ptr), n, d, 1.0, ctypes.byref(o), ctypes.byref(jo), ctypes.byref(hi),
                          ctypes.byref(hr))
    t.append(time.perf_counter())
    r = m.Result(hr.value)
    t.append(time.perf_counter())
    ix = m.Index(hi.value)
    t.append(time.perf_counter())
    c = r.counters
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    r.free()
    ix.free()
    if it >= 5:
        for k, name in enumerate(["points_arg", "join_opts", "C call", "Result()", "Index()", "counters", "sync"]):
            acc.setdefault(name, []).append((t[k + 1] - t[k]) * 1e6)
for name, v in acc.items():
    v.sort()
    print(f"{name:12s} median {v[len(v) // 2]:8.1f} us")
