import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen, paper_1803_04120_b200 as sj
P = torch.from_numpy(datagen.skewed(15_228_633, 2)).cuda()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    idx = sj.build_index(P, 0.02)
    torch.cuda.synchronize(); print("build", (time.perf_counter() - t) * 1e3, idx.timings(), idx.geometry()["dir_k"], flush=True)
    del idx
