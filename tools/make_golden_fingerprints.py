"""Write tests/golden/fingerprints.json: the ORACLE's |S| and order-independent fingerprints
(F_a, F_b of the pair multiset, F_c of the per-query count vector; oracle/sj_oracle.c
orc_grid_digest) for the BASELINE.json configs whose results are too large to compare pair by pair
inside the GPU test run (C2 2-D, C3 eps >= 16, C4, C5).

Calls only datagen (seeded inputs) and oracle/ -- nothing from the CUDA path (task rule ③).

    python tools/make_golden_fingerprints.py [--only KEY ...] [--threads T]
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fingerprints.json")

# key -> (config, d, eps); points = datagen's BASELINE.json generator for that config
CASES = {
    "C2/d2/eps1": ("C2", 2, 1.0),
    "C3/d6/eps16": ("C3", 6, 16.0),
    "C3/d6/eps20": ("C3", 6, 20.0),
    "C3/d6/eps24": ("C3", 6, 24.0),
    "C4/d2/eps0.002": ("C4", 2, 0.002),
    "C4/d2/eps0.005": ("C4", 2, 0.005),
    "C4/d2/eps0.01": ("C4", 2, 0.01),
    "C4/d2/eps0.02": ("C4", 2, 0.02),
    "C4/d3/eps0.05": ("C4", 3, 0.05),
    "C4/d3/eps0.1": ("C4", 3, 0.1),
    "C4/d3/eps0.2": ("C4", 3, 0.2),
    "C5/d4/eps2": ("C5", 4, 2.0),
    "C5/d6/eps8": ("C5", 6, 8.0),
}


def points(cfg, d):
    if cfg == "C4":
        return datagen.skewed(15_228_633, d)
    return datagen.uniform_config(cfg, d)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    keys = a.only or list(CASES)
    cache = {}
    for key in keys:
        cfg, d, eps = CASES[key]
        if (cfg, d) not in cache:
            cache.clear()
            cache[(cfg, d)] = points(cfg, d)
        P = cache[(cfg, d)]
        t0 = time.time()
        dg = oracle.grid_digest(P, eps, nthreads=a.threads)
        dt = time.time() - t0
        data[key] = {"config": cfg, "d": d, "eps": eps, "n": int(len(P)), "pairs": dg["pairs"],
                     "fa": f"{dg['fa']:016x}", "fb": f"{dg['fb']:016x}", "fc": f"{dg['fc']:016x}",
                     "oracle": "oracle.grid_digest (orc_grid_digest: full 3^d hash-grid scan, FP64 RN, "
                               "no FMA)", "seconds": round(dt, 1), "threads": a.threads,
                     "host": platform.node()}
        print(key, data[key], flush=True)
        with open(OUT + ".tmp", "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)
        os.replace(OUT + ".tmp", OUT)


if __name__ == "__main__":
    main()
