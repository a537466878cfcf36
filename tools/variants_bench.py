"""Device timing of the SURVEY §8(f) rank-4 variants (variants.cu) on the BASELINE configs' point sets.

    python tools/variants_bench.py [--steps K] [--warmup W] [--only sets,knn,knnjoin,f32] [--json]

Each case: W untimed calls, then K calls timed with CUDA events on torch's stream around the whole
library call (it blocks until its result is complete), the L2 flushed (512 MB write) before each.  Work
counters come from the library (cells probed, candidates tested); the FP64 fraction is
3d ops per candidate / time against sj_diag_fp64_peak; the pair-write HBM fraction is 8 B per pair / time
against MEASURED_PEAKS.json (fallback 7.7 TB/s).
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1803_04120_b200 as sj  # noqa: E402


def hbm_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        for k in ("hbm_copy_gbs", "hbm_gbs", "copy_gbs"):
            if k in d:
                return float(d[k])
        for v in d.values():
            if isinstance(v, dict) and "hbm_gbs" in v:
                return float(v["hbm_gbs"])
    except Exception:
        pass
    return 7700.0


def knn_radius(n, d, k, L=100.0):
    vol = k / n * L ** d
    return (vol * math.gamma(1 + d / 2) / math.pi ** (d / 2)) ** (1.0 / d)


def timeit(fn, steps, warmup, flush):
    for _ in range(warmup):
        out = fn()
        del out
    torch.cuda.synchronize()
    ms = []
    out = None
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if hasattr(out, "free") and _ < steps - 1:
            out.free()
    return float(np.median(ms)), float(np.min(ms)), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--only", default="sets,knn,f32")
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args()
    sj.load_library()
    fp = sj.fp64_peak(0)
    fp64 = min(fp["dadd_ops_per_s"], fp["dmul_ops_per_s"])
    hbm = hbm_peak()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    only = set(a.only.split(","))

    if "sets" in only:
        for cfg, d, eps in (("C2", 6, 1.0), ("C3", 6, 8.0), ("C2", 3, 1.0), ("C2", 2, 1.0)):
            P = torch.from_numpy(datagen.uniform_config(cfg, d)).cuda()
            Q = torch.from_numpy(datagen.uniform(P.shape[0], d, seed=777 + d)).cuda()
            idx = sj.build_index(P, eps)
            med, mn, res = timeit(lambda: sj.join_sets(idx, Q), a.steps, a.warmup, flush)
            st = res.stats
            pairs = res.n_pairs
            rows.append(dict(variant="two-set join J(Q,P)", config=f"{cfg} {d}-D P 2M x Q 2M uniform, eps={eps}",
                             ms=med, ms_min=mn, pairs=pairs, pairs_per_s=pairs / (med / 1e3),
                             queries_per_s=Q.shape[0] / (med / 1e3), cells_probed=st["cells_probed"],
                             candidates_tested=st["candidates_tested"],
                             fp64_frac=3 * d * st["candidates_tested"] / (med / 1e3) / fp64,
                             pair_write_hbm_frac=8 * pairs / (med / 1e3) / 1e9 / hbm,
                             note="queries sorted by cell; >= 65536 queries: sampled plan, one fill pass (counters: sample + fill)"))
            res.free()
            del idx, P, Q
            torch.cuda.empty_cache()

    if "knn" in only:
        for cfg, d, k in (("C2", 6, 8), ("C2", 4, 16), ("C2", 2, 16)):
            P = torch.from_numpy(datagen.uniform_config(cfg, d)).cuda()
            eps0 = 1.3 * knn_radius(P.shape[0], d, k)
            info = {}

            def run():
                ids, s2, st = sj.knn_self(P, k, eps0, with_stats=True)
                info.update(st)
                return ids
            med, mn, _ = timeit(run, a.steps, a.warmup, flush)
            rows.append(dict(variant="kNN self-join", config=f"{cfg} {d}-D 2M uniform, k={k}, eps0={eps0:.4g}",
                             ms=med, ms_min=mn, queries_per_s=P.shape[0] / (med / 1e3), rounds=info["rounds"],
                             eps_final=info["eps_final"], cells_probed=info["cells_probed"],
                             candidates_tested=info["candidates_tested"],
                             fp64_frac=3 * d * info["candidates_tested"] / (med / 1e3) / fp64,
                             note="includes one index build per round"))
            del P
            torch.cuda.empty_cache()

    if "knnjoin" in only or "knn" in only:
        for cfg, d, k in (("C2", 6, 8), ("C2", 2, 16)):
            P = torch.from_numpy(datagen.uniform_config(cfg, d)).cuda()
            Q = torch.from_numpy(datagen.uniform(P.shape[0], d, seed=777 + d)).cuda()
            eps0 = 1.3 * knn_radius(P.shape[0], d, k)
            info = {}

            def runj():
                ids, s2, st = sj.knn_join(P, Q, k, eps0, with_stats=True)
                info.update(st)
                return ids
            med, mn, _ = timeit(runj, a.steps, a.warmup, flush)
            rows.append(dict(variant="kNN join", config=f"{cfg} {d}-D P 2M x Q 2M uniform, k={k}, eps0={eps0:.4g}",
                             ms=med, ms_min=mn, queries_per_s=Q.shape[0] / (med / 1e3), rounds=info["rounds"],
                             cells_probed=info["cells_probed"], candidates_tested=info["candidates_tested"],
                             fp64_frac=3 * d * info["candidates_tested"] / (med / 1e3) / fp64))
            del P, Q
            torch.cuda.empty_cache()

    if "f32" in only:
        for cfg, d, eps in (("C2", 6, 8.0), ("C2", 3, 1.0), ("C2", 2, 1.0)):
            P = torch.from_numpy(datagen.uniform_config(cfg, d).astype(np.float32)).cuda()
            med, mn, res = timeit(lambda: sj.self_join_f32(P, eps), a.steps, a.warmup, flush)
            st = res.stats
            pairs = res.n_pairs
            rows.append(dict(variant="FP32 self-join", config=f"{cfg} {d}-D 2M uniform float32, eps={eps}",
                             ms=med, ms_min=mn, pairs=pairs, pairs_per_s=pairs / (med / 1e3),
                             cells_probed=st["cells_probed"], candidates_tested=st["candidates_tested"],
                             pair_write_hbm_frac=8 * pairs / (med / 1e3) / 1e9 / hbm,
                             note="the self-join path (build, estimate, unicomp batches) with the binary32 predicate"))
            res.free()
            del P
            torch.cuda.empty_cache()

    for r in rows:
        if a.json:
            print(json.dumps(r))
        else:
            print(f"{r['variant']:<22} {r['config']:<48} {r['ms']:9.3f} ms  " +
                  "  ".join(f"{k}={v:.4g}" if isinstance(v, float) else f"{k}={v}" for k, v in r.items()
                            if k not in ("variant", "config", "ms", "note")))


if __name__ == "__main__":
    main()
