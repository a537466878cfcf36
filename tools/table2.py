"""PAPER.md Table 2 analogue on B200 (f1: unicomp ablation with kernel metrics).

    python tools/table2.py run  --work syn6d --mode uni|full     (one build + one join; ncu target)
    python tools/table2.py report                                 (runs ncu per workload x mode, prints the table)

Per workload x mode: join time (CUDA events, best of 3 without a profiler), and from ncu over the
join's emitting refine launches (time-weighted): theoretical and achieved occupancy and the L1/TEX
("unified cache") throughput in GB/s.  Ratios are unicomp / full like the paper's."""
import csv
import io
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORK = {"c4_2d": ("C4 2-D skewed 15.2M (real-data stand-in)", 0.005),
        "syn5d": ("Syn-5D 2M", 8.0), "syn6d": ("Syn-6D 2M", 8.0)}
METRICS = ["gpu__time_duration.sum", "sm__maximum_warps_per_active_cycle_pct",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum.per_second",
           "l1tex__t_sector_hit_rate.pct"]


def points(work):
    import datagen
    if work == "c4_2d":
        return datagen.skewed(15_228_633, 2)
    d = 5 if work == "syn5d" else 6
    return datagen.uniform(2_000_000, d, datagen.seed_for(d, "C2"))


def run(work, mode, reps):
    import torch
    import paper_1803_04120_b200 as sj
    P = torch.from_numpy(points(work)).cuda()
    eps = WORK[work][1]
    idx = sj.build_index(P, eps)
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = sj.self_join(idx, unicomp=(mode == "uni"))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
        n = r.n_pairs
        r.free()
    print(f"JOIN {work} {mode} {best * 1e3:.3f} ms pairs={n}", flush=True)


def ncu(work, mode):
    cmd = ["ncu", "--metrics", ",".join(METRICS), "--csv", "-k", "regex:^k_refine", sys.executable,
           os.path.abspath(__file__), "run", "--work", work, "--mode", mode, "--reps", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900).stdout
    rows = list(csv.DictReader(io.StringIO("\n".join(l for l in out.splitlines() if l.startswith('"')))))
    launches = {}
    for r in rows:
        name = r["Kernel Name"]
        emit = "k_refine_dense" in name or "k_refine_q" in name or (
            "k_refine<" in name and name.split("<")[1].split(",")[1].strip() == "0")
        if not emit:
            continue
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] else 0.0
        unit = r.get("Metric Unit", "")
        scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "byte/second": 1.0,
                 "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9, "Tbyte/second": 1e12}.get(unit, 1.0)
        launches.setdefault(r["ID"], {})[r["Metric Name"]] = v * scale
    tot = sum(l.get("gpu__time_duration.sum", 0) for l in launches.values())
    w = lambda k: sum(l.get(k, 0) * l.get("gpu__time_duration.sum", 0) for l in launches.values()) / max(tot, 1e-12)
    return {"theo_occ": w("sm__maximum_warps_per_active_cycle_pct"),
            "ach_occ": w("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "l1_gbs": w("l1tex__t_bytes.sum.per_second") / 1e9, "l1_hit": w("l1tex__t_sector_hit_rate.pct"),
            "launches": len(launches)}


def report():
    print("| workload | eps | time full (ms) | time unicomp (ms) | ratio resp. time (full/uni) | theo. occ. full | "
          "theo. occ. uni | achieved occ. full / uni | L1/TEX GB/s full | L1/TEX GB/s uni | ratio occ. | ratio cache |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for work, (label, eps) in WORK.items():
        t = {}
        for mode in ("full", "uni"):
            out = subprocess.run([sys.executable, os.path.abspath(__file__), "run", "--work", work, "--mode", mode,
                                  "--reps", "3"], capture_output=True, text=True, timeout=900).stdout
            t[mode] = float([l for l in out.splitlines() if l.startswith("JOIN")][-1].split()[3])
        m = {mode: ncu(work, mode) for mode in ("full", "uni")}
        f, u = m["full"], m["uni"]
        print(f"| {label} | {eps} | {t['full']:.2f} | {t['uni']:.2f} | {t['full'] / t['uni']:.2f} | "
              f"{f['theo_occ']:.1f}% | {u['theo_occ']:.1f}% | {f['ach_occ']:.1f}% / {u['ach_occ']:.1f}% | "
              f"{f['l1_gbs']:.0f} | {u['l1_gbs']:.0f} | {u['theo_occ'] / max(f['theo_occ'], 1e-9):.2f} | "
              f"{u['l1_gbs'] / max(f['l1_gbs'], 1e-9):.2f} |", flush=True)


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["run", "report"])
    ap.add_argument("--work", default="syn6d")
    ap.add_argument("--mode", default="uni")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    if a.cmd == "run":
        run(a.work, a.mode, a.reps)
    else:
        report()
