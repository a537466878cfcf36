"""Key metrics of an ncu --set full report (one line per metric), for profiles/ summaries."""
import csv
import subprocess
import sys

WANT = ["Duration", "Elapsed Cycles", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Executed Ipc Active", "Issue Slots Busy", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "L1/TEX Hit Rate", "L2 Hit Rate", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Shared Memory Configuration Size", "Block Size", "Grid Size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
seen = set()
for r in rows[1:]:
    if r[mi] in WANT and (r[ki], r[mi]) not in seen:
        seen.add((r[ki], r[mi]))
        print(f"{r[ki][:48]:48s} {r[mi]:36s} {r[vi]:>12s} {r[ui]}")
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if rr:
    hh = rr[0]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors_op_read.sum",
                 "sm__inst_executed.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
                 "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"):
        if name in hh:
            j = hh.index(name)
            for r in rr[2:]:
                print(f"{r[hh.index('Kernel Name')][:48]:48s} {name:36s} {r[j]:>12s} {rr[1][j]}")
