#!/bin/bash
# Capture the round's ncu evidence (run under gpurun, 1 GPU):
#   1. launch list of a short bench run (per-kernel device time shares)
#   2. --set full of the refine kernel (every emit launch of one join), the radix scatter and the
#      compaction/gather kernels of the 6-D eps=1 workload
set -e
R=${1:-r01}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --also-eps 0 > gpurun_out/${R}_launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_refine|k_bucket_scatter|k_bucket_sort|k_compact_gather|k_keys|k_minmax" \
    -c 14 -o gpurun_out/${R}_full python tools/prof_join.py > gpurun_out/${R}_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_refine -s 1 -c 1 \
    -o gpurun_out/${R}_refine_eps8 python tools/prof_join.py --eps 8 > gpurun_out/${R}_refine_eps8.log 2>&1
echo done
