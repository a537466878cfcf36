#!/bin/bash
# Compare libsj variants (tools/variants.sh) on a few workloads: refine span / join / build ms.
#   tools/cmp_variants.sh ["--d 6 --eps 1" ...]
cd "$(dirname "$0")/.."
if [ $# -eq 0 ]; then set -- "--d 6 --eps 1" "--d 6 --eps 8" "--d 2 --eps 1" "--d 3 --eps 1" "--d 4 --eps 1"; fi
for lib in paper_1803_04120_b200/libsj.so build/variants/*.so; do
  [ -f "$lib" ] || continue
  echo "== $lib"
  for args in "$@"; do
    SJ_LIBRARY=$lib python tools/prof_join.py $args --reps 4 --quiet 2>&1 | tail -1
  done
done
