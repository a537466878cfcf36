# A/B of a variant library (tools/variants.sh) against the default build on the headline bench:
#   bash tools/ab_lib.sh NAME [reps]      (NAME: build/variants/libsj_NAME.so)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
V=$1; R=${2:-3}
for r in $(seq $R); do for lib in default $V; do
  if [ $lib = default ]; then L=paper_1803_04120_b200/libsj.so; else L=build/variants/libsj_$lib.so; fi
  SJ_LIBRARY=$L timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --also-eps 0 > gpurun_out/ab_$lib.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$lib.json').read().strip().splitlines()[-1]); p=d['phases']; print('$lib', round(d['ms_per_step'],4), 'build', round(p['build_total_ms'],4), 'join', round(p['join_total_ms'],4))"
done; done
