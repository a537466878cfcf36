# A/B of an env switch on the headline bench: bash tools/ab.sh VAR [reps]
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
V=$1; R=${2:-3}
for r in $(seq $R); do for x in 0 1; do
  env $V=$x timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --traffic off --also-eps 0 > gpurun_out/ab_$x.json 2>/dev/null
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$x.json').read().strip().splitlines()[-1]); p=d['phases']; print('$V=$x', round(d['ms_per_step'],4), 'build', round(p['build_total_ms'],4), 'join', round(p['join_total_ms'],4))"
done; done
