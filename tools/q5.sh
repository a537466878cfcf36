# quick: dense + build parity subset, C2 sweep, headline bench (no e2e/cpu), timeline, in-situ build profile
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or uniform_matrix or structured or lattice or index_matches or c1 or tiny or errors" > gpurun_out/q5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q5_tests.log
tail -3 gpurun_out/q5_tests.log
timeout 600 python tools/sweep.py --set c2 --reps 3 > gpurun_out/q5_sweep.txt 2>&1; cat gpurun_out/q5_sweep.txt | cut -c1-200
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --also-eps 0 > gpurun_out/q5_bench.json 2> gpurun_out/q5_bench.err
python -c "import json; d=json.loads(open('gpurun_out/q5_bench.json').read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], {k: round(v,4) if isinstance(v,float) else v for k,v in d['phases'].items() if 'ms' in k})"
bash tools/insitu.sh "--d 6 --eps 1" q5_insitu > /dev/null 2>&1; head -14 gpurun_out/q5_insitu_summary.txt
