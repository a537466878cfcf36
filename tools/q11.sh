cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/q11_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q11_tests.log
tail -2 gpurun_out/q11_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C2-d6 or C2-d5 or C2-d4 or C3-d6-eps2 or C3-d6-eps4" > gpurun_out/q11_full.log 2>&1; echo "rc=$?" >> gpurun_out/q11_full.log
tail -2 gpurun_out/q11_full.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --also-eps 8 > gpurun_out/q11_bench.json 2> gpurun_out/q11_bench.err
python -c "import json; d=json.loads(open('gpurun_out/q11_bench.json').read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], {k: round(v,4) if isinstance(v,float) else v for k,v in d['phases'].items() if 'ms' in k}, d['also']['ms_per_step'])"
bash tools/insitu.sh "--d 6 --eps 1 --points" q11_insitu > /dev/null 2>&1; head -16 gpurun_out/q11_insitu_summary.txt
