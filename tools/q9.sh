cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/q9_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q9_tests.log
tail -3 gpurun_out/q9_tests.log
ncu --set full --import-source on --clock-control none -k regex:k_refine_dense -s 1 -c 1 -o gpurun_out/dense2d_c python tools/prof_join.py --d 2 --eps 1 > gpurun_out/dense2d_c.log 2>&1; python tools/ncu_summary.py gpurun_out/dense2d_c.ncu-rep > gpurun_out/dense2d_c_summary.txt; cat gpurun_out/dense2d_c_summary.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --also-eps 8 > gpurun_out/q9_bench.json 2> gpurun_out/q9_bench.err
python -c "import json; d=json.loads(open('gpurun_out/q9_bench.json').read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], {k: round(v,4) if isinstance(v,float) else v for k,v in d['phases'].items() if 'ms' in k}, d['also']['ms_per_step'])"
SJ_TRACE=2 timeout 120 python tools/timeline.py --steps 4 --points > gpurun_out/tl_points.txt 2>&1; tail -24 gpurun_out/tl_points.txt
