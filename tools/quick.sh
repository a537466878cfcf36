# Quick GPU checks between commits (run under gpurun; logs into gpurun_out/):
#   bash tools/quick.sh headline   parity + multirank + full-size subset, headline bench, in-situ build/refine profile
#   bash tools/quick.sh dense      dense-kernel parity subset, full-size dense configs, C2/C3/C4 sweep
#   bash tools/quick.sh extras     CSR drain, DBSCAN, C3 eps=20/24 device / host / CSR-drain joins
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
case "${1:-headline}" in
headline)
    timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -q -x > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
    tail -2 gpurun_out/quick_tests.log
    timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C2-d6 or C2-d5 or C2-d4 or C3-d6-eps2 or C3-d6-eps4" > gpurun_out/quick_full.log 2>&1; echo "rc=$?" >> gpurun_out/quick_full.log
    tail -2 gpurun_out/quick_full.log
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --also-eps 8 > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
    python -c "import json; d=json.loads(open('gpurun_out/quick_bench.json').read().strip().splitlines()[-1]); print('ms/step', d['ms_per_step'], {k: round(v,4) if isinstance(v,float) else v for k,v in d['phases'].items() if 'ms' in k}, d['also']['ms_per_step'])"
    bash tools/insitu.sh "--d 6 --eps 1 --points" quick_insitu > /dev/null 2>&1; head -20 gpurun_out/quick_insitu_summary.txt
    ;;
dense)
    timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or uniform_matrix or structured or lattice or batching or c1 or csr or sort_pairs or lanes" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
    tail -2 gpurun_out/quick_tests.log
    timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C2-d2 or C2-d3 or C2/d2 or eps16 or eps0.02 or eps0.2" > gpurun_out/quick_full.log 2>&1; echo "rc=$?" >> gpurun_out/quick_full.log
    tail -2 gpurun_out/quick_full.log
    timeout 900 python tools/sweep.py --set c2,c3,c4 --reps 3 2>&1 | cut -c1-220
    ;;
extras)
    timeout 900 python -m pytest tests/test_gpu_csr_drain.py tests/test_gpu_dbscan.py -m gpu -q -x > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
    tail -2 gpurun_out/quick_tests.log
    timeout 600 python tools/c3_large.py 2>&1 | tail -8
    ;;
esac
