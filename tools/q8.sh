cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or uniform_matrix or structured or lattice or batching or c1 or csr or sort_pairs or lanes" > gpurun_out/q8_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q8_tests.log
tail -3 gpurun_out/q8_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C2-d2 or C2-d3 or C2/d2 or eps16 or eps0.02 or eps0.2" > gpurun_out/q8_full.log 2>&1; echo "rc=$?" >> gpurun_out/q8_full.log
tail -3 gpurun_out/q8_full.log
timeout 900 python tools/sweep.py --set c2,c3,c4 --reps 3 2>&1 | cut -c1-220
SJ_TRACE=2 timeout 120 python tools/timeline.py --steps 4 --points > gpurun_out/tl_points.txt 2>&1; tail -32 gpurun_out/tl_points.txt
