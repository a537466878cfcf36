# dense-kernel check: parity tests that exercise k_refine_dense, then the dense sweep (C2 2-D/3-D, C3 large eps, C4 2-D)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or uniform_matrix or structured or lattice or batching or c1 or csr or sort_pairs" > gpurun_out/qd_tests.log 2>&1; echo "rc=$?" >> gpurun_out/qd_tests.log
tail -3 gpurun_out/qd_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C2-d2 or C2-d3 or C2/d2 or eps16 or eps0.02 or eps0.2" > gpurun_out/qd_full.log 2>&1; echo "rc=$?" >> gpurun_out/qd_full.log
tail -3 gpurun_out/qd_full.log
timeout 600 python tools/sweep.py --set ${1:-c2,c3,c4} --reps 2 > gpurun_out/qd_sweep.txt 2>&1; cat gpurun_out/qd_sweep.txt
