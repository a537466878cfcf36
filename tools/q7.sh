cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/q7_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q7_tests.log
tail -3 gpurun_out/q7_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C3 or C5" > gpurun_out/q7_full.log 2>&1; echo "rc=$?" >> gpurun_out/q7_full.log
tail -3 gpurun_out/q7_full.log
timeout 600 python tools/sweep.py --set c3,c5 --reps 2 2>&1 | cut -c1-240
