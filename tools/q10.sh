cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "dense or uniform_matrix or structured or lattice or batching or c1 or csr or sort_pairs or lanes" > gpurun_out/q10_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q10_tests.log
tail -2 gpurun_out/q10_tests.log
timeout 900 python tools/sweep.py --set c2,c3,c4 --reps 3 2>&1 | cut -c1-200
ncu --set full --import-source on --clock-control none -k regex:k_refine_dense -s 1 -c 1 -o gpurun_out/dense2d_d python tools/prof_join.py --d 2 --eps 1 > gpurun_out/dense2d_d.log 2>&1; python tools/ncu_summary.py gpurun_out/dense2d_d.ncu-rep > gpurun_out/dense2d_d_summary.txt; cat gpurun_out/dense2d_d_summary.txt | grep -i "duration\|occupancy\|issue\|ipc\|dram__bytes_write\|active threads"
