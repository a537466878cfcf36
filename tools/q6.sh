cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sweep.py --set c2 --reps 3 > gpurun_out/q6_sweep.txt 2>&1; cat gpurun_out/q6_sweep.txt | cut -c1-200
for C in 4 16 32; do echo "SJ_DIR_CAP=$C"; SJ_DIR_CAP=$C timeout 600 python tools/sweep.py --set c3 --reps 2 2>&1 | cut -c1-240; done
