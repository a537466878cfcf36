cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; lscpu | head -20; nvidia-smi) > gpurun_out/r02_box.txt 2>&1
SJ_TRACE=2 bash tools/trace_step.sh > gpurun_out/r02_trace_6d.txt 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench0.json 2> gpurun_out/r02_bench0.err
