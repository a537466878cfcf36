# full GPU checkpoint: test suite, default bench line, ncu launch list + full captures (profiles/<R>_*)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
R=${1:-r02}
bash tools/gpu_tests.sh tests > /dev/null 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; tail -c 600 gpurun_out/${R}_bench.json
timeout 1200 bash tools/profile_round.sh $R > gpurun_out/${R}_profile.log 2>&1; tail -2 gpurun_out/${R}_profile.log
python tools/ncu_launches.py gpurun_out/${R}_launches.csv > gpurun_out/${R}_launches_summary.txt 2>&1; head -30 gpurun_out/${R}_launches_summary.txt
python tools/ncu_summary.py gpurun_out/${R}_full.ncu-rep > gpurun_out/${R}_ncu_full_6d_eps1.txt 2>&1
python tools/ncu_summary.py gpurun_out/${R}_refine_eps8.ncu-rep > gpurun_out/${R}_ncu_refine_6d_eps8.txt 2>&1
ls gpurun_out | grep $R
