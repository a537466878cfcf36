# quick GPU check after build-path changes: index/parity tests, bench, timeline, in-situ profile
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${1:-"index or prefix or bucket or imported or uniform_matrix or structured or tiny or build_time or fig2 or masks or dense_tasks"}
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > gpurun_out/q2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q2_tests.log
tail -15 gpurun_out/q2_tests.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C2 or eps8 or eps4 or C5" > gpurun_out/q2_full.log 2>&1; echo "rc=$?" >> gpurun_out/q2_full.log
tail -5 gpurun_out/q2_full.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/q2_bench.json 2> gpurun_out/q2_bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/q2_bench.json").read().strip().splitlines()[-1])
print("ms/step", d["ms_per_step"], "pairs/s", d["value"], "also", d["also"]["ms_per_step"] if d["also"] else None)
print({k: (round(v,4) if isinstance(v,float) else v) for k,v in d["phases"].items() if not isinstance(v, dict)})
PY
SJ_TRACE=2 python tools/timeline.py --steps 3 --points > gpurun_out/q2_tl.txt 2>&1; tail -40 gpurun_out/q2_tl.txt
bash tools/insitu.sh "--d 6 --eps 1" q2_insitu6 > /dev/null 2>&1; cat gpurun_out/q2_insitu6_summary.txt
