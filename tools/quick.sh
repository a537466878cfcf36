# quick GPU check: selected tests + headline bench (no e2e/cpu) + eps=8 + 2-D sweep line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
K=${1:-"imported or dense_tasks or uniform_matrix or structured or lanes or masks"}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "$K" > gpurun_out/quick_tests.log 2>&1; echo "rc=$?" >> gpurun_out/quick_tests.log
tail -3 gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/quick_bench.json").read().strip().splitlines()[-1])
print("ms/step", d["ms_per_step"], "pairs/s", d["value"], "also", d["also"]["ms_per_step"] if d["also"] else None)
print({k: (round(v,4) if isinstance(v,float) else v) for k,v in d["phases"].items() if not isinstance(v, dict)})
print("fp64", d["roofline"]["fp64"])
PY
timeout 300 python tools/sweep.py --set c2 --reps 2 > gpurun_out/quick_sweep.txt 2>&1; cat gpurun_out/quick_sweep.txt
