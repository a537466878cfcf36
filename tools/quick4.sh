cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/q4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q4_tests.log
tail -4 gpurun_out/q4_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k "C3 or C5" > gpurun_out/q4_full.log 2>&1; echo "rc=$?" >> gpurun_out/q4_full.log
tail -4 gpurun_out/q4_full.log
for Q in 0 1; do
SJ_NO_QUEUE=$Q timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --eps 8 --also-eps 0 > gpurun_out/q4_bench$Q.json 2> gpurun_out/q4_bench$Q.err
SJ_NO_QUEUE=$Q python - <<'PY'
import json, os
d=json.loads(open("gpurun_out/q4_bench%s.json" % os.environ["SJ_NO_QUEUE"]).read().strip().splitlines()[-1])
print("no_queue", os.environ["SJ_NO_QUEUE"], "eps8 ms/step", d["ms_per_step"], "span", d["phases"]["refine_span_ms"], "fp64 frac", d["roofline"]["fp64"]["frac"])
PY
done
python tools/prof_join.py --eps 8 --reps 3 --quiet 2>&1 | tail -1; python tools/prof_join.py --eps 8 --reps 3 --quiet --full 2>&1 | tail -1
timeout 300 python tools/sweep.py --set c3 --reps 2 > gpurun_out/q4_sweep.txt 2>&1; cat gpurun_out/q4_sweep.txt
