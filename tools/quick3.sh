cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -c "
from cuda.bindings import runtime as rt
for a in ('cudaDevAttrL2CacheSize','cudaDevAttrMaxAccessPolicyWindowSize','cudaDevAttrMaxPersistingL2CacheSize'):
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
"
K=${1:-"index or prefix or bucket or imported or uniform_matrix or structured or tiny or build_time or fig2 or masks or dense_tasks"}
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "$K" > gpurun_out/q3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q3_tests.log
tail -4 gpurun_out/q3_tests.log
for P in 1 0; do
SJ_L2_PERSIST=$P timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --traffic off --also-eps 0 > gpurun_out/q3_bench$P.json 2> gpurun_out/q3_bench$P.err
SJ_L2_PERSIST=$P python - <<'PY'
import json, os
d=json.loads(open("gpurun_out/q3_bench%s.json" % os.environ["SJ_L2_PERSIST"]).read().strip().splitlines()[-1])
print("persist", os.environ["SJ_L2_PERSIST"], "ms/step", d["ms_per_step"], "pairs/s", d["value"])
print({k: (round(v,4) if isinstance(v,float) else v) for k,v in d["phases"].items() if not isinstance(v, dict)})
PY
SJ_L2_PERSIST=$P bash tools/insitu.sh "--d 6 --eps 1" q3_insitu6_p$P > /dev/null 2>&1; cat gpurun_out/q3_insitu6_p${P}_summary.txt
done
SJ_TRACE=2 python tools/timeline.py --steps 3 --points > gpurun_out/q3_tl.txt 2>&1; tail -36 gpurun_out/q3_tl.txt
