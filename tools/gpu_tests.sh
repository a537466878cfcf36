# run the GPU test suite (or a subset) on the box; logs into gpurun_out/
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-tests}
shift
timeout 2400 python -m pytest $T -m gpu -q -x --durations=25 "$@" > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
tail -40 gpurun_out/gpu_tests.log
