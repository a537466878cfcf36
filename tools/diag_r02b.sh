cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sanitizer.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q -x -k "sanitizer or sharded or dense_tasks or fingerprint or freed or trim" > gpurun_out/r02b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout 600 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --also-eps 0 > gpurun_out/r02b_bench2.json 2> gpurun_out/r02b_bench2.err
tail -3 gpurun_out/r02b_tests.log
