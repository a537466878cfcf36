cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_csr_drain.py -m gpu -q -x > gpurun_out/q12_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q12_tests.log
tail -15 gpurun_out/q12_tests.log
timeout 600 python tools/c3_large.py --help > /dev/null 2>&1
timeout 600 python - <<'PY'
import time, torch, datagen, paper_1803_04120_b200 as sj
P = torch.from_numpy(datagen.uniform_config("C3", 6)).cuda()
for eps in (20.0, 24.0):
    idx = sj.build_index(P, eps)
    for mode in ("device", "host", "csr"):
        best = None
        for rep in range(2):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            r = sj.self_join(idx, result_on_host=(mode != "device"), drain_csr=(mode == "csr"))
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            n = r.n_pairs; nb = r.n_batches; r.free()
        print(f"C3 eps={eps} {mode:6s} pairs={n} batches={nb} join={best*1e3:.1f} ms", flush=True)
    idx.free()
PY
