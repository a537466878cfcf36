"""bench.py's multi-rank launch path on CPU: `--gpus 2` outside torchrun
re-launches itself under torch.distributed.run with 2 ranks; --dry-run runs the plumbing (gloo
rendezvous on 127.0.0.1, header + packed index-buffer broadcast, counter all-reduce, max-over-ranks
timing) and rank 0 alone prints ONE JSON line with n_gpus = 2."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_dry_run_spawns_two_ranks():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--steps", "2", "--warmup", "0", "--n", "20000"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["broadcast_ok"] is True
    assert d["queries_covered"] == 20000
    assert d["metric"].startswith("self-join result pairs/s")
