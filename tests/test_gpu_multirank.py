"""Multi-rank path on ONE GPU: two processes (gloo, both ranks on cuda:0) run the full sharded
step -- rank-0 build, broadcast of the index arrays, sj_index_import on rank 1, per-rank shard
join, all-reduce -- and the union of the ranks' pairs must equal the oracle's S exactly.
(NCCL refuses two ranks on one GPU; the collective calls are the same torch.distributed ones.)"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q, d, n, eps):
    import torch.distributed as dist
    import datagen
    from paper_1803_04120_b200 import distributed as sjd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pts = datagen.uniform(n, d, seed=77 + d)
        P = torch.from_numpy(pts).cuda() if rank == 0 else None
        res, total, idx = sjd.sharded_self_join(P, eps, 0)
        mine = res.to_numpy(sort=False) if res is not None else np.empty(0, np.uint64)
        out_q.put((rank, mine, total))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,n,eps,world", [(3, 6000, 8.0, 2), (6, 8000, 30.0, 3)])
def test_sharded_union_equals_oracle(d, n, eps, world):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    import datagen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, d, n, eps)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    want = oracle.brute_force(datagen.uniform(n, d, seed=77 + d), eps)
    allp = np.sort(np.concatenate([g[1] for g in got]))
    assert np.array_equal(allp, want)
    assert all(g[2] == len(want) for g in got)
