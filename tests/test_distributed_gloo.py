"""Multi-process CPU tests (gloo, world_size 2) of the multi-GPU glue (paper_1803_04120_b200.distributed):
index broadcast (bit-exact arrays + geometry), shard planning, count all-reduce.  The CUDA import
step (sj_index_import) is exercised on the GPU by test_gpu_parity.test_query_range_shards_union."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_04120_b200 import distributed as sjd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ref_index():
    """Index arrays of a small dataset from the oracle's statement of the index (test-side), laid
    out in ONE packed byte buffer the way sj_index_view.packed is (X, A, pcell, G, masks, B)."""
    import datagen
    from oracle import index_ref as ir
    pts = datagen.uniform(500, 3, seed=3)
    idx = ir.build_index(pts, 9.0)
    g = idx.geom
    geom = dict(d=3, key_bits=int(g.n_cells - 1).bit_length(), eps=9.0, eps2=81.0, w=g.w,
                mins=g.mins.tolist(), cpd=g.cpd, strides=g.strides, mask_offsets=[0, 7, 14, 21])
    n, nG = len(pts), len(idx.B)
    parts = {"X": pts[idx.A].T.copy().view(np.uint8).ravel(),
             "A": idx.A.astype(np.uint32).view(np.uint8),
             "pcell": np.repeat(np.arange(nG), np.diff(idx.G)).astype(np.uint32).view(np.uint8),
             "G": idx.G.astype(np.uint32).view(np.uint8),
             "masks": np.array([0x12345], dtype=np.uint32).view(np.uint8),
             "B": np.array(idx.B, dtype=np.uint64).view(np.uint8)}
    layout, off = {}, 0
    for k, v in parts.items():
        layout[k] = off
        off += (len(v) + 255) // 256 * 256
    buf = np.zeros(off, dtype=np.uint8)
    for k, v in parts.items():
        buf[layout[k]:layout[k] + len(v)] = v
    layout["packed_bytes"] = off
    cuts = sjd.plan_shards(n, 2)
    meta = sjd.pack_meta(geom, n, nG, 21, layout, cuts)
    return meta, torch.from_numpy(buf), geom, parts, layout


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        meta, buf, geom, parts, layout = _ref_index()
        args = (meta, buf, None) if rank == 0 else (None, None, None)
        m, got, masks = sjd.broadcast_index(*args, torch.device("cpu"))
        ok = np.array_equal(m, meta) and masks is None
        lay, cuts = sjd.unpack_layout(m)
        ok &= lay == {k: (layout[k] if k in layout else -1) for k in lay}
        g = got.numpy()
        for k, v in parts.items():
            ok &= np.array_equal(g[lay[k]:lay[k] + len(v)], v)
        g2, n2, nG2, mb2 = sjd.unpack_meta(m)
        ok &= g2["w"] == geom["w"] and g2["cpd"] == geom["cpd"] and g2["mins"] == geom["mins"]
        # shard cuts travel in the header; the count all-reduce sums the shards
        mine = int(cuts[rank + 1] - cuts[rank])
        tot = sjd.allreduce_counts([mine, 1, 2, 3], torch.device("cpu"))
        mx = sjd.allreduce_counts([float(rank + 0.5)], torch.device("cpu"), op="max")[0]
        out_q.put((rank, bool(ok), int(tot[0]), float(mx), tot[1:].tolist()))
    finally:
        dist.destroy_process_group()


def test_broadcast_and_allreduce_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert [r[0] for r in res] == [0, 1]
    assert all(r[1] for r in res), res
    assert all(r[2] == 500 for r in res)
    assert all(r[3] == 1.5 for r in res)
    assert all(r[4] == [2, 4, 6] for r in res)


def test_meta_roundtrip_is_bit_exact():
    geom = dict(d=6, key_bits=41, eps=1.0, eps2=1.0, w=1.0000000000000069, mins=[-0.0, 5e-324, 1e308, -3.5, 0.1, 2.0],
                cpd=[102, 2 ** 40, 3, 4, 5, 6], strides=[1, 102, 2 ** 47, 2 ** 62 + 5, 7, 8],
                mask_offsets=[0, 1, 2, 3, 4, 5, 6])
    m = sjd.pack_meta(geom, 123, 45, 6, {"packed_bytes": 4096, "X": 0, "A": 512, "pcell": 1024, "G": 1536,
                                          "masks": -1, "B": 2048}, [0, 50, 123])
    g, n, nG, mb = sjd.unpack_meta(m)
    lay, cuts = sjd.unpack_layout(m)
    assert lay["masks"] == -1 and lay["B"] == 2048 and cuts.tolist() == [0, 50, 123]
    assert (n, nG, mb) == (123, 45, 6)
    for k in ("eps", "eps2", "w"):
        assert np.float64(g[k]).tobytes() == np.float64(geom[k]).tobytes()
    assert [np.float64(x).tobytes() for x in g["mins"]] == [np.float64(x).tobytes() for x in geom["mins"]]
    assert g["cpd"] == geom["cpd"] and g["strides"] == geom["strides"]


@pytest.mark.parametrize("n,world", [(10, 3), (2_000_000, 8), (5, 8), (0, 2)])
def test_plan_shards_partition(n, world):
    cuts = sjd.plan_shards(n, world)
    assert cuts[0] == 0 and cuts[-1] == n and len(cuts) == world + 1
    assert np.all(np.diff(cuts) >= 0)
    assert np.max(np.diff(cuts)) - np.min(np.diff(cuts)) <= 1


def test_plan_shards_weighted():
    w = np.ones(1000)
    w[:100] = 50.0      # a hot region gets fewer queries per shard
    cuts = sjd.plan_shards(1000, 4, weights=w)
    parts = [w[a:b].sum() for a, b in zip(cuts[:-1], cuts[1:])]
    assert cuts[-1] == 1000 and max(parts) - min(parts) <= 50.0
