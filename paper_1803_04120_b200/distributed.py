"""Multi-GPU glue: query sharding with a replicated index (north_star "Partitioning").

One process per GPU (torchrun), ``torch.distributed`` for the plumbing:
  1. rank 0 builds the index (sj_build_index) and plans the shards from the build's sampled
     result-size estimate (sj_plan_shards: contiguous A-order query ranges of equal estimated work);
  2. rank 0 broadcasts a small int64 header (geometry, sizes, array offsets, shard cuts) and then the
     index's arrays as ONE packed device buffer (sj_index_view.packed: X, A, pcell, G, masks, B) --
     the one exchange step of the path (NCCL over NVLink on B200; gloo in the CPU tests);
  3. every other rank imports the received buffer in place (sj_index_import_borrowed: no copy; the
     prefix directory, occupancy bitmaps and dense-cell tasks are rebuilt from B and G) and joins its
     own query range (sj_self_join with query_begin/query_end); with unicomp a rank emits both
     orientations of every pair its queries decide, so the shards partition S exactly;
  4. [pairs, cells_probed, candidates_tested, retries] are all-reduced (SUM); pairs stay on their rank.

Everything here is marshalling: no step of the method runs in Python.
"""
from __future__ import annotations

import struct
from typing import Optional, Sequence, Tuple

import numpy as np

SJ_MAX_DIM = 6
MAX_WORLD = 64
# header layout (int64 words):
#   [0:5]   n, d, n_cells, key_bits, mask_bits
#   [5:8]   eps, eps2, w (float64 bit patterns)
#   [8:26]  mins (bits), cpd, strides (SJ_MAX_DIM each)
#   [26:33] mask_offsets (SJ_MAX_DIM + 1)
#   [33:41] packed_bytes, off_X, off_A, off_pcell, off_G, off_masks (-1: separate), off_B, world
#   [41:41+MAX_WORLD+1] shard cuts
_GEOM_WORDS = 5 + 3 + SJ_MAX_DIM * 3 + (SJ_MAX_DIM + 1)
_META_WORDS = _GEOM_WORDS + 8 + MAX_WORLD + 1


def _f2i(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(x)))[0]


def _i2f(x: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(x)))[0]


def _u2i(x: int) -> int:
    return int(np.uint64(x).astype(np.int64))


def _i2u(x) -> int:
    return int(np.int64(x).astype(np.uint64))


def pack_meta(geom: dict, n: int, n_cells: int, mask_bits: int, layout: Optional[dict] = None,
              cuts: Optional[Sequence[int]] = None) -> np.ndarray:
    """Geometry, packed-buffer layout and shard cuts of an index as int64 words (float64 fields
    bit-cast, so the transfer is exact)."""
    d = int(geom["d"])
    m = np.zeros(_META_WORDS, dtype=np.int64)
    m[0:5] = [n, d, n_cells, geom["key_bits"], mask_bits]
    m[5:8] = [_f2i(geom["eps"]), _f2i(geom["eps2"]), _f2i(geom["w"])]
    o = 8
    for j in range(d):
        m[o + j] = _f2i(geom["mins"][j])
        m[o + SJ_MAX_DIM + j] = _u2i(geom["cpd"][j])
        m[o + 2 * SJ_MAX_DIM + j] = _u2i(geom["strides"][j])
    o += 3 * SJ_MAX_DIM
    for j in range(d + 1):
        m[o + j] = geom["mask_offsets"][j]
    o = _GEOM_WORDS
    if layout is not None:
        m[o:o + 7] = [layout["packed_bytes"], layout["X"], layout["A"], layout["pcell"], layout["G"],
                      layout.get("masks", -1), layout["B"]]
    if cuts is not None:
        w = len(cuts) - 1
        if w > MAX_WORLD:
            raise ValueError(f"world > {MAX_WORLD}")
        m[o + 7] = w
        m[o + 8:o + 8 + w + 1] = np.asarray(cuts, dtype=np.int64)
    return m


def unpack_meta(m: np.ndarray) -> Tuple[dict, int, int, int]:
    m = np.asarray(m, dtype=np.int64)
    n, d, n_cells, key_bits, mask_bits = (int(v) for v in m[0:5])
    geom = dict(d=d, key_bits=key_bits, eps=_i2f(m[5]), eps2=_i2f(m[6]), w=_i2f(m[7]))
    o = 8
    geom["mins"] = [_i2f(m[o + j]) for j in range(d)]
    geom["cpd"] = [_i2u(m[o + SJ_MAX_DIM + j]) for j in range(d)]
    geom["strides"] = [_i2u(m[o + 2 * SJ_MAX_DIM + j]) for j in range(d)]
    o += 3 * SJ_MAX_DIM
    geom["mask_offsets"] = [int(m[o + j]) for j in range(d + 1)]
    return geom, n, n_cells, mask_bits


def unpack_layout(m: np.ndarray) -> Tuple[dict, np.ndarray]:
    m = np.asarray(m, dtype=np.int64)
    o = _GEOM_WORDS
    keys = ("packed_bytes", "X", "A", "pcell", "G", "masks", "B")
    layout = {k: int(v) for k, v in zip(keys, m[o:o + 7])}
    w = int(m[o + 7])
    cuts = m[o + 8:o + 8 + w + 1].copy() if w > 0 else np.zeros(0, dtype=np.int64)
    return layout, cuts


def index_meta(idx, cuts=None) -> Tuple[np.ndarray, "torch.Tensor", Optional["torch.Tensor"]]:
    """(header words, packed uint8 device buffer, separate masks tensor or None) of a built index."""
    v = idx.view
    g = idx.geometry()
    has_masks = bool(v.masks)
    mask_bits = int(g["mask_offsets"][-1]) if has_masks else 0
    sep = has_masks and int(v.off_masks) == 0xFFFFFFFFFFFFFFFF
    layout = {"packed_bytes": int(v.packed_bytes), "X": int(v.off_X), "A": int(v.off_A),
              "pcell": int(v.off_pcell), "G": int(v.off_G), "B": int(v.off_B),
              "masks": -1 if (sep or not has_masks) else int(v.off_masks)}
    meta = pack_meta(g, idx.n, idx.n_cells, mask_bits, layout, cuts)
    buf = idx.packed()
    masks = idx.arrays()["masks"] if sep else None
    return meta, buf, masks


def view_from_packed(meta: np.ndarray, buf, masks, device: int):
    """sj_index_view whose arrays point into the received packed buffer (+ separate masks)."""
    import ctypes
    from . import sj
    geom, n, n_cells, mask_bits = unpack_meta(meta)
    layout, _ = unpack_layout(meta)
    v = sj.IndexView()
    d = geom["d"]
    v.d, v.device, v.n, v.n_cells = d, device, n, n_cells
    v.eps, v.eps2, v.w = geom["eps"], geom["eps2"], geom["w"]
    for j in range(d):
        v.mins[j] = geom["mins"][j]
        v.cpd[j] = geom["cpd"][j]
        v.strides[j] = geom["strides"][j]
    v.key_bits = geom["key_bits"]
    for j in range(d + 1):
        v.mask_offsets[j] = geom["mask_offsets"][j]
    base = buf.data_ptr()
    for name in ("B", "G", "A", "pcell", "X"):
        setattr(v, name, ctypes.c_void_p(base + layout[name]))
    if mask_bits:
        v.masks = ctypes.c_void_p(masks.data_ptr() if layout["masks"] < 0 else base + layout["masks"])
    else:
        v.masks = None
    v.packed = ctypes.c_void_p(base)
    v.packed_bytes = layout["packed_bytes"]
    return v


def broadcast_index(meta: Optional[np.ndarray], buf, masks, device, group=None, src: int = 0):
    """Broadcast the header, then the packed index buffer (and, rarely, masks too large for the
    packed buffer) from `src`.  Non-src ranks pass None and receive fresh tensors on `device`.
    Returns (meta, buf, masks) on every rank."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    mt = torch.zeros(_META_WORDS, dtype=torch.int64, device=device)
    if rank == src:
        mt.copy_(torch.from_numpy(np.asarray(meta, dtype=np.int64)))
    dist.broadcast(mt, src=src, group=group)
    meta = mt.cpu().numpy()
    geom, n, n_cells, mask_bits = unpack_meta(meta)
    layout, _ = unpack_layout(meta)
    if rank != src:
        buf = torch.empty(layout["packed_bytes"], dtype=torch.uint8, device=device)
    dist.broadcast(buf, src=src, group=group)
    if mask_bits and layout["masks"] < 0:
        if rank != src:
            masks = torch.empty((mask_bits + 31) // 32, dtype=torch.int32, device=device)
        else:
            masks = masks.view(torch.int32)
        dist.broadcast(masks, src=src, group=group)
    return meta, buf, masks


def plan_shards(n: int, world: int, weights: Optional[Sequence[float]] = None) -> np.ndarray:
    """Host-side shard cuts for tests and the dry run: equal query counts, or equal cumulative
    weight.  (The GPU path uses sj_plan_shards, balanced by the sampled estimate.)"""
    if world < 1:
        raise ValueError("world must be >= 1")
    if weights is None:
        return np.array([n * r // world for r in range(world + 1)], dtype=np.int64)
    w = np.asarray(weights, dtype=np.float64)
    if len(w) != n:
        raise ValueError("one weight per query")
    c = np.concatenate([[0.0], np.cumsum(w)])
    tot = c[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(c, tot * r / world, side="left")))
    cuts.append(n)
    return np.maximum.accumulate(np.array(cuts, dtype=np.int64))


def allreduce_counts(values: Sequence[int], device, op: str = "sum", group=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.int64 if op == "sum" else torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=group)
    return t.cpu().numpy()


COUNTERS = ("pairs", "cells_probed", "candidates_tested", "retries")


def sharded_self_join(points, eps: float, device: int, group=None, stats: bool = False, **join_kw):
    """Full multi-GPU step: rank-0 build + shard plan -> broadcast (header + packed buffer) ->
    borrowed import -> shard join -> all-reduce of the work counters.

    Returns (local Result or None, global pair count, local Index) -- and with stats=True also the
    dict of all-reduced counters."""
    import torch
    import torch.distributed as dist
    from . import sj
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    dev = torch.device("cuda", device)
    if world == 1:
        # one library call (sj_self_join_points): build + join without a return to Python between them
        res, idx = sj.join_points(points, eps, device=device, **join_kw)
        if stats:
            return res, res.n_pairs, idx, res.counters
        return res, res.n_pairs, idx
    if rank == 0:
        idx = sj.build_index(points, eps, device=device)
        cuts = sj.plan_shards(idx, world)
        meta, buf, masks = index_meta(idx, cuts)
    else:
        idx, meta, buf, masks = None, None, None, None
    meta, buf, masks = broadcast_index(meta, buf, masks, dev, group=group)
    if rank != 0:
        idx = sj.import_index(view_from_packed(meta, buf, masks, device), device, borrow=(buf, masks))
    _, cuts = unpack_layout(meta)
    a, b = int(cuts[rank]), int(cuts[rank + 1])
    res = sj.self_join(idx, query_begin=a, query_end=b, **join_kw) if b > a else None
    if res is not None:
        c = res.counters
        local = [c[k] for k in COUNTERS]
    else:
        local = [0] * len(COUNTERS)
    tot = allreduce_counts(local, dev, group=group)
    if stats:
        return res, int(tot[0]), idx, dict(zip(COUNTERS, (int(x) for x in tot)))
    return res, int(tot[0]), idx
