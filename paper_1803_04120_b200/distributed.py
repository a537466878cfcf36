"""Multi-GPU glue: query sharding with a replicated index (north_star "Partitioning").

One process per GPU (torchrun), ``torch.distributed`` for the plumbing:
  1. rank 0 builds the index (sj_build_index);
  2. the index arrays (B, G, A, pcell, X, masks) and its geometry are broadcast from rank 0
     (NCCL over NVLink on B200; gloo in the CPU tests) -- the one exchange step of the path;
  3. every rank imports the arrays (sj_index_import) and joins its own contiguous A-order
     query range (sj_self_join with query_begin/query_end); with unicomp a rank emits both
     orientations of every pair its queries decide, so the shards partition S exactly;
  4. pair counts are combined with an all-reduce (SUM); pairs stay on their rank.

Everything here is marshalling: no step of the method runs in Python.
"""
from __future__ import annotations

import struct
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

SJ_MAX_DIM = 6
# meta layout (int64 words): n, d, n_cells, key_bits, mask_bits, device-independent geometry
_META_WORDS = 5 + 3 + SJ_MAX_DIM * 3 + (SJ_MAX_DIM + 1)


def _f2i(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", float(x)))[0]


def _i2f(x: int) -> float:
    return struct.unpack("<d", struct.pack("<q", int(x)))[0]


def pack_meta(geom: dict, n: int, n_cells: int, mask_bits: int) -> np.ndarray:
    """Geometry of an index as int64 words (float64 fields bit-cast, so transfer is exact)."""
    d = int(geom["d"])
    m = np.zeros(_META_WORDS, dtype=np.int64)
    m[0:5] = [n, d, n_cells, geom["key_bits"], mask_bits]
    m[5:8] = [_f2i(geom["eps"]), _f2i(geom["eps2"]), _f2i(geom["w"])]
    o = 8
    for j in range(d):
        m[o + j] = _f2i(geom["mins"][j])
        m[o + SJ_MAX_DIM + j] = np.uint64(geom["cpd"][j]).astype(np.int64)
        m[o + 2 * SJ_MAX_DIM + j] = np.uint64(geom["strides"][j]).astype(np.int64)
    o += 3 * SJ_MAX_DIM
    for j in range(d + 1):
        m[o + j] = geom["mask_offsets"][j]
    return m


def unpack_meta(m: np.ndarray) -> Tuple[dict, int, int, int]:
    m = np.asarray(m, dtype=np.int64)
    n, d, n_cells, key_bits, mask_bits = (int(v) for v in m[0:5])
    geom = dict(d=d, key_bits=key_bits, eps=_i2f(m[5]), eps2=_i2f(m[6]), w=_i2f(m[7]))
    o = 8
    geom["mins"] = [_i2f(m[o + j]) for j in range(d)]
    geom["cpd"] = [int(np.int64(m[o + SJ_MAX_DIM + j]).astype(np.uint64)) for j in range(d)]
    geom["strides"] = [int(np.int64(m[o + 2 * SJ_MAX_DIM + j]).astype(np.uint64)) for j in range(d)]
    o += 3 * SJ_MAX_DIM
    geom["mask_offsets"] = [int(m[o + j]) for j in range(d + 1)]
    return geom, n, n_cells, mask_bits


ARRAY_SPECS = ("B", "G", "A", "pcell", "X", "masks")


def _shapes(n: int, d: int, n_cells: int, mask_bits: int) -> Dict[str, Tuple[tuple, str]]:
    # torch has no unsigned 64/32-bit collectives: int64/int32 carry the same bits
    return {"B": ((n_cells,), "int64"), "G": ((n_cells + 1,), "int32"), "A": ((n,), "int32"),
            "pcell": ((n,), "int32"), "X": ((d, n), "float64"), "masks": (((mask_bits + 31) // 32,), "int32")}


def broadcast_index_arrays(arrays: Optional[Dict[str, "torch.Tensor"]], meta: Optional[np.ndarray],
                           device, group=None, src: int = 0):
    """Broadcast geometry + index arrays from `src`.  Returns (meta, arrays) on every rank.

    `arrays` (rank src only): B, G, A, pcell, X[, masks] as tensors on `device` (dtype bits as in
    ``_shapes``).  Other ranks pass None and receive freshly allocated tensors.
    """
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    mt = torch.zeros(_META_WORDS, dtype=torch.int64, device=device)
    if rank == src:
        mt.copy_(torch.from_numpy(np.asarray(meta, dtype=np.int64)))
    dist.broadcast(mt, src=src, group=group)
    meta = mt.cpu().numpy()
    geom, n, n_cells, mask_bits = unpack_meta(meta)
    out = {}
    for name, (shape, dt) in _shapes(n, geom["d"], n_cells, mask_bits).items():
        if name == "masks" and mask_bits == 0:
            continue
        if rank == src:
            t = arrays[name]
            t = t.view(getattr(torch, dt)) if t.dtype != getattr(torch, dt) else t
            t = t.reshape(shape).contiguous()
        else:
            t = torch.empty(shape, dtype=getattr(torch, dt), device=device)
        dist.broadcast(t, src=src, group=group)
        out[name] = t
    return meta, out


def index_to_arrays(idx) -> Tuple[np.ndarray, Dict[str, "torch.Tensor"]]:
    """(meta, arrays) of a built sj index, arrays as zero-copy device tensors."""
    import torch
    g = idx.geometry()
    arr = idx.arrays()
    mask_bits = int(g["mask_offsets"][-1]) if "masks" in arr else 0
    meta = pack_meta(g, idx.n, idx.n_cells, mask_bits)
    conv = {"B": torch.int64, "G": torch.int32, "A": torch.int32, "pcell": torch.int32, "masks": torch.int32}
    out = {k: (v.view(conv[k]) if k in conv else v) for k, v in arr.items()}
    return meta, out


def arrays_to_index(meta: np.ndarray, arrays: Dict[str, "torch.Tensor"], device: int):
    """sj_index_import of broadcast arrays (copied into a library-owned index)."""
    import ctypes
    from . import sj
    geom, n, n_cells, mask_bits = unpack_meta(meta)
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
    for name in ("B", "G", "A", "pcell", "X"):
        setattr(v, name, ctypes.c_void_p(arrays[name].data_ptr()))
    v.masks = ctypes.c_void_p(arrays["masks"].data_ptr()) if mask_bits and "masks" in arrays else None
    return sj.import_index(v, device)


def plan_shards(n: int, world: int, weights: Optional[Sequence[float]] = None) -> np.ndarray:
    """Contiguous A-order query ranges [cuts[r], cuts[r+1]) for `world` ranks.

    With per-query work weights (e.g. sampled estimator counts expanded to queries), ranges are
    cut at equal cumulative weight; otherwise at equal query counts."""
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
    cuts = np.maximum.accumulate(np.array(cuts, dtype=np.int64))
    return cuts


def allreduce_counts(values: Sequence[int], device, op: str = "sum", group=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.int64 if op == "sum" else torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=group)
    return t.cpu().numpy()


def sharded_self_join(points, eps: float, device: int, group=None, **join_kw):
    """Full multi-GPU step: rank-0 build -> broadcast -> import -> shard join -> all-reduce.

    Returns (local Result, global pair count, local index)."""
    import torch
    import torch.distributed as dist
    from . import sj
    if dist.is_available() and dist.is_initialized():
        rank, world = dist.get_rank(group), dist.get_world_size(group)
    else:
        rank, world = 0, 1
    dev = torch.device("cuda", device)
    if world == 1:
        idx = sj.build_index(points, eps, device=device)
        res = sj.self_join(idx, **join_kw)
        return res, res.n_pairs, idx
    if rank == 0:
        idx0 = sj.build_index(points, eps, device=device)
        meta, arrays = index_to_arrays(idx0)
    else:
        idx0, meta, arrays = None, None, None
    meta, arrays = broadcast_index_arrays(arrays, meta, dev, group=group)
    idx = idx0 if rank == 0 else arrays_to_index(meta, arrays, device)
    n = idx.n
    cuts = plan_shards(n, world)
    a, b = int(cuts[rank]), int(cuts[rank + 1])
    res = sj.self_join(idx, query_begin=a, query_end=b, **join_kw) if b > a else None
    local = res.n_pairs if res is not None else 0
    total = int(allreduce_counts([local], dev, group=group)[0])
    return res, total, idx
