"""Thin Python binding of libsj (include/sj.h) -- argument marshalling only.

Every step of the self-join runs in the CUDA library; there is no CPU fallback: if libsj.so is
missing or no GPU is present the calls raise (``SJError`` / ``RuntimeError``).

    idx = build_index(points, eps)              # points: torch tensor (cuda or cpu) or numpy N x d f64
    res = self_join(idx)                        # device-resident batches (torch uint64 views)
    pairs = res.to_numpy(sort=True)             # canonical order
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SJ_LIB") or os.path.join(_PKG, "libsj.so")   # SJ_LIB: experiment override

SJ_MAX_DIM = 6
STATUS = {0: "SJ_OK", 1: "SJ_ERR_ARG", 2: "SJ_ERR_NONFINITE", 3: "SJ_ERR_DIM", 4: "SJ_ERR_KEY_OVERFLOW",
          5: "SJ_ERR_NOMEM", 6: "SJ_ERR_CUDA", 7: "SJ_ERR_EPS_MISMATCH", 8: "SJ_ERR_STATE"}

u64, u32, i32, dbl, f32, vp = (ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double,
                               ctypes.c_float, ctypes.c_void_p)


class BuildOpts(ctypes.Structure):
    _fields_ = [("device", i32), ("points_on_device", i32), ("stream", vp), ("build_masks", i32),
                ("speculative_estimate", i32)]


class JoinOpts(ctypes.Structure):
    _fields_ = [("unicomp", i32), ("include_self", i32), ("batch_capacity_pairs", u64),
                ("min_batches", i32), ("n_streams", i32), ("result_on_host", i32),
                ("query_begin", u64), ("query_end", u64), ("use_masks", i32), ("lanes_per_query", i32),
                ("dense_cells", i32), ("sort_pairs", i32), ("drain_csr", i32)]


class Stats(ctypes.Structure):
    _fields_ = [("pairs", u64), ("cells_probed", u64), ("candidates_tested", u64),
                ("estimated_pairs", u64), ("batches", u32), ("retries", u32),
                ("estimate_ms", f32), ("refine_ms", f32), ("refine_max_ms", f32), ("total_ms", f32),
                ("refine_launches", u32), ("refine_span_ms", f32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class KnnStats(ctypes.Structure):
    _fields_ = [("rounds", ctypes.c_uint32), ("eps_final", ctypes.c_double), ("cells_probed", ctypes.c_uint64),
                ("candidates_tested", ctypes.c_uint64)]


class IndexView(ctypes.Structure):
    _fields_ = [("d", i32), ("device", i32), ("n", u64), ("n_cells", u64),
                ("eps", dbl), ("eps2", dbl), ("w", dbl),
                ("mins", dbl * SJ_MAX_DIM), ("cpd", u64 * SJ_MAX_DIM), ("strides", u64 * SJ_MAX_DIM),
                ("key_bits", i32), ("mask_offsets", u64 * (SJ_MAX_DIM + 1)),
                ("B", vp), ("G", vp), ("A", vp), ("pcell", vp), ("X", vp), ("masks", vp),
                ("dir_k", i32), ("dir_entries", u64), ("dir", vp),
                ("t_h2d_ms", f32), ("t_geometry_ms", f32), ("t_keys_ms", f32), ("t_sort_ms", f32),
                ("t_compact_ms", f32), ("t_total_ms", f32),
                ("packed", vp), ("packed_bytes", u64), ("off_X", u64), ("off_A", u64), ("off_pcell", u64),
                ("off_G", u64), ("off_masks", u64), ("off_B", u64)]


class SJError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libsj.so (fails loudly: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SJ_LIBRARY", path)      # experiment builds (tools/variants.sh); same ABI
    if not os.path.exists(path):
        raise RuntimeError(f"libsj.so not built at {path}: run `python -m paper_1803_04120_b200.build` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(path)
    P = ctypes.POINTER
    L.sj_build_opts_default.argtypes = [P(BuildOpts)]
    L.sj_build_opts_default.restype = None
    L.sj_join_opts_default.argtypes = [P(JoinOpts)]
    L.sj_join_opts_default.restype = None
    L.sj_build_index.argtypes = [vp, u64, i32, dbl, P(BuildOpts), P(vp)]
    L.sj_build_index.restype = i32
    L.sj_self_join.argtypes = [vp, P(JoinOpts), P(vp)]
    L.sj_self_join.restype = i32
    L.sj_self_join_points.argtypes = [vp, u64, i32, dbl, P(BuildOpts), P(JoinOpts), P(vp), P(vp)]
    L.sj_self_join_points.restype = i32
    L.sj_free_result.argtypes = [vp]
    L.sj_free_result.restype = None
    L.sj_free_result_async.argtypes = [vp, vp]
    L.sj_free_result_async.restype = None
    L.sj_result_fingerprint.argtypes = [vp, vp, vp]
    L.sj_result_fingerprint.restype = i32
    L.sj_plan_shards.argtypes = [vp, u32, vp]
    L.sj_plan_shards.restype = i32
    L.sj_diag_fp64_peak.argtypes = [i32, P(dbl), P(dbl)]
    L.sj_diag_fp64_peak.restype = i32
    L.sj_trim.argtypes = [i32]
    L.sj_trim.restype = i32
    L.sj_set_result_cache_limit.argtypes = [u64]
    L.sj_set_result_cache_limit.restype = None
    L.sj_free_index.argtypes = [vp]
    L.sj_free_index.restype = None
    L.sj_result_info.argtypes = [vp, P(u64), P(u32), P(Stats)]
    L.sj_result_info.restype = i32
    L.sj_result_batch.argtypes = [vp, u32, P(vp), P(u64), P(i32)]
    L.sj_result_batch.restype = i32
    L.sj_result_batch_csr.argtypes = [vp, u32, P(vp), P(vp), P(u64), P(u64)]
    L.sj_result_batch_csr.restype = i32
    L.sj_dbscan.argtypes = [vp, u32, vp, P(u64), P(u64), P(u64)]
    L.sj_dbscan.restype = i32
    L.sj_result_n_points.argtypes = [vp, P(u64)]
    L.sj_result_n_points.restype = i32
    L.sj_result_counters.argtypes = [vp, P(u64)]
    L.sj_result_counters.restype = i32
    L.sj_result_copy_to_host.argtypes = [vp, vp, u64]
    L.sj_result_copy_to_host.restype = i32
    L.sj_result_to_csr.argtypes = [vp, u64, vp, vp]
    L.sj_result_to_csr.restype = i32
    L.sj_neighbor_counts.argtypes = [vp, P(JoinOpts), vp, P(u64)]
    L.sj_neighbor_counts.restype = i32
    L.sj_brute_force_join.argtypes = [vp, u64, i32, dbl, P(BuildOpts), P(JoinOpts), P(vp)]
    L.sj_brute_force_join.restype = i32
    L.sj_join_sets.argtypes = [vp, vp, u64, i32, P(JoinOpts), P(vp)]
    L.sj_join_sets.restype = i32
    L.sj_self_join_f32.argtypes = [vp, u64, i32, ctypes.c_float, P(BuildOpts), P(JoinOpts), P(vp)]
    L.sj_self_join_f32.restype = i32
    L.sj_knn_join.argtypes = [vp, u64, vp, u64, i32, u32, dbl, P(BuildOpts), vp, vp, P(KnnStats)]
    L.sj_knn_join.restype = i32
    L.sj_knn_self.argtypes = [vp, u64, i32, u32, dbl, P(BuildOpts), vp, vp, P(KnnStats)]
    L.sj_knn_self.restype = i32
    L.sj_index_export.argtypes = [vp, P(IndexView)]
    L.sj_index_export.restype = i32
    L.sj_index_timings.argtypes = [vp, P(IndexView)]
    L.sj_index_timings.restype = i32
    L.sj_index_import.argtypes = [P(IndexView), i32, P(vp)]
    L.sj_index_import.restype = i32
    L.sj_index_import_borrowed.argtypes = [P(IndexView), i32, P(vp)]
    L.sj_index_import_borrowed.restype = i32
    L.sj_set_allocator.argtypes = [vp, vp, vp]
    L.sj_set_allocator.restype = None
    L.sj_plan_batches.argtypes = [vp, u64, u64, u64, u64, u64, i32, dbl, vp, u32, P(u32), P(u64)]
    L.sj_plan_batches.restype = i32
    L.sj_kernel_launches.argtypes = []
    L.sj_kernel_launches.restype = u64
    L.sj_last_error.argtypes = []
    L.sj_last_error.restype = ctypes.c_char_p
    L.sj_abi_version.argtypes = []
    L.sj_abi_version.restype = i32
    _lib = L
    return L


def _check(st: int):
    if st != 0:
        msg = _lib.sj_last_error().decode(errors="replace")
        raise SJError(st, msg)


def kernel_launches() -> int:
    return int(load_library().sj_kernel_launches())


_JOIN_DEFAULTS = None


def join_opts(**kw) -> JoinOpts:
    global _JOIN_DEFAULTS
    if _JOIN_DEFAULTS is None:
        d0 = JoinOpts()
        load_library().sj_join_opts_default(ctypes.byref(d0))
        _JOIN_DEFAULTS = bytes(d0)
    o = JoinOpts.from_buffer_copy(_JOIN_DEFAULTS)
    for k, v in kw.items():
        if v is None:
            continue
        if not hasattr(o, k):
            raise TypeError(f"unknown join option {k}")
        setattr(o, k, int(v))
    return o


class Index:
    """An sj_index handle (device-resident, immutable)."""

    def __init__(self, handle: int, keepalive=None):
        self._h = ctypes.c_void_p(handle)
        self._keep = keepalive
        self.view = IndexView()
        _check(load_library().sj_index_export(self._h, ctypes.byref(self.view)))

    @property
    def handle(self):
        return self._h

    @property
    def n(self) -> int:
        return int(self.view.n)

    @property
    def d(self) -> int:
        return int(self.view.d)

    @property
    def n_cells(self) -> int:
        return int(self.view.n_cells)

    @property
    def device(self) -> int:
        return int(self.view.device)

    def geometry(self) -> dict:
        v = self.view
        d = v.d
        return dict(d=d, n=v.n, n_cells=v.n_cells, eps=v.eps, eps2=v.eps2, w=v.w,
                    mins=list(v.mins[:d]), cpd=list(v.cpd[:d]), strides=list(v.strides[:d]),
                    key_bits=v.key_bits, mask_offsets=list(v.mask_offsets[:d + 1]),
                    dir_k=v.dir_k, dir_entries=v.dir_entries)

    def timings(self) -> dict:
        v = IndexView()
        _check(load_library().sj_index_timings(self._h, ctypes.byref(v)))
        return dict(h2d_ms=v.t_h2d_ms, geometry_ms=v.t_geometry_ms, keys_ms=v.t_keys_ms,
                    sort_ms=v.t_sort_ms, compact_ms=v.t_compact_ms, total_ms=v.t_total_ms)

    def arrays(self) -> dict:
        """Zero-copy torch views of the device arrays (B, G, A, pcell, X, masks)."""
        import torch
        v = self.view
        n, nG, d = int(v.n), int(v.n_cells), int(v.d)
        out = {
            "B": _device_tensor(v.B, (nG,), torch.uint64, self.device, self),
            "G": _device_tensor(v.G, (nG + 1,), torch.uint32, self.device, self),
            "A": _device_tensor(v.A, (n,), torch.uint32, self.device, self),
            "pcell": _device_tensor(v.pcell, (n,), torch.uint32, self.device, self),
            "X": _device_tensor(v.X, (d, n), torch.float64, self.device, self),
        }
        if v.masks:
            words = (int(v.mask_offsets[d]) + 31) // 32
            out["masks"] = _device_tensor(v.masks, (words,), torch.uint32, self.device, self)
        if v.dir:
            out["dir"] = _device_tensor(v.dir, (int(v.dir_entries),), torch.uint32, self.device, self)
        return out

    def packed(self):
        """Zero-copy uint8 device tensor of the index's contiguous array buffer
        (sj_index_view.packed: X, A, pcell, G, masks, B at the view's off_* offsets), or None."""
        import torch
        v = self.view
        if not v.packed:
            return None
        return _device_tensor(v.packed, (int(v.packed_bytes),), torch.uint8, self.device, self)

    def free(self):
        if self._h and self._h.value:
            load_library().sj_free_index(self._h)
            self._h = ctypes.c_void_p(0)
        self._keep = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class _CudaArray:
    """__cuda_array_interface__ wrapper so torch.as_tensor can view library-owned memory."""

    def __init__(self, ptr: int, shape, typestr: str, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr or 0), False), "version": 3, "strides": None}
        self._owner = owner


_TYPESTR = {"uint64": "<u8", "uint32": "<u4", "float64": "<f8", "uint8": "|u1"}


def _device_tensor(ptr, shape, dtype, device, owner):
    import torch
    name = str(dtype).replace("torch.", "")
    if int(np.prod(shape)) == 0:
        return torch.empty(shape, dtype=dtype, device=f"cuda:{device}")
    t = torch.as_tensor(_CudaArray(ptr, shape, _TYPESTR[name], owner), device=f"cuda:{device}")
    return t


_BUILD_DEFAULTS = None
_torch = None


def _current_stream(dev: int) -> int:
    """torch's current CUDA stream of a device as a raw handle (the cheap accessor when present: this
    sits in every step's host path)."""
    raw = getattr(_torch._C, "_cuda_getCurrentRawStream", None)
    return raw(dev) if raw is not None else _torch.cuda.current_stream(dev).cuda_stream


def _points_arg(points, device, stream, build_masks=True, speculative_estimate=True):
    """(BuildOpts, pointer, n, d, keepalive) for sj_build_index / sj_self_join_points."""
    global _BUILD_DEFAULTS, _torch
    if _BUILD_DEFAULTS is None:
        d0 = BuildOpts()
        load_library().sj_build_opts_default(ctypes.byref(d0))
        _BUILD_DEFAULTS = bytes(d0)
    o = BuildOpts.from_buffer_copy(_BUILD_DEFAULTS)
    o.build_masks = int(build_masks)
    o.speculative_estimate = int(speculative_estimate)
    if _torch is None:
        try:
            import torch
            _torch = torch
        except ImportError:  # pragma: no cover
            _torch = False
    is_torch = bool(_torch) and isinstance(points, _torch.Tensor)
    if is_torch:
        t = points
        if t.dtype != _torch.float64 or t.dim() != 2:
            raise TypeError("points must be a 2-D float64 tensor")
        if not t.is_contiguous():
            t = t.contiguous()
        n, d = t.shape
        if t.is_cuda:
            o.points_on_device = 1
            dev = t.get_device()
            o.device = dev if device is None else device
            o.stream = ctypes.c_void_p(_current_stream(dev)) if stream is None else ctypes.c_void_p(stream)
        else:
            o.points_on_device = 0
            o.device = 0 if device is None else device
        return o, t.data_ptr(), n, d, t
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim != 2:
        raise TypeError("points must be N x d")
    n, d = a.shape
    o.points_on_device = 0
    o.device = 0 if device is None else device
    return o, a.ctypes.data, n, d, a


def build_index(points, eps: float, device: Optional[int] = None, stream=None, build_masks: bool = True,
                speculative_estimate: bool = True) -> Index:
    """sj_build_index.  points: N x d float64 (torch cuda/cpu tensor or numpy array)."""
    L = load_library()
    o, ptr, n, d, keep = _points_arg(points, device, stream, build_masks, speculative_estimate)
    h = ctypes.c_void_p()
    _check(L.sj_build_index(ctypes.c_void_p(ptr), n, d, float(eps), ctypes.byref(o), ctypes.byref(h)))
    del keep
    return Index(h.value)


def join_points(points, eps: float, device: Optional[int] = None, stream=None, keep_index: bool = True,
                **join_kw):
    """sj_self_join_points: build + join in one library call -> (Result, Index or None)."""
    L = load_library()
    o, ptr, n, d, keep = _points_arg(points, device, stream)
    jo = join_opts(**join_kw)
    hi, hr = ctypes.c_void_p(), ctypes.c_void_p()
    _check(L.sj_self_join_points(ctypes.c_void_p(ptr), n, d, float(eps), ctypes.byref(o), ctypes.byref(jo),
                                 ctypes.byref(hi) if keep_index else None, ctypes.byref(hr)))
    del keep
    r = Result(hr.value)
    r.device = o.device
    return r, (Index(hi.value) if keep_index else None)


class Result:
    """An sj_result handle; batches are zero-copy views (torch on device, numpy on host)."""

    def __init__(self, handle: int):
        self._h = ctypes.c_void_p(handle)
        L = load_library()
        n, nb = u64(), u32()
        _check(L.sj_result_info(self._h, ctypes.byref(n), ctypes.byref(nb), None))
        self.n_pairs = int(n.value)
        self.n_batches = int(nb.value)
        self._stats = None
        self.device = None

    @property
    def stats(self) -> dict:
        """Work counters and device timings (the timings are computed from the join's CUDA
        events on this first access, off the join's critical path)."""
        if self._stats is None:
            st = Stats()
            _check(load_library().sj_result_info(self._h, None, None, ctypes.byref(st)))
            self._stats = st.as_dict()
        return self._stats

    @property
    def counters(self) -> dict:
        """sj_result_counters: pairs, cells_probed, candidates_tested, retries (no event queries)."""
        c = (u64 * 4)()
        _check(load_library().sj_result_counters(self._h, c))
        return {"pairs": int(c[0]), "cells_probed": int(c[1]), "candidates_tested": int(c[2]), "retries": int(c[3])}

    def batch(self, b: int):
        L = load_library()
        p, n, dev = vp(), u64(), i32()
        _check(L.sj_result_batch(self._h, b, ctypes.byref(p), ctypes.byref(n), ctypes.byref(dev)))
        if dev.value:
            import torch
            d = torch.cuda.current_device() if self.device is None else self.device
            return _device_tensor(p.value, (int(n.value),), torch.uint64, d, self)
        if n.value == 0:
            return np.empty(0, dtype=np.uint64)
        buf = (ctypes.c_uint64 * int(n.value)).from_address(p.value)
        arr = np.ctypeslib.as_array(buf)
        arr.flags.writeable = False
        return arr

    def batch_csr(self, b: int):
        """sj_result_batch_csr (drain_csr results) -> (row_offsets uint32[N+1], neighbors uint32[n]):
        zero-copy numpy views of the pinned host block; the neighbours of key i held by batch b are
        neighbors[row_offsets[i]:row_offsets[i+1]]."""
        L = load_library()
        po, pn, rows, n = vp(), vp(), u64(), u64()
        _check(L.sj_result_batch_csr(self._h, b, ctypes.byref(po), ctypes.byref(pn), ctypes.byref(rows),
                                     ctypes.byref(n)))
        offs = np.ctypeslib.as_array((ctypes.c_uint32 * (int(rows.value) + 1)).from_address(po.value))
        nb = (np.ctypeslib.as_array((ctypes.c_uint32 * int(n.value)).from_address(pn.value)) if n.value
              else np.empty(0, dtype=np.uint32))
        offs.flags.writeable = False
        nb.flags.writeable = False
        return offs, nb

    def batches(self):
        return [self.batch(b) for b in range(self.n_batches)]

    def to_numpy(self, sort: bool = True) -> np.ndarray:
        out = np.empty(self.n_pairs, dtype=np.uint64)
        _check(load_library().sj_result_copy_to_host(self._h, out.ctypes.data, self.n_pairs))
        if sort:
            out.sort()
        return out

    def to_csr(self, n_points: int):
        """sj_result_to_csr -> (row_offsets int64[n_points+1], neighbors int32[n_pairs]) on the device;
        neighbours of point i (original ids) are neighbors[row_offsets[i]:row_offsets[i+1]], ascending."""
        import torch
        dev = f"cuda:{self.device if self.device is not None else 0}"
        offsets = torch.empty(n_points + 1, dtype=torch.int64, device=dev)
        nbrs = torch.empty(max(self.n_pairs, 1), dtype=torch.int32, device=dev)
        _check(load_library().sj_result_to_csr(self._h, n_points, ctypes.c_void_p(offsets.data_ptr()),
                                               ctypes.c_void_p(nbrs.data_ptr())))
        return offsets, nbrs[:self.n_pairs]

    def fingerprint(self, counts: bool = False, n_points: Optional[int] = None):
        """sj_result_fingerprint -> (F_a, F_b) of the pair multiset, and with counts=True also the
        per-key counts (torch uint32 on the device, n_points entries = the joined N)."""
        fp = (ctypes.c_uint64 * 2)()
        cnt = None
        if counts:
            import torch
            dev = self.device if self.device is not None else 0
            cnt = torch.empty(int(n_points), dtype=torch.uint32, device=f"cuda:{dev}")
        _check(load_library().sj_result_fingerprint(self._h, fp, ctypes.c_void_p(cnt.data_ptr()) if counts else None))
        return (int(fp[0]), int(fp[1]), cnt) if counts else (int(fp[0]), int(fp[1]))

    def dbscan(self, min_pts: int):
        """sj_dbscan -> (labels torch.int32[N] on the device, {clusters, core, noise}): DBSCAN read off
        this (whole) self-join result; see include/sj.h for the label conventions."""
        import torch
        dev = self.device if self.device is not None else 0
        npts = self._n_points()
        labels = torch.empty(max(npts, 1), dtype=torch.int32, device=f"cuda:{dev}")
        nc, ncore, nn = u64(), u64(), u64()
        _check(load_library().sj_dbscan(self._h, int(min_pts), ctypes.c_void_p(labels.data_ptr()), ctypes.byref(nc),
                                        ctypes.byref(ncore), ctypes.byref(nn)))
        return labels[:npts], {"clusters": int(nc.value), "core": int(ncore.value), "noise": int(nn.value)}

    def _n_points(self) -> int:
        n = u64()
        _check(load_library().sj_result_n_points(self._h, ctypes.byref(n)))
        return int(n.value)

    def free(self, stream=None):
        """Release the result; its device buffers are reused only after the work queued on
        `stream` (default: torch's current stream of the result's device) completed."""
        if self._h and self._h.value:
            L = load_library()
            st = stream
            if st is None and self.device is not None:
                try:
                    import torch
                    st = torch.cuda.current_stream(self.device).cuda_stream
                except Exception:
                    st = None
            L.sj_free_result_async(self._h, ctypes.c_void_p(st) if st else None)
            self._h = ctypes.c_void_p(0)

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def fp64_peak(device: int = 0) -> dict:
    """sj_diag_fp64_peak: measured DADD / DMUL throughput (operations/s) of the FP64 pipe."""
    a, m = dbl(), dbl()
    _check(load_library().sj_diag_fp64_peak(int(device), ctypes.byref(a), ctypes.byref(m)))
    return {"dadd_ops_per_s": a.value, "dmul_ops_per_s": m.value}


_ALLOC_CB = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p)
_RELEASE_CB = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p)
_hook_refs = None


def use_torch_allocator(enable: bool = True):
    """sj_set_allocator wired to PyTorch's caching allocator: every device allocation of the library
    (index arrays, result batches, build scratch) then comes from -- and returns to -- torch's pool,
    so the library and the surrounding PyTorch program share one device-memory budget
    (north_star: "PyTorch used only for device memory, streams and process groups").  enable=False
    restores the library's own stream-ordered pool.  Allocations made under one allocator are
    released by the same one (the library records each allocation's provenance)."""
    global _hook_refs
    L = load_library()
    if not enable:
        L.sj_set_allocator(None, None, None)
        _hook_refs = None
        return
    import torch

    def _alloc(nbytes, dev, stream, ctx):
        try:
            return int(torch.cuda.caching_allocator_alloc(int(nbytes), int(dev), int(stream or 0)))
        except Exception:
            return None

    def _release(ptr, ctx):
        if ptr:
            torch.cuda.caching_allocator_delete(int(ptr))

    a, r = _ALLOC_CB(_alloc), _RELEASE_CB(_release)
    _hook_refs = (a, r)                       # the C library keeps raw pointers to these thunks
    L.sj_set_allocator(ctypes.cast(a, ctypes.c_void_p), ctypes.cast(r, ctypes.c_void_p), None)


def trim(device: int = -1):
    """sj_trim: release the library's caches (result batches, build scratch, pinned blocks, pool)."""
    _check(load_library().sj_trim(int(device)))


def set_result_cache_limit(nbytes: int):
    load_library().sj_set_result_cache_limit(int(nbytes))


def self_join(index: Index, unicomp: bool = True, include_self: bool = True,
              batch_capacity_pairs: Optional[int] = None, min_batches: Optional[int] = None,
              n_streams: Optional[int] = None, result_on_host: bool = False,
              query_begin: int = 0, query_end: int = 0, use_masks: bool = True,
              lanes_per_query: int = 0, dense_cells: bool = True, sort_pairs: bool = False,
              drain_csr: bool = False) -> Result:
    """sj_self_join over the index; see include/sj.h for the option semantics."""
    L = load_library()
    o = join_opts(unicomp=unicomp, include_self=include_self, batch_capacity_pairs=batch_capacity_pairs,
                  min_batches=min_batches, n_streams=n_streams, result_on_host=result_on_host,
                  query_begin=query_begin, query_end=query_end, use_masks=use_masks,
                  lanes_per_query=lanes_per_query, dense_cells=dense_cells, sort_pairs=sort_pairs,
                  drain_csr=drain_csr)
    h = ctypes.c_void_p()
    _check(L.sj_self_join(index.handle, ctypes.byref(o), ctypes.byref(h)))
    r = Result(h.value)
    r.device = index.device
    return r


def neighbor_counts(index: Index, unicomp: bool = True, include_self: bool = True,
                    query_begin: int = 0, query_end: int = 0, out=None, lanes_per_query: int = 0):
    """sj_neighbor_counts -> (torch uint32 counts by original id on the device, total)."""
    import torch
    L = load_library()
    o = join_opts(unicomp=unicomp, include_self=include_self, query_begin=query_begin, query_end=query_end,
                  lanes_per_query=lanes_per_query)
    if out is None:
        out = torch.empty(index.n, dtype=torch.uint32, device=f"cuda:{index.device}")
    tot = u64()
    _check(L.sj_neighbor_counts(index.handle, ctypes.byref(o), ctypes.c_void_p(out.data_ptr()), ctypes.byref(tot)))
    return out, int(tot.value)


def brute_force_join(points, eps: float, include_self: bool = True, result_on_host: bool = False,
                     sort_pairs: bool = False, device: Optional[int] = None) -> Result:
    """sj_brute_force_join: all-pairs GPU join, O(N^2)."""
    import torch
    L = load_library()
    bo = BuildOpts()
    L.sj_build_opts_default(ctypes.byref(bo))
    if isinstance(points, torch.Tensor):
        t = points.contiguous()
        if t.dtype != torch.float64 or t.dim() != 2:
            raise TypeError("points must be a 2-D float64 tensor")
        keep, ptr = t, t.data_ptr()
        bo.points_on_device = int(t.is_cuda)
        bo.device = (t.device.index if t.is_cuda else 0) if device is None else device
        n, d = t.shape
    else:
        a = np.ascontiguousarray(points, dtype=np.float64)
        keep, ptr = a, a.ctypes.data
        bo.points_on_device = 0
        bo.device = 0 if device is None else device
        n, d = a.shape
    o = join_opts(include_self=include_self, result_on_host=result_on_host, sort_pairs=sort_pairs)
    h = ctypes.c_void_p()
    _check(L.sj_brute_force_join(ctypes.c_void_p(ptr), n, d, float(eps), ctypes.byref(bo), ctypes.byref(o),
                                 ctypes.byref(h)))
    del keep
    r = Result(h.value)
    r.device = bo.device
    return r


def join_sets(index: Index, queries, batch_capacity_pairs: Optional[int] = None, min_batches: Optional[int] = None,
              result_on_host: bool = False, sort_pairs: bool = False) -> Result:
    """sj_join_sets ("the related similarity join"; R19): pairs (i<<32|k) of query
    row i and index point k within the index's eps.  queries: nq x d float64 torch tensor (cuda on the
    index's device, or cpu) or numpy array."""
    import torch
    L = load_library()
    if isinstance(queries, torch.Tensor):
        t = queries.contiguous()
        if t.dtype != torch.float64 or t.dim() != 2:
            raise TypeError("queries must be a 2-D float64 tensor")
        keep, ptr, on_dev = t, t.data_ptr(), int(t.is_cuda)
        nq, d = t.shape
    else:
        a = np.ascontiguousarray(queries, dtype=np.float64)
        if a.ndim != 2:
            raise TypeError("queries must be nq x d")
        keep, ptr, on_dev = a, a.ctypes.data, 0
        nq, d = a.shape
    if d != index.d:
        raise ValueError(f"queries have d={d}, the index d={index.d}")
    kw = dict(result_on_host=result_on_host, sort_pairs=sort_pairs)
    if batch_capacity_pairs is not None:
        kw["batch_capacity_pairs"] = batch_capacity_pairs
    if min_batches is not None:
        kw["min_batches"] = min_batches
    o = join_opts(**kw)
    h = ctypes.c_void_p()
    _check(L.sj_join_sets(index.handle, ctypes.c_void_p(ptr if nq else None), nq, on_dev, ctypes.byref(o),
                          ctypes.byref(h)))
    del keep
    r = Result(h.value)
    r.device = index.device
    return r


def self_join_f32(points, eps: float, include_self: bool = True, result_on_host: bool = False,
                  sort_pairs: bool = False, batch_capacity_pairs: Optional[int] = None,
                  min_batches: Optional[int] = None, device: Optional[int] = None) -> Result:
    """sj_self_join_f32 (PAPER.md:393 32-bit floats; R21): the self-join of float32 points with
    the predicate evaluated in binary32.  points: n x d float32 torch tensor (cuda or cpu) or numpy."""
    import torch
    L = load_library()
    bo = BuildOpts()
    L.sj_build_opts_default(ctypes.byref(bo))
    if isinstance(points, torch.Tensor):
        t = points.contiguous()
        if t.dtype != torch.float32 or t.dim() != 2:
            raise TypeError("points must be a 2-D float32 tensor")
        keep, ptr = t, t.data_ptr()
        bo.points_on_device = int(t.is_cuda)
        bo.device = (t.device.index if t.is_cuda else 0) if device is None else device
        n, d = t.shape
    else:
        a = np.ascontiguousarray(points, dtype=np.float32)
        if a.ndim != 2:
            raise TypeError("points must be n x d")
        keep, ptr = a, a.ctypes.data
        bo.points_on_device = 0
        bo.device = 0 if device is None else device
        n, d = a.shape
    kw = dict(include_self=include_self, result_on_host=result_on_host, sort_pairs=sort_pairs)
    if batch_capacity_pairs is not None:
        kw["batch_capacity_pairs"] = batch_capacity_pairs
    if min_batches is not None:
        kw["min_batches"] = min_batches
    o = join_opts(**kw)
    h = ctypes.c_void_p()
    _check(L.sj_self_join_f32(ctypes.c_void_p(ptr), n, d, float(np.float32(eps)), ctypes.byref(bo), ctypes.byref(o),
                              ctypes.byref(h)))
    del keep
    r = Result(h.value)
    r.device = bo.device
    return r


def knn_self(points, k: int, eps0: float, device: Optional[int] = None, with_stats: bool = False):
    """sj_knn_self (PAPER.md:609 kNN; R20): for every point its k nearest other points,
    ascending in (s, id) -> (ids int32 [n, k], dist2 float64 [n, k]) cuda tensors (+ stats dict)."""
    import torch
    L = load_library()
    bo, ptr, n, d, keep = _points_arg(points, device, None)
    bo.stream = None
    bo.speculative_estimate = 0
    dev = bo.device
    ids = torch.empty((n, k), dtype=torch.int32, device=f"cuda:{dev}")
    dist2 = torch.empty((n, k), dtype=torch.float64, device=f"cuda:{dev}")
    st = KnnStats()
    _check(L.sj_knn_self(ctypes.c_void_p(ptr), n, d, int(k), float(eps0), ctypes.byref(bo),
                         ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(dist2.data_ptr()), ctypes.byref(st)))
    del keep
    if with_stats:
        return ids, dist2, dict(rounds=st.rounds, eps_final=st.eps_final, cells_probed=st.cells_probed,
                                candidates_tested=st.candidates_tested)
    return ids, dist2


def knn_join(points, queries, k: int, eps0: float, device: Optional[int] = None, with_stats: bool = False):
    """sj_knn_join: for every query row its k nearest points (ascending (s, id)), nothing excluded ->
    (ids int32 [nq, k], dist2 float64 [nq, k]) cuda tensors (+ stats).  points / queries: both torch cuda
    tensors on one device, or both host (numpy / cpu tensors)."""
    import torch
    L = load_library()
    bo, ptr, n, d, keep = _points_arg(points, device, None)
    bo.stream = None
    bo.speculative_estimate = 0
    if isinstance(queries, torch.Tensor):
        qt = queries.contiguous()
        if qt.dtype != torch.float64 or qt.dim() != 2:
            raise TypeError("queries must be a 2-D float64 tensor")
        if bool(qt.is_cuda) != bool(bo.points_on_device):
            raise ValueError("points and queries must both be on the device or both on the host")
        qkeep, qptr = qt, qt.data_ptr()
        nq, dq = qt.shape
    else:
        if bo.points_on_device:
            raise ValueError("points and queries must both be on the device or both on the host")
        qa = np.ascontiguousarray(queries, dtype=np.float64)
        qkeep, qptr = qa, qa.ctypes.data
        nq, dq = qa.shape
    if dq != d:
        raise ValueError("dimension mismatch")
    dev = bo.device
    ids = torch.empty((nq, k), dtype=torch.int32, device=f"cuda:{dev}")
    dist2 = torch.empty((nq, k), dtype=torch.float64, device=f"cuda:{dev}")
    st = KnnStats()
    _check(L.sj_knn_join(ctypes.c_void_p(ptr), n, ctypes.c_void_p(qptr if nq else None), nq, d, int(k), float(eps0),
                         ctypes.byref(bo), ctypes.c_void_p(ids.data_ptr()), ctypes.c_void_p(dist2.data_ptr()),
                         ctypes.byref(st)))
    del keep, qkeep
    if with_stats:
        return ids, dist2, dict(rounds=st.rounds, eps_final=st.eps_final, cells_probed=st.cells_probed,
                                candidates_tested=st.candidates_tested)
    return ids, dist2


def plan_shards(index: Index, world: int) -> np.ndarray:
    """sj_plan_shards: A-order query cuts (world + 1 entries) balanced by the sampled estimate."""
    cuts = np.zeros(int(world) + 1, dtype=np.uint64)
    _check(load_library().sj_plan_shards(index.handle, int(world), cuts.ctypes.data))
    return cuts.astype(np.int64)


def import_index(view: IndexView, device: int, borrow=None) -> Index:
    """sj_index_import (arrays copied), or with borrow=<object owning the arrays>
    sj_index_import_borrowed: the index reads the view's arrays in place and keeps `borrow` alive."""
    L = load_library()
    h = ctypes.c_void_p()
    if borrow is None:
        _check(L.sj_index_import(ctypes.byref(view), device, ctypes.byref(h)))
        return Index(h.value)
    _check(L.sj_index_import_borrowed(ctypes.byref(view), device, ctypes.byref(h)))
    return Index(h.value, keepalive=borrow)


def plan_batches(sample_counts, step: int, q_begin: int, q_end: int, capacity: int, min_batches: int = 3,
                 margin: float = 0.25):
    """Host-only batch planner (sj_plan_batches): returns (cuts, estimated_total)."""
    L = load_library()
    c = np.ascontiguousarray(sample_counts, dtype=np.uint32)
    max_cuts = max(16, int(len(c)) * 4 + min_batches + 8)
    cuts = np.zeros(max_cuts + 1, dtype=np.uint64)
    k, tot = u32(), u64()
    _check(L.sj_plan_batches(c.ctypes.data if len(c) else None, len(c), step, q_begin, q_end, capacity,
                             min_batches, margin, cuts.ctypes.data, max_cuts, ctypes.byref(k), ctypes.byref(tot)))
    return cuts[: k.value + 1].copy(), int(tot.value)
