"""TEST INFRASTRUCTURE ONLY -- the independent CPU oracle for the epsilon self-join.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with the CUDA path
(``paper_1803_04120_b200``) and never imports it; the only thing both sides share is the
seeded input generators in ``datagen`` (which hold none of the method's arithmetic).

Contents, each citing the passage it follows (PAPER.md line numbers, SPEC.md as S.<line>):

* ``brute_force`` / ``grid_join`` / ``rows`` -- the join itself (§3), in plain C
  (``sj_oracle.c``, gcc -O2 -ffp-contract=off): brute force is the definition written out;
  the grid join is a filter with its own robust width and a full 3^d neighbourhood.
* ``index_ref`` -- the grid index of §4.2-4.4 (geometry, cell coordinates, linearisation, B, G,
  A, M) and the Alg. 1 / Alg. 2 cell enumerations, in plain numpy / Python, following the
  paper's notation with the DESIGN.md readings R6-R13.
* ``join_sets`` / ``knn`` -- the SURVEY.md §8(f) rank-4 variants on the same predicate
  (``sj_variants_oracle.c``): the two-set similarity join J(Q,P) (reading R19) by
  brute force or a sorted-tuple grid, and the kNN self-join (reading R20) by brute
  force with ties broken by the smaller id; ``brute_force_f32`` -- the self-join in binary32
  (reading R21).
* ``expected_pairs_uniform`` -- the exact expectation of |S| for iid uniform points (SURVEY.md
  §8(c) P4), used as a statistical pin.

Pins (tests/test_oracle_pins.py) tie every function here to something other than itself:
closed forms on integer lattices, the tie/self-pair worked examples of SPEC S.235-236,
S.272-273, S.316-317, the Figure 2 facts of PAPER.md:179/201-202, the P4 expectation,
symmetry, and brute force on tiny inputs.  ``estimate`` / batching has no oracle: "parity
unpinned" by design (reading R13) -- the result set is invariant to batching.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from typing import Iterable, Sequence

import numpy as np

from . import index_ref  # noqa: F401  (re-export)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sj_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "sj_variants_oracle.c")]
_LIB = os.path.join(_HERE, "libsj_oracle.so")
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fno-unsafe-math-optimizations",
          "-shared", "-fPIC", "-pthread", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile the C oracle (building the checker is not using it)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        p = ctypes.c_void_p
        lib.orc_pair_within.argtypes = [p, p, i32, dbl]
        lib.orc_pair_within.restype = i32
        lib.orc_brute_force.argtypes = [p, i64, i32, dbl, i32, p, i64]
        lib.orc_brute_force.restype = i64
        lib.orc_rows.argtypes = [p, i64, i32, dbl, i32, p, i64, i32, p, p]
        lib.orc_rows.restype = i64
        lib.orc_grid_join.argtypes = [p, i64, i32, dbl, i32, i64, i64, i32, p, p, i64]
        lib.orc_grid_join.restype = i64
        lib.orc_grid_digest.argtypes = [p, i64, i32, dbl, i32, i64, i64, i32, p, p]
        lib.orc_grid_digest.restype = i64
        lib.orc_join_sets_brute.argtypes = [p, i64, p, i64, i32, dbl, p, i64]
        lib.orc_join_sets_brute.restype = i64
        lib.orc_join_sets_grid.argtypes = [p, i64, p, i64, i32, dbl, i32, p, p, i64]
        lib.orc_join_sets_grid.restype = i64
        lib.orc_brute_force_f32.argtypes = [p, i64, i32, ctypes.c_float, i32, p, i64]
        lib.orc_brute_force_f32.restype = i64
        lib.orc_join_sets_digest.argtypes = [p, i64, p, i64, i32, dbl, i32, p, p]
        lib.orc_join_sets_digest.restype = i64
        lib.orc_knn.argtypes = [p, i64, p, p, i64, i32, i32, i32, p, p]
        lib.orc_knn.restype = i32
        lib.orc_mix.argtypes = [i32, ctypes.c_uint64]
        lib.orc_mix.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _pts(points) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("points must be N x d")
    return a


def default_threads() -> int:
    return os.cpu_count() or 1


def pair_within(a: Sequence[float], b: Sequence[float], eps: float) -> bool:
    """The predicate s(a,b) <= fl(eps*eps) (R1) as the C oracle evaluates it."""
    A = np.ascontiguousarray(a, dtype=np.float64)
    B = np.ascontiguousarray(b, dtype=np.float64)
    return bool(_load().orc_pair_within(_ptr(A), _ptr(B), len(A), float(eps)))


def brute_force(points, eps: float, include_self: bool = True) -> np.ndarray:
    """All ordered pairs (i<<32|k) with s(p_i,p_k) <= fl(eps^2), sorted."""
    P = _pts(points)
    n, d = P.shape
    lib = _load()
    total = lib.orc_brute_force(_ptr(P), n, d, float(eps), int(include_self), None, 0)
    if total < 0:
        raise ValueError("bad arguments")
    out = np.empty(total, dtype=np.uint64)
    lib.orc_brute_force(_ptr(P), n, d, float(eps), int(include_self), _ptr(out), total)
    return out


def grid_join(points, eps: float, include_self: bool = True, q0: int = 0, q1: int | None = None,
              nthreads: int | None = None, count_only: bool = False):
    """Pairs (or per-query counts) of queries [q0,q1) against all points; full 3^d scan."""
    P = _pts(points)
    n, d = P.shape
    q1 = n if q1 is None else q1
    nthreads = nthreads or default_threads()
    lib = _load()
    counts = np.zeros(max(q1 - q0, 0), dtype=np.int64)
    if count_only:
        total = lib.orc_grid_join(_ptr(P), n, d, float(eps), int(include_self), q0, q1, nthreads,
                                  _ptr(counts), None, 0)
        if total < 0:
            raise ValueError("bad arguments")
        return counts
    total = lib.orc_grid_join(_ptr(P), n, d, float(eps), int(include_self), q0, q1, nthreads,
                              _ptr(counts), None, 0)
    if total < 0:
        raise ValueError("bad arguments")
    out = np.empty(total, dtype=np.uint64)
    got = lib.orc_grid_join(_ptr(P), n, d, float(eps), int(include_self), q0, q1, nthreads,
                            None, _ptr(out), total)
    assert got == total
    return out


def grid_digest(points, eps: float, include_self: bool = True, q0: int = 0, q1: int | None = None,
                nthreads: int | None = None, with_counts: bool = False):
    """Order-independent fingerprints of S restricted to queries [q0,q1) (sj_oracle.c
    orc_grid_digest): returns dict(pairs=|S|, fa=F_a, fb=F_b, fc=F_c[, counts=per-query counts]).
    Fingerprints are sums mod 2^64, so they add over disjoint query ranges."""
    P = _pts(points)
    n, d = P.shape
    q1 = n if q1 is None else q1
    nthreads = nthreads or default_threads()
    counts = np.zeros(max(q1 - q0, 0), dtype=np.int64) if with_counts else None
    fp = np.zeros(3, dtype=np.uint64)
    total = _load().orc_grid_digest(_ptr(P), n, d, float(eps), int(include_self), q0, q1, nthreads,
                                    _ptr(counts) if counts is not None else None, _ptr(fp))
    if total < 0:
        raise ValueError("bad arguments")
    out = dict(pairs=int(total), fa=int(fp[0]), fb=int(fp[1]), fc=int(fp[2]))
    if with_counts:
        out["counts"] = counts
    return out


def mix(which: int, x: int) -> int:
    """The fingerprint mixers of sj_oracle.c (0: SplitMix64 output, 1: MurmurHash3 fmix64)."""
    return int(_load().orc_mix(int(which), ctypes.c_uint64(int(x) & (2**64 - 1))))


def fingerprint_pairs(pairs: np.ndarray) -> tuple:
    """(F_a, F_b) of an explicit pair array, via the C mixers (slow path for small arrays: tests)."""
    fa = fb = 0
    for x in np.asarray(pairs, dtype=np.uint64).tolist():
        fa = (fa + mix(0, x)) & (2**64 - 1)
        fb = (fb + mix(1, x)) & (2**64 - 1)
    return fa, fb


def rows(points, eps: float, qids: Iterable[int], include_self: bool = True,
         nthreads: int | None = None):
    """Brute-force neighbour rows of the given queries: (counts[nq], concatenated pairs)."""
    P = _pts(points)
    n, d = P.shape
    q = np.ascontiguousarray(np.asarray(list(qids) if not isinstance(qids, np.ndarray) else qids,
                                        dtype=np.int64))
    nthreads = nthreads or default_threads()
    lib = _load()
    counts = np.zeros(len(q), dtype=np.int64)
    total = lib.orc_rows(_ptr(P), n, d, float(eps), int(include_self), _ptr(q), len(q), nthreads,
                         _ptr(counts), None)
    out = np.empty(total, dtype=np.uint64)
    lib.orc_rows(_ptr(P), n, d, float(eps), int(include_self), _ptr(q), len(q), nthreads,
                 _ptr(counts), _ptr(out))
    return counts, out


def pair_counts(pairs: np.ndarray, n: int) -> np.ndarray:
    """cnt[i] = |{k : (i,k) in S}|."""
    keys = (np.asarray(pairs, dtype=np.uint64) >> np.uint64(32)).astype(np.int64)
    return np.bincount(keys, minlength=n)


def transpose_pairs(pairs: np.ndarray) -> np.ndarray:
    p = np.asarray(pairs, dtype=np.uint64)
    lo = p & np.uint64(0xFFFFFFFF)
    hi = p >> np.uint64(32)
    return np.sort((lo << np.uint64(32)) | hi)


def expected_pairs_uniform(n: int, d: int, eps: float, L: float = 100.0) -> float:
    """E|S| for n iid uniform points in [0,L]^d, self pairs included.

    E|S| = n + n(n-1) F_d(r), r = eps/L, where F_d(r) = P(|X-Y| <= r) for X,Y iid uniform in the
    unit cube: F_d(r) = sum_k (-1)^k C(d,k) pi^{(d-k)/2} / Gamma(1+(d+k)/2) r^{d+k}, exact for r<=1
    (the (d-k)-dim ball volume times the mixed-volume correction of the cube's boundary).
    """
    r = eps / L
    if r > 1.0:
        raise ValueError("formula exact only for eps <= L")
    F = 0.0
    for k in range(d + 1):
        F += ((-1) ** k) * math.comb(d, k) * math.pi ** ((d - k) / 2) / math.gamma(1 + (d + k) / 2) \
            * r ** (d + k)
    return n + n * (n - 1) * F


def join_sets(queries, points, eps: float, method: str = "grid", nthreads: int | None = None,
              count_only: bool = False):
    """J(Q,P) = {(i,k) : s(q_i,p_k) <= fl(eps^2)} packed (i<<32|k), sorted (sj_variants_oracle.c;
    PAPER.md:52 "the related similarity join", reading R19).  method: "brute" (the definition
    written out) or "grid" (sorted-tuple filter, full 3^d scan).  count_only: per-query counts."""
    Q = _pts(queries)
    P = _pts(points)
    if Q.shape[1] != P.shape[1]:
        raise ValueError("dimension mismatch")
    nq, d = Q.shape
    n = P.shape[0]
    lib = _load()
    if method == "brute":
        if count_only:
            raise ValueError("count_only needs method='grid'")
        total = lib.orc_join_sets_brute(_ptr(Q), nq, _ptr(P), n, d, float(eps), None, 0)
        if total < 0:
            raise ValueError("bad arguments")
        out = np.empty(total, dtype=np.uint64)
        lib.orc_join_sets_brute(_ptr(Q), nq, _ptr(P), n, d, float(eps), _ptr(out), total)
        return out
    nthreads = nthreads or default_threads()
    counts = np.zeros(nq, dtype=np.int64)
    total = lib.orc_join_sets_grid(_ptr(Q), nq, _ptr(P), n, d, float(eps), nthreads, _ptr(counts), None, 0)
    if total < 0:
        raise ValueError("bad arguments")
    if count_only:
        return counts
    out = np.empty(total, dtype=np.uint64)
    got = lib.orc_join_sets_grid(_ptr(Q), nq, _ptr(P), n, d, float(eps), nthreads, None, _ptr(out), total)
    assert got == total
    return out


def knn(points, k: int, qids: Iterable[int] | None = None, queries=None, nthreads: int | None = None):
    """k nearest neighbours by brute force (sj_variants_oracle.c orc_knn, reading R20):
    for each query, the k points of `points` with the smallest (s, id), s the predicate's distance.

    Self kNN (queries=None): query i is points[i] for i in qids (default all) and excludes itself.
    Two-set (queries given): rows of `queries`, nothing excluded.
    Returns (ids int64 [nq, k] (-1 = fewer than k points), s float64 [nq, k] (+inf there))."""
    P = _pts(points)
    n, d = P.shape
    if queries is None:
        q = np.arange(n, dtype=np.int64) if qids is None else np.ascontiguousarray(np.asarray(list(qids) if not isinstance(qids, np.ndarray) else qids, dtype=np.int64))
        Q = np.ascontiguousarray(P[q])
        qself = q
    else:
        Q = _pts(queries)
        qself = None
    nq = Q.shape[0]
    ids = np.empty((nq, k), dtype=np.int64)
    s = np.empty((nq, k), dtype=np.float64)
    rc = _load().orc_knn(_ptr(Q), nq, _ptr(qself) if qself is not None else None, _ptr(P), n, d, int(k),
                         nthreads or default_threads(), _ptr(ids), _ptr(s))
    if rc != 0:
        raise ValueError("bad arguments")
    return ids, s


def brute_force_f32(points, eps: float, include_self: bool = True) -> np.ndarray:
    """The self-join in binary32 (sj_variants_oracle.c orc_brute_force_f32; PAPER.md:393 SuperEGO's
    32-bit floats, R21): points and eps as float32, s32 <= fl32(eps*eps), pairs sorted."""
    P = np.ascontiguousarray(points, dtype=np.float32)
    if P.ndim != 2:
        raise ValueError("points must be N x d")
    n, d = P.shape
    e = float(np.float32(eps))
    lib = _load()
    total = lib.orc_brute_force_f32(_ptr(P), n, d, e, int(include_self), None, 0)
    if total < 0:
        raise ValueError("bad arguments")
    out = np.empty(total, dtype=np.uint64)
    lib.orc_brute_force_f32(_ptr(P), n, d, e, int(include_self), _ptr(out), total)
    return out


def join_sets_digest(queries, points, eps: float, nthreads: int | None = None, with_counts: bool = False):
    """|J(Q,P)| and the order-independent fingerprints F_a, F_b of the pair multiset (the grid join of
    join_sets, accumulated instead of stored; the mixers of sj_oracle.c): dict(pairs, fa, fb[, counts])."""
    Q = _pts(queries)
    P = _pts(points)
    nq, d = Q.shape
    counts = np.zeros(nq, dtype=np.int64) if with_counts else None
    fp = np.zeros(2, dtype=np.uint64)
    total = _load().orc_join_sets_digest(_ptr(Q), nq, _ptr(P), P.shape[0], d, float(eps), nthreads or default_threads(),
                                         _ptr(counts) if counts is not None else None, _ptr(fp))
    if total < 0:
        raise ValueError("bad arguments")
    out = dict(pairs=int(total), fa=int(fp[0]), fb=int(fp[1]))
    if with_counts:
        out["counts"] = counts
    return out
