"""TEST INFRASTRUCTURE ONLY -- plain numpy/Python statement of the paper's grid index.

Follows PAPER.md §4.2-4.4 (lines 155-183) and Alg. 1-2 (lines 216-251, 293-341) step by step,
with the DESIGN.md readings where the paper is silent or garbled:

  R6  cell width  w = eps + 2^-44 (eps + R),  R = max_j (max_j - min_j)      (PAPER.md:168 assumes
      "eps evenly divides the range"; a width of exactly eps drops FP knife-edge pairs)
  R7  c_j = 1 + floor(fl(fl(x_j - min_j) / w)),  |g_j| = cpd_j = 3 + floor(fl(fl(max_j-min_j)/w))
      (PAPER.md:156 pads the range by one cell on each side "to avoid boundary conditions")
  R8  linear id with dimension 1 fastest: id = sum_j c_j * stride_j, stride_1 = 1,
      stride_{j+1} = stride_j * cpd_j  (reproduces Fig. 2's ids 22,23,29,30,36,37)
  R9  M_j = set of occupied coordinates in dimension j
  R12/R13 unicomp in n-D: for every dimension j with c_j odd, the cells whose dims < j range over
      the (masked) adjacent values, dim j differs from c_j, dims > j equal c (PAPER.md:285-289,
      Alg. 2 with its third block's "C_a.y is odd" read as "C_a.z is odd")
  R14 A lists point ids in ascending (linear id, point id) order (stable sort).

Nothing here is imported by, or imports, the CUDA path.  Python ints are used for linear ids so
no overflow can hide a mistake; numpy float64 arithmetic is IEEE round-to-nearest with no FMA.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Geometry:
    d: int
    eps: float
    mins: np.ndarray      # [d] exact per-dimension minima
    maxs: np.ndarray      # [d] exact per-dimension maxima
    R: float              # max_j fl(max_j - min_j)
    w: float              # cell width (R6)
    cpd: list             # cells per dimension |g_j| (R7), python ints
    strides: list         # python ints (R8)

    @property
    def n_cells(self) -> int:
        p = 1
        for c in self.cpd:
            p *= c
        return p


def geometry(points: np.ndarray, eps: float) -> Geometry:
    """§4.2 "Index Properties" with readings R6-R8."""
    P = np.asarray(points, dtype=np.float64)
    d = P.shape[1]
    mins = P.min(axis=0)
    maxs = P.max(axis=0)
    ranges = maxs - mins                         # fl(max_j - min_j)
    R = float(ranges.max())
    w = float(np.float64(eps) + np.ldexp(np.float64(eps) + np.float64(R), -44))
    cpd = [3 + int(np.floor(np.float64(ranges[j]) / np.float64(w))) for j in range(d)]
    strides = [1]
    for j in range(d - 1):
        strides.append(strides[-1] * cpd[j])
    g = Geometry(d, float(eps), mins, maxs, R, w, cpd, strides)
    if g.n_cells >= 2 ** 64:
        raise OverflowError("prod(cpd) >= 2^64: use a larger eps")
    return g


def cell_coords(g: Geometry, points: np.ndarray) -> np.ndarray:
    """c_j = 1 + floor(fl(fl(x_j - min_j)/w)) (R7); returns int64 [N, d]."""
    P = np.asarray(points, dtype=np.float64)
    t = np.floor((P - g.mins[None, :]) / np.float64(g.w))
    return (1 + t).astype(np.int64)


def linearize(g: Geometry, c) -> int:
    """getLinearCoord (Alg. 1 line 10), dimension 1 fastest (R8)."""
    return int(sum(int(c[j]) * g.strides[j] for j in range(g.d)))


@dataclass
class Index:
    geom: Geometry
    B: list               # sorted linear ids of non-empty cells, |B| = |G|
    G: np.ndarray         # int64 [|G|+1]: cell h holds A[G[h] : G[h+1]]      (A_h^min..A_h^max)
    A: np.ndarray         # int64 [N]: point ids grouped by cell               (|A| = |D|)
    M: list               # M[j] = sorted occupied coordinates in dimension j  (R9)
    coords: np.ndarray = field(repr=False, default=None)   # [N, d] per input point
    keys: list = field(repr=False, default=None)           # linear id per input point


def build_index(points: np.ndarray, eps: float) -> Index:
    """§4.3 "Index Components": B, G, A, M over non-empty cells only."""
    g = geometry(points, eps)
    c = cell_coords(g, points)
    keys = [linearize(g, row) for row in c]
    n = len(keys)
    # stable sort by linear id: ties keep input order (R14)
    A = sorted(range(n), key=lambda i: (keys[i], i))
    B, starts = [], []
    for pos, i in enumerate(A):
        if not B or keys[i] != B[-1]:
            B.append(keys[i])
            starts.append(pos)
    starts.append(n)
    M = [sorted(set(int(v) for v in c[:, j])) for j in range(g.d)]
    return Index(g, B, np.asarray(starts, dtype=np.int64), np.asarray(A, dtype=np.int64), M, c, keys)


def lookup(idx: Index, lid: int):
    """Binary search of B (Alg. 1 line 11): cell position h or None."""
    lo, hi = 0, len(idx.B)
    while lo < hi:
        mid = (lo + hi) // 2
        if idx.B[mid] < lid:
            lo = mid + 1
        else:
            hi = mid
    return lo if lo < len(idx.B) and idx.B[lo] == lid else None


def adjacent_ranges(idx: Index, c) -> list:
    """getAdjCells (Alg. 1 line 5): O_j = [c_j - 1, c_j + 1] within [0, |g_j|-1]."""
    return [(max(0, int(c[j]) - 1), min(idx.geom.cpd[j] - 1, int(c[j]) + 1)) for j in range(idx.geom.d)]


def mask_ranges(idx: Index, O) -> list:
    """maskCellRange (Alg. 1 line 6): O_j ∩ M_j as sorted lists."""
    return [[v for v in range(lo, hi + 1) if v in set(idx.M[j])] for j, (lo, hi) in enumerate(O)]


def alg1_probes(idx: Index, c):
    """Alg. 1 lines 5-11 for one query cell: (probed linear ids, those present in B)."""
    masked = mask_ranges(idx, adjacent_ranges(idx, c))
    probed = [linearize(idx.geom, t) for t in itertools.product(*masked)]
    hits = [lid for lid in probed if lookup(idx, lid) is not None]
    return probed, hits


def unicomp_cells(c, masked) -> list:
    """Alg. 2 generalised to n dimensions (reading R12/R13; SPEC S.242).

    For each dimension j (0-based here) with c[j] odd: every tuple with dims < j from the
    masked lists, dim j from masked[j] minus c[j], dims > j equal to c.  The home cell is never
    emitted.
    """
    n = len(c)
    out = []
    for j in range(n):
        if int(c[j]) % 2 == 0:
            continue
        lower = [masked[i] for i in range(j)]
        mids = [v for v in masked[j] if v != int(c[j])]
        for pre in itertools.product(*lower):
            for v in mids:
                out.append(tuple(pre) + (v,) + tuple(int(x) for x in c[j + 1:]))
    return out


def alg2_as_printed_3d(c, masked) -> list:
    """Alg. 2 exactly as printed: the third block tests 'C_a.y is odd'.

    Kept only to pin reading R12: this version does NOT cover each adjacent cell pair once.
    """
    out = []
    x, y, z = (int(v) for v in c)
    if x % 2 == 1:
        out += [(v, y, z) for v in masked[0] if v != x]
    if y % 2 == 1:
        out += [(a, b, z) for a in masked[0] for b in masked[1] if b != y]
    if y % 2 == 1:   # sic
        out += [(a, b, cz) for a in masked[0] for b in masked[1] for cz in masked[2] if cz != z]
    return out
