"""TEST INFRASTRUCTURE ONLY -- DBSCAN clustering read off an epsilon self-join result (SURVEY.md
§8(f) rank 4, "DBSCAN-style epsilon-neighbourhood table"; "the DBSCAN clustering
algorithm requires range queries that search the neighborhood of all data points to find those
within a given distance", citing Ester et al. 1996).

The self-join S (ordered pairs, self pairs included) IS the table of
epsilon-neighbourhoods N_eps(p) = {q : (p, q) in S}.  DBSCAN's definitions on it (Ester 1996):

* p is a CORE point iff |N_eps(p)| >= min_pts (p counts itself: (p, p) is in S);
* core points p, q with (p, q) in S are directly density-reachable from each other; the clusters
  are the connected components of the core points under that relation;
* a non-core point with at least one core neighbour is a BORDER point of that neighbour's cluster;
  a point with no core neighbour is NOISE.

Where the 1996 definition leaves a choice (reading R17): a border point adjacent to
several clusters joins the one with the smallest label (the original algorithm assigns it to the
first cluster that reaches it -- visit order), and a cluster's label is the smallest point id
among its core points, so the labelling is unique.  Noise is -1.

Plain Python: a dictionary-free union-find over the core-core pairs, in pair order, then the
border rule.  Parity pins: tests/test_oracle_pins.py (scikit-learn's DBSCAN on the same
neighbourhood graph -- core set and noise set exactly, core partition up to relabelling -- and a
hand-built fixture with known clusters).
"""
from __future__ import annotations

import numpy as np


def dbscan_from_pairs(pairs: np.ndarray, n: int, min_pts: int) -> np.ndarray:
    """Labels (int64[n]) of DBSCAN(eps, min_pts) given the eps self-join's packed pairs
    (uint64 (p << 32) | q, both orientations, self pairs included)."""
    pairs = np.asarray(pairs, dtype=np.uint64)
    p = (pairs >> np.uint64(32)).astype(np.int64)
    q = (pairs & np.uint64(0xFFFFFFFF)).astype(np.int64)
    # |N_eps(p)|: the number of pairs keyed by p (self pair included)
    count = np.bincount(p, minlength=n)
    core = count >= min_pts
    parent = list(range(n))

    def find(x: int) -> int:
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    # clusters: connected components of core points under (p, q) in S
    for a, b in zip(p.tolist(), q.tolist()):
        if a < b and core[a] and core[b]:
            ra, rb = find(a), find(b)
            if ra != rb:
                if ra < rb:
                    parent[rb] = ra          # the smaller id stays the root: root = min core id
                else:
                    parent[ra] = rb
    labels = np.full(n, -1, dtype=np.int64)
    for i in range(n):
        if core[i]:
            labels[i] = find(i)
    # border points: the smallest label among their core neighbours (reading R17); else noise
    for a, b in zip(p.tolist(), q.tolist()):
        if not core[a] and core[b]:
            lb = labels[b]
            if labels[a] < 0 or lb < labels[a]:
                labels[a] = lb
    return labels
