"""Seeded synthetic input generators for the epsilon self-join (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no grid, no distance, no predicate): it only
draws point sets.  Both the oracle (``oracle/``) and the CUDA path consume the same arrays,
which is the only thing the two sides share (task rule ③).

Recipes:
  * uniform  -- PAPER.md:357-358 (§6.1): "64-bit floating point value uniformly distributed in
    the range [0,100] in each dimension"; ``numpy.random.default_rng(seed).uniform(0,100,(N,d))``.
  * skewed   -- synthetic stand-in for the paper's SW-/SDSS- real datasets (PAPER.md:359-380,
    Table 1), galaxy-like clustered 2-D cloud (+ smooth 3rd coordinate for the 3-D variant);
    exact numpy call order from SURVEY.md §8(d) "C4 skewed stand-in".
  * lattice / knife-edge / duplicates -- structured inputs whose join has a closed form or sits
    on the predicate's tie.
"""
from __future__ import annotations

import numpy as np

# seed = 1803_04120 + 100*d + config#
BASE_SEED = 1803_04120

# BASELINE.json configs (index = config#; 0-based like BASELINE.json "configs")
CONFIGS = {
    # C1: Syn-2D 10,000 uniform points, eps for ~20 neighbours/point (incl. self)
    "C1": dict(kind="uniform", n=10_000, dims=(2,), eps=(2.5,)),
    # C2: Syn-2D..6D 2M uniform, eps=1 (Fig. 1(a) set-up)
    "C2": dict(kind="uniform", n=2_000_000, dims=(2, 3, 4, 5, 6), eps=(1.0,)),
    # C3: Syn-6D 2M eps sweep, result sets larger than one buffer at the top end
    "C3": dict(kind="uniform", n=2_000_000, dims=(6,), eps=(1.0, 2.0, 4.0, 8.0, 12.0, 16.0, 20.0, 24.0)),
    # C4: skewed 2-D/3-D, 15,228,633 points (SDSS2DB size)
    "C4": dict(kind="skewed", n=15_228_633, dims=(2, 3),
               eps={2: (0.002, 0.005, 0.01, 0.02), 3: (0.05, 0.1, 0.2)}),
    # C5: Syn-4D / Syn-6D 16M uniform (scaling run)
    "C5": dict(kind="uniform", n=16_000_000, dims=(4, 6), eps={4: (2.0,), 6: (8.0,)}),
}
CONFIG_NUMBER = {"C1": 0, "C2": 1, "C3": 2, "C4": 3, "C5": 4}


def seed_for(d: int, config: str) -> int:
    return BASE_SEED + 100 * d + CONFIG_NUMBER[config]


def uniform(n: int, d: int, seed: int, lo: float = 0.0, hi: float = 100.0) -> np.ndarray:
    """N x d float64, iid uniform in [lo, hi) per coordinate."""
    r = np.random.default_rng(seed)
    return np.ascontiguousarray(r.uniform(lo, hi, (n, d)), dtype=np.float64)


def uniform_config(config: str, d: int, n: int | None = None) -> np.ndarray:
    """The BASELINE.json config's uniform array (optionally truncated to its first n rows)."""
    spec = CONFIGS[config]
    full_n = spec["n"]
    pts = uniform(full_n if n is None else n, d, seed_for(d, config))
    return pts


def skewed(n: int, d: int, seed: int = 1803041200, n_clusters: int = 25_000) -> np.ndarray:
    """Clustered 'galaxy-like' cloud in [0,100]^d, d in {2,3} (SURVEY.md §8(d) C4 recipe).

    Call order is fixed so the statistics quoted in SURVEY.md Appendix A reproduce:
    centres, pareto weights, background count, multinomial counts, log-normal widths,
    gaussian members, uniform background, clip, optional smooth z, shuffle.
    """
    if d not in (2, 3):
        raise ValueError("skewed generator supports d in {2,3}")
    r = np.random.default_rng(seed)
    K = n_clusters
    centres = r.uniform(0, 100, (K, 2))
    w = r.pareto(1.5, K) + 1.0
    w /= w.sum()
    n_bg = int(0.15 * n)
    counts = r.multinomial(n - n_bg, w)
    sigma = 0.05 * np.exp(r.normal(0, 0.5, K))
    idx = np.repeat(np.arange(K), counts)
    members = centres[idx] + r.normal(size=(n - n_bg, 2)) * sigma[idx][:, None]
    pts = np.concatenate([members, r.uniform(0, 100, (n_bg, 2))], axis=0)
    pts = np.clip(pts, 0.0, 100.0)
    if d == 3:
        x, y = pts[:, 0], pts[:, 1]
        z = 50.0 + 30.0 * np.sin(x / 15.0) * np.cos(y / 20.0) + r.normal(0, 3, n)
        pts = np.concatenate([pts, np.clip(z, 0.0, 100.0)[:, None]], axis=1)
    r.shuffle(pts)
    return np.ascontiguousarray(pts, dtype=np.float64)


def lattice(L: int, d: int, spacing: float = 1.0, origin: float = 0.0) -> np.ndarray:
    """All points of {origin + i*spacing : i = 0..L-1}^d (row-major, last coordinate fastest)."""
    axes = [origin + spacing * np.arange(L, dtype=np.float64)] * d
    grid = np.meshgrid(*axes, indexing="ij")
    return np.ascontiguousarray(np.stack([g.ravel() for g in grid], axis=1), dtype=np.float64)


def knife_edge(n: int, d: int, eps: float, seed: int, span_cells: int = 12) -> np.ndarray:
    """Points on an eps-spaced lattice with random +-0..2 ulp perturbations.

    Many pairs sit exactly at, or one rounding step around, distance eps and exactly on
    cell boundaries -- the inputs where a grid with cell side exactly eps drops pairs
    (SURVEY.md §8(c) O7, Appendix B.1).
    """
    r = np.random.default_rng(seed)
    i = r.integers(0, span_cells, size=(n, d)).astype(np.float64)
    pts = i * eps  # fl(i*eps): the lattice as the FP unit sees it
    steps = r.integers(-2, 3, size=(n, d))
    for s in (-2, -1, 1, 2):
        m = steps == s
        direction = np.inf if s > 0 else -np.inf
        v = pts[m]
        for _ in range(abs(s)):
            v = np.nextafter(v, direction)
        pts[m] = v
    return np.ascontiguousarray(pts, dtype=np.float64)


def duplicates(m: int, d: int, value: float = 3.25) -> np.ndarray:
    """m coincident points (join = all m^2 ordered pairs)."""
    return np.full((m, d), value, dtype=np.float64)


def clustered_small(n: int, d: int, seed: int, n_clusters: int = 8, sigma: float = 0.5,
                    box: float = 20.0) -> np.ndarray:
    """Small, dense, duplicate-prone clustered cloud for parity tests of skewed cells."""
    r = np.random.default_rng(seed)
    centres = r.uniform(0, box, (n_clusters, d))
    lab = r.integers(0, n_clusters, n)
    pts = centres[lab] + r.normal(0, sigma, (n, d))
    # quantise a fraction of the coordinates to create exact duplicates and ties
    q = r.random((n, d)) < 0.3
    pts[q] = np.round(pts[q] * 4.0) / 4.0
    return np.ascontiguousarray(pts, dtype=np.float64)
