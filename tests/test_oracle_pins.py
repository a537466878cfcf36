"""Pins of the oracle to things other than itself (task rule ③).

Every test here is CPU-only.  Each names the passage or closed form it checks.
"""
import itertools
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import datagen
import oracle
from oracle import index_ref as ir

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def as_pairs(lst):
    return np.array(sorted((i << 32) | k for i, k in lst), dtype=np.uint64)


# ---------------------------------------------------------------- worked examples (SPEC)
def test_tie_included_and_excluded():
    """S.235-236: (0,0),(3,4): eps=5 -> 4 pairs (tie dist == eps included, PAPER.md:130 '<=');
    eps=4.9 -> only the 2 self pairs."""
    P = np.array([[0.0, 0.0], [3.0, 4.0]])
    assert np.array_equal(oracle.brute_force(P, 5.0), as_pairs([(0, 0), (0, 1), (1, 0), (1, 1)]))
    assert np.array_equal(oracle.brute_force(P, 4.9), as_pairs([(0, 0), (1, 1)]))
    assert np.array_equal(oracle.grid_join(P, 5.0), as_pairs([(0, 0), (0, 1), (1, 0), (1, 1)]))
    assert np.array_equal(oracle.grid_join(P, 4.9), as_pairs([(0, 0), (1, 1)]))


def test_collinear_chain():
    """S.316: points 0,1,2 on a line, eps=1 -> {(0,0),(0,1),(1,0),(1,1),(1,2),(2,1),(2,2)}."""
    P = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    want = as_pairs([(0, 0), (0, 1), (1, 0), (1, 1), (1, 2), (2, 1), (2, 2)])
    assert np.array_equal(oracle.brute_force(P, 1.0), want)
    assert np.array_equal(oracle.grid_join(P, 1.0), want)


@pytest.mark.parametrize("m", [1, 2, 7, 33])
@pytest.mark.parametrize("d", [2, 6])
def test_coincident_points_give_m_squared(m, d):
    """S.272-273 (1 point -> 1 pair, 2 coincident -> 4) and P7: m coincident points -> m^2."""
    P = datagen.duplicates(m, d)
    assert len(oracle.brute_force(P, 0.5)) == m * m
    assert len(oracle.grid_join(P, 0.5)) == m * m
    assert len(oracle.grid_join(P, 0.5, include_self=False)) == m * m - m


def test_eps_below_min_separation_gives_self_pairs_only():
    """S.317: eps smaller than the minimum inter-point distance -> only self pairs."""
    P = datagen.lattice(5, 3, spacing=1.0)
    got = oracle.brute_force(P, 0.999)
    assert np.array_equal(got, as_pairs([(i, i) for i in range(len(P))]))


# ---------------------------------------------------------------- closed forms (P2, P3)
@pytest.mark.parametrize("d,L", [(2, 6), (3, 5), (4, 4)])
def test_lattice_eps1_closed_form_bruteforce(d, L):
    """P2: unit lattice {0..L-1}^d, eps=1: interior point has 1+2d neighbours (self incl.),
    total = L^d + 2d(L-1)L^(d-1) (each of the d axes has (L-1)L^(d-1) adjacent pairs, x2)."""
    P = datagen.lattice(L, d)
    S = oracle.brute_force(P, 1.0)
    assert len(S) == L ** d + 2 * d * (L - 1) * L ** (d - 1)
    cnt = oracle.pair_counts(S, len(P))
    interior = np.all((P > 0) & (P < L - 1), axis=1)
    assert np.all(cnt[interior] == 1 + 2 * d)


@pytest.mark.parametrize("d,L", [(2, 9), (3, 6), (4, 5), (5, 4), (6, 4)])
def test_lattice_eps1_closed_form_grid(d, L):
    P = datagen.lattice(L, d)
    S = oracle.grid_join(P, 1.0)
    assert len(S) == L ** d + 2 * d * (L - 1) * L ** (d - 1)


@pytest.mark.parametrize("d", [2, 3, 4])
def test_lattice_sqrt2_uses_squared_eps(d):
    """P3: eps = fl(sqrt 2): fl(eps*eps) = 2.0000000000000004 > 2, so the face diagonals
    (squared distance exactly 2) are accepted: interior count 1 + 2d + 4*C(d,2) = 1 + 2d^2.
    One ulp below fl(sqrt 2) the square rounds below 2 and the count falls back to 1 + 2d."""
    eps = math.sqrt(2.0)
    assert eps * eps > 2.0
    L = 5
    P = datagen.lattice(L, d)
    interior = np.all((P > 0) & (P < L - 1), axis=1)
    cnt = oracle.pair_counts(oracle.grid_join(P, eps), len(P))
    assert np.all(cnt[interior] == 1 + 2 * d * d)
    below = np.nextafter(eps, 0.0)
    assert below * below < 2.0
    cnt2 = oracle.pair_counts(oracle.grid_join(P, below), len(P))
    assert np.all(cnt2[interior] == 1 + 2 * d)


# ---------------------------------------------------------------- predicate readings (O1, O5)
def test_squared_form_not_sqrt_form():
    """Reading R1: accept iff s <= fl(eps^2).  Find a point pair whose computed
    s is one ulp above fl(eps^2) although fl(sqrt(s)) <= eps (the sqrt form of PAPER.md:130
    would accept it); the oracle must reject it."""
    rng = np.random.default_rng(7)

    def case(e):
        E = e * e
        T = float(np.nextafter(E, np.inf))
        if math.sqrt(T) > e:
            return None
        x = float(np.nextafter(e, 0.0))
        for _ in range(4):
            x2 = x * x
            if x2 < T:
                y = math.sqrt(T - x2)
                for _ in range(64):
                    s = x2 + y * y
                    if s == T:
                        return (e, x, y)
                    y = float(np.nextafter(y, np.inf if s < T else 0.0))
            x = float(np.nextafter(x, 0.0))
        return None

    found = None
    for e in rng.uniform(0.5, 50.0, 2000):
        found = case(float(e))
        if found:
            break
    assert found, "no knife-edge case found"
    e, x, y = found
    assert math.sqrt(x * x + y * y) <= e          # the sqrt form would accept ...
    assert not oracle.pair_within([0.0, 0.0], [x, y], e)   # ... the squared form rejects
    assert oracle.pair_within([0.0, 0.0], [e, 0.0], e)


def _round(fr: Fraction) -> float:
    return float(fr)  # CPython int/int true division is correctly rounded (RN-even)


def test_no_fma_contraction():
    """Reading R1/O5: each *, + is a separate RN operation.  Find (t0, t1) where the fused
    fl(t0^2 + t1*t1 exactly) decides differently from fl(fl(t0^2)+fl(t1^2)); the oracle
    must follow the unfused order."""
    rng = np.random.default_rng(11)
    found = None
    for _ in range(200000):
        t0, t1 = (float(v) for v in rng.uniform(0.1, 1.0, 2))
        s = (t0 * t0) + (t1 * t1)                      # python floats: RN, no FMA
        fused = _round(Fraction(t0 * t0) + Fraction(t1) * Fraction(t1))
        if fused != s:
            found = (t0, t1, s, fused)
            break
    assert found
    t0, t1, s, fused = found
    # choose eps so that E = fl(eps^2) lies between the two sums
    lo, hi = min(s, fused), max(s, fused)
    eps = math.sqrt(lo)
    while eps * eps < lo:
        eps = np.nextafter(eps, np.inf)
    while eps * eps > lo:
        eps = np.nextafter(eps, 0)
    E = eps * eps
    if not (lo <= E < hi):
        pytest.skip("no representable eps between the two sums")
    want = s <= E
    assert oracle.pair_within([0.0, 0.0], [t0, t1], float(eps)) == want


def test_predicate_symmetric_on_knife_edge():
    """O5: fl(a-b) = -fl(b-a), so s(a,b) = s(b,a) and S is symmetric (P5)."""
    P = datagen.knife_edge(3000, 3, 0.1, seed=5)
    S = oracle.grid_join(P, 0.1)
    assert np.array_equal(S, oracle.transpose_pairs(S))


# ---------------------------------------------------------------- brute force vs grid (P1)
CASES = []
for d in range(2, 7):
    CASES += [("uniform", d, 400, 12.0 + 4 * d), ("clustered", d, 500, 0.6), ("knife", d, 400, 0.1)]


@pytest.mark.parametrize("kind,d,n,eps", CASES)
def test_grid_join_equals_brute_force(kind, d, n, eps):
    seed = 100 * d + n
    if kind == "uniform":
        P = datagen.uniform(n, d, seed)
    elif kind == "clustered":
        P = datagen.clustered_small(n, d, seed)
    else:
        P = datagen.knife_edge(n, d, eps, seed)
    for inc in (True, False):
        bf = oracle.brute_force(P, eps, include_self=inc)
        gj = oracle.grid_join(P, eps, include_self=inc)
        assert np.array_equal(bf, gj)
        assert np.array_equal(bf, oracle.transpose_pairs(bf))                   # P5
        if inc:
            assert np.all(oracle.pair_counts(bf, n) >= 1)                       # (i,i) in S


def test_bruteforce_equals_python_definition_tiny():
    """The C brute force against the definition evaluated with Python floats (RN, no FMA)."""
    P = datagen.knife_edge(60, 3, 0.25, seed=3)
    eps = 0.25
    E = eps * eps
    want = []
    for i in range(len(P)):
        for k in range(len(P)):
            s = 0.0
            for j in range(3):
                t = float(P[i, j]) - float(P[k, j])
                s = s + t * t
            if s <= E:
                want.append((i, k))
    assert np.array_equal(oracle.brute_force(P, eps), as_pairs(want))


def test_rows_and_query_ranges_match_full_join():
    P = datagen.uniform(3000, 4, 99)
    eps = 15.0
    full = oracle.grid_join(P, eps)
    q = np.array([0, 17, 1500, 2999])
    cnt, rows = oracle.rows(P, eps, q)
    keys = full >> np.uint64(32)
    want = np.concatenate([full[keys == np.uint64(i)] for i in q])
    assert np.array_equal(rows, want)
    part = oracle.grid_join(P, eps, q0=1000, q1=2000)
    assert np.array_equal(part, full[(keys >= 1000) & (keys < 2000)])
    c = oracle.grid_join(P, eps, count_only=True)
    assert np.array_equal(c, oracle.pair_counts(full, len(P)))                  # P6


# ---------------------------------------------------------------- fingerprints (full-size parity)
def test_fingerprint_mixers_match_published_values():
    """mix_a is SplitMix64's output function: its first four outputs from state 0 are the
    published e220a8397b1dcdaf, 6e789e6aa1b965f4, 06c45d188009454f, f88bb8a8724c81ec (Steele, Lea
    & Flood 2014 reference implementation); mix_b is MurmurHash3's fmix64 (fmix64(0) = 0,
    fmix64(1) = b456bcfc34c2cb2c) applied to x ^ 0xC2B2AE3D27D4EB4F."""
    gamma = 0x9E3779B97F4A7C15
    want = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F, 0xF88BB8A8724C81EC]
    assert [oracle.mix(0, (i * gamma) % 2**64) for i in range(4)] == want
    assert oracle.mix(1, 0xC2B2AE3D27D4EB4F) == 0
    assert oracle.mix(1, 1 ^ 0xC2B2AE3D27D4EB4F) == 0xB456BCFC34C2CB2C
    import fingerprints
    x = np.random.default_rng(1).integers(0, 2**63, 2000, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    assert [int(v) for v in fingerprints.mix_a(x)] == [oracle.mix(0, int(v)) for v in x]
    assert [int(v) for v in fingerprints.mix_b(x)] == [oracle.mix(1, int(v)) for v in x]


@pytest.mark.parametrize("kind,d,n,eps", [("uniform", 2, 2000, 4.0), ("clustered", 3, 2500, 0.6),
                                          ("knife", 4, 1500, 0.1), ("uniform", 6, 1500, 40.0)])
def test_grid_digest_equals_brute_force_fingerprint(kind, d, n, eps):
    """orc_grid_digest (|S|, F_a, F_b, F_c, per-query counts) equals the fingerprints of the brute
    force's explicit S (P1), for any split of the queries (fingerprints add over query ranges)."""
    P = {"uniform": datagen.uniform, "clustered": datagen.clustered_small}.get(kind, None)
    P = P(n, d, 7 * n + d) if P else datagen.knife_edge(n, d, eps, 7 * n + d)
    bf = oracle.brute_force(P, eps)
    cnt = oracle.pair_counts(bf, n)
    dg = oracle.grid_digest(P, eps, with_counts=True)
    assert dg["pairs"] == len(bf) and np.array_equal(dg["counts"], cnt)
    import fingerprints
    assert (dg["fa"], dg["fb"]) == fingerprints.fingerprint(bf)
    assert dg["fc"] == fingerprints.count_fingerprint(cnt)
    parts = [oracle.grid_digest(P, eps, q0=a, q1=b) for a, b in ((0, n // 3), (n // 3, n - 1), (n - 1, n))]
    M = 2**64
    assert sum(p["pairs"] for p in parts) == dg["pairs"]
    for key in ("fa", "fb", "fc"):
        assert sum(p[key] for p in parts) % M == dg[key]
    # a single dropped, added or altered pair changes both fingerprints
    assert fingerprints.fingerprint(bf[1:]) != fingerprints.fingerprint(bf)
    alt = bf.copy()
    alt[len(alt) // 2] ^= np.uint64(1)
    fa, fb = fingerprints.fingerprint(alt)
    assert fa != dg["fa"] and fb != dg["fb"]


# ---------------------------------------------------------------- expectation (P4)
@pytest.mark.parametrize("d,eps,tol", [(2, 2.5, 0.01), (3, 8.0, 0.02), (4, 20.0, 0.03),
                                       (6, 40.0, 0.04)])
def test_uniform_expectation(d, eps, tol):
    """P4: E|S| = N + N(N-1)F_d(eps/L) for iid uniform points in [0,L]^d (exact for eps<=L)."""
    n = 20000
    P = datagen.uniform(n, d, seed=1234 + d)
    got = int(oracle.grid_join(P, eps, count_only=True).sum())
    exp = oracle.expected_pairs_uniform(n, d, eps)
    assert abs(got - exp) / exp < tol


def test_p4_formula_d1_d2_closed_forms():
    """F_1(r) = 2r - r^2 and F_2(r) = pi r^2 - 8/3 r^3 + r^4/2 (textbook line / square picking)."""
    for r in (0.01, 0.2, 0.7):
        assert math.isclose((oracle.expected_pairs_uniform(2, 1, r, 1.0) - 2) / 2, 2 * r - r * r)
        assert math.isclose((oracle.expected_pairs_uniform(2, 2, r, 1.0) - 2) / 2,
                            math.pi * r * r - 8 / 3 * r ** 3 + r ** 4 / 2)


def test_c1_config_full():
    """C1 (BASELINE.json configs[0]): 10K Syn-2D, eps=2.5: brute force == grid join, and the
    total sits within 1% of the P4 expectation (~2.02e5 pairs)."""
    P = datagen.uniform_config("C1", 2)
    bf = oracle.brute_force(P, 2.5)
    gj = oracle.grid_join(P, 2.5)
    assert np.array_equal(bf, gj)
    exp = oracle.expected_pairs_uniform(10_000, 2, 2.5)
    assert abs(len(bf) - exp) / exp < 0.01


def test_mean_neighbours_decrease_with_dimension():
    """PAPER.md:71 / Fig. 1(a) trend (SPEC criterion 6): fixed N and eps=1, mean neighbours per
    point strictly decreases from 2-D to 6-D."""
    n = 100_000
    means = []
    for d in range(2, 7):
        P = datagen.uniform(n, d, seed=77 + d)
        means.append(oracle.grid_join(P, 1.0, count_only=True).mean())
    assert all(a > b for a, b in zip(means, means[1:]))
    assert abs(means[0] - (1 + (n - 1) * math.pi / 1e4)) / means[0] < 0.1  # S.402 density check


# ---------------------------------------------------------------- index (§4.2-4.4)
def load_fig2():
    P = np.loadtxt(os.path.join(GOLDEN, "fig2_points.txt"))
    return P


def test_fig2_index_facts():
    """PAPER.md:179, 201-202 (Fig. 2 worked example) under readings R6-R9."""
    P = load_fig2()
    idx = ir.build_index(P, 1.0)
    assert len(idx.B) == 11 and len(idx.G) - 1 == 11                       # |B| = |G| = 11
    assert idx.geom.cpd[0] == 7                                              # id = c1 + 7*c2
    assert idx.B[6] == 30                                                    # C_7 -> linear id 30
    assert idx.B[5] == 22                                                    # C_6 -> linear id 22
    a = 20
    c = idx.coords[a]
    assert ir.linearize(idx.geom, c) == 30
    O = ir.adjacent_ranges(idx, c)
    assert O == [(1, 3), (3, 5)]                                             # O_1, O_2
    masked = ir.mask_ranges(idx, O)
    assert masked == [[1, 2], [3, 4, 5]]                                     # O_j ∩ M_j
    probed, hits = ir.alg1_probes(idx, c)
    assert sorted(probed) == [22, 23, 29, 30, 36, 37]
    assert sorted(hits) == [22, 30, 36]
    h = ir.lookup(idx, 22)
    assert set(idx.A[idx.G[h]:idx.G[h + 1]].tolist()) == {35, 6}             # {p36, p7}


def _check_invariants(P, eps):
    idx = ir.build_index(P, eps)
    n = len(P)
    nG = len(idx.B)
    assert nG == len(idx.G) - 1 <= n                                         # |B|=|G|<=|D|
    assert sorted(idx.A.tolist()) == list(range(n))                          # A permutation
    assert all(a < b for a, b in zip(idx.B, idx.B[1:]))                      # B strictly sorted
    assert idx.G[0] == 0 and idx.G[-1] == n and np.all(np.diff(idx.G) >= 1)  # non-empty cells
    for h in range(nG):
        for i in idx.A[idx.G[h]:idx.G[h + 1]]:
            assert idx.keys[i] == idx.B[h]                                   # re-linearises
    for j in range(idx.geom.d):
        assert idx.M[j] == sorted(set(idx.coords[:, j].tolist()))
        assert idx.coords[:, j].min() >= 1 and idx.coords[:, j].max() <= idx.geom.cpd[j] - 2  # R7
    return idx


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
def test_index_invariants(d):
    """SPEC S.117-125, S.184-187, S.405 (criterion 8)."""
    _check_invariants(datagen.uniform(800, d, seed=d), 9.0)
    _check_invariants(datagen.clustered_small(800, d, seed=d), 0.4)
    _check_invariants(datagen.knife_edge(500, d, 0.1, seed=d), 0.1)


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
def test_index_is_a_complete_filter(d):
    """Reading R6: with w = eps + 2^-44(eps+R), every accepted pair (brute force) lies in cells
    whose coordinates differ by at most 1 in every dimension, on knife-edge inputs."""
    for eps in (0.1, 0.3, 1.0 / 3.0):
        P = datagen.knife_edge(1500, d, eps, seed=d + 31)
        idx = ir.build_index(P, eps)
        S = oracle.brute_force(P, eps)
        i = (S >> np.uint64(32)).astype(np.int64)
        k = (S & np.uint64(0xFFFFFFFF)).astype(np.int64)
        assert np.abs(idx.coords[i] - idx.coords[k]).max() <= 1


def test_cell_side_exactly_eps_is_not_complete():
    """Why R6 exists: with cell side exactly eps (origin
    at the minimum) an accepted knife-edge pair can land two cells apart."""
    rng = np.random.default_rng(1)
    found = None
    for _ in range(20000):
        eps = float(rng.uniform(0.05, 2.0))
        k = int(rng.integers(1, 200))
        o = float(rng.uniform(0.1, 50))
        x = o + k * eps
        for _ in range(16):                       # largest x still in cell k-1
            if math.floor((x - o) / eps) < k:
                break
            x = float(np.nextafter(x, 0))
        y = x + eps
        for _ in range(6):
            if math.floor((x - o) / eps) < k and math.floor((y - o) / eps) >= k + 1:
                P = np.array([[o, 0.0], [x, 0.0], [y, 0.0]])
                if len(oracle.brute_force(P, eps)) == 5:     # (x,y) accepted both ways
                    found = (P, eps)
                    break
            y = float(np.nextafter(y, np.inf))
        if found:
            break
    assert found
    P, eps = found
    c_exact = np.floor((P - P.min(axis=0)) / eps).astype(np.int64)
    assert abs(c_exact[2, 0] - c_exact[1, 0]) == 2               # side eps: two cells apart
    idx = ir.build_index(P, eps)
    assert abs(idx.coords[2, 0] - idx.coords[1, 0]) <= 1          # R6 width: adjacent


# ---------------------------------------------------------------- unicomp (Alg. 2, R12/R13)
def test_unicomp_spec_examples():
    """SPEC S.245-247: 2-D (2,4) -> nothing; 2-D (1,3) -> all 8 neighbours; 3-D (1,2,2) -> 2."""
    assert ir.unicomp_cells((2, 4), [[1, 2, 3], [3, 4, 5]]) == []
    got = ir.unicomp_cells((1, 3), [[0, 1, 2], [2, 3, 4]])
    assert sorted(got) == sorted([(0, 3), (2, 3), (0, 2), (1, 2), (2, 2), (0, 4), (1, 4), (2, 4)])
    assert ir.unicomp_cells((1, 2, 2), [[0, 1, 2], [1, 2, 3], [1, 2, 3]]) == [(0, 2, 2), (2, 2, 2)]


@pytest.mark.parametrize("d", [2, 3, 4, 5])
def test_unicomp_covers_each_adjacent_pair_once(d):
    """R13: on a 5^d grid, each unordered pair of distinct adjacent cells {a,b} is searched by
    exactly one of them (the one odd in the highest differing dimension), and each cell
    searches 1 + (3^d - 1)/2 cells on average over the parity classes."""
    side = 5 if d <= 4 else 4
    cells = list(itertools.product(range(side), repeat=d))
    cellset = set(cells)
    U = {}
    for c in cells:
        masked = [[v for v in (c[j] - 1, c[j], c[j] + 1) if 0 <= v < side] for j in range(d)]
        lst = ir.unicomp_cells(c, masked)
        assert len(lst) == len(set(lst)) and c not in lst
        U[c] = set(lst)
    for a in cells:
        for off in itertools.product((-1, 0, 1), repeat=d):
            if not any(off):
                continue
            b = tuple(x + o for x, o in zip(a, off))
            if b not in cellset:
                continue
            assert (b in U[a]) + (a in U[b]) == 1
    # parity-class mean on a full 3^d neighbourhood (all values available)
    tot = 0
    for par in itertools.product((0, 1), repeat=d):
        c = tuple(2 + p for p in par)
        masked = [[c[j] - 1, c[j], c[j] + 1] for j in range(d)]
        tot += 1 + len(ir.unicomp_cells(c, masked))
    assert tot / 2 ** d == 1 + (3 ** d - 1) / 2


def test_alg2_as_printed_double_covers():
    """R12: Alg. 2's third block as printed ('C_a.y is odd') does not cover each
    adjacent pair exactly once on a 5^3 grid; the z-parity reading does (test above)."""
    side = 5
    cells = list(itertools.product(range(side), repeat=3))
    U = {}
    for c in cells:
        masked = [[v for v in (c[j] - 1, c[j], c[j] + 1) if 0 <= v < side] for j in range(3)]
        U[c] = set(ir.alg2_as_printed_3d(c, masked))
    bad = 0
    for a in cells:
        for off in itertools.product((-1, 0, 1), repeat=3):
            b = tuple(x + o for x, o in zip(a, off))
            if any(off) and all(0 <= v < side for v in b):
                bad += ((b in U[a]) + (a in U[b])) != 1
    assert bad > 0


def test_generators_deterministic():
    a = datagen.uniform(100, 3, 42)
    b = datagen.uniform(100, 3, 42)
    assert np.array_equal(a, b) and a.min() >= 0 and a.max() < 100
    s = datagen.skewed(20000, 3, seed=5)
    assert s.shape == (20000, 3) and s.min() >= 0 and s.max() <= 100


# ------------------------------------------------------------------ f4: DBSCAN on the join (R17)
def _sk_dbscan(pairs, n, min_pts):
    """scikit-learn's DBSCAN (an independent implementation) on the same eps-neighbourhood graph:
    a sparse precomputed 'distance' matrix whose stored entries are exactly the pairs of S."""
    from scipy.sparse import csr_matrix
    from sklearn.cluster import DBSCAN
    p = (pairs >> np.uint64(32)).astype(np.int64)
    q = (pairs & np.uint64(0xFFFFFFFF)).astype(np.int64)
    G = csr_matrix((np.full(len(p), 0.1), (p, q)), shape=(n, n))
    m = DBSCAN(eps=0.5, min_samples=min_pts, metric="precomputed").fit(G)
    core = np.zeros(n, bool)
    core[m.core_sample_indices_] = True
    return m.labels_, core


@pytest.mark.parametrize("seed,d,n,eps,min_pts", [(1, 2, 1500, 0.35, 4), (2, 2, 2000, 0.5, 8),
                                                  (3, 3, 1200, 0.8, 5), (4, 2, 800, 2.0, 3),
                                                  (5, 4, 1000, 1.2, 6)])
def test_dbscan_oracle_matches_sklearn(seed, d, n, eps, min_pts):
    """oracle.dbscan against scikit-learn on the same neighbourhood table: the core set and the
    noise set exactly, the core partition up to relabelling; every border label is the smallest
    label among the point's core neighbours (reading R17: the unique choice)."""
    from oracle.dbscan import dbscan_from_pairs
    pts = datagen.clustered_small(n, d, seed=seed) if seed % 2 else datagen.uniform(n, d, seed=seed, hi=12.0)
    pairs = oracle.brute_force(pts, eps)
    lab = dbscan_from_pairs(pairs, n, min_pts)
    sk_lab, sk_core = _sk_dbscan(pairs, n, min_pts)
    cnt = np.bincount((pairs >> np.uint64(32)).astype(np.int64), minlength=n)
    core = cnt >= min_pts
    assert np.array_equal(core, sk_core)
    assert np.array_equal(lab == -1, sk_lab == -1)                   # noise: no core neighbour
    # core partition identical up to relabelling (a bijection between label sets on core points)
    pairs_cl = set(zip(lab[core].tolist(), sk_lab[core].tolist()))
    assert len(pairs_cl) == len(set(lab[core].tolist())) == len(set(sk_lab[core].tolist()))
    # labels are the smallest core id of each cluster
    for c in set(lab[core].tolist()):
        assert c == np.flatnonzero(core & (lab == c)).min()
    # border: smallest label among core neighbours
    p = (pairs >> np.uint64(32)).astype(np.int64)
    q = (pairs & np.uint64(0xFFFFFFFF)).astype(np.int64)
    for i in np.flatnonzero(~core & (lab != -1)):
        nb = q[(p == i)]
        assert lab[i] == min(lab[j] for j in nb if core[j])
    assert np.any(core) and len(set(lab[core].tolist())) >= 1


def test_dbscan_oracle_fixture():
    """Hand-built, on a line (y = 0), eps = 1 (ties included), min_pts = 4: two clusters of five
    points 0.25 apart, a bridge point at x = 2 seeing 1.0, 2.0 and 3.0 only (3 < 4: not core, but a
    border of BOTH clusters -> the smaller label, reading R17), and an isolated point (noise).
    Neighbourhood sizes by hand: [5,5,5,5,6, 3, 6,5,5,5,5, 1]."""
    from oracle.dbscan import dbscan_from_pairs
    xs = [0.0, 0.25, 0.5, 0.75, 1.0, 2.0, 3.0, 3.25, 3.5, 3.75, 4.0, 10.0]
    pts = np.array([[x, 0.0] for x in xs])
    pairs = oracle.brute_force(pts, 1.0)
    cnt = np.bincount((pairs >> np.uint64(32)).astype(np.int64), minlength=len(pts))
    assert list(cnt) == [5, 5, 5, 5, 6, 3, 6, 5, 5, 5, 5, 1]
    lab = dbscan_from_pairs(pairs, len(pts), 4)
    assert list(lab) == [0, 0, 0, 0, 0, 0, 6, 6, 6, 6, 6, -1]
    # min_pts = 6: only 1.0 and 3.0 are core, each its own cluster; the rest are their borders
    # (the bridge takes the smaller label) or noise
    lab6 = dbscan_from_pairs(pairs, len(pts), 6)
    assert list(lab6) == [4, 4, 4, 4, 4, 4, 6, 6, 6, 6, 6, -1]
