"""Pins of the variant oracles (sj_variants_oracle.c: two-set join, kNN) to
things other than themselves (task rule ③): scipy's KD-tree (an independent library route), lattice
closed forms with exact binary-fraction distances, tie rules worked by hand, the already-pinned
self-join oracle as the Q = P special case, and transposition symmetry.  CPU only.
"""
import itertools

import numpy as np
import pytest

import datagen
import oracle

scipy_spatial = pytest.importorskip("scipy.spatial")


def _lin(c, L):
    """Row-major id of lattice point c in datagen.lattice(L, d) (last coordinate fastest)."""
    i = 0
    for x in c:
        i = i * L + int(x)
    return i


# ---------------------------------------------------------------- two-set join
@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("method", ["brute", "grid"])
def test_join_sets_equals_kdtree_ball_query(d, method):
    """J(Q,P) on continuous random data (no knife edges) == scipy cKDTree.query_ball_point with r=eps
    (an independent implementation of the same ball predicate)."""
    rng = np.random.default_rng(100 + d)
    P = rng.uniform(0.0, 10.0, (700, d))
    Q = rng.uniform(-2.0, 12.0, (500, d))           # queries reach outside P's bounding box
    eps = [1.2, 2.0, 3.0, 3.8, 4.5][d - 2]
    got = oracle.join_sets(Q, P, eps, method=method)
    tree = scipy_spatial.cKDTree(P)
    want = []
    for i, row in enumerate(tree.query_ball_point(Q, eps)):
        want.extend((i << 32) | k for k in row)
    want = np.array(sorted(want), dtype=np.uint64)
    assert len(want) > 100
    assert np.array_equal(got, want)


@pytest.mark.parametrize("d,L", [(2, 7), (3, 5), (4, 4), (6, 3)])
def test_join_sets_shifted_lattice_closed_form(d, L):
    """P = {0..L-1}^d, Q = P + (1/4) e_0, eps = 1: (v_0 - 1/4)^2 + sum_{j>0} v_j^2 <= 1 holds exactly
    (binary fractions) for the lattice displacements v = 0 and v = e_0 only, so
    |J| = L^d + (L-1) L^(d-1) and every pair is (i, i) or (i, i + e_0)."""
    P = datagen.lattice(L, d)
    Q = P.copy()
    Q[:, 0] += 0.25
    for method in ("brute", "grid"):
        got = oracle.join_sets(Q, P, 1.0, method=method)
        assert len(got) == L ** d + (L - 1) * L ** (d - 1)
        want = []
        for c in itertools.product(range(L), repeat=d):
            i = _lin(c, L)
            want.append((i << 32) | i)
            if c[0] + 1 < L:
                want.append((i << 32) | _lin((c[0] + 1,) + c[1:], L))
        assert np.array_equal(got, np.array(sorted(want), dtype=np.uint64))


@pytest.mark.parametrize("d", [2, 4, 6])
def test_join_sets_of_a_set_with_itself_is_the_self_join(d):
    """J(P,P) == S(P) with self pairs (the pinned self-join oracle; the self-join is the
    similarity join of a set with itself)."""
    P = datagen.clustered_small(600, d, seed=5 + d)
    eps = [0.6, 1.2, 2.0][d // 2 - 1]
    want = oracle.brute_force(P, eps, include_self=True)
    assert len(want) > 600
    assert np.array_equal(oracle.join_sets(P, P, eps, method="brute"), want)
    assert np.array_equal(oracle.join_sets(P, P, eps), want)


def test_join_sets_transpose_and_degenerate():
    """J(Q,P) = transpose(J(P,Q)) (the predicate is symmetric); empty Q / far-away Q give no pairs;
    the knife-edge tie s == fl(eps^2) is included as in the self-join (S.235: (0,0),(3,4), eps=5)."""
    rng = np.random.default_rng(7)
    P = rng.uniform(0, 5, (300, 3))
    Q = rng.uniform(0, 5, (200, 3))
    a = oracle.join_sets(Q, P, 0.9)
    assert np.array_equal(a, oracle.transpose_pairs(oracle.join_sets(P, Q, 0.9)))
    assert len(oracle.join_sets(np.empty((0, 3)), P, 0.9)) == 0
    assert len(oracle.join_sets(P + 1e6, P, 0.9)) == 0
    A = np.array([[0.0, 0.0]])
    B = np.array([[3.0, 4.0], [3.0, 4.0000001]])
    for m in ("brute", "grid"):
        assert oracle.join_sets(A, B, 5.0, method=m).tolist() == [0]   # (0,0) only: B[1] is just outside
        assert oracle.join_sets(A, B, 4.9, method=m).tolist() == []


# ---------------------------------------------------------------- kNN
@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("k", [1, 7, 32])
def test_knn_equals_kdtree(d, k):
    """Self kNN on continuous random data (all distances distinct): ids == scipy cKDTree.query(k+1)
    minus the query itself; s == the squared distances up to the library's own rounding."""
    rng = np.random.default_rng(200 + d)
    P = rng.uniform(0.0, 10.0, (900, d))
    ids, s = oracle.knn(P, k)
    dist, nbr = scipy_spatial.cKDTree(P).query(P, k + 1)
    assert np.array_equal(nbr[:, 0], np.arange(len(P)))      # the query itself first (distance 0)
    assert np.array_equal(ids, nbr[:, 1:])
    np.testing.assert_allclose(np.sqrt(s), dist[:, 1:], rtol=1e-12)


def test_knn_lattice_ties_broken_by_id():
    """Interior point c of {0..4}^d: its 2d axis neighbours sit at s = 1 exactly and the 2d(d-1) diagonal neighbours of the next
    shell at s = 2, so the k = 2d nearest are exactly the axis neighbours in ascending id, and the
    (2d+1)-th is the smallest-id point at s = 2 (the tie rule of reading R20)."""
    for d in (2, 3, 4):
        L = 5
        P = datagen.lattice(L, d)
        c = (2,) * d
        i = _lin(c, L)
        axis = sorted(_lin(c[:j] + (c[j] + e,) + c[j + 1:], L) for j in range(d) for e in (-1, 1))
        diag = sorted(_lin(tuple(c[t] + (a if t == j1 else b if t == j2 else 0) for t in range(d)), L)
                      for j1, j2 in itertools.combinations(range(d), 2)
                      for a in (-1, 1) for b in (-1, 1))
        ids, s = oracle.knn(P, 2 * d + 1, qids=[i])
        assert ids[0, :2 * d].tolist() == axis
        assert s[0, :2 * d].tolist() == [1.0] * (2 * d)
        assert ids[0, 2 * d] == diag[0] and s[0, 2 * d] == 2.0


def test_knn_duplicates_and_short_rows():
    """m coincident points: every query's neighbours are the other m-1 ids ascending at s = 0; with
    k > m-1 the row ends with -1 / +inf (fewer than k other points)."""
    P = datagen.duplicates(6, 3)
    ids, s = oracle.knn(P, 5)
    for i in range(6):
        assert ids[i].tolist() == [k for k in range(6) if k != i]
        assert s[i].tolist() == [0.0] * 5
    ids, s = oracle.knn(P, 7)
    assert ids[0].tolist() == [1, 2, 3, 4, 5, -1, -1] and np.isinf(s[0, 5:]).all()


def test_knn_two_set_form_and_sample_rows():
    """The qids / queries forms agree with the full self kNN row for row (queries form: nothing is
    excluded, so a query equal to a point of P gets it first at s = 0)."""
    rng = np.random.default_rng(9)
    P = rng.uniform(0, 1, (400, 4))
    ids, s = oracle.knn(P, 6)
    q = [3, 77, 399]
    i2, s2 = oracle.knn(P, 6, qids=q)
    assert np.array_equal(i2, ids[q]) and np.array_equal(s2, s[q])
    i3, s3 = oracle.knn(P, 7, queries=P[q])
    assert i3[:, 0].tolist() == q and (s3[:, 0] == 0).all()
    assert np.array_equal(i3[:, 1:], ids[q])


# ---------------------------------------------------------------- FP32 self-join (R21)
@pytest.mark.parametrize("d,L", [(2, 8), (3, 6), (4, 4), (6, 3)])
def test_f32_lattice_closed_form(d, L):
    """Integer lattice, eps = 1: every coordinate, difference and square is an exact small integer in
    binary32, so S32 = S = L^d + 2d(L-1)L^(d-1) pairs (the same closed form as the FP64 join)."""
    P = datagen.lattice(L, d).astype(np.float32)
    got = oracle.brute_force_f32(P, 1.0)
    assert len(got) == L ** d + 2 * d * (L - 1) * L ** (d - 1)
    assert np.array_equal(got, oracle.brute_force(P.astype(np.float64), 1.0))


def test_f32_rounding_accepts_what_fp64_rejects():
    """Worked by hand: a = (0,0), b = (1, 2^-13), eps = 1.  Exactly s = 1 + 2^-26 > 1, which binary64
    keeps (rejects the pair); in binary32 1 + 2^-26 is below half an ulp of 1 (2^-24) and rounds to 1,
    so the FP32 predicate accepts it.  (3,4) at eps 5 is the exact tie both include (S.235)."""
    P = np.array([[0.0, 0.0], [1.0, 2.0 ** -13]])
    assert oracle.brute_force_f32(P, 1.0).tolist() == [0, 1, 1 << 32, (1 << 32) | 1]
    assert oracle.brute_force(P, 1.0).tolist() == [0, (1 << 32) | 1]
    T = np.array([[0.0, 0.0], [3.0, 4.0]])
    assert len(oracle.brute_force_f32(T, 5.0)) == 4 and len(oracle.brute_force_f32(T, 4.99)) == 2


@pytest.mark.parametrize("d", [2, 4, 6])
def test_f32_bracketed_by_fp64(d):
    """Random float32 points: the FP32 set lies between the (pinned) FP64 joins at eps(1 -+ 1e-5)
    (binary32 rounding moves a distance by < 1e-6 relative), and is exactly the FP64 set whenever no
    pair sits inside that bracket."""
    P = datagen.uniform(1500, d, seed=60 + d, hi=10.0).astype(np.float32)
    eps = float(np.float32([0.4, 2.5, 4.0][d // 2 - 1]))
    got = set(oracle.brute_force_f32(P, eps).tolist())
    P64 = P.astype(np.float64)
    lo = set(oracle.brute_force(P64, eps * (1 - 1e-5)).tolist())
    hi = set(oracle.brute_force(P64, eps * (1 + 1e-5)).tolist())
    assert lo <= got <= hi
    assert len(got) > 2 * len(P)
    if lo == hi:
        assert got == lo


def test_join_sets_digest_matches_explicit_pairs():
    """The two-set digest (|J|, F_a, F_b, per-query counts) equals the fingerprints of the explicit grid
    join (itself pinned above), on clustered data with duplicates."""
    P = datagen.clustered_small(2500, 3, seed=12)
    Q = P[::2] + 0.01                             # near P's clusters (and its quantised duplicates)
    want = oracle.join_sets(Q, P, 0.6, method="brute")
    dg = oracle.join_sets_digest(Q, P, 0.6, with_counts=True)
    assert dg["pairs"] == len(want) > 1000
    assert (dg["fa"], dg["fb"]) == oracle.fingerprint_pairs(want)
    assert np.array_equal(dg["counts"], np.bincount((want >> np.uint64(32)).astype(np.int64), minlength=len(Q)))


@pytest.mark.parametrize("d", [2, 4, 6])
def test_knn_join_form_equals_kdtree(d):
    """kNN join (queries form, nothing excluded) on continuous random data == scipy cKDTree.query(k) of
    the queries against the points: ids exactly, distances to the library's rounding."""
    rng = np.random.default_rng(400 + d)
    P = rng.uniform(0.0, 10.0, (800, d))
    Q = rng.uniform(-3.0, 13.0, (300, d))
    ids, s = oracle.knn(P, 9, queries=Q)
    dist, nbr = scipy_spatial.cKDTree(P).query(Q, 9)
    assert np.array_equal(ids, nbr)
    np.testing.assert_allclose(np.sqrt(s), dist, rtol=1e-12)
