"""GPU parity of the SURVEY.md §8(f) rank-4 variants (variants.cu) against the oracle
(sj_variants_oracle.c), through the C ABI:

* two-set join J(Q,P) (sj_join_sets; R19): pair sets bit-exact after canonical sort;
* kNN self-join (sj_knn_self; R20): ids AND the float64 bits of s bit-exact (the same operation order on
  both sides, ties broken by id), at sizes spanning many warps and radius rounds, and on sampled rows
  at full size;
* FP32 self-join (sj_self_join_f32; R21): pair sets bit-exact against the binary32 oracle.
"""
import math

import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sj():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1803_04120_b200 as m
    m.load_library()
    return m


def _eps_for(n, d, mean_nbrs, L=100.0):
    vol = mean_nbrs / n * L ** d
    return (vol * math.gamma(1 + d / 2) / math.pi ** (d / 2)) ** (1.0 / d)


def gpu_sets(sj, P, Q, eps, build_masks=True, q_on_device=True, **kw):
    idx = sj.build_index(torch.from_numpy(P).cuda(), eps, build_masks=build_masks)
    Qa = torch.from_numpy(Q).cuda() if q_on_device else Q
    res = sj.join_sets(idx, Qa, **kw)
    got = res.to_numpy(sort=True)
    assert len(got) == res.n_pairs
    return got, res


# ------------------------------------------------------------------ two-set join
SETS = [(d, m) for d in (2, 3, 4, 5, 6) for m in (1, 20, 200)]


@pytest.mark.parametrize("d,m", SETS)
def test_join_sets_matrix_exact(sj, d, m):
    """Uniform P (6000 points) against Q (4000 points reaching 10 % outside P's box), ~m neighbours."""
    P = datagen.uniform(6000, d, seed=40 + d)
    Q = datagen.uniform(4000, d, seed=80 + d, lo=-10.0, hi=110.0)
    eps = _eps_for(6000, d, m)
    want = oracle.join_sets(Q, P, eps)
    got, res = gpu_sets(sj, P, Q, eps)
    assert np.array_equal(got, want)
    assert res.n_batches >= 3 or len(want) < 3


@pytest.mark.parametrize("d", [2, 3, 6])
def test_join_sets_knife_edge_clustered_and_options(sj, d):
    """Knife-edge lattices (pairs at exactly eps and +-2 ulp across cell boundaries) and clustered
    duplicates; masks on/off, host queries, host results, sorted batches and small capacities give the
    same set."""
    eps = 0.75
    P = datagen.knife_edge(3000, d, eps, seed=5 + d)
    Q = datagen.knife_edge(2000, d, eps, seed=9 + d)
    want = oracle.join_sets(Q, P, eps)
    assert len(want) > 0
    for kw in (dict(), dict(build_masks=False), dict(q_on_device=False), dict(result_on_host=True),
               dict(sort_pairs=True), dict(batch_capacity_pairs=257, min_batches=5)):
        got, _ = gpu_sets(sj, P, Q, eps, **kw)
        assert np.array_equal(got, want), kw
    P = datagen.clustered_small(5000, d, seed=3)
    Q = datagen.clustered_small(3000, d, seed=4)
    eps = 0.5
    got, _ = gpu_sets(sj, P, Q, eps, batch_capacity_pairs=1000)
    assert np.array_equal(got, oracle.join_sets(Q, P, eps))


@pytest.mark.parametrize("d,L", [(2, 40), (3, 12), (6, 4)])
def test_join_sets_shifted_lattice_on_gpu(sj, d, L):
    """The closed form pinned for the oracle: Q = P + e_0/4, eps = 1 -> |J| = L^d + (L-1) L^(d-1)."""
    P = datagen.lattice(L, d)
    Q = P.copy()
    Q[:, 0] += 0.25
    got, _ = gpu_sets(sj, P, Q, 1.0)
    assert len(got) == L ** d + (L - 1) * L ** (d - 1)
    assert np.array_equal(got, oracle.join_sets(Q, P, 1.0))


def test_join_sets_degenerate(sj):
    """No queries; queries far outside the grid; one query; Q == P gives the full (3^d) self-join with
    self pairs; a NaN query is rejected (SJ_ERR_NONFINITE)."""
    P = datagen.uniform(3000, 3, seed=1)
    idx = sj.build_index(torch.from_numpy(P).cuda(), 4.0)
    r = sj.join_sets(idx, torch.empty((0, 3), dtype=torch.float64, device="cuda"))
    assert r.n_pairs == 0
    far = np.full((50, 3), 1e9)
    far[::2] = -1e300
    assert sj.join_sets(idx, torch.from_numpy(far).cuda()).n_pairs == 0
    one = P[7:8]
    assert np.array_equal(sj.join_sets(idx, one).to_numpy(sort=True), oracle.join_sets(one, P, 4.0))
    full = sj.join_sets(idx, torch.from_numpy(P).cuda()).to_numpy(sort=True)
    assert np.array_equal(full, oracle.brute_force(P, 4.0))
    assert np.array_equal(full, sj.self_join(idx, unicomp=False).to_numpy(sort=True))
    bad = P[:10].copy()
    bad[3, 1] = np.nan
    with pytest.raises(sj.SJError) as e:
        sj.join_sets(idx, bad)
    assert e.value.status == 2
    res = sj.join_sets(idx, P[:100])
    with pytest.raises(sj.SJError):
        res.dbscan(3)


@pytest.mark.parametrize("cfg,d,eps", [("C2", 6, 1.0), ("C2", 3, 1.0), ("C3", 6, 8.0)])
def test_join_sets_full_size(sj, cfg, d, eps):
    """Full-size: the config's 2 M points P against 2 M independent uniform queries Q; the whole
    canonical-sorted J(Q,P) against the oracle's grid join."""
    P = datagen.uniform_config(cfg, d)
    Q = datagen.uniform(len(P), d, seed=777 + d)
    got, res = gpu_sets(sj, P, Q, eps)
    want = oracle.join_sets(Q, P, eps)
    assert len(got) == len(want)
    assert np.array_equal(got, want)
    res.free()


# ------------------------------------------------------------------ kNN
def gpu_knn(sj, P, k, eps0, **kw):
    ids, s, st = sj.knn_self(torch.from_numpy(P).cuda(), k, eps0, with_stats=True, **kw)
    return ids.cpu().numpy().astype(np.int64), s.cpu().numpy(), st


KNN = [(d, k, f) for d in (2, 3, 4, 5, 6) for k in (1, 8, 32) for f in (0.3, 1.5)]


@pytest.mark.parametrize("d,k,f", KNN)
def test_knn_matrix_exact(sj, d, k, f):
    """5000 uniform points; eps0 = f x the radius holding ~k neighbours (f = 0.3 forces radius rounds);
    ids and the bits of s identical to the oracle's brute force."""
    P = datagen.uniform(5000, d, seed=300 + 10 * d + k)
    eps0 = f * _eps_for(5000, d, k)
    ids, s, st = gpu_knn(sj, P, k, eps0)
    want_i, want_s = oracle.knn(P, k)
    assert np.array_equal(ids, want_i)
    assert np.array_equal(s.view(np.uint64), want_s.view(np.uint64))
    if f < 1:
        assert st["rounds"] >= 2


@pytest.mark.parametrize("d", [2, 3, 6])
def test_knn_ties_duplicates_clusters(sj, d):
    """Exact ties: a lattice (whole shells at equal s), 40 coincident copies of one point (s = 0 ties),
    clustered data with quantised coordinates: ties go to the smaller id on both sides."""
    L = {2: 30, 3: 10, 6: 3}[d]
    P = datagen.lattice(L, d)
    for k in (2 * d, 2 * d + 1, 32):
        if k >= len(P):
            continue
        ids, s, _ = gpu_knn(sj, P, k, 1.0)
        wi, ws = oracle.knn(P, k)
        assert np.array_equal(ids, wi) and np.array_equal(s, ws), k
    P = np.concatenate([datagen.uniform(500, d, seed=2), datagen.duplicates(40, d, value=50.0)])
    ids, s, _ = gpu_knn(sj, P, 16, 0.5)
    wi, ws = oracle.knn(P, 16)
    assert np.array_equal(ids, wi) and np.array_equal(s, ws)
    P = datagen.clustered_small(4000, d, seed=11)
    ids, s, _ = gpu_knn(sj, P, 12, 0.05)
    wi, ws = oracle.knn(P, 12)
    assert np.array_equal(ids, wi) and np.array_equal(s, ws)


def test_knn_edges(sj):
    """k = n - 1 (every other point); host points; bad k / n rejected."""
    P = datagen.uniform(33, 4, seed=5)
    ids, s, _ = gpu_knn(sj, P, 32, 1.0)
    wi, ws = oracle.knn(P, 32)
    assert np.array_equal(ids, wi) and np.array_equal(s, ws)
    ids2, s2 = sj.knn_self(P, 32, 1.0)
    assert np.array_equal(ids2.cpu().numpy(), wi) and np.array_equal(s2.cpu().numpy(), ws)
    for k in (0, 33):
        with pytest.raises(sj.SJError):
            sj.knn_self(P, k, 1.0)
    with pytest.raises(sj.SJError):
        sj.knn_self(P[:5], 5, 1.0)


@pytest.mark.parametrize("cfg,d,k,eps0", [("C2", 6, 8, 6.0), ("C2", 2, 16, 0.3), ("C2", 4, 32, 2.5)])
def test_knn_full_size_sampled_rows(sj, cfg, d, k, eps0):
    """Full size (2 M points): every row is certified; sampled rows (random + the queries that needed
    the most rounds' radius, i.e. the largest k-th distance) equal the oracle's brute force over all N."""
    P = datagen.uniform_config(cfg, d)
    ids, s, st = gpu_knn(sj, P, k, eps0)
    assert (ids >= 0).all() and (ids < len(P)).all()
    assert (np.diff(s, axis=1) >= 0).all()
    rng = np.random.default_rng(d)
    q = np.unique(np.concatenate([rng.integers(0, len(P), 300), np.argsort(s[:, -1])[-100:]]))
    wi, ws = oracle.knn(P, k, qids=q)
    assert np.array_equal(ids[q], wi)
    assert np.array_equal(s[q].view(np.uint64), ws.view(np.uint64))


# ------------------------------------------------------------------ FP32 self-join (R21)
F32 = [(d, m) for d in (2, 3, 4, 5, 6) for m in (2, 50)]


@pytest.mark.parametrize("d,m", F32)
def test_f32_self_join_exact(sj, d, m):
    """float32 uniform points, ~m neighbours: the GPU's binary32 join == the oracle's, pair for pair,
    with and without self pairs, device and host input."""
    P = datagen.uniform(4000, d, seed=500 + d, hi=50.0).astype(np.float32)
    eps = float(np.float32(_eps_for(4000, d, m, L=50.0)))
    want = oracle.brute_force_f32(P, eps)
    res = sj.self_join_f32(torch.from_numpy(P).cuda(), eps)
    assert np.array_equal(res.to_numpy(sort=True), want)
    assert res.n_batches >= 3
    ns = sj.self_join_f32(P, eps, include_self=False, batch_capacity_pairs=999).to_numpy(sort=True)
    assert np.array_equal(ns, oracle.brute_force_f32(P, eps, include_self=False))


@pytest.mark.parametrize("d", [2, 3, 6])
def test_f32_knife_edge_and_rounding(sj, d):
    """Knife-edge float lattices (pairs at eps and +-1-2 float ulps), the hand-worked (1, 2^-13) case
    (binary32 accepts, binary64 rejects) and the lattice closed form."""
    eps = 0.75
    P = datagen.knife_edge(3000, d, eps, seed=21 + d).astype(np.float32)
    assert np.array_equal(sj.self_join_f32(P, eps).to_numpy(sort=True), oracle.brute_force_f32(P, eps))
    A = np.zeros((2, d), np.float32)
    A[1, 0] = 1.0
    A[1, 1] = 2.0 ** -13
    assert sj.self_join_f32(A, 1.0).to_numpy(sort=True).tolist() == [0, 1, 1 << 32, (1 << 32) | 1]
    L = {2: 30, 3: 10, 6: 3}[d]
    Lp = datagen.lattice(L, d).astype(np.float32)
    assert sj.self_join_f32(Lp, 1.0).n_pairs == L ** d + 2 * d * (L - 1) * L ** (d - 1)


def test_f32_full_size(sj):
    """Syn-6D 2 M (C2) rounded to float32 at eps = 8 (the C3 density): the GPU set lies between the
    (pinned) FP64 oracle joins at eps(1 -+ 1e-5), and every pair inside that bracket is decided as the
    FP32 oracle decides it on the pair alone."""
    P32 = datagen.uniform_config("C2", 6).astype(np.float32)
    res = sj.self_join_f32(torch.from_numpy(P32).cuda(), 8.0)
    got = res.to_numpy(sort=True)
    P64 = P32.astype(np.float64)
    lo = oracle.grid_join(P64, 8.0 * (1 - 1e-5))
    hi = oracle.grid_join(P64, 8.0 * (1 + 1e-5))
    assert np.isin(lo, got).all() and np.isin(got, hi).all()
    diff = np.setdiff1d(hi, lo)
    assert len(diff) < 5000
    ing = np.isin(diff, got)
    for x, g in zip(diff.tolist(), ing.tolist()):
        i, k = x >> 32, x & 0xFFFFFFFF
        want = len(oracle.brute_force_f32(P32[[i, k]], 8.0, include_self=False)) == 2
        assert g == want, (i, k)
    res.free()


def test_join_sets_nonfinite_in_a_tiled_warp(sj):
    """A NaN query among queries of one populous cell (the tiled path takes the whole warp) is still
    reported (SJ_ERR_NONFINITE), and so is one among a few queries."""
    P = np.concatenate([datagen.uniform(3000, 2, seed=1), np.full((200, 2), 50.0)])
    idx = sj.build_index(torch.from_numpy(P).cuda(), 2.0)
    Q = np.full((64, 2), 50.25)
    Q[37, 0] = np.nan
    with pytest.raises(sj.SJError) as e:
        sj.join_sets(idx, Q)
    assert e.value.status == 2
    Q2 = np.full((3, 2), 50.25)
    Q2[1, 1] = np.inf
    with pytest.raises(sj.SJError):
        sj.join_sets(idx, Q2)
    ok = np.full((64, 2), 50.25)
    assert np.array_equal(sj.join_sets(idx, ok).to_numpy(sort=True), oracle.join_sets(ok, P, 2.0))


@pytest.mark.parametrize("cfg,d,eps", [("C2", 2, 1.0), ("C3", 6, 16.0), ("C4", 2, 0.005)])
def test_join_sets_full_size_fingerprints(sj, cfg, d, eps):
    """Full-size two-set results too large to hold twice (1.2e9 pairs at C2 2-D): |J|, the multiset
    fingerprints F_a / F_b (device, over all batches) and the per-query counts against the oracle's
    grid digest.  C4: P = the 15.2 M skewed cloud, Q = 2 M points of another skewed draw (the tiled
    path's populous cells and the per-query path's sparse ones in one join)."""
    if cfg == "C4":
        P = datagen.skewed(15_228_633, d)
        Q = datagen.skewed(2_000_000, d, seed=5)
    else:
        P = datagen.uniform_config(cfg, d)
        Q = datagen.uniform(len(P), d, seed=779 + d)
    idx = sj.build_index(torch.from_numpy(P).cuda(), eps)
    res = sj.join_sets(idx, torch.from_numpy(Q).cuda())
    want = oracle.join_sets_digest(Q, P, eps, with_counts=True)
    assert res.n_pairs == want["pairs"]
    fa, fb, cnt = res.fingerprint(counts=True, n_points=max(len(P), len(Q)))
    assert (fa, fb) == (want["fa"], want["fb"])
    assert np.array_equal(cnt.cpu().numpy()[:len(Q)].astype(np.int64), want["counts"])
    res.free()


@pytest.mark.parametrize("cap", [None, 20_000, 3_000])
def test_join_sets_sampled_plan(sj, cap):
    """>= 65536 queries take the sampled one-pass plan (the estimate-then-batch scheme, reading R15):
    skewed queries (clusters + background) and small capacities force many batches and overflowed
    batches re-filled from their exact cursor; the set is unchanged, and a NaN query is still caught."""
    P = datagen.clustered_small(20_000, 2, seed=21, n_clusters=5, sigma=0.8)
    rng = np.random.default_rng(3)
    Q = np.concatenate([datagen.clustered_small(60_000, 2, seed=22, n_clusters=5, sigma=0.8),
                        rng.uniform(-2, 22, (12_000, 2))])
    rng.shuffle(Q)
    eps = 0.15
    want = oracle.join_sets(Q, P, eps)
    kw = {} if cap is None else dict(batch_capacity_pairs=cap)
    got, res = gpu_sets(sj, P, Q, eps, **kw)
    assert np.array_equal(got, want)
    assert res.stats["estimated_pairs"] > 0
    if cap is not None:
        assert res.n_batches >= len(want) // cap
    bad = Q.copy()
    bad[40_000, 1] = np.inf
    with pytest.raises(sj.SJError):
        gpu_sets(sj, P, bad, eps, **kw)


@pytest.mark.parametrize("d,k", [(2, 1), (2, 16), (3, 8), (4, 32), (6, 8)])
def test_knn_join_exact(sj, d, k):
    """kNN join of query rows against points (sj_knn_join): ids and the bits of s equal the oracle's
    brute force (queries form: nothing excluded); queries include copies of points (s = 0, tie by id
    with duplicates) and points far outside the points' box (many radius steps)."""
    P = datagen.uniform(4000, d, seed=600 + d)
    rng = np.random.default_rng(d)
    Q = np.concatenate([datagen.uniform(1500, d, seed=700 + d), P[:50], rng.uniform(-80, 180, (30, d))])
    eps0 = 0.8 * _eps_for(4000, d, k)
    ids, s, st = sj.knn_join(torch.from_numpy(P).cuda(), torch.from_numpy(Q).cuda(), k, eps0, with_stats=True)
    wi, ws = oracle.knn(P, k, queries=Q)
    assert np.array_equal(ids.cpu().numpy().astype(np.int64), wi)
    assert np.array_equal(s.cpu().numpy().view(np.uint64), ws.view(np.uint64))
    assert st["rounds"] >= 2


def test_knn_join_edges(sj):
    """Host inputs; k = n (every point); no queries; a NaN query is rejected; mixed residency rejected."""
    P = datagen.uniform(20, 3, seed=1)
    Q = datagen.uniform(7, 3, seed=2)
    ids, s = sj.knn_join(P, Q, 20, 5.0)
    wi, ws = oracle.knn(P, 20, queries=Q)
    assert np.array_equal(ids.cpu().numpy(), wi) and np.array_equal(s.cpu().numpy(), ws)
    ids0, _ = sj.knn_join(P, np.empty((0, 3)), 4, 5.0)
    assert ids0.shape == (0, 4)
    bad = Q.copy()
    bad[3, 0] = np.nan
    with pytest.raises(sj.SJError) as e:
        sj.knn_join(P, bad, 4, 5.0)
    assert e.value.status == 2
    with pytest.raises(sj.SJError):
        sj.knn_join(P, Q, 21, 5.0)
    with pytest.raises(ValueError):
        sj.knn_join(torch.from_numpy(P).cuda(), Q, 4, 5.0)
