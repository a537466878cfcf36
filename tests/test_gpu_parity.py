"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by element.

Bar (task rule ③): integer pair sets bit-exact after canonical sort; the FP64 predicate is
evaluated with the same operation order on both sides, so there is no tolerance anywhere.
"""
import math
import os

import numpy as np
import pytest

import datagen
import oracle
from oracle import index_ref as ir

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sj():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1803_04120_b200 as m
    m.load_library()
    return m


def gpu_pairs(sj, pts, eps, **kw):
    on_dev = kw.pop("points_on_device", True)
    P = torch.from_numpy(pts).cuda() if on_dev else pts
    idx = sj.build_index(P, eps)
    res = sj.self_join(idx, **kw)
    out = res.to_numpy(sort=True)
    assert len(out) == res.n_pairs
    return out, res, idx


# ------------------------------------------------------------------ small exact parity matrix
def _eps_for(n, d, mean_nbrs, L=100.0):
    # eps such that the expected neighbours per point ~ mean_nbrs (ball volume, no boundary)
    vol = mean_nbrs / n * L ** d
    return (vol * math.gamma(1 + d / 2) / math.pi ** (d / 2)) ** (1.0 / d)


MATRIX = [(d, n, m) for d in (2, 3, 4, 5, 6) for n in (10, 100, 1000, 5000) for m in (1, 10, 100)]


@pytest.mark.parametrize("d,n,m", MATRIX)
def test_uniform_matrix_exact(sj, d, n, m):
    """SPEC criterion 1 (S.398): n in {10..5000}, d in 2..6, mean neighbours ~{1,10,100}."""
    pts = datagen.uniform(n, d, seed=1000 * d + n + m)
    eps = _eps_for(n, d, m)
    want = oracle.brute_force(pts, eps)
    got, res, _ = gpu_pairs(sj, pts, eps)
    assert np.array_equal(got, want)
    assert res.n_batches >= 3 or n < 3


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("kind", ["clustered", "knife", "dups", "lattice"])
def test_structured_inputs_exact(sj, d, kind):
    if kind == "clustered":
        pts, eps = datagen.clustered_small(3000, d, seed=d), 0.5
    elif kind == "knife":
        pts, eps = datagen.knife_edge(3000, d, 0.1, seed=d), 0.1
    elif kind == "dups":
        pts = np.concatenate([datagen.duplicates(300, d), datagen.uniform(700, d, seed=d, hi=5.0)])
        eps = 0.7
    else:
        L = {2: 40, 3: 12, 4: 6, 5: 4, 6: 3}[d]
        pts, eps = datagen.lattice(L, d), 1.0
    want = oracle.brute_force(pts, eps)
    for unicomp in (True, False):
        got, _, _ = gpu_pairs(sj, pts, eps, unicomp=unicomp)
        assert np.array_equal(got, want), f"unicomp={unicomp}"


@pytest.mark.parametrize("d,L", [(2, 30), (3, 10), (4, 6), (6, 3)])
def test_lattice_closed_form(sj, d, L):
    """P2 on the GPU: |S| = L^d + 2d(L-1)L^(d-1) (eps = 1, unit lattice)."""
    got, _, _ = gpu_pairs(sj, datagen.lattice(L, d), 1.0)
    assert len(got) == L ** d + 2 * d * (L - 1) * L ** (d - 1)


def test_sqrt2_lattice(sj):
    """P3: eps = fl(sqrt 2) accepts the face diagonals (interior count 1 + 2d^2)."""
    d, L = 3, 6
    P = datagen.lattice(L, d)
    got, _, _ = gpu_pairs(sj, P, math.sqrt(2.0))
    cnt = oracle.pair_counts(got, len(P))
    interior = np.all((P > 0) & (P < L - 1), axis=1)
    assert np.all(cnt[interior] == 1 + 2 * d * d)


def test_worked_examples(sj):
    """SPEC S.235-236, S.272-273, S.316."""
    P = np.array([[0.0, 0.0], [3.0, 4.0]])
    assert gpu_pairs(sj, P, 5.0)[0].tolist() == [0, 1, (1 << 32), (1 << 32) | 1]
    assert gpu_pairs(sj, P, 4.9)[0].tolist() == [0, (1 << 32) | 1]
    assert gpu_pairs(sj, np.array([[1.5, 2.5]]), 1.0)[0].tolist() == [0]
    assert len(gpu_pairs(sj, np.array([[1.0, 1.0], [1.0, 1.0]]), 1.0)[0]) == 4
    P = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0]])
    assert len(gpu_pairs(sj, P, 1.0)[0]) == 7


def test_include_self_false(sj):
    pts = datagen.uniform(3000, 3, seed=5)
    want = oracle.brute_force(pts, 6.0, include_self=False)
    for unicomp in (True, False):
        got, _, _ = gpu_pairs(sj, pts, 6.0, include_self=False, unicomp=unicomp)
        assert np.array_equal(got, want)


def test_host_points_and_host_results(sj):
    pts = datagen.uniform(4000, 4, seed=9)
    want = oracle.brute_force(pts, 12.0)
    got, res, _ = gpu_pairs(sj, pts, 12.0, points_on_device=False, result_on_host=True)
    assert np.array_equal(got, want)
    b0 = res.batch(0)
    assert isinstance(b0, np.ndarray)


@pytest.mark.parametrize("host", [False, True])
def test_batching_invariance_and_overflow(sj, host):
    """SPEC criterion 4 (S.401): identical output for any capacity / min_batches; tiny
    capacities force overflow re-runs (device: exact realloc; host: split)."""
    pts = datagen.uniform(6000, 2, seed=3)
    eps = 2.0
    want = oracle.brute_force(pts, eps)
    for cap, mb in ((1 << 28, 3), (1000, 5), (100, 8), (10_000_000, 1)):
        got, res, _ = gpu_pairs(sj, pts, eps, batch_capacity_pairs=cap, min_batches=mb, result_on_host=host)
        assert np.array_equal(got, want)
        assert res.n_batches >= min(mb, 1)
        if cap == 100:
            assert res.stats["retries"] > 0


@pytest.mark.parametrize("streams", [1, 2, 5])
def test_stream_count_invariance(sj, streams):
    pts = datagen.uniform(5000, 3, seed=4)
    want = oracle.brute_force(pts, 7.0)
    for host in (False, True):
        got, _, _ = gpu_pairs(sj, pts, 7.0, n_streams=streams, result_on_host=host)
        assert np.array_equal(got, want)


def test_query_range_shards_union(sj):
    """North star sharding: the union over a partition of [0,N) in A-order is S (no dups)."""
    pts = datagen.uniform(5000, 4, seed=12)
    eps = 15.0
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    for parts in (2, 3, 8):
        cuts = np.linspace(0, 5000, parts + 1).astype(int)
        allp = np.concatenate([sj.self_join(idx, query_begin=int(a), query_end=int(b)).to_numpy(sort=False)
                               for a, b in zip(cuts[:-1], cuts[1:])])
        allp.sort()
        assert np.array_equal(allp, want)


def test_neighbor_counts(sj):
    """P6: per-point counts equal the oracle's; the total equals |S|."""
    pts = datagen.clustered_small(4000, 3, seed=8)
    eps = 0.6
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    for unicomp in (True, False):
        cnt, tot = sj.neighbor_counts(idx, unicomp=unicomp)
        assert tot == len(want)
        assert np.array_equal(cnt.cpu().numpy().astype(np.int64), oracle.pair_counts(want, len(pts)))


# ------------------------------------------------------------------ index parity
@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
def test_index_matches_oracle_index(sj, d):
    """a1-a4 vs the oracle's statement of §4.2-4.4: geometry, B, G, A, masks bit-exact."""
    for pts, eps in ((datagen.uniform(3000, d, seed=d), 9.0), (datagen.knife_edge(2000, d, 0.1, seed=d), 0.1),
                     (datagen.clustered_small(2500, d, seed=d), 0.3)):
        ref = ir.build_index(pts, eps)
        idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
        g = idx.geometry()
        assert g["w"] == ref.geom.w and g["cpd"] == ref.geom.cpd and g["strides"] == ref.geom.strides
        assert g["mins"] == ref.geom.mins.tolist()
        arr = idx.arrays()
        assert arr["B"].cpu().numpy().tolist() == ref.B
        assert arr["G"].cpu().numpy().astype(np.int64).tolist() == ref.G.tolist()
        assert np.array_equal(arr["A"].cpu().numpy().astype(np.int64), ref.A)
        X = arr["X"].cpu().numpy()
        assert np.array_equal(X, pts[ref.A].T)
        pc = arr["pcell"].cpu().numpy().astype(np.int64)
        assert np.array_equal(pc, np.repeat(np.arange(len(ref.B)), np.diff(ref.G)))
        if "masks" in arr:
            words = arr["masks"].cpu().numpy().astype(np.uint64)
            bits = ((words[:, None] >> np.arange(32, dtype=np.uint64)) & np.uint64(1)).reshape(-1)
            off = g["mask_offsets"]
            for j in range(d):
                assert np.nonzero(bits[off[j]:off[j + 1]])[0].tolist() == ref.M[j]


def test_fig2_fixture_on_gpu(sj):
    """the GPU index of the Fig. 2 replica."""
    P = np.loadtxt(os.path.join(GOLDEN, "fig2_points.txt"))
    idx = sj.build_index(torch.from_numpy(P).cuda(), 1.0)
    arr = idx.arrays()
    B = arr["B"].cpu().numpy().tolist()
    assert len(B) == 11 and B[5] == 22 and B[6] == 30
    G = arr["G"].cpu().numpy()
    A = arr["A"].cpu().numpy()
    assert set(A[G[5]:G[6]].tolist()) == {35, 6}
    assert np.array_equal(gpu_pairs(sj, P, 1.0)[0], oracle.brute_force(P, 1.0))


def test_errors(sj):
    P = datagen.uniform(100, 3, seed=1)
    bad = P.copy()
    bad[17, 2] = np.nan
    with pytest.raises(sj.SJError) as e:
        sj.build_index(torch.from_numpy(bad).cuda(), 1.0)
    assert e.value.name == "SJ_ERR_NONFINITE"
    with pytest.raises(sj.SJError) as e:
        sj.build_index(torch.from_numpy(datagen.uniform(100, 6, seed=2, hi=1e6)).cuda(), 1e-3)
    assert e.value.name == "SJ_ERR_KEY_OVERFLOW"
    idx = sj.build_index(torch.from_numpy(P).cuda(), 1.0)
    with pytest.raises(sj.SJError) as e:
        sj.self_join(idx, query_begin=5, query_end=1000)
    assert e.value.name == "SJ_ERR_ARG"


def test_c1_config_exact(sj):
    """BASELINE.json configs[0]: Syn-2D 10K, eps=2.5 -- full pair set."""
    pts = datagen.uniform_config("C1", 2)
    want = oracle.grid_join(pts, 2.5)
    for unicomp in (True, False):
        got, _, _ = gpu_pairs(sj, pts, 2.5, unicomp=unicomp)
        assert np.array_equal(got, want)


def _gapped(n, d, seed):
    """Points in separated slabs: whole coordinate columns of the grid are empty, so the
    masks M_j actually remove adjacent coordinates."""
    rng = np.random.default_rng(seed)
    P = rng.uniform(0, 10, (n, d))
    P[:, 0] = np.where(rng.random(n) < 0.5, P[:, 0], P[:, 0] + 3.0)   # shifted half
    P[:, 1] = np.floor(P[:, 1] * 2.0) / 2.0 * 1.5                     # quantised rows
    return P


@pytest.mark.parametrize("d", [2, 3, 5, 6])
def test_masks_option_invariance(sj, d):
    pts = _gapped(4000, d, seed=d)
    eps = 0.6
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    for use_masks in (True, False):
        for unicomp in (True, False):
            got = sj.self_join(idx, use_masks=use_masks, unicomp=unicomp).to_numpy()
            assert np.array_equal(got, want), (use_masks, unicomp)


@pytest.mark.parametrize("d,n,eps", [(2, 5000, 1.5), (3, 8000, 4.0), (4, 20000, 6.0), (6, 30000, 20.0),
                                     (6, 3000, 0.5), (2, 50, 1e-3)])
def test_prefix_directory_definition(sj, d, n, eps):
    """dir[p] = lower_bound(B, p * stride_{d-k}) for every prefix p (index_build.cu)."""
    pts = datagen.uniform(n, d, seed=n + d)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    g = idx.geometry()
    arr = idx.arrays()
    B = arr["B"].cpu().numpy().astype(object)
    k = g["dir_k"]
    div = 1
    for j in range(d - k):
        div *= g["cpd"][j]
    P = 1
    for j in range(d - k, d):
        P *= g["cpd"][j]
    assert g["dir_entries"] == P + 1
    Bn = np.array([int(b) // div for b in B], dtype=np.int64)
    want = np.searchsorted(Bn, np.arange(P + 1), side="left")
    assert np.array_equal(arr["dir"].cpu().numpy().astype(np.int64), want)
    assert np.array_equal(sj.self_join(idx).to_numpy(), oracle.brute_force(pts, eps)) if n <= 8000 else True


@pytest.mark.parametrize("d,n,eps", [(2, 4000, 2.0), (3, 5000, 6.0), (4, 6000, 12.0), (6, 5000, 25.0),
                                     (6, 4000, 60.0), (5, 3000, 8.0)])
def test_lanes_per_query_invariance(sj, d, n, eps):
    """S is independent of how many lanes cooperate on a query (G = 1..32), in every search
    mode the index picks (dense rows / cell scan / rows), unicomp and full."""
    pts = datagen.uniform(n, d, seed=5 * n + d)
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    for G in (1, 2, 4, 8, 16, 32):
        for unicomp in (True, False):
            got = sj.self_join(idx, lanes_per_query=G, unicomp=unicomp).to_numpy()
            assert np.array_equal(got, want), (G, unicomp)
        cnt, tot = sj.neighbor_counts(idx, lanes_per_query=G)
        assert tot == len(want)


@pytest.mark.parametrize("kind,d,eps", [("uniform", 2, 3.0), ("uniform", 3, 9.0), ("clustered", 2, 0.4),
                                        ("clustered", 3, 0.5), ("clustered", 6, 1.2), ("dups", 4, 0.5)])
def test_dense_cells_path_invariance(sj, kind, d, eps):
    """The warp-per-task dense path (cells with >= 16 points, warp-buffered emission) gives the
    same S as the per-query path, for unicomp and full search, device and host batches, and with
    capacities small enough to overflow inside the warp buffers' flushes."""
    if kind == "uniform":
        pts = datagen.uniform(6000, d, seed=d)
    elif kind == "clustered":
        pts = datagen.clustered_small(6000, d, seed=d, sigma=0.3)
    else:
        pts = np.concatenate([datagen.duplicates(700, d), datagen.uniform(1500, d, seed=d, hi=4.0)])
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    for dense in (True, False):
        for unicomp in (True, False):
            got = sj.self_join(idx, dense_cells=dense, unicomp=unicomp).to_numpy()
            assert np.array_equal(got, want), (dense, unicomp)
    for cap in (5000, 300):
        got = sj.self_join(idx, batch_capacity_pairs=cap, result_on_host=True).to_numpy()
        assert np.array_equal(got, want)


# ------------------------------------------------------------------ NEXT rows f2, f3
@pytest.mark.parametrize("host", [False, True])
def test_sort_pairs_per_batch(sj, host):
    """f2: with sort_pairs every batch comes back sorted by (key, value), and the
    batches still partition S."""
    pts = datagen.clustered_small(5000, 3, seed=21)
    eps = 0.5
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    res = sj.self_join(idx, sort_pairs=True, result_on_host=host, batch_capacity_pairs=20000)
    parts = []
    for b in res.batches():
        a = b.cpu().numpy().view(np.uint64) if isinstance(b, torch.Tensor) else np.asarray(b)
        assert np.all(a[1:] >= a[:-1])
        parts.append(a)
    assert res.n_batches >= 3
    assert np.array_equal(np.sort(np.concatenate(parts)), want)


@pytest.mark.parametrize("d,n,eps", [(2, 3000, 3.0), (4, 2500, 15.0), (6, 2000, 35.0)])
def test_brute_force_join(sj, d, n, eps):
    """f3: the GPU all-pairs join equals the oracle's brute force and the grid
    join, with and without self pairs; sort_pairs returns it in canonical order."""
    pts = datagen.uniform(n, d, seed=n + 3 * d)
    for inc in (True, False):
        want = oracle.brute_force(pts, eps, include_self=inc)
        got = sj.brute_force_join(torch.from_numpy(pts).cuda(), eps, include_self=inc).to_numpy()
        assert np.array_equal(got, want)
    r = sj.brute_force_join(pts, eps, sort_pairs=True, result_on_host=True)
    b = np.asarray(r.batch(0))
    assert np.array_equal(b, oracle.brute_force(pts, eps))
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    assert np.array_equal(sj.self_join(idx).to_numpy(), b)


@pytest.mark.parametrize("d,eps", [(2, 2.0), (3, 4.0), (4, 8.0), (5, 12.0), (6, 18.0)])
def test_unicomp_halves_the_work(sj, d, eps):
    """f1 / SPEC criterion 3 (S.400, PAPER.md:346 'reduces ... distance calculations roughly by a
    factor of two'): uniform 10^5 points, >= 10 neighbours: unicomp's candidate tests are within
    [0.4, 0.6] of the full 3^d search, with identical pair sets."""
    pts = datagen.uniform(100_000, d, seed=300 + d)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    ru = sj.self_join(idx, unicomp=True)
    rf = sj.self_join(idx, unicomp=False)
    assert ru.n_pairs == rf.n_pairs and ru.n_pairs / len(pts) >= 10
    ratio = ru.stats["candidates_tested"] / rf.stats["candidates_tested"]
    assert 0.4 <= ratio <= 0.6, ratio
    assert np.array_equal(ru.to_numpy(), rf.to_numpy())


@pytest.mark.parametrize("m", [3000, 7000])
def test_prefix_bucket_sort_big_buckets(sj, m):
    """a3 prefix-bucket sort (sparse 6-D keys, N <= 2P): one top-k prefix holds m points -- a
    bucket sorted in shared memory by one CTA (m <= 4096) or, beyond that, flagged on the device
    and rebuilt with the LSD radix sort.  Either way A must equal the stable order (R14)."""
    rng = np.random.default_rng(m)
    n = 20000
    pts = rng.uniform(0, 100, (n, 6))
    pts[:m, 4:] = 50.25 + rng.uniform(0, 0.5, (m, 2))      # same (c_4, c_5) cell prefix
    pts[:m, :4] = rng.uniform(40, 60, (m, 4))               # neighbours inside the cluster
    rng.shuffle(pts)
    eps = 1.0
    ref = ir.build_index(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    arr = idx.arrays()
    assert arr["B"].cpu().numpy().tolist() == ref.B
    assert np.array_equal(arr["A"].cpu().numpy().astype(np.int64), ref.A)
    assert np.array_equal(arr["X"].cpu().numpy(), pts[ref.A].T)
    got = sj.self_join(idx).to_numpy(sort=True)
    assert np.array_equal(got, oracle.brute_force(pts, eps))


@pytest.mark.parametrize("host", [False, True])
def test_csr_output(sj, host):
    """f2 CSR neighbour lists (4 B/pair + offsets) equal the oracle's pairs grouped by key, rows
    ascending -- across several batches, device- and host-resident."""
    n, d, eps = 4000, 3, 6.0
    pts = datagen.uniform(n, d, seed=31)
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    res = sj.self_join(idx, result_on_host=host, min_batches=5)
    assert res.n_batches >= 5
    offsets, nbrs = res.to_csr(n)
    keys = (want >> np.uint64(32)).astype(np.int64)
    want_off = np.concatenate([[0], np.cumsum(np.bincount(keys, minlength=n))])
    assert np.array_equal(offsets.cpu().numpy(), want_off)
    assert np.array_equal(nbrs.cpu().numpy().astype(np.uint32), (want & np.uint64(0xFFFFFFFF)).astype(np.uint32))


def test_lazy_timings_and_stats(sj):
    """Build/join device timings are computed on request from pooled CUDA events
    (sj_index_timings, sj_result_info with stats): positive and consistent with the work done."""
    pts = datagen.uniform(200000, 4, seed=5)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), 2.0, speculative_estimate=False)
    res = sj.self_join(idx)
    t = idx.timings()
    assert t["total_ms"] > 0 and t["total_ms"] >= t["sort_ms"] >= 0
    st = res.stats
    assert st["refine_ms"] > 0 and st["refine_span_ms"] > 0 and st["refine_max_ms"] <= st["refine_ms"] + 1e-6
    assert st["estimate_ms"] > 0 and st["batches"] == res.n_batches >= 3
    # unicomp: every accepted test emits both orientations, self pairs need no test
    assert st["pairs"] == res.n_pairs and 2 * st["candidates_tested"] + len(pts) >= res.n_pairs


@pytest.mark.parametrize("d,n,eps", [(6, 300000, 1.0), (5, 200000, 1.5), (4, 200000, 3.0), (3, 200000, 2.0),
                                     (2, 100000, 0.3)])
def test_build_time_estimate_is_the_join_estimate(sj, d, n, eps):
    """The default join's a5 estimate run by the build (before its final sync) equals the join's own
    estimate (same deterministic sample): same estimated_pairs, same batch plan, same pairs.  Covers
    both sort paths (prefix buckets, LSD) and all three search modes."""
    pts = torch.from_numpy(datagen.uniform(n, d, seed=9 + d)).cuda()
    a = sj.self_join(sj.build_index(pts, eps, speculative_estimate=True))
    b = sj.self_join(sj.build_index(pts, eps, speculative_estimate=False))
    assert a.stats["estimated_pairs"] == b.stats["estimated_pairs"] and a.n_batches == b.n_batches
    assert a.n_pairs == b.n_pairs
    assert b.stats["estimate_ms"] > 0


@pytest.mark.parametrize("d", [2, 3, 4, 5, 6])
def test_tiny_inputs(sj, d):
    """Degenerate sizes: one point, two identical points, two points just outside eps -- device and
    host results, CSR output."""
    for pts, eps in ((np.zeros((1, d)), 1.0), (np.ones((2, d)), 0.5),
                     (np.stack([np.zeros(d), np.full(d, 1.0)]), 0.999)):
        want = oracle.brute_force(pts, eps)
        for host in (False, True):
            got, res, _ = gpu_pairs(sj, pts, eps, result_on_host=host)
            assert np.array_equal(got, want)
            off, nb = res.to_csr(len(pts))
            keys = (want >> np.uint64(32)).astype(np.int64)
            assert np.array_equal(off.cpu().numpy(), np.concatenate([[0], np.cumsum(np.bincount(keys, minlength=len(pts)))]))


@pytest.mark.parametrize("host", [False, True])
def test_dense_tasks_small_batches(sj, host):
    """Dense-cell tasks with batches of ~100 queries over runs of 16-25-point cells:
    a batch intersects more tasks than (q1-q0)/dense_T when cell tails are short, and every one of
    them must run (their self pairs sit in fixed slots)."""
    n = 20000
    pts = datagen.uniform(n, 2, seed=41)
    eps = 3.16          # ~1000 cells of ~20 points (w ~ eps)
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    per_query = len(want) / n
    for nq in (37, 100, 230):
        cap = int(nq * per_query * 1.3)
        res = sj.self_join(idx, batch_capacity_pairs=cap, result_on_host=host)
        assert res.n_batches > n // (2 * nq)
        assert np.array_equal(res.to_numpy(), want), nq


def test_fingerprint_device_and_host_batches(sj):
    """sj_result_fingerprint over device batches and over pinned host batches (read through the UVA
    mapping) equals the fingerprint of the oracle's explicit S; per-key counts too."""
    import fingerprints as F
    pts = datagen.clustered_small(6000, 3, seed=17)
    eps = 0.5
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    for host in (False, True):
        res = sj.self_join(idx, result_on_host=host, min_batches=4)
        fa, fb, cnt = res.fingerprint(counts=True, n_points=len(pts))
        assert (fa, fb) == F.fingerprint(want)
        assert np.array_equal(cnt.cpu().numpy().astype(np.int64), oracle.pair_counts(want, len(pts)))
        with pytest.raises(sj.SJError):
            res.to_csr(len(pts) - 1)              # n_points below the joined N is rejected
        res.free()


def test_freed_buffers_reused_after_pending_reads(sj):
    """A result freed while an async read of its zero-copy batch view is still queued: the next
    join reuses the cached buffer only after that read completed (sj_free_result_async)."""
    pts = datagen.uniform(300_000, 2, seed=8)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), 0.4)
    # a different point set of the same shape: the next join writes different pairs into the buffers
    idx2 = sj.build_index(torch.from_numpy(datagen.uniform(300_000, 2, seed=9)).cuda(), 0.4)
    ref = sj.self_join(idx)
    want = sum(int(b.view(torch.int64).sum().item()) for b in ref.batches())
    ref.free()
    side = torch.cuda.Stream()
    for _ in range(3):
        res = sj.self_join(idx)
        with torch.cuda.stream(side):
            torch.cuda._sleep(20_000_000)         # keep the side stream busy (~10 ms)
            sums = [b.view(torch.int64).sum() for b in res.batches()]
            res.free(stream=side.cuda_stream)
        nxt = sj.self_join(idx2)                 # may get the same buffers from the cache
        side.synchronize()
        assert sum(int(x.item()) for x in sums) == want
        nxt.free()


def test_trim_and_cache_limit(sj):
    pts = datagen.uniform(200_000, 3, seed=2)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), 2.0)
    want = sj.self_join(idx).to_numpy()
    sj.set_result_cache_limit(0)
    r = sj.self_join(idx)
    r.free()
    sj.trim()
    sj.set_result_cache_limit(48 << 30)
    assert np.array_equal(sj.self_join(idx).to_numpy(), want)


@pytest.mark.parametrize("d,n,eps", [(6, 2_000_000, 1.0), (6, 2_000_000, 4.0), (5, 2_000_000, 1.0),
                                     (4, 300_000, 3.0), (2, 200_000, 0.5)])
def test_imported_index_equals_built(sj, d, n, eps):
    """The multi-GPU import path: an index imported from the exported arrays (copied)
    and one imported in place from the packed buffer (sj_index_import_borrowed, what a non-zero rank
    does with the broadcast buffer) join to the same S as the built index -- same |S| and
    fingerprints -- in the sparse regimes whose occupancy bitmaps (occ, occ2) are rebuilt on import."""
    from paper_1803_04120_b200 import distributed as sjd
    pts = torch.from_numpy(datagen.uniform(n, d, seed=91 + d)).cuda()
    idx = sj.build_index(pts, eps)
    r0 = sj.self_join(idx)
    want = (r0.n_pairs, r0.fingerprint())
    r0.free()
    copied = sj.import_index(idx.view, 0)
    meta, buf, masks = sjd.index_meta(idx, sj.plan_shards(idx, 3))
    buf2 = buf.clone()                         # stands for the received broadcast buffer
    borrowed = sj.import_index(sjd.view_from_packed(meta, buf2, masks, 0), 0, borrow=(buf2, masks))
    for imp in (copied, borrowed):
        assert imp.n_cells == idx.n_cells
        r = sj.self_join(imp)
        assert (r.n_pairs, r.fingerprint()) == want
        r.free()
        # and sharded: the three ranges of the plan
        _, cuts = sjd.unpack_layout(meta)
        fa = fb = tot = 0
        for a, b in zip(cuts[:-1], cuts[1:]):
            r = sj.self_join(imp, query_begin=int(a), query_end=int(b))
            x, y = r.fingerprint()
            fa, fb, tot = (fa + x) % 2**64, (fb + y) % 2**64, tot + r.n_pairs
            r.free()
        assert (tot, (fa, fb)) == want


def test_torch_allocator_hook(sj):
    """sj_set_allocator wired to torch's caching allocator (sj.use_torch_allocator): the index and
    the device result batches are carved from torch's pool (torch.cuda.memory_allocated grows by at
    least the index's SoA copy while they live, and returns when they are freed); S is unchanged."""
    pts = datagen.uniform(20_000, 3, seed=77)
    want = oracle.grid_join(pts, 4.0)
    P = torch.from_numpy(pts).cuda()
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    sj.use_torch_allocator(True)
    try:
        idx = sj.build_index(P, 4.0)
        res = sj.self_join(idx)
        torch.cuda.synchronize()
        during = torch.cuda.memory_allocated()
        assert during - base >= pts.nbytes          # X (8dN) alone lives in torch's pool
        assert np.array_equal(res.to_numpy(), want)
        res.free()
        idx.free()
        torch.cuda.synchronize()
        assert torch.cuda.memory_allocated() == base
    finally:
        sj.use_torch_allocator(False)
    # and the library's own pool again
    idx = sj.build_index(P, 4.0)
    assert np.array_equal(sj.self_join(idx).to_numpy(), want)


def test_cell_coordinates_at_cell_boundaries(sj):
    """The key pass's division-free c_j (cell_floor: fl(t * fl(1/w)) with an exact-division fallback
    near integers) against the oracle's floor(fl(t / w)) on coordinates AT the cell boundaries:
    k * w and its neighbours within +-3 ulps for every k, so t / w sits within ulps of integers."""
    rng = np.random.default_rng(1234)
    for d, eps in ((3, 0.7), (6, 3.3), (2, 0.013)):
        base = np.array([[0.0] * d, [100.0] * d])
        w = ir.build_index(base, eps).geom.w
        vals = []
        for k in range(0, int(100.0 / w) + 1):
            x = k * w
            for s in range(-3, 4):
                y = x
                for _ in range(abs(s)):
                    y = np.nextafter(y, np.inf if s > 0 else -np.inf)
                if 0.0 <= y <= 100.0:
                    vals.append(y)
        vals = np.array(vals)
        pts = np.vstack([base, vals[rng.integers(0, len(vals), (4000, d))]])
        ref = ir.build_index(pts, eps)
        assert ref.geom.w == w
        idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
        arr = idx.arrays()
        assert arr["B"].cpu().numpy().tolist() == ref.B
        assert np.array_equal(arr["A"].cpu().numpy().astype(np.int64), ref.A)
        assert np.array_equal(sj.self_join(idx).to_numpy(), oracle.grid_join(pts, eps))


def test_build_after_failed_build(sj):
    """Regression: the key pass launches programmatically behind the min/max pass and must read the
    geometry only after griddepcontrol.wait.  A small 2-D build, a failed build (NaN -> SJ_ERR_NONFINITE,
    overflow -> SJ_ERR_KEY_OVERFLOW) and then C1 once faulted in the compaction: the key pass had read
    the failed build's status (a load the compiler hoisted above the wait) and skipped its keys."""
    P = datagen.uniform(5000, 2, seed=3)
    sj.build_index(torch.from_numpy(P).cuda(), 4.0).free()
    bad = datagen.uniform(100, 3, seed=1)
    bad[17, 2] = np.nan
    with pytest.raises(sj.SJError):
        sj.build_index(torch.from_numpy(bad).cuda(), 1.0)
    pts = datagen.uniform_config("C1", 2)
    got, _, _ = gpu_pairs(sj, pts, 2.5)
    assert np.array_equal(got, oracle.grid_join(pts, 2.5))
    with pytest.raises(sj.SJError):
        sj.build_index(torch.from_numpy(datagen.uniform(100, 6, seed=2, hi=1e6)).cuda(), 1e-3)
    got, _, _ = gpu_pairs(sj, pts, 2.5)
    assert np.array_equal(got, oracle.grid_join(pts, 2.5))
