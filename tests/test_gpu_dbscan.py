"""f4: DBSCAN read off the self-join on the GPU (sj_dbscan) against the oracle
(oracle/dbscan.py, itself pinned to scikit-learn and a hand-built fixture in test_oracle_pins.py).
The labelling is unique (reading R17), so labels are compared element by element."""
import numpy as np
import pytest

import datagen
import oracle
from oracle.dbscan import dbscan_from_pairs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sj():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1803_04120_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("kind,d,n,eps,min_pts", [("clustered", 2, 20_000, 0.3, 5), ("clustered", 3, 15_000, 0.6, 10),
                                                  ("uniform", 2, 30_000, 0.6, 4), ("uniform", 6, 20_000, 14.0, 3),
                                                  ("clustered", 2, 20_000, 0.3, 1), ("clustered", 5, 8_000, 1.5, 6)])
@pytest.mark.parametrize("host", [False, True])
def test_dbscan_equals_oracle(sj, kind, d, n, eps, min_pts, host):
    pts = datagen.clustered_small(n, d, seed=d + n) if kind == "clustered" else datagen.uniform(n, d, seed=d + n, hi=30.0)
    pairs = oracle.grid_join(pts, eps)
    want = dbscan_from_pairs(pairs, n, min_pts)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    res = sj.self_join(idx, result_on_host=host, batch_capacity_pairs=max(len(pairs) // 5, 1000))
    assert res.n_batches >= 3
    lab, info = res.dbscan(min_pts)
    got = lab.cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)
    core = np.bincount((pairs >> np.uint64(32)).astype(np.int64), minlength=n) >= min_pts
    assert info["core"] == int(core.sum())
    assert info["noise"] == int((want == -1).sum())
    assert info["clusters"] == len(set(want[core].tolist()))
    res.free()


def test_dbscan_without_self_pairs_and_full_mode(sj):
    """include_self = 0 (|N_eps(p)| then counts p itself implicitly) and the full 3^n search give the
    same labels."""
    pts = datagen.clustered_small(10_000, 2, seed=4)
    want = dbscan_from_pairs(oracle.grid_join(pts, 0.3), len(pts), 6)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), 0.3)
    for kw in ({"include_self": False}, {"unicomp": False}):
        res = sj.self_join(idx, **kw)
        assert np.array_equal(res.dbscan(6)[0].cpu().numpy().astype(np.int64), want), kw
        res.free()


def test_dbscan_rejects_partial_results(sj):
    pts = datagen.uniform(5000, 2, seed=9)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), 2.0)
    res = sj.self_join(idx, query_begin=0, query_end=2500)
    with pytest.raises(Exception):
        res.dbscan(4)
    res.free()
    res = sj.self_join(idx, result_on_host=True, drain_csr=True)
    with pytest.raises(Exception):
        res.dbscan(4)
    res.free()
