"""drain_csr: host-drained batches crossing PCIe as CSR neighbour lists, 4 B per pair + 4 B per row
(PAPER.md:209 sorted key/value pairs; the D2H drain named as the bottleneck at
PAPER.md:262/601).  The pair set must be exactly the oracle's; every batch's rows must partition that
batch's pairs by key; with sort_pairs the rows are ascending."""
import json
import os

import numpy as np
import pytest

import datagen
import fingerprints as F
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fingerprints.json")))


@pytest.fixture(scope="module")
def sj():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1803_04120_b200 as m
    m.load_library()
    return m


def _expand(offs, nb):
    keys = np.repeat(np.arange(len(offs) - 1, dtype=np.uint64), np.diff(offs.astype(np.int64)))
    return (keys << np.uint64(32)) | nb.astype(np.uint64)


@pytest.mark.parametrize("kind,d,n,eps,cap", [("uniform", 2, 10_000, 2.5, None),
                                              ("uniform", 2, 10_000, 2.5, 30_000),
                                              ("clustered", 2, 20_000, 0.4, 50_000),
                                              ("uniform", 3, 8_000, 6.0, 20_000),
                                              ("uniform", 6, 6_000, 30.0, 40_000)])
@pytest.mark.parametrize("sort", [False, True])
def test_csr_drain_equals_oracle(sj, kind, d, n, eps, cap, sort):
    pts = datagen.uniform(n, d, seed=11 * n + d) if kind == "uniform" else datagen.clustered_small(n, d, seed=3 + d)
    want = oracle.brute_force(pts, eps)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), eps)
    res = sj.self_join(idx, result_on_host=True, drain_csr=True, sort_pairs=sort, batch_capacity_pairs=cap)
    assert res.n_pairs == len(want)
    total = 0
    parts = []
    for b in range(res.n_batches):
        offs, nb = res.batch_csr(b)
        assert len(offs) == n + 1 and offs[0] == 0 and offs[-1] == len(nb)
        assert np.all(np.diff(offs.astype(np.int64)) >= 0)
        pb = _expand(offs, nb)
        if sort:                               # rows ascending: the expanded batch is sorted
            assert np.all(pb[1:] >= pb[:-1])
        parts.append(pb)
        total += len(nb)
    assert total == len(want)
    got = np.sort(np.concatenate(parts)) if parts else np.empty(0, np.uint64)
    assert np.array_equal(got, want)
    assert np.array_equal(res.to_numpy(sort=True), want)            # sj_result_copy_to_host expands
    assert res.fingerprint() == F.fingerprint(want)                   # CSR-aware fingerprint
    with pytest.raises(Exception):
        res.batch(0)                                                  # pairs view refused for CSR
    res.free()


def test_csr_drain_requires_host_results(sj):
    pts = datagen.uniform(1000, 2, seed=5)
    idx = sj.build_index(torch.from_numpy(pts).cuda(), 3.0)
    with pytest.raises(Exception):
        sj.self_join(idx, drain_csr=True)
    # a device-resident result has no CSR batches
    res = sj.self_join(idx)
    with pytest.raises(Exception):
        res.batch_csr(0)
    res.free()


def test_csr_drain_full_size_c3_eps16(sj):
    """C3 eps=16 (2.6e8 pairs, ~1 buffer): the CSR-drained result's |S|, F_a, F_b and per-key count
    fingerprint equal the oracle's golden values."""
    g = GOLD["C3/d6/eps16"]
    P = datagen.uniform_config("C3", 6)
    idx = sj.build_index(torch.from_numpy(P).cuda(), g["eps"])
    res = sj.self_join(idx, result_on_host=True, drain_csr=True)
    assert res.n_pairs == g["pairs"]
    fa, fb, cnt = res.fingerprint(counts=True, n_points=len(P))
    assert f"{fa:016x}" == g["fa"] and f"{fb:016x}" == g["fb"]
    assert f"{F.count_fingerprint(cnt.cpu().numpy()):016x}" == g["fc"]
    res.free()
