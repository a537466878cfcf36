"""CPU-side checks of the C ABI: the library loads, exports every symbol include/sj.h declares,
validates arguments on the host before touching CUDA, and plans batches (host-only logic)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sj():
    from paper_1803_04120_b200 import build as b
    b.build()
    import paper_1803_04120_b200 as m
    m.load_library()
    return m


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "sj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sj_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(sj):
    syms = declared_symbols()
    assert "sj_build_index" in syms and "sj_self_join" in syms and "sj_free_result" in syms
    lib = ctypes.CDLL(sj.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s


def test_abi_struct_sizes_match_header(sj):
    """The ctypes mirrors have the C layout (checked against offsets computed by the compiler
    would need a GPU-free C program; here: field count and 8-byte alignment sanity)."""
    assert ctypes.sizeof(sj.sj.JoinOpts) % 8 == 0
    assert ctypes.sizeof(sj.sj.Stats) == 8 * 4 + 4 * 2 + 4 * 4 + 4 + 4
    assert sj.load_library().sj_abi_version() == 5


def test_defaults(sj):
    o = sj.sj.join_opts()
    assert (o.unicomp, o.include_self, o.batch_capacity_pairs, o.min_batches, o.n_streams,
            o.result_on_host, o.use_masks, o.lanes_per_query) == (1, 1, 1 << 28, 3, 3, 0, 1, 0)


def test_argument_errors_before_cuda(sj):
    with pytest.raises(sj.SJError) as e:
        sj.build_index(np.zeros((10, 7)), 1.0)
    assert e.value.name == "SJ_ERR_DIM"
    with pytest.raises(sj.SJError) as e:
        sj.build_index(np.zeros((10, 1)), 1.0)
    assert e.value.name == "SJ_ERR_DIM"
    for bad in (0.0, -1.0, float("nan"), float("inf"), 1e-200):
        with pytest.raises(sj.SJError) as e:
            sj.build_index(np.zeros((10, 2)), bad)
        assert e.value.name == "SJ_ERR_ARG"
    with pytest.raises(sj.SJError) as e:
        sj.build_index(np.zeros((0, 2)), 1.0)
    assert e.value.name == "SJ_ERR_ARG"


def test_null_handles_are_safe(sj):
    L = sj.load_library()
    L.sj_free_result(None)
    L.sj_free_index(None)
    st = L.sj_self_join(None, None, ctypes.byref(ctypes.c_void_p()))
    assert sj.sj.STATUS[st] == "SJ_ERR_STATE"


def test_planner_min_batches_and_capacity(sj):
    """at least 3 batches; S.264: est 1e6 pairs with capacity 1e5 -> ~10 batches
    (here capacity/(1+margin) is the per-batch target)."""
    cuts, tot = sj.plan_batches(np.full(100, 10, np.uint32), 10, 0, 1000, 1 << 28, 3)
    assert len(cuts) - 1 == 3 and cuts[0] == 0 and cuts[-1] == 1000 and tot == 10_000
    cuts, tot = sj.plan_batches(np.full(1000, 1000, np.uint32), 1, 0, 1000, 100_000, 3, margin=0.0)
    assert tot == 1_000_000 and len(cuts) - 1 == 10
    assert np.all(np.diff(cuts.astype(np.int64)) > 0)


def test_planner_skewed_and_tiny(sj):
    c = np.zeros(200, np.uint32)
    c[50] = 100000      # one hot sample bucket
    cuts, tot = sj.plan_batches(c, 50, 0, 10_000, 1_000_000, 3)
    assert cuts[0] == 0 and cuts[-1] == 10_000 and np.all(np.diff(cuts.astype(np.int64)) > 0)
    assert len(cuts) - 1 >= 5   # the hot bucket (5e6 est) is split to respect the capacity
    cuts, _ = sj.plan_batches(np.array([1], np.uint32), 1, 0, 1, 1 << 28, 3)
    assert cuts.tolist() == [0, 1]      # one query cannot make 3 batches
    cuts, _ = sj.plan_batches(np.array([], np.uint32), 1, 5, 5, 1 << 28, 3)
    assert cuts.tolist() == [5, 5]
