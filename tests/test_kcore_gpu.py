"""GPU: vertex ordering before the path — kcore_parallel,
coreness_order and reorder against the reference library (oracle/_ref), including the
reference tests' known answers (tests/test_kcore.cpp, python/test_smoke.py)."""
import numpy as np
import pytest

from helpers import build_fixture, gpu_graph, load_fixtures

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def td():
    from paper_1707_02000_b200 import trussdec
    return trussdec


def test_coreness_known_answer(td, oracle):
    """python/test_smoke.py:27-32: triangle + pendant -> cores [2, 2, 2, 1]."""
    g = gpu_graph(oracle.canonicalize([(0, 1), (0, 2), (1, 2), (2, 3)]))
    r = td.kcore_parallel(g)
    assert r.core.tolist() == [2, 2, 2, 1] and r.c_max == 2


def test_kcore_closed_forms(td, oracle):
    for n in range(2, 9):
        r = td.kcore_parallel(gpu_graph(oracle.complete_graph(n)))
        assert (r.core == n - 1).all() and r.c_max == n - 1
    assert (td.kcore_parallel(gpu_graph(oracle.cycle_graph(7))).core == 2).all()
    assert (td.kcore_parallel(gpu_graph(oracle.star_graph(5))).core == 1).all()


@pytest.mark.parametrize("rec", load_fixtures()[::3], ids=lambda r: r["name"])
def test_kcore_order_reorder_match_reference(td, oracle, ref, rec):
    c = build_fixture(oracle, rec)
    g = gpu_graph(c)
    core, cmax, perm = ref.kcore_order(c, 4)
    r = td.kcore_parallel(g)
    assert (r.core == core).all() and r.c_max == cmax
    p = td.coreness_order(r)
    assert (p == perm).all()
    if c.n:
        g2 = td.reorder(g, p)
        c2 = ref.reorder(c, perm)
        assert (g2.offsets == c2.offsets).all() and (g2.neighbors == c2.neighbors).all()


def test_reorder_preserves_truss_histogram(td, oracle):
    """python/test_smoke.py:30-33 and acceptance.cpp:126-138: kcore order keeps the truss
    histogram and reduces sum d+^2 on RMAT."""
    g = gpu_graph(oracle.rmat_graph(12, 16, 2))
    r = td.reorder(g, td.coreness_order(td.kcore_parallel(g)))
    a, b = td.truss_parallel(g).result, td.truss_parallel(r).result
    assert a.kclass_sizes == b.kclass_sizes
    assert td.stats(r).sum_dplus_sq < td.stats(g).sum_dplus_sq


def test_reorder_rejects_non_bijection(td, oracle):
    g = gpu_graph(oracle.complete_graph(4))
    with pytest.raises(ValueError):
        td.reorder(g, np.array([0, 0, 1, 2], np.uint32))
