"""GPU: maximal k-trusses against the reference's ktruss_subgraphs
(truss_serial.cpp:176-210), run from the reference library (oracle/_ref)."""
import pytest

from helpers import build_fixture, gpu_graph, load_fixtures

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def td():
    from paper_1707_02000_b200 import trussdec
    return trussdec


def test_two_diamond_two_3_trusses(td, oracle):
    """test_truss_serial.cpp:62-72: two maximal 3-trusses."""
    g = gpu_graph(oracle.canonicalize([(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (4, 5), (4, 6), (4, 7), (5, 6),
                                       (6, 7), (3, 4), (1, 7)]))
    res = td.truss_parallel(g).result
    comps = td.ktruss_subgraphs(g, res, 3)
    assert len(comps) == 2 and sorted(len(c) for c in comps) == [5, 5]
    assert len(td.ktruss_subgraphs(g, res, 2)) == 1


def test_labelled_components(td, oracle):
    """python/test_smoke.py:35-38: two disjoint triangles -> two 3-trusses; k > t_max raises."""
    g = gpu_graph(oracle.canonicalize([(10, 11), (10, 12), (11, 12), (20, 21), (20, 22), (21, 22)]))
    res = td.truss_parallel(g).result
    assert len(td.ktruss_subgraphs(g, res, 3)) == 2
    with pytest.raises(ValueError):
        td.ktruss_subgraphs(g, res, 9)
    with pytest.raises(ValueError):
        td.ktruss_subgraphs(g, res, 1)


@pytest.mark.parametrize("rec", [r for r in load_fixtures() if r["m"] > 0][::4], ids=lambda r: r["name"])
def test_ktruss_matches_reference(td, oracle, ref, rec):
    c = build_fixture(oracle, rec)
    g = gpu_graph(c)
    res = td.truss_parallel(g).result
    for k in sorted(k for k in {2, 3, res.t_max // 2, res.t_max} if 2 <= k <= res.t_max):
        assert td.ktruss_subgraphs(g, res, k) == ref.ktruss_subgraphs(c, res.truss, k), (rec["name"], k)
    with pytest.raises(ValueError):  # truss_serial.cpp:179-180 on both sides
        td.ktruss_subgraphs(g, res, res.t_max + 1)
    with pytest.raises(RuntimeError):
        ref.ktruss_subgraphs(c, res.truss, res.t_max + 1)
