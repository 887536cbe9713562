"""GPU: ingest — canonicalize (graph.cpp:19-71) on the GPU against the
reference library's canonicalize on the same raw streams (tests/test_graph.cpp semantics:
first-appearance ids, loops dropped, duplicates and both orientations merged)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def td():
    from paper_1707_02000_b200 import trussdec
    return trussdec


def _same(g, r, labels_expected=None):
    assert (g.n, g.m) == (r.n, r.m)
    assert (g.offsets == r.offsets).all() and (g.neighbors == r.neighbors).all()


def test_first_appearance_labels(td):
    g = td.canonicalize([(10, 11), (11, 10), (10, 12), (12, 12), (11, 12), (7, 10)])
    assert g.labels.tolist() == [10, 11, 12, 7]
    assert (g.n, g.m) == (4, 4)
    assert g.offsets.tolist() == [0, 3, 5, 7, 8]
    assert g.neighbors.tolist() == [1, 2, 3, 0, 2, 0, 1, 0]


def test_empty_and_loop_only(td):
    g = td.canonicalize(np.zeros((0, 2), np.uint64))
    assert (g.n, g.m) == (0, 0)
    g = td.canonicalize([(5, 5), (6, 6)])
    assert (g.n, g.m) == (2, 0) and g.labels.tolist() == [5, 6]


@pytest.mark.parametrize("seed", range(6))
def test_random_streams_match_reference(td, ref, oracle, seed):
    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 5000))
    span = int(rng.choice([8, 300, 1 << 40]))
    pairs = rng.integers(0, span, size=(k, 2), dtype=np.int64)
    g = td.canonicalize(pairs.astype(np.uint64))
    r = ref.make_graph(2, 0, 0.0, 0, pairs=pairs)
    _same(g, r)
    o = oracle.canonicalize(pairs.astype(np.uint64))
    assert (g.labels == o.labels).all()


def test_generator_streams(td, ref, oracle):
    for scale, ef, s in [(8, 8, 1), (10, 16, 3)]:
        raw = oracle.generate_rmat(scale, ef, s)
        g = td.canonicalize(raw)
        _same(g, ref.make_graph(1, scale, ef, s))
    raw = oracle.generate_er(300, 0.05, 9)
    _same(td.canonicalize(raw), ref.make_graph(0, 300, 0.05, 9))
