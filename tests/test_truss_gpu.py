"""GPU parity: the CUDA path (through the C-ABI) against the reference's golden outputs
and the oracle, mirroring the reference's own tests (paths relative to
/root/reference/proj/tests). Integer work: every comparison is bit-exact."""
import numpy as np
import pytest

from helpers import build_fixture, gpu_graph, load_fixtures, sha

pytestmark = pytest.mark.gpu

FIXTURES = load_fixtures()


@pytest.fixture(scope="module")
def td():
    from paper_1707_02000_b200 import trussdec
    return trussdec


@pytest.mark.parametrize("rec", FIXTURES, ids=lambda r: r["name"])
def test_truss_parallel_matches_reference(td, oracle, rec):
    """acceptance.cpp criteria 1-4, 7: truss, nsl, barriers identical to the reference."""
    g = gpu_graph(build_fixture(oracle, rec))
    dec = td.truss_parallel(g, 4)
    assert sha(dec.result.truss) == rec["truss_sha"]
    assert dec.trace.nsl == rec["nsl"]
    assert dec.trace.barriers == rec["barriers"]
    if g.m:
        assert dec.trace.barriers == dec.trace.expected_barriers(dec.result.t_max)
        assert dec.gpu["triangles"] == rec["triangles"]


@pytest.mark.parametrize("rec", FIXTURES, ids=lambda r: r["name"])
def test_support_matches_reference(td, oracle, rec):
    """acceptance.cpp criterion 2 / test_triangle.cpp: am4 == oracle, sum = 3|T|."""
    g = gpu_graph(build_fixture(oracle, rec))
    s = td.support_am4(g, 4)
    assert sha(s) == rec["support_sha"]
    if "support" in rec:
        assert s.tolist() == rec["support"]


def test_build_truss_graph_matches_oracle(td, oracle):
    """graph.cpp:73-101 layout: eo, eid (both mirror slots), el in ascending (u,v)."""
    for rec in FIXTURES[:80] + [r for r in FIXTURES if r["name"].startswith("rmat_")]:
        c = build_fixture(oracle, rec)
        tg = td.build_truss_graph(gpu_graph(c))
        eo, eid, el = oracle.build_truss_graph(c)
        assert (tg.eo == eo).all() and (tg.eid == eid).all() and (tg.el == el).all(), rec["name"]


def test_stats_match_oracle(td, oracle):
    for rec in FIXTURES[:40]:
        c = build_fixture(oracle, rec)
        if c.m == 0:
            continue
        st = td.stats(gpu_graph(c))
        o = oracle.stats(c)
        assert (st.d_max, st.sum_deg_sq, st.sum_dplus_sq, st.wedge_count) == \
               (o["d_max"], o["sum_deg_sq"], o["sum_dplus_sq"], o["wedge_count"])
        assert (st.deg_sum_dplus_sq, st.deg_s1) == (o["deg_order_sum_dplus_sq"], o["deg_order_s1"])


def test_closed_forms(td, oracle):
    """acceptance.cpp:109-124 and test_truss_serial.cpp:43-48."""
    for n in range(3, 9):
        assert (td.truss_parallel(gpu_graph(oracle.complete_graph(n))).result.truss == n).all()
    for n in range(4, 17):
        assert (td.truss_parallel(gpu_graph(oracle.cycle_graph(n))).result.truss == 2).all()
    for k in range(1, 9):
        assert (td.truss_parallel(gpu_graph(oracle.star_graph(k))).result.truss == 2).all()


def test_k4_trace(td, oracle):
    """test_truss_parallel.cpp:107-116."""
    dec = td.truss_parallel(gpu_graph(oracle.complete_graph(4)), 4)
    assert dec.result.truss.tolist() == [4] * 6
    assert dec.trace.nsl == [0, 0, 1]
    assert dec.trace.barriers == dec.trace.expected_barriers(dec.result.t_max)


def test_triangle_plus_pendant(td, oracle):
    """test_truss_parallel.cpp:118-126, test_cli.cpp:82-86 (hist 2:1, 3:3)."""
    dec = td.truss_parallel(gpu_graph(oracle.canonicalize([(0, 1), (0, 2), (1, 2), (0, 3)])), 2)
    assert dec.result.kclass_sizes == {2: 1, 3: 3}
    assert dec.result.t_max == 3


def test_two_diamond(td, oracle):
    """test_truss_serial.cpp:62-72."""
    g = oracle.canonicalize([(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (4, 5), (4, 6), (4, 7), (5, 6), (6, 7),
                             (3, 4), (1, 7)])
    dec = td.truss_parallel(gpu_graph(g))
    assert dec.result.kclass_sizes == {2: 2, 3: 10}


def test_empty_and_edgeless_graphs(td):
    """m == 0: empty result, one barrier (truss_parallel.cpp:113, loop never runs)."""
    for n in (0, 1, 5):
        g = td.CsrGraph.from_arrays(np.zeros(n + 1, np.int64), np.zeros(0, np.int32))
        dec = td.truss_parallel(g)
        assert len(dec.result.truss) == 0 and dec.trace.nsl == [] and dec.trace.barriers == 1
        assert len(td.support_am4(g)) == 0


def test_isolated_vertices_and_ragged_ids(td, oracle):
    """Isolated vertices kept: CSR with gaps in the id space."""
    pairs = [(0, 5), (5, 9), (0, 9), (9, 20), (20, 21), (21, 9), (20, 5)]
    from paper_1707_02000_b200 import graphgen
    n, m, off, nb = graphgen.from_pairs(pairs, n_hint=32)
    from oracle import Csr
    c = Csr(n, m, off, nb)
    dec = td.truss_parallel(gpu_graph(c))
    r = oracle.truss_pkt(c)
    assert (dec.result.truss == r.truss).all() and dec.trace.nsl == r.nsl


def test_scan_step(td, oracle):
    """test_truss_parallel.cpp:25-49."""
    g = gpu_graph(oracle.complete_graph(4))
    s = td.support_am4(g)
    f = td.LevelFrontier(6)
    td.scan(s, 0, f)
    assert f.curr_size == 0
    td.scan(s, 2, f)
    assert sorted(f.curr[: f.curr_size].tolist()) == list(range(6))
    assert (f.in_curr == 1).all()
    c = oracle.er_graph(120, 0.12, 3)
    s = td.support_am4(gpu_graph(c))
    f = td.LevelFrontier(c.m)
    td.scan(s, 1, f)
    assert sorted(f.curr[: f.curr_size].tolist()) == np.nonzero(s == 1)[0].tolist()


def test_process_sublevel_lone_edge(td, oracle):
    """test_truss_parallel.cpp:51-70 (hand-built state, level 0 with a live triangle)."""
    g = gpu_graph(oracle.complete_graph(3))
    s = np.array([0, 1, 1], np.uint32)
    f = td.LevelFrontier(3)
    f.curr[0] = 0
    f.curr_size = 1
    f.in_curr[0] = 1
    td.process_sublevel(f, g, s, 0, td.MarkScratchPool(2, 3), 2)
    assert s.tolist() == [0, 0, 0]
    assert sorted(f.next[: f.next_size].tolist()) == [1, 2]
    assert f.in_next[1] == 1 and f.in_next[2] == 1
    assert f.processed[0] == 1 and f.in_curr[0] == 0


def test_process_sublevel_ownership(td, oracle):
    """test_truss_parallel.cpp:72-88: the third edge is decremented exactly once."""
    g = gpu_graph(oracle.complete_graph(3))
    for _ in range(3):
        s = np.array([0, 0, 1], np.uint32)
        f = td.LevelFrontier(3)
        f.curr[0], f.curr[1] = 0, 1
        f.curr_size = 2
        f.in_curr[0] = f.in_curr[1] = 1
        td.process_sublevel(f, g, s, 0)
        assert s[2] == 0
        assert f.next_size == 1 and f.next[0] == 2


def test_process_sublevel_full_k4(td, oracle):
    """test_truss_parallel.cpp:90-105: no underflow, empty next."""
    g = gpu_graph(oracle.complete_graph(4))
    s = np.full(6, 2, np.uint32)
    f = td.LevelFrontier(6)
    f.curr[:6] = np.arange(6)
    f.in_curr[:] = 1
    f.curr_size = 6
    td.process_sublevel(f, g, s, 2)
    assert s.tolist() == [2] * 6 and f.next_size == 0 and (f.processed == 1).all()


def test_manual_frontier_loop(td, oracle):
    """test_truss_parallel.cpp:150-184: every edge enters curr once; s + 2 == truss."""
    c = oracle.er_graph(80, 0.2, 7)
    g = gpu_graph(c)
    m = c.m
    s = td.support_am4(g).copy()
    expect = oracle.truss_wc(c)
    f = td.LevelFrontier(m)
    entered = np.zeros(m, np.int64)
    total = 0
    while f.todo > 0:
        td.scan(s, f.level, f)
        while f.curr_size > 0:
            cs = f.curr_size
            total += cs
            f.todo -= cs
            np.add.at(entered, f.curr[:cs], 1)
            f.next_size = 0
            td.process_sublevel(f, g, s, f.level)
            f.curr, f.next = f.next, f.curr
            f.in_curr, f.in_next = f.in_next, f.in_curr
            f.curr_size = f.next_size
            f.next_size = 0
        f.level += 1
    assert total == m and (entered == 1).all() and (f.processed == 1).all()
    assert ((s + 2) == expect).all()


def test_vertex_order_invariance(td, oracle):
    """Trussness per (labelled) edge and nsl are invariant to vertex relabelling."""
    c = oracle.rmat_graph(12, 16, 7)
    base = td.truss_parallel(gpu_graph(c))
    rng = np.random.default_rng(5)
    perm = rng.permutation(c.n)
    el = np.repeat(np.arange(c.n), np.diff(c.offsets))
    pairs = np.stack([perm[el], perm[c.neighbors]], 1)
    from paper_1707_02000_b200 import graphgen
    n, m, off, nb = graphgen.from_pairs(pairs, n_hint=c.n)
    dec = td.truss_parallel(td.CsrGraph.from_arrays(off, nb))
    assert dec.trace.nsl == base.trace.nsl
    assert dec.result.kclass_sizes == base.result.kclass_sizes
    # per-edge: map both through canonical labelled keys
    def keyed(offs, nbrs, truss, relabel):
        src = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
        up = src < nbrs
        u, v = relabel[src[up]], relabel[nbrs[up]]
        k = np.minimum(u, v).astype(np.int64) << 32 | np.maximum(u, v)
        return dict(zip(k.tolist(), truss.tolist()))
    ident = np.arange(c.n)
    a = keyed(c.offsets, c.neighbors, base.result.truss, perm)
    b = keyed(off, nb, dec.result.truss, ident)
    assert a == b


def test_repeated_calls_and_context_reuse(td, oracle):
    c = oracle.rmat_graph(10, 16, 1)
    ctx = td.Context(0)
    outs = [ctx.truss(gpu_graph(c))[0].copy() for _ in range(3)]
    small = oracle.complete_graph(5)
    assert (ctx.truss(gpu_graph(small))[0] == 5).all()  # smaller graph on grown buffers
    outs.append(ctx.truss(gpu_graph(c))[0])
    assert all((o == outs[0]).all() for o in outs)
    ctx.close()


def test_bad_input_raises(td):
    g = td.CsrGraph(3, 2, np.array([0, 1, 2, 3], np.int64), np.array([1, 0, 2, 1], np.int32))
    with pytest.raises(ValueError):
        td.truss_parallel(g)  # offsets[n] != 2m


@pytest.mark.parametrize("rec", FIXTURES[::3], ids=lambda r: r["name"])
def test_triangle_count_matches_reference(td, oracle, rec):
    """triangle.cpp:90-116 against the reference's own count."""
    assert td.triangle_count(gpu_graph(build_fixture(oracle, rec))) == rec["triangles"]


def test_triangle_count_closed_forms(td, oracle):
    """test_triangle.cpp:42-52: K5 has C(5,3) = 10 triangles, K3,3 none."""
    assert td.triangle_count(gpu_graph(oracle.complete_graph(5))) == 10
    k33 = oracle.canonicalize([(a, b) for a in range(3) for b in range(3, 6)])
    assert td.triangle_count(gpu_graph(k33)) == 0
