"""CPU: pin the C restatement (oracle/oracle.c) before trusting it.

Checked against (1) the golden fixtures produced by the reference library itself
(tests/golden/fixtures.json, made by tests/golden/make_golden.py from oracle/_ref), and
(2) the known answers in the reference's own tests (paths relative to
/root/reference/proj/tests).
"""
import numpy as np
import pytest

from helpers import build_fixture, load_fixtures, sha


def test_mt19937_64_known_answer(oracle):
    # std::mt19937_64 with the default seed 5489: the 10000th output (C++11 [rand.predef]).
    assert oracle.mt64(5489, 10000)[-1] == 9981545732273789042


@pytest.mark.parametrize("rec", load_fixtures(), ids=lambda r: r["name"])
def test_oracle_matches_reference_fixture(oracle, rec):
    g = build_fixture(oracle, rec)
    assert (g.n, g.m) == (rec["n"], rec["m"])
    assert sha(g.offsets) + sha(g.neighbors) == rec["csr_sha"]  # generators + canonicalize pinned
    r = oracle.truss_pkt(g)
    assert sha(r.truss) == rec["truss_sha"]
    assert sha(r.support) == rec["support_sha"]
    assert r.nsl == rec["nsl"]
    assert r.barriers == rec["barriers"]
    if "truss" in rec:
        assert r.truss.tolist() == rec["truss"]
    if g.m:
        assert int(r.support.astype(np.int64).sum()) == 3 * rec["triangles"]  # acceptance.cpp:100
        assert (oracle.truss_wc(g) == r.truss).all()                          # wc == pkt
        assert (r.truss <= r.support + 2).all()                               # test_truss_serial.cpp:90-96
        assert r.barriers == int(r.truss.max()) + 2 * sum(r.nsl)              # truss_parallel.hpp:37-39


def test_reference_known_answers(oracle):
    # test_triangle.cpp:13-22
    assert oracle.support_am4(oracle.complete_graph(3)).tolist() == [1, 1, 1]
    k4 = oracle.support_am4(oracle.complete_graph(4))
    assert k4.tolist() == [2] * 6 and k4.sum() == 12
    assert oracle.support_am4(oracle.canonicalize([(0, 1), (1, 2)])).tolist() == [0, 0]
    # test_triangle.cpp:58-60
    cnt, s = oracle.triangle_oracle(oracle.complete_graph(6))
    assert cnt == 20 and (s == 4).all()
    # test_truss_parallel.cpp:107-116 (K4 trace)
    r = oracle.truss_pkt(oracle.complete_graph(4))
    assert r.truss.tolist() == [4] * 6 and r.nsl == [0, 0, 1]
    assert r.barriers == 4 + 2 * 1
    # test_truss_parallel.cpp:118-126 / test_cli.cpp:82-86 (hist "2\t1\n3\t3\n")
    r = oracle.truss_pkt(oracle.canonicalize([(0, 1), (0, 2), (1, 2), (0, 3)]))
    assert sorted(r.truss.tolist()) == [2, 3, 3, 3]
    # test_truss_serial.cpp:62-68 (two diamonds)
    g = oracle.canonicalize([(0, 1), (0, 2), (0, 3), (1, 2), (2, 3), (4, 5), (4, 6), (4, 7), (5, 6), (6, 7),
                             (3, 4), (1, 7)])
    t = oracle.truss_pkt(g).truss
    assert (t == 2).sum() == 2 and (t == 3).sum() == 10
    # acceptance.cpp:109-124 closed forms
    for n in range(3, 9):
        assert (oracle.truss_pkt(oracle.complete_graph(n)).truss == n).all()
    for n in range(4, 17):
        assert (oracle.truss_pkt(oracle.cycle_graph(n)).truss == 2).all()
    for k in range(1, 9):
        assert (oracle.truss_pkt(oracle.star_graph(k)).truss == 2).all()


def test_oracle_step_functions_reference_states(oracle):
    """Hand-built frontier states of test_truss_parallel.cpp:25-105."""
    k3 = oracle.complete_graph(3)
    # lone curr edge decrements both peers (:51-70)
    s = np.array([0, 1, 1], np.uint32)
    curr = np.array([0, 0, 0], np.uint32)
    in_curr = np.array([1, 0, 0], np.uint8)
    in_next = np.zeros(3, np.uint8)
    proc = np.zeros(3, np.uint8)
    nxt = np.zeros(3, np.uint32)
    ns = oracle.process_sublevel(k3, s, 0, curr, 1, in_curr, in_next, proc, nxt)
    assert s.tolist() == [0, 0, 0] and sorted(nxt[:ns].tolist()) == [1, 2]
    assert in_next.tolist() == [0, 1, 1] and proc[0] == 1 and in_curr[0] == 0
    # ownership rule: the third edge is decremented once (:72-88)
    s = np.array([0, 0, 1], np.uint32)
    curr = np.array([0, 1, 0], np.uint32)
    in_curr = np.array([1, 1, 0], np.uint8)
    in_next = np.zeros(3, np.uint8)
    proc = np.zeros(3, np.uint8)
    ns = oracle.process_sublevel(k3, s, 0, curr, 2, in_curr, in_next, proc, nxt)
    assert s[2] == 0 and ns == 1 and nxt[0] == 2
    # scan on K4 (:25-36)
    k4 = oracle.complete_graph(4)
    s = oracle.support_am4(k4)
    in_curr = np.zeros(6, np.uint8)
    curr = np.zeros(6, np.uint32)
    assert oracle.scan(s, 0, np.zeros(6, np.uint8), in_curr, curr) == 0
    assert oracle.scan(s, 2, np.zeros(6, np.uint8), in_curr, curr) == 6
    assert sorted(curr.tolist()) == list(range(6)) and (in_curr == 1).all()


def test_oracle_build_truss_graph_matches_reference(oracle, ref):
    for rec in load_fixtures()[:60]:
        g = build_fixture(oracle, rec)
        eo, eid, el = oracle.build_truss_graph(g)
        reo, reid, rel = ref.build_truss_graph(g)
        assert (eo == reo).all() and (eid == reid).all() and (el == rel).all()


def test_oracle_matches_reference_library_directly(oracle, ref):
    g = oracle.rmat_graph(12, 16, 4)
    r = oracle.truss_pkt(g)
    d = ref.truss_parallel(g, 4)
    assert (r.truss == d.truss).all() and r.nsl == d.nsl and r.barriers == d.barriers
    assert (ref.support_am4(g, 3) == r.support).all()
