"""CPU: the config generator (include/tdg_gen.h) — determinism, CSR invariants, and its
RMAT stream pinned to the reference's generate_rmat via the oracle restatement."""
import numpy as np
import pytest

from paper_1707_02000_b200 import graphgen


def check_csr(n, m, off, nb):
    assert off[0] == 0 and off[-1] == 2 * m and len(off) == n + 1
    assert (np.diff(off) >= 0).all()
    src = np.repeat(np.arange(n), np.diff(off))
    assert (src != nb).all()                                    # no loops
    key = src.astype(np.int64) * n + nb
    assert (np.diff(key) > 0).all()                             # sorted, no duplicates
    rev = np.sort(nb.astype(np.int64) * n + src)
    assert (rev == key).all()                                   # symmetric


def test_rmat_stream_matches_reference_generate_rmat(oracle):
    """Unpermuted generator output == the reference generate_rmat draws (generate.cpp:58-92)
    restated in oracle.c, deduped with ids kept."""
    for scale, ef, seed in [(6, 8, 1), (8, 8, 2), (10, 16, 3), (9, 4, 99)]:
        raw = oracle.generate_rmat(scale, ef, seed)
        n1, m1, o1, b1 = graphgen.rmat(scale, ef, seed, permute=False)
        n2, m2, o2, b2 = graphgen.from_pairs(raw.astype(np.int64), n_hint=1 << scale)
        assert (n1, m1) == (n2, m2)
        assert (o1 == o2).all() and (b1 == b2).all()


def test_permutation_rule(oracle):
    """Appendix B.2: Fisher-Yates j = rng() % (i+1) on the continuing stream."""
    scale, ef, seed = 7, 8, 5
    mt = oracle.mt64(seed, (1 << scale) * ef * scale + (1 << scale))
    pos = (1 << scale) * ef * scale
    p = list(range(1 << scale))
    for i in range((1 << scale) - 1, 0, -1):
        j = mt[pos] % (i + 1)
        pos += 1
        p[i], p[j] = p[j], p[i]
    raw = oracle.generate_rmat(scale, ef, seed)
    perm = np.array(p, np.int64)
    n2, m2, o2, b2 = graphgen.from_pairs(perm[raw.astype(np.int64)], n_hint=1 << scale)
    n1, m1, o1, b1 = graphgen.rmat(scale, ef, seed, permute=True)
    assert (o1 == o2).all() and (b1 == b2).all()


def test_c1_shape_and_determinism():
    n, m, off, nb = graphgen.config(1)
    assert (n, m) == (65536, 909956)  # SURVEY.md §1 flag 1: reference generator gives 909,956
    check_csr(n, m, off, nb)
    n2, m2, off2, nb2 = graphgen.config(1)
    assert (off == off2).all() and (nb == nb2).all()


def test_gnm_and_planted_small():
    n, m, off, nb = graphgen.gnm(1000, 5000, 7)
    assert m == 5000
    check_csr(n, m, off, nb)
    n, m, off, nb = graphgen.planted(2000, 4000, 5, 8, 20, 3)
    check_csr(n, m, off, nb)
    assert m >= 4000


def test_from_pairs_drops_loops_and_duplicates():
    n, m, off, nb = graphgen.from_pairs([(0, 1), (1, 0), (2, 2), (1, 2), (1, 2)], n_hint=4)
    assert (n, m) == (4, 2)
    assert off.tolist() == [0, 1, 3, 4, 4] and nb.tolist() == [1, 0, 2, 1]


def test_generator_errors():
    with pytest.raises(RuntimeError):
        graphgen.rmat(0)
    with pytest.raises(RuntimeError):
        graphgen.gnm(3, 10, 1)
