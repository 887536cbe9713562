"""GPU: both ways of choosing a key's filter word give the reference's results, and the build
picks hash mode exactly when vertex ids are clustered. An unpermuted RMAT graph (hubs and
their neighbours at low ids) must switch to hash mode; its permuted twin must stay in rank
mode; both must match the oracle's restatement of truss_parallel (truss_parallel.cpp:106-150)
bit for bit, truss and sub-level trace."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("permute,want_hashed", [(False, True), (True, False)])
def test_filter_mode_choice_and_parity(oracle, permute, want_hashed):
    from oracle import Csr
    from paper_1707_02000_b200 import graphgen, trussdec
    n, m, off, nb = graphgen.rmat(15, 16, 21, permute=permute)
    ctx = trussdec.Context(0)
    truss, nsl, _, _ = ctx.truss(trussdec.CsrGraph(n, m, off, nb))
    hashed, est = ctx.filter_mode()
    assert hashed == want_hashed, est
    assert (est > 0.08) == want_hashed
    ref = oracle.truss_pkt(Csr(n, m, np.ascontiguousarray(off, np.int64), np.ascontiguousarray(nb[: 2 * m], np.int32)))
    assert np.array_equal(np.asarray(truss, np.uint32), ref.truss)
    assert list(nsl) == ref.nsl
    ctx.close()
