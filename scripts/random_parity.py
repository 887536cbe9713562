"""Randomized parity sweep (GPU box): seeded random graphs of several families — RMAT with
and without id permutation (rank / hash filter modes), G(n,m) at several densities, planted
cliques, unions of a hub clique with a sparse background — decomposed through the C-ABI and
compared bit for bit (truss, nsl, support) with the UNMODIFIED reference library
(oracle/_ref) on the same CSR. Prints one line per graph and a final tally.
Usage: python scripts/random_parity.py [count] [seed]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import Csr, Reference  # noqa: E402
from paper_1707_02000_b200 import graphgen, trussdec  # noqa: E402


def main():
    count = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
    R = Reference()
    ctx = trussdec.Context(0)
    threads = os.cpu_count() or 1
    bad = 0
    t_start = time.time()
    for i in range(count):
        fam = i % 5
        seed = int(rng.integers(1, 1 << 30))
        if fam == 0:
            sc = int(rng.integers(10, 18))
            n, m, off, nb = graphgen.rmat(sc, int(rng.integers(4, 24)), seed, permute=True)
            name = f"rmat{sc} permuted"
        elif fam == 1:
            sc = int(rng.integers(10, 17))
            n, m, off, nb = graphgen.rmat(sc, int(rng.integers(8, 32)), seed, permute=False)
            name = f"rmat{sc} unpermuted"
        elif fam == 2:
            n_ = int(rng.integers(1 << 10, 1 << 17))
            m_ = int(n_ * rng.uniform(1.0, 24.0))
            m_ = min(m_, n_ * (n_ - 1) // 4)
            n, m, off, nb = graphgen.gnm(n_, m_, seed)
            name = f"gnm n={n_}"
        elif fam == 3:
            n_ = int(rng.integers(1 << 12, 1 << 16))
            n, m, off, nb = graphgen.planted(n_, int(n_ * rng.uniform(2, 8)), int(rng.integers(5, 200)), 4,
                                             int(rng.integers(8, 200)), seed)
            name = f"planted n={n_}"
        else:  # a clique of k vertices (hub lists) inside a sparse random graph
            n_ = int(rng.integers(1 << 12, 1 << 15))
            k = int(rng.integers(200, 1200))
            r2 = np.random.default_rng(seed)
            bg = r2.integers(0, n_, size=(int(n_ * r2.uniform(2, 10)), 2), dtype=np.int64)
            cl = r2.choice(n_, size=k, replace=False).astype(np.int64)
            iu = np.triu_indices(k, 1)
            pairs = np.concatenate([bg, np.stack([cl[iu[0]], cl[iu[1]]], 1)])
            n, m, off, nb = graphgen.from_pairs(pairs, n_)
            name = f"clique{k}+sparse n={n_}"
        c = Csr(n, m, np.ascontiguousarray(off, np.int64), np.ascontiguousarray(nb[: 2 * m], np.int32))
        g = trussdec.CsrGraph(n, m, off, nb)
        truss, nsl, sup, _ = ctx.truss(g, want_support=True)
        hashed, est = ctx.filter_mode() if m else (False, 0.0)
        ref = R.truss_parallel(c, threads)
        sref = R.support_am4(c, threads)
        ok = bool(np.array_equal(np.asarray(truss, np.uint32), ref.truss) and list(nsl) == ref.nsl and
                  np.array_equal(np.asarray(sup, np.uint32), sref))
        bad += 0 if ok else 1
        print(f"{i:3d} {name:28s} seed={seed:10d} n={n:7d} m={m:9d} t_max={int(ref.truss.max()) if m else 0:4d} "
              f"sublevels={sum(ref.nsl):5d} filter={'hash' if hashed else 'rank'}({est:.3f}) {'ok' if ok else 'MISMATCH'}",
              flush=True)
    print(f"{count} graphs, {bad} mismatches, {time.time() - t_start:.0f} s")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
