"""Decompose an RMAT graph (scale, seed, permute 0/1) through the C-ABI and print phase times
and the sha256 of the trussness array (A/B driver: filter word choice on clustered vertex ids;
select the library with TDG_SO)."""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1707_02000_b200 import _lib, graphgen, trussdec  # noqa: E402

scale, seed, permute = int(sys.argv[1]), int(sys.argv[2]), bool(int(sys.argv[3]))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
n, m, off, nb = graphgen.rmat(scale, 16, seed, permute=permute)
ctx = trussdec.Context(0)
g = trussdec.CsrGraph(n, m, off, nb)
for _ in range(reps):
    truss, nsl, _, t = ctx.truss(g)
    sha = hashlib.sha256(np.ascontiguousarray(truss, np.uint32).tobytes()).hexdigest()[:16]
    print(f"rmat{scale} seed{seed} permute={int(permute)} m={m} lib={os.path.relpath(_lib.TDG_SO, ROOT)} truss_sha={sha} "
          f"sublevels={sum(nsl)}", {k: round(v, 1) for k, v in t.items() if k in ("build_ms", "support_ms", "peel_ms", "total_ms")},
          flush=True)
