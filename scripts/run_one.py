"""Run one decomposition of a BASELINE config through the C-ABI (profiling driver, no torch)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1707_02000_b200 import graphgen, trussdec  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
n, m, off, nb = graphgen.config(cfg)
ctx = trussdec.Context(0)
g = trussdec.CsrGraph(n, m, off, nb)
for _ in range(reps):
    t0 = time.time()
    truss, nsl, _, t = ctx.truss(g)
    print(f"C{cfg} m={m} wall={time.time()-t0:.3f}s", {k: round(v, 2) if isinstance(v, float) else v for k, v in t.items()})
