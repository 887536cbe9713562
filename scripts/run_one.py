"""Run decompositions of a BASELINE config through the C-ABI (profiling / A-B driver, no
torch): prints per-run phase times and whether truss + nsl match the committed golden."""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1707_02000_b200 import _lib, graphgen, trussdec  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "configs.json")))["configs"].get(str(cfg), {})
n, m, off, nb = graphgen.config(cfg)
ctx = trussdec.Context(0)
g = trussdec.CsrGraph(n, m, off, nb)
for _ in range(reps):
    t0 = time.time()
    truss, nsl, _, t = ctx.truss(g)
    ok = hashlib.sha256(np.ascontiguousarray(truss, np.uint32).tobytes()).hexdigest() == gold.get("truss_sha") \
        and nsl == gold.get("nsl")
    keep = ("build_ms", "support_ms", "peel_ms", "scan_ms", "process_ms", "compact_ms", "rebuild_ms", "table_rebuilds", "total_ms", "probes",
            "support_probes", "sublevels")
    print(f"C{cfg} m={m} wall={time.time()-t0:.3f}s parity={'ok' if ok else 'FAIL'} lib={os.path.relpath(_lib.TDG_SO, ROOT)}",
          {k: round(v, 2) if isinstance(v, float) else v for k, v in t.items() if k in keep}, flush=True)
