"""Driver for compute-sanitizer runs (memcheck / racecheck / synccheck, one tool per GPU
call): every golden fixture graph through tdg_truss (+ support), the reference tests'
hand-built frontier states through tdg_scan / tdg_process_sublevel, the edge-list parser,
and (unless --no-c1) BASELINE config 1 — each checked against the committed goldens, so a
sanitizer run is also a parity run. No torch import (keeps the sanitized process small).

Usage: compute-sanitizer --tool memcheck --error-exitcode 99 python scripts/sanitize.py [--no-c1] [--max N]
"""
import argparse
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import build_fixture, load_configs, load_fixtures, sha  # noqa: E402

from oracle import Oracle  # noqa: E402
from paper_1707_02000_b200 import graphgen, trussdec  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--no-c1", action="store_true")
    ap.add_argument("--max", type=int, default=0, help="only the first N fixtures")
    a = ap.parse_args()
    O = Oracle()
    ctx = trussdec.Context(0)
    fx = load_fixtures()
    if a.max:
        fx = fx[: a.max]
    bad = 0
    for rec in fx:
        g = build_fixture(O, rec)
        cg = trussdec.CsrGraph.from_arrays(g.offsets, g.neighbors, g.labels)
        truss, nsl, sup, _ = ctx.truss(cg, want_support=True)
        ok = sha(truss.astype(np.uint32)) == rec["truss_sha"] and nsl == rec["nsl"] and \
            sha(sup.astype(np.uint32)) == rec["support_sha"]
        bad += 0 if ok else 1
    # step functions on hand-built states (tests/test_truss_parallel.cpp:25-105): K4
    k4 = O.complete_graph(4)
    cg = trussdec.CsrGraph.from_arrays(k4.offsets, k4.neighbors)
    tg = trussdec.build_truss_graph(cg)
    s = trussdec.support_am4(tg).copy()
    f = trussdec.LevelFrontier(tg.m())
    trussdec.scan(s, 2, f)
    bad += 0 if f.curr_size == 6 else 1
    trussdec.process_sublevel(f, tg, s, 2, trussdec.MarkScratchPool(1, tg.n()))
    bad += 0 if (s == 2).all() and f.processed.sum() == 6 else 1
    # edge-list parser
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "g.txt")
        with open(p, "w") as fh:
            fh.write("# c\n0 1\n 1\t2 \n\n2 0\n" * 1000)
        bad += 0 if trussdec.read_edge_list(p).shape == (3000, 2) else 1
    n_cases = len(fx) + 3
    if not a.no_c1:
        gold = load_configs().get("1")
        n, m, off, nb = graphgen.config(1)
        truss, nsl, _, _ = ctx.truss(trussdec.CsrGraph(n, m, off, nb))
        bad += 0 if (gold and sha(truss.astype(np.uint32)) == gold["truss_sha"] and nsl == gold["nsl"]) else 1
        n_cases += 1
    ctx.close()
    print(f"sanitize driver: {n_cases} cases, {bad} mismatches")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
