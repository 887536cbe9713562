#!/usr/bin/env python3
"""Generate tests/golden/*.json by running the UNMODIFIED reference library.

The reference (/root/reference/proj/src, compiled by oracle/Makefile into
oracle/_ref/libtrussdec_ref.so) is executed here, in the build container; its outputs
are committed so the GPU box (which has no /root/reference) can check against them.

  fixtures.json : the reference tests' own graphs (tests/helpers.hpp fixtures,
                  closed forms, the 200-graph acceptance suite of acceptance.cpp:43-52)
                  with the reference's truss / support / nsl / barriers.
  configs.json  : BASELINE configs C1..C5 built by the repo generator (graphgen) with
                  sha256 pins of the CSR and of the reference's truss / support arrays,
                  plus nsl, t_max, k-class sizes and triangle counts.

Usage: python tests/golden/make_golden.py fixtures
       python tests/golden/make_golden.py configs 1 2 3 4 [5]   (C3 ~5 min, C5 hours)
       python tests/golden/make_golden.py configs-kcore 5
           same record, but the reference runs on its own preprocessed graph
           (kcore_parallel -> coreness_order -> reorder, trussdec.cpp:92-97) and the
           per-edge truss / support are mapped back to the input's edge ids by (u,v).
           Trussness, support and nsl are invariant under vertex relabelling, so the
           record is the same; the reordered graph peels far faster on a CPU.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import Csr, Reference  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def suite_recipes():
    """acceptance.cpp:43-52: 100 seeds x (ER(n,p,s), RMAT(4+s%5, 8, s))."""
    out = []
    for s in range(1, 101):
        n = 4 + (s * 97) % 253
        p = 0.02 + 0.48 * float((s * 31) % 100) / 99.0
        out.append({"name": f"suite_er_{s}", "kind": "er", "n": n, "p": p, "seed": s})
        out.append({"name": f"suite_rmat_{s}", "kind": "rmat", "scale": 4 + s % 5, "ef": 8, "seed": s})
    return out


def named_recipes():
    r = []
    for n in range(3, 9):
        r.append({"name": f"K{n}", "kind": "pairs", "pairs": [[u, v] for u in range(n) for v in range(u + 1, n)]})
    for n in range(4, 17):
        r.append({"name": f"C{n}", "kind": "pairs", "pairs": [[u, (u + 1) % n] for u in range(n)]})
    for k in range(1, 9):
        r.append({"name": f"star{k}", "kind": "pairs", "pairs": [[0, v] for v in range(1, k + 1)]})
    r.append({"name": "triangle_pendant", "kind": "pairs", "pairs": [[0, 1], [0, 2], [1, 2], [0, 3]]})
    r.append({"name": "path3", "kind": "pairs", "pairs": [[0, 1], [1, 2]]})
    r.append({"name": "single_edge", "kind": "pairs", "pairs": [[0, 1]]})
    r.append({"name": "two_triangles", "kind": "pairs", "pairs": [[0, 1], [0, 2], [1, 2], [1, 3], [2, 3]]})
    r.append({"name": "two_diamond", "kind": "pairs", "pairs": [[0, 1], [0, 2], [0, 3], [1, 2], [2, 3], [4, 5], [4, 6],
                                                                 [4, 7], [5, 6], [6, 7], [3, 4], [1, 7]]})
    r.append({"name": "K33", "kind": "pairs", "pairs": [[a, b] for a in range(3) for b in range(3, 6)]})
    r.append({"name": "labels_sparse", "kind": "pairs", "pairs": [[10, 11], [10, 12], [11, 12], [20, 21], [20, 22],
                                                                   [21, 22], [12, 20]]})
    for n, p, s in [(100, 0.15, 2), (140, 0.1, 17), (80, 0.2, 7), (120, 0.12, 3), (150, 0.08, 8), (200, 0.1, 5),
                    (130, 0.1, 21), (100, 0.12, 5), (90, 0.12, 6), (256, 0.5, 11)]:
        r.append({"name": f"er_{n}_{p}_{s}", "kind": "er", "n": n, "p": p, "seed": s})
    for sc, ef, s in [(8, 8, 2), (10, 16, 1), (12, 16, 3), (14, 16, 1)]:
        r.append({"name": f"rmat_{sc}_{ef}_{s}", "kind": "rmat", "scale": sc, "ef": ef, "seed": s})
    return r


def make_graph(R: Reference, rec) -> Csr:
    if rec["kind"] == "er":
        return R.make_graph(0, rec["n"], rec["p"], rec["seed"])
    if rec["kind"] == "rmat":
        return R.make_graph(1, rec["scale"], rec["ef"], rec["seed"])
    return R.make_graph(2, 0, 0.0, 0, pairs=rec["pairs"])


def fixtures():
    R = Reference()
    out = []
    for rec in named_recipes() + suite_recipes():
        g = make_graph(R, rec)
        d = R.truss_parallel(g, 4)
        sup = R.support_am4(g, 2)
        tri = R.triangle_count(g, 2)
        ent = {"name": rec["name"], "recipe": rec}
        ent.update({"n": g.n, "m": g.m, "csr_sha": sha(g.offsets) + sha(g.neighbors),
                    "nsl": d.nsl, "barriers": d.barriers, "triangles": tri,
                    "t_max": int(d.truss.max()) if g.m else 0})
        if g.m <= 20000 and not rec["name"].startswith("suite_"):
            ent["truss"] = d.truss.tolist()
            ent["support"] = sup.tolist()
        ent["truss_sha"] = sha(d.truss)
        ent["support_sha"] = sha(sup)
        if g.n <= 512 and g.m:
            assert (R.truss_oracle(g) == d.truss).all(), rec["name"]
        out.append(ent)
    with open(os.path.join(HERE, "fixtures.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py (reference library oracle/_ref)",
                   "fixtures": out}, f, separators=(",", ":"))
    print(f"fixtures.json: {len(out)} graphs")


def edge_keys(off, nb) -> np.ndarray:
    """u<<32|v for every edge u<v in reference edge-id order (graph.cpp:86-99: ascending (u,v))."""
    n = len(off) - 1
    deg = np.diff(off)
    src = np.repeat(np.arange(n, dtype=np.uint32), deg)
    keep = nb.view(np.uint32) > src
    k = src[keep].astype(np.uint64) << np.uint64(32)
    del src
    k |= nb[keep].astype(np.uint64)
    return k


def mapped_back(R: Reference, g: Csr, workers: int):
    """Reference pipeline on the reordered graph; truss/support returned in g's edge-id order."""
    t0 = time.time()
    core, cmax, perm = R.kcore_order(g, workers)
    r = R.reorder(g, perm)
    t1 = time.time()
    print(f"  kcore+reorder {t1 - t0:.1f}s c_max={cmax}", flush=True)
    d = R.truss_parallel(r, workers)
    t2 = time.time()
    print(f"  truss_parallel {t2 - t1:.1f}s {d.times}", flush=True)
    sup_r = R.support_am4(r, workers)
    kr = edge_keys(r.offsets, r.neighbors)
    del r
    ko = edge_keys(g.offsets, g.neighbors)
    p = perm.astype(np.uint64)
    a = p[(ko >> np.uint64(32)).astype(np.int64)]
    b = p[(ko & np.uint64(0xFFFFFFFF)).astype(np.int64)]
    del ko
    key = (np.minimum(a, b) << np.uint64(32)) | np.maximum(a, b)
    del a, b
    idx = np.searchsorted(kr, key)
    assert (kr[idx] == key).all()
    del kr, key
    truss = d.truss[idx]
    sup = sup_r[idx]
    d.times["kcore_reorder"] = t1 - t0
    return d, truss, sup


def configs(ids, kcore=False):
    from paper_1707_02000_b200 import graphgen
    R = Reference()
    path = os.path.join(HERE, "configs.json")
    doc = json.load(open(path)) if os.path.exists(path) else {"configs": {}}
    for c in ids:
        t0 = time.time()
        n, m, off, nb = graphgen.config(c)
        g = Csr(n, m, off, nb)
        tg = time.time() - t0
        workers = int(os.environ.get("TDG_GOLDEN_WORKERS", os.cpu_count() or 8))
        if kcore:
            d, truss, sup = mapped_back(R, g, workers)
            d.truss = truss
        else:
            d = R.truss_parallel(g, workers)
            sup = R.support_am4(g, workers)
        vals, cnt = np.unique(d.truss, return_counts=True)
        doc["configs"][str(c)] = {
            "name": graphgen.CONFIG_NAMES[c], "n": n, "m": m,
            "offsets_sha": sha(off), "neighbors_sha": sha(nb),
            "truss_sha": sha(d.truss), "support_sha": sha(sup),
            "nsl": d.nsl, "sublevels": int(sum(d.nsl)), "barriers": d.barriers,
            "t_max": int(d.truss.max()), "kclass_sizes": {int(v): int(k) for v, k in zip(vals, cnt)},
            "triangles": int(sup.astype(np.uint64).sum() // 3),
            "sum_tau_minus_1": int(d.truss.astype(np.uint64).sum() - m),
            "ref_times_s": d.times, "ref_workers": workers, "gen_s": tg,
            "ref_pipeline": "kcore->coreness_order->reorder, mapped back" if kcore else "input order",
        }
        json.dump(doc, open(path, "w"), indent=1)
        print(f"C{c}: n={n} m={m} t_max={int(d.truss.max())} sublevels={sum(d.nsl)} ({time.time()-t0:.1f}s)")


if __name__ == "__main__":
    if sys.argv[1] == "fixtures":
        fixtures()
    else:
        configs([int(x) for x in sys.argv[2:]], kcore=sys.argv[1] == "configs-kcore")
