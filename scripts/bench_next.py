#!/usr/bin/env python3
"""Measure the SURVEY §8(f) rows on one config: GPU (through the C-ABI, host buffers, wall
clock incl. copies) vs the reference library (oracle/_ref) on all host threads, with a
parity check of every output. One JSON line per row."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Csr, Reference  # noqa: E402
from paper_1707_02000_b200 import graphgen, trussdec  # noqa: E402


def timed(f, reps=1):
    best, out = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        out = f()
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return best, out


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    threads = os.cpu_count() or 1
    n, m, off, nb = graphgen.config(cfg)
    c = Csr(n, m, off, nb)
    g = trussdec.CsrGraph(n, m, off, nb)
    R = Reference()
    ctx = trussdec.default_context()
    ctx.truss(trussdec.CsrGraph.from_arrays([0, 1, 2], [1, 0]))  # warm the CUDA modules
    rows = []

    tg, cnt_g = timed(lambda: trussdec.triangle_count(g), 2)
    tr, cnt_r = timed(lambda: R.triangle_count(c, threads))
    rows.append({"row": "triangle_count (triangle.cpp:90-116)", "gpu_s": tg, "ref_s": tr, "equal": cnt_g == cnt_r,
                 "value": cnt_g})

    tg, kc = timed(lambda: trussdec.kcore_parallel(g), 2)
    tg2, perm = timed(lambda: trussdec.coreness_order(kc), 2)
    tg3, g2 = timed(lambda: trussdec.reorder(g, perm), 1)
    t0 = time.perf_counter()
    core_r, cmax_r, perm_r = R.kcore_order(c, threads)
    tr = time.perf_counter() - t0
    tr3, c2 = timed(lambda: R.reorder(c, perm_r))
    rows.append({"row": "kcore_parallel + coreness_order (kcore.cpp:68-138)", "gpu_s": tg + tg2, "ref_s": tr,
                 "equal": bool((kc.core == core_r).all() and kc.c_max == cmax_r and (perm == perm_r).all()),
                 "c_max": kc.c_max})
    rows.append({"row": "reorder (graph.cpp:103-133)", "gpu_s": tg3, "ref_s": tr3,
                 "equal": bool((g2.offsets == c2.offsets).all() and (g2.neighbors == c2.neighbors).all())})

    truss, _, _, _ = ctx.truss(g)
    res = trussdec.TrussnessResult(truss)
    res.finalize()
    k = max(2, res.t_max // 2)
    tg, comps_g = timed(lambda: trussdec.ktruss_subgraphs(g, res, k), 1)
    tr, comps_r = timed(lambda: R.ktruss_subgraphs(c, truss, k))
    rows.append({"row": f"ktruss_subgraphs k={k} (truss_serial.cpp:176-210)", "gpu_s": tg, "ref_s": tr,
                 "equal": comps_g == comps_r, "components": len(comps_g)})

    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(off))
    up = src < nb
    pairs = np.stack([src[up], nb[up].astype(np.int64)], 1)
    rng = np.random.default_rng(1)
    pairs = pairs[rng.permutation(len(pairs))]
    flip = rng.random(len(pairs)) < 0.5
    pairs[flip] = pairs[flip][:, ::-1]
    pairs = np.ascontiguousarray(pairs)
    tg, gc = timed(lambda: trussdec.canonicalize(pairs.astype(np.uint64)), 1)
    if m <= 70_000_000:
        tr, rc = timed(lambda: R.make_graph(2, 0, 0.0, 0, pairs=pairs))
        eq = bool(gc.n == rc.n and (gc.offsets == rc.offsets).all() and (gc.neighbors == rc.neighbors).all())
    else:
        tr, eq = None, None
    rows.append({"row": "canonicalize (graph.cpp:19-71), shuffled+flipped edge stream", "gpu_s": tg, "ref_s": tr,
                 "equal": eq})

    # sharded support pass: R shards one after another on this GPU; the shards'
    # partial supports must sum to the reference's support_am4, and the slowest shard shows the
    # work balance (ideal = full / R)
    t_full, s_full = timed(lambda: ctx.support(g)[0], 2)
    tr, s_ref = timed(lambda: R.support_am4(c, threads))
    for shards in (2, 8):
        ts, acc = [], np.zeros(m, np.uint64)
        for r_ in range(shards):
            t_, part = timed(lambda: ctx.support_shard(g, r_, shards)[1]["support_ms"], 1)
            ts.append(part)
            acc += ctx.support_shard(g, r_, shards)[0]
        rows.append({"row": f"support_am4 sharded x{shards} (triangle.cpp:26-61; kernel ms of the slowest shard)",
                     "gpu_s": max(ts) * 1e-3, "ref_s": tr, "equal": bool((acc.astype(np.uint32) == s_ref).all()),
                     "shard_ms": [round(x, 2) for x in ts], "full_kernel_ms": round(ctx.support(g)[1]["support_ms"], 2)})

    # read_edge_list on a text file of the first 4M edges (graph.cpp:152-200)
    import tempfile
    k4 = min(len(pairs), 4_000_000)
    with tempfile.NamedTemporaryFile("w", suffix=".txt", delete=False) as f:
        f.write("# bench_next\n")
        np.savetxt(f, pairs[:k4], fmt="%d")
        path = f.name
    tg, pg = timed(lambda: trussdec.read_edge_list(path), 2)
    tr, pr = timed(lambda: R.read_edge_list(path))
    os.unlink(path)
    rows.append({"row": f"read_edge_list, {k4} text lines (graph.cpp:152-200)", "gpu_s": tg, "ref_s": tr,
                 "equal": bool(np.array_equal(np.asarray(pg, np.uint64).reshape(-1, 2), np.asarray(pr, np.uint64).reshape(-1, 2)))})

    for r in rows:
        r.update({"config": graphgen.CONFIG_NAMES[cfg], "m": m, "ref_threads": threads,
                  "speedup": (r["ref_s"] / r["gpu_s"]) if r.get("ref_s") else None})
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
