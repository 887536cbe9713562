"""Time the UNMODIFIED reference (oracle/_ref/libtrussdec_ref.so) on BASELINE configs on the
host it runs on (the GPU box's own cores when launched through gpurun). Baseline
infrastructure only: variant (i) = the config CSR as given,
variant (ii) = the reference's own preprocessing kcore_parallel -> coreness_order -> reorder
(trussdec.cpp:92-97) before build_truss_graph + truss_parallel.

Usage: python scripts/ref_host_run.py OUT.jsonl CFG:VARIANTS [CFG:VARIANTS ...]
       e.g. 2:i,ii 4:i,ii 5:ii
"""
import os
import sys

# OpenMP placement must be in the environment before libgomp is loaded (with the library)
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import json  # noqa: E402
import platform  # noqa: E402
import time  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import Csr, Reference  # noqa: E402
from paper_1707_02000_b200 import graphgen  # noqa: E402


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main():
    out = sys.argv[1]
    R = Reference()
    threads = os.cpu_count() or 1
    for spec in sys.argv[2:]:
        cfg, variants = spec.split(":")
        cfg = int(cfg)
        t0 = time.time()
        n, m, off, nb = graphgen.config(cfg)
        gen_s = time.time() - t0
        g = Csr(n, m, off, nb)
        for v in variants.split(","):
            t0 = time.time()
            if v == "i":
                d = R.truss_parallel(g, threads)
                ph = dict(d.times)
                engine = ph["engine"]
            else:
                ph = R.truss_parallel_kcore(g, threads)
                engine = ph["engine"]
            wall = time.time() - t0
            rec = {"config": cfg, "workload": graphgen.CONFIG_NAMES[cfg], "variant": v, "n": n, "m": m,
                   "threads": threads, "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")},
                   "cpu": cpu_model(), "phases_s": ph, "engine_s": engine, "wall_s": wall,
                   "engine_medges_s": m / engine / 1e6, "gen_s": gen_s}
            print(json.dumps(rec), flush=True)
            with open(out, "a") as f:
                f.write(json.dumps(rec) + "\n")


if __name__ == "__main__":
    main()
