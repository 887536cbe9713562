#!/usr/bin/env python3
"""bench.py — PKT truss decomposition on B200 (BASELINE.json metric).

A "step" = one full decomposition of the workload graph (default: BASELINE config 5,
RMAT-25): edge-id map + degree orientation + hash tables (build), support pass,
device-resident level-synchronous peel, truss = s + 2.

  value : Medges/s with the CSR already resident in HBM (tdg_truss_device), whole job over
          all ranks (replicas only: every rank decomposes its own copy; no data-path
          collective — SURVEY §8(e)).
  e2e   : the same through the host-pointer C-ABI call tdg_truss with pinned host buffers:
          H2D of the CSR and D2H of truss[m] inside every timed step.
  roofline : the dominant kernel (k_peel) against the measured HBM copy bandwidth, with
          ELEMENT-level algorithmic bytes of the algorithm as implemented (access tallies
          of a diagnostic count-mode run x bytes per access), a sector-level
          upper bound, the SURVEY §8(d) PKT model, and ncu's DRAM bytes (profiles/).
  cpu_baseline : the reference (oracle/_ref = the unmodified reference sources) on this
          host's cores on a SAME-CONFIG pair — BASELINE config 4 decomposed here on the GPU
          and by the reference, input order (i) and the reference's own kcore -> coreness
          order -> reorder preprocessing (ii, the headline CPU variant, trussdec.cpp:92-97).
  --impl reference : the reference's truss_parallel on BASELINE config --ref-config
          (default 4; preprocessing (ii) once, each step = one engine run), rank 0 only.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
With --gpus N > 1 and no torchrun environment, bench.py launches N ranks itself
(torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1).
"""
from __future__ import annotations

import os

# OpenMP placement of the reference library (libgomp reads it once, when it is loaded)
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import argparse  # noqa: E402
import csv  # noqa: E402
import hashlib  # noqa: E402
import io  # noqa: E402
import json  # noqa: E402
import socket  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "truss decomposition Medges/s on 1 B200; achieved HBM GB/s vs peak"
UNIT = "Medges/s"
L2_BYTES = 126 * 2 ** 20
GOLDEN = os.path.join(ROOT, "tests", "golden", "configs.json")
NCU_FILE = os.path.join(ROOT, "profiles", "ncu_traffic.json")
CSRC = os.path.join(ROOT, "paper_1707_02000_b200", "csrc")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=int(os.environ.get("TDG_BENCH_CONFIG", "5")))
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--ref-config", type=int, default=4, help="BASELINE config of the CPU reference runs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-counts", action="store_true", help="skip the untimed count-mode run (byte model)")
    ap.add_argument("--launcher-check", action="store_true", help=argparse.SUPPRESS)  # CPU test of the N-rank launch
    return ap.parse_args(argv)


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(args, argv) -> int:
    """--gpus N without a torchrun environment: launch N ranks (one process per GPU) with
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd, cwd=ROOT)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy test)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def max_over_ranks(x: float, dev=None) -> float:
    """Max of a per-rank scalar over all ranks (gloo on CPU, nccl on GPU); x if single rank."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=dev if dev is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(world: int, m: int, ms_per_step: float) -> float:
    """Replicas only: every rank decomposes its own copy, so the job processes world*m edges
    per step; the step time is the max over ranks."""
    return world * m / (ms_per_step * 1e-3) / 1e6


def golden(cfg: int) -> dict | None:
    try:
        return json.load(open(GOLDEN))["configs"].get(str(cfg))
    except Exception:
        return None


def src_sha() -> str:
    """Hash of the CUDA sources: ties an ncu capture in profiles/ to the code it measured."""
    h = hashlib.sha256()
    for f in sorted(os.listdir(CSRC)):
        if f.endswith((".cu", ".cuh", ".h")):
            h.update(f.encode())
            h.update(open(os.path.join(CSRC, f), "rb").read())
    return h.hexdigest()[:16]


# ----------------------------------------------------------------------------- byte models
def peel_bytes(c: dict, n: int, m: int, probes: int) -> dict:
    """Bytes k_peel moves for the algorithm AS IMPLEMENTED, from the access
    tallies c of a count-mode run (tdg_counters): element-level (every access charged its
    own width — what an ideal memory system moves) and sector-level (every random access a
    full 32 B sector, no L2 reuse — an upper bound). Returns {"elem": {...}, "sector": {...}}."""
    g = lambda k: int(c.get(k, 0))  # noqa: E731
    elem = {
        # probe: list element + edge id (coalesced), filter word, processed-bitmap word, one
        # 16 B key vector per table bucket read, the 4 B value and two edge-state words per
        # hit, atomics as read + write, appends (+ stamp store)
        "process": 8 * probes + 8 * g("filter") + 4 * g("pbits") + 16 * g("slots") + 20 * g("hits")
                   + 8 * g("dec") + 8 * g("repair") + 8 * g("next") + 4 * g("cross"),
        # per task: curr + el + 2 dl + off(a) + off(b), off(b+1) read, descriptor + work prefix written and
        # re-read by the process phase
        "prep": 84 * g("tasks"),
        "sort": 44 * g("sorted"),
        # live-list entry + edge state read, list entry written; one curr stamp per edge
        "scan": 12 * g("scan_in") + 4 * g("scan_out") + 4 * m,
        # adj + eid + processed bit read; kept entries written (long lists staged: 3 passes)
        "compact": 12 * g("comp_in") + 8 * g("comp_kept") + 24 * g("comp_long"),
        "marks": 8 * g("marks"),
        "init": 12 * m + 4 * n,
    }
    sec = {
        "process": 8 * probes + 32 * g("filter") + 32 * g("pbits") + 32 * g("slots")
                   + 64 * g("hits") + 32 * g("dec") + 4 * g("next") + 4 * g("cross"),
        "prep": 216 * g("tasks"),
        "sort": 204 * g("sorted"),
        "scan": 36 * g("scan_in") + 4 * g("scan_out"),
        "compact": 40 * g("comp_in") + 8 * g("comp_kept") + 24 * g("comp_long"),
        "marks": 36 * g("marks"),
        "init": 12 * m + 4 * n,
    }
    elem["total"] = sum(elem.values())
    sec["total"] = sum(sec.values())
    return {"elem": elem, "sector": sec}


def support_bytes(c: dict, m: int, probes: int, triangles: int) -> int:
    """Element-level bytes of the support pass as implemented: per task (oriented edge)
    the descriptor loads (slot, owner, neighbour, edge id, 2 x 2 list bounds) and the work
    prefix (written by prep, read back); per probe one N+(y) element; per triangle three
    atomics (read + write); owner lists loaded into shared-memory tables; searched items;
    zeroing and summing s."""
    return 32 * m + 24 * m + 8 * m + 4 * probes + 24 * triangles + 4 * int(c.get("sup_tab_elems", 0)) \
        + 4 * int(c.get("sup_search", 0)) + 8 * m


def survey_bytes(S1: int, S2: int, T: int, m: int, sum_tau_m1: int) -> tuple[int, int]:
    """SURVEY §8(d)'s PKT model (full-list scans): (B_sup, B_peel)."""
    return 4 * S1 + 24 * m + 32 * T, 4 * S2 + 48 * T + 55 * m + 5 * sum_tau_m1


REF_HOST = os.path.join(ROOT, "profiles", "r02_ref_host.jsonl")


def reference_host_record(cfg: int, variant: str = "ii") -> dict | None:
    """The reference's full run on this config on the GPU box's host, recorded once
    (scripts/ref_host_run.py -> profiles/r02_ref_host.jsonl): the workload itself is too slow
    for every bench run (C5: ~52 min on 16 cores)."""
    try:
        for line in open(REF_HOST):
            d = json.loads(line)
            if d["config"] == cfg and d["variant"] == variant:
                return {"value": d["engine_medges_s"], "unit": UNIT, "engine_s": d["engine_s"], "threads": d["threads"],
                        "cpu": d.get("cpu"), "phases_s": d["phases_s"], "variant": variant,
                        "source": "profiles/r02_ref_host.jsonl (scripts/ref_host_run.py on the GPU box host)"}
    except Exception:
        return None
    return None


def ncu_traffic(cfg: int) -> dict | None:
    """ncu DRAM bytes per launch for this config, if profiles/ncu_traffic.json was captured
    on the current CUDA sources (src_sha match); else None."""
    try:
        d = json.load(open(NCU_FILE))
    except Exception:
        return None
    if d.get("src_sha") != src_sha():
        return {"stale": True, "src_sha": d.get("src_sha")}
    return d.get(f"C{cfg}")


# ----------------------------------------------------------------------------- CPU arm
def reference_pair(cfg: int, threads: int, variants=("i", "ii")) -> dict:
    """The reference on config cfg, each variant prepared once and its engine run once:
    (i) input order, (ii) kcore_parallel -> coreness_order -> reorder (trussdec.cpp:92-97)."""
    from oracle import Csr, Reference
    from paper_1707_02000_b200 import graphgen
    R = Reference()
    n, m, off, nb = graphgen.config(cfg)
    g = Csr(n, m, off, nb)
    out = {"workload": graphgen.CONFIG_NAMES[cfg], "n": n, "m": m, "threads": threads}
    for v in variants:
        h, prep = R.prepare(g, threads, kcore=(v == "ii"))
        try:
            run = R.run(h, threads)
        finally:
            R.free(h)
        out[v] = {"prep_s": prep, "engine_s": run["engine"], "support_s": run["support"],
                  "peel_s": run["scan"] + run["processing"], "t_max": run["t_max"],
                  "value": m / run["engine"] / 1e6}
    return out


def bench_reference(args):
    """--impl reference: the reference's own truss_parallel (oracle/_ref, unmodified sources)
    on all host threads; rank 0 only (other ranks exit without work)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    from oracle import Csr, Reference
    from paper_1707_02000_b200 import graphgen
    threads = os.cpu_count() or 1
    cfg = args.ref_config
    R = Reference()
    n, m, off, nb = graphgen.config(cfg)
    g = Csr(n, m, off, nb)
    h, prep = R.prepare(g, threads, kcore=True)
    steps, warmup = max(1, args.steps), min(max(0, args.warmup), 1)
    runs = []
    try:
        for i in range(warmup + steps):
            r = R.run(h, threads)
            if i >= warmup:
                runs.append(r)
    finally:
        R.free(h)
    t = float(np.median([r["engine"] for r in runs]))
    val = m / t / 1e6
    gold = golden(cfg)
    sample = (f"{graphgen.CONFIG_NAMES[cfg]} (BASELINE config {cfg}, m={m}): one full truss_parallel per step "
              f"after the reference's own kcore -> coreness_order -> reorder preprocessing (done once, "
              f"trussdec.cpp:92-97); the C5 workload itself takes ~1 h per run on this host class")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator)",
            "config": {"workload": graphgen.CONFIG_NAMES[cfg], "n": n, "m": m, "threads": threads,
                       "variant": "ii (kcore preprocessing)"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "prep_s": prep,
            "c5_reference_host": reference_host_record(5),
            "phases_s": {k: float(np.median([r[k] for r in runs])) for k in ("support", "scan", "processing", "engine")},
            "t_max": runs[-1]["t_max"], "t_max_golden": gold and gold.get("t_max"),
            "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")}}
    print(json.dumps(line), flush=True)
    return line


# ----------------------------------------------------------------------------- GPU arm
class ClockSampler:
    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        rows = [r for r in csv.reader(io.StringIO(out)) if len(r) == len(self.FIELDS)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        reasons = set()
        for r in rows:
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def truss_sha(truss_u32: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(truss_u32, np.uint32).tobytes()).hexdigest()


def gpu_same_config(ctx, stream, dev, cfg: int, steps: int = 5, warmup: int = 3) -> dict:
    """Config cfg decomposed on this GPU with the device-resident C-ABI call (median of
    `steps` after `warmup`, L2 flushed between steps), checked against the golden."""
    import torch

    from paper_1707_02000_b200 import graphgen
    n, m, off, nb = graphgen.config(cfg)
    off_d = torch.from_numpy(off).to(dev)
    nb_d = torch.from_numpy(np.ascontiguousarray(nb)).to(dev)
    truss_d = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)
    nsl = np.zeros(n + 2, np.uint32)
    ms = []
    for i in range(warmup + steps):
        flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nlen, t = ctx.truss_device(n, m, off_d.data_ptr(), nb_d.data_ptr(), truss_d.data_ptr(), nsl)
        b.record(stream)
        torch.cuda.synchronize()
        if i >= warmup:
            ms.append(a.elapsed_time(b))
    gold = golden(cfg) or {}
    sha = truss_sha(truss_d[:m].cpu().numpy().view(np.uint32))
    t_ms = float(np.median(ms))
    res = {"workload": graphgen.CONFIG_NAMES[cfg], "m": m, "ms": t_ms, "value": m / (t_ms * 1e-3) / 1e6,
           "truss_sha_ok": sha == gold.get("truss_sha"), "nsl_ok": [int(x) for x in nsl[:nlen]] == gold.get("nsl")}
    del off_d, nb_d, truss_d, flush
    torch.cuda.empty_cache()
    return res


def bench_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1707_02000_b200 import graphgen, trussdec

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    # ---- workload (every rank builds the same seeded graph: replicas only)
    pinned = {}

    def alloc(n, m):
        pinned["off"] = torch.empty(n + 1, dtype=torch.int64, pin_memory=True)
        pinned["nb"] = torch.empty(max(2 * m, 1), dtype=torch.int32, pin_memory=True)
        return pinned["off"].numpy(), pinned["nb"].numpy()

    t0 = time.time()
    n, m, off_np, nb_np = graphgen.config(args.config, 0, alloc)
    gen_s = time.time() - t0
    off_h, nb_h = pinned["off"], pinned["nb"]
    off_d = off_h.to(dev, non_blocking=True)
    nb_d = nb_h.to(dev, non_blocking=True)
    truss_d = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    truss_h = torch.empty(max(m, 1), dtype=torch.int32, pin_memory=True)
    torch.cuda.synchronize()
    in_bytes = (n + 1) * 8 + 2 * m * 4
    flush = None if in_bytes > 2 * L2_BYTES else torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev)

    ctx = trussdec.Context(local)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    nsl = np.zeros(n + 2, np.uint32)

    def step_device():
        return ctx.truss_device(n, m, off_d.data_ptr(), nb_d.data_ptr(), truss_d.data_ptr(), nsl)

    for _ in range(max(args.warmup, 0)):
        step_device()
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs)
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    recs = []
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i)
        evs[i][0].record(stream)
        nlen, t = step_device()
        evs[i][1].record(stream)
        recs.append(t)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = max_over_ranks(float(sum(step_ms)), dev)
    ms_per_step = total_ms / args.steps
    value = whole_job_value(world, m, ms_per_step)
    timed_counts = ctx.counters()

    # ---- parity of the timed run's output against the committed golden (reference output)
    truss = truss_d[:m].cpu().numpy().view(np.uint32)
    gold = golden(args.config) or {}
    parity = {"truss_sha_ok": truss_sha(truss) == gold.get("truss_sha"),
              "nsl_ok": [int(x) for x in nsl[:nlen]] == gold.get("nsl"),
              "t_max_ok": int(recs[-1]["t_max"]) == gold.get("t_max"),
              "golden": "tests/golden/configs.json (reference library output on the same CSR)"}
    if not (parity["truss_sha_ok"] and parity["nsl_ok"]):
        print(json.dumps({"error": "timed run does not match the golden", "parity": parity}), file=sys.stderr, flush=True)
    tri = recs[-1]["triangles"]
    sum_tau_m1 = int(truss.astype(np.uint64).sum()) - m if m else 0

    # ---- e2e through the host-pointer C-ABI (pinned buffers; H2D + D2H inside each step)
    e2e = None
    if not args.no_e2e:
        ctx.truss_host_ptrs(n, m, off_h.data_ptr(), nb_h.data_ptr(), truss_h.data_ptr(), nsl)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_ms = []
        for _ in range(args.steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.truss_host_ptrs(n, m, off_h.data_ptr(), nb_h.data_ptr(), truss_h.data_ptr(), nsl)
            b.record(stream)
            torch.cuda.synchronize()
            e_ms.append(a.elapsed_time(b))
        et = max_over_ranks(float(sum(e_ms)), dev)
        assert (truss_h[:m].numpy().view(np.uint32) == truss).all()
        e2e = {"value": whole_job_value(world, m, et / args.steps), "unit": UNIT,
               "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": 4 * m,
               "ms_per_step": et / args.steps}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- access tallies of one untimed count-mode decomposition (deterministic: the same
    # sub-level sets as the timed runs) -> the byte model of the kernels as implemented
    counts = None
    if not args.no_counts:
        os.environ["TDG_COUNT"] = "1"
        try:
            step_device()
            counts = ctx.counters()
        finally:
            os.environ.pop("TDG_COUNT", None)
        torch.cuda.synchronize()
    c = counts or timed_counts
    avg = {k: float(np.mean([r[k] for r in recs])) for k in
           ("build_ms", "support_ms", "peel_ms", "scan_ms", "process_ms", "compact_ms", "total_ms")}
    probes = int(recs[-1]["probes"])
    sup_probes = int(recs[-1]["support_probes"])
    pb = peel_bytes(c, n, m, probes)
    b_sup = support_bytes(c, m, sup_probes, tri)
    st = ctx.stats(trussdec.CsrGraph(n, m, off_np, nb_np[: 2 * m]))
    sv_sup, sv_peel = survey_bytes(st.deg_s1, st.sum_deg_sq, tri, m, sum_tau_m1)
    peak, peak_src = peaks()
    k_ms = avg["peel_ms"]
    gbs = lambda b, ms: b / (ms * 1e-3) / 1e9  # noqa: E731
    achieved = gbs(pb["elem"]["total"], k_ms)
    ncu = ncu_traffic(args.config)
    traffic = ncu.get("k_peel", {}).get("dram_bytes") if ncu and not ncu.get("stale") else None
    roofline = {
        "bound": "hbm", "kernel": "k_peel (persistent cooperative level loop; CUDA events around its launch)",
        "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
        "peak_source": peak_src, "kernel_ms": k_ms, "algorithmic_bytes": pb["elem"]["total"],
        "model": "element-level bytes of the implemented algorithm: tdg_counters tallies of a count-mode run "
                 "x bytes per access (bench.py peel_bytes, DESIGN.md §4)",
        "bytes_by_phase": pb["elem"],
        "sector_model": {"bytes": pb["sector"]["total"], "frac": gbs(pb["sector"]["total"], k_ms) / peak,
                         "note": "every random access a full 32 B sector, no L2 reuse (upper bound)"},
        "dram_frac_ncu": (traffic / (k_ms * 1e-3) / 1e9 / peak) if traffic else None,
        "ncu": ncu,
        "survey_model": {"bytes": sv_peel, "frac": gbs(sv_peel, k_ms) / peak,
                         "note": "SURVEY §8(d) PKT model (4*S2 full-list scans the hash-probe design never does)"},
        "support": {"kernel": "k_support_tab", "ms": avg["support_ms"], "bytes": b_sup,
                    "GBps": gbs(b_sup, avg["support_ms"]), "frac": gbs(b_sup, avg["support_ms"]) / peak,
                    "traffic": (ncu.get("k_support_tab", {}).get("dram_bytes") if ncu and not ncu.get("stale") else None),
                    "survey_model_bytes": sv_sup},
        "counts": c,
        "counts_consistent": None if counts is None else all(
            counts[k] == timed_counts[k] for k in ("scan_in", "scan_out", "tasks", "sorted", "marks")),
    }

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = os.cpu_count() or 1
        try:
            gpu_pair = gpu_same_config(ctx, stream, dev, args.ref_config)
            ref = reference_pair(args.ref_config, threads)
            cpu = {"value": ref["ii"]["value"], "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"{ref['workload']} (BASELINE config {args.ref_config}, m={ref['m']}): the reference's "
                             f"truss_parallel once per variant on this host; value = variant (ii), its own "
                             f"kcore -> coreness_order -> reorder preprocessing (trussdec.cpp:92-97)",
                   "workload": ref["workload"], "variant_i": ref["i"], "variant_ii": ref["ii"],
                   "gpu_same_config": gpu_pair,
                   "speedup_same_config": {"vs_i": gpu_pair["value"] / ref["i"]["value"],
                                           "vs_ii": gpu_pair["value"] / ref["ii"]["value"]},
                   "workload_reference_host": reference_host_record(args.config),
                   "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")}}
        except Exception as e:  # the checker is optional on a box without oracle/_ref
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded generator, include/tdg_gen.h)",
        "config": {"workload": graphgen.CONFIG_NAMES[args.config], "n": n, "m": m, "triangles": tri,
                   "t_max": recs[-1]["t_max"], "sublevels": recs[-1]["sublevels"], "scans": recs[-1]["scans"],
                   "parallelism": f"replicas x{world}", "l2": "inputs larger than L2" if flush is None
                   else "L2 flushed between steps", "gen_s": gen_s},
        "phases_ms": avg,
        "parity": parity,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": int(sum(r["kernel_launches"] for r in recs)),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def launcher_check(args):
    """CPU check of the N-rank launch (tests/test_bench_dist.py): every rank reports its
    rank / local rank over gloo; rank 0 prints them with n_gpus = world size."""
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    info = {"rank": rank, "local_rank": local, "pid": os.getpid()}
    allinfo = [None] * world
    if world > 1:
        dist.all_gather_object(allinfo, info)
    else:
        allinfo = [info]
    mx = max_over_ranks(float(rank + 1))
    if rank == 0:
        print(json.dumps({"n_gpus": world, "ranks": allinfo, "max_over_ranks": mx}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args, argv))
    if args.launcher_check:
        launcher_check(args)
    elif args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
