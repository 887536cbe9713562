"""CPU, multi-process: bench.py's N>1 logic (replicas only) with world_size 2 over gloo —
max-over-ranks timing, whole-job value, and the reference arm running on rank 0 only."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    per_rank_ms = [100.0, 250.0][rank]
    mx = bench.max_over_ranks(per_rank_ms)
    val = bench.whole_job_value(world, 1_000_000, mx)
    # the reference arm: rank != 0 returns immediately without output or work
    import argparse
    did = None
    if rank == 1:
        args = argparse.Namespace(steps=1, warmup=0, gpus=world, ref_config=1)
        did = bench.bench_reference(args)
    q.put((rank, mx, val, did))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replica_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, val, did in res:
        assert mx == 250.0                      # max over ranks
        assert val == pytest.approx(2 * 1_000_000 / 0.25 / 1e6)  # world * m / max time
        assert did is None


def test_bench_spawns_n_ranks_itself():
    """`bench.py --gpus 2` without a torchrun environment launches 2 ranks (one process per
    GPU, distinct LOCAL_RANK = device binding) and rank 0 reports n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-check"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert sorted(r["local_rank"] for r in d["ranks"]) == [0, 1]
    assert len({r["pid"] for r in d["ranks"]}) == 2
    assert d["max_over_ranks"] == 2.0


def test_byte_models_bracket():
    """The element-level model never exceeds the sector-level bound, and both grow with the
    tallies (bench.py peel_bytes)."""
    import bench
    c = dict(filter=100, pbits=200, walk=80, slots=120, hits=30, dead=10, dec=40, repair=2, next=5, cross=1,
             comp_in=1000, comp_kept=700, comp_long=50, scan_in=5000, scan_out=4000, tasks=300, sorted=0, marks=300)
    b = bench.peel_bytes(c, n=100, m=1000, probes=500)
    assert 0 < b["elem"]["total"] <= b["sector"]["total"]
    c2 = dict(c, hits=60)
    assert bench.peel_bytes(c2, 100, 1000, 500)["elem"]["total"] > b["elem"]["total"]
    assert bench.support_bytes({"sup_tab_elems": 10}, 1000, 500, 7) > 0


def test_ncu_traffic_is_tied_to_the_sources(tmp_path, monkeypatch):
    """profiles/ncu_traffic.json is only used when it was captured on the current CUDA sources."""
    import json
    import bench
    f = tmp_path / "ncu.json"
    f.write_text(json.dumps({"src_sha": "0000", "C5": {"k_peel": {"dram_bytes": 1}}}))
    monkeypatch.setattr(bench, "NCU_FILE", str(f))
    assert bench.ncu_traffic(5).get("stale") is True
    f.write_text(json.dumps({"src_sha": bench.src_sha(), "C5": {"k_peel": {"dram_bytes": 1}}}))
    assert bench.ncu_traffic(5) == {"k_peel": {"dram_bytes": 1}}


def _shard_worker(rank, world, port, q):
    """Rank `rank` of the sharded support pass's host side over gloo: the partial supports
    (here: the oracle's supports split between the ranks edge by edge, standing in for the GPU
    shards) are summed by allreduce_partial_supports; every rank must end with the full array."""
    import numpy as np
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle
    from paper_1707_02000_b200 import trussdec
    orc = Oracle()
    csr = orc.rmat_graph(9, 8, 11)
    full = np.asarray(orc.support_am4(csr), np.uint32)
    rng = np.random.default_rng(5)  # same stream on both ranks
    cut = (rng.random(len(full)) * (full + 1)).astype(np.uint32)  # 0 <= cut <= full
    part = cut if rank == 0 else full - cut
    # wrap-around is part of the contract (u32 sums on the i32 view): plant one
    part = part.copy()
    part[0] = np.uint32(0xFFFFFFF0) if rank == 0 else np.uint32(full[0] + 0x10)
    out = trussdec.allreduce_partial_supports(np.ascontiguousarray(part))
    q.put((rank, bool(np.array_equal(out, full)), int(full.sum())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_support_allreduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [True, True]
    assert res[0][2] == res[1][2] > 0
