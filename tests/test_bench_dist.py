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
        args = argparse.Namespace(steps=1, warmup=0, gpus=world, ref_scale=4)
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
