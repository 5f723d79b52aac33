"""Multi-process host logic of bench.py (replicas only, SURVEY §8 e) with
the gloo backend on CPU, world_size 2: max-over-ranks timing, the whole-job
replica throughput, barriers, and the reference arm running on rank 0 only."""

from __future__ import annotations

import io
import os
import sys
from contextlib import redirect_stdout
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    sys.path.insert(0, str(ROOT))
    import bench

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, r, loc = bench.dist_setup(None)
        # rank 1 is the slow replica: the job time is its time
        t_local = 2.0 if rank == 1 else 1.0
        t_max, value = bench.replica_throughput(t_local, 10, world)
        bench.barrier(world)

        class A:
            steps, warmup, config = 1, 0, 2

        buf = io.StringIO()
        if rank != 0:
            with redirect_stdout(buf):
                bench.run_reference(A, world, rank)  # rank 0 alone runs the CPU arm
        q.put((rank, w, r, loc, t_max, value, buf.getvalue()))
    finally:
        dist.destroy_process_group()


def test_bench_replicas_gloo_world2():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, w, r, loc, t_max, value, out in res:
        assert (w, r, loc) == (2, rank, rank)
        assert t_max == 2.0  # max over ranks, identical on every rank
        assert value == pytest.approx(2 * 10 / 2.0)  # whole-job steps/s
    assert res[1][6] == ""  # the reference arm prints nothing off rank 0
