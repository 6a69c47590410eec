"""The N > 1 host path of bench.py on CPU (gloo, world size 2): N independent
replicas, timed as the max over ranks, value = N * m / that time; the
reference arm prints on rank 0 only (replicas only)."""
import io
import os
import socket
import sys
from contextlib import redirect_stdout

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms = bench.reduce_max_ms(1.5 + rank, dist, "cpu")   # rank 1 is the slow one
    dist.barrier()
    q.put((rank, ms, bench.job_value(world, 1000, ms)))
    dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
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
    assert [r[1] for r in res] == [2.5, 2.5]                    # every rank sees the max
    assert all(r[2] == pytest.approx(2 * 1000 / 2.5e-3) for r in res)


def test_reference_arm_prints_on_rank0_only(monkeypatch):
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2"])
    buf = io.StringIO()
    with redirect_stdout(buf):
        assert bench.run_reference(bench.parse_args()) == 0
    assert buf.getvalue() == ""


def test_single_process_identity():
    assert bench.reduce_max_ms(3.25, None, "cpu") == 3.25
    assert bench.job_value(1, 500, 2.0) == pytest.approx(500 / 2e-3)
