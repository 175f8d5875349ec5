"""N > 1 host logic of bench.py on CPU: world_size-2 gloo ranks (replicas only).
Each rank times its own replica; the job throughput divides all ranks' dofs by the slowest rank's time."""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = [0.004, 0.005][rank]                       # rank 1 is the slow one
        tmax = bench.reduce_max(t, world, torch.device("cpu"))
        out[rank] = (tmax, bench.replica_value(1000, world, tmax))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_two_rank_max_and_replica_value():
    port = _free_port()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert out[0] == out[1]
    tmax, value = out[0]
    assert tmax == pytest.approx(0.005)
    assert value == pytest.approx(2 * 1000 / 0.005 / 1e9)


def test_single_rank_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.reduce_max(0.25, 1, None) == 0.25
    assert bench.replica_value(2146689, 1, 1e-3) == pytest.approx(2.146689)
