"""World-size-2 `gloo` test of the multi-rank host logic of bench.py (CPU):
replicas only -- each rank runs a full step, the job's
time is the slowest rank's, and value = units of all ranks / that time."""
import importlib.util
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port), "RANK": str(rank),
                       "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank)})
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=world)
    b = _bench()
    ws, r, local = b.dist_env()
    per_rank_ms = [10.0, 25.0][rank]
    mx = b.max_over_ranks(per_rank_ms, "cpu")
    val = b.job_value(1000, 4, ws, mx)
    dist.barrier()
    out[rank] = (ws, r, local, mx, val)
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_replicas_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        ws, r, local, mx, val = out[rank]
        assert (ws, r, local) == (2, rank, rank)
        assert mx == 25.0                                   # the slowest rank's time
        assert abs(val - 1000 * 4 * 2 / 0.025) < 1e-6       # all ranks' units / max time


def test_single_rank_is_identity():
    b = _bench()
    assert b.max_over_ranks(3.5, "cpu") == 3.5
    assert abs(b.job_value(10, 2, 1, 1000.0) - 20.0) < 1e-12
