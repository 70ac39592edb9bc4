"""N>1 plumbing on CPU: world_size-2 gloo ranks exercise bench.py's
max-over-ranks timing and whole-job aggregation (replicas, no data-path
collective — SURVEY §8e)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    local_ms = 10.0 + 5.0 * rank  # rank 1 is the slow replica
    ms = bench.max_over_ranks(local_ms, dist, torch.device("cpu"))
    value = bench.aggregate_value(1000, world, ms)
    dist.barrier()
    out[rank] = (ms, value)
    dist.destroy_process_group()


def test_two_rank_max_and_aggregate():
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()  # no fork of a process that already runs OpenMP threads
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    assert out[0] == out[1]
    ms, value = out[0]
    assert ms == 15.0
    assert value == pytest.approx(2 * 1000 / 0.015)


def test_single_process_passthrough():
    import bench

    assert bench.max_over_ranks(3.5, None, torch.device("cpu")) == 3.5
    assert bench.aggregate_value(10, 1, 1000.0) == 10.0


def test_reference_arm_under_torchrun_two_ranks():
    """`bench.py --impl reference` launched as the driver launches it for N>1:
    rank 0 alone runs and prints one JSON line, the other rank exits 0."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference", "--gpus", "2",
           "--config", "1", "--steps", "1", "--warmup", "1"]
    res = subprocess.run(cmd, cwd=root, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
