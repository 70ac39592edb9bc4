"""Row-slab sharding host logic on CPU: the row partition, the
test-side row slab the plans are built on, and the one collective of the path
(gathering y slabs) over world_size-2 gloo ranks."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_00995_b200.shard import gather_rows, row_partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,world", [(642, 1), (642, 2), (10242, 8), (5, 8), (0, 3)])
def test_row_partition_covers_rows_once(n, world):
    parts = row_partition(n, world)
    assert len(parts) == world
    assert parts[0][0] == 0 and parts[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
    sizes = [r1 - r0 for r0, r1 in parts]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 0


def test_row_slab_plan_statistics(galerk):
    """A slab plan sees the slab's rows and every trial location, keeps the full
    plan's guard radius, and the slabs together evaluate at most ~1/3 more
    pairs than one non-symmetric plan of the whole matrix (the x halo along the
    slab cuts: measured 1.16 / 1.22 / 1.26 for 2 / 3 / 8 slabs of cfg 2)."""
    m = galerk.build_sphere(642, 1.0)
    d = galerk.make_domain(m, 3)
    sp = galerk.make_fem(m, "P1")
    kern = galerk.green_kernel("[exp(ikr)/r]", 2 * math.pi / (10 * galerk.edge_stats(m).mean_len))
    full = galerk.plan_info_dry(d, d, sp, kern, sp, galerk.BemOptions(), 0)
    n = sp.free_count()
    tot = 0
    for r0, r1 in row_partition(n, 3):
        info = galerk.plan_info_dry_rows(d, d, sp, kern, sp, galerk.BemOptions(), r0, r1)
        assert info["rows"] == r1 - r0 and info["cols"] == n
        assert info["y_locations"] == full["y_locations"]
        assert info["symmetric"] is False
        assert info["eps"] == full["eps"]  # same guard radius: the bbox is the trial side's
        tot += info["pairs_evaluated"]
    assert full["pairs_evaluated"] <= tot < 1.35 * full["pairs_evaluated"]


def _worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    y = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    r0, r1 = row_partition(n, world)[rank]
    got = gather_rows(torch.tensor(y[r0:r1]), n)
    out[rank] = bool(np.array_equal(got.numpy(), y)) and got.dtype == torch.complex128
    dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 7])
def test_gather_rows_two_ranks(n):
    port = _free_port()
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, n, out), nprocs=2, join=True)
    assert out[0] and out[1]


def test_empty_and_out_of_range_slabs(galerk):
    """More ranks than rows leave empty slabs (a valid, empty plan); a range
    outside the test side is rejected like the reference's bad arguments."""
    m = galerk.build_sphere(12, 1.0)
    d = galerk.make_domain(m, 3)
    sp = galerk.make_fem(m, "P1")
    kern = galerk.green_kernel("[1/r]", 0.0)
    info = galerk.plan_info_dry_rows(d, d, sp, kern, sp, galerk.BemOptions(), 5, 5)
    assert info["rows"] == 0 and info["pairs_evaluated"] == 0 and info["tiles"] == 0
    with pytest.raises(ValueError):
        galerk.plan_info_dry_rows(d, d, sp, kern, sp, galerk.BemOptions(), 3, 13)
