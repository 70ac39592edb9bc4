"""GPU: row-slab sharding.  The slabs a multi-GPU job assembles
(one per rank) are built here one after another on the single GPU — no rank
waits on another — and must reproduce the whole-matrix plan's rows, and the
slab matvecs its product."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_target,family,world", [(642, "P1", 3), (2562, "P0", 4), (642, "P1", 1)])
def test_row_slabs_match_whole_matrix(galerk, n_target, family, world):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1804_00995_b200.shard import row_partition

    m = galerk.build_sphere(n_target, 1.0)
    d = galerk.make_domain(m, 3)
    sp = galerk.make_fem(m, family)
    kern = galerk.green_kernel("[exp(ikr)/r]", 2 * math.pi / (10 * galerk.edge_stats(m).mean_len))
    n = sp.free_count()
    full = galerk.AssemblyPlan(d, d, sp, kern, sp)
    A = torch.empty(n * n, dtype=torch.complex128, device="cuda")
    full.assemble(A.data_ptr(), n, 0)
    x = torch.tensor(galerk.complex_normal(5, n), device="cuda")
    y = torch.empty(n, dtype=torch.complex128, device="cuda")
    galerk.matvec(A.data_ptr(), n, n, n, x.data_ptr(), y.data_ptr(), 0)
    torch.cuda.synchronize()
    An = A.cpu().numpy().reshape(n, n).T
    yn = y.cpu().numpy()
    ys = []
    for r0, r1 in row_partition(n, world):
        plan = galerk.AssemblyPlan(d, d, sp, kern, sp, galerk.BemOptions(), -1, r0, r1)
        info = plan.info()
        assert info["rows"] == r1 - r0 and info["cols"] == n
        assert bool(info["symmetric"]) == (world == 1)  # a proper slab is never symmetric
        lda = max(1, r1 - r0)
        S = torch.empty(n * lda, dtype=torch.complex128, device="cuda")
        plan.assemble(S.data_ptr(), lda, 0)
        yl = torch.empty(r1 - r0, dtype=torch.complex128, device="cuda")
        galerk.matvec(S.data_ptr(), r1 - r0, n, lda, x.data_ptr(), yl.data_ptr(), 0)
        torch.cuda.synchronize()
        Sn = S.cpu().numpy().reshape(n, lda).T[: r1 - r0]
        ref = An[r0:r1]
        assert np.linalg.norm(Sn - ref) <= 1e-13 * np.linalg.norm(ref)
        ys.append(yl.cpu().numpy())
    yc = np.concatenate(ys)
    assert np.linalg.norm(yc - yn) <= 1e-13 * np.linalg.norm(yn)


def test_sharded_operator_single_rank(galerk):
    """ShardedOperator without a process group is the whole matrix on one GPU."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1804_00995_b200.shard import ShardedOperator

    m = galerk.build_sphere(642, 1.0)
    d = galerk.make_domain(m, 3)
    sp = galerk.make_fem(m, "P1")
    kern = galerk.green_kernel("[exp(ikr)/r]", 2 * math.pi / (10 * galerk.edge_stats(m).mean_len))
    n = sp.free_count()
    op = ShardedOperator(d, d, sp, kern, sp).assemble()
    x = torch.tensor(galerk.complex_normal(6, n), device="cuda")
    y = op.matvec(x)
    torch.cuda.synchronize()
    A = galerk.bem_dense(d, d, sp, kern, sp)
    ref = np.asarray(A) @ x.cpu().numpy()
    assert y.shape == (n,)
    assert np.linalg.norm(y.cpu().numpy() - ref) <= 1e-12 * np.linalg.norm(ref)


def test_matrix_free_target_slabs(galerk):
    """Matrix-free matvec sharded by targets (sources replicated, no reduction):
    each target slab's plan reproduces its rows of the whole plan's product."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1804_00995_b200.shard import row_partition

    m = galerk.build_sphere(2562, 1.0)
    d = galerk.make_domain(m, 3)
    pts, w, _ = galerk.quadrature(d)
    pts = np.asarray(pts)
    k = 2 * math.pi / (10 * galerk.edge_stats(m).mean_len)
    kern = galerk.green_kernel("[exp(ikr)/r]", k)
    q = torch.tensor(np.asarray(w) * galerk.complex_normal(4, len(w)), device="cuda")
    whole = galerk.GreenPlan(pts, pts, kern)
    y = torch.empty(len(w), dtype=torch.complex128, device="cuda")
    whole.matvec(q.data_ptr(), y.data_ptr(), galerk.FP64, 0)
    torch.cuda.synchronize()
    yn = y.cpu().numpy()
    for r0, r1 in row_partition(len(w), 3):
        plan = galerk.GreenPlan(np.ascontiguousarray(pts[r0:r1]), pts, kern)
        assert plan.info()["eps"] == whole.info()["eps"]  # the guard radius sees every source
        ys = torch.empty(r1 - r0, dtype=torch.complex128, device="cuda")
        plan.matvec(q.data_ptr(), ys.data_ptr(), galerk.FP64, 0)
        torch.cuda.synchronize()
        ref = yn[r0:r1]
        assert np.linalg.norm(ys.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
