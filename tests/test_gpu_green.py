"""GPU parity: matrix-free Green-kernel matvec (K5), fp64 and fp32 variants."""
import math

import numpy as np
import pytest

from tests._support import rel_fro

pytestmark = pytest.mark.gpu
FP32_TOL = 2e-4  # stated bound for the complex64/fp32 variant (relative l2)


def _setup(galerk, n_target):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    m = galerk.build_sphere(n_target, 1.0)
    dom = galerk.make_domain(m, 3)
    pts, w, _ = galerk.quadrature(dom)
    hbar = galerk.edge_stats(m).mean_len
    k = 2 * math.pi / (10 * hbar)
    q = np.asarray(w) * galerk.complex_normal(4, len(w))
    return torch, m, pts, q, k


@pytest.mark.parametrize("n_target", [642, 10242])
def test_green_matvec_fp64_and_fp32(galerk, oracle, n_target):
    torch, m, pts, q, k = _setup(galerk, n_target)
    plan = galerk.GreenPlan(pts, pts, galerk.green_kernel("[exp(ikr)/r]", k))
    info = plan.info()
    assert info["unique_targets"] == len(pts) // 2  # every point has one bit-identical twin
    qd = torch.tensor(q, device="cuda")
    y64 = torch.empty(len(pts), dtype=torch.complex128, device="cuda")
    y32 = torch.empty_like(y64)
    plan.matvec(qd.data_ptr(), y64.data_ptr(), galerk.FP64, 0)
    plan.matvec(qd.data_ptr(), y32.data_ptr(), galerk.FP32, 0)
    torch.cuda.synchronize()
    ids = sorted(set(np.random.default_rng(1).choice(len(pts), 64, replace=False).tolist()) | {0, 1})
    ref = np.array(oracle.green_matvec("[exp(ikr)/r]", k, pts, pts, q, info["eps"], ids, 8))
    y64n, y32n = y64.cpu().numpy(), y32.cpu().numpy()
    assert rel_fro(y64n[ids], ref) <= 1e-10
    assert rel_fro(y32n[ids], ref) <= FP32_TOL
    # twins get identical outputs
    assert y64n[0] == y64n[np.flatnonzero((pts == pts[0]).all(axis=1))[-1]]


def test_green_matvec_laplace(galerk, oracle):
    torch, m, pts, q, _ = _setup(galerk, 162)
    plan = galerk.GreenPlan(pts, pts[::2].copy(), galerk.green_kernel("[1/r]", 0.0))
    qd = torch.tensor(q[::2].copy(), device="cuda")
    y = torch.empty(len(pts), dtype=torch.complex128, device="cuda")
    plan.matvec(qd.data_ptr(), y.data_ptr(), galerk.FP64, 0)
    torch.cuda.synchronize()
    ids = list(range(len(pts)))
    ref = np.array(oracle.green_matvec("[1/r]", 0.0, pts, pts[::2].copy(), q[::2].copy(), plan.info()["eps"], ids, 8))
    assert rel_fro(y.cpu().numpy(), ref) <= 1e-10


@pytest.mark.parametrize("name,npts", [("[exp(ikr)/r]", None), ("[1/r]", None), ("[exp(ikr)/r]", 1001)])
def test_green_matvec_symmetric_path(galerk, oracle, monkeypatch, name, npts):
    """targets == sources: the symmetric fp64 path (each unordered block pair
    once, rotating column sums) agrees with the general path and the oracle,
    including a ragged last block (npts not a multiple of the block size)."""
    torch, m, pts, q, k = _setup(galerk, 2562)
    if npts is not None:
        pts, q = pts[:npts].copy(), q[:npts].copy()
    kk = k if name != "[1/r]" else 0.0
    kern = galerk.green_kernel(name, kk)
    qd = torch.tensor(q, device="cuda")
    ys = torch.empty(len(pts), dtype=torch.complex128, device="cuda")
    yg = torch.empty_like(ys)
    galerk.GreenPlan(pts, pts, kern).matvec(qd.data_ptr(), ys.data_ptr(), galerk.FP64, 0)
    monkeypatch.setenv("GK_GREEN_SYM", "0")
    plan_g = galerk.GreenPlan(pts, pts, kern)
    plan_g.matvec(qd.data_ptr(), yg.data_ptr(), galerk.FP64, 0)
    torch.cuda.synchronize()
    ysn, ygn = ys.cpu().numpy(), yg.cpu().numpy()
    assert np.all(np.isfinite(ysn))
    assert rel_fro(ysn, ygn) <= 1e-13
    ids = sorted(set(np.random.default_rng(2).choice(len(pts), 48, replace=False).tolist()) | {0, len(pts) - 1})
    ref = np.array(oracle.green_matvec(name, kk, pts, pts, q, plan_g.info()["eps"], ids, 8))
    assert rel_fro(ysn[ids], ref) <= 1e-10


def test_config5_full_size_sampled_targets(galerk, oracle):
    """BASELINE cfg 5 at full size: L7 sphere, 983,040 Gauss points as targets
    and sources (symmetric path, 1,920 blocks in groups), charges = weight x
    complex N(0,1) from seed 4; sampled targets vs the oracle (fp64 1e-10,
    fp32 within FP32_TOL)."""
    torch, m, pts, q, k = _setup(galerk, 163842)
    assert len(pts) == 983040
    plan = galerk.GreenPlan(pts, pts, galerk.green_kernel("[exp(ikr)/r]", k))
    info = plan.info()
    assert info["unique_targets"] == 491520
    qd = torch.tensor(q, device="cuda")
    y64 = torch.empty(len(pts), dtype=torch.complex128, device="cuda")
    y32 = torch.empty_like(y64)
    plan.matvec(qd.data_ptr(), y64.data_ptr(), galerk.FP64, 0)
    plan.matvec(qd.data_ptr(), y32.data_ptr(), galerk.FP32, 0)
    torch.cuda.synchronize()
    ids = sorted(set(np.random.default_rng(5).choice(len(pts), 24, replace=False).tolist()) | {0, len(pts) - 1})
    ref = np.array(oracle.green_matvec("[exp(ikr)/r]", k, pts, pts, q, info["eps"], ids, 16))
    assert rel_fro(y64.cpu().numpy()[ids], ref) <= 1e-10
    assert rel_fro(y32.cpu().numpy()[ids], ref) <= FP32_TOL


def test_green_matvec_near_coincident_points(galerk, oracle):
    """Points closer than eps but not bitwise equal (an unwelded mesh nudged by
    ~1e-14): the distance mask, not the twin merge, must drop those pairs, on
    the symmetric and the general path alike."""
    import torch

    base = galerk.build_sphere(162, 1.0)
    v0, e0 = np.asarray(base.vertices), np.asarray(base.elements)
    rng = np.random.default_rng(9)
    v = v0[e0].reshape(-1, 3) * (1.0 + 1e-14 * rng.uniform(-1, 1, size=(3 * len(e0), 1)))
    e = np.arange(3 * len(e0), dtype=np.int32).reshape(-1, 3)
    dom = galerk.make_domain(galerk.Mesh(v, e), 3)
    pts, w, _ = galerk.quadrature(dom)
    q = np.asarray(w) * galerk.complex_normal(4, len(w))
    kern = galerk.green_kernel("[exp(ikr)/r]", 4.0)
    plan = galerk.GreenPlan(pts, pts, kern)
    assert plan.info()["symmetric"]
    qd = torch.tensor(q, device="cuda")
    y = torch.empty(len(pts), dtype=torch.complex128, device="cuda")
    plan.matvec(qd.data_ptr(), y.data_ptr(), galerk.FP64, 0)
    torch.cuda.synchronize()
    ids = list(range(0, len(pts), 7))
    ref = np.array(oracle.green_matvec("[exp(ikr)/r]", 4.0, pts, pts, q, plan.info()["eps"], ids, 8))
    yn = y.cpu().numpy()
    assert np.all(np.isfinite(yn)) and rel_fro(yn[ids], ref) <= 1e-10
