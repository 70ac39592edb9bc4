"""GPU parity: the streamed one-shot gk_bem_dense (column slabs, tables built
ahead on worker threads, slab s assembled while slab s-1 drains to the host).

GK_SLAB_COLS forces the streamed path and its slab width at small sizes; the
results must match the oracle (<= 1e-10 relative Frobenius) and the
whole-matrix path, for pageable and pinned destinations, padded lda, mixed
spaces, point targets and the all-masked (unwelded mesh) case.
"""
import math

import numpy as np
import pytest

from tests._support import rel_fro, sphere_problem

pytestmark = pytest.mark.gpu
P0, P1 = 0, 1
FAM = {"P0": P0, "P1": P1}
TOL = 1e-10


def _torch():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.fixture
def slab(monkeypatch):
    def set_width(w):
        monkeypatch.setenv("GK_SLAB_COLS", str(w))
    return set_width


@pytest.mark.parametrize("n,gauss,fam,name,k,w", [
    (642, 3, "P1", "[exp(ikr)/r]", 4.0, 64),
    (642, 3, "P1", "[1/r]", 0.0, 100),      # width not a multiple of the tile, ragged last slab
    (162, 6, "P0", "[exp(ikr)/r]", 5.0, 7),  # many tiny slabs
    (162, 3, "P1", "[exp(ikr)/r]", 2.0, 1000),  # one slab
])
def test_streamed_matches_oracle_and_whole_path(galerk, oracle, slab, n, gauss, fam, name, k, w):
    m, dom, sp, _ = sphere_problem(galerk, n, gauss, fam)
    kern = galerk.green_kernel(name, k)
    slab(0)
    whole = galerk.bem_dense(dom, dom, sp, kern, sp)
    slab(w)
    A = galerk.bem_dense(dom, dom, sp, kern, sp)
    ref = oracle.bem_dense(m.vertices, m.elements, gauss, FAM[fam], m.vertices, m.elements, gauss, FAM[fam],
                           name, k, threads=8)
    assert rel_fro(A, ref) <= TOL
    assert rel_fro(A, whole) <= 1e-13
    if k == 0.0:
        assert np.all(A.imag == 0.0)


def test_streamed_mixed_spaces_and_points(galerk, oracle, slab):
    slab(32)
    mx = galerk.build_sphere(162, 1.0)
    vy = galerk.build_sphere(642, 1.0).vertices * 0.7 + np.array([0.3, 0.0, 0.1])
    my = galerk.Mesh(vy, galerk.build_sphere(642, 1.0).elements)
    dx, dy = galerk.make_domain(mx, 3), galerk.make_domain(my, 7)
    t, u = galerk.make_fem(mx, "P1"), galerk.make_fem(my, "P0")
    A = galerk.bem_dense(dx, dy, t, galerk.green_kernel("[exp(ikr)/r]", 6.0), u)
    ref = oracle.bem_dense(mx.vertices, mx.elements, 3, P1, my.vertices, my.elements, 7, P0, "[exp(ikr)/r]", 6.0)
    assert A.shape == (162, 1280) and rel_fro(A, ref) <= TOL
    pts = np.random.default_rng(4).normal(size=(300, 3)) * 1.3
    R = galerk.radiation_dense(pts, dy, galerk.green_kernel("[exp(ikr)/r]", 3.0), u)
    refr = oracle.radiation_dense(pts, my.vertices, my.elements, 7, P0, "[exp(ikr)/r]", 3.0)
    assert rel_fro(R, refr) <= TOL


def test_streamed_unwelded_mesh_masks_every_tile(galerk, oracle, slab):
    slab(64)
    base = galerk.build_sphere(162, 1.0)
    v0, e0 = np.asarray(base.vertices), np.asarray(base.elements)
    rng = np.random.default_rng(9)
    v = v0[e0].reshape(-1, 3) * (1.0 + 1e-14 * rng.uniform(-1, 1, size=(3 * len(e0), 1)))
    e = np.arange(3 * len(e0), dtype=np.int32).reshape(-1, 3)
    m = galerk.Mesh(v, e)
    dom = galerk.make_domain(m, 3)
    sp = galerk.make_fem(m, "P0")
    A = galerk.bem_dense(dom, dom, sp, galerk.green_kernel("[exp(ikr)/r]", 4.0), sp)
    ref = oracle.bem_dense(v, e, 3, P0, v, e, 3, P0, "[exp(ikr)/r]", 4.0)
    assert np.all(np.isfinite(A)) and rel_fro(A, ref) <= TOL


def test_streamed_pinned_destination_with_padding(galerk, slab):
    torch = _torch()
    m, dom, sp, _ = sphere_problem(galerk, 642, 3, "P1")
    kern = galerk.green_kernel("[exp(ikr)/r]", 4.2)
    n, lda = 642, 650
    slab(0)
    whole = galerk.bem_dense(dom, dom, sp, kern, sp)
    slab(96)
    host = torch.full((n * lda,), float("nan"), dtype=torch.complex128, pin_memory=True)
    galerk.bem_dense_into(dom, dom, sp, kern, sp, galerk.BemOptions(), host.data_ptr(), lda)
    a = host.numpy().reshape(n, lda)  # row c = column c of A
    assert np.isnan(a[:, n:].real).all()  # padding untouched
    assert rel_fro(a[:, :n].T, whole) <= 1e-13


def test_streamed_errors_match_whole_path(galerk, slab):
    m, dom, sp, _ = sphere_problem(galerk, 162, 3, "P1")
    opts = galerk.BemOptions()
    opts.memory_cap_bytes = 1000
    slab(16)
    with pytest.raises(RuntimeError, match="exceeds the cap"):
        galerk.bem_dense(dom, dom, sp, galerk.green_kernel("[exp(ikr)/r]", 1.0), sp, opts)


def test_config2_one_shot_default_streams_and_matches_plan_path(galerk, oracle, monkeypatch):
    """BASELINE cfg 2 through the one-shot call as bench.py's e2e leg runs it
    (default slab width, pinned destination) against the device plan path."""
    torch = _torch()
    monkeypatch.delenv("GK_SLAB_COLS", raising=False)
    monkeypatch.delenv("GK_STREAM", raising=False)
    m, dom, sp, hbar = sphere_problem(galerk, 10242, 3, "P1")
    k = 2 * math.pi / (10 * hbar)
    kern = galerk.green_kernel("[exp(ikr)/r]", k)
    n = 10242
    host = torch.empty(n * n, dtype=torch.complex128, pin_memory=True)
    galerk.bem_dense_into(dom, dom, sp, kern, sp, galerk.BemOptions(), host.data_ptr(), n)
    plan = galerk.AssemblyPlan(dom, dom, sp, kern, sp, galerk.BemOptions(), -1)
    dev = torch.empty(n * n, dtype=torch.complex128, device="cuda")
    plan.assemble(dev.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    d = dev.cpu().numpy()
    h = host.numpy()
    assert np.linalg.norm(h - d) <= 1e-13 * np.linalg.norm(d)
    rows = [0, 17, 5000, n - 1]
    ref = oracle.bem_dense(m.vertices, m.elements, 3, P1, m.vertices, m.elements, 3, P1, "[exp(ikr)/r]", k,
                           rows=rows, threads=8)
    assert rel_fro(h.reshape(n, n)[:, rows].T, ref) <= TOL
