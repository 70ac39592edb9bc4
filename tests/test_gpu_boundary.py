"""Boundary entry points added in round 2:

* gk_evaluate_blocks / Kernel::evaluate_blocks — the kept reference API
  kernels.hpp:37-39 (kernels.cpp:76-131) as a device panel, including the
  mask=false raising path with the reference's "(i,j)" message
  (kernels.cpp:104-108), checked against the oracle and, where built, the
  reference's own kernels.cpp (oracle/_ref);
* gk_plan_set_wavenumber — one plan serving a frequency sweep.
"""
import math

import numpy as np
import pytest

from tests._support import colmajor_from_torch, load_ref, rel_fro, sphere_problem

pytestmark = pytest.mark.gpu
ref = load_ref()


@pytest.mark.parametrize("name,k", [("[exp(ikr)/r]", 3.7), ("[exp(ikr)/r]", 66.8), ("[1/r]", 4.0)])
def test_evaluate_blocks_panel(galerk, oracle, name, k):
    rng = np.random.default_rng(17)
    X = rng.normal(size=(300, 3))
    Y = np.vstack([rng.normal(size=(200, 3)), X[:7]])  # coincident pairs: masked to 0
    eps = oracle.singular_guard_radius(X, Y)
    got = galerk.evaluate_blocks(X, Y, galerk.green_kernel(name, k), eps, True)
    want = oracle.evaluate(name, k, X, Y, True, eps)
    assert got.shape == (300, 207)
    assert rel_fro(got, want) <= 1e-13
    assert np.count_nonzero(got == 0) == 7
    if name == "[1/r]":
        assert np.all(got.imag == 0.0)
    if ref is not None:
        assert rel_fro(got, ref.evaluate(name, k, X, Y, True, eps)) <= 1e-13


def test_evaluate_blocks_raises_like_the_reference(galerk, oracle):
    X = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [2.0, 0.0, 0.0]])
    Y = np.array([[5.0, 0.0, 0.0], [2.0, 0.0, 0.0], [1.0, 0.0, 0.0]])  # pairs (2,1) and (1,2) coincide
    eps = oracle.singular_guard_radius(X, Y)
    with pytest.raises(RuntimeError) as e_dev:
        galerk.evaluate_blocks(X, Y, galerk.green_kernel("[exp(ikr)/r]", 2.0), eps, False)
    with pytest.raises(RuntimeError) as e_or:
        oracle.evaluate("[exp(ikr)/r]", 2.0, X, Y, False, eps)
    assert "(2,1)" in str(e_dev.value)  # first in the reference's loop order: j outer, i inner
    assert str(e_dev.value) == str(e_or.value)
    if ref is not None:
        with pytest.raises(RuntimeError) as e_ref:
            ref.evaluate("[exp(ikr)/r]", 2.0, X, Y, False, eps)
        assert str(e_dev.value) == str(e_ref.value)


def test_plan_frequency_sweep(galerk, oracle):
    import torch

    m, dom, sp, hbar = sphere_problem(galerk, 642, 3, "P1")
    plan = galerk.AssemblyPlan(dom, dom, sp, galerk.green_kernel("[exp(ikr)/r]", 1.0), sp)
    n = plan.info()["rows"]
    A = torch.empty(n * n, dtype=torch.complex128, device="cuda")
    for k in (1.0, 2 * math.pi / (10 * hbar), 0.0, 25.0):
        plan.set_wavenumber(k)
        plan.assemble(A.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        want = oracle.bem_dense(m.vertices, m.elements, 3, 1, m.vertices, m.elements, 3, 1, "[exp(ikr)/r]", k,
                                threads=8)
        assert rel_fro(colmajor_from_torch(A, n, n, n), want) <= 1e-10, k
    # a "[1/r]" plan keeps k = 0 (kernels.cpp:47-49)
    lap = galerk.AssemblyPlan(dom, dom, sp, galerk.green_kernel("[1/r]", 0.0), sp)
    lap.set_wavenumber(5.0)
    lap.assemble(A.data_ptr(), n, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = colmajor_from_torch(A, n, n, n)
    assert np.all(got.imag == 0.0)
    want = oracle.bem_dense(m.vertices, m.elements, 3, 1, m.vertices, m.elements, 3, 1, "[1/r]", 0.0, threads=8)
    assert rel_fro(got, want) <= 1e-10
    with pytest.raises(ValueError):
        plan.set_wavenumber(float("nan"))
