"""Oversized dofs: a dof supported by more quadrature locations
than a tile holds (128 x locations / 112 y records) — the apex of a fan of 24
triangles with the 6- or 7-point rule has 144 / 168 — is constrained out of
the tiles and filled by k_big_entries.  The reference's bem_product has no
such limit (assembly.cpp:192-222), so the device must match the oracle here
too, through the plan, the one-shot bem_dense and a non-symmetric pairing.
"""
import math

import numpy as np
import pytest

from tests._support import colmajor_from_torch, rel_fro

P0, P1 = 0, 1
FAM = {"P0": P0, "P1": P1}
TOL = 1e-10


def double_cone(n=24, h=1.0):
    """Closed double cone: ring of n vertices, apexes of degree n (fan caps)."""
    ring = [[math.cos(2 * math.pi * i / n), math.sin(2 * math.pi * i / n), 0.0] for i in range(n)]
    v = np.array(ring + [[0.0, 0.0, h], [0.0, 0.0, -h]])
    e = []
    for i in range(n):
        j = (i + 1) % n
        e.append([n, i, j])
        e.append([n + 1, j, i])
    return v, np.array(e, dtype=np.int32)


def test_oversized_dofs_plan_on_cpu(galerk):
    v, e = double_cone()
    m = galerk.Mesh(v, e)
    for g in (3, 7):
        dom = galerk.make_domain(m, g)
        sp = galerk.make_fem(m, "P1")
        info = galerk.plan_info_dry(dom, dom, sp, galerk.green_kernel("[exp(ikr)/r]", 2.0), sp, galerk.BemOptions())
        assert info["rows"] == 26


@pytest.mark.gpu
@pytest.mark.parametrize("g,fam,name,k", [(7, "P1", "[exp(ikr)/r]", 2.0), (7, "P1", "[1/r]", 0.0),
                                          (3, "P1", "[exp(ikr)/r]", 3.0), (7, "P0", "[exp(ikr)/r]", 2.0)])
def test_oversized_dofs_match_oracle(galerk, oracle, g, fam, name, k):
    import torch

    n = 24 if g == 7 else 120  # apex locations: 24 x 7 = 168 (7-point), 120 edge midpoints (3-point)
    v, e = double_cone(n)
    m = galerk.Mesh(v, e)
    dom = galerk.make_domain(m, g)
    sp = galerk.make_fem(m, fam)
    kern = galerk.green_kernel(name, k)
    plan = galerk.AssemblyPlan(dom, dom, sp, kern, sp)
    N = plan.info()["rows"]
    A = torch.full((N * N,), float("nan"), dtype=torch.complex128, device="cuda")
    plan.assemble(A.data_ptr(), N, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = colmajor_from_torch(A, N, N, N)
    ref = oracle.bem_dense(v, e, g, FAM[fam], v, e, g, FAM[fam], name, k)
    assert not np.isnan(got).any()
    assert rel_fro(got, ref) <= TOL
    # the one-shot drop-in (whole-matrix path for oversized dofs)
    one = galerk.bem_dense(dom, dom, sp, kern, sp)
    assert rel_fro(one, ref) <= TOL


@pytest.mark.gpu
def test_oversized_dofs_nonsymmetric(galerk, oracle):
    # test side: the double cone P1 7-point (oversized apex rows); trial side:
    # a sphere P0 3-point — non-symmetric plan, big rows only
    import torch

    v, e = double_cone()
    vs, es = oracle.build_sphere(162, 1.3)
    mx, my = galerk.Mesh(v, e), galerk.Mesh(np.asarray(vs), np.asarray(es))
    dx, dy = galerk.make_domain(mx, 7), galerk.make_domain(my, 3)
    sx, sy = galerk.make_fem(mx, "P1"), galerk.make_fem(my, "P0")
    kern = galerk.green_kernel("[exp(ikr)/r]", 3.0)
    plan = galerk.AssemblyPlan(dx, dy, sx, kern, sy)
    info = plan.info()
    R, C = info["rows"], info["cols"]
    A = torch.full((R * C,), float("nan"), dtype=torch.complex128, device="cuda")
    plan.assemble(A.data_ptr(), R, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got = colmajor_from_torch(A, R, C, R)
    ref = oracle.bem_dense(v, e, 7, P1, vs, es, 3, P0, "[exp(ikr)/r]", 3.0)
    assert rel_fro(got, ref) <= TOL
    # and transposed roles: big columns
    plan2 = galerk.AssemblyPlan(dy, dx, sy, kern, sx)
    A2 = torch.full((R * C,), float("nan"), dtype=torch.complex128, device="cuda")
    plan2.assemble(A2.data_ptr(), C, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    got2 = colmajor_from_torch(A2, C, R, C)
    ref2 = oracle.bem_dense(vs, es, 3, P0, v, e, 7, P1, "[exp(ikr)/r]", 3.0)
    assert rel_fro(got2, ref2) <= TOL
