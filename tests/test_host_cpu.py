"""CPU-side checks of the product: host tables bit-identical to the oracle,
reference error behaviour at the API, and the C-ABI exports (no GPU needed)."""
import ctypes
import math
import re

import numpy as np
import pytest

from tests._support import ROOT

P0, P1 = 0, 1


@pytest.mark.parametrize("n", [12, 162, 642, 10242])
def test_build_sphere_bitwise_equals_oracle(galerk, oracle, n):
    m = galerk.build_sphere(n, 1.0)
    v, e = oracle.build_sphere(n, 1.0)
    assert np.array_equal(m.vertices, v) and np.array_equal(m.elements, e)
    assert galerk.edge_stats(m).mean_len == oracle.edge_stats(v, e)[2]


def test_perturbed_sphere_bitwise_equals_oracle(galerk, oracle):
    m = galerk.perturb_radial(galerk.build_sphere(10242, 1.0), 2, 0.02)
    v, e = oracle.build_sphere(10242, 1.0)
    v2, _ = oracle.perturb_radial(v, e, 2, 0.02)
    assert np.array_equal(m.vertices, v2)
    r = np.linalg.norm(m.vertices, axis=1)
    assert r.min() >= 0.98 - 1e-15 and r.max() <= 1.02 + 1e-15


@pytest.mark.parametrize("gauss", [1, 3, 6, 7])
def test_quadrature_bitwise_equals_oracle(galerk, oracle, gauss):
    m = galerk.build_sphere(642, 1.0)
    pts, w, elem = galerk.quadrature(galerk.make_domain(m, gauss))
    opts, ow, oelem = oracle.quadrature(m.vertices, m.elements, gauss)
    assert np.array_equal(pts, opts) and np.array_equal(w, ow) and list(elem) == list(oelem)


def test_rng_streams(galerk, oracle):
    assert np.array_equal(galerk.uniform01(7, 1000), oracle.uniform01_stream(7, 1000))
    z = galerk.complex_normal(1, 20000)
    assert abs(z.real.mean()) < 0.03 and abs(z.imag.std() - 1) < 0.03
    # Box-Muller, cos branch first
    u = galerk.uniform01(3, 2)
    assert galerk.normal(3, 1)[0] == math.sqrt(-2 * math.log(1 - u[0])) * math.cos(2 * math.pi * u[1])


def test_reference_error_behaviour(galerk):
    m = galerk.build_sphere(12, 1.0)
    with pytest.raises(ValueError, match="1,3,7"):
        galerk.make_domain(m, 5)  # test_quadrature.cpp:35
    with pytest.raises(ValueError):
        galerk.make_fem(m, "Q7")
    with pytest.raises(ValueError):
        galerk.green_kernel("[foo]", 1.0)
    assert galerk.green_kernel("[1/r]", 3.0).wavenumber() == 0.0  # kernels.cpp:47-49
    dom = galerk.make_domain(m, 3)
    p1 = galerk.make_fem(m, "P1")
    tiny = galerk.BemOptions()
    tiny.memory_cap_bytes = 1000
    with pytest.raises(RuntimeError, match="tol"):  # test_assembly.cpp:176-179
        galerk.bem_dense(dom, dom, p1, galerk.green_kernel("[exp(ikr)/r]", 2.0), p1, tiny)
    with pytest.raises(ValueError, match=r"\(1,3,1\)"):  # contraction(), assembly.cpp:44-46
        galerk.bem_dense(dom, dom, p1, galerk.green_kernel("grady[1/r]", 0.0), p1)
    with pytest.raises(ValueError, match="custom"):
        galerk.bem_dense(dom, dom, p1, galerk.Kernel.custom(1), p1)
    assert galerk.radiation_dense(np.zeros((0, 3)), dom, galerk.green_kernel("[1/r]", 0), p1).shape == (0, 12)


def test_config3_memory_cap_refuses_at_defaults(galerk):
    m = galerk.perturb_radial(galerk.build_sphere(10242, 1.0), 2, 0.02)
    dom = galerk.make_domain(m, 6)
    p0 = galerk.make_fem(m, "P0")
    with pytest.raises(RuntimeError, match="tol"):  # SURVEY trap 5: 9.06e9 > 8e9
        galerk.AssemblyPlan(dom, dom, p0, galerk.green_kernel("[exp(ikr)/r]", 15.0), p0)


def _header_functions():
    text = open(f"{ROOT}/include/galerk_b200.h").read()
    return sorted(set(re.findall(r"\b(gk_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_exports_every_declared_symbol():
    lib = ctypes.CDLL(f"{ROOT}/paper_1804_00995_b200/_build/libgalerk_b200.so")
    names = _header_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    lib.gk_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.gk_version()


def test_c_abi_argument_errors_without_device():
    lib = ctypes.CDLL(f"{ROOT}/paper_1804_00995_b200/_build/libgalerk_b200.so")
    lib.gk_last_error.restype = ctypes.c_char_p
    # null sides -> GK_EINVAL before any device work
    out = ctypes.c_void_p()
    assert lib.gk_plan_create(None, None, None, None, ctypes.byref(out)) == 1
    assert b"null" in lib.gk_last_error()
    assert lib.gk_matvec(None, -1, 0, 0, None, None, None) == 1
    i64, vp = ctypes.c_int64, ctypes.c_void_p
    lib.gk_matvec_multi.argtypes = [vp, i64, i64, i64, vp, i64, vp, i64, ctypes.c_int32, vp]
    assert lib.gk_matvec_multi(None, 4, 4, 4, None, 4, None, 4, -1, None) == 1
    assert b"negative" in lib.gk_last_error()


def test_no_cpu_fallback(galerk):
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    m = galerk.build_sphere(12, 1.0)
    dom = galerk.make_domain(m, 3)
    p1 = galerk.make_fem(m, "P1")
    with pytest.raises(RuntimeError, match="no CUDA device"):
        galerk.bem_dense(dom, dom, p1, galerk.green_kernel("[1/r]", 0.0), p1)


@pytest.mark.parametrize("nv,fam,gauss", [(40962, "P0", 3), (10242, "P1", 7), (2562, "P1", 3)])
def test_threaded_location_numbering_equals_serial(galerk, nv, fam, gauss):
    """Large sides number their locations on several host threads (hash-sharded,
    gk_plan.cpp build_locations); the ids must be the serial first-seen ones,
    so plans (and matrices) do not depend on the host's thread count."""
    import numpy as np

    g = galerk
    mesh = g.build_sphere(nv, 1.0)
    dom = g.make_domain(mesh, gauss)
    sp = g.make_fem(mesh, fam)
    loc_t, n_t, xyz_t = g.location_ids(dom, sp, False)
    loc_s, n_s, xyz_s = g.location_ids(dom, sp, True)
    assert n_t == n_s
    assert np.array_equal(loc_t, loc_s)
    assert np.array_equal(np.asarray(xyz_t)[: 3 * n_t], np.asarray(xyz_s)[: 3 * n_s])
    # first-seen order: ids appear in increasing order of their first point
    first = np.full(n_s, -1, dtype=np.int64)
    ids = np.asarray(loc_s)
    _, idx = np.unique(ids, return_index=True)
    assert np.array_equal(np.sort(idx), idx)  # id u's first point precedes id u+1's
    pts, _, _ = g.quadrature(dom)
    pts = np.asarray(pts).reshape(-1, 3)
    assert np.array_equal(np.asarray(xyz_s)[: 3 * n_s].reshape(-1, 3)[ids], pts + 0.0)
