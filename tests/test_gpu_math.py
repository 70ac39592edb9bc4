"""GPU: accuracy of the device scalar math the kernels are built from (gk_math.cuh).

Every transcendental on the hot path is hand-written (quarter-turn sin/cos of
the pair kernel, the refined reciprocal square root, and the near-field
kernel's quotient-free log, division and branch-free atan2), so each one is
checked here against numpy's extended precision (x86 80-bit long double) on
seeded arguments spanning the ranges the kernels feed them.  Bounds are in
ulps of the double result (sin/cos: absolute, as their polynomials are fitted
for absolute error on [-1/2, 1/2] quarter turns).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

LOG_RATIO, ATAN2, DIV, SIN_Q, COS_Q, RSQRT = range(6)
PI_L = np.longdouble("3.14159265358979323846264338327950288")


def _run(galerk, fn, a, b=None):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    da = torch.tensor(a, dtype=torch.float64, device="cuda")
    db = torch.tensor(b, dtype=torch.float64, device="cuda") if b is not None else None
    out = torch.empty_like(da)
    galerk.diag_math(fn, len(a), da.data_ptr(), db.data_ptr() if db is not None else 0, out.data_ptr(), 0)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _ulps(got, exact):
    exact = np.asarray(exact, dtype=np.longdouble)
    err = np.abs(got.astype(np.longdouble) - exact)
    return (err / np.spacing(np.abs(exact.astype(np.float64)))).astype(np.float64)


def _rng():
    return np.random.default_rng(20261020)


def test_log_ratio(galerk):
    rng = _rng()
    n = 200000
    # the edge logs see ratios near 1 (far points) up to ~1e12 (near a vertex)
    num = np.exp(rng.uniform(-28, 28, n)) * rng.uniform(0.5, 2, n)
    log_ratio = np.concatenate([rng.uniform(-1e-6, 1e-6, n // 4), rng.uniform(-0.5, 0.5, n // 4),
                                rng.uniform(-3, 3, n // 4), rng.uniform(-28, 28, n - 3 * (n // 4))])
    den = num * np.exp(log_ratio)
    got = _run(galerk, LOG_RATIO, num, den)
    nl, dl = num.astype(np.longdouble), den.astype(np.longdouble)
    # log1p of the (exact) difference near 1: a long-double quotient would carry
    # more error than the device result there
    near = np.abs(nl / dl - 1) < 0.25
    exact = np.where(near, np.log1p((nl - dl) / dl), np.log(nl / dl))
    big = np.abs(exact) > 1e-300
    u = _ulps(got[big], exact[big])
    assert np.percentile(u, 99.9) <= 2.0 and u.max() <= 4.0, (u.max(), np.percentile(u, 99.9))


def test_atan2(galerk):
    rng = _rng()
    n = 200000
    ang = rng.uniform(-np.pi, np.pi, n)
    r = np.exp(rng.uniform(-20, 20, n))
    y, x = r * np.sin(ang), r * np.cos(ang)
    got = _run(galerk, ATAN2, y, x)
    exact = np.arctan2(y.astype(np.longdouble), x.astype(np.longdouble))
    u = _ulps(got, exact)
    assert u.max() <= 2.0, u.max()
    # the solid angle at a vertex hits atan2(0, 0): 0, finite
    z = _run(galerk, ATAN2, np.zeros(2), np.array([0.0, 1.0]))
    assert np.all(z == 0.0)


def test_div(galerk):
    rng = _rng()
    n = 200000
    d = rng.uniform(-10, 10, n) * np.exp(rng.uniform(-5, 5, n))
    s = np.exp(rng.uniform(-20, 20, n))
    got = _run(galerk, DIV, d, s)
    exact = d.astype(np.longdouble) / s.astype(np.longdouble)
    u = _ulps(got, exact)
    assert u.max() <= 1.0, u.max()


def test_sincos_quarter(galerk):
    rng = _rng()
    # phases u = k r 2/pi up to ~170 quarter turns (cfg 5: max kr = 134)
    u = np.concatenate([rng.uniform(-0.5, 0.5, 100000), rng.uniform(0, 170, 100000)])
    s = _run(galerk, SIN_Q, u)
    c = _run(galerk, COS_Q, u)
    ang = PI_L / 2 * u.astype(np.longdouble)
    es = np.abs(s.astype(np.longdouble) - np.sin(ang)).max()
    ec = np.abs(c.astype(np.longdouble) - np.cos(ang)).max()
    # polynomial error 3.6e-15 (sin, degree 5) / 1.75e-16 (cos, degree 6)
    # plus the rounding of f = u - q (scripts/derive_polys.py); odd quadrants
    # swap the two polynomials, so both outputs carry the sine's error
    assert es <= 4e-15 and ec <= 4e-15, (float(es), float(ec))


def test_rsqrt(galerk):
    rng = _rng()
    x = np.exp(rng.uniform(-60, 60, 200000))
    got = _run(galerk, RSQRT, x)
    exact = 1 / np.sqrt(x.astype(np.longdouble))
    u = _ulps(got, exact)
    assert u.max() <= 1.0, u.max()
