"""Derivation of the device polynomials in paper_1804_00995_b200/csrc/gk_math.cuh:
Chebyshev interpolants (in z = f^2) of the quarter-turn sine and cosine,
sin(pi f / 2) = f P(f^2), cos(pi f / 2) = Q(f^2) for f in [-1/2, 1/2], computed
from 40-digit mpmath values and converted to the power basis; prints the
coefficients and the max abs error of their double-precision Horner
evaluation on a dense grid.  (The device's cosine coefficients come from an
earlier fit of the same kind, 1.75e-16 measured; its sine is this script's
degree-5 output.)  The device copies are checked on the GPU by
tests/test_gpu_math.py.

    python scripts/derive_polys.py [sin_degree cos_degree]   (device: 5 6)
"""
import sys

import mpmath as mp
import numpy as np
from numpy.polynomial import chebyshev as C

mp.mp.dps = 40


def fit(fun, deg, zmax, n=3000):
    k = np.arange(n)
    zn = np.cos(np.pi * (k + 0.5) / n)
    z = (zn + 1) / 2 * zmax
    y = np.array([float(fun(mp.mpf(v))) for v in z])
    p = C.cheb2poly(C.chebfit(zn, y, deg))
    return np.polynomial.Polynomial(p)(np.polynomial.Polynomial([-1, 2 / zmax])).coef


def horner(c, z):
    acc = np.full_like(z, c[-1])
    for a in c[-2::-1]:
        acc = acc * z + a
    return acc


def main():
    ds, dc = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (5, 6)
    sin_p = fit(lambda z: mp.sin(mp.pi / 2 * mp.sqrt(z)) / mp.sqrt(z) if z > 0 else mp.pi / 2, ds, 0.25)
    cos_q = fit(lambda z: mp.cos(mp.pi / 2 * mp.sqrt(z)), dc, 0.25)
    f = np.linspace(-0.5, 0.5, 20001)
    ts = np.array([float(mp.sin(mp.pi / 2 * mp.mpf(x))) for x in f])
    tc = np.array([float(mp.cos(mp.pi / 2 * mp.mpf(x))) for x in f])
    es = np.abs(f * horner(sin_p, f * f) - ts).max()
    ec = np.abs(horner(cos_q, f * f) - tc).max()
    print(f"sin degree {ds} in z: max abs error {es:.2e}")
    print("  c_sinP =", ", ".join(repr(float(c)) for c in sin_p))
    print(f"cos degree {dc} in z: max abs error {ec:.2e}")
    print("  c_cosQ =", ", ".join(repr(float(c)) for c in cos_q))


if __name__ == "__main__":
    main()
