"""Derive the quarter-turn sin/cos polynomials used by the sm_100a kernels.

The device kernels reduce the phase in quarter turns:  u = k r * (2/pi),
q = rint(u), f = u - q in [-1/2, 1/2], then
    sin(pi f / 2) = f * P(f^2),   cos(pi f / 2) = Q(f^2)
with P, Q polynomials in z = f^2 on [0, 1/4].  Coefficients are Chebyshev
interpolants computed in 50-digit arithmetic (near-minimax); the script then
emulates the device Horner evaluation in IEEE double (numpy) and reports the
max error against mpmath.  Output is pasted into csrc/gk_math.cuh.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
ZMAX = mp.mpf(1) / 4
HALF_PI = mp.pi / 2


def cheb_fit(fun, deg):
    n = deg + 1
    nodes = [ZMAX / 2 * (1 - mp.cos(mp.pi * (2 * i + 1) / (2 * n))) for i in range(n)]
    A = mp.matrix([[z ** j for j in range(n)] for z in nodes])
    b = mp.matrix([fun(z) for z in nodes])
    return list(mp.lu_solve(A, b))


def p_fun(z):  # sin(pi/2 sqrt z)/sqrt z
    if z == 0:
        return HALF_PI
    s = mp.sqrt(z)
    return mp.sin(HALF_PI * s) / s


def q_fun(z):
    return mp.cos(HALF_PI * mp.sqrt(z))


def horner(coefs, z):
    acc = np.float64(coefs[-1])
    for c in reversed(coefs[:-1]):
        acc = np.float64(np.fma(acc, z, np.float64(c))) if hasattr(np, "fma") else acc * z + np.float64(c)
    return acc


def check(P, Q, n=20001):
    fs = np.linspace(-0.5, 0.5, n)
    worst_s = worst_c = 0.0
    for f in fs:
        f = float(f)
        z = f * f
        pd = float(P[-1])
        for c in reversed(P[:-1]):
            pd = float(mp.mpf(pd) * z + float(c))  # fma emulation: exact then round
        qd = float(Q[-1])
        for c in reversed(Q[:-1]):
            qd = float(mp.mpf(qd) * z + float(c))
        s = f * pd
        es = abs(s - mp.sin(HALF_PI * f))
        ec = abs(qd - mp.cos(HALF_PI * f))
        worst_s = max(worst_s, float(es))
        worst_c = max(worst_c, float(ec))
    return worst_s, worst_c


if __name__ == "__main__":
    # degrees used by gk_math.cuh: P degree 6 (7 terms), Q degree 6 (7 terms)
    P = cheb_fit(p_fun, 6)
    Q = cheb_fit(q_fun, 6)
    ws, wc = check(P, Q, 4001)
    print("max abs err sin %.3e cos %.3e" % (ws, wc))
    for name, cs in (("P", P), ("Q", Q)):
        for i, c in enumerate(cs):
            print(f"{name}{i} = {mp.nstr(c, 21)}")
