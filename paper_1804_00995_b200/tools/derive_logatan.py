"""Derive the reduced-argument log and atan polynomials of the near-field kernel (K3).

gk_nearfield.cu evaluates, after its argument reductions,
    log((1+s)/(1-s)) = 2 s + s z R(z),   z = s^2, |s| <= (sqrt2-1)/(sqrt2+1)   (log_ratio)
    atan(s)          =   s + s z P(z),   z = s^2, |s| <= tan(pi/16)            (atan2_fast)
R and P used to be the truncated Taylor series (9 and 11 terms).  Here they are
Chebyshev interpolants in z computed in 50-digit arithmetic (near-minimax), so
that fewer terms reach the same accuracy.  The script emulates the device
evaluation in IEEE double (Horner with fused multiply-adds, then the final
fused step) and prints the max error in ulps of the result for each degree,
for the Taylor series and for the fits; the chosen coefficients are pasted into
csrc/gk_nearfield.cu.
"""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
S_LOG = (mp.sqrt(2) - 1) / (mp.sqrt(2) + 1)
S_ATAN = mp.tan(mp.pi / 16)


def r_fun(z):  # (log((1+s)/(1-s)) - 2s) / (s z)
    if z == 0:
        return mp.mpf(2) / 3
    s = mp.sqrt(z)
    return (mp.log((1 + s) / (1 - s)) - 2 * s) / (s * z)


def p_fun(z):  # (atan(s) - s) / (s z)
    if z == 0:
        return -mp.mpf(1) / 3
    s = mp.sqrt(z)
    return (mp.atan(s) - s) / (s * z)


def cheb_fit(fun, zmax, deg):
    n = deg + 1
    nodes = [zmax / 2 * (1 - mp.cos(mp.pi * (2 * i + 1) / (2 * n))) for i in range(n)]
    A = mp.matrix([[z ** j for j in range(n)] for z in nodes])
    b = mp.matrix([fun(z) for z in nodes])
    return [float(c) for c in mp.lu_solve(A, b)]


def fma(a, b, c):  # one rounding
    return float(mp.mpf(a) * mp.mpf(b) + mp.mpf(c))


def ulp(x):
    return float(np.spacing(abs(np.float64(x))))


def worst_log(R, n=3001):
    w = 0.0
    for s in np.linspace(-float(S_LOG), float(S_LOG), n):
        s = float(s)
        if s == 0.0:
            continue
        z = s * s
        r = R[-1]
        for c in reversed(R[:-1]):
            r = fma(r, z, c)
        v = fma(s * z, r, 2.0 * s)
        exact = mp.log((1 + mp.mpf(s)) / (1 - mp.mpf(s)))
        w = max(w, abs(float(mp.mpf(v) - exact)) / ulp(float(exact)))
    return w


def worst_atan(P, n=3001):
    w = 0.0
    for s in np.linspace(-float(S_ATAN), float(S_ATAN), n):
        s = float(s)
        if s == 0.0:
            continue
        z = s * s
        p = P[-1]
        for c in reversed(P[:-1]):
            p = fma(p, z, c)
        v = fma(s * z, p, s)
        exact = mp.atan(mp.mpf(s))
        w = max(w, abs(float(mp.mpf(v) - exact)) / ulp(float(exact)))
    return w


if __name__ == "__main__":
    taylor_r = [2.0 / (2 * k + 3) for k in range(9)]
    taylor_p = [(-1) ** (k + 1) / (2 * k + 3) for k in range(11)]
    print("log: Taylor 9 terms  max %.2f ulp" % worst_log(taylor_r))
    for deg in (5, 6, 7):
        R = cheb_fit(r_fun, S_LOG ** 2, deg)
        print("log: Chebyshev deg %d (%d terms) max %.2f ulp" % (deg, deg + 1, worst_log(R)), R)
    print("atan: Taylor 11 terms max %.2f ulp" % worst_atan(taylor_p))
    for deg in (5, 6, 7):
        P = cheb_fit(p_fun, S_ATAN ** 2, deg)
        print("atan: Chebyshev deg %d (%d terms) max %.2f ulp" % (deg, deg + 1, worst_atan(P)), P)
