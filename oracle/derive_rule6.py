"""Derive the symmetric 6-point degree-4 triangle rule used by config 3.

TEST/BUILD INFRASTRUCTURE. The reference (`proj/src/quadrature.cpp:126-136`)
supports only 1/3/7-point triangle rules; BASELINE config 3 asks for a 6-point
rule, so both the oracle and the product add the same new rule.  The rule has
two S21 orbits (a,a,1-2a) and (b,b,1-2b) with per-point weights wa, wb.  The
four unknowns are fixed by exactness on the S3-invariant polynomials of degree
<= 4 on the reference triangle (1, e2, e3, e2^2 in the barycentric elementary
symmetric functions), whose normalised moments are
    E[1] = 1, E[e2] = 1/4, E[e3] = 1/60, E[e2^2] = 1/15
(from  (1/|T|) int lam1^p lam2^q lam3^r = 2 p! q! r! / (p+q+r+2)!).
Solved with mpmath Newton at 40 digits; prints the constants written into
oracle/galerk_oracle.cpp and paper_1804_00995_b200/csrc/host/quadrature.cpp.
"""
import mpmath as mp

mp.mp.dps = 40


def orbit(a):
    e2 = 2 * a - 3 * a * a
    e3 = a * a * (1 - 2 * a)
    return e2, e3


def equations(a, b, wa, wb):
    ea2, ea3 = orbit(a)
    eb2, eb3 = orbit(b)
    return [
        3 * wa + 3 * wb - 1,
        3 * wa * ea2 + 3 * wb * eb2 - mp.mpf(1) / 4,
        3 * wa * ea3 + 3 * wb * eb3 - mp.mpf(1) / 60,
        3 * wa * ea2 ** 2 + 3 * wb * eb2 ** 2 - mp.mpf(1) / 15,
    ]


def solve():
    # start: one orbit near the edge midpoints, one near the vertices
    sol = mp.findroot(lambda a, b, wa, wb: equations(a, b, wa, wb), (0.44, 0.09, 0.22, 0.11))
    a, b, wa, wb = sol
    return a, b, wa, wb


if __name__ == "__main__":
    a, b, wa, wb = solve()
    res = equations(a, b, wa, wb)
    assert max(abs(r) for r in res) < mp.mpf(10) ** -35
    assert wa > 0 and wb > 0 and 0 < a < 0.5 and 0 < b < 0.5
    for name, v in (("a", a), ("b", b), ("wa", wa), ("wb", wb)):
        print(f"{name} = {mp.nstr(v, 25)}")
