#!/usr/bin/env python
"""Near-minimax (Chebyshev-fit) coefficients for the fp64 polynomials of
csrc/gvx_math.cuh, at a chosen number of terms, with the max error of the
double-rounded coefficients on the reduced range (mpmath, 40 digits).
Usage: python tools/fit_poly.py  -> prints candidate tables and their errors."""
import mpmath as mp

mp.mp.dps = 40


def fit(f, a, b, n):
    """Chebyshev fit of f on [a, b] with n coefficients (highest degree first)."""
    c, err = mp.chebyfit(f, [a, b], n, error=True)
    return [float(x) for x in c]


def horner(c, z):
    p = mp.mpf(c[0])
    for x in c[1:]:
        p = p * z + mp.mpf(x)
    return p


def grid(a, b, n=2000):
    return [a + (b - a) * mp.mpf(i) / n for i in range(n + 1)]


def exp_split(nq):
    L = mp.log(2) / 2 * (1 + mp.mpf(1e-12))
    s_hi = L * L
    fe = lambda s: (mp.cosh(mp.sqrt(s)) - 1 - s / 2) / (s * s) if s > 0 else mp.mpf(1) / 24
    fo = lambda s: (mp.sinh(mp.sqrt(s)) / mp.sqrt(s) - 1 - s / 6) / (s * s) if s > 0 else mp.mpf(1) / 120
    qe, qo = fit(fe, 0, s_hi, nq), fit(fo, 0, s_hi, nq)
    w = 0
    for r in grid(-L, L):
        s = r * r
        E = 1 + s * (mp.mpf(0.5) + s * horner(qe, s))
        O = r * (1 + s * (mp.mpf(0.16666666666666666) + s * horner(qo, s)))
        w = max(w, abs(E - mp.cosh(r)) / mp.cosh(r), abs(O - mp.sinh(r)))
    return qe, qo, w


def sin_cos_quarter(nsin, ncos):
    R = mp.pi / 4 * (1 + mp.mpf(1e-12))
    fs = lambda z: (mp.sqrt(z) - mp.sin(mp.sqrt(z))) / (z * mp.sqrt(z)) if z > 0 else mp.mpf(1) / 6
    fc = lambda z: (mp.cos(mp.sqrt(z)) - 1 + z / 2) / (z * z) if z > 0 else mp.mpf(1) / 24
    P, Q = fit(fs, 0, R * R, nsin), fit(fc, 0, R * R, ncos)
    ws = wc = 0
    for r in grid(-R, R):
        z = r * r
        ws = max(ws, abs(r - r ** 3 * horner(P, z) - mp.sin(r)))
        wc = max(wc, abs(1 + z * (mp.mpf(-0.5) + z * horner(Q, z)) - mp.cos(r)))
    return P, Q, ws, wc


if __name__ == "__main__":
    for nq in (4, 3, 2):
        qe, qo, w = exp_split(nq)
        print(f"exp even/odd, {nq} coefs each (degree {2 * nq + 2}/{2 * nq + 3}): max err {float(w):.3e}")
        print("  QE", qe)
        print("  QO", qo)
    for ns, nc in ((6, 5), (5, 4), (4, 4)):
        P, Q, ws, wc = sin_cos_quarter(ns, nc)
        print(f"sin {ns} / cos {nc} coefs: sin err {float(ws):.3e}, cos err {float(wc):.3e}")
        print("  SIN", P)
        print("  COSQ", Q)
