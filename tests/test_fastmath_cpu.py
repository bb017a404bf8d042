"""The GPU path's polynomial and reduction constants (csrc/gvx_math.cuh kCoef) are
checked on the CPU: each polynomial, evaluated exactly (mpmath) with the double
coefficients as written in the table, must approximate its function to the bound
DESIGN.md §5 budgets on the range its Cody-Waite reduction produces. A typo in a
constant fails here before any GPU run."""
import os
import re

import mpmath as mp
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2312_02756_b200", "csrc", "gvx_math.cuh")
mp.mp.dps = 40


def table():
    src = open(SRC).read()
    body = re.search(r"__constant__ double kCoef\[K_NCOEF\] = \{(.*?)\};", src, re.S).group(1)
    body = re.sub(r"//[^\n]*", "", body)
    vals = [float(x) for x in re.findall(r"[-+]?\d[\d.]*(?:e[-+]?\d+)?", body)]
    enum = re.search(r"enum : int \{(.*?)\};", src, re.S).group(1)
    enum = re.sub(r"//[^\n]*", "", enum)
    idx, i = {}, 0
    for tok in [t.strip() for t in enum.split(",") if t.strip()]:
        if "=" in tok:
            name, v = [x.strip() for x in tok.split("=")]
            i = int(v)
        else:
            name = tok
        idx[name] = i
        i += 1
    assert len(vals) == idx["K_NCOEF"], (len(vals), idx["K_NCOEF"])
    return vals, idx


def horner(coefs, z):
    p = mp.mpf(coefs[0])
    for c in coefs[1:]:
        p = p * z + mp.mpf(c)
    return p


def grid(a, b, n=400):
    return [a + (b - a) * mp.mpf(i) / n for i in range(n + 1)]


@pytest.fixture(scope="module")
def K():
    return table()


def test_exp_even_odd(K):
    v, ix = K
    qe = v[ix["K_EXP_QE"]:ix["K_EXP_QE"] + 4]
    qo = v[ix["K_EXP_QO"]:ix["K_EXP_QO"] + 4]
    L = mp.log(2) / 2
    worst = 0
    for r in grid(-L * (1 + mp.mpf(1e-12)), L * (1 + mp.mpf(1e-12))):
        s = r * r
        E = 1 + s * (mp.mpf(0.5) + s * horner(qe, s))
        O = r * (1 + s * (mp.mpf(0.16666666666666666) + s * horner(qo, s)))
        worst = max(worst, abs(E - mp.cosh(r)) / mp.cosh(r), abs(O - mp.sinh(r)))
    assert worst < 5e-16, worst


def test_sin_cos_quarter(K):
    v, ix = K
    P = v[ix["K_SIN"]:ix["K_SIN"] + 6]
    Q = v[ix["K_COSQ"]:ix["K_COSQ"] + 5]
    R = mp.pi / 4 * (1 + mp.mpf(1e-12))
    ws = wc = 0
    for r in grid(-R, R):
        z = r * r
        ws = max(ws, abs(r - r ** 3 * horner(P, z) - mp.sin(r)))
        wc = max(wc, abs(1 + z * (mp.mpf(-0.5) + z * horner(Q, z)) - mp.cos(r)))
    assert ws < 3e-16 and wc < 1e-15, (ws, wc)


def test_cos_half(K):
    v, ix = K
    C = v[ix["K_COSH"]:ix["K_COSH"] + 9]
    R = mp.pi / 2 * (1 + mp.mpf(1e-12))
    w = max(abs(horner(C, r * r) - mp.cos(r)) for r in grid(-R, R))
    assert w < 5e-16, w


def test_reduction_constants(K):
    v, ix = K
    assert abs(mp.mpf(v[ix["K_LN2_HI"]]) + mp.mpf(v[ix["K_LN2_LO"]]) - mp.log(2)) < 1e-25
    assert abs(mp.mpf(v[ix["K_PI_HI"]]) + mp.mpf(v[ix["K_PI_LO"]]) - mp.pi) < 1e-31
    assert abs(mp.mpf(v[ix["K_PIO2_HI"]]) + mp.mpf(v[ix["K_PIO2_LO"]]) - mp.pi / 2) < 1e-31
    # k * LN2_HI must be exact for |k| < 2^10: LN2_HI has <= 43 significant bits
    m, e = mp.frexp(mp.mpf(v[ix["K_LN2_HI"]]))
    assert (m * 2 ** 43) == int(m * 2 ** 43)
    assert abs(v[ix["K_LOG2E"]] - float(1 / mp.log(2))) == 0
    assert abs(v[ix["K_INV_PI"]] - float(1 / mp.pi)) == 0
    assert abs(v[ix["K_2_PI"]] - float(2 / mp.pi)) == 0
