"""Pins for the CPU oracle (oracle/) against things other than itself.

Each test checks the oracle against what the paper/SPEC and mathematics fix:
the SPEC's printed worked examples (tests/golden/spec_examples.json), closed
forms named in BASELINE.json's north_star, invariants (Lorentz invariance,
metric preservation, β then −β), 40-digit mpmath truth computed along a
DIFFERENT algebraic route than the oracle's (so a dropped term, a wrong sign,
a swapped sin/cos or a transposed index fails), and exact rational brute force
for the histogram binning. No expected value here comes from the CUDA path.
"""
import json
import math
import os
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")
MMU = synth.MUON_MASS
mp.mp.dps = 40


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def O(oracle_lib):
    return oracle_lib


# --------------------------------------------------------------------------
# High-precision truth along an independent route
# --------------------------------------------------------------------------

def truth_mass2_ptetaphim(a, b):
    """M² and E_lab from the rapidity-angle form (not the oracle's Cartesian sum):
    M² = m1|m1| + m2|m2| + 2(E1E2 − pt1pt2(cos(φ1−φ2) + sinh η1 sinh η2)),
    E_i = sqrt(m_i|m_i| + pt_i² cosh² η_i); valid when no E² clamp applies."""
    pt1, e1, f1, m1 = (mp.mpf(float(x)) for x in a)
    pt2, e2, f2, m2 = (mp.mpf(float(x)) for x in b)
    E1 = mp.sqrt(m1 * abs(m1) + (pt1 * mp.cosh(e1)) ** 2)
    E2 = mp.sqrt(m2 * abs(m2) + (pt2 * mp.cosh(e2)) ** 2)
    M2 = m1 * abs(m1) + m2 * abs(m2) + 2 * (E1 * E2 - pt1 * pt2 * (mp.cos(f1 - f2) + mp.sinh(e1) * mp.sinh(e2)))
    return M2, E1 + E2


def truth_boost(v, beta):
    """Boost by rapidity ζ = atanh|β| along n = β/|β| (a different route than Λ):
    E' = cosh ζ E + sinh ζ p∥,  p' = p + ((cosh ζ − 1) p∥ + sinh ζ E) n."""
    px, py, pz, E = (mp.mpf(float(x)) for x in v)
    bx, by, bz = (mp.mpf(float(x)) for x in beta)
    b = mp.sqrt(bx * bx + by * by + bz * bz)
    if b == 0:
        return [px, py, pz, E]
    nx, ny, nz = bx / b, by / b, bz / b
    z = mp.atanh(b)
    ppar = px * nx + py * ny + pz * nz
    k = (mp.cosh(z) - 1) * ppar + mp.sinh(z) * E
    return [px + k * nx, py + k * ny, pz + k * nz, mp.cosh(z) * E + mp.sinh(z) * ppar]


def signed_sq(x):
    return x * abs(x)


# --------------------------------------------------------------------------
# SPEC worked examples (golden)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_golden_conversion_at_rest(O, golden, dt):
    for ex in golden["conversion_ptetaphim_to_pxpypze"]:
        # single vector paired with the zero vector: E_lab = E, M = m
        m, e = O.invariant_mass(np.array([ex["in"]], dt), np.zeros((1, 4), dt))
        assert e[0] == ex["out"][3], ex["cite"]
        assert m[0] == ex["in"][3], ex["cite"]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_golden_mass_pxpypze(O, golden, dt):
    z = np.zeros((1, 4), dt)
    for ex in golden["mass_pxpypze"]:
        m, _ = O.invariant_mass(np.array([ex["v"]], dt), z, coords="pxpypze")
        if "mass" in ex:
            assert m[0] == ex["mass"], ex["cite"]
        else:
            assert m[0] == dt(math.sqrt(ex["mass_squared"])), ex["cite"]
    for ex in golden["batch_mass_pxpypze"] + golden["add_pxpypze"]:
        a = np.array([ex.get("v1", ex.get("a"))] * 7, dt)
        b = np.array([ex.get("v2", ex.get("b"))] * 7, dt)
        m, e = O.invariant_mass(a, b, coords="pxpypze")
        if "mass" in ex:
            assert np.all(m == ex["mass"]), ex["cite"]
        elif "mass_squared" in ex:
            assert np.all(m == dt(math.sqrt(ex["mass_squared"]))), ex["cite"]
        else:  # additive examples: check through the sum's energy and mass
            s = ex["sum"]
            assert np.all(e == s[3]), ex["cite"]
            exp_m2 = s[3] ** 2 - (s[0] ** 2 + s[1] ** 2 + s[2] ** 2)
            assert np.allclose(m * np.abs(m), exp_m2, rtol=1e-6 if dt == np.float32 else 1e-15)


def test_golden_batch_empty(O, golden):
    for dt in (np.float32, np.float64):
        m, e = O.invariant_mass(np.zeros((0, 4), dt), np.zeros((0, 4), dt))
        assert m.shape == (0,)
        out, s = O.boost(np.zeros((0, 4), dt), np.zeros((0, 3), dt))
        assert out.shape == (0, 4)
        bins, _ = O.mass_histogram(np.zeros((0, 4), dt), np.zeros((0, 4), dt), 0.25, 300.0, 1000)
        assert bins.sum() == 0


def boost_matrix_from_oracle(O, beta, dt=np.float64):
    """Columns of Λ = oracle boost applied to the 4 basis vectors."""
    basis = np.eye(4, dtype=dt)
    out, _ = O.boost(basis, np.array([beta] * 4, dt))
    return out.T  # out[j] = Λ e_j = column j


def test_golden_boost_matrix(O, golden):
    for ex in golden["boost_matrix"]:
        L = boost_matrix_from_oracle(O, ex["beta"])
        if ex.get("identity"):
            assert np.array_equal(L, np.eye(4)), ex["cite"]
            continue
        assert L[2, 2] == pytest.approx(ex["L_zz"], abs=1e-15), ex["cite"]
        assert L[2, 3] == pytest.approx(ex["L_zt"], abs=1e-15), ex["cite"]
        assert L[3, 2] == pytest.approx(ex["L_tz"], abs=1e-15), ex["cite"]
        assert L[3, 3] == pytest.approx(ex["L_tt"], abs=1e-15), ex["cite"]
        assert L[0, 0] == ex["L_xx"] and L[1, 1] == ex["L_yy"], ex["cite"]
        assert L[0, 1] == 0 and L[0, 3] == 0 and L[1, 3] == 0


def test_golden_boost_apply(O, golden):
    for ex in golden["boost_apply"]:
        m = ex["rest_mass"]
        for dt, tol in ((np.float64, 1e-15), (np.float32, 1e-6)):
            out, _ = O.boost(np.array([[0, 0, 0, m]], dt), np.array([ex["beta"]], dt))
            assert np.allclose(out[0], np.array(ex["out_over_m"]) * m, rtol=tol, atol=tol), ex["cite"]


def test_golden_boost_domain(O, golden):
    for ex in golden["boost_domain_error"]:
        with pytest.raises(O.DomainError):
            O.boost_uniform(np.zeros((3, 4)), *ex["beta"])
        out, s = O.boost(np.ones((1, 4)), np.array([ex["beta"]]))
        assert np.all(np.isnan(out)) and np.isnan(s[0]), ex["cite"]
    # |β| = 1 exactly is also rejected (b2 < 1 is required)
    out, _ = O.boost(np.ones((1, 4)), np.array([[0.0, 0.0, 1.0]]))
    assert np.all(np.isnan(out))


# --------------------------------------------------------------------------
# Closed forms from the north star
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_single_vector_mass_is_m(O, dt):
    rng = np.random.default_rng(1)
    v = np.stack([rng.uniform(1, 100, 200), rng.uniform(-2.5, 2.5, 200), rng.uniform(-np.pi, np.pi, 200),
                  rng.uniform(0.1, 90, 200)], axis=1).astype(dt)
    m, e = O.invariant_mass(v, np.zeros_like(v))
    # |M² − m²| ≤ τ·E² (τ = the north-star tolerance of the dtype)
    tau = 1e-12 if dt == np.float64 else 1e-5
    assert np.all(np.abs(signed_sq(m.astype(np.float64)) - signed_sq(v[:, 3].astype(np.float64)))
                  <= tau * e.astype(np.float64) ** 2)
    # spacelike sign convention: pt = 1, m = −0.5 → −0.5
    m, _ = O.invariant_mass(np.array([[1.0, 0.0, 0.0, -0.5]], dt), np.zeros((1, 4), dt))
    assert m[0] < 0 and m[0] == pytest.approx(-0.5, rel=4 * np.finfo(dt).eps)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_back_to_back_massless_pair(O, dt):
    # pt = 25, η = ±1.1, Δφ = π → M = 2·pt·cosh η (north star: "back-to-back massless pairs give M = 2E")
    a = np.array([[25.0, 1.1, 0.3, 0.0]], dt)
    b = np.array([[25.0, -1.1, 0.3 - math.pi, 0.0]], dt)
    m, e = O.invariant_mass(a, b)
    exact = 2 * 25 * mp.cosh(mp.mpf(float(dt(1.1))))
    tau = 1e-12 if dt == np.float64 else 1e-5
    assert abs(mp.mpf(float(m[0])) ** 2 - exact ** 2) <= tau * exact ** 2
    assert float(exact) == pytest.approx(83.425927691112816634, rel=1e-15 if dt == np.float64 else 1e-6)


def test_v_plus_v_is_twice_m(O):
    # PtEtaPhiM(3, 0.5, 1.0, 1) + itself → mass 2
    v = np.array([[3.0, 0.5, 1.0, 1.0]])
    m, _ = O.invariant_mass(v, v)
    assert m[0] == pytest.approx(2.0, abs=1e-14)


def test_spec_conversion_example_mpmath(O):
    # (10, 1.2, 0.5, 0.105) → E = sqrt(0.105² + 10² cosh² 1.2); M of (v, 0) = 0.105
    v = np.array([[10.0, 1.2, 0.5, 0.105]])
    m, e = O.invariant_mass(v, np.zeros_like(v))
    E = mp.sqrt(mp.mpf(0.105) ** 2 + 100 * mp.cosh(mp.mpf(1.2)) ** 2)
    assert abs(e[0] - E) <= 4e-16 * E
    assert float(E) == pytest.approx(18.106860118426809386, rel=1e-16)
    # the Cartesian image: boosting by β = 0 and reading back through the pxpypze mass path
    px, py, pz = 10 * mp.cos(0.5), 10 * mp.sin(0.5), 10 * mp.sinh(1.2)
    assert float(px) == pytest.approx(8.7758256189037271612, rel=1e-16)
    assert float(pz) == pytest.approx(15.09461355412172616, rel=1e-16)
    mc, ec = O.invariant_mass(np.array([[float(px), float(py), float(pz), float(E)]]), np.zeros((1, 4)),
                              coords="pxpypze")
    assert ec[0] == pytest.approx(e[0], rel=1e-16)
    assert abs(mc[0] ** 2 - m[0] ** 2) <= 1e-12 * E ** 2


def test_dimuon_pins(O):
    a = np.array([[45.0, 0.3, 0.1, MMU]])
    b = np.array([[40.0, -0.8, 2.9, MMU]])
    m, e = O.invariant_mass(a, b)
    assert m[0] == pytest.approx(96.946954876884514685, rel=1e-14)
    assert e[0] == pytest.approx(100.53785398749637737, rel=1e-15)
    # near-collinear pair (cancellation regime, M/E = 1.6e-3)
    a = np.array([[20.0, 2.4, -3.0, MMU]])
    b = np.array([[20.0, 2.39, -3.01, MMU]])
    m, e = O.invariant_mass(a, b)
    M2t, Et = truth_mass2_ptetaphim(a[0], b[0])
    assert float(mp.sqrt(M2t)) == pytest.approx(0.35306635229398653897, rel=1e-15)
    assert abs(m[0] ** 2 - M2t) <= 1e-14 * Et ** 2


# --------------------------------------------------------------------------
# Random events against 40-digit truth along the rapidity route
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt,bound", [(np.float64, 1e-14), (np.float32, 2e-6)])
def test_mass_random_vs_mpmath(O, dt, bound):
    v1, v2 = synth.muon_pairs(np.arange(400), seed=7, dtype=dt)
    # add heavier, wider-η and spacelike-free variety
    rng = np.random.default_rng(3)
    extra1 = np.stack([rng.uniform(0.5, 500, 100), rng.uniform(-5, 5, 100), rng.uniform(-20, 20, 100),
                       rng.uniform(0, 100, 100)], 1).astype(dt)
    extra2 = np.stack([rng.uniform(0.5, 500, 100), rng.uniform(-5, 5, 100), rng.uniform(-20, 20, 100),
                       rng.uniform(0, 100, 100)], 1).astype(dt)
    v1 = np.concatenate([v1, extra1])
    v2 = np.concatenate([v2, extra2])
    m, e = O.invariant_mass(v1, v2)
    worst = 0.0
    for i in range(len(m)):
        M2t, Et = truth_mass2_ptetaphim(v1[i], v2[i])
        err = abs(signed_sq(mp.mpf(float(m[i]))) - M2t) / Et ** 2
        worst = max(worst, float(err))
        assert abs(mp.mpf(float(e[i])) - Et) <= 4 * np.finfo(dt).eps * Et
    assert worst <= bound, worst


@pytest.mark.parametrize("dt,bound", [(np.float64, 1e-14), (np.float32, 1e-5)])
def test_boost_random_vs_rapidity_truth(O, dt, bound):
    v, beta = synth.boost_inputs(np.arange(300), seed=11, dtype=dt)
    out, s = O.boost(v, beta)
    worst = 0.0
    for i in range(len(v)):
        t = truth_boost(v[i], beta[i])
        S = float(s[i])
        for c in range(4):
            worst = max(worst, float(abs(mp.mpf(float(out[i, c])) - t[c])) / S)
    assert worst <= bound, worst


def test_boost_metric_preservation(O):
    # Λᵀ g Λ = g, g = diag(−1, −1, −1, +1)
    g = np.diag([-1.0, -1.0, -1.0, 1.0])
    _, beta = synth.boost_inputs(np.arange(200), seed=5)
    for b in beta:
        L = boost_matrix_from_oracle(O, b)
        assert np.max(np.abs(L.T @ g @ L - g)) <= 1e-12
        assert np.allclose(L, L.T, atol=0)  # a pure boost is symmetric


def test_boost_inverse_and_invariance(O):
    v, beta = synth.boost_inputs(np.arange(2000), seed=9)
    out, s = O.boost(v, beta)
    back, _ = O.boost(out, -beta)
    assert np.max(np.abs(back - v) / s[:, None]) <= 1e-13  # β then −β = identity
    m0, _ = O.invariant_mass(v, np.zeros_like(v), coords="pxpypze")
    m1, _ = O.invariant_mass(out, np.zeros_like(out), coords="pxpypze")
    assert np.max(np.abs(signed_sq(m1) - signed_sq(m0)) / s ** 2) <= 1e-13  # M invariant under boosts
    # rest particle → E = γm, |p| = γβm (north star), β = (0.3, −0.4, 0.5)
    out, _ = O.boost(np.array([[0.0, 0.0, 0.0, 1.0]]), np.array([[0.3, -0.4, 0.5]]))
    g = 1 / mp.sqrt(1 - mp.mpf(0.3) ** 2 - mp.mpf(0.4) ** 2 - mp.mpf(0.5) ** 2)
    assert out[0, 3] == pytest.approx(float(g), rel=2e-16)
    assert float(g) == pytest.approx(1.4142135623730950645, rel=1e-16)
    assert math.sqrt(out[0, 0] ** 2 + out[0, 1] ** 2 + out[0, 2] ** 2) == pytest.approx(1.0000000000000000222, rel=4e-16)
    assert out[0, 0] == pytest.approx(0.3 * float(g), rel=4e-16)
    assert out[0, 1] == pytest.approx(-0.4 * float(g), rel=4e-16)


def test_boost_uniform_equals_per_event(O):
    v, _ = synth.boost_inputs(np.arange(50), seed=2)
    b = (0.1, 0.2, -0.3)
    u = O.boost_uniform(v, *b)
    p, _ = O.boost(v, np.array([b] * 50))
    assert np.array_equal(u, p)


# --------------------------------------------------------------------------
# CM boost (reading R11)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_cm_mass_invariance_and_rest_frame(O, dt):
    v1, v2 = synth.muon_pairs(np.arange(3000), seed=21, dtype=dt)
    mcm, e, bo = O.cm_mass(v1, v2, want_boosted=True)
    mlab, _ = O.invariant_mass(v1, v2)
    ok = np.isfinite(mcm)
    if dt == np.float64:
        assert ok.all()
        tau = 1e-12
    else:
        tau = 1e-5
    e = e.astype(np.float64)
    assert np.all(np.abs(signed_sq(mcm[ok].astype(np.float64)) - signed_sq(mlab[ok].astype(np.float64)))
                  <= tau * e[ok] ** 2)
    if dt == np.float64:
        P = bo[:, 0:3] + bo[:, 4:7]
        E = bo[:, 3] + bo[:, 7]
        S = e ** 2 / np.maximum(mlab, 1e-300)  # γ·E scale of the CM boost
        assert np.max(np.abs(P).max(1) / S) <= 1e-14  # total momentum vanishes
        assert np.max(np.abs(E - mlab) / S) <= 1e-14  # E' = M
    # dimuon pin: E' = M
    m, _, bo = O.cm_mass(np.array([[45.0, 0.3, 0.1, MMU]]), np.array([[40.0, -0.8, 2.9, MMU]]), want_boosted=True)
    assert m[0] == pytest.approx(96.946954876884514685, rel=1e-13)
    assert bo[0, 3] + bo[0, 7] == pytest.approx(96.946954876884514685, rel=1e-13)


def test_cm_degenerate(O):
    # already at rest in the CM: β = 0 → boosted = input
    a = np.array([[3.0, 4.0, 5.0, 13.0]])
    b = np.array([[-3.0, -4.0, -5.0, 13.0]])
    m, _, bo = O.cm_mass(a, b, coords="pxpypze", want_boosted=True)
    assert m[0] == 26.0 and np.array_equal(bo[0], np.concatenate([a[0], b[0]]))
    # zero-energy pair → NaN (reading R11) → overflow bin
    z = np.zeros((1, 4))
    m, _ = O.cm_mass(z, z)
    assert np.isnan(m[0])
    bins, _ = O.mass_histogram(z, z, 0.25, 300.0, 1000, cm=True)
    assert bins[1001] == 1 and bins.sum() == 1
    # lightlike collinear pair: β² = 1 → NaN
    a = np.array([[0.0, 0.0, 5.0, 5.0]])
    m, _ = O.cm_mass(a, a, coords="pxpypze")
    assert np.isnan(m[0])


# --------------------------------------------------------------------------
# Histogram binning vs exact rational brute force
# --------------------------------------------------------------------------

def brute_bin(x, lo, hi, nbins):
    """Scan the edges lo + b·(hi−lo)/nbins exactly (rationals)."""
    if math.isnan(x):
        return nbins + 1
    if math.isinf(x):
        return 0 if x < 0 else nbins + 1
    X, L, H = Fraction(x), Fraction(lo), Fraction(hi)
    if X < L:
        return 0
    if X >= H:
        return nbins + 1
    w = (H - L) / nbins
    for b in range(1, nbins + 1):
        if L + (b - 1) * w <= X < L + b * w:
            return b
    raise AssertionError


def test_find_bin_vs_brute_force(O):
    lo, hi, nb = 0.25, 300.0, 1000
    rng = np.random.default_rng(0)
    xs = list(rng.uniform(lo - 20, hi + 20, 3000)) + [lo, hi, -0.0, 0.0, float("nan"), float("inf"),
                                                      -float("inf"), np.nextafter(lo, -1), np.nextafter(hi, -1)]
    w = (hi - lo) / nb
    for x in xs:
        b_or = O.find_bin(x, lo, hi, nb)
        b_bf = brute_bin(x, lo, hi, nb)
        # the only allowed disagreement: within float tolerance of an interior edge
        near_edge = (lo <= x < hi) and abs((x - lo) / w - round((x - lo) / w)) < 1e-9
        assert b_or == b_bf or near_edge, (x, b_or, b_bf)
    assert O.find_bin(float("nan"), lo, hi, nb) == nb + 1
    assert O.find_bin(hi, lo, hi, nb) == nb + 1
    assert O.find_bin(lo, lo, hi, nb) == 1
    assert O.find_bin(-0.0, 0.0, 1.0, 10) == 1
    assert O.find_bin(0.15, 0.0, 1.0, 10) == brute_bin(0.15, 0.0, 1.0, 10)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("cm", [False, True])
def test_histogram_is_bincount_of_masses(O, dt, cm):
    v1, v2 = synth.muon_pairs(np.arange(5000), seed=4, dtype=dt)
    bins, m = O.mass_histogram(v1, v2, 0.25, 300.0, 1000, cm=cm)
    assert bins.sum() == 5000
    ref = np.zeros(1002, np.uint64)
    for x in m:
        ref[brute_bin(float(x), 0.25, 300.0, 1000)] += 1
    assert np.array_equal(bins, ref)
    if cm:
        mm, _ = O.cm_mass(v1, v2)
    else:
        mm, _ = O.invariant_mass(v1, v2)
    assert np.array_equal(m, mm, equal_nan=True)
    # accumulation: a second call adds
    O.mass_histogram(v1, v2, 0.25, 300.0, 1000, cm=cm, bins=bins)
    assert np.array_equal(bins, 2 * ref)


def test_histogram_single_bin_stress(O):
    # every pair has the same mass → all counts in one bin
    v = np.tile(np.array([[0.0, 0.0, 0.0, 45.5]]), (1000, 1))
    bins, _ = O.mass_histogram(v, v, 0.25, 300.0, 1000, coords="pxpypze")
    b = brute_bin(91.0, 0.25, 300.0, 1000)
    assert bins[b] == 1000 and bins.sum() == 1000


# --------------------------------------------------------------------------
# Other 4D coordinate systems
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_pxpypzm_closed_forms(O, dt):
    z = np.zeros((1, 4), dt)
    # |p| = 13 (3-4-12): m = 0 -> lightlike; m = 5 -> E = sqrt(194), mass 5
    m, e = O.invariant_mass(np.array([[3, 4, 12, 0]], dt), z, coords="pxpypzm")
    assert m[0] == 0 and e[0] == 13
    m, e = O.invariant_mass(np.array([[3, 4, 12, 5]], dt), z, coords="pxpypzm")
    assert m[0] == pytest.approx(5, rel=8 * np.finfo(dt).eps) and e[0] == dt(np.sqrt(194.0))
    # spacelike m = -5: E^2 = 169 - 25 = 144 -> M = -5 (R3/R4)
    m, e = O.invariant_mass(np.array([[3, 4, 12, -5]], dt), z, coords="pxpypzm")
    assert e[0] == 12 and m[0] == pytest.approx(-5, rel=8 * np.finfo(dt).eps)
    # clamp (R2): m = -20 -> E = 0, M = -|p| = -13
    m, e = O.invariant_mass(np.array([[3, 4, 12, -20]], dt), z, coords="pxpypzm")
    assert e[0] == 0 and m[0] == -13


def test_coordinate_systems_agree(O):
    """The same physical pairs written in all four systems give the same mass (mpmath
    conversions at 40 digits, independent of the oracle's own conversion code)."""
    v1, v2 = synth.muon_pairs(np.arange(300), seed=13)
    def forms(v):
        out = {k: [] for k in ("ptetaphim", "pxpypze", "pxpypzm", "ptetaphie")}
        for pt, eta, phi, m in v:
            pt, eta, phi, m = (mp.mpf(float(x)) for x in (pt, eta, phi, m))
            px, py, pz = pt * mp.cos(phi), pt * mp.sin(phi), pt * mp.sinh(eta)
            E = mp.sqrt(m * m + px * px + py * py + pz * pz)
            out["ptetaphim"].append([float(pt), float(eta), float(phi), float(m)])
            out["pxpypze"].append([float(px), float(py), float(pz), float(E)])
            out["pxpypzm"].append([float(px), float(py), float(pz), float(m)])
            out["ptetaphie"].append([float(pt), float(eta), float(phi), float(E)])
        return {k: np.array(x) for k, x in out.items()}
    f1, f2 = forms(v1), forms(v2)
    ref, e = O.invariant_mass(f1["ptetaphim"], f2["ptetaphim"])
    for c in ("pxpypze", "pxpypzm", "ptetaphie"):
        m, _ = O.invariant_mass(f1[c], f2[c], coords=c)
        assert np.max(np.abs(m * np.abs(m) - ref * np.abs(ref)) / e ** 2) <= 1e-14, c
        mc, _ = O.cm_mass(f1[c], f2[c], coords=c)
        assert np.max(np.abs(mc * np.abs(mc) - ref * np.abs(ref)) / e ** 2) <= 1e-13, c


def test_ptetaphie_single_vector_mpmath(O):
    rng = np.random.default_rng(17)
    v = np.stack([rng.uniform(1, 100, 100), rng.uniform(-3, 3, 100), rng.uniform(-np.pi, np.pi, 100),
                  np.zeros(100)], 1)
    v[:, 3] = v[:, 0] * np.cosh(v[:, 1]) * rng.uniform(1.0, 1.5, 100)  # timelike E
    m, e = O.invariant_mass(v, np.zeros_like(v), coords="ptetaphie")
    for i in range(100):
        pt, eta, E = (mp.mpf(float(x)) for x in (v[i, 0], v[i, 1], v[i, 3]))
        M2 = E * E - (pt * mp.cosh(eta)) ** 2
        assert abs(mp.mpf(float(m[i])) ** 2 - M2) <= 1e-14 * E * E


# --------------------------------------------------------------------------
# Jagged dimuon selection (reading R21)
# --------------------------------------------------------------------------

def test_dimuon_selection_brute_force(O):
    mu, q, off = synth.jagged_events(0, 20_000, seed=3)
    bins, m, sel = O.dimuon_histogram(mu, q, off, 0.25, 300.0, 1000)
    k = np.diff(off)
    expect_sel = 0
    ref = np.zeros(1002, np.uint64)
    for e in range(off.size - 1):
        a, b = off[e], off[e + 1]
        if b - a == 2 and q[a] != q[a + 1]:  # exactly two, opposite charge (q = ±1)
            expect_sel += 1
            mm, _ = O.invariant_mass(mu[a:a + 1], mu[a + 1:a + 2])
            assert m[e] == mm[0]
            ref[O.find_bin(float(mm[0]), 0.25, 300.0, 1000)] += 1
        else:
            assert np.isnan(m[e])
    assert sel == expect_sel == int(bins.sum())
    assert np.array_equal(bins, ref)
    # the multiplicity / charge recipe: P(k = 2) = 0.30, opposite charges half of those
    assert abs((k == 2).mean() - 0.30) < 0.01
    assert abs(sel / off.size - 0.15) < 0.01


def test_dimuon_closed_forms(O):
    m_mu = synth.MUON_MASS
    mu = np.array([[45, 0.3, 0.1, m_mu], [40, -0.8, 2.9, m_mu],     # event 0: opposite -> selected
                   [45, 0.3, 0.1, m_mu], [40, -0.8, 2.9, m_mu],     # event 1: same sign -> rejected
                   [25, 1.1, 0.3, 0], [25, -1.1, 0.3 - np.pi, 0],   # event 2: back-to-back massless
                   [10, 0, 0, m_mu], [10, 0, 1, m_mu], [10, 0, 2, m_mu]])  # event 3: three muons -> rejected
    q = np.array([1, -1, -1, -1, 1, -1, 1, -1, 1], np.int32)
    off = np.array([0, 2, 4, 6, 9, 9])  # event 4: empty
    bins, m, sel = O.dimuon_histogram(mu, q, off, 0.25, 300.0, 1000)
    assert sel == 2
    assert m[0] == pytest.approx(96.946954876884514685, rel=1e-14)
    assert m[2] == pytest.approx(2 * 25 * np.cosh(1.1), rel=1e-12)
    assert np.isnan(m[1]) and np.isnan(m[3]) and np.isnan(m[4])
    # no events
    bins, m, sel = O.dimuon_histogram(np.zeros((0, 4)), np.zeros(0, np.int32), np.zeros(1, np.int64), 0.25, 300.0, 1000)
    assert sel == 0 and m.size == 0


# --------------------------------------------------------------------------
# General 4x4 Lorentz transformation (f2)
# --------------------------------------------------------------------------

def rot_z(theta):
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[c, -s, 0, 0], [s, c, 0, 0], [0, 0, 1, 0], [0, 0, 0, 1.0]])


def test_lorentz_transform_pins(O):
    v, beta = synth.boost_inputs(np.arange(500), seed=19)
    # a pure boost matrix (columns = oracle boost of the basis) reproduces the uniform boost bitwise (f64)
    b = (0.3, -0.4, 0.5)
    L = boost_matrix_from_oracle(O, b)
    assert np.array_equal(O.lorentz_transform(v, L), O.boost_uniform(v, *b))
    # a quarter turn about z: (px, py) -> (-py, px) exactly (cos(pi/2) rounds to 6e-17)
    out = O.lorentz_transform(np.array([[1.0, 2.0, 3.0, 10.0]]), rot_z(math.pi / 2))
    assert np.allclose(out[0], [-2.0, 1.0, 3.0, 10.0], atol=1e-15)
    # identity
    assert np.array_equal(O.lorentz_transform(v, np.eye(4)), v)
    # composition Λ(β)·R(θ): metric preserved, masses invariant, equals boost(rotate(v))
    LR = L @ rot_z(0.7)
    out = O.lorentz_transform(v, LR)
    two = O.boost_uniform(O.lorentz_transform(v, rot_z(0.7)), *b)
    assert np.max(np.abs(out - two) / v[:, 3:4]) <= 1e-14
    m0, _ = O.invariant_mass(v, np.zeros_like(v), coords="pxpypze")
    m1, _ = O.invariant_mass(out, np.zeros_like(out), coords="pxpypze")
    assert np.max(np.abs(m1 * np.abs(m1) - m0 * np.abs(m0)) / (v[:, 3] * 3) ** 2) <= 1e-13
    # not Lorentz (a plain scaling) -> domain error (SPEC.md:191 spirit: invalid transforms rejected)
    with pytest.raises(O.DomainError):
        O.lorentz_transform(v, 2 * np.eye(4))
    with pytest.raises(O.DomainError):
        O.lorentz_transform(v, np.full((4, 4), np.nan))


# --------------------------------------------------------------------------
# CM decay angle cos θ* (reading R22)
# --------------------------------------------------------------------------

def _rest_frame_decay_in_lab(pstar, theta, phi, m, beta):
    """Two-body decay at rest (vector 1 at polar angle θ, azimuth φ; vector 2 opposite),
    then boosted into the lab by β along the rapidity route (mpmath, 40 digits)."""
    with mp.workdps(40):
        ps, th, ph, mm = (mp.mpf(x) for x in (pstar, theta, phi, m))
        E = mp.sqrt(ps * ps + mm * mm)
        p1 = [ps * mp.sin(th) * mp.cos(ph), ps * mp.sin(th) * mp.sin(ph), ps * mp.cos(th), E]
        p2 = [-p1[0], -p1[1], -p1[2], E]
        return [float(x) for x in truth_boost(p1, beta)], [float(x) for x in truth_boost(p2, beta)]


def test_costheta_recovers_rest_frame_angle(O):
    """Closed form: boosting a rest-frame decay by β and then applying the CM path gives back
    the rest-frame angle, because β_cm = −P/E = −β and two pure boosts along one axis
    compose to the identity (no Wigner rotation)."""
    rng = np.random.default_rng(3)
    rows1, rows2, want, gam = [], [], [], []
    for _ in range(300):
        th = rng.uniform(0, np.pi)
        ph = rng.uniform(-np.pi, np.pi)
        pstar = rng.uniform(1.0, 60.0)
        d = rng.normal(size=3)
        b = 0.99 * rng.uniform() ** (1 / 3) * d / np.linalg.norm(d)
        a, c = _rest_frame_decay_in_lab(pstar, th, ph, MMU, b)
        rows1.append(a)
        rows2.append(c)
        want.append(math.cos(th))
        gam.append(1 / math.sqrt(1 - b @ b))
    v1, v2 = np.array(rows1), np.array(rows2)
    _, _, m, cos = O.cm_costheta(v1, v2, coords="pxpypze")
    err = np.abs(cos - np.array(want))
    # input rounding (1e-16 relative on lab components ~ γE) maps to ~γ² 1e-16 E/p* in cos θ*
    assert err.max() <= 1e-12, err.max()
    # swapping the two vectors flips the angle (p2' = −p1' in the CM)
    _, _, _, cos_sw = O.cm_costheta(v2, v1, coords="pxpypze")
    assert np.max(np.abs(cos_sw + cos)) <= 1e-12
    # f32: same pins at the fp32 scale (γ ≤ 7.1 here)
    _, _, _, c32 = O.cm_costheta(v1.astype(np.float32), v2.astype(np.float32), coords="pxpypze")
    g = np.array(gam)
    assert np.all(np.abs(c32.astype(np.float64) - want) <= 2e-5 * g * g)


def _truth_costheta(a, b):
    """cos θ* along the rapidity route: β_cm = −P/E, vector 1 boosted by truth_boost."""
    with mp.workdps(40):
        A = [mp.mpf(float(x)) for x in a]
        B = [mp.mpf(float(x)) for x in b]
        E = A[3] + B[3]
        beta = [-(A[k] + B[k]) / E for k in range(3)]
        p = truth_boost(A, beta)
        return float(p[2] / mp.sqrt(p[0] ** 2 + p[1] ** 2 + p[2] ** 2)), float(E), float(
            mp.sqrt(p[0] ** 2 + p[1] ** 2 + p[2] ** 2))


@pytest.mark.parametrize("dt,bound", [(np.float64, 1e-13), (np.float32, 5e-6)])
def test_costheta_random_vs_rapidity_truth(O, dt, bound):
    v1, v2 = synth.muon_pairs(np.arange(400), seed=31, dtype=dt)
    _, _, mcm, cos = O.cm_costheta(v1, v2)
    # truth from the Cartesian inputs the oracle itself forms (the conversion is pinned elsewhere)
    a = np.array([[x[0] * np.cos(x[2]), x[0] * np.sin(x[2]), x[0] * np.sinh(x[1]),
                   np.sqrt(x[3] ** 2 + (x[0] * np.cosh(x[1])) ** 2)] for x in v1.astype(np.float64)])
    b = np.array([[x[0] * np.cos(x[2]), x[0] * np.sin(x[2]), x[0] * np.sinh(x[1]),
                   np.sqrt(x[3] ** 2 + (x[0] * np.cosh(x[1])) ** 2)] for x in v2.astype(np.float64)])
    worst = 0.0
    for i in range(v1.shape[0]):
        t, E, pstar = _truth_costheta(a[i], b[i])
        S = E * E / max(float(mcm[i]), 1e-300)  # γ·E scale of the CM boost (as for M_cm)
        worst = max(worst, abs(float(cos[i]) - t) * pstar / S)
    assert worst <= bound, worst
    assert np.all(np.abs(cos.astype(np.float64)) <= 1 + 4 * np.finfo(dt).eps)


def test_costheta_degenerate_and_histograms(O):
    # pair at rest back to back along +z: β = 0, cos θ* = 1 exactly → overflow bin of [−1, 1)
    a = np.array([[0.0, 0.0, 3.0, 5.0], [4.0, 0.0, 0.0, 5.0], [0.0, 0.0, -3.0, 5.0]])
    b = np.array([[0.0, 0.0, -3.0, 5.0], [-4.0, 0.0, 0.0, 5.0], [0.0, 0.0, 3.0, 5.0]])
    mb, cb, m, c = O.cm_costheta(a, b, coords="pxpypze", c_axis=(-1.0, 1.0, 4))
    assert np.array_equal(c, [1.0, 0.0, -1.0]) and np.array_equal(m, [10.0, 10.0, 10.0])
    assert cb.tolist() == [0, 1, 0, 1, 0, 1]  # −1 → bin 1, 0 → bin 3, +1 → overflow
    # zero pair, lightlike collinear pair → NaN (reading R11) → overflow of both axes
    z = np.zeros((2, 4))
    z[1] = [0.0, 0.0, 5.0, 5.0]
    mb, cb, m, c = O.cm_costheta(z, np.array([[0.0] * 4, [0.0, 0.0, 5.0, 5.0]]), coords="pxpypze")
    assert np.isnan(m).all() and np.isnan(c).all() and mb[-1] == 2 and cb[-1] == 2
    # the histograms are the bincounts of the per-event values; mass axis == the CM histogram
    v1, v2 = synth.muon_pairs(np.arange(5000), seed=4, dtype=np.float64)
    mb, cb, m, c = O.cm_costheta(v1, v2, c_axis=(-1.0, 1.0, 50))
    ref_m, _ = O.mass_histogram(v1, v2, 0.25, 300.0, 1000, cm=True)
    assert np.array_equal(mb, ref_m)
    ref_c = np.zeros(52, np.uint64)
    for x in c:
        ref_c[O.find_bin(float(x), -1.0, 1.0, 50)] += 1
    assert np.array_equal(cb, ref_c)
    # isotropic-ish sample: both hemispheres populated, accumulation doubles
    assert cb[1:26].sum() > 1000 and cb[26:51].sum() > 1000
    mb2, cb2, _, _ = O.cm_costheta(v1, v2, c_axis=(-1.0, 1.0, 50), m_bins=mb.copy(), c_bins=cb.copy())
    assert np.array_equal(cb2, 2 * cb) and np.array_equal(mb2, 2 * mb)


def test_boost_high_beta_stress(O):
    """Reading R10's fp64 stress set: |β| up to 0.9999 (γ ≈ 71). The literal Λ stays within
    τ·S of the rapidity-route truth (the rounding of 1 − β² grows as 1/(1 − β²))."""
    rng = np.random.default_rng(77)
    n = 300
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    mag = np.concatenate([np.full(n // 3, 0.999), np.full(n // 3, 0.9995), np.full(n - 2 * (n // 3), 0.9999)])
    beta = d * mag[:, None]
    v, _ = synth.boost_inputs(np.arange(n), seed=3)
    out, S = O.boost(v, beta)
    worst = 0.0
    for i in range(n):
        t = truth_boost(v[i], beta[i])
        worst = max(worst, max(abs(float(out[i, k]) - float(t[k])) for k in range(4)) / float(S[i]))
    assert worst <= 1e-12, worst


# --------------------------------------------------------------------------
# The boost tolerance scale S = γ(E + |β||p|) (reading R5), pinned by closed forms
# --------------------------------------------------------------------------

@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_boost_scale_closed_forms(O, dt):
    """S is the denominator of every boost parity check, so it is pinned to quantities
    computed along the rapidity route, not by retyping its formula:
    * a massless vector along β̂ has E' = γ(1 + |β|)E (the Doppler factor), and S = E' there;
    * a particle at rest has E' = γm and S = γm;
    * for physical vectors (|p| ≤ E) S bounds every row of |Λ|·|v| and is within 2× of the
      largest row: max_r Σ_j |Λ_rj||v_j| ≤ S ≤ 2 max_r Σ_j |Λ_rj||v_j|."""
    eps = float(np.finfo(dt).eps)
    rng = np.random.default_rng(404)
    for bmag in (0.1, 0.5, 0.9, 0.99):
        for _ in range(6):
            n = rng.normal(size=3)
            n /= np.linalg.norm(n)
            for E in (1.0, 37.5):
                v = np.array([[E * n[0], E * n[1], E * n[2], E]], dt)
                beta = np.array([bmag * n], dt)
                _, s = O.boost(v, beta)
                Ep = truth_boost(v[0], beta[0])[3]  # the boosted energy, rapidity route
                g2 = 1 / (1 - bmag * bmag)
                assert abs(mp.mpf(float(s[0])) - Ep) <= 16 * eps * g2 * Ep, (bmag, E, float(s[0]), float(Ep))
                # and the closed form γ(1+β)E = E·sqrt((1+β)/(1−β)) itself
                assert float(Ep) == pytest.approx(E * math.sqrt((1 + bmag) / (1 - bmag)), rel=64 * eps * g2)
            # rest particle of mass m: S = γm = E'
            m = 0.1056583755 if dt == np.float64 else 5.0
            v = np.array([[0.0, 0.0, 0.0, m]], dt)
            beta = np.array([bmag * n], dt)
            _, s = O.boost(v, beta)
            Ep = truth_boost(v[0], beta[0])[3]
            assert abs(mp.mpf(float(s[0])) - Ep) <= 16 * eps * g2 * Ep
    # random physical events: S bounds |Λ|·|v| row by row, tightly (40-digit Λ from β)
    v, beta = synth.boost_inputs(np.arange(300), seed=13, dtype=dt)
    _, s = O.boost(v, beta)
    for i in range(len(v)):
        bx, by, bz = (mp.mpf(float(x)) for x in beta[i])
        b2 = bx * bx + by * by + bz * bz
        g = 1 / mp.sqrt(1 - b2)
        bg = g * g / (1 + g)
        b = [bx, by, bz]
        L = [[(1 if r == c else 0) + bg * b[r] * b[c] for c in range(3)] + [g * b[r]] for r in range(3)]
        L.append([g * bx, g * by, g * bz, g])
        av = [abs(mp.mpf(float(x))) for x in v[i]]
        rows = max(sum(abs(L[r][c]) * av[c] for c in range(4)) for r in range(4))
        S = mp.mpf(float(s[i]))
        assert rows * (1 - 64 * eps) <= S <= 2 * rows * (1 + 64 * eps), (i, float(S), float(rows))


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_ptetaphim_energy_clamp(O, dt):
    """Reading R2 (SPEC.md:81 is silent on m·|m| + pt² + pz² < 0): E² is clamped to 0, so a
    spacelike vector whose |m| exceeds its |p| has E = 0 and, alone, mass −|p|:
    (pt=1, η=0, φ=0, m=−5): E² = −24 → E = 0, M² = −1, M = −1;
    (3, 0, 0, −4): E² = −7 → E = 0, M = −3; (3, 0, 0, −3): E² = 0 → E = 0, M = −3.
    (√|E²| instead of the clamp would give E = √24 and M = +√23.)"""
    z = np.zeros((1, 4), dt)
    for v, M in (((1.0, 0.0, 0.0, -5.0), -1.0), ((3.0, 0.0, 0.0, -4.0), -3.0), ((3.0, 0.0, 0.0, -3.0), -3.0),
                 ((2.0, 0.0, 1.0, -7.5), -2.0)):
        m, e = O.invariant_mass(np.array([v], dt), z)
        # (φ = 1: cos² + sin² is 1 only to a few ulp)
        assert e[0] == 0.0 and m[0] == pytest.approx(M, rel=4 * np.finfo(dt).eps), (v, float(e[0]), float(m[0]))
    # a clamped vector in a pair: E_lab = E of the other vector only; M² = E2² − |p1 + p2|²
    a = np.array([[1.0, 0.0, 0.0, -5.0]], dt)   # p = (1, 0, 0), E = 0
    b = np.array([[4.0, 0.0, 0.0, 3.0]], dt)    # p = (4, 0, 0), E = 5
    m, e = O.invariant_mass(a, b)
    assert e[0] == 5.0 and m[0] == 0.0         # M² = 25 − 25
    # the same clamp on the CM path: the pair (a, b) is lightlike, E = 5 > 0, β = −1 → NaN (R11)
    mc, _ = O.cm_mass(a, b)
    assert np.isnan(mc[0])


def test_boost_unit_speed_is_a_domain_error(O):
    """|β| ≥ 1 → domain error — |β| = 1 exactly included (pre: b² < 1)."""
    for b in ((0.0, 0.0, 1.0), (-1.0, 0.0, 0.0), (0.0, 1.0, 0.0)):
        for dt in (np.float64, np.float32):
            with pytest.raises(O.DomainError):
                O.boost_uniform(np.ones((2, 4), dt), *b)


def test_cm_conversion_components_spec_example(O):
    """The Cartesian components of the conversion, seen through the CM boost (a pair's mass alone
    only sees cos(φ1 − φ2), which a px <-> py swap leaves unchanged): SPEC.md:88's vector
    a = PtEtaPhiM(10, 1.2, 0.5, 0.105) and SPEC.md:87's rest vector b = (0, 0, 0, 5). In the CM
    frame b' is the rest particle boosted by β_cm = −p_a/(E_a + 5), so its momentum is
    5γβ_cm = −5γ p_a/(E_a + 5) with p_a = (10 cos 0.5, 10 sin 0.5, 10 sinh 1.2), at 40 digits."""
    a = np.array([[10.0, 1.2, 0.5, 0.105]])
    b = np.array([[0.0, 0.0, 0.0, 5.0]])
    m, _, bo = O.cm_mass(a, b, want_boosted=True)
    p = [10 * mp.cos(mp.mpf(0.5)), 10 * mp.sin(mp.mpf(0.5)), 10 * mp.sinh(mp.mpf(1.2))]
    Ea = mp.sqrt(mp.mpf(0.105) ** 2 + 100 * mp.cosh(mp.mpf(1.2)) ** 2)
    E = Ea + 5
    beta = [-x / E for x in p]
    g = 1 / mp.sqrt(1 - sum(x * x for x in beta))
    for k in range(3):
        want = 5 * g * beta[k]
        assert abs(bo[0, 4 + k] - want) <= 1e-14 * E, (k, bo[0, 4 + k], float(want))
        assert abs(bo[0, k] + want) <= 1e-14 * E  # p'_a = −p'_b in the CM frame
    assert abs(bo[0, 7] - 5 * g) <= 1e-14 * E
    assert float(p[0]) == pytest.approx(8.7758256189037271612, rel=1e-16)   # S:88 as printed
    assert float(p[1]) == pytest.approx(4.7942553860420300027, rel=1e-16)


def test_cm_negative_energy_pair_has_no_rest_frame(O):
    """Reading R11: β_cm = −P/E needs E > 0. A pair with negative total energy and P = 0 has
    β_cm = 0 (|β| < 1) but no centre-of-mass frame: its CM mass is NaN (→ overflow bin)."""
    a = np.array([[0.0, 0.0, 0.0, -5.0]])
    b = np.array([[0.0, 0.0, 0.0, -3.0]])
    m, _ = O.cm_mass(a, b, coords="pxpypze")
    assert np.isnan(m[0])
    bins, _ = O.mass_histogram(a, b, 0.25, 300.0, 1000, cm=True, coords="pxpypze")
    assert bins[1001] == 1
    # the lab mass of the same pair is defined: E² − p² = 64 → 8
    ml, _ = O.invariant_mass(a, b, coords="pxpypze")
    assert ml[0] == 8.0


# --------------------------------------------------------------------------
# Mixed-coordinate pairs ("two particles expressed in any 4-dimensional
# coordinate system")
# --------------------------------------------------------------------------

SYSTEMS = ("ptetaphim", "pxpypze", "pxpypzm", "ptetaphie")


def mp_cartesian(system, comps):
    """40-digit PxPyPzE of a vector given in `system` (R2 clamp)."""
    a, b, c, d = (mp.mpf(float(x)) for x in comps)
    if system in ("ptetaphim", "ptetaphie"):
        px, py, pz = a * mp.cos(c), a * mp.sin(c), a * mp.sinh(b)
        if system == "ptetaphie":
            return px, py, pz, d
        e2 = d * abs(d) + a * a + pz * pz
        return px, py, pz, mp.sqrt(max(e2, 0))
    if system == "pxpypze":
        return a, b, c, d
    e2 = a * a + b * b + c * c + d * abs(d)
    return a, b, c, mp.sqrt(max(e2, 0))


def represent(system, pt, eta, phi, m):
    """The physics vector (pt, η, φ, m) written in `system` at 40 digits, then rounded."""
    pt, eta, phi, m = (mp.mpf(float(x)) for x in (pt, eta, phi, m))
    px, py, pz = pt * mp.cos(phi), pt * mp.sin(phi), pt * mp.sinh(eta)
    E = mp.sqrt(m * m + (pt * mp.cosh(eta)) ** 2)
    return {"ptetaphim": (pt, eta, phi, m), "pxpypze": (px, py, pz, E), "pxpypzm": (px, py, pz, m),
            "ptetaphie": (pt, eta, phi, E)}[system]


def test_mixed_pair_closed_form(O):
    """SPEC.md:88's vector in PtEtaPhiM and its mirror image in PxPyPzE with the components S:88
    prints, (−px, −py, −pz, E): back to back with equal energies, so M = 2E (to the 20 printed
    digits). A swapped or mis-signed Cartesian component anywhere breaks it by O(1)."""
    a = np.array([[10.0, 1.2, 0.5, 0.105]])
    b = np.array([[-8.7758256189037271612, -4.7942553860420300027, -15.09461355412172616, 18.106860118426809386]])
    for dt in (np.float64, np.float32):
        m, e = O.invariant_mass(a.astype(dt), b.astype(dt), coords="ptetaphim", coords2="pxpypze")
        assert e[0] == pytest.approx(2 * 18.106860118426809386, rel=4 * np.finfo(dt).eps)
        tau = 1e-12 if dt == np.float64 else 1e-5
        assert abs(float(m[0]) ** 2 - (2 * 18.106860118426809386) ** 2) <= tau * float(e[0]) ** 2, (dt, m[0])
        # the other order, and the CM path (already at rest: M_cm = M)
        m2, _ = O.invariant_mass(b.astype(dt), a.astype(dt), coords="pxpypze", coords2="ptetaphim")
        assert m2[0] == m[0]
        mc, _ = O.cm_mass(a.astype(dt), b.astype(dt), coords="ptetaphim", coords2="pxpypze")
        assert abs(float(mc[0]) ** 2 - (2 * 18.106860118426809386) ** 2) <= tau * float(e[0]) ** 2


@pytest.mark.parametrize("dt,bound", [(np.float64, 1e-14), (np.float32, 2e-6)])
def test_mixed_pairs_vs_cartesian_mpmath(O, dt, bound):
    """Every (system of v1, system of v2) combination against the 40-digit all-Cartesian mass of the
    same rounded inputs: |M²_oracle − M²_truth| ≤ bound·E_lab². The same physics pair written in
    different systems gives the same mass to that bound. Lab and CM masses and the
    histogram agree with the same-system calls when the systems coincide."""
    v1, v2 = synth.muon_pairs(np.arange(60), seed=31)
    for s1 in SYSTEMS:
        for s2 in SYSTEMS:
            a = np.array([[float(x) for x in represent(s1, *r)] for r in v1], dt)
            b = np.array([[float(x) for x in represent(s2, *r)] for r in v2], dt)
            m, e = O.invariant_mass(a, b, coords=s1, coords2=s2)
            for i in range(len(m)):
                p = mp_cartesian(s1, a[i])
                q = mp_cartesian(s2, b[i])
                E = p[3] + q[3]
                M2 = E * E - sum((p[k] + q[k]) ** 2 for k in range(3))
                err = abs(signed_sq(mp.mpf(float(m[i]))) - M2) / E ** 2
                assert err <= bound, (s1, s2, i, float(err))
                assert abs(mp.mpf(float(e[i])) - E) <= 8 * np.finfo(dt).eps * E
            if s1 == s2:
                ms, es = O.invariant_mass(a, b, coords=s1)
                assert np.array_equal(ms, m) and np.array_equal(es, e)
            # CM mass = lab mass (Lorentz invariance) for the mixed pair too
            mc, _ = O.cm_mass(a, b, coords=s1, coords2=s2)
            ok = np.isfinite(mc)
            if dt == np.float64:
                assert ok.all()
            tau = 1e-12 if dt == np.float64 else 1e-5
            assert np.all(np.abs(signed_sq(mc[ok].astype(np.float64)) - signed_sq(m[ok].astype(np.float64)))
                          <= tau * e[ok].astype(np.float64) ** 2)
            h, hm = O.mass_histogram(a, b, 0.25, 300.0, 1000, coords=s1, coords2=s2)
            assert np.array_equal(hm, m) and int(h.sum()) == len(m)
