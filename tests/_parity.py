"""Parity predicates shared by the GPU tests (test infrastructure only).

Tolerances are the north star's (BASELINE.json): |ΔM²| ≤ τ·E² and
component-wise |Δ| ≤ τ·E, τ = 1e-12 (f64) / 1e-5 (f32), with the scales of
DESIGN.md reading R5 (E_lab for masses, S = γ(E + |β||p|) for boosts), and the
histogram exemption rule of reading R14.
"""
from __future__ import annotations

import numpy as np

TAU = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}


def tau_of(dtype) -> float:
    return TAU[np.dtype(dtype)]


def energy_scale(O, v1, v2, coords="ptetaphim"):
    """Reading R5: the "E" of |ΔM²| ≤ τ·E² is Σ_i max(E_i, |p_i|) — equal to the oracle's
    E_lab = E1 + E2 for every timelike or lightlike vector, and the right rounding scale
    for spacelike inputs whose E² the conversion clamps to 0 (R2)."""
    z = np.zeros_like(v1)
    _, e1 = O.invariant_mass(v1, z, coords=coords)
    _, e2 = O.invariant_mass(v2, z, coords=coords)
    a = np.asarray(v1, np.float64)
    b = np.asarray(v2, np.float64)
    with np.errstate(over="ignore", invalid="ignore"):
        if coords == "ptetaphim":
            p1 = np.abs(a[:, 0]) * np.cosh(a[:, 1])
            p2 = np.abs(b[:, 0]) * np.cosh(b[:, 1])
        else:
            p1 = np.sqrt((a[:, :3] ** 2).sum(1))
            p2 = np.sqrt((b[:, :3] ** 2).sum(1))
        return np.fmax(e1.astype(np.float64), p1) + np.fmax(e2.astype(np.float64), p2)


def mass_violations(m_gpu, m_ref, e_lab, tau):
    """Indices where the GPU mass breaks |M_g|M_g| − M_o|M_o|| ≤ τ·E_lab², or where
    exactly one side is non-finite."""
    g = np.asarray(m_gpu, np.float64)
    o = np.asarray(m_ref, np.float64)
    e = np.asarray(e_lab, np.float64)
    fin_g, fin_o = np.isfinite(g), np.isfinite(o)
    bad = fin_g != fin_o
    both = fin_g & fin_o
    with np.errstate(invalid="ignore", over="ignore"):
        err = np.abs(g * np.abs(g) - o * np.abs(o))
        lim = tau * e * e
    bad |= both & ~(err <= lim)
    return np.nonzero(bad)[0]


def boost_violations(out_gpu, out_ref, scale, tau):
    g = np.asarray(out_gpu, np.float64)
    o = np.asarray(out_ref, np.float64)
    s = np.asarray(scale, np.float64)
    fin_g, fin_o = np.isfinite(g), np.isfinite(o)
    bad = (fin_g != fin_o).any(axis=1)
    with np.errstate(invalid="ignore"):
        err = np.where(fin_g & fin_o, np.abs(g - o), 0.0).max(axis=1)
    bad |= ~(err <= tau * np.where(np.isfinite(s), s, np.inf))
    return np.nonzero(bad)[0]


def find_bin_np(x, lo, hi, nbins):
    """Vectorised ROOT FindFixBin in double (same operation order as the oracle)."""
    x = np.asarray(x, np.float64)
    with np.errstate(invalid="ignore"):
        q = (float(nbins) * (x - lo)) / (hi - lo)
        inner = 1 + np.trunc(np.where(np.isfinite(q), q, 0)).astype(np.int64)
    b = np.where(x < lo, 0, np.where(~(x < hi), nbins + 1, inner))
    return b.astype(np.int64)


def hist_check(h_gpu, m_ref, e_lab, tau, lo, hi, nbins, nan_possible=None, m_window_center=None):
    """Reading R14. Returns ``(failures, n_ambiguous)`` (no failures = pass).

    δ_i = τ·E_i² / max(|M_i|, √τ·E_i); event i is ambiguous if an edge of the axis lies
    within δ_i of its oracle mass M_i. Events flagged in ``nan_possible`` may also land in
    the overflow bin; their window is centred on ``m_window_center`` (the lab mass) when
    the oracle's own mass is NaN. See hist_check_delta for the rule itself."""
    m = np.asarray(m_ref, np.float64).copy()
    e = np.asarray(e_lab, np.float64)
    nanp = np.zeros(m.size, bool) if nan_possible is None else np.asarray(nan_possible, bool)
    if m_window_center is not None:
        c = np.asarray(m_window_center, np.float64)
        m = np.where(np.isnan(m) & nanp, c, m)
    with np.errstate(invalid="ignore", divide="ignore"):
        delta = tau * e * e / np.maximum(np.abs(m), np.sqrt(tau) * e)
    return hist_check_delta(h_gpu, m_ref, delta, lo, hi, nbins, nan_possible=nanp, window_center=m)


def hist_check_delta(h_gpu, x_ref, delta, lo, hi, nbins, nan_possible=None, window_center=None):
    """Histogram parity with per-event uncertainty windows [x_i − δ_i, x_i + δ_i] (R14, R22).

    Event i is ambiguous if an edge of the axis lies within δ_i of its oracle value (or it
    is flagged in ``nan_possible``). h_s = oracle histogram of the non-ambiguous events.
    Require h_gpu ≥ h_s bin-wise, Σ(h_gpu − h_s) = #ambiguous, and each bin's excess ≤
    #ambiguous events whose window touches it (nan_possible events may also count in the
    overflow bin). ``window_center`` replaces x_ref as the window centre where given."""
    h_gpu = np.asarray(h_gpu, np.int64)
    x0 = np.asarray(x_ref, np.float64)
    x = x0 if window_center is None else np.asarray(window_center, np.float64)
    delta = np.asarray(delta, np.float64)
    n = x.size
    nanp = np.zeros(n, bool) if nan_possible is None else np.asarray(nan_possible, bool)
    w = (hi - lo) / nbins
    fin = np.isfinite(x)
    with np.errstate(invalid="ignore"):
        k = np.clip(np.round((x - lo) / w), 0, nbins)
        nearest_edge = lo + k * w
        amb = fin & (np.abs(x - nearest_edge) <= delta + 1e-12 * np.abs(x)) & (x > lo - delta - w) & (x < hi + delta + w)
    amb |= nanp
    b_ref = find_bin_np(x0, lo, hi, nbins)
    h_s = np.bincount(b_ref[~amb], minlength=nbins + 2).astype(np.int64)
    fails = []
    if (h_gpu < h_s).any():
        bad = np.nonzero(h_gpu < h_s)[0][:10]
        fails.append(f"bins below the unambiguous oracle count: {bad.tolist()}")
    excess = h_gpu - h_s
    if excess.sum() != amb.sum():
        fails.append(f"total excess {excess.sum()} != #ambiguous {amb.sum()}")
    allowed = np.zeros(nbins + 2, np.int64)
    for i in np.nonzero(amb)[0]:
        if np.isfinite(x[i]) and np.isfinite(delta[i]):
            b0 = find_bin_np(x[i] - delta[i], lo, hi, nbins)
            b1 = find_bin_np(x[i] + delta[i], lo, hi, nbins)
            allowed[int(b0):int(b1) + 1] += 1
        elif np.isfinite(x[i]):  # unbounded window: anywhere
            allowed += 1
        if nanp[i] or not np.isfinite(x[i]):
            allowed[nbins + 1] += 1
    if (excess > allowed).any():
        bad = np.nonzero(excess > allowed)[0][:10]
        fails.append(f"bins exceed their ambiguous allowance: {bad.tolist()}")
    return fails, int(amb.sum())
