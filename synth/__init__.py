"""Seeded, counter-based synthetic event generator — shared input source for the
oracle (tests) and the CUDA path (tests, bench).

This module holds NONE of the method's arithmetic (no coordinate conversion,
no 4-vector sum, no mass, no boost, no binning). It only draws events.

Every value is a deterministic function of ``(seed, stream, global event
index)``: Philox4x32-10 (Salmon et al., SC'11) turns the counter into four
32-bit words, and the words are mapped to physics-shaped values with IEEE-754
basic operations only (+, −, ×, ÷, sqrt, floor, ldexp — all exactly rounded),
in a fixed order, with no fused multiply-add. The twin device generator in
``synth/synth_gen.cu`` performs the same operations in the same order with
``__dmul_rn``/``__dadd_rn``/``__dsqrt_rn`` (no contraction), so both sides
produce the same bits for the same event index — a GPU test asserts this.
Any subset of events (e.g. a sample of a 1e9-event device batch) can thus be
regenerated on the host for the oracle without reading device memory back.

Distributions ("input recipe"; shaped after the paper's
dimuon-style workloads — PAPER.md:263 "invariant masses from two arrays of
particles and the boosting of one array", BASELINE.json north_star "pt
exponential/log-normal around tens of GeV, |eta| < 2.5, uniform phi, m near
the muon mass"):

* muon (PtEtaPhiM): pt = exp(ln 30 + 0.5·z) GeV (log-normal around 30 GeV),
  z = (u0+u1+u2+u3 − 2)·√3 (Irwin–Hall(4), zero mean, unit variance);
  eta = −2.5 + 5·u; phi = −π + 2π·u; m = 0.1056583755 GeV.
* boost input (PxPyPzE): p_i = 30·z_i GeV for i = x, y, z; E = sqrt(|p|² + m_μ²).
* per-event beta: isotropic direction g/|g| (g_i Irwin–Hall normals) times
  |β| = 0.99·max(u_a, u_b, u_c) — the max of three uniforms has density
  3r², i.e. β uniform in the ball of radius 0.99.
* optional resonance admixture (``muon_pairs(..., f_res)``): a
  fraction f_res of the pairs peaks at the Z mass (see muon_pairs).
"""
from __future__ import annotations

import numpy as np

# Philox4x32 constants (Random123).
_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)

# Stream ids (counter word 3).
STREAM_V1 = 1
STREAM_V2 = 2
STREAM_BOOST_P = 3
STREAM_BOOST_BETA = 4
STREAM_JAGGED_N = 5     # per-event muon multiplicity
STREAM_JAGGED_MU = 6    # muon j of event e: counter e * 8 + j (j < 8)
STREAM_RES = 7          # resonance admixture: selector, then two normals
Z_MASS = 91.1876
Z_HALF_WIDTH = 1.2476   # Gamma_Z / 2
JAGGED_SLOTS = 8
# multiplicity k = 0..4 with P = 0.25, 0.30, 0.30, 0.10, 0.05 (cumulative thresholds)
JAGGED_CDF = (0.25, 0.55, 0.85, 0.95)

DEFAULT_SEED = 12345

# Constants, written as decimal literals that numpy and nvcc both round
# correctly to the same doubles.
MUON_MASS = 0.1056583755
MUON_MASS2 = 0.011163692328303140  # any fixed double; only used as "m²" input term
LN30 = 3.4011973816621555
SQRT3 = 1.7320508075688772
PI = 3.141592653589793
TWO_PI = 6.283185307179586
INV_LN2 = 1.4426950408889634
LN2_HI = 0.693145751953125          # 0x3FE62E4000000000: 21 significant bits
LN2_LO = 1.4286068203094173e-06     # ln 2 − LN2_HI rounded to double
TWO_M32 = 2.3283064365386963e-10    # 2^-32 exactly
# Taylor coefficients 1/k!, k = 0..13 (Horner, highest first).
EXP_COEF = (
    1.6059043836821613e-10, 2.08767569878681e-09, 2.505210838544172e-08,
    2.755731922398589e-07, 2.7557319223985893e-06, 2.48015873015873e-05,
    0.0001984126984126984, 0.001388888888888889, 0.008333333333333333,
    0.041666666666666664, 0.16666666666666666, 0.5, 1.0, 1.0,
)


def philox4x32(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 on uint64 arrays holding 32-bit words; returns 4 word arrays."""
    c0 = np.asarray(c0, np.uint64)
    c1 = np.asarray(c1, np.uint64)
    c2 = np.asarray(c2, np.uint64)
    c3 = np.asarray(c3, np.uint64)
    k0 = np.uint64(k0) & _MASK
    k1 = np.uint64(k1) & _MASK
    for r in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK
        hi1, lo1 = p1 >> _S32, p1 & _MASK
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
        if r < 9:
            k0 = (k0 + _W0) & _MASK
            k1 = (k1 + _W1) & _MASK
    return c0, c1, c2, c3


def _draw(idx, call, stream, seed):
    idx = np.asarray(idx, np.uint64)
    seed = np.uint64(seed)
    return philox4x32(idx & _MASK, idx >> _S32, np.full_like(idx, call), np.full_like(idx, stream),
                      seed & _MASK, seed >> _S32)


def _u(word):
    """uint32 word -> uniform double in (0, 1): (w + 0.5)·2^-32 (exact)."""
    return (word.astype(np.float64) + 0.5) * TWO_M32


def _normal(w):
    """Irwin–Hall(4) standard normal from four words: (u0+u1+u2+u3 − 2)·√3."""
    s = ((_u(w[0]) + _u(w[1])) + _u(w[2])) + _u(w[3])
    return (s - 2.0) * SQRT3


def _exp_det(x):
    """exp(x) for |x| < 700 from basic operations only (deterministic across CPU/GPU)."""
    k = np.floor(x * INV_LN2 + 0.5)
    r = (x - k * LN2_HI) - k * LN2_LO
    p = np.full_like(r, EXP_COEF[0])
    for c in EXP_COEF[1:]:
        p = p * r + c
    return np.ldexp(p, k.astype(np.int64))


def muons(idx, stream, seed=DEFAULT_SEED, dtype=np.float64):
    """PtEtaPhiM muons for the given global event indices -> [len(idx), 4] of dtype."""
    return _muons64(idx, stream, seed).astype(dtype)


def _muons64(idx, stream, seed=DEFAULT_SEED):
    idx = np.asarray(idx, np.uint64).reshape(-1)
    w0 = _draw(idx, 0, stream, seed)
    w1 = _draw(idx, 1, stream, seed)
    pt = _exp_det(LN30 + 0.5 * _normal(w0))
    eta = -2.5 + 5.0 * _u(w1[0])
    phi = -PI + TWO_PI * _u(w1[1])
    out = np.empty((idx.size, 4), np.float64)
    out[:, 0] = pt
    out[:, 1] = eta
    out[:, 2] = phi
    out[:, 3] = MUON_MASS
    return out


def muon_pairs(idx, seed=DEFAULT_SEED, dtype=np.float64, f_res=0.0):
    """(v1, v2): two independent PtEtaPhiM muons per event index; with ``f_res`` > 0 that
    fraction of the events is re-drawn as a resonance pair (SURVEY §8(d) "resonance
    admixture"): a Z-like mass x = 91.1876 + 1.2476·z1/z2 (ratio of normals: a Breit–Wigner
    shape; outside [60, 120] GeV it falls back to 91.1876 + 1.2476·z1), muon 2 put back to back
    in φ with the pt that gives a massless pair this mass, pt2 = x² / (2·pt1·(cosh Δη + 1)).
    Choosing pt2 inverts the massless back-to-back relation; no 4-vector arithmetic of the
    method (conversion, sum, mass, boost) is done here."""
    idx = np.asarray(idx, np.uint64).reshape(-1)
    a = _muons64(idx, STREAM_V1, seed)
    b = _muons64(idx, STREAM_V2, seed)
    if f_res > 0.0:
        sel = _u(_draw(idx, 0, STREAM_RES, seed)[0]) < f_res
        if sel.any():
            ii = idx[sel]
            z1 = _normal(_draw(ii, 1, STREAM_RES, seed))
            z2 = _normal(_draw(ii, 2, STREAM_RES, seed))
            with np.errstate(divide="ignore", invalid="ignore"):
                x = Z_MASS + Z_HALF_WIDTH * (z1 / z2)
            x = np.where((x >= 60.0) & (x <= 120.0), x, Z_MASS + Z_HALF_WIDTH * z1)
            d = a[sel, 1] - b[sel, 1]
            ch = (_exp_det(d) + _exp_det(-d)) * 0.5
            b[sel, 0] = (x * x) / ((2.0 * a[sel, 0]) * (ch + 1.0))
            phi2 = a[sel, 2] + PI
            b[sel, 2] = np.where(phi2 >= PI, phi2 - TWO_PI, phi2)
    return a.astype(dtype), b.astype(dtype)


def boost_inputs(idx, seed=DEFAULT_SEED, dtype=np.float64):
    """(v [N,4] PxPyPzE on the muon mass shell, beta [N,3] uniform in |β| ≤ 0.99)."""
    idx = np.asarray(idx, np.uint64).reshape(-1)
    px = 30.0 * _normal(_draw(idx, 0, STREAM_BOOST_P, seed))
    py = 30.0 * _normal(_draw(idx, 1, STREAM_BOOST_P, seed))
    pz = 30.0 * _normal(_draw(idx, 2, STREAM_BOOST_P, seed))
    e = np.sqrt(((px * px + py * py) + pz * pz) + MUON_MASS2)
    gx = _normal(_draw(idx, 0, STREAM_BOOST_BETA, seed))
    gy = _normal(_draw(idx, 1, STREAM_BOOST_BETA, seed))
    gz = _normal(_draw(idx, 2, STREAM_BOOST_BETA, seed))
    wm = _draw(idx, 3, STREAM_BOOST_BETA, seed)
    mag = 0.99 * np.maximum(np.maximum(_u(wm[0]), _u(wm[1])), _u(wm[2]))
    scale = mag / np.sqrt((gx * gx + gy * gy) + gz * gz)
    v = np.stack([px, py, pz, e], axis=1).astype(dtype)
    beta = np.stack([gx * scale, gy * scale, gz * scale], axis=1).astype(dtype)
    return v, beta


def jagged_counts(event_idx, seed=DEFAULT_SEED):
    """Muon multiplicity of each event (0..4), from one uniform per event."""
    idx = np.asarray(event_idx, np.uint64).reshape(-1)
    u = _u(_draw(idx, 0, STREAM_JAGGED_N, seed)[0])
    k = np.zeros(idx.size, np.int64)
    for t in JAGGED_CDF:
        k += (u >= t)
    return k


def jagged_events(first_event: int, n_events: int, seed=DEFAULT_SEED, dtype=np.float64):
    """A flat, RDataFrame-style muon collection for events first_event .. first_event+n_events-1:
    ``(muons [M, 4] PtEtaPhiM, charge int32 [M], offsets int64 [n_events + 1])``. Muon j of
    event e is drawn from counter e * 8 + j, charge = +1 / -1 with probability 1/2, so any
    shard of events regenerates identically."""
    ev = np.arange(first_event, first_event + n_events, dtype=np.uint64)
    k = jagged_counts(ev, seed)
    offsets = np.zeros(n_events + 1, np.int64)
    np.cumsum(k, out=offsets[1:])
    ev_of = np.repeat(ev, k)
    j = np.arange(offsets[-1], dtype=np.int64) - np.repeat(offsets[:-1], k)
    midx = ev_of * np.uint64(JAGGED_SLOTS) + j.astype(np.uint64)
    mu = muons(midx, STREAM_JAGGED_MU, seed, dtype)
    q = np.where(_u(_draw(midx, 2, STREAM_JAGGED_MU, seed)[0]) < 0.5, 1, -1).astype(np.int32)
    return mu, q, offsets


def shard_range(n_total: int, rank: int, world: int):
    """Contiguous index shard of rank r: [floor(r·N/G), floor((r+1)·N/G))."""
    return (n_total * rank) // world, (n_total * (rank + 1)) // world
