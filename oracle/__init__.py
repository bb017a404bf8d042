"""CPU oracle of the GenVectorX hot path (arXiv 2312.02756) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package. The product path
(``paper_2312_02756_b200``) never imports it and shares no code with it.

The arithmetic lives in plain C (``gvx_oracle.c`` / ``gvx_oracle_body.inc``),
compiled by gcc ``-O2 -ffp-contract=off`` against glibc libm into
``liboracle.so``; this module only marshals numpy arrays through ctypes.
Each function cites the PAPER.md / SPEC.md passage its C body follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_SOURCES = ["gvx_oracle.c", "gvx_oracle_body.inc", "gvx_oracle.h"]

PTETAPHIM = 0
PXPYPZE = 1
PXPYPZM = 2
PTETAPHIE = 3
_COORDS = {"ptetaphim": PTETAPHIM, "pxpypze": PXPYPZE, "pxpypzm": PXPYPZM, "ptetaphie": PTETAPHIE}


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, no FMA contraction)."""
    src_mtime = max(os.path.getmtime(os.path.join(_HERE, s)) for s in _SOURCES)
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= src_mtime:
        return _LIB_PATH
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared",
           "-Wall", "-Wextra", "-o", _LIB_PATH + ".tmp", os.path.join(_HERE, "gvx_oracle.c"), "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        for sfx, T in (("f32", ctypes.c_float), ("f64", ctypes.c_double)):
            getattr(lib, f"gvx_ref_invariant_mass_{sfx}").argtypes = [ctypes.c_int, ctypes.c_int, P, P, I64, P, P]
            getattr(lib, f"gvx_ref_boost_{sfx}").argtypes = [P, P, I64, P, P]
            f = getattr(lib, f"gvx_ref_boost_uniform_{sfx}")
            f.argtypes = [P, T, T, T, I64, P]
            f.restype = ctypes.c_int
            f = getattr(lib, f"gvx_ref_lorentz_transform_{sfx}")
            f.argtypes = [P, P, I64, P]
            f.restype = ctypes.c_int
            getattr(lib, f"gvx_ref_cm_mass_{sfx}").argtypes = [ctypes.c_int, ctypes.c_int, P, P, I64, P, P, P]
            getattr(lib, f"gvx_ref_mass_histogram_{sfx}").argtypes = [
                ctypes.c_int, ctypes.c_int, P, P, I64, ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                ctypes.c_int, P, P]
            getattr(lib, f"gvx_ref_cm_costheta_{sfx}").argtypes = [
                ctypes.c_int, ctypes.c_int, P, P, I64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, P,
                ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, P, P]
            f = getattr(lib, f"gvx_ref_dimuon_histogram_{sfx}")
            f.argtypes = [P, P, P, I64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, P]
            f.restype = I64
        lib.gvx_ref_find_bin.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int32]
        lib.gvx_ref_find_bin.restype = ctypes.c_int32
        _lib = lib
    return _lib


def _sfx(dtype) -> str:
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise TypeError(f"oracle supports float32/float64, got {dtype}")


def _vecs(a, ncomp: int, dtype=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=dtype)
    if a.ndim == 1 and a.size == ncomp:
        a = a.reshape(1, ncomp)
    if a.ndim != 2 or a.shape[1] != ncomp:
        raise ValueError(f"expected an [N, {ncomp}] array, got shape {a.shape}")
    return a


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _c2(coords: str, coords2):
    """(coords of v1, coords of v2): the pair functions take each operand's coordinate system
    ("two particles expressed in any 4-dimensional coordinate system")."""
    return _COORDS[coords], _COORDS[coords2 if coords2 is not None else coords]


def invariant_mass(v1, v2, coords: str = "ptetaphim", coords2=None):
    """InvariantMasses, PAPER.md:141-151 (Fig. 1): ``m[i] = (v1[i] + v2[i]).mass()``.

    ``v1`` is in ``coords``, ``v2`` in ``coords2`` (default: the same system).
    Returns ``(M, E_lab)``, both of v1's dtype; ``E_lab = E1 + E2`` is the
    tolerance scale (reading R5).
    """
    v1 = _vecs(v1, 4)
    v2 = _vecs(v2, 4, v1.dtype)
    if v1.shape != v2.shape:
        raise ValueError(f"length mismatch: {v1.shape[0]} vs {v2.shape[0]}")
    n = v1.shape[0]
    m = np.empty(n, v1.dtype)
    e = np.empty(n, v1.dtype)
    getattr(_load(), f"gvx_ref_invariant_mass_{_sfx(v1.dtype)}")(
        *_c2(coords, coords2), _ptr(v1), _ptr(v2), n, _ptr(m), _ptr(e))
    return m, e


def boost(v, beta):
    """Per-event Lorentz boost, PAPER.md:136 / SPEC.md:188-200.

    ``v`` is [N, 4] PxPyPzE, ``beta`` [N, 3]. Returns ``(out, S)`` with
    ``S = γ(E + |β||p|)`` the tolerance scale (reading R5); |β| ≥ 1 → NaN×4.
    """
    v = _vecs(v, 4)
    beta = _vecs(beta, 3, v.dtype)
    if v.shape[0] != beta.shape[0]:
        raise ValueError(f"length mismatch: {v.shape[0]} vs {beta.shape[0]}")
    n = v.shape[0]
    out = np.empty_like(v)
    s = np.empty(n, v.dtype)
    getattr(_load(), f"gvx_ref_boost_{_sfx(v.dtype)}")(_ptr(v), _ptr(beta), n, _ptr(out), _ptr(s))
    return out, s


class DomainError(ValueError):
    pass


def boost_uniform(v, bx, by, bz):
    """The paper's single-matrix ApplyBoost; |β| ≥ 1 raises DomainError
    (SPEC.md:191)."""
    v = _vecs(v, 4)
    n = v.shape[0]
    out = np.empty_like(v)
    rc = getattr(_load(), f"gvx_ref_boost_uniform_{_sfx(v.dtype)}")(_ptr(v), bx, by, bz, n, _ptr(out))
    if rc != 0:
        raise DomainError(f"|beta|^2 = {bx*bx + by*by + bz*bz} >= 1")
    return out


def lorentz_transform(v, L):
    """General 4x4 Lorentz transformation ("orthosymplectic matrix"): out = L·v.
    ``L`` 4x4 (row-major, double); raises DomainError unless L^T g L = g (to 1e-9)."""
    v = _vecs(v, 4)
    Lm = np.ascontiguousarray(L, np.float64).reshape(4, 4)
    out = np.empty_like(v)
    rc = getattr(_load(), f"gvx_ref_lorentz_transform_{_sfx(v.dtype)}")(_ptr(Lm), _ptr(v), v.shape[0], _ptr(out))
    if rc != 0:
        raise DomainError("L is not a Lorentz transformation (L^T g L != g)")
    return out


def cm_mass(v1, v2, coords: str = "ptetaphim", want_boosted: bool = False, coords2=None):
    """Boost each pair to its CM frame (β = −P/E), then the signed mass (reading R11).

    Returns ``(M_cm, E_lab[, boosted])``; boosted is [N, 8] (vector 1, vector 2).
    """
    v1 = _vecs(v1, 4)
    v2 = _vecs(v2, 4, v1.dtype)
    if v1.shape != v2.shape:
        raise ValueError(f"length mismatch: {v1.shape[0]} vs {v2.shape[0]}")
    n = v1.shape[0]
    m = np.empty(n, v1.dtype)
    e = np.empty(n, v1.dtype)
    bo = np.empty((n, 8), v1.dtype) if want_boosted else None
    getattr(_load(), f"gvx_ref_cm_mass_{_sfx(v1.dtype)}")(
        *_c2(coords, coords2), _ptr(v1), _ptr(v2), n, _ptr(m), _ptr(e), _ptr(bo))
    return (m, e, bo) if want_boosted else (m, e)


def mass_histogram(v1, v2, lo: float, hi: float, nbins: int, cm: bool = False,
                   coords: str = "ptetaphim", bins=None, coords2=None):
    """Fused mass histogram (north_star; reading R12). Returns ``(bins uint64[nbins+2], M)``.

    ``bins`` accumulates if given (the caller's zeroed array)."""
    v1 = _vecs(v1, 4)
    v2 = _vecs(v2, 4, v1.dtype)
    if v1.shape != v2.shape:
        raise ValueError(f"length mismatch: {v1.shape[0]} vs {v2.shape[0]}")
    n = v1.shape[0]
    if bins is None:
        bins = np.zeros(nbins + 2, np.uint64)
    assert bins.dtype == np.uint64 and bins.shape == (nbins + 2,) and bins.flags.c_contiguous
    m = np.empty(n, v1.dtype)
    getattr(_load(), f"gvx_ref_mass_histogram_{_sfx(v1.dtype)}")(
        *_c2(coords, coords2), _ptr(v1), _ptr(v2), n, lo, hi, nbins, int(bool(cm)), _ptr(bins), _ptr(m))
    return bins, m


def cm_costheta(v1, v2, m_axis=(0.25, 300.0, 1000), c_axis=(-1.0, 1.0, 100),
                coords: str = "ptetaphim", m_bins=None, c_bins=None, coords2=None):
    """CM decay angle (reading R22): cos θ* = p'1z/|p'1| of vector 1 after
    the CM boost of reading R11, with the CM mass and cos θ* histograms (reading R12).
    Returns ``(m_bins, c_bins, M_cm, cos_theta)``; bins accumulate if given."""
    v1 = _vecs(v1, 4)
    v2 = _vecs(v2, 4, v1.dtype)
    if v1.shape != v2.shape:
        raise ValueError(f"length mismatch: {v1.shape[0]} vs {v2.shape[0]}")
    n = v1.shape[0]
    if m_bins is None:
        m_bins = np.zeros(m_axis[2] + 2, np.uint64)
    if c_bins is None:
        c_bins = np.zeros(c_axis[2] + 2, np.uint64)
    m = np.empty(n, v1.dtype)
    c = np.empty(n, v1.dtype)
    getattr(_load(), f"gvx_ref_cm_costheta_{_sfx(v1.dtype)}")(
        *_c2(coords, coords2), _ptr(v1), _ptr(v2), n, float(m_axis[0]), float(m_axis[1]), int(m_axis[2]),
        _ptr(m_bins), float(c_axis[0]), float(c_axis[1]), int(c_axis[2]), _ptr(c_bins), _ptr(m), _ptr(c))
    return m_bins, c_bins, m, c


def dimuon_histogram(muons, charge, offsets, lo: float, hi: float, nbins: int, bins=None):
    """Jagged dimuon selection + histogram (reading R21): events with exactly two muons of
    opposite charge. ``muons`` [M, 4] PtEtaPhiM, ``charge`` int32 [M], ``offsets`` int64
    [n_events + 1]. Returns ``(bins uint64[nbins+2], M_per_event (NaN if not selected), n_selected)``."""
    muons = _vecs(muons, 4)
    charge = np.ascontiguousarray(charge, np.int32)
    offsets = np.ascontiguousarray(offsets, np.int64)
    if charge.shape != (muons.shape[0],):
        raise ValueError("charge must have one entry per muon")
    n_events = offsets.shape[0] - 1
    if n_events < 0 or (n_events > 0 and (offsets[0] < 0 or offsets[-1] > muons.shape[0] or
                                          np.any(np.diff(offsets) < 0))):
        raise ValueError("offsets must be non-decreasing within [0, n_muons]")
    if bins is None:
        bins = np.zeros(nbins + 2, np.uint64)
    m = np.empty(max(n_events, 0), muons.dtype)
    sel = getattr(_load(), f"gvx_ref_dimuon_histogram_{_sfx(muons.dtype)}")(
        _ptr(muons), _ptr(charge), _ptr(offsets), max(n_events, 0), lo, hi, nbins, _ptr(bins), _ptr(m))
    return bins, m, int(sel)


def find_bin(x: float, lo: float, hi: float, nbins: int) -> int:
    """ROOT FindFixBin in double (reading R12)."""
    return int(_load().gvx_ref_find_bin(float(x), float(lo), float(hi), int(nbins)))
