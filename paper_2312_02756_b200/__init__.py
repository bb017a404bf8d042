"""B200-native GenVectorX hot path (arXiv 2312.02756): Python binding.

Thin marshalling over the C ABI of ``include/gvx.h`` (``libgvx.so``, hand-
written sm_100a CUDA). Torch supplies device memory and the current stream
only; every step of the path runs in the library's kernels. There is no CPU
fallback: importing this package on a machine where ``libgvx.so`` is missing
raises, and calling an op with CPU tensors raises.

Names follow the paper ("InvariantMasses", "ApplyBoost"):

* :func:`invariant_mass` — ``m[i] = (v1[i] + v2[i]).mass()`` (Fig. 1)
* :func:`boost` / :func:`boost_uniform` — Lorentz boost by per-event / one β
* :func:`mass_histogram` — fused mass (+ optional CM boost) histogram
* :func:`sharded_mass_histogram` — per-rank histogram + NCCL bin all-reduce

Pair calls take ``coords2`` for mixed pairs (v2 in another system than v1; ABI v7).

Vector arguments are CUDA tensors ``[N, 4]`` (AoS, any row stride — e.g. the
``[:, 0, :]`` view of interleaved ``[N, 2, 4]`` pairs) or a 4-sequence of
``[N]`` tensors sharing one stride (SoA). Components are (pt, eta, phi, m)
for ``coords="ptetaphim"``, (px, py, pz, E) for ``"pxpypze"``, (px, py, pz, m)
for ``"pxpypzm"`` and (pt, eta, phi, E) for ``"ptetaphie"``.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Union

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# GVX_LIB may point at the tuning build (tools/libgvx_tune.so) for A/B runs.
LIB_PATH = os.environ.get("GVX_LIB") or os.path.join(_PKG, "libgvx.so")

GVX_OK = 0
GVX_ERR_INVALID_ARGUMENT = 1
GVX_ERR_DOMAIN = 2
GVX_ERR_UNSUPPORTED = 3
GVX_ERR_CUDA = 4
GVX_F32 = 0
GVX_F64 = 1
GVX_PTETAPHIM = 0
GVX_PXPYPZE = 1
GVX_PXPYPZM = 2
GVX_PTETAPHIE = 3
GVX_HIST_BOOST_TO_CM = 0x1
ABI_VERSION = 8

# The default histogram of the north star: 1000 bins over the dimuon range
# (reading R13).
DEFAULT_LO = 0.25
DEFAULT_HI = 300.0
DEFAULT_NBINS = 1000


class Vec4CView(ctypes.Structure):
    _fields_ = [("c", ctypes.c_void_p * 4), ("stride", ctypes.c_int64)]


class Vec4View(ctypes.Structure):
    _fields_ = [("c", ctypes.c_void_p * 4), ("stride", ctypes.c_int64)]


class Vec3CView(ctypes.Structure):
    _fields_ = [("c", ctypes.c_void_p * 3), ("stride", ctypes.c_int64)]


class GvxError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class DomainError(GvxError, ValueError):
    pass


def _load_lib():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    I64 = ctypes.c_int64
    st = ctypes.c_int
    lib.gvx_invariant_mass.argtypes = [st, st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec4CView), P, I64, P]
    lib.gvx_invariant_mass.restype = st
    lib.gvx_boost.argtypes = [st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec3CView), ctypes.POINTER(Vec4View),
                              I64, P]
    lib.gvx_boost.restype = st
    lib.gvx_boost_uniform.argtypes = [st, ctypes.POINTER(Vec4CView), ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, ctypes.POINTER(Vec4View), I64, P]
    lib.gvx_boost_uniform.restype = st
    lib.gvx_mass_histogram.argtypes = [st, st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec4CView), I64,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, ctypes.c_uint32, P,
                                       ctypes.POINTER(Vec4View), P]
    lib.gvx_mass_histogram.restype = st
    lib.gvx_lorentz_transform.argtypes = [st, ctypes.POINTER(Vec4CView), P, ctypes.POINTER(Vec4View), I64, P]
    lib.gvx_lorentz_transform.restype = st
    lib.gvx_dimuon_histogram.argtypes = [st, ctypes.POINTER(Vec4CView), P, P, I64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_int32, P, P, P]
    lib.gvx_dimuon_histogram.restype = st
    lib.gvx_pair_histograms.argtypes = [st, st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec4CView), I64,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, P, P, P, P]
    lib.gvx_pair_histograms.restype = st
    lib.gvx_pair_histograms_boost.argtypes = [st, st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec4CView), I64,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, P, P, P,
                                              ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec3CView),
                                              ctypes.POINTER(Vec4View), I64, P]
    lib.gvx_pair_histograms_boost.restype = st
    lib.gvx_mass_histogram_peers.argtypes = [st, st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec4CView), I64,
                                             ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, ctypes.c_int32,
                                             P, P, ctypes.c_uint32, P, P]
    lib.gvx_mass_histogram_peers.restype = st
    lib.gvx_cm_costheta_histogram.argtypes = [st, st, ctypes.POINTER(Vec4CView), ctypes.POINTER(Vec4CView), I64,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_int32, P,
                                              ctypes.c_double, ctypes.c_double, ctypes.c_int32, P, P, P, P]
    lib.gvx_cm_costheta_histogram.restype = st
    # mixed-coordinate pairs (ABI v7): the calls above with (coords1, coords2)
    lib.gvx_invariant_mass_mixed.argtypes = [st, st] + lib.gvx_invariant_mass.argtypes[1:]
    lib.gvx_invariant_mass_mixed.restype = st
    lib.gvx_mass_histogram_mixed.argtypes = [st, st] + lib.gvx_mass_histogram.argtypes[1:]
    lib.gvx_mass_histogram_mixed.restype = st
    lib.gvx_pair_histograms_mixed.argtypes = [st, st] + lib.gvx_pair_histograms.argtypes[1:]
    lib.gvx_pair_histograms_mixed.restype = st
    lib.gvx_pair_histograms_boost_mixed.argtypes = [st, st] + lib.gvx_pair_histograms_boost.argtypes[1:]
    lib.gvx_pair_histograms_boost_mixed.restype = st
    lib.gvx_status_string.argtypes = [st]
    lib.gvx_status_string.restype = ctypes.c_char_p
    lib.gvx_last_cuda_error_string.argtypes = []
    lib.gvx_last_cuda_error_string.restype = ctypes.c_char_p
    lib.gvx_abi_version.restype = ctypes.c_int
    if lib.gvx_abi_version() != ABI_VERSION:
        raise ImportError(f"libgvx ABI {lib.gvx_abi_version()} != binding ABI {ABI_VERSION}")
    return lib


lib = _load_lib()

VecArg = Union[torch.Tensor, Sequence[torch.Tensor]]


def _check(status: int, what: str) -> None:
    if status == GVX_OK:
        return
    name = lib.gvx_status_string(status).decode()
    if status == GVX_ERR_CUDA:
        raise GvxError(status, f"{what}: {name}: {lib.gvx_last_cuda_error_string().decode()}")
    if status == GVX_ERR_DOMAIN:
        raise DomainError(status, f"{what}: {name}")
    raise GvxError(status, f"{what}: {name}")


def _dtype_code(dt: torch.dtype) -> int:
    if dt == torch.float64:
        return GVX_F64
    if dt == torch.float32:
        return GVX_F32
    raise TypeError(f"gvx supports float32 and float64, got {dt}")


def _coords_code(coords: str) -> int:
    try:
        return {"ptetaphim": GVX_PTETAPHIM, "pxpypze": GVX_PXPYPZE, "pxpypzm": GVX_PXPYPZM,
                "ptetaphie": GVX_PTETAPHIE}[coords]
    except KeyError:
        raise ValueError(f"coords must be one of ptetaphim, pxpypze, pxpypzm, ptetaphie; got {coords!r}") from None


def _coords_args(coords: str, coords2: Optional[str]):
    """-> (mixed, codes): the single-system call's (coords,) or the mixed call's (coords1, coords2)."""
    if coords2 is None:
        return False, (_coords_code(coords),)
    return True, (_coords_code(coords), _coords_code(coords2))


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (gvx has no CPU fallback)")


def _view(x: VecArg, ncomp: int, name: str, writable: bool = False):
    """-> (ctypes view struct, n, dtype, device, keepalive)."""
    if isinstance(x, torch.Tensor):
        _require_cuda(x, name)
        if x.dim() != 2 or x.shape[1] != ncomp:
            raise ValueError(f"{name} must be [N, {ncomp}] or a {ncomp}-sequence of [N] tensors, got {tuple(x.shape)}")
        es = x.element_size()
        base = x.data_ptr()
        s0, s1 = x.stride()
        n = x.shape[0]
        ptrs = [base + k * s1 * es for k in range(ncomp)]
        if n > 1 and s0 < 1:
            raise ValueError(f"{name}: row stride {s0} is not supported (broadcast or flipped views); "
                             "make the tensor contiguous")
        stride = s0 if n > 1 else max(s0, 1)
        dtype, dev = x.dtype, x.device
        keep = (x,)
    else:
        comps = list(x)
        if len(comps) != ncomp:
            raise ValueError(f"{name} must have {ncomp} components, got {len(comps)}")
        for i, c in enumerate(comps):
            _require_cuda(c, f"{name}[{i}]")
            if c.dim() != 1:
                raise ValueError(f"{name}[{i}] must be 1-D")
        n = comps[0].shape[0]
        dtype, dev = comps[0].dtype, comps[0].device
        if any(c.shape[0] != n or c.dtype != dtype or c.device != dev for c in comps):
            raise ValueError(f"{name}: components differ in length, dtype or device")
        strides = {c.stride(0) for c in comps} if n > 1 else {1}
        if len(strides) != 1:
            raise ValueError(f"{name}: components must share one stride")
        stride = strides.pop()
        if stride < 1:
            raise ValueError(f"{name}: stride {stride} is not supported (broadcast or flipped views)")
        ptrs = [c.data_ptr() for c in comps]
        keep = tuple(comps)
    if ncomp == 4:
        v = (Vec4View if writable else Vec4CView)()
    else:
        v = Vec3CView()
    for k in range(ncomp):
        v.c[k] = ptrs[k]
    v.stride = max(int(stride), 1)
    return v, n, dtype, dev, keep


def _stream(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def invariant_mass(v1: VecArg, v2: VecArg, out: Optional[torch.Tensor] = None,
                   coords: str = "ptetaphim", coords2: Optional[str] = None) -> torch.Tensor:
    """InvariantMasses: ``out[i] = (v1[i] + v2[i]).mass()``, signed (ROOT convention).
    ``v1`` is in ``coords``; ``v2`` in ``coords2`` if given (mixed pairs), else in ``coords``."""
    a, n, dt, dev, k1 = _view(v1, 4, "v1")
    b, n2, dt2, dev2, k2 = _view(v2, 4, "v2")
    if n != n2:
        raise ValueError(f"length mismatch: v1 has {n} vectors, v2 has {n2}")
    if dt != dt2 or dev != dev2:
        raise ValueError("v1 and v2 must share dtype and device")
    if out is None:
        out = torch.empty(n, dtype=dt, device=dev)
    else:
        _require_cuda(out, "out")
        if out.shape != (n,) or out.dtype != dt or not out.is_contiguous() or out.device != dev:
            raise ValueError("out must be a contiguous [N] tensor of the inputs' dtype and device")
    with torch.cuda.device(dev):
        mixed, cc = _coords_args(coords, coords2)
        fn = lib.gvx_invariant_mass_mixed if mixed else lib.gvx_invariant_mass
        _check(fn(_dtype_code(dt), *cc, ctypes.byref(a), ctypes.byref(b), out.data_ptr() if n else None, n,
                  _stream(dev)), "gvx_invariant_mass")
    return out


def _boost_out(v_t, n, dt, dev, out):
    if out is None:
        out = torch.empty((n, 4), dtype=dt, device=dev)
    o, no, dto, devo, ko = _view(out, 4, "out", writable=True)
    if no != n or dto != dt or devo != dev:
        raise ValueError("out must match v in length, dtype and device")
    return out, o


def boost(v: VecArg, beta: VecArg, out: Optional[VecArg] = None) -> VecArg:
    """ApplyBoost with per-event β: ``out[i] = Λ(β[i])·v[i]``.

    ``v`` PxPyPzE; ``out`` may be ``v`` itself (in place). |β[i]| ≥ 1 → NaN×4.
    """
    a, n, dt, dev, k1 = _view(v, 4, "v")
    b, nb, dtb, devb, k2 = _view(beta, 3, "beta")
    if nb != n:
        raise ValueError(f"length mismatch: v has {n} vectors, beta has {nb}")
    if dtb != dt or devb != dev:
        raise ValueError("v and beta must share dtype and device")
    out, o = _boost_out(v, n, dt, dev, out)
    with torch.cuda.device(dev):
        _check(lib.gvx_boost(_dtype_code(dt), ctypes.byref(a), ctypes.byref(b), ctypes.byref(o), n, _stream(dev)),
               "gvx_boost")
    return out


def boost_uniform(v: VecArg, beta: Sequence[float], out: Optional[VecArg] = None) -> VecArg:
    """The paper's single-matrix ApplyBoost; |β| ≥ 1 raises :class:`DomainError`."""
    a, n, dt, dev, k1 = _view(v, 4, "v")
    bx, by, bz = (float(x) for x in beta)
    out, o = _boost_out(v, n, dt, dev, out)
    with torch.cuda.device(dev):
        _check(lib.gvx_boost_uniform(_dtype_code(dt), ctypes.byref(a), bx, by, bz, ctypes.byref(o), n,
                                     _stream(dev)), "gvx_boost_uniform")
    return out


def lorentz_transform(v: VecArg, L, out: Optional[VecArg] = None) -> VecArg:
    """ApplyBoost with a general 4x4 Lorentz matrix: ``out[i] = L @ v[i]``.
    ``L`` is any 4x4 array-like (row-major); non-Lorentz L raises :class:`DomainError`."""
    import numpy as _np
    Lm = _np.ascontiguousarray(_np.asarray(L, dtype=_np.float64).reshape(4, 4))
    a, n, dt, dev, k1 = _view(v, 4, "v")
    out, o = _boost_out(v, n, dt, dev, out)
    with torch.cuda.device(dev):
        _check(lib.gvx_lorentz_transform(_dtype_code(dt), ctypes.byref(a), Lm.ctypes.data, ctypes.byref(o), n,
                                         _stream(dev)), "gvx_lorentz_transform")
    return out


def new_bins(nbins: int = DEFAULT_NBINS, device=None) -> torch.Tensor:
    """Zeroed counters: [nbins + 2] int64 (0 = underflow, nbins + 1 = overflow)."""
    return torch.zeros(nbins + 2, dtype=torch.int64, device=device or torch.device("cuda"))


def mass_histogram(v1: VecArg, v2: VecArg, lo: float = DEFAULT_LO, hi: float = DEFAULT_HI,
                   nbins: int = DEFAULT_NBINS, bins: Optional[torch.Tensor] = None, cm: bool = False,
                   m_out: Optional[torch.Tensor] = None, boosted_out: Optional[VecArg] = None,
                   coords: str = "ptetaphim", coords2: Optional[str] = None) -> torch.Tensor:
    """Fused mass histogram (north star). Accumulates into ``bins`` ([nbins+2] int64, zeroed by the caller
    or allocated here) and returns it. ``cm=True`` boosts each pair to its CM frame first.
    ``boosted_out`` ([2N, 4], CM only) receives the boosted pair (vectors 2i, 2i+1)."""
    a, n, dt, dev, k1 = _view(v1, 4, "v1")
    b, n2, dt2, dev2, k2 = _view(v2, 4, "v2")
    if n != n2:
        raise ValueError(f"length mismatch: v1 has {n} vectors, v2 has {n2}")
    if dt != dt2 or dev != dev2:
        raise ValueError("v1 and v2 must share dtype and device")
    if bins is None:
        bins = new_bins(nbins, dev)
    _require_cuda(bins, "bins")
    if bins.shape != (nbins + 2,) or bins.dtype != torch.int64 or not bins.is_contiguous():
        raise ValueError(f"bins must be a contiguous int64 tensor of shape [{nbins + 2}]")
    mptr = None
    if m_out is not None:
        _require_cuda(m_out, "m_out")
        if m_out.shape != (n,) or m_out.dtype != dt or not m_out.is_contiguous():
            raise ValueError("m_out must be a contiguous [N] tensor of the inputs' dtype")
        mptr = m_out.data_ptr()
    bo_ref = None
    if boosted_out is not None:
        if not cm:
            raise ValueError("boosted_out requires cm=True")
        bo, nbo, dtbo, devbo, kbo = _view(boosted_out, 4, "boosted_out", writable=True)
        if nbo != 2 * n or dtbo != dt:
            raise ValueError("boosted_out must hold 2N vectors of the inputs' dtype")
        bo_ref = ctypes.byref(bo)
    flags = GVX_HIST_BOOST_TO_CM if cm else 0
    with torch.cuda.device(dev):
        mixed, cc = _coords_args(coords, coords2)
        fn = lib.gvx_mass_histogram_mixed if mixed else lib.gvx_mass_histogram
        _check(fn(_dtype_code(dt), *cc, ctypes.byref(a), ctypes.byref(b), n, float(lo), float(hi), int(nbins),
                  bins.data_ptr(), flags, mptr, bo_ref, _stream(dev)), "gvx_mass_histogram")
    return bins


def _out_1d(t: Optional[torch.Tensor], n: int, dt, name: str):
    if t is None:
        return None
    _require_cuda(t, name)
    if t.shape != (n,) or t.dtype != dt or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous [N] tensor of the inputs' dtype")
    return t.data_ptr()


def _bins_arg(bins: Optional[torch.Tensor], nbins: int, dev, name: str) -> torch.Tensor:
    if bins is None:
        bins = new_bins(nbins, dev)
    _require_cuda(bins, name)
    if bins.shape != (nbins + 2,) or bins.dtype != torch.int64 or not bins.is_contiguous():
        raise ValueError(f"{name} must be a contiguous int64 tensor of shape [{nbins + 2}]")
    return bins


def cm_costheta_histogram(v1: VecArg, v2: VecArg, m_axis=(DEFAULT_LO, DEFAULT_HI, DEFAULT_NBINS),
                          c_axis=(-1.0, 1.0, 100), m_bins: Optional[torch.Tensor] = None,
                          c_bins: Optional[torch.Tensor] = None, m_out: Optional[torch.Tensor] = None,
                          cos_out: Optional[torch.Tensor] = None, coords: str = "ptetaphim"):
    """CM decay angle (DESIGN R22): boost each pair to its CM frame, then bin the CM mass on
    ``m_axis`` and cos θ* = p'1z/|p'1| on ``c_axis`` (each ``(lo, hi, nbins)``) in one pass.
    Returns ``(m_bins, c_bins)`` ([nbins+2] int64 each, accumulated)."""
    a, n, dt, dev, _ = _view(v1, 4, "v1")
    b, n2, dt2, dev2, _ = _view(v2, 4, "v2")
    if n != n2:
        raise ValueError(f"length mismatch: v1 has {n} vectors, v2 has {n2}")
    if dt != dt2 or dev != dev2:
        raise ValueError("v1 and v2 must share dtype and device")
    m_lo, m_hi, m_nb = float(m_axis[0]), float(m_axis[1]), int(m_axis[2])
    c_lo, c_hi, c_nb = float(c_axis[0]), float(c_axis[1]), int(c_axis[2])
    m_bins = _bins_arg(m_bins, m_nb, dev, "m_bins")
    c_bins = _bins_arg(c_bins, c_nb, dev, "c_bins")
    mptr = _out_1d(m_out, n, dt, "m_out")
    cptr = _out_1d(cos_out, n, dt, "cos_out")
    with torch.cuda.device(dev):
        _check(lib.gvx_cm_costheta_histogram(_dtype_code(dt), _coords_code(coords), ctypes.byref(a), ctypes.byref(b),
                                             n, m_lo, m_hi, m_nb, m_bins.data_ptr(), c_lo, c_hi, c_nb,
                                             c_bins.data_ptr(), mptr, cptr, _stream(dev)),
               "gvx_cm_costheta_histogram")
    return m_bins, c_bins


def dimuon_histogram(muons: VecArg, charge: torch.Tensor, offsets: torch.Tensor, lo: float = DEFAULT_LO,
                     hi: float = DEFAULT_HI, nbins: int = DEFAULT_NBINS, bins: Optional[torch.Tensor] = None,
                     m_out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Jagged events (RDataFrame-style, DESIGN R21): events with exactly two opposite-charge
    muons; their pair masses are binned into ``bins`` ([nbins+2] int64, accumulated).
    ``muons`` [M, 4] PtEtaPhiM (or SoA), ``charge`` int32 [M], ``offsets`` int64 [n_events + 1]."""
    a, m, dt, dev, k1 = _view(muons, 4, "muons")
    _require_cuda(charge, "charge")
    _require_cuda(offsets, "offsets")
    if charge.dtype != torch.int32 or charge.shape != (m,) or not charge.is_contiguous():
        raise ValueError("charge must be a contiguous int32 tensor with one entry per muon")
    if offsets.dtype != torch.int64 or offsets.dim() != 1 or not offsets.is_contiguous() or offsets.shape[0] < 1:
        raise ValueError("offsets must be a contiguous int64 tensor of n_events + 1 entries")
    n_events = offsets.shape[0] - 1
    if bins is None:
        bins = new_bins(nbins, dev)
    if bins.shape != (nbins + 2,) or bins.dtype != torch.int64 or not bins.is_contiguous():
        raise ValueError(f"bins must be a contiguous int64 tensor of shape [{nbins + 2}]")
    mptr = None
    if m_out is not None:
        if m_out.shape != (n_events,) or m_out.dtype != dt or not m_out.is_contiguous():
            raise ValueError("m_out must be a contiguous [n_events] tensor of the muons' dtype")
        mptr = m_out.data_ptr()
    with torch.cuda.device(dev):
        _check(lib.gvx_dimuon_histogram(_dtype_code(dt), ctypes.byref(a), charge.data_ptr(), offsets.data_ptr(),
                                        n_events, float(lo), float(hi), int(nbins), bins.data_ptr(), mptr,
                                        _stream(dev)), "gvx_dimuon_histogram")
    return bins


def sharded_mass_histogram(v1: VecArg, v2: VecArg, lo: float = DEFAULT_LO, hi: float = DEFAULT_HI,
                           nbins: int = DEFAULT_NBINS, cm: bool = False, group=None,
                           coords: str = "ptetaphim", bins: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Per-rank fused histogram of this rank's event shard, then ONE all-reduce(SUM) of the
    nbins+2 counters over the process group (NCCL over NVLink on B200s; gloo on CPU tests).
    Returns the global histogram on every rank."""
    bins = mass_histogram(v1, v2, lo, hi, nbins, bins=bins, cm=cm, coords=coords)
    return allreduce_bins(bins, group)


def pair_histograms(v1: VecArg, v2: VecArg, lo: float = DEFAULT_LO, hi: float = DEFAULT_HI,
                    nbins: int = DEFAULT_NBINS, lab_bins: Optional[torch.Tensor] = None,
                    cm_bins: Optional[torch.Tensor] = None, m_out: Optional[torch.Tensor] = None,
                    cm_m_out: Optional[torch.Tensor] = None, coords: str = "ptetaphim",
                    coords2: Optional[str] = None):
    """gvx_pair_histograms: lab mass + lab histogram + CM mass + CM histogram of the pairs in ONE
    pass over the inputs (bit-identical to invariant_mass / mass_histogram / mass_histogram(cm=True)).
    Returns ``(lab_bins, cm_bins)`` ([nbins+2] int64 each, accumulated)."""
    a, n, dt, dev, _ = _view(v1, 4, "v1")
    b, n2, dt2, dev2, _ = _view(v2, 4, "v2")
    if n != n2:
        raise ValueError(f"length mismatch: v1 has {n} vectors, v2 has {n2}")
    if dt != dt2 or dev != dev2:
        raise ValueError("v1 and v2 must share dtype and device")
    lab_bins = _bins_arg(lab_bins, nbins, dev, "lab_bins")
    cm_bins = _bins_arg(cm_bins, nbins, dev, "cm_bins")
    mptr = _out_1d(m_out, n, dt, "m_out")
    cptr = _out_1d(cm_m_out, n, dt, "cm_m_out")
    with torch.cuda.device(dev):
        mixed, cc = _coords_args(coords, coords2)
        fn = lib.gvx_pair_histograms_mixed if mixed else lib.gvx_pair_histograms
        _check(fn(_dtype_code(dt), *cc, ctypes.byref(a), ctypes.byref(b), n, float(lo), float(hi), int(nbins),
                  lab_bins.data_ptr(), cm_bins.data_ptr(), mptr, cptr, _stream(dev)), "gvx_pair_histograms")
    return lab_bins, cm_bins


def pair_histograms_boost(v1: VecArg, v2: VecArg, bv: VecArg, beta: VecArg, lo: float = DEFAULT_LO,
                          hi: float = DEFAULT_HI, nbins: int = DEFAULT_NBINS, lab_bins: Optional[torch.Tensor] = None,
                          cm_bins: Optional[torch.Tensor] = None, m_out: Optional[torch.Tensor] = None,
                          cm_m_out: Optional[torch.Tensor] = None, out: Optional[VecArg] = None,
                          coords: str = "ptetaphim", coords2: Optional[str] = None):
    """gvx_pair_histograms_boost: pair_histograms(v1, v2) and boost(bv, beta) in ONE launch
    (bit-identical to the two calls). Returns ``(lab_bins, cm_bins, boosted)``."""
    a, n, dt, dev, _ = _view(v1, 4, "v1")
    b, n2, dt2, dev2, _ = _view(v2, 4, "v2")
    if n != n2:
        raise ValueError(f"length mismatch: v1 has {n} vectors, v2 has {n2}")
    c, nb, dtc, devc, _ = _view(bv, 4, "bv")
    d, nb2, dtd, devd, _ = _view(beta, 3, "beta")
    if nb != nb2:
        raise ValueError(f"length mismatch: bv has {nb} vectors, beta has {nb2}")
    if len({dt, dt2, dtc, dtd}) != 1 or len({dev, dev2, devc, devd}) != 1:
        raise ValueError("all inputs must share dtype and device")
    lab_bins = _bins_arg(lab_bins, nbins, dev, "lab_bins")
    cm_bins = _bins_arg(cm_bins, nbins, dev, "cm_bins")
    mptr = _out_1d(m_out, n, dt, "m_out")
    cptr = _out_1d(cm_m_out, n, dt, "cm_m_out")
    out, o = _boost_out(bv, nb, dt, dev, out)
    with torch.cuda.device(dev):
        mixed, cc = _coords_args(coords, coords2)
        fn = lib.gvx_pair_histograms_boost_mixed if mixed else lib.gvx_pair_histograms_boost
        _check(fn(_dtype_code(dt), *cc, ctypes.byref(a), ctypes.byref(b), n, float(lo), float(hi), int(nbins),
                  lab_bins.data_ptr(), cm_bins.data_ptr(), mptr, cptr, ctypes.byref(c), ctypes.byref(d),
                  ctypes.byref(o), nb, _stream(dev)), "gvx_pair_histograms_boost")
    return lab_bins, cm_bins, out


_PEER_WORK = {}


def _peer_work(nbins: int, dev: torch.device, slot) -> torch.Tensor:
    """The zeroed device workspace gvx_mass_histogram_peers pre-reduces into (nbins+2 partial
    sums and a ticket word; every call leaves it zeroed), one per (device, nbins, slot)."""
    key = (dev.index, nbins, slot)
    if key not in _PEER_WORK:
        _PEER_WORK[key] = torch.zeros(nbins + 3, dtype=torch.int64, device=dev)
    return _PEER_WORK[key]


def mass_histogram_peers(v1: VecArg, v2: VecArg, peer_bins_dev: int, npeers: int, lo: float = DEFAULT_LO,
                         hi: float = DEFAULT_HI, nbins: int = DEFAULT_NBINS, cm: bool = False,
                         m_out: Optional[torch.Tensor] = None, coords: str = "ptetaphim",
                         mc_bins: Optional[int] = None, work: Optional[torch.Tensor] = None) -> None:
    """gvx_mass_histogram_peers: the fused histogram whose CTAs pre-reduce into a device-local
    workspace (``work``: int64[nbins+3], zero, left zero; default: one cached per device, nbins
    and stream) and whose last CTA adds the totals into every peer's bins (``peer_bins_dev``:
    device address of an array of ``npeers`` device pointers) or into one multicast address
    (``mc_bins``). The caller owns the cross-rank barriers around the call (see
    allreduce_mass_histogram)."""
    a, n, dt, dev, _ = _view(v1, 4, "v1")
    b, n2, dt2, dev2, _ = _view(v2, 4, "v2")
    if n != n2:
        raise ValueError(f"length mismatch: v1 has {n} vectors, v2 has {n2}")
    if dt != dt2 or dev != dev2:
        raise ValueError("v1 and v2 must share dtype and device")
    mptr = _out_1d(m_out, n, dt, "m_out")
    if work is None:
        work = _peer_work(int(nbins), dev, _stream(dev))
    elif work.dtype != torch.int64 or work.device != dev or work.numel() < nbins + 3 or not work.is_contiguous():
        raise ValueError(f"work must be a contiguous int64 tensor of >= nbins+3 = {nbins + 3} on {dev}")
    with torch.cuda.device(dev):
        _check(lib.gvx_mass_histogram_peers(_dtype_code(dt), _coords_code(coords), ctypes.byref(a), ctypes.byref(b), n,
                                            float(lo), float(hi), int(nbins), int(peer_bins_dev) or None,
                                            int(npeers), mc_bins, work.data_ptr(), GVX_HIST_BOOST_TO_CM if cm else 0,
                                            mptr, _stream(dev)), "gvx_mass_histogram_peers")


_SYMM_BINS = {}


def allreduce_mass_histogram(v1: VecArg, v2: VecArg, lo: float = DEFAULT_LO, hi: float = DEFAULT_HI,
                             nbins: int = DEFAULT_NBINS, cm: bool = False, group=None,
                             coords: str = "ptetaphim", multicast: bool = False, slot: int = 0) -> torch.Tensor:
    """Global histogram of every rank's shard with the all-reduce fused into the kernel tail
    (SURVEY §8(e)): the bins live in torch symmetric memory (one int64[nbins+2] per rank,
    peer-mapped over NVLink); a device barrier after zeroing, the kernel adds each CTA's counts
    into all ranks' bins (P2P atomics, or one multimem.red to the NVSwitch multicast address when
    ``multicast`` and the group supports it), a device barrier, and every rank holds the total.
    Returns this rank's symmetric bins tensor, one per (group, nbins, device, ``slot``), reused
    across calls: copy it (or use another slot) to keep a result."""
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    a, _, _, dev, _ = _view(v1, 4, "v1")
    group = group or dist.group.WORLD
    key = (id(group), nbins, dev.index, slot)
    if key not in _SYMM_BINS:
        bins = symm.empty(nbins + 2, dtype=torch.int64, device=dev)
        hdl = symm.rendezvous(bins, group)
        # this tensor's address in every rank's mapping (its offset inside the symmetric buffer
        # is the same on all ranks), as a device array for the kernel
        off = bins.data_ptr() - int(hdl.buffer_ptrs[hdl.rank])
        ptrs = torch.tensor([int(p) + off for p in hdl.buffer_ptrs], dtype=torch.int64, device=dev)
        try:  # 0 when the group has no NVSwitch multicast object
            mcp = int(hdl.multicast_ptr or 0)
        except (RuntimeError, TypeError):
            mcp = 0
        mc = mcp + off if mcp else None
        _SYMM_BINS[key] = (bins, hdl, ptrs, mc)
    bins, hdl, ptrs, mc = _SYMM_BINS[key]
    bins.zero_()
    hdl.barrier(channel=0)
    mass_histogram_peers(v1, v2, ptrs.data_ptr(), ptrs.numel(), lo, hi, nbins, cm=cm, coords=coords,
                         mc_bins=mc if multicast else None)
    hdl.barrier(channel=0)
    return bins


def allreduce_bins(bins: torch.Tensor, group=None) -> torch.Tensor:
    """The path's only cross-rank exchange: all-reduce(SUM) of the int64
    bin counters, in place. No-op without an initialised multi-rank process group."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(bins, op=dist.ReduceOp.SUM, group=group)
    return bins
