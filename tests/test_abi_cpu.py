"""Host-side checks that need no GPU: the C-ABI library loads, exports every
symbol include/gvx.h declares, and its synchronous validation returns the
documented status codes without enqueuing anything (no CUDA call is reached)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gvx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_boundary():
    names = declared("gvx.h")
    for want in ("gvx_invariant_mass", "gvx_boost", "gvx_boost_uniform", "gvx_mass_histogram",
                 "gvx_status_string", "gvx_abi_version", "gvx_last_cuda_error_string"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2312_02756_b200", "libgvx.so"))
    for name in declared("gvx.h"):
        assert hasattr(lib, name), name


@pytest.fixture(scope="module")
def gvx():
    import paper_2312_02756_b200 as g
    return g


def _view(ptr=0x1000, stride=4, es=8):
    v = __import__("paper_2312_02756_b200").Vec4CView()
    for k in range(4):
        v.c[k] = ptr + k * es if ptr else None
    v.stride = stride
    return v


def test_validation_codes(gvx):
    L = gvx.lib
    a, b = _view(), _view()
    by = ctypes.byref
    assert L.gvx_abi_version() == gvx.ABI_VERSION
    assert L.gvx_status_string(gvx.GVX_ERR_DOMAIN) == b"GVX_ERR_DOMAIN"
    # n < 0, bad dtype, bad coords
    assert L.gvx_invariant_mass(gvx.GVX_F64, gvx.GVX_PTETAPHIM, by(a), by(b), 0x2000, -1, None) == 1
    assert L.gvx_invariant_mass(7, gvx.GVX_PTETAPHIM, by(a), by(b), 0x2000, 4, None) == 1
    assert L.gvx_invariant_mass(gvx.GVX_F64, 9, by(a), by(b), 0x2000, 4, None) == 1
    # n == 0 is OK with nothing launched, even with NULL views
    assert L.gvx_invariant_mass(gvx.GVX_F64, gvx.GVX_PTETAPHIM, None, None, None, 0, None) == 0
    # NULL component pointer, stride < 1, misaligned pointer, NULL output
    assert L.gvx_invariant_mass(gvx.GVX_F64, gvx.GVX_PTETAPHIM, by(_view(0)), by(b), 0x2000, 4, None) == 1
    assert L.gvx_invariant_mass(gvx.GVX_F64, gvx.GVX_PTETAPHIM, by(_view(stride=0)), by(b), 0x2000, 4, None) == 1
    assert L.gvx_invariant_mass(gvx.GVX_F64, gvx.GVX_PTETAPHIM, by(_view(0x1004)), by(b), 0x2000, 4, None) == 1
    assert L.gvx_invariant_mass(gvx.GVX_F64, gvx.GVX_PTETAPHIM, by(a), by(b), None, 4, None) == 1
    # uniform boost: |β| ≥ 1 and non-finite β are domain errors
    o = gvx.Vec4View()
    for k in range(4):
        o.c[k] = 0x3000 + 8 * k
    o.stride = 4
    assert L.gvx_boost_uniform(gvx.GVX_F64, by(a), 0.9, 0.9, 0.0, by(o), 4, None) == 2
    assert L.gvx_boost_uniform(gvx.GVX_F64, by(a), 0.0, 0.0, 1.0, by(o), 4, None) == 2
    assert L.gvx_boost_uniform(gvx.GVX_F32, by(a), float("nan"), 0.0, 0.0, by(o), 4, None) == 2
    assert L.gvx_boost_uniform(gvx.GVX_F64, by(a), 0.1, 0.0, 0.0, by(o), 0, None) == 0
    # histogram: bad range / nbins / flags / boosted_out without CM
    H = L.gvx_mass_histogram
    assert H(gvx.GVX_F64, 0, by(a), by(b), 4, 1.0, 1.0, 10, 0x4000, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, float("inf"), 10, 0x4000, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 0, 0x4000, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0x80, None, None, None) == 1
    assert H(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0, None, by(o), None) == 1
    assert H(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, None, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, 0, by(a), by(b), 0, 0.0, 1.0, 10, None, 0, None, None, None) == 0


def test_cm_costheta_validation(gvx):
    """gvx_cm_costheta_histogram (ABI v3) validates both axes, both bin arrays and the
    optional outputs synchronously; n == 0 is OK with nothing launched."""
    L = gvx.lib
    by = ctypes.byref
    a, b = _view(), _view()
    C = L.gvx_cm_costheta_histogram
    ok_m, ok_c = (0.25, 300.0, 1000), (-1.0, 1.0, 100)

    def call(n=4, m=ok_m, c=ok_c, mb=0x4000, cb=0x5000, mo=None, co=None, dt=gvx.GVX_F64, coords=0):
        return C(dt, coords, by(a), by(b), n, m[0], m[1], m[2], mb, c[0], c[1], c[2], cb, mo, co, None)

    assert call(m=(1.0, 1.0, 10)) == 1                    # lo >= hi (mass axis)
    assert call(c=(1.0, -1.0, 10)) == 1                   # lo >= hi (angle axis)
    assert call(c=(-1.0, float("nan"), 10)) == 1          # non-finite edge
    assert call(m=(0.0, 1.0, 0)) == 1                     # nbins < 1
    assert call(c=(0.0, 1.0, 1 << 29)) == 1               # nbins too large
    assert call(mb=None) == 1 and call(cb=None) == 1      # missing bins
    assert call(cb=0x5004) == 1                           # misaligned bins
    assert call(co=0x6001) == 1                           # misaligned cos output
    assert call(dt=7) == 1 and call(coords=9) == 1 and call(n=-1) == 1
    assert call(n=0, mb=None, cb=None) == 0               # n == 0: OK, nothing launched
    assert call(n=0, m=(1.0, 1.0, 10)) == 1               # ... but a bad axis is still an error


def test_pair_histograms_validation(gvx):
    """gvx_pair_histograms (ABI v5) validates the axis, both bin arrays and the optional mass
    outputs synchronously; n == 0 is OK with nothing launched."""
    L = gvx.lib
    by = ctypes.byref
    a, b = _view(), _view()
    P = L.gvx_pair_histograms

    def call(n=4, ax=(0.25, 300.0, 1000), lb=0x4000, cb=0x5000, mo=None, co=None, dt=gvx.GVX_F64, coords=0):
        return P(dt, coords, by(a), by(b), n, ax[0], ax[1], ax[2], lb, cb, mo, co, None)

    assert call(ax=(1.0, 1.0, 10)) == 1                   # lo >= hi
    assert call(ax=(float("-inf"), 1.0, 10)) == 1         # non-finite edge
    assert call(ax=(0.0, 1.0, 0)) == 1 and call(ax=(0.0, 1.0, 1 << 29)) == 1
    assert call(lb=None) == 1 and call(cb=None) == 1      # missing bins
    assert call(lb=0x4004) == 1 and call(cb=0x5002) == 1  # misaligned bins
    assert call(mo=0x6001) == 1 and call(co=0x7003) == 1  # misaligned mass outputs
    assert call(dt=7) == 1 and call(coords=9) == 1 and call(n=-1) == 1
    assert call(n=0, lb=None, cb=None) == 0               # n == 0: OK, nothing launched
    assert call(n=0, ax=(1.0, 1.0, 10)) == 1              # ... but a bad axis is still an error


def test_pair_histograms_boost_validation(gvx):
    """gvx_pair_histograms_boost (ABI v6) validates the axis, the pair and the boost arguments
    synchronously; empty batches are OK with nothing launched."""
    L = gvx.lib
    by = ctypes.byref
    a, b, v = _view(), _view(), _view()
    beta = gvx.Vec3CView()
    beta.c[0], beta.c[1], beta.c[2], beta.stride = 0x9000, 0x9008, 0x9010, 3
    out = gvx.Vec4View()
    for k in range(4):
        out.c[k] = 0xA000 + 8 * k
    out.stride = 4
    F = L.gvx_pair_histograms_boost

    def call(n=4, nb=4, ax=(0.25, 300.0, 1000), lb=0x4000, cb=0x5000, dt=gvx.GVX_F64, coords=0, bo=out):
        return F(dt, coords, by(a), by(b), n, ax[0], ax[1], ax[2], lb, cb, None, None, by(v), by(beta), by(bo), nb,
                 None)

    assert call(ax=(1.0, 1.0, 10)) == 1 and call(ax=(0.0, 1.0, 0)) == 1
    assert call(lb=None) == 1 and call(cb=0x5004) == 1
    assert call(n=-1) == 1 and call(nb=-1) == 1 and call(dt=7) == 1 and call(coords=9) == 1
    bad = gvx.Vec4View()
    bad.c[0], bad.stride = 0xA001, 4
    assert call(bo=bad) == 1                              # misaligned boost output
    assert call(n=0, nb=0, lb=None, cb=None) == 0         # both batches empty: nothing launched


def test_mass_histogram_peers_validation(gvx):
    """The fused-reduction entry point (ABI v4) checks its sink arguments synchronously."""
    L = gvx.lib
    by = ctypes.byref
    a, b = _view(), _view()
    P = L.gvx_mass_histogram_peers
    W = 0x6000  # an aligned (never dereferenced) workspace address
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, None, 2, None, W, 0, None, None) == 1     # no peers
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0, None, W, 0, None, None) == 1   # npeers < 1
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, 0x4004, 2, None, W, 0, None, None) == 1   # misaligned
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, None, 0, 0x5001, W, 0, None, None) == 1   # misaligned mc
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 1.0, 1.0, 10, 0x4000, 2, None, W, 0, None, None) == 1   # bad axis
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 2, None, None, 0, None, None) == 1  # no work
    assert P(gvx.GVX_F64, 0, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 2, None, W + 4, 0, None, None) == 1  # misaligned
    assert P(gvx.GVX_F64, 0, by(a), by(b), 0, 0.0, 1.0, 10, 0x4000, 2, None, W, 0, None, None) == 0   # n == 0


def test_dimuon_axis_limit(gvx):
    """gvx_dimuon_histogram privatises its counters in shared memory: nbins + 2 > 49152 is
    GVX_ERR_UNSUPPORTED (documented in gvx.h), returned before anything is launched."""
    L = gvx.lib
    mu = _view()
    r = L.gvx_dimuon_histogram(gvx.GVX_F64, ctypes.byref(mu), 0x5000, 0x6000, 10, 0.0, 1.0, 60_000, 0x7000, None,
                               None)
    assert r == 3
    assert L.gvx_dimuon_histogram(gvx.GVX_F64, ctypes.byref(mu), 0x5000, 0x6000, 10, 1.0, 1.0, 10, 0x7000, None,
                                  None) == 1


def test_lorentz_matrix_validation(gvx):
    """gvx_lorentz_transform checks L^T g L = g on the host before anything is enqueued."""
    L = gvx.lib
    by = ctypes.byref
    a, o = _view(), gvx.Vec4View()
    for k in range(4):
        o.c[k] = 0x3000 + 8 * k
    o.stride = 4
    D = ctypes.c_double * 16
    eye = D(*[1.0 if i % 5 == 0 else 0.0 for i in range(16)])
    two = D(*[2.0 if i % 5 == 0 else 0.0 for i in range(16)])
    nan = D(*[float("nan")] * 16)
    import math
    g, b = 1 / math.sqrt(1 - 0.36), 0.6
    boost_z = D(1, 0, 0, 0, 0, 1, 0, 0, 0, 0, g, g * b, 0, 0, g * b, g)
    assert L.gvx_lorentz_transform(gvx.GVX_F64, by(a), eye, by(o), 0, None) == 0
    assert L.gvx_lorentz_transform(gvx.GVX_F64, by(a), boost_z, by(o), 0, None) == 0
    assert L.gvx_lorentz_transform(gvx.GVX_F64, by(a), two, by(o), 4, None) == 2
    assert L.gvx_lorentz_transform(gvx.GVX_F32, by(a), nan, by(o), 4, None) == 2
    assert L.gvx_lorentz_transform(gvx.GVX_F64, by(a), None, by(o), 4, None) == 1


def test_host_pipeline_validation():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2312_02756_b200", "libgvx.so"))
    P = ctypes.c_void_p
    lib.gvx_host_pipeline_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.POINTER(P)]
    lib.gvx_host_pairs.argtypes = [P, ctypes.c_int, P, P, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_int32, P, P, P, P]
    lib.gvx_host_boost.argtypes = [P, P, P, ctypes.c_int64, P, P]
    lib.gvx_host_pipeline_destroy.argtypes = [P]
    out = P()
    assert lib.gvx_host_pipeline_create(9, 1024, ctypes.byref(out)) == 1          # bad dtype
    assert lib.gvx_host_pipeline_create(1, 0, ctypes.byref(out)) == 1             # chunk < 1
    assert lib.gvx_host_pipeline_create(1, 1 << 40, ctypes.byref(out)) == 1       # chunk > 2^31
    assert lib.gvx_host_pairs(None, 0, None, None, 4, 0.0, 1.0, 10, None, None, None, None) == 1
    assert lib.gvx_host_boost(None, None, None, 4, None, None) == 1
    assert lib.gvx_host_pipeline_destroy(None) == 1


def test_python_binding_rejects_cpu_tensors(gvx):
    import torch
    with pytest.raises(ValueError, match="CUDA"):
        gvx.invariant_mass(torch.zeros(3, 4, dtype=torch.float64), torch.zeros(3, 4, dtype=torch.float64))


def test_oracle_is_test_infrastructure_only():
    """The product package never imports the oracle (no CPU fallback path)."""
    pkg = os.path.join(ROOT, "paper_2312_02756_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).lower().replace("no oracle", ""), f


def test_binding_rejects_unsupported_strides(gvx, monkeypatch):
    """Broadcast (stride 0) views are rejected before any call (checked with a fake CUDA tensor
    flag: _view only inspects shapes and strides)."""
    import torch
    t = torch.zeros(1, 4, dtype=torch.float64).expand(5, 4)
    monkeypatch.setattr(gvx, "_require_cuda", lambda x, name: None)
    with pytest.raises(ValueError, match="stride"):
        gvx._view(t, 4, "v1")


def test_mixed_coords_validation(gvx):
    """The mixed-coordinate entry points (ABI v7) validate both systems and the rest of their
    arguments synchronously, exactly as the single-system calls; n == 0 launches nothing."""
    L = gvx.lib
    by = ctypes.byref
    a, b = _view(), _view()
    PM, PE = gvx.GVX_PTETAPHIM, gvx.GVX_PXPYPZE
    M = L.gvx_invariant_mass_mixed
    assert M(gvx.GVX_F64, PM, 9, by(a), by(b), 0x2000, 4, None) == 1      # bad coords2
    assert M(gvx.GVX_F64, 9, PE, by(a), by(b), 0x2000, 4, None) == 1      # bad coords1
    assert M(gvx.GVX_F64, PM, PE, by(a), by(b), 0x2000, -1, None) == 1
    assert M(7, PM, PE, by(a), by(b), 0x2000, 4, None) == 1
    assert M(gvx.GVX_F64, PM, PE, by(a), by(b), None, 4, None) == 1       # NULL output
    assert M(gvx.GVX_F64, PM, PE, by(_view(0x1004)), by(b), 0x2000, 4, None) == 1
    assert M(gvx.GVX_F64, PM, PE, None, None, None, 0, None) == 0         # empty: OK
    H = L.gvx_mass_histogram_mixed
    assert H(gvx.GVX_F64, PM, PE, by(a), by(b), 4, 1.0, 1.0, 10, 0x4000, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, PM, PE, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0x80, None, None, None) == 1
    assert H(gvx.GVX_F64, PM, PE, by(a), by(b), 4, 0.0, 1.0, 10, None, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, PM, 5, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0, None, None, None) == 1
    assert H(gvx.GVX_F64, PM, PE, by(a), by(b), 0, 0.0, 1.0, 10, None, 0, None, None, None) == 0
    P = L.gvx_pair_histograms_mixed
    assert P(gvx.GVX_F32, PM, PE, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, None, None, None, None) == 1
    assert P(gvx.GVX_F32, PM, PE, by(a), by(b), 4, 0.0, 1.0, 0, 0x4000, 0x5000, None, None, None) == 1
    assert P(gvx.GVX_F32, PM, PE, by(a), by(b), 0, 0.0, 1.0, 10, None, None, None, None, None) == 0
    beta = gvx.Vec3CView()
    beta.c[0], beta.c[1], beta.c[2], beta.stride = 0x9000, 0x9008, 0x9010, 3
    out = gvx.Vec4View()
    for k in range(4):
        out.c[k] = 0xA000 + 8 * k
    out.stride = 4
    F = L.gvx_pair_histograms_boost_mixed
    assert F(gvx.GVX_F64, PM, PE, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0x5000, None, None, by(a), by(beta),
             by(out), -1, None) == 1
    bad = gvx.Vec4View()
    bad.c[0], bad.stride = 0xA001, 4
    # a bad boost half is caught before the pair half is enqueued
    assert F(gvx.GVX_F64, PM, PE, by(a), by(b), 4, 0.0, 1.0, 10, 0x4000, 0x5000, None, None, by(a), by(beta),
             by(bad), 4, None) == 1
    assert F(gvx.GVX_F64, PM, PE, by(a), by(b), 0, 0.0, 1.0, 10, None, None, None, None, None, None, None, 0,
             None) == 0


def test_host_pipeline_validation(gvx):
    """gvx_host_pairs validates coords and the axis before anything is enqueued (no pipeline
    needed to reach these checks: a NULL pipeline is itself INVALID_ARGUMENT)."""
    import paper_2312_02756_b200.hostpipe  # noqa: F401  (sets the host-pipeline argtypes)
    L = gvx.lib
    assert L.gvx_host_pairs(None, 0, 0x1000, 0x2000, 4, 0.0, 1.0, 10, None, 0x3000, None, None) == 1
    assert L.gvx_host_pipeline_create(7, 1024, ctypes.byref(ctypes.c_void_p())) == 1
    assert L.gvx_host_pipeline_create(gvx.GVX_F64, 0, ctypes.byref(ctypes.c_void_p())) == 1
