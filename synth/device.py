"""Device twin of :mod:`synth` (libgvxsynth.so): fills CUDA tensors with the same
events the host generator draws for the same global indices. Not the method's
arithmetic — only the shared input generator (see synth/__init__.py)."""
from __future__ import annotations

import ctypes
import os

import torch

from . import DEFAULT_SEED

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libgvxsynth.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_LIB)
        for f in (lib.gvx_synth_muon_pairs, lib.gvx_synth_boost_inputs):
            f.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                          ctypes.c_void_p, ctypes.c_void_p]
            f.restype = ctypes.c_int
        lib.gvx_synth_muon_pairs.argtypes = lib.gvx_synth_muon_pairs.argtypes + [ctypes.c_double]
        lib.gvx_synth_jagged_counts.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, ctypes.c_void_p,
                                                ctypes.c_void_p]
        lib.gvx_synth_jagged_counts.restype = ctypes.c_int
        lib.gvx_synth_jagged_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.gvx_synth_jagged_fill.restype = ctypes.c_int
        lib.gvx_synth_stream_read.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        lib.gvx_synth_stream_read.restype = ctypes.c_int
        _lib = lib
    return _lib


def _code(dtype):
    return 1 if dtype == torch.float64 else 0


def muon_pairs(n: int, first: int = 0, seed: int = DEFAULT_SEED, dtype=torch.float64, device="cuda", out=None,
               f_res: float = 0.0):
    """(v1, v2) [n, 4] PtEtaPhiM AoS for global event indices first .. first+n-1 (``f_res``: the
    fraction of Z-like resonance pairs, see synth.muon_pairs)."""
    dev = torch.device(device)
    if out is None:
        v1 = torch.empty((n, 4), dtype=dtype, device=dev)
        v2 = torch.empty((n, 4), dtype=dtype, device=dev)
    else:
        v1, v2 = out
    with torch.cuda.device(dev):
        rc = _load().gvx_synth_muon_pairs(_code(dtype), seed, first, n, v1.data_ptr(), v2.data_ptr(),
                                          torch.cuda.current_stream(dev).cuda_stream, float(f_res))
    if rc:
        raise RuntimeError(f"gvx_synth_muon_pairs: cuda error {rc}")
    return v1, v2


def boost_inputs(n: int, first: int = 0, seed: int = DEFAULT_SEED, dtype=torch.float64, device="cuda", out=None):
    """(v [n, 4] PxPyPzE, beta [n, 3]) for global event indices first .. first+n-1."""
    dev = torch.device(device)
    if out is None:
        v = torch.empty((n, 4), dtype=dtype, device=dev)
        beta = torch.empty((n, 3), dtype=dtype, device=dev)
    else:
        v, beta = out
    with torch.cuda.device(dev):
        rc = _load().gvx_synth_boost_inputs(_code(dtype), seed, first, n, v.data_ptr(), beta.data_ptr(),
                                            torch.cuda.current_stream(dev).cuda_stream)
    if rc:
        raise RuntimeError(f"gvx_synth_boost_inputs: cuda error {rc}")
    return v, beta


def jagged_events(first_event: int, n_events: int, seed: int = DEFAULT_SEED, dtype=torch.float64, device="cuda"):
    """Device twin of synth.jagged_events: (muons [M, 4], charge int32 [M], offsets int64 [n+1])."""
    dev = torch.device(device)
    with torch.cuda.device(dev):
        st = torch.cuda.current_stream(dev).cuda_stream
        counts = torch.empty(n_events, dtype=torch.int64, device=dev)
        rc = _load().gvx_synth_jagged_counts(seed, first_event, n_events, counts.data_ptr(), st)
        if rc:
            raise RuntimeError(f"gvx_synth_jagged_counts: cuda error {rc}")
        offsets = torch.zeros(n_events + 1, dtype=torch.int64, device=dev)
        torch.cumsum(counts, 0, out=offsets[1:])
        m = int(offsets[-1].item())
        mu = torch.empty((m, 4), dtype=dtype, device=dev)
        q = torch.empty(m, dtype=torch.int32, device=dev)
        rc = _load().gvx_synth_jagged_fill(_code(dtype), seed, first_event, n_events, offsets.data_ptr(),
                                           mu.data_ptr(), q.data_ptr(), st)
        if rc:
            raise RuntimeError(f"gvx_synth_jagged_fill: cuda error {rc}")
    return mu, q, offsets


def stream_read_gbs(buffers, reps: int = 5) -> float:
    """K5: achievable HBM read bandwidth, GB/s, of one streaming pass over the
    given device tensors (each read once per rep; take buffers much larger than L2), CUDA
    events on the current stream, best of ``reps``."""
    lib = _load()
    dev = buffers[0].device
    sink = torch.zeros(1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    total = 0
    for b in buffers:
        total += (b.numel() * b.element_size()) // 16384 * 16384  # whole 16-KB tiles
    best = float("inf")
    for _ in range(reps + 1):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for b in buffers:
            rc = lib.gvx_synth_stream_read(b.data_ptr(), b.numel() * b.element_size(), sink.data_ptr(),
                                           st.cuda_stream)
            if rc != 0:
                raise RuntimeError(f"gvx_synth_stream_read: cuda error {rc}")
        z.record(st)
        z.synchronize()
        best = min(best, a.elapsed_time(z))
    return total / (best * 1e-3) / 1e9
