"""Transfer-inclusive mode ("handling the device
memory allocation and transfers if necessary"): the hot-path step on inputs that
live in pinned HOST memory, through the C ABI's host pipeline
(``gvx_host_pipeline_*``, ``gvx_host_pairs``, ``gvx_host_boost`` in
include/gvx.h; csrc/gvx_host.cu).

The native pipeline owns three CUDA streams and a ring of device staging slots;
within one call, chunk c's H2D copy, chunk c-1's kernels and chunk c-2's D2H copy
overlap. This module only allocates the pinned output buffers and marshals
pointers; the caller's current stream is made to wait for each call, so CUDA
events recorded on it bracket the whole transfer-inclusive step.
"""
from __future__ import annotations

import ctypes

import torch

from . import (DEFAULT_HI, DEFAULT_LO, DEFAULT_NBINS, GVX_HIST_BOOST_TO_CM, _check, _coords_code, _dtype_code,
               lib)

_P = ctypes.c_void_p
lib.gvx_host_pipeline_create.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.POINTER(_P)]
lib.gvx_host_pipeline_create.restype = ctypes.c_int
lib.gvx_host_pipeline_destroy.argtypes = [_P]
lib.gvx_host_pipeline_destroy.restype = ctypes.c_int
lib.gvx_host_pairs.argtypes = [_P, ctypes.c_int, _P, _P, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                               ctypes.c_int32, _P, _P, _P, _P]
lib.gvx_host_pairs.restype = ctypes.c_int
lib.gvx_host_boost.argtypes = [_P, _P, _P, ctypes.c_int64, _P, _P]
lib.gvx_host_boost.restype = ctypes.c_int

assert GVX_HIST_BOOST_TO_CM == 1


def _host_ptr(t: torch.Tensor, name: str, shape, dtype) -> int:
    if t.is_cuda:
        raise ValueError(f"{name} must be a host (pinned) tensor")
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)}")
    return t.data_ptr()


class HostPipeline:
    """Reusable transfer-inclusive runner for batches of ``n`` events."""

    def __init__(self, n: int, dtype: torch.dtype, device, nbins: int = DEFAULT_NBINS, lo: float = DEFAULT_LO,
                 hi: float = DEFAULT_HI, chunk: int = 1 << 21, coords: str = "ptetaphim"):
        self.n, self.dtype, self.dev = n, dtype, torch.device(device)
        self.nbins, self.lo, self.hi, self.coords = nbins, lo, hi, coords
        self.chunk = max(1, min(chunk, max(n, 1)))
        self._p = _P()
        with torch.cuda.device(self.dev):
            _check(lib.gvx_host_pipeline_create(_dtype_code(dtype), self.chunk, ctypes.byref(self._p)),
                   "gvx_host_pipeline_create")
        self.h_m = torch.empty(n, dtype=dtype, pin_memory=True)
        self.h_bout = torch.empty((n, 4), dtype=dtype, pin_memory=True)
        self.h_bins = torch.empty((2, nbins + 2), dtype=torch.int64, pin_memory=True)
        es = torch.empty((), dtype=dtype).element_size()
        self.h2d_bytes = n * (4 + 4 + 4 + 3) * es
        self.d2h_bytes = n * (1 + 4) * es + 2 * (nbins + 2) * 8

    def step(self, h_v1, h_v2, h_bv, h_bb):
        """One transfer-inclusive step: masses, lab and CM histograms of the pairs, and the
        boosted vectors; returns the pinned host outputs (masses, boosted, bins[2])."""
        n = self.n
        p1 = _host_ptr(h_v1, "h_v1", (n, 4), self.dtype)
        p2 = _host_ptr(h_v2, "h_v2", (n, 4), self.dtype)
        pv = _host_ptr(h_bv, "h_bv", (n, 4), self.dtype)
        pb = _host_ptr(h_bb, "h_bb", (n, 3), self.dtype)
        with torch.cuda.device(self.dev):
            st = torch.cuda.current_stream(self.dev).cuda_stream
            _check(lib.gvx_host_pairs(self._p, _coords_code(self.coords), p1, p2, n, self.lo, self.hi, self.nbins,
                                      self.h_m.data_ptr(), self.h_bins[0].data_ptr(), self.h_bins[1].data_ptr(), st),
                   "gvx_host_pairs")
            _check(lib.gvx_host_boost(self._p, pv, pb, n, self.h_bout.data_ptr(), st), "gvx_host_boost")
        return self.h_m, self.h_bout, self.h_bins

    def close(self):
        if self._p:
            lib.gvx_host_pipeline_destroy(self._p)
            self._p = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
