"""Transfer-inclusive mode ("handling the device
memory allocation and transfers if necessary"): run the whole hot-path step on
inputs that live in pinned HOST memory.

The batch is cut into chunks that cycle through ``nslots`` device buffers. For
chunk c: the copy-in stream uploads it (H2D), the compute stream runs the four
kernels on it, and the copy-out stream downloads its masses and boosted vectors
(D2H). Events order the three streams, so the upload of chunk c+1 and the
download of chunk c-1 overlap the kernels of chunk c; the bins stay on the
device until the last chunk and are downloaded once. The caller's current
stream waits for everything, so CUDA events recorded on it bracket the whole
transfer-inclusive step.
"""
from __future__ import annotations

import torch

from . import boost, invariant_mass, mass_histogram


class HostPipeline:
    def __init__(self, n: int, dtype: torch.dtype, device, nbins: int = 1000, lo: float = 0.25,
                 hi: float = 300.0, chunk: int = 1 << 23, nslots: int = 2):
        self.n, self.dtype, self.dev = n, dtype, torch.device(device)
        self.nbins, self.lo, self.hi = nbins, lo, hi
        self.chunk = max(1, min(chunk, n))
        self.nslots = nslots
        c = self.chunk
        mk = lambda *s: torch.empty(s, dtype=dtype, device=self.dev)  # noqa: E731
        self.slots = [dict(v1=mk(c, 4), v2=mk(c, 4), bv=mk(c, 4), bb=mk(c, 3), m=mk(c), bout=mk(c, 4))
                      for _ in range(nslots)]
        self.bins = torch.zeros(2, nbins + 2, dtype=torch.int64, device=self.dev)
        self.h_m = torch.empty(n, dtype=dtype, pin_memory=True)
        self.h_bout = torch.empty((n, 4), dtype=dtype, pin_memory=True)
        self.h_bins = torch.empty((2, nbins + 2), dtype=torch.int64, pin_memory=True)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.ev_in = [torch.cuda.Event() for _ in range(nslots)]
        self.ev_cmp = [torch.cuda.Event() for _ in range(nslots)]
        self.ev_free = [torch.cuda.Event() for _ in range(nslots)]
        es = torch.empty((), dtype=dtype).element_size()
        self.h2d_bytes = n * (4 + 4 + 4 + 3) * es
        self.d2h_bytes = n * (1 + 4) * es + 2 * (nbins + 2) * 8

    def step(self, h_v1, h_v2, h_bv, h_bb):
        """One transfer-inclusive step; returns pinned host (masses, boosted vectors, bins[2])."""
        cur = torch.cuda.current_stream(self.dev)
        for s in (self.s_in, self.s_cmp, self.s_out):
            s.wait_stream(cur)
        with torch.cuda.stream(self.s_cmp):
            self.bins.zero_()
        for c, a in enumerate(range(0, self.n, self.chunk)):
            b = min(a + self.chunk, self.n)
            k = b - a
            j = c % self.nslots
            sl = self.slots[j]
            if c >= self.nslots:
                self.s_in.wait_event(self.ev_free[j])
            with torch.cuda.stream(self.s_in):
                sl["v1"][:k].copy_(h_v1[a:b], non_blocking=True)
                sl["v2"][:k].copy_(h_v2[a:b], non_blocking=True)
                sl["bv"][:k].copy_(h_bv[a:b], non_blocking=True)
                sl["bb"][:k].copy_(h_bb[a:b], non_blocking=True)
                self.ev_in[j].record(self.s_in)
            self.s_cmp.wait_event(self.ev_in[j])
            with torch.cuda.stream(self.s_cmp):
                invariant_mass(sl["v1"][:k], sl["v2"][:k], out=sl["m"][:k])
                boost(sl["bv"][:k], sl["bb"][:k], out=sl["bout"][:k])
                mass_histogram(sl["v1"][:k], sl["v2"][:k], self.lo, self.hi, self.nbins, bins=self.bins[0])
                mass_histogram(sl["v1"][:k], sl["v2"][:k], self.lo, self.hi, self.nbins, bins=self.bins[1],
                               cm=True)
                self.ev_cmp[j].record(self.s_cmp)
            self.s_out.wait_event(self.ev_cmp[j])
            with torch.cuda.stream(self.s_out):
                self.h_m[a:b].copy_(sl["m"][:k], non_blocking=True)
                self.h_bout[a:b].copy_(sl["bout"][:k], non_blocking=True)
                self.ev_free[j].record(self.s_out)
        self.s_out.wait_stream(self.s_cmp)
        with torch.cuda.stream(self.s_out):
            self.h_bins.copy_(self.bins, non_blocking=True)
        cur.wait_stream(self.s_out)
        cur.wait_stream(self.s_in)
        return self.h_m, self.h_bout, self.h_bins
