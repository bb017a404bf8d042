"""Jagged dimuon (f4) vs the device's L2 fetch granularity (cudaLimitMaxL2FetchGranularity):
the kernel gathers one 32-B (f64) muon row per load, scattered; ncu showed DRAM bytes equal to
128-B segments of those gathers. Times gvx.dimuon_histogram at the default limit, then at 64 and
32 B. Probe only (a library must not change a device-wide limit behind its caller's back)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from cuda.bindings import runtime as rt  # noqa: E402

import paper_2312_02756_b200 as gvx  # noqa: E402
import synth.device as sd  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) for a, b in ev)
    return t[0], t[len(t) // 2]


out = []
for dt in (torch.float64, torch.float32):
    mu, q, off = sd.jagged_events(0, 100_000_000, dtype=dt)
    torch.cuda.synchronize()
    ref = gvx.dimuon_histogram(mu, q, off).clone()
    for lim in (None, 128, 64, 32):
        if lim is not None:
            err, = rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, lim)
            assert err == rt.cudaError_t.cudaSuccess, err
        err, cur = rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity)
        best, med = timed(lambda: gvx.dimuon_histogram(mu, q, off))
        same = torch.equal(gvx.dimuon_histogram(mu, q, off), ref)
        rec = {"dtype": str(dt).split(".")[-1], "limit_set": lim, "limit_now": cur, "ms_best": best,
               "ms_median": med, "bins_equal": same}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    rt.cudaDeviceSetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity, 128)
    del mu, q, off
    torch.cuda.empty_cache()
