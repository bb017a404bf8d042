"""Probe: does running the HBM-bound boost concurrently with the FP64-bound CM histogram
(two streams) shorten their combined time? Not a benchmark; prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02756_b200 as gvx  # noqa: E402
import synth.device as sd  # noqa: E402

n = int(float(os.environ.get("N", "1e8")))
dt = torch.float64
v1, v2 = sd.muon_pairs(n, dtype=dt)
bv, bb = sd.boost_inputs(n, dtype=dt)
out = torch.empty_like(bv)
bins = gvx.new_bins()
s1 = torch.cuda.Stream()
s2 = torch.cuda.Stream()


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def boost():
    gvx.boost(bv, bb, out=out)


def cm():
    gvx.mass_histogram(v1, v2, bins=bins, cm=True)


def both_seq():
    boost()
    cm()


def both_conc():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        boost()
    with torch.cuda.stream(s2):
        cm()
    cur.wait_stream(s1)
    cur.wait_stream(s2)


r = {"cfg": os.environ.get("GVX_TMA_CFG", "default"), "boost": timed(boost), "cm": timed(cm),
     "seq": timed(both_seq), "concurrent": timed(both_conc)}
print(json.dumps(r))
