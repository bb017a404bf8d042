"""Probe: transfer-inclusive step time (hostpipe) vs chunk size, f64, N = 1e8 pinned host
batch. Prints JSON lines. Not a benchmark."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth.device as sd  # noqa: E402
from paper_2312_02756_b200 import hostpipe  # noqa: E402

n = int(float(os.environ.get("N", "1e8")))
dt = torch.float64
v1, v2 = sd.muon_pairs(n, dtype=dt)
bv, bb = sd.boost_inputs(n, dtype=dt)
h = [torch.empty(t.shape, dtype=dt, pin_memory=True) for t in (v1, v2, bv, bb)]
for hh, d in zip(h, (v1, v2, bv, bb)):
    hh.copy_(d)
del v1, v2, bv, bb
for lg in (20, 21, 22, 23):
    pipe = hostpipe.HostPipeline(n, dt, "cuda", chunk=1 << lg)
    pipe.step(*h)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        pipe.step(*h)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 3
    print(json.dumps({"chunk_log2": lg, "ms": ms, "events_per_s": n / (ms * 1e-3)}), flush=True)
    pipe.close()
    del pipe
