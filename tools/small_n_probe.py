"""Probe: histogram kernels at small N (L2 flushed between reps), best of 10 — to choose the
TMA ring vs register-kernel crossover. Prints JSON lines. Not a benchmark."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02756_b200 as gvx  # noqa: E402
import synth.device as sd  # noqa: E402

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for dt in (torch.float64, torch.float32):
    for n in (10_000, 100_000, 300_000, 1_000_000, 3_000_000):
        v1, v2 = sd.muon_pairs(n, dtype=dt)
        bins = gvx.new_bins()
        for cm in (False, True):
            best = 1e9
            for _ in range(12):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                gvx.mass_histogram(v1, v2, bins=bins, cm=cm)
                b.record()
                b.synchronize()
                best = min(best, a.elapsed_time(b))
            print(json.dumps({"dtype": str(dt)[6:], "n": n, "cm": cm, "us": best * 1e3,
                              "tma": os.environ.get("GVX_DISABLE_TMA") != "1"}))
