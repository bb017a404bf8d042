"""Probe: the bench step as two launches (pair_histograms + boost) vs one launch
(pair_histograms_boost), N = 1e8 each, CUDA events, median of 20. Prints JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2312_02756_b200 as gvx  # noqa: E402
import synth.device as sd  # noqa: E402

for dtn in sys.argv[1:] or ["f64", "f32"]:
    dt = torch.float64 if dtn == "f64" else torch.float32
    n = int(float(os.environ.get("N", "1e8")))
    v1, v2 = sd.muon_pairs(n, dtype=dt)
    bv, bb = sd.boost_inputs(n, dtype=dt)
    m = torch.empty(n, dtype=dt, device="cuda")
    out = torch.empty_like(bv)
    lab, cmb = gvx.new_bins(), gvx.new_bins()

    def two():
        gvx.pair_histograms(v1, v2, lab_bins=lab, cm_bins=cmb, m_out=m)
        gvx.boost(bv, bb, out=out)

    def one():
        gvx.pair_histograms_boost(v1, v2, bv, bb, lab_bins=lab, cm_bins=cmb, m_out=m, out=out)

    res = {"dtype": dtn, "n": n}
    for name, f in (("two_launches", two), ("one_launch", one), ("two_launches_again", two), ("one_launch_again", one)):
        for _ in range(3):
            f()
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            f()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b))
        ts.sort()
        res[name] = ts[len(ts) // 2]
    print(json.dumps(res), flush=True)
