"""One launch of each hot-path kernel at the bench configuration (N = 1e8 per kernel,
AoS), for `ncu --set full` captures. Not a benchmark: numbers printed under a
profiler are never reported."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2312_02756_b200 as gvx  # noqa: E402
import synth.device as sd  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--dtype", default="f64")
p.add_argument("--events", type=float, default=1e8)
p.add_argument("--reps", type=int, default=1)
p.add_argument("--layout", default="aos")
a = p.parse_args()
tdt = torch.float64 if a.dtype == "f64" else torch.float32
n = int(a.events)
v1, v2 = sd.muon_pairs(n, dtype=tdt)
bv, bb = sd.boost_inputs(n, dtype=tdt)
if a.layout == "soa":
    v1 = [v1[:, k].contiguous() for k in range(4)]
    v2 = [v2[:, k].contiguous() for k in range(4)]
m = torch.empty(n, dtype=tdt, device="cuda")
out = torch.empty((n, 4), dtype=tdt, device="cuda")
bins = gvx.new_bins()
torch.cuda.synchronize()
for _ in range(a.reps):
    gvx.invariant_mass(v1, v2, out=m)
    gvx.boost(bv, bb, out=out)
    gvx.mass_histogram(v1, v2, bins=bins)
    gvx.mass_histogram(v1, v2, bins=bins, cm=True)
    gvx.cm_costheta_histogram(v1, v2)
    gvx.pair_histograms(v1, v2, m_out=m)
    gvx.pair_histograms_boost(v1, v2, bv, bb, m_out=m, out=out)
torch.cuda.synchronize()
print("prof_step done")
