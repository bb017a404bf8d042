"""One dimuon_histogram launch on 1e8 jagged events (for ncu). Not a benchmark."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2312_02756_b200 as gvx  # noqa: E402
import synth.device as sd  # noqa: E402
dt = torch.float64 if (len(sys.argv) < 2 or sys.argv[1] == "f64") else torch.float32
mu, q, off = sd.jagged_events(0, 100_000_000, dtype=dt)
torch.cuda.synchronize()
gvx.dimuon_histogram(mu, q, off)
torch.cuda.synchronize()
