"""Debug: repeat the f64 mass on the same inputs and compare run to run and to the oracle."""
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2312_02756_b200 as gvx, synth.device as sd, synth, oracle
n = (1 << 20) + 12345
v1, v2 = sd.muon_pairs(n, dtype=torch.float64)
ref = gvx.invariant_mass(v1, v2).cpu()
bad_runs = 0
for r in range(20):
    m = gvx.invariant_mass(v1, v2).cpu()
    d = torch.nonzero(m != ref).flatten()
    if d.numel(): bad_runs += 1; print('run', r, 'differs at', d.numel(), d[:8].tolist())
idx = np.array([7265, 7266, 7272, 100, 200000])
a, b = synth.muon_pairs(idx)
mo, e = oracle.invariant_mass(a, b)
print('oracle', mo, 'gpu', ref[idx].numpy(), 'bad runs', bad_runs)
