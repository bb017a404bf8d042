import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2312_02756_b200 as gvx, synth.device as sd
from paper_2312_02756_b200 import hostpipe
n = (1 << 20) + 12345
for tdt in (torch.float64, torch.float32):
    v1, v2 = sd.muon_pairs(n, dtype=tdt)
    bv, bb = sd.boost_inputs(n, dtype=tdt)
    m = gvx.invariant_mass(v1, v2); bo = gvx.boost(bv, bb)
    h = gvx.mass_histogram(v1, v2); hc = gvx.mass_histogram(v1, v2, cm=True)
    hs = [t.cpu().pin_memory() for t in (v1, v2, bv, bb)]
    pipe = hostpipe.HostPipeline(n, tdt, "cuda", chunk=1 << 18)
    hm, hbo, hbins = pipe.step(*hs)
    torch.cuda.synchronize()
    for name, a, b in (("m", hm, m.cpu()), ("bo", hbo, bo.cpu()), ("h", hbins[0], h.cpu()), ("hc", hbins[1], hc.cpu())):
        d = (a != b) if a.dtype.is_floating_point is False else ~((a == b) | (torch.isnan(a) & torch.isnan(b)))
        idx = torch.nonzero(d.reshape(d.shape[0], -1).any(1)).flatten()
        print(tdt, name, 'mismatches', idx.numel(), idx[:10].tolist(), (a.reshape(a.shape[0],-1)[idx[:3]] if idx.numel() else ''), (b.reshape(b.shape[0],-1)[idx[:3]] if idx.numel() else ''))
