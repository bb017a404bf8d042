import numpy as np, torch, sys
sys.path.insert(0,'.')
import paper_2312_02756_b200 as gvx, synth
from tests.test_gpu_parity import mixed_inputs
for dt in (np.float64,):
    n, nb = (1<<20)+37, (1<<20)+11
    v1, v2 = mixed_inputs(n, dt, seed=21)
    t1, t2 = torch.from_numpy(v1).cuda(), torch.from_numpy(v2).cuda()
    x, beta = synth.boost_inputs(np.arange(nb), dtype=dt, seed=8)
    tx, tb = torch.from_numpy(x).cuda(), torch.from_numpy(beta).cuda()
    lab, cmb, out = gvx.pair_histograms_boost(t1, t2, tx, tb)
    ref = gvx.boost(tx, tb)
    o, r = out.cpu().numpy(), ref.cpu().numpy()
    bad = ~((o == r) | (np.isnan(o) & np.isnan(r)))
    rows = np.where(bad.any(1))[0]
    print('bad rows', rows.size, 'first', rows[:10], 'tail start', (nb//256)*256)
    if rows.size:
        i = rows[0]; print(o[i], r[i], x[i], beta[i])
        rel = np.abs(o[bad]-r[bad])/np.maximum(np.abs(r[bad]),1e-300); print('max rel', rel.max(), 'median', np.median(rel))
        print('rows mod 256 hist', np.bincount(rows % 256)[:8], 'tile ids', np.unique(rows//256)[:10])
