export GVX_LIB=$PWD/tools/libgvx_tune.so
for dt in f64 f32; do for c in 0 1 2 3 4 5 6 7 8 9; do
  GVX_DIMUON_CFG=$c timeout 120 python -c "
import sys, torch, json
sys.path.insert(0,'.')
import paper_2312_02756_b200 as gvx, synth.device as sd
dt = torch.float64 if '$dt'=='f64' else torch.float32
mu,q,off = sd.jagged_events(0, 100_000_000, dtype=dt)
for _ in range(2): gvx.dimuon_histogram(mu,q,off)
torch.cuda.synchronize()
ev=[(torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)) for _ in range(10)]
for a,b in ev:
    a.record(); gvx.dimuon_histogram(mu,q,off); b.record()
torch.cuda.synchronize()
t=sorted(a.elapsed_time(b) for a,b in ev)
print('$dt cfg $c', round(t[0],4), round(t[5],4))
"
done; done
