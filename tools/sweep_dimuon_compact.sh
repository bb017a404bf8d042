#!/bin/bash
# A/B sweep of the stream-compacted dimuon kernel's tile / block / occupancy
# variants (tools/libgvx_tune.so, GVX_DIMUON_CFG; see launch_dimuon_compact).
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_dimuon_compact.jsonl; : > $out
for dt in f64 f32; do for c in ${CFGS:-0 1 2 3 4 5 6}; do
  echo "{\"variant\":\"compact$c-$dt\"}" >> $out
  GVX_DIMUON_CFG=$c python bench.py --steps 5 --warmup 3 --extended --no-e2e --no-cpu-baseline --dtype $dt >> $out 2>>gpurun_out/sweep.err
done; done
