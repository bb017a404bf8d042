#!/bin/bash
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_dimuon.jsonl; : > $out
for dt in f64 f32; do for c in 0 1 2 3 4; do
  echo "{\"variant\":\"dimuon$c-$dt\"}" >> $out
  GVX_DIMUON_CFG=$c python bench.py --steps 5 --warmup 3 --extended --no-e2e --no-cpu-baseline --dtype $dt >> $out 2>>gpurun_out/sweep.err
done; done
