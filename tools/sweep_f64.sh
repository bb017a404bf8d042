#!/bin/bash
# A/B sweep of f64 kernel variants from the tuning build (tools/libgvx_tune.so).
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_f64.jsonl; : > $out
for c in 0 1 2 3 4 5; do
  echo "{\"variant\":\"tma$c\"}" >> $out
  GVX_TMA_CFG=$c python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $out 2>>gpurun_out/sweep.err
done
for c in 0 1 2 3 4; do
  echo "{\"variant\":\"ldg$c\"}" >> $out
  GVX_DISABLE_TMA=1 GVX_LDG_CFG=$c python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $out 2>>gpurun_out/sweep.err
done
