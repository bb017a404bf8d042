#!/bin/bash
# Ring-geometry sweep of the fused pair pass (tools/libgvx_tune.so: GVX_TMA_CFG for
# f64, GVX_TMA_CFG32 for f32); one bench line per variant.
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_pairs_cfg.jsonl; : > $out
for c in ${CFGS64:-8 9 13 14 15 16 17}; do
  echo "{\"variant\":\"f64cfg$c\"}" >> $out
  GVX_FORCE_TMA=1 GVX_TMA_CFG=$c python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline >> $out 2>>gpurun_out/sweep.err
done
for c in ${CFGS32:-0 1 2 3 4 6 7 8}; do
  echo "{\"variant\":\"f32cfg$c\"}" >> $out
  GVX_FORCE_TMA=1 GVX_TMA_CFG32=$c python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --dtype f32 >> $out 2>>gpurun_out/sweep.err
done
