#!/bin/bash
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_f32.jsonl; : > $out
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --dtype f32"
for c in 0 1 2 3; do
  echo "{\"variant\":\"f32tma$c\"}" >> $out
  GVX_FORCE_TMA=1 GVX_TMA_CFG32=$c $B >> $out 2>>gpurun_out/sweep.err
done
echo "{\"variant\":\"f32ldg\"}" >> $out
GVX_DISABLE_TMA=1 $B >> $out 2>>gpurun_out/sweep.err
