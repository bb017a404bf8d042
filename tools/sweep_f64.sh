#!/bin/bash
# A/B sweep of kernel variants from the tuning build (tools/libgvx_tune.so).
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_f64.jsonl; : > $out
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
for c in ${TMA_CFGS:-0 2 6 8}; do
  echo "{\"variant\":\"tma$c\"}" >> $out
  GVX_FORCE_TMA=1 GVX_TMA_CFG=$c $B >> $out 2>>gpurun_out/sweep.err
done
for c in ${LDG_CFGS:-0 2}; do
  echo "{\"variant\":\"ldg$c\"}" >> $out
  GVX_DISABLE_TMA=1 GVX_LDG_CFG=$c $B >> $out 2>>gpurun_out/sweep.err
done
if [ -n "$F32" ]; then
for m in tma ldg; do
  echo "{\"variant\":\"f32_$m\"}" >> $out
  if [ $m = tma ]; then GVX_FORCE_TMA=1 $B --dtype f32 >> $out 2>>gpurun_out/sweep.err;
  else GVX_DISABLE_TMA=1 $B --dtype f32 >> $out 2>>gpurun_out/sweep.err; fi
done
fi
