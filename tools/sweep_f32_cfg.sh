#!/bin/bash
# f32 TMA-ring geometry sweep (tools/libgvx_tune.so, GVX_TMA_CFG32) over every
# f32 pair kernel incl. the cos theta* mode (bench.py --extended).
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_f32_cfg.jsonl; : > $out
for c in ${CFGS:-0 1 2 3 4 5 6}; do
  echo "{\"variant\":\"f32cfg$c\"}" >> $out
  GVX_FORCE_TMA=1 GVX_TMA_CFG32=$c python bench.py --steps 10 --warmup 3 --extended --no-e2e --no-cpu-baseline --dtype f32 >> $out 2>>gpurun_out/sweep.err
done
