#!/bin/bash
# Warp-specialised (setmaxnreg) ring variants vs the product configs, tools/libgvx_tune.so:
# GVX_TMA_CFG (f64 pair kernels), GVX_TMA_CFG32 (f32), GVX_STEP_CFG (the one-launch step).
export GVX_LIB=$PWD/tools/libgvx_tune.so
out=gpurun_out/sweep_ws.jsonl; : > $out
run() {  # label, env...
  local label=$1; shift
  env "$@" python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw.tmp 2>>gpurun_out/sweep_ws.err
  python - "$label" >> $out <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/sw.tmp") if l.startswith("{")][-1])
k = d["kernels"]
print(json.dumps({"variant": sys.argv[1], "step_ms": d["ms_per_step"],
                  **{n: round(v["ms"], 4) for n, v in k.items()}}))
PY
  tail -1 $out
}
for c in ${CFGS64:-14 20 21 22 23}; do run f64cfg$c GVX_FORCE_TMA=1 GVX_TMA_CFG=$c; done
for c in ${CFGS32:-1 9 10 11}; do run f32cfg$c GVX_FORCE_TMA=1 GVX_TMA_CFG32=$c; done
for c in ${STEPS:-2 3 4}; do run step$c GVX_STEP_CFG=$c; done
