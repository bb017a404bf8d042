#!/bin/bash
# f32 ring configs and the f32 one-launch step after the FindBin fix (tuning build)
export GVX_LIB=$PWD/tools/libgvx_tune.so
mkdir -p gpurun_out; out=gpurun_out/sweep_f32_s3.jsonl; : > $out
run() {
  local label=$1; shift
  local extra=""
  if [ "${@: -1}" = "--one-launch" ]; then extra="--one-launch"; set -- "${@:1:$(($#-1))}"; fi
  env "$@" python bench.py $extra --dtype f32 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/sw.tmp 2>>gpurun_out/sweep32.err
  python - "$label" >> $out <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/sw.tmp") if l.startswith("{")][-1])
k = d["kernels"]
k.setdefault("pairs", {"ms": 0.0}); k.setdefault("boost", {"ms": 0.0})
print(json.dumps({"variant": sys.argv[1], "step_ms": round(d["ms_per_step"], 4), "pairs": round(k["pairs"]["ms"], 4), "boost": round(k["boost"]["ms"], 4), "pairs_f32": round(k["pairs_f32"]["ms"], 4)}))
PY
}
run default
for c in ${CFGS32:-1 2 3 4 6 7 8 9 10 11}; do run f32cfg$c GVX_FORCE_TMA=1 GVX_TMA_CFG32=$c; done
run onelaunch_default --one-launch
for c in 1 2 3 4; do run step32cfg$c GVX_STEP32_CFG=$c --one-launch; done
run default_again
