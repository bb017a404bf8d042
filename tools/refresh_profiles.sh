#!/bin/bash
# Refresh the committed measurements of the step in gpurun batches (each call's
# gpurun_out must stay under 64 MiB, so the ncu captures go one per call):
#   bash tools/refresh_profiles.sh bench     # bench lines, launch list, widened rows, CFG2 sweep
#   bash tools/refresh_profiles.sh ncu f64   # ncu --set full of every step kernel (then tools/ncu_summary.py)
#   bash tools/refresh_profiles.sh ncu f32
#   bash tools/refresh_profiles.sh ncu f64 "k_step|k_boost" a   # a subset per call (report suffix a) when one
#   bash tools/refresh_profiles.sh ncu f64 "k_pair_tma" b       # report would exceed gpurun_out's 64 MiB cap
set -x
mkdir -p gpurun_out
if [ "$1" = bench ]; then
  python bench.py > gpurun_out/bench_f64.jsonl 2> gpurun_out/bench_f64.err
  python bench.py --dtype f32 > gpurun_out/bench_f32.jsonl 2> gpurun_out/bench_f32.err
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_f64.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  python bench.py --extended --no-e2e --no-cpu-baseline > gpurun_out/bench_extended_f64.jsonl 2>> gpurun_out/refresh.err
  python bench.py --extended --dtype f32 --no-e2e --no-cpu-baseline > gpurun_out/bench_extended_f32.jsonl 2>> gpurun_out/refresh.err
  python bench.py --sweep --sweep-out gpurun_out/nsweep_cfg2.jsonl > gpurun_out/sweep.log 2>> gpurun_out/refresh.err
elif [ "$1" = ncu ]; then
  dt=${2:-f64}
  kre=${3:-"k_step|k_pair_tma|k_boost|k_invariant_mass|k_mass_histogram|k_cm_costheta"}
  ncu --set full --import-source on --clock-control none -k regex:"$kre" \
      -f -o gpurun_out/prof_$dt$4 python tools/prof_step.py --dtype $dt > gpurun_out/prof_$dt$4.log 2>&1
fi
