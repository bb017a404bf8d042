#!/bin/bash
# One gpurun batch that refreshes the committed measurements of the step:
# bench lines (f64, f32), the ncu launch list of the bench command, and
# ncu --set full captures of every step kernel (summarised by tools/ncu_summary.py).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_f64.jsonl 2> gpurun_out/bench_f64.err
python bench.py --dtype f32 > gpurun_out/bench_f32.jsonl 2> gpurun_out/bench_f32.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_f64.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for dt in f64 f32; do
  ncu --set full --import-source on --clock-control none -k regex:"k_pair_tma|k_boost|k_invariant_mass|k_mass_histogram|k_cm_costheta" \
      -f -o gpurun_out/prof_$dt python tools/prof_step.py --dtype $dt > gpurun_out/prof_$dt.log 2>&1
done
