#!/usr/bin/env python
"""Summarise `ncu --set full` captures of the hot-path kernels into
profiles/<round>/ncu_summary_<dtype>.md and profiles/ncu_traffic.json.

Usage: python tools/ncu_summary.py <dtype> <report.ncu-rep>[,<report2.ncu-rep>...] <round-dir> [n_events]
(several reports: one capture per gpurun call when a single one would exceed gpurun_out's size cap)

ncu_traffic.json maps dtype -> bench kernel name -> DRAM bytes per launch
(dram__bytes_read.sum + dram__bytes_write.sum) and the algorithmic bytes of the
same launch, which bench.py reports as roofline.traffic.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "DRAM read % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def kernel_key(name: str):
    if "k_boost_inputs" in name or "k_muon_pairs" in name or "k_jagged" in name:
        return None  # the input generator (synth/), not a hot-path kernel
    if "k_step" in name:
        return "step"
    if "k_boost" in name:
        return "boost"
    cm = None
    if "k_pair_tma" in name:
        mode = name.split("k_pair_tma<")[1].split(",")[2].strip()
        return {"0": "invariant_mass", "1": "mass_histogram", "2": "mass_histogram_cm", "3": "cm_costheta_hist",
                "4": "pairs"}[mode]
    if "k_cm_costheta" in name:
        return "cm_costheta_hist"
    if "k_invariant_mass" in name:
        return "invariant_mass"
    if "k_mass_histogram" in name:
        cm = name.split("k_mass_histogram<")[1].split(",")[3].strip()
        return "mass_histogram_cm" if cm in ("1", "true") else "mass_histogram"
    return name[:40]


def main():
    dtype, rep, rdir = sys.argv[1], sys.argv[2], sys.argv[3]
    n = int(float(sys.argv[4])) if len(sys.argv) > 4 else 100_000_000
    es = 8 if dtype == "f64" else 4
    algo = {"invariant_mass": 9 * es, "boost": 11 * es, "mass_histogram": 8 * es, "mass_histogram_cm": 8 * es,
            "cm_costheta_hist": 8 * es, "pairs": 9 * es, "step": 20 * es}
    reps = rep.split(",")
    missing = [r for r in reps if not os.path.exists(r)]
    if missing:
        sys.exit(f"missing report(s): {missing}")  # never overwrite the summary / traffic with nothing
    rows, h = [], None  # rows: (values, units) aligned to the first report's columns
    for rp in reps:
        out = subprocess.run(["ncu", "-i", rp, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rr = list(csv.reader(out.splitlines()))
        if h is None:
            h = rr[0]
        hh, uu = rr[0], dict(zip(rr[0], rr[1]))
        for r in rr[2:]:
            d = dict(zip(hh, r))
            rows.append(([d.get(k, "") for k in h], [uu.get(k, "") for k in h]))
    lines = [f"# ncu --set full summary ({dtype}, N = {n:.0e} events per launch)", "",
             f"Source: `{', '.join(os.path.basename(r) for r in reps)}` (captured on a B200 under gpurun with "
             "`--clock-control none`; per-launch replays are cold-cache and serialised).", "",
             "| kernel | " + " | ".join(lbl for _, lbl in METRICS) + " | algorithmic bytes | DRAM/algorithmic "
             "| DRAM GB/s (bytes / duration) |",
             "|" + "---|" * (len(METRICS) + 4)]
    traffic = {}
    for r, units in rows:
        if len(r) < len(h):
            continue
        name = r[h.index("Kernel Name")]
        key = kernel_key(name)
        if key is None:
            continue
        vals = []
        for m, _ in METRICS:
            if m not in h and m.startswith("gpu__dram_throughput") and "dram__throughput.avg.pct_of_peak_sustained_elapsed" in h:
                m = "dram__throughput.avg.pct_of_peak_sustained_elapsed"  # older ncu name
            if m in h:
                i = h.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("n/a")

        def num(m):
            i = h.index(m)
            v = float(r[i].replace(",", ""))
            u = units[i]
            return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)

        dram = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        ab = algo.get(key, 0) * n
        dur = num("gpu__time_duration.sum") * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3,
                                                "ms": 1e-3, "nsecond": 1e-9}.get(units[h.index("gpu__time_duration.sum")], 1e-9)
        lines.append(f"| `{key}` ({name[:60]}) | " + " | ".join(vals) + f" | {ab:.3e} | {dram / ab if ab else 0:.3f} "
                     f"| {dram / dur / 1e9:.0f} |")
        traffic[key] = {"dram_bytes_per_launch": dram, "algorithmic_bytes_per_launch": ab, "events_per_launch": n,
                        "dram_bytes_per_event": dram / n, "kernel": name[:120]}
    os.makedirs(rdir, exist_ok=True)
    with open(os.path.join(rdir, f"ncu_summary_{dtype}.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    allt = {}
    if os.path.exists(tpath):
        with open(tpath) as f:
            allt = json.load(f)
    allt[dtype] = traffic
    with open(tpath, "w") as f:
        json.dump(allt, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
