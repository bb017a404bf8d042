#!/usr/bin/env python
"""Per-event SASS instruction mix and warp-stall breakdown of one kernel in an
`ncu --set full --import-source on` report (its source page, SASS view).

Usage: python tools/ncu_instmix.py <report.ncu-rep> <kernel-name-regex> <events> [top]
Prints markdown: thread instructions per event by opcode (executed warp instructions
x 32 / events), each opcode's share of the warp-state samples, and the stall reasons."""
import collections
import csv
import re
import subprocess
import sys


def main():
    rep, kre, n = sys.argv[1], sys.argv[2], float(sys.argv[3])
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 24
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    # one section per captured launch: a "Kernel Name" row, the header row, the SASS rows;
    # take the first launch whose name matches the regex
    sec = None
    for i, r in enumerate(rows):
        if r and r[0] == "Kernel Name" and len(r) > 1 and re.search(kre, r[1]):
            sec = i
            break
    if sec is None:
        sys.exit(f"no launch matching /{kre}/ in {rep}")
    hdr = rows[sec + 1]
    data = []
    for r in rows[sec + 2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(hdr):
            data.append(r)
    i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
    i_w = hdr.index("Warp Stall Sampling (All Samples)")
    stall_cols = [(h[6:], hdr.index(h)) for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    ex, smp, stalls = collections.Counter(), collections.Counter(), collections.Counter()
    for r in data:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[i_src].strip())
        op = m.group(2) if m else "?"
        ex[op] += int(r[i_ex] or 0)
        smp[op] += int(r[i_w] or 0)
        for name, i in stall_cols:
            stalls[name] += int(r[i] or 0)
    tot, ts, tst = sum(ex.values()), sum(smp.values()) or 1, sum(stalls.values()) or 1
    print(f"kernel /{kre}/ of `{rep.split('/')[-1]}`: {tot * 32 / n:.1f} thread instructions per event "
          f"({n:.0e} events)\n")
    print("| opcode | per event | share of stall samples |\n|---|---|---|")
    for op, c in ex.most_common(top):
        print(f"| {op} | {c * 32 / n:.2f} | {100 * smp[op] / ts:.1f} % |")
    print("\nwarp-state samples: " + ", ".join(f"{k} {100 * v / tst:.1f} %" for k, v in stalls.most_common(10)))


if __name__ == "__main__":
    main()
