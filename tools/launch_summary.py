#!/usr/bin/env python
"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`):
per kernel the launch count, total and mean device time, and each kernel's
share of the bench step (the kernels launched inside the timed loop: Vanka
patch + gather + SpMV). ncu times are cold-cache and serialised: compare
shares, not absolutes.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/<round>/launches_summary.txt
"""
import csv
import re
import sys
from collections import OrderedDict

STEP = ("vanka_patch_kernel", "vanka_gather_kernel", "vanka_gather_seq_kernel", "spmv_kernel")


def short(name):
    name = re.sub(r"\(.*\)$", "", name.replace("sag::", ""))
    return name.replace("void ", "")


def main():
    rows = []
    with open(sys.argv[1]) as fh:
        lines = [l for l in fh if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "gpu__time_duration.sum":
            rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) / 1e3))
    agg = OrderedDict()
    for k, t in rows:
        c, s = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, s + t)
    print(f"{len(rows)} launches")
    print(f"{'kernel':60s} {'count':>6s} {'total_us':>10s} {'mean_us':>9s}")
    for k, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:60s} {c:6d} {s:10.1f} {s / c:9.1f}")
    step = {k: v for k, v in agg.items() if k.startswith(STEP)}
    tot = sum(s / c for c, s in step.values())
    print("\nshare of one bench step (mean launch time per kernel):")
    for k, (c, s) in step.items():
        print(f"  {k:58s} {s / c:9.1f} us  {100 * (s / c) / tot:5.1f} %")


if __name__ == "__main__":
    main()
