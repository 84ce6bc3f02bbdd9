#!/usr/bin/env python
"""DRAM traffic per launch from an ncu capture of tools/prof_once.py (two
rounds; the second is kept), merged into profiles/<round>/ncu_traffic.json
under a workload key ("<workload>" for K0, "<workload>/ISO0" for ISO0):

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep profiles/r02/ncu_traffic.json \
        sv_cavity_256x256_barycentric/ISO0 "<source note>"

Keys: "vanka_patch" = the patch stage of one sweep (sum over its size-class
launches), "vanka_gather", "spmv" (the Store epilogue); also the per-launch
kernel names and durations.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TUNIT = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        def get(k):
            i = hdr.index(k)
            return row[i], units[i]
        name = row[hdr.index("Kernel Name")]
        rd = float(get("dram__bytes_read.sum")[0]) * UNIT.get(get("dram__bytes_read.sum")[1], 1)
        wr = float(get("dram__bytes_write.sum")[0]) * UNIT.get(get("dram__bytes_write.sum")[1], 1)
        t, tu = get("gpu__time_duration.sum")
        res.append((name, rd + wr, float(t) * TUNIT.get(tu, 1e-9)))
    return res


def kind(name):
    if re.search(r"vanka_(patch|subwarp|fixed)_kernel", name):
        return "vanka_patch"
    if "vanka_gather" in name:
        return "vanka_gather"
    if "spmv_kernel" in name:
        return "spmv"
    return None


def main():
    rep, dst, key = sys.argv[1:4]
    note = sys.argv[4] if len(sys.argv) > 4 else ""
    rs = [r for r in rows(rep) if kind(r[0])]
    half = rs[len(rs) // 2:]  # second round
    agg, launches = {}, []
    for name, b, t in half:
        k = kind(name)
        agg[k] = agg.get(k, 0) + int(b)
        launches.append({"kernel": name[:120], "dram_bytes": int(b), "us": t * 1e6})
    d = {"workloads": {}}
    if os.path.exists(dst):
        with open(dst) as f:
            d = json.load(f)
    d.setdefault("workloads", {})[key] = dict(agg, launches=launches, source=note)
    os.makedirs(os.path.dirname(dst) or ".", exist_ok=True)
    with open(dst, "w") as f:
        json.dump(d, f, indent=1, sort_keys=True)
    print(json.dumps(d["workloads"][key], indent=1))


if __name__ == "__main__":
    main()
