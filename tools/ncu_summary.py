#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) into the numbers the roofline
uses: duration, DRAM bytes, DRAM throughput, occupancy, stall reasons.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [algorithmic_bytes] > profiles/...txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 sector hit rate"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard / issue"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait / issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio_throttle / issue"),
    ("smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio", "stall lg_throttle / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "stall math_pipe / issue"),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "stall sleeping / issue"),
    # where the L2 traffic and its DRAM fills come from
    ("lts__t_sectors_op_read.sum", "L2 sectors read"),
    ("lts__t_sectors_op_write.sum", "L2 sectors written"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 sectors read by SMs"),
    ("lts__t_sectors_srcunit_tex_op_write.sum", "L2 sectors written by SMs"),
    ("lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "L2 read misses (SM reads)"),
    ("lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum", "L2 write misses (SM writes)"),
    ("lts__t_sectors_srcunit_tex_lookup_miss.sum", "L2 misses (SM)"),
    ("lts__t_sectors_srcnode_gpc_op_read_lookup_miss.sum", "L2 read misses (GPC)"),
    ("lts__t_sectors_srcunit_ltcfabric.sum", "L2 sectors over the die fabric"),
    ("dram__sectors_read.sum", "dram sectors read"),
    ("dram__sectors_write.sum", "dram sectors written"),
    ("l1tex__m_xbar2l1tex_read_sectors.sum", "L2 -> L1 sectors"),
    ("smsp__inst_executed_op_shared_ld.sum", "shared loads"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots %"),
]


def to_bytes(val, unit):
    m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    return float(val) * m.get(unit, 1)


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        vals = {}
        for key, label in KEYS:
            if key in hdr:
                i = hdr.index(key)
                vals[key] = (r[i], units[i])
                print(f"  {label:34s} {r[i]} {units[i]}")
        if "dram__bytes_read.sum" in vals and "gpu__time_duration.sum" in vals:
            rd = to_bytes(*vals["dram__bytes_read.sum"])
            wr = to_bytes(*vals["dram__bytes_write.sum"])
            t = float(vals["gpu__time_duration.sum"][0])
            tu = vals["gpu__time_duration.sum"][1]
            ts = t * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(tu, 1e-9)
            print(f"  {'dram traffic (read+write)':34s} {(rd + wr) / 1e6:.1f} MB  -> {(rd + wr) / ts / 1e9:.0f} GB/s")
            if alg:
                print(f"  {'algorithmic bytes':34s} {alg / 1e6:.1f} MB  (traffic/alg = {(rd + wr) / alg:.3f})")


if __name__ == "__main__":
    main()
