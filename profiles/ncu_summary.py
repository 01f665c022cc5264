#!/usr/bin/env python
"""Summarise an `ncu --set full` report: per kernel duration, DRAM/L2 traffic, occupancy
and the top warp-stall reasons.  Usage: python profiles/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thru %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM thru %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM thru %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__occupancy_limit_registers", "CTA limit (regs)"),
    ("smsp__inst_executed.sum", "warp instrs"),
    ("lts__t_requests_srcunit_tex_op_red.sum", "L2 red requests"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sectors"),
]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    for d in data:
        name = d[idx["Kernel Name"]].split("(")[0].split("::")[-1]
        print(f"== {name}")
        for key, label in KEYS:
            if key in idx:
                print(f"   {label:18s} {d[idx[key]]:>16s} {units[idx[key]]}")
        stalls = []
        for h, i in idx.items():
            if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith(".ratio"):
                try:
                    stalls.append((float(d[i]), h[len("smsp__average_warp_latency_issue_stalled_"):-6]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        if stalls:
            print("   stalls (cycles/issued instr): " +
                  ", ".join(f"{n}={v:.1f}" for v, n in stalls[:6]))


if __name__ == "__main__":
    main(sys.argv[1])
