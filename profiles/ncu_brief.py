"""Print the headline ncu metrics of every kernel in a report.
usage: python profiles/ncu_brief.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate", "Executed Ipc Active")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
seen = {}
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in WANT:
        key = (d["ID"], d["Kernel Name"].split("(")[0][-40:])
        seen.setdefault(key, []).append(f"{d['Metric Name']}={d['Metric Value']}{d['Metric Unit']}")
for (i, k), v in seen.items():
    print(i, k)
    print("   ", "; ".join(v))
