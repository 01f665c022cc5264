#!/usr/bin/env python
"""Record the per-launch DRAM traffic and L2 hit rate of the step's kernels from one
`ncu --set full` capture into profiles/ncu_traffic.json, keyed by workload, per-GPU ray
count and the build id of the kernel sources (bench.build_id) -- bench.py reports
`roofline.traffic` / `dram_frac` / `l2_hit_pct` only for a capture of the build it runs.

usage: python profiles/ncu_traffic_update.py <report.ncu-rep> <workload> <rays_per_gpu> [summary-file]
The capture must be of the current sources (run on the GPU box right after building them).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
KERNELS = ("k_march", "k_forward", "k_backward_pipe")


def main(rep, workload, rays, summary=None):
    from bench import build_id

    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, data = rows[0], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def val(d, k):
        v = float(d[ix[k]].replace(",", ""))
        unit = rows[1][ix[k]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)

    entry = {"workload": workload, "rays_per_gpu": int(rays), "build_id": build_id(), "report": os.path.basename(rep),
             "file": summary, "dram_bytes": {}, "l2_hit_pct": {}, "duration_ms": {}, "instances": {}}
    for d in data:
        full = d[ix["Kernel Name"]]
        name = full.split("(")[0].split("::")[-1].split("<")[0].strip()
        name = name.replace("void ", "")
        if name not in KERNELS or name in entry["dram_bytes"]:
            continue
        entry["dram_bytes"][name] = int(val(d, "dram__bytes_read.sum") + val(d, "dram__bytes_write.sum"))
        entry["l2_hit_pct"][name] = float(d[ix["lts__t_sector_hit_rate.pct"]])
        entry["duration_ms"][name] = val(d, "gpu__time_duration.sum") / 1e6 if rows[1][ix["gpu__time_duration.sum"]] == "ns" \
            else float(d[ix["gpu__time_duration.sum"]])
        entry["instances"][name] = full[:160]
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    doc = json.load(open(path)) if os.path.exists(path) else {"captures": []}
    doc["source"] = ("ncu --set full captures: dram__bytes_read.sum + dram__bytes_write.sum per launch "
                     "(bench.py roofline.traffic) and lts__t_sector_hit_rate.pct, per workload, rays per GPU "
                     "and kernel-source build id")
    doc["captures"] = [e for e in doc["captures"]
                       if not (e.get("workload") == workload and e.get("rays_per_gpu") == int(rays))] + [entry]
    with open(path, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:4], sys.argv[4] if len(sys.argv) > 4 else None)
