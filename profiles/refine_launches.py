"""Launch list of the refinement step (bench.bench_refine's workload): run under
`ncu --metrics gpu__time_duration.sum --csv`, then summarise with
`python profiles/refine_launches.py --summarise <csv>` (mean ms per kernel name per step)."""
import csv
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def summarise(path, steps):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(float)
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        v = float(r[mv].replace(",", ""))
        v = v / 1e6 if r[mu] in ("ns", "nsecond") else (v / 1e3 if r[mu] in ("us", "usecond") else v)
        name = r[kn].replace("<unnamed>", "anon").split("(")[0].split("<")[0].replace("void ", "")
        name = name.split("::")[-1] if not name.startswith("cub") else name
        tot[name] += v
    total = sum(tot.values())
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:50s} {v / steps:8.3f} ms/step  {100 * v / total:5.1f} %")
    print(f"{'total':50s} {total / steps:8.3f} ms/step")


if __name__ == "__main__":
    if sys.argv[1:2] == ["--summarise"]:
        summarise(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 5)
    else:
        import torch

        import bench

        dev = torch.device("cuda", 0)
        s = torch.cuda.Stream(dev)
        torch.cuda.set_stream(s)
        print(bench.bench_refine(dev, s, steps=5))
