"""One device step out of an `ncu --metrics gpu__time_duration.sum --csv --log-file` launch
list: the launches from the k-th `k_ray_keys_dir` (a step starts with the pre-march ray
order) up to the next one.  usage: python profiles/launch_list.py launches.csv [k]"""
import csv
import re
import sys


def main(path, k=4):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        full = r["Kernel Name"].removeprefix("void ")
        if full.startswith("cub::"):
            name = full.split("<")[0]
        else:
            name = re.sub(r"\(.*", "", full).replace("svr_dev::<unnamed>::", "")
        rows.append((name, us))
    starts = [i for i, (n, _) in enumerate(rows) if n.startswith("k_ray_keys_dir")]
    a = starts[k - 1]
    b = starts[k] if len(starts) > k else len(rows)
    step = rows[a:b]
    tot = sum(us for _, us in step)
    for n, us in step:
        print(f"{n[:64]:64s} {us:10.1f} us {100 * us / tot:5.1f}%")
    print(f"{'total':64s} {tot:10.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 4)
