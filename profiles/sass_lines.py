#!/usr/bin/env python
"""Per-source-line instruction counts and stall samples of one kernel.

Joins an ncu SASS source page (`ncu -i rep --page source --csv --print-source sass
--kernel-name regex:K > k.csv`) with `nvdisasm --print-line-info` of the same build's cubin
(extracted from libsvr_b200.so with `cuobjdump -xelf all`), matching instructions by their
offset from the function start.  usage:
  python profiles/sass_lines.py k.csv svr_render.sm_100a.cubin <mangled-name-regex> [top]
"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, fn_re):
    out = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True,
                         check=True).stdout
    rx = re.compile(fn_re)
    m, cur, inside = {}, "?", False
    for ln in out.splitlines():
        if ln.startswith("//----") and ".text." in ln:
            inside = bool(rx.search(ln))
            continue
        if not inside:
            continue
        s = ln.strip()
        if s.startswith("//## File"):
            f = re.search(r'"([^"]+)", line (\d+)', s)
            cur = f"{f.group(1).split('/')[-1]}:{f.group(2)}"
        else:
            a = re.match(r"/\*([0-9a-f]{4,})\*/", s)
            if a:
                m[int(a.group(1), 16)] = cur
    return m


def main(csv_path, cubin, fn_re, top=40):
    lm = line_map(cubin, fn_re)
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    base = None
    inst, samp, ninst = collections.Counter(), collections.Counter(), 0
    tot_i = tot_s = 0
    for r in rows[2:]:
        try:
            addr = int(r[ix["Address"]], 16)
            n = int(r[ix["Instructions Executed"]])
            s = int(r[ix["Warp Stall Sampling (All Samples)"]])
        except (ValueError, IndexError):
            continue
        base = addr if base is None else base
        key = lm.get(addr - base, "?")
        inst[key] += n
        samp[key] += s
        tot_i += n
        tot_s += s
        ninst += 1
    print(f"{ninst} SASS instructions, {tot_i / 1e6:.1f}M executed, {tot_s} stall samples; "
          f"{len(lm)} mapped offsets")
    keys = sorted(set(inst) | set(samp), key=lambda k: -(inst[k] / max(tot_i, 1) + samp[k] / max(tot_s, 1)))
    for k in keys[:top]:
        print(f"{k:28s} inst {100 * inst[k] / tot_i:5.1f}%  stall {100 * samp[k] / tot_s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 40)
