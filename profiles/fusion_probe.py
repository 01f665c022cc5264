"""cfg3 fusion + denoise driver for timing / ncu.
usage: python profiles/fusion_probe.py [reps] [knob=value ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_13220_b200 import SparseDenseGrid  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
knobs = dict(a.split("=") for a in sys.argv[2:])
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
cfg = bench.CFG3
scene = bench.make_scene(cfg)
cams = scene.cameras(cfg["act_frames"])
depth, rgb, sem = scene.frames(cams)
g = SparseDenseGrid(cfg["h"], 8, cfg["C"], device=0)
g.set_stream(stream)
for k, v in knobs.items():
    if k not in ("radius",):
        g.set_tuning(k, int(v))
g.allocate_for_frames(depth, cams, cfg["dilation"])
mu = 8 * cfg["h"] * cfg["dilation"]
dd, dr, ds = (torch.from_numpy(a).to(dev) for a in (depth, rgb, sem))
torch.cuda.synchronize()
r = int(knobs.get("radius", 1))
out = {"blocks": g.block_count(),
       "fuse_all_ms": bench._events_ms(stream, lambda: g.fuse_all(dd, cams, mu, rgb=dr, semantic=ds), reps),
       "denoise_ms": bench._events_ms(stream, lambda: g.denoise(1.0, r), reps)}
print(json.dumps(out))
