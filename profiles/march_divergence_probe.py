"""How much of k_march is SIMT divergence?  The cfg3 grid; 1,048,576 distinct bench rays vs
the first 32,768 of them each repeated 32 times (the march's pre-sort puts the copies in one
warp: no divergence at all, same per-ray work on average).  Run under
`ncu --metrics gpu__time_duration.sum -k regex:k_march`; prints nothing itself but the sizes.
usage: python profiles/march_divergence_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_13220_b200 import SparseDenseGrid  # noqa: E402

cfg = dict(bench.CFG3)
dev = torch.device("cuda", 0)
scene = bench.make_scene(cfg)
cams, depth = bench.activation_frames(scene, cfg)
g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
g.allocate_for_frames(depth, cams, cfg["dilation"])
bench.fill_in_chunks(scene, cfg, g.coords(), lambda f, n, p: g.set_payload(f, n, **p))
o, d = (torch.from_numpy(a).to(dev) for a in bench.rays_for_rank(scene, cfg, 0, 1)[:2])
S, step, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
o2 = o[:32768].repeat_interleave(32, dim=0).contiguous()
d2 = d[:32768].repeat_interleave(32, dim=0).contiguous()
for name, (oo, dd) in (("distinct", (o, d)), ("x32", (o2, d2))):
    for _ in range(2):
        out = g.render_forward(oo, dd, step, S, beta)
    torch.cuda.synchronize()
    print(name, oo.shape[0], int(out["n_samples"].sum()), flush=True)
