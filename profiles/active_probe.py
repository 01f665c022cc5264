"""How much gradient a cfg3 step produces: active blocks and nonzero voxels per step (sizes
the multi-GPU all-reduce)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_13220_b200 import SparseDenseGrid  # noqa: E402

cfg = bench.CFG3
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
scene = bench.make_scene(cfg)
cams, depth = bench.activation_frames(scene, cfg)
g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
g.set_stream(stream)
g.allocate_for_frames(depth, cams, cfg["dilation"])
bench.fill_in_chunks(scene, cfg, g.coords(), lambda f, n, p: g.set_payload(f, n, **p))
o, d, dC, dD, dN = bench.rays_for_rank(scene, cfg, 0, 1)
A = g.block_count()
out = {"blocks": A}
for n_rays in (1 << 17, 1 << 18, 1 << 20):
    g.grad_zero()
    g.render_forward(o[:n_rays], d[:n_rays], cfg["h"] / 2, 64, 2 * cfg["h"])
    g.render_backward(dC[:n_rays], dD[:n_rays], dN[:n_rays])
    act = g.active_mask()
    gs, gr = g.grads()
    nz = (gs != 0) | (gr != 0).any(-1)
    na = int(act.sum())
    sub = nz.reshape(A, 4, 2, 4, 2, 4, 2).any(axis=(2, 4, 6)).reshape(A, 64)
    out[n_rays] = {"active_blocks": na, "active_frac": na / A,
                   "nonzero_voxels": int(nz.sum()), "nonzero_frac_of_active_voxels": float(nz.sum() / (na * 512)),
                   "touched_2cubed_subblocks_frac": float(sub[act.astype(bool)].mean()),
                   "allreduce_bytes_dense": na * 512 * 16, "allreduce_bytes_nonzero": int(nz.sum()) * 16}
print(json.dumps(out, indent=1))
