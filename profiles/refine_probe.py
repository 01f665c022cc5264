"""Refinement demo / timing: fuse distorted depth, refine, mesh (profiles/ evidence).
usage: python profiles/refine_probe.py [steps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_13220_b200 import SparseDenseGrid  # noqa: E402
from paper_2305_13220_b200.refine import RefineConfig, Refiner, frames_to_device  # noqa: E402
from fixtures import SyntheticScene  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
sc = SyntheticScene(n_frames=32, width=320, height=240, label_channels=4, n_objects=4, seed=1)
cams = sc.cameras()
depth, rgb, sem, nrm = sc.frames(cams, normals=True)
h = 0.02
g = SparseDenseGrid(h, 8, 4)
g.allocate_for_frames(depth, cams, 2)
rng = np.random.default_rng(0)
scale = 1.0 + 0.08 * np.sin(np.linspace(0, 3, depth.shape[2]))[None, None, :]
bad = (depth * scale * (1 + 0.02 * rng.normal(size=depth.shape))).astype(np.float32)
mu = 8 * h * 2
g.fuse_all(bad, cams, mu, rgb=rgb, semantic=sem)


def surface_err():
    m = g.marching_cubes(0.0)
    v = m["vertices"]
    return {"vertices": len(v), "mean_abs_gt_sdf": float(np.mean(np.abs(sc.sdf(v)))),
            "frac_within_1cm": float(np.mean(np.abs(sc.sdf(v)) < 0.01))}


e0 = surface_err()
r, dp, nm = frames_to_device(rgb, bad, nrm)
ref = Refiner(g, cams, r, dp, nm, step_m=h / 2, beta=2 * h, mu=mu, config=RefineConfig(max_samples=256))
ref.run(3)
torch.cuda.synchronize()
t0 = time.perf_counter()
trace = ref.run(steps, log_every=max(steps // 6, 1))
torch.cuda.synchronize()
dt = time.perf_counter() - t0
e1 = surface_err()
print(json.dumps({"blocks": g.block_count(), "rays_per_step": ref.n, "steps": steps,
                  "ms_per_step_with_logging": dt / steps * 1e3, "init": e0, "refined": e1,
                  "trace": [{k: round(v, 6) if isinstance(v, float) else v for k, v in t.items()} for t in trace]},
                 indent=1))
