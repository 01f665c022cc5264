"""The BASELINE.json workloads as input recipes, shared by bench.py and the
full-size parity tests.  Every input is generated on the host by a scene generator with the
SyntheticScene interface: ``fixtures.SyntheticScene`` (the restatement, our arm) or
``oracle.RefScene`` (the reference's own synthetic.cpp, the reference arm) -- the two are
equal bit for bit (tests/test_synthetic.py).
"""
from __future__ import annotations

import numpy as np

# cfg3 (BASELINE.json configs[2]): ScanNet-scale synthetic room 11 x 11 x 3 m, 1 cm voxels,
# 8^3 blocks activated with L-inf dilation R = 2 from the GT depth of 64 ring cameras;
# 1M rays per GPU per step = 64 poses x 16384 random pixels, <= 64 samples at h/2, beta = 2h
CFG3 = dict(room=(11.0, 11.0, 3.0), h=0.01, dilation=2, C=4, width=640, height=480,
            n_objects=4, seed=1, fov=70.0, act_frames=64, ray_poses=64, rays_per_pose=16384,
            max_samples=64, name="cfg3")
# cfg5 (configs[4]): the cfg3 grid, 8M rays per step in total split over the ranks (strong)
CFG5 = dict(CFG3, rays_per_pose=131072, strong=True, name="cfg5")
# cfg1 / cfg2 (configs[0] / [1]): 5 x 5 x 3 m room, 2 cm voxels, R = 2 from 24 ring frames
CFG1 = dict(CFG3, room=(5.0, 5.0, 3.0), h=0.02, act_frames=24, ray_poses=24, name="cfg1")
# cfg4 (configs[3]): the cfg3 geometry, activation from 300 ring frames, then a query sweep
CFG4 = dict(CFG3, act_frames=300, ray_poses=300, name="cfg4")

WORKLOADS = {
    "cfg3": ("cfg3: ScanNet-scale synthetic room 11x11x3 m, 1 cm voxels, 8^3 blocks, R=2 activation from 64 "
             "ring-camera GT depth frames, 1M rays/GPU/step (64 poses x 16384 px), <=64 samples/ray, fwd+bwd"),
    "cfg5": ("cfg5: the cfg3 grid (11x11x3 m, 1 cm voxels, R=2 from 64 GT depth frames), 8M rays/step in total "
             "(64 poses x 131072 px) split contiguously over the GPUs, <=64 samples/ray, fwd+bwd"),
}


def scene_spec(cfg) -> dict:
    r = cfg["room"]
    return dict(room_w=r[0], room_d=r[1], room_h=r[2], n_objects=cfg["n_objects"], width=cfg["width"],
                height=cfg["height"], n_frames=cfg["ray_poses"], fov_deg=cfg["fov"], label_channels=cfg["C"],
                seed=cfg["seed"])


def make_scene(cfg, reference: bool = False):
    """The restated fixture generator, or the reference's own (oracle/_ref) when reference."""
    if reference:
        from oracle import RefScene

        return RefScene(**scene_spec(cfg))
    from fixtures import SyntheticScene

    return SyntheticScene(**scene_spec(cfg))


def uniform(scene, n: int, seed: int) -> np.ndarray:
    """U(-1, 1) floats from mt19937_64(seed) with the scene's own generator library."""
    f = getattr(scene, "uniform_floats", None)
    if f is not None:
        return f(n, seed)
    from fixtures import uniform_floats

    return uniform_floats(n, seed)


def activation_frames(scene, cfg):
    cams = scene.cameras(cfg["act_frames"])
    return cams, scene.depth(cams)


def rays_for_rank(scene, cfg, rank: int, world: int):
    """(o, d, dC, dD, dN) of rank's contiguous shard.  Weak scaling: the global ray set is
    world x (poses x rays_per_pose); strong (cfg5): poses x rays_per_pose whatever the world."""
    poses, rpp = cfg["ray_poses"], cfg["rays_per_pose"]
    if cfg.get("strong"):
        if (poses * rpp) % world:
            raise SystemExit(f"{poses * rpp} rays do not split evenly over {world} ranks")
        o, d = scene.rays(poses, rpp, seed=0)
        n = poses * rpp // world
    else:
        o, d = scene.rays(poses * world, rpp, seed=0)
        n = poses * rpp
    u = uniform(scene, 7 * n * world, 1).reshape(n * world, 7)[rank * n:(rank + 1) * n]
    o, d = o[rank * n:(rank + 1) * n], d[rank * n:(rank + 1) * n]
    c = np.ascontiguousarray
    return c(o), c(d), c(u[:, :3]), c(u[:, 3]), c(u[:, 4:])


def fill_in_chunks(scene, cfg, coords, sink, chunk=8192):
    """Synthetic payload (sdf clamped at mu = L*R, weight 1, rgb, one-hot logits)."""
    h, R = cfg["h"], cfg["dilation"]
    mu = 8 * h * R  # PAPER.md:502, mu = L * R
    for f in range(0, len(coords), chunk):
        c = coords[f:f + chunk]
        sink(f, len(c), scene.fill_payload(h, c, mu, cfg["C"]))
