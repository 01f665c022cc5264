"""Shared fixtures: identical grids/rays for the GPU library and the CPU oracle.

Grids are activated by the ORACLE (ascending packed-key order), then replayed into the
GPU grid with allocate_blocks in the same order, so block indices agree and gradient
planes can be compared element-wise.  Payloads come from the synthetic scene
(paper_2305_13220_b200.synthetic, restating proj/src/core/synthetic.cpp:42-192).
"""
from __future__ import annotations

import functools

import numpy as np

from oracle import OracleGrid
from fixtures import SyntheticScene, uniform_floats

# render tolerance: |gpu - oracle| <= RTOL*|oracle| + ATOL_FRAC*max|oracle|
RTOL = 1e-4
ATOL_FRAC = 1e-6


def assert_close(gpu, ref, rtol=RTOL, atol_frac=ATOL_FRAC, what=""):
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    assert gpu.shape == ref.shape, (what, gpu.shape, ref.shape)
    scale = float(np.abs(ref).max()) if ref.size else 0.0
    err = np.abs(gpu - ref)
    bound = rtol * np.abs(ref) + atol_frac * scale
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(f"{what}: {int(bad.sum())}/{bad.size} outside tolerance; worst at {i}: "
                             f"gpu={gpu[i]!r} ref={ref[i]!r} err={err[i]:.3e} bound={bound[i]:.3e}")


@functools.lru_cache(maxsize=8)
def scene_case(room=(2.4, 2.2, 2.0), h=0.04, dilation=1, n_frames=8, width=64, height=48,
               C=4, n_objects=2, n_poses=8, rays_per_pose=64, seed=0):
    """Small synthetic scene: oracle grid + payload + rays + upstream grads."""
    sc = SyntheticScene(room_w=room[0], room_d=room[1], room_h=room[2], n_objects=n_objects,
                        width=width, height=height, n_frames=n_frames, label_channels=C)
    cams = sc.cameras()
    depth = sc.depth(cams)
    og = OracleGrid(h, 8, C)
    og.allocate_frames(depth, cams, dilation)
    coords = og.coords()
    pay = sc.fill_payload(h, coords, 8 * h * dilation if dilation else 8 * h, C)
    og.set_payload(0, len(coords), **pay)
    o, d = sc.rays(n_poses, rays_per_pose, seed=seed)
    n = len(o)
    u = uniform_floats(7 * n, 1).reshape(n, 7)
    return {"scene": sc, "cams": cams, "depth": depth, "oracle": og, "coords": coords, "pay": pay,
            "o": o, "d": d, "dC": np.ascontiguousarray(u[:, :3]), "dD": np.ascontiguousarray(u[:, 3]),
            "dN": np.ascontiguousarray(u[:, 4:]), "h": h, "C": C, "step": h / 2, "beta": 2 * h}


def gpu_grid_from(case, lookup=None):
    """Replay the oracle's blocks (same order => same indices) into a GPU grid."""
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(case["h"], 8, case["C"])
    idx = g.allocate_blocks(case["coords"])
    assert np.array_equal(idx, np.arange(len(case["coords"]), dtype=np.uint32))
    g.set_payload(0, len(case["coords"]), **case["pay"])
    if lookup is not None:
        g.set_lookup(lookup)
    # the test batches are small: keep the production (sorted) ordering path under test
    g.set_tuning("sort_min_rays", 0)
    return g
