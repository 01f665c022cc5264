#!/usr/bin/env python
"""Regenerate tests/golden/*.npz from the REFERENCE's own code.

Runs only where /root/reference exists: oracle/_ref/libsvr_ref.so is the reference's
grid.cpp / allocation.cpp / camera.cpp / grid_io.cpp / scale_field.cpp compiled verbatim
(oracle/Makefile).  Inputs are drawn from fixed numpy seeds and stored next to the
reference outputs, so the fixtures are self-contained on machines without the reference.
The renderer golden comes from ref_capi.cpp's spec-restated renderer running on the
reference grid API (the reference itself has no renderer: SURVEY.md section 0.2).

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from oracle import RefGrid  # noqa: E402
from fixtures import SyntheticScene, uniform_floats  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"{name}: {os.path.getsize(path) / 1024:.1f} KiB")


def canonical(coords):
    c = np.asarray(coords, np.int64)
    return c[np.lexsort((c[:, 0], c[:, 1], c[:, 2]))].astype(np.int32)


def golden_hash(rng):
    # test_grid.cpp:33 shape at 2e4 coords (duplicates included) + 1000 misses
    coords = rng.integers(-4000, 4001, size=(20000, 3), dtype=np.int32)
    coords[5000:5200] = coords[:200]  # explicit duplicates: insert returns existing value
    g = RefGrid(0.015, 8, 2, capacity=1 << 16)
    idx = g.allocate_blocks(coords)
    far = rng.integers(10000, 20001, size=(1000, 3), dtype=np.int32)
    save("hash.npz", coords=coords, idx=idx, found=g.find(coords), far=far, far_found=g.find(far))


def golden_activation(rng):
    out = {}
    pts = rng.uniform(-0.5, 0.5, size=(500, 3))
    out["points"] = pts
    for R in (0, 1, 2):
        g = RefGrid(0.015, 8, 2)
        rep = g.allocate_points(pts, R)
        out[f"points_R{R}_coords"] = canonical(g.coords())
        out[f"points_R{R}_report"] = np.array([rep.blocks_added, rep.blocks_requested, rep.pixels_used])
    sc = SyntheticScene(room_w=2.4, room_d=2.2, room_h=2.0, n_objects=2, width=40, height=30, n_frames=6)
    cams = sc.cameras()
    depth = sc.depth(cams)
    depth[:, ::7, ::5] = 0.0  # invalid pixels (allocation.cpp:68-69)
    scales = rng.uniform(0.8, 1.25, size=(len(cams), 4, 5))
    out["depth"] = depth
    out["cams"] = np.array([[c.fx, c.fy, c.cx, c.cy, c.width, c.height, *c.R, *c.t] for c in cams])
    out["scales"] = scales
    for R in (0, 1):
        for use_scales in (False, True):
            g = RefGrid(0.04, 8, 2)
            rep = g.allocate_frames(depth, cams, R, scales if use_scales else None)
            key = f"frames_R{R}_s{int(use_scales)}"
            out[key + "_coords"] = canonical(g.coords())
            out[key + "_report"] = np.array([rep.blocks_added, rep.blocks_requested, rep.pixels_used])
    save("activation.npz", **out)


def small_grid(rng, h=0.02, n_pts=4, R=1, C=3, frac_invalid=0.02):
    g = RefGrid(h, 8, C)
    pts = rng.uniform(-0.3, 0.3, size=(n_pts, 3))
    g.allocate_points(pts, R)
    coords = g.coords()
    n = len(coords)
    q = lambda a: (np.round(a * 256) / 256).astype(np.float32)  # noqa: E731  (compressible)
    pay = {"sdf": q(rng.uniform(-1, 1, size=(n, 512))),
           "weight": (rng.uniform(0, 1, size=(n, 512)) > frac_invalid).astype(np.float32),
           "rgb": q(rng.uniform(0, 1, size=(n, 512, 3))),
           "logits": q(rng.uniform(-1, 1, size=(n, 512, C)))}
    g.set_payload(0, n, **pay)
    return g, coords, pay


def golden_query(rng):
    g, coords, pay = small_grid(rng)
    lo, hi = coords.min(0) * 0.16, (coords.max(0) + 1) * 0.16
    x = rng.uniform(lo - 0.05, hi + 0.05, size=(4000, 3))
    q = g.query(x)
    save("query.npz", h=0.02, C=3, coords=coords, x=x, **{f"pay_{k}": v for k, v in pay.items()},
         **{f"q_{k}": v for k, v in q.items()})


def golden_march(rng):
    # test_grid.cpp:298-331 shape: 10 scenes x 100 rays, step 0.008
    out = {}
    for scene in range(10):
        g = RefGrid(0.015, 8, 2)
        pts = rng.uniform(-0.6, 0.6, size=(40, 3))
        g.allocate_points(pts, 1 if scene % 3 == 0 else 0)
        o = rng.uniform(-1.8, 1.8, size=(100, 3))
        d = rng.uniform(-1, 1, size=(100, 3))
        d[::17, 0] = 0.0  # axis-parallel rays exercise the dir == 0 branches
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        m = g.march(o, d, 0.008, 96)
        out[f"s{scene}_coords"] = g.coords()
        out[f"s{scene}_o"], out[f"s{scene}_d"] = o, d
        out[f"s{scene}_counts"] = m["counts"]
        out[f"s{scene}_t"] = m["t"]
        out[f"s{scene}_delta"] = m["delta"]
    save("march.npz", **out)


def golden_render(rng):
    sc = SyntheticScene(room_w=2.4, room_d=2.2, room_h=2.0, n_objects=2, width=48, height=36, n_frames=6)
    cams = sc.cameras()
    depth = sc.depth(cams)
    h = 0.05
    g = RefGrid(h, 8, 4)
    g.allocate_frames(depth, cams, 1)
    coords = g.coords()
    pay = sc.fill_payload(h, coords, 8 * h, 4)
    g.set_payload(0, len(coords), **pay)
    o, d = sc.rays(6, 32, seed=0)
    n = len(o)
    u = uniform_floats(7 * n, 1).reshape(n, 7)
    f = g.render_forward(o, d, h / 2, 64, 2 * h)
    g.render_backward(u[:, :3], u[:, 3], u[:, 4:])
    gs, gr = g.grads()
    keep = np.nonzero(np.abs(gs).sum(1) + np.abs(gr).sum((1, 2)))[0]
    save("render.npz", h=h, coords=coords, o=o, d=d, dC=u[:, :3], dD=u[:, 3], dN=u[:, 4:],
         rgb=f["rgb"], depth=f["depth"], normal=f["normal"], wsum=f["wsum"], n_valid=f["n_valid"],
         grad_blocks=coords[keep], grad_sdf=gs[keep], grad_rgb=gr[keep], scene_room=np.array([2.4, 2.2, 2.0]))


def golden_sdgv(rng):
    g, coords, pay = small_grid(rng, n_pts=4, R=0, C=2)
    path = os.path.join(HERE, "ref_small.sdgv")
    g.save(path)
    print(f"ref_small.sdgv: {os.path.getsize(path) / 1024:.1f} KiB")


def main():
    if not os.path.isdir(oracle.REF_ROOT):
        sys.exit("make_golden.py needs /root/reference (the compiled reference is the source of truth)")
    oracle.build(ref=True)
    rng = np.random.default_rng(20240518)
    golden_hash(rng)
    golden_activation(rng)
    golden_query(rng)
    golden_march(rng)
    golden_render(rng)
    golden_sdgv(rng)


if __name__ == "__main__":
    main()
