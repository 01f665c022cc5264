#!/usr/bin/env python
"""How many gradient reductions would the backward issue under different merge schemes?

On a sample of the cfg3 bench rays (oracle march on the CPU, the GPU's post-march ray order
does not matter here: merging is per ray), for every valid sample and every corner parity p
(the parity-p voxel of the sample's cell, the key k_backward_pipe merges on):
  * updates   -- 8 per valid sample (no merging),
  * lane      -- a lane's two samples merged when they share the voxel (no hand-off),
  * handoff   -- the shipped scheme: plus a lane's first run handed to the previous lane when it
                 continues that lane's last run (one step),
  * runs      -- one reduction per maximal run of equal keys along the ray (a full segmented
                 reduction over the warp).
usage: python profiles/merge_probe.py [rays]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(nrays=16384):
    from fixtures.workloads import CFG3, activation_frames, fill_in_chunks, make_scene, rays_for_rank
    from oracle import OracleGrid

    cfg = CFG3
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    og = OracleGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    og.allocate_frames(depth, cams, cfg["dilation"])
    o, d = rays_for_rank(scene, cfg, 0, 1)[:2]
    idx = np.linspace(0, len(o) - 1, nrays).astype(np.int64)
    o, d = o[idx], d[idx]
    h, S = cfg["h"], cfg["max_samples"]
    m = og.march(o, d, h / 2, S)
    cnt, t = m["counts"], m["t"]
    k = np.arange(S)[None, :]
    valid = k < cnt[:, None]
    x = o[:, None, :] + t[:, :, None] * d[:, None, :]
    base = np.floor(x * (1.0 / h)).astype(np.int64)
    tot = {"updates": 0, "lane": 0, "handoff": 0, "runs": 0}
    hist = {}
    for p in range(8):
        pb = np.array([(p >> a) & 1 for a in range(3)])
        vox = base + ((base & 1) != pb[None, None, :])
        key = (vox[..., 0] + (1 << 20)) | ((vox[..., 1] + (1 << 20)) << 21) | ((vox[..., 2] + (1 << 20)) << 42)
        key = np.where(valid, key, -1)
        tot["updates"] += int(valid.sum())
        # maximal runs of equal valid keys along each ray
        newrun = valid & np.concatenate([np.ones((len(key), 1), bool), key[:, 1:] != key[:, :-1]], axis=1)
        tot["runs"] += int(newrun.sum())
        # lane pairs (2l, 2l+1)
        k0, k1 = key[:, 0::2], key[:, 1::2]
        v0, v1 = valid[:, 0::2], valid[:, 1::2]
        two = v0 & v1 & (k0 != k1)
        lane = two.astype(np.int64) + (v0 | v1)
        tot["lane"] += int(lane.sum())
        first = np.where(v0, k0, k1)
        last = np.where(v1, k1, k0)
        prev_last = np.concatenate([np.full((len(key), 1), -2), last[:, :-1]], axis=1)
        give = (first != -1) & (first == prev_last)
        recv = np.concatenate([give[:, 1:], np.zeros((len(key), 1), bool)], axis=1)
        # a lane that gives its first run away saves one reduction (the receiver folds it in),
        # except a single-run lane that also receives: it still reduces the next lane's run
        tot["handoff"] += int(lane.sum() - give.sum() + (~two & give & recv).sum())
        # pass-through lanes (one run, continued from the previous lane and into the next) per
        # chain: a forwarding depth of 1 (pass-throughs hand on what they received) saves the
        # reductions of chains with at most one pass-through, and so on
        pt = ~two & give & recv
        # length of consecutive pass-through stretches
        run_len = np.zeros(pt.shape, np.int64)
        for j in range(pt.shape[1]):
            run_len[:, j] = np.where(pt[:, j], (run_len[:, j - 1] if j else 0) + 1, 0)
        ends = pt & ~np.concatenate([pt[:, 1:], np.zeros((len(pt), 1), bool)], axis=1)
        lens = run_len[ends]
        for L in range(1, 5):
            hist[min(L, 4)] = hist.get(min(L, 4), 0) + int((lens == L).sum() if L < 4 else (lens >= 4).sum())
    n = tot["updates"]
    print(f"{nrays} rays, {int(valid.sum())} valid-slot samples (march slots; the renderer also drops "
          f"samples whose corners are missing)")
    for kx, v in tot.items():
        print(f"  {kx:8s} {v:12d}  {v / n * 8:6.3f} per sample  ({v / n:.3f} of updates)")
    print("  chains by pass-through lanes (1, 2, 3, >= 4):", [hist.get(L, 0) for L in range(1, 5)])


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 16384)
