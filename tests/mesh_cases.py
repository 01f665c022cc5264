"""Grids for the marching-cubes parity tests (meshing.cpp:168-273), built identically in the
CPU oracle, the compiled reference and the GPU library."""
from __future__ import annotations

import numpy as np


def fibonacci_sphere(c, r, n):
    """test_meshing.cpp:18-30."""
    i = np.arange(n)
    z = 1.0 - 2.0 * (i + 0.5) / n
    rad = np.sqrt(1.0 - z * z)
    th = np.pi * (3.0 - np.sqrt(5.0)) * i
    return np.asarray(c) + r * np.stack([rad * np.cos(th), rad * np.sin(th), z], 1)


def voxel_centres(coords, h, B=8):
    v = np.arange(B ** 3)
    loc = np.stack([v % B, (v // B) % B, v // (B * B)], 1)
    return (coords[:, None, :] * B + loc[None]) * h


def sphere_payload(og, r, h, C=2, holes=0.0, seed=0, B=8, centre=(0.0, 0.0, 0.0)):
    """sphere_grid (test_meshing.cpp:32-40) + optional unobserved voxels, random rgb/logits."""
    og.allocate_points(fibonacci_sphere(np.array(centre), r, 6000), 1)
    cs = og.coords()
    A, V = len(cs), B ** 3
    X = voxel_centres(cs, h, B)
    rng = np.random.default_rng(seed)
    pay = {"sdf": (np.linalg.norm(X - np.array(centre), axis=2) - r).astype(np.float32),
           "weight": (rng.uniform(size=(A, V)) >= holes).astype(np.float32),
           "rgb": rng.uniform(-0.2, 1.2, (A, V, 3)).astype(np.float32),
           "logits": rng.normal(size=(A, V, C)).astype(np.float32)}
    og.set_payload(0, A, **pay)
    return cs, pay


def all_cases_payload(C=2, seed=0):
    """2x2x1 blocks (16x16x8 voxels): the cell anchored at (2i, 2j, 2k) gets case i + 8j + 64k
    (corner c negative iff bit c), magnitudes varied so crossings are not at midpoints."""
    cs = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0]], np.int32)
    sdf = np.zeros((4, 512), np.float32)
    for cfg in range(256):
        i, j, k = cfg % 8, (cfg // 8) % 8, cfg // 64
        for c in range(8):
            vx, vy, vz = 2 * i + (c & 1), 2 * j + ((c >> 1) & 1), 2 * k + (c >> 2)
            b = (vx // 8) + 2 * (vy // 8)
            mag = 0.25 + 0.07 * c + 0.003 * (cfg % 11)
            sdf[b, vx % 8 + 8 * (vy % 8) + 64 * vz] = -mag if (cfg >> c) & 1 else mag
    rng = np.random.default_rng(seed)
    pay = {"sdf": sdf, "weight": np.ones((4, 512), np.float32),
           "rgb": rng.uniform(0, 1, (4, 512, 3)).astype(np.float32),
           "logits": rng.normal(size=(4, 512, C)).astype(np.float32)}
    return cs, pay
