#!/usr/bin/env python
"""Break down the host-buffer (e2e) path of one cfg3 step: raw pinned H2D/D2H bandwidth
vs. the C-ABI calls with pinned host arrays (wall clock, synchronised)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_13220_b200 import SparseDenseGrid  # noqa: E402


def wall(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    cfg = dict(bench.CFG3)
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    scene = bench.make_scene(cfg)
    cams, depth = bench.activation_frames(scene, cfg)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    g.set_stream(stream)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    bench.fill_in_chunks(scene, cfg, g.coords(), lambda f, n, p: g.set_payload(f, n, **p))
    arrs = bench.rays_for_rank(scene, cfg, 0, 1)
    hp = [torch.from_numpy(a).pin_memory() for a in arrs]
    dv = [a.to(dev) for a in hp]
    n = hp[0].shape[0]
    S, step, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    outs_h = {k: torch.empty(s, dtype=torch.float32).pin_memory()
              for k, s in (("rgb", (n, 3)), ("depth", (n,)), ("normal", (n, 3)), ("wsum", (n,)))}
    outs_h["n_samples"] = None
    outs_d = {k: v.to(dev) for k, v in outs_h.items() if v is not None}
    outs_d["n_samples"] = None
    h2d = sum(a.numel() * a.element_size() for a in hp)
    d2h = sum(v.numel() * v.element_size() for v in outs_d.values() if v is not None)
    print(f"bytes h2d={h2d / 1e6:.1f} MB d2h={d2h / 1e6:.1f} MB")
    print(f"torch pinned H2D all inputs : {wall(lambda: [a.to(dev, non_blocking=True) for a in hp]):7.2f} ms")
    print(f"torch pinned D2H all outputs: "
          f"{wall(lambda: [outs_h[k].copy_(outs_d[k], non_blocking=True) for k in ('rgb', 'depth', 'normal', 'wsum')]):7.2f} ms")
    print(f"fwd device                  : {wall(lambda: g.render_forward(dv[0], dv[1], step, S, beta, out=outs_d)):7.2f} ms")
    print(f"fwd host in/out             : {wall(lambda: g.render_forward(hp[0], hp[1], step, S, beta, out=outs_h)):7.2f} ms")
    print(f"bwd device                  : {wall(lambda: g.render_backward(dv[2], dv[3], dv[4])):7.2f} ms")
    print(f"bwd host                    : {wall(lambda: g.render_backward(hp[2], hp[3], hp[4])):7.2f} ms")
    print(f"zero_active                 : {wall(lambda: g.grad_zero_active()):7.2f} ms")

    def step_host():
        g.render_forward(hp[0], hp[1], step, S, beta, out=outs_h)
        g.render_backward(hp[2], hp[3], hp[4])
        g.grad_zero_active()

    print(f"e2e step                    : {wall(step_host):7.2f} ms")


if __name__ == "__main__":
    main()
