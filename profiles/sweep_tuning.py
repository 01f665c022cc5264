#!/usr/bin/env python
"""Sweep the renderer's performance knobs (svr_grid_set_tuning; results unaffected) on the
cfg3 workload in one process.  Knobs and values come from SWEEP, e.g.
    SWEEP="ray_sort=1,3;bwd_pipe=0,1;pipe_min_blocks=2,3" python profiles/sweep_tuning.py
Prints per-config device times (CUDA events, mean of 4 after 2 warm-up steps) of the
forward call (sort + march + sort + forward) and the backward call."""
import itertools
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2305_13220_b200 import SparseDenseGrid  # noqa: E402


def main():
    spec = os.environ.get("SWEEP", "ray_sort=3")
    knobs = []
    for part in spec.split(";"):
        if part.strip():
            k, vals = part.split("=")
            knobs.append((k.strip(), [int(v) for v in vals.split(",")]))
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
    o, d, dC, dD, dN = (torch.from_numpy(a).to(dev) for a in bench.rays_for_rank(scene, cfg, 0, 1))
    n = o.shape[0]
    outs = {k: torch.empty(s, dtype=torch.float32, device=dev)
            for k, s in (("rgb", (n, 3)), ("depth", (n,)), ("normal", (n, 3)), ("wsum", (n,)))}
    outs["n_samples"] = None
    S, step, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    print(f"blocks={g.block_count()} rays={n}", flush=True)
    first = None
    for combo in itertools.product(*[v for _, v in knobs]):
        for (k, _), v in zip(knobs, combo):
            g.set_tuning(k, v)
        f_ms, b_ms = [], []
        for it in range(2 + int(os.environ.get("ITERS", "4"))):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record(stream)
            g.render_forward(o, d, step, S, beta, out=outs)
            e[1].record(stream)
            g.render_backward(dC, dD, dN)
            e[2].record(stream)
            g.grad_zero_active()
            torch.cuda.synchronize()
            if it >= 2:
                f_ms.append(e[0].elapsed_time(e[1]))
                b_ms.append(e[1].elapsed_time(e[2]))
        tag = " ".join(f"{k}={v}" for (k, _), v in zip(knobs, combo))
        got = torch.cat([outs[k].reshape(n, -1) for k in ("rgb", "depth", "normal", "wsum")], 1).cpu()
        if first is None:
            first = got
        same = "same" if torch.equal(got, first) else f"DIFF max {float((got - first).abs().max()):.3g}"
        print(f"{tag}: fwd {statistics.mean(f_ms):7.3f} ms  bwd {statistics.mean(b_ms):7.3f} ms  "
              f"total {statistics.mean(f_ms) + statistics.mean(b_ms):7.3f}  outputs vs first config: {same}",
              flush=True)


if __name__ == "__main__":
    main()
