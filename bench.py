#!/usr/bin/env python
"""Benchmark: differentiable SDF volume rendering over the sparse-dense block grid.

Workload (BASELINE.json configs[2], "cfg3"): ScanNet-scale synthetic room 11 x 11 x 3 m,
1 cm voxels, 8^3 blocks activated with L-inf dilation R=2 from the GT depth of the ring
cameras, 1M rays per GPU per step (64 poses x 16384 random pixels), <= 64 samples per
ray at step h/2, Laplace beta = 2h.  One step = render_forward (march + fused forward)
+ render_backward (fused adjoint + vector-atomic scatter) + active-block gradient
reduction (N > 1) + zeroing of the active gradients.

`--workload cfg5` (BASELINE.json configs[4]): the same grid, 8M rays per step in total split
over the GPUs (strong scaling).

`--impl reference`: the reference's CPU path on the host cores -- its own grid code and
synthetic generator compiled verbatim (oracle/_ref) with the spec renderer on its API -- for
the same workload, config and metric; rank 0 only.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg3|cfg5]
With --gpus N > 1 outside torchrun the script re-launches itself under torch.distributed.run
(one rank per GPU); rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import ctypes
import hashlib
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from fixtures.workloads import (CFG1, CFG3, CFG4, CFG5, WORKLOADS, activation_frames,  # noqa: E402
                                fill_in_chunks, make_scene, rays_for_rank)

METRIC = "rays/s and samples/s fwd+bwd per GPU (1/2/4/8 B200); % HBM roofline vs CPU"
# algorithmic bytes per VALID interpolated sample / per ray
FWD_B_SAMPLE, FWD_B_RAY = 182.8, 80.0
BWD_B_SAMPLE, BWD_B_RAY = 256.0, 28.0
STEP_B_SAMPLE, STEP_B_RAY = FWD_B_SAMPLE + BWD_B_SAMPLE, FWD_B_RAY + BWD_B_RAY
# SURVEY.md 8(d) "cfg4 bytes": activation 4 B per pixel read + per new block a 16 B slot, a 12 B
# coordinate and the zero-initialised payload 512 (20 + 4 C) B; query 127 B per point
ACT_B_PIXEL = 4.0
QUERY_B_POINT = 8 * (4 + 4) + 22.8 + 24 + 16


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


STEP_KERNELS = ("k_march", "k_forward", "k_backward_pipe")


def build_id(so_path=None) -> str:
    """Hash of the SASS of the step's kernels in the built library (cuobjdump): ncu captures are
    tied to the machine code they profiled, host-code or comment edits do not orphan them.
    Falls back to the kernel sources without comments when cuobjdump is unavailable."""
    so = so_path or os.path.join(ROOT, "paper_2305_13220_b200", "libsvr_b200.so")
    try:
        out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, timeout=120,
                             check=True).stdout
        h = hashlib.sha256()
        keep = False
        for line in out.splitlines():
            if "Function :" in line:  # the mangled name embeds a build-path hash: not hashed
                name = line.split("Function :")[1].strip()
                keep = any(f"{len(k)}{k}" in name and ("EN" in name.split(k, 1)[1][:2]) for k in STEP_KERNELS)
                if keep:
                    h.update(next(k for k in STEP_KERNELS if f"{len(k)}{k}" in name).encode())
                continue
            if keep:
                h.update(line.strip().encode())
        return "sass-" + h.hexdigest()[:16]
    except Exception:
        pass
    import re

    h = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2305_13220_b200", "csrc")
    for f in sorted(os.listdir(csrc)):
        if f.endswith((".cu", ".cuh", ".h")):
            with open(os.path.join(csrc, f), encoding="utf-8") as fh:
                src = fh.read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            src = re.sub(r"//[^\n]*", "", src)
            h.update(f.encode() + " ".join(src.split()).encode())
    return h.hexdigest()[:16]


def traffic_from_profiles(workload, rays_per_gpu, bid, path=None):
    """Per-launch DRAM bytes (ncu dram__bytes_read.sum + dram__bytes_write.sum) and L2 hit
    rates captured for this workload, per-GPU ray count AND this build; else {}."""
    try:
        with open(path or os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            entries = json.load(f)["captures"]
    except Exception:
        return {}
    for e in entries:
        if e.get("workload") == workload and e.get("rays_per_gpu") == rays_per_gpu and e.get("build_id") == bid:
            return e
    return {}


def workload_config(cfg, blocks, rays, valid, world):
    """The `config` object of the JSON line -- identical for both arms of the same workload."""
    return {"workload": WORKLOADS[cfg["name"]], "blocks": int(blocks), "rays_per_gpu": int(rays),
            "valid_samples_per_gpu": int(valid), "max_samples": cfg["max_samples"], "step_m": cfg["h"] / 2,
            "beta_m": 2 * cfg["h"], "parallelism": f"rays sharded over {world} GPU(s), grid replicated",
            "l2": f"no flush: inputs exceed L2 (payload + gradient planes {blocks * 512 * 32 / 1e9:.1f} GB "
                  f"vs 126 MB L2)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []  # (perf_counter, line)
        self.t0 = self.t1 = None

    def _reader(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line))

    def start(self):
        """Start nvidia-smi -lms 50 and wait for its first sample, so the timed region that
        follows is covered (nvidia-smi needs ~100+ ms to come up)."""
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        threading.Thread(target=self._reader, daemon=True).start()
        deadline = time.perf_counter() + 5.0
        while not self.lines and time.perf_counter() < deadline:
            time.sleep(0.01)

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def have_samples(self) -> bool:
        t0 = self.t0 if self.t0 is not None else 0.0
        return any(t >= t0 for t, _ in self.lines)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if self.t1 is None:
            self.t1 = time.perf_counter()
        time.sleep(0.06)  # one more sample period
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        t0 = self.t0 if self.t0 is not None else 0.0
        # samples inside the timed region, plus the one straddling its end
        inside = [ln for t, ln in self.lines if t0 <= t <= self.t1 + 0.06]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in inside:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "region_s": self.t1 - t0}


# ----------------------------------------------------------------------------------
# CPU arms (oracle/, only here and in tests)
# ----------------------------------------------------------------------------------
def run_reference(args, cfg, rank, world):
    """--impl reference: the reference CPU path on all host threads, rank 0 only.  Inputs come
    from the reference's own SyntheticScene (synthetic.cpp, oracle/_ref); activation is its
    allocate_for_frames (allocation.cpp:56-83, single thread as written); each step renders
    the whole per-GPU ray set forward + backward with the spec renderer on its grid API
    (march_ray -> gather_corners -> sdf_at / sdf_gradient_at / color_at, parallel_chunks over
    rays, float atomics: SPEC.md:340-341).  No product code is loaded."""
    if rank != 0:
        return
    import oracle

    t_setup = time.perf_counter()
    ref = oracle.ref_available()
    scene = make_scene(cfg, reference=ref)  # fixture restatement only if _ref was not built
    cams, depth = activation_frames(scene, cfg)
    o, d, dC, dD, dN = rays_for_rank(scene, cfg, 0, world)
    Grid = oracle.RefGrid if ref else oracle.OracleGrid
    g = Grid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    t0 = time.perf_counter()
    g.allocate_frames(depth, cams, cfg["dilation"])
    act_s = time.perf_counter() - t0
    coords = g.coords()
    fill_in_chunks(scene, cfg, coords, lambda f, n, p: g.set_payload(f, n, **p))
    cores = os.cpu_count() or 1
    Grid.set_threads(cores)
    S, step_len, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    log(f"[reference] setup {time.perf_counter() - t_setup:.1f}s: {len(coords)} blocks "
        f"(allocate_for_frames {act_s:.1f}s), {len(o)} rays, {cores} threads")

    def step():
        f = g.render_forward(o, d, step_len, S, beta)
        if ref:
            g.render_backward(dC, dD, dN)
        else:
            g.render_backward(o, d, step_len, S, beta, dC, dD, dN)
        return f

    # setup, untimed: the reference renderer allocates its gradient shadow buffers
    # (VoxelBlock::grad_sdf / grad_color, grid.hpp:69) on its first backward
    f0 = g.render_forward(o[:1024], d[:1024], step_len, S, beta)
    g.render_backward(dC[:1024], dD[:1024], dN[:1024]) if ref else None
    del f0
    for _ in range(args.warmup):
        step()
    times, nvalid = [], 0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        f = step()
        times.append(time.perf_counter() - t0)
        nvalid = int(f["n_valid"].sum())
    t = sum(times) / len(times)
    value = nvalid / t
    kind = "reference" if ref else "port"
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic", "impl": "reference", "rays_per_s": len(o) / t,
            "config": workload_config(cfg, len(coords), len(o), nvalid, world),
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": kind,
                             "sample": f"the whole per-GPU step: {len(o)} {cfg['name']} rays fwd+bwd per step, "
                                       f"{nvalid} valid samples"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def parity_report(gpu, ref, what):
    """|gpu - oracle| <= 1e-4 |oracle| + 1e-6 max|oracle| element-wise."""
    g = np.asarray(gpu, np.float64).ravel()
    r = np.asarray(ref, np.float64).ravel()
    scale = float(np.abs(r).max()) if r.size else 0.0
    err = np.abs(g - r)
    bound = 1e-4 * np.abs(r) + 1e-6 * scale
    rel = err / np.maximum(np.abs(r), 1e-6 * scale if scale > 0 else 1e-30)
    return {"n": int(r.size), "outside": int((err > bound).sum()), "max_abs_err": float(err.max(initial=0.0)),
            "max_err_over_bound": float((err / np.maximum(bound, 1e-300)).max(initial=0.0)),
            "max_rel_err": float(rel.max(initial=0.0))}


def cpu_leg_and_parity(grid, coords, payload_chunks, o, d, dC, dD, dN, cfg):
    """The restated oracle (oracle/liboracle.so, fp64) on all host cores renders the SAME rays
    on the SAME grid (same block order) forward + backward: timed as cpu_baseline, and compared
    with the GPU's outputs, gradients and active set (the `parity` object)."""
    from oracle import OracleGrid

    og = OracleGrid(cfg["h"], 8, cfg["C"], capacity=max(len(coords), 1 << 21))
    og.allocate_blocks(coords)
    for f, n, p in payload_chunks():
        og.set_payload(f, n, **p)
    cores = os.cpu_count() or 1
    OracleGrid.set_threads(cores)
    S, step_len, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    t0 = time.perf_counter()
    ref = og.render_forward(o, d, step_len, S, beta)
    gs_o, gr_o, act_o = og.render_backward(o, d, step_len, S, beta, dC, dD, dN)
    dt = time.perf_counter() - t0
    OracleGrid.set_threads(1)
    nvalid = int(ref["n_valid"].sum())
    cpu = {"value": nvalid / dt, "unit": "samples/s", "cores": cores, "kind": "port", "rays_per_s": len(o) / dt,
           "sample": f"the whole step: {len(o)} {cfg['name']} rays fwd+bwd, {nvalid} valid samples in {dt:.2f} s"}
    # the GPU: one forward + backward of the same rays into zeroed gradient planes
    grid.grad_zero()
    out = grid.render_forward(o, d, step_len, S, beta)
    grid.render_backward(dC, dD, dN)
    gs, gr = grid.grads()
    act = grid.active_mask()
    par = {"rays": len(o), "tolerance": "|gpu - oracle| <= 1e-4 |oracle| + 1e-6 max|oracle| (SURVEY.md 8(c))",
           "oracle": "oracle/liboracle.so (fp64 restatement, pinned to the compiled reference)",
           "n_samples_equal": bool(np.array_equal(out["n_samples"], ref["n_samples"])),
           "active_set_equal": bool(np.array_equal(act, act_o)), "active_blocks": int(act_o.sum())}
    for k in ("rgb", "depth", "normal", "wsum"):
        par[k] = parity_report(out[k], ref[k], k)
    par["grad_sdf"] = parity_report(gs, gs_o, "grad_sdf")
    par["grad_rgb"] = parity_report(gr, gr_o, "grad_rgb")
    par["green"] = bool(par["n_samples_equal"] and par["active_set_equal"] and
                        all(par[k]["outside"] == 0 for k in ("rgb", "depth", "normal", "wsum", "grad_sdf",
                                                              "grad_rgb")))
    return cpu, par


# ----------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------
def _all_reduce(dist, t, op=None):
    """all_reduce that also works on a gloo group (CPU round trip)."""
    op = dist.ReduceOp.SUM if op is None else op
    if dist.get_backend() == "gloo" and t.is_cuda:
        c = t.cpu()
        dist.all_reduce(c, op=op)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=op)


def run_ours(args, cfg, rank, world, local_rank):
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid

    dist = None
    if world > 1:
        import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    # a real (non-legacy) stream shared by torch, NCCL ordering and the library
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    t_setup = time.perf_counter()
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    grid = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22, device=local_rank)
    grid.set_stream(stream)
    # A/B hook for the result-neutral knobs: SVR_TUNING="key=v,key=v"
    for kv in filter(None, os.environ.get("SVR_TUNING", "").split(",")):
        k, v = kv.split("=")
        grid.set_tuning(k.strip(), int(v))
    if args.lookup == "hash":
        grid.set_lookup(1)
    rep = grid.allocate_for_frames(depth, cams, cfg["dilation"])
    coords = grid.coords()
    chunks = []
    keep_host = rank == 0 and world == 1 and not args.no_cpu_baseline

    def sink(f, n, p):
        grid.set_payload(f, n, **p)
        if keep_host:
            chunks.append((f, n, p))

    fill_in_chunks(scene, cfg, coords, sink)
    o, d, dC, dD, dN = rays_for_rank(scene, cfg, rank, world)
    n_rays = len(o)
    log(f"[rank {rank}] setup {time.perf_counter() - t_setup:.1f}s: {len(coords)} blocks "
        f"({rep.pixels_used} px), {n_rays} rays, lookup {'dense' if grid.info().lookup_mode == 2 else 'hash'}")

    S, step_len, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    o_d = torch.from_numpy(o).to(dev)
    d_d = torch.from_numpy(d).to(dev)
    dC_d, dD_d, dN_d = (torch.from_numpy(a).to(dev) for a in (dC, dD, dN))
    outs = {"rgb": torch.empty((n_rays, 3), dtype=torch.float32, device=dev),
            "depth": torch.empty((n_rays,), dtype=torch.float32, device=dev),
            "normal": torch.empty((n_rays, 3), dtype=torch.float32, device=dev),
            "wsum": torch.empty((n_rays,), dtype=torch.float32, device=dev),
            "n_samples": None}
    grid.grad_zero()
    reducer = make_reducer(args, grid, dev, dist, rank) if dist is not None else None

    ev = []

    def step(record):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if record else None
        if e:
            e[0].record(stream)
        grid.render_forward(o_d, d_d, step_len, S, beta, out=outs)  # K4 march + K5 forward
        if e:
            e[1].record(stream)
        grid.render_backward(dC_d, dD_d, dN_d)  # K6 backward
        if e:
            e[2].record(stream)
            ev.append(e)
        if reducer is not None:
            reducer["fn"]()  # active-block gradient all-reduce across the ranks
        grid.grad_zero_active()

    if reducer is not None:
        calibrate_reducer(reducer, step, stream, dev, dist)
    for _ in range(max(args.warmup, 3)):
        step(False)
    torch.cuda.synchronize(dev)
    stats = grid.render_stats()
    valid_per_step = int(stats.valid_samples)
    marched_per_step = int(stats.samples)
    info = grid.info()

    clocks = ClockSampler(local_rank)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    clocks.mark_start()
    t0.record(stream)
    for _ in range(args.steps):
        step(True)
    grid.join()  # the last step's pending zeroing (fused into the next forward otherwise) is timed too
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark_stop()
    # a timed region shorter than nvidia-smi's sampling period may hold no sample: keep the
    # GPU under the same load with untimed steps until one arrives (at most 1 s).  Rank 0
    # decides for all ranks, so every rank runs the same number of steps (collectives).
    extended = 0
    t_ext = time.perf_counter()

    def more():
        want = rank == 0 and not clocks.have_samples() and time.perf_counter() - t_ext < 1.0
        if dist is None:
            return want
        f = torch.tensor([1.0 if want else 0.0], dtype=torch.float64, device=dev)
        _all_reduce(dist, f, dist.ReduceOp.MAX)
        return f.item() > 0

    while more():
        step(False)
        torch.cuda.synchronize(dev)
        extended += 1
    if extended:
        clocks.mark_stop()
    if dist is not None:
        dist.barrier()
    clk = clocks.stop()
    if extended:
        clk["extended_untimed_steps"] = extended
    ms = t0.elapsed_time(t1) / args.steps
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    bwd_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    if dist is not None:
        t = torch.tensor([ms, fwd_ms, bwd_ms], dtype=torch.float64, device=dev)
        _all_reduce(dist, t, dist.ReduceOp.MAX)
        ms, fwd_ms, bwd_ms = (float(v) for v in t.tolist())
        vt = torch.tensor([valid_per_step, marched_per_step], dtype=torch.float64, device=dev)
        _all_reduce(dist, vt)
        valid_total, marched_total = (int(v) for v in vt.tolist())
    else:
        valid_total, marched_total = valid_per_step, marched_per_step
    rays_total = n_rays * world

    # --- e2e: the same step through the C-ABI with pinned HOST buffers -----------------
    pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    o_h, d_h, dC_h, dD_h, dN_h = (pin(a) for a in (o, d, dC, dD, dN))
    outs_h = {"rgb": torch.empty((n_rays, 3), dtype=torch.float32).pin_memory(),
              "depth": torch.empty((n_rays,), dtype=torch.float32).pin_memory(),
              "normal": torch.empty((n_rays, 3), dtype=torch.float32).pin_memory(),
              "wsum": torch.empty((n_rays,), dtype=torch.float32).pin_memory(), "n_samples": None}

    def step_host():
        grid.render_forward(o_h, d_h, step_len, S, beta, out=outs_h)
        grid.render_backward(dC_h, dD_h, dN_h)
        if reducer is not None:
            reducer["fn"]()
        grid.grad_zero_active()

    # host_async: pinned host arrays move on the library's copy streams through double-buffered
    # device slots, so step i+1's H2D overlaps step i's kernels (every step still copies its
    # own inputs in and its outputs out inside the timed region)
    grid.set_tuning("host_async", 1)
    for _ in range(2):
        step_host()
    grid.synchronize()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    e2e_steps = max(3, args.steps)  # as many steps as the device-timed region (pipeline fill / drain amortised the same way)
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        step_host()
    grid.synchronize()
    torch.cuda.synchronize(dev)
    e2e_s = (time.perf_counter() - w0) / e2e_steps
    grid.set_tuning("host_async", 0)
    if dist is not None:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        _all_reduce(dist, t, dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = n_rays * (48 + 28)
    d2h = n_rays * 32

    if rank != 0:
        return
    peak, peak_kind = peaks()
    bid = build_id()
    # dominant kernel: K6 backward (one launch: k_backward_pipe); the forward call (ordering,
    # k_march, k_forward) is reported beside it
    bwd_bytes = valid_per_step * BWD_B_SAMPLE + n_rays * BWD_B_RAY
    fwd_bytes = valid_per_step * FWD_B_SAMPLE + n_rays * FWD_B_RAY
    step_bytes = valid_per_step * STEP_B_SAMPLE + n_rays * STEP_B_RAY
    cap = traffic_from_profiles(cfg["name"] + ("_hash" if args.lookup == "hash" else ""), n_rays, bid)
    dom, dom_ms, dom_bytes = "k_backward_pipe", bwd_ms, bwd_bytes
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    dram = cap.get("dram_bytes", {})
    step_dram = sum(dram.get(k, 0) for k in ("k_march", "k_forward", "k_backward_pipe", "k_grad_zero_active"))
    line = {
        "metric": METRIC,
        "value": valid_total / (ms * 1e-3),
        "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong" if cfg.get("strong") else "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "rays_per_s": rays_total / (ms * 1e-3),
        "samples_marched_per_s": marched_total / (ms * 1e-3),
        "config": workload_config(cfg, info.block_count, n_rays, valid_per_step, world),
        "build": {"id": bid, "lookup": "dense" if info.lookup_mode == 2 else "hash",
                  "grad_reduction": ({"used": reducer["used"], "calibration_ms_per_step": reducer["calib_ms"]}
                                     if reducer is not None else None)},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_kind,
                     "traffic": dram.get(dom),
                     "traffic_capture": cap.get("file"),
                     "bytes_model": "SURVEY.md 8(d): fwd 182.8 B/valid sample + 80 B/ray; "
                                    "bwd 256 B/valid sample + 28 B/ray",
                     # measured DRAM traffic of the same kernel over its duration: the byte model
                     # charges every corner read-modify-write to HBM, L2 serves most of them, so
                     # frac (model) can exceed 1 while the DRAM itself runs at dram_frac
                     "dram_achieved": (dram[dom] / (dom_ms * 1e-3) / 1e9) if dram.get(dom) else None,
                     "dram_frac": (dram[dom] / (dom_ms * 1e-3) / 1e9 / peak) if dram.get(dom) else None,
                     "l2_hit_pct": cap.get("l2_hit_pct", {}).get(dom),
                     "kernel_ms": dom_ms, "fwd_call_ms": fwd_ms, "bwd_ms": bwd_ms,
                     "fwd_call_frac": fwd_bytes / (fwd_ms * 1e-3) / 1e9 / peak,
                     "step_frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                     # whole-step measured DRAM bytes (ncu, this build) over the device step time
                     "step_dram_frac": (step_dram / (ms * 1e-3) / 1e9 / peak) if step_dram else None},
        "e2e": {"value": valid_total / e2e_s, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_s * 1e3,
                "path": "SparseDenseGrid.render_forward/backward via C-ABI with pinned host buffers, "
                        "host_async (copies of step i+1 overlap kernels of step i)"},
        "gpu_launches": LAUNCHES_PER_STEP * args.steps + 1,
        "library_launches": {"cub_radix_sort": LIBRARY_LAUNCHES_PER_STEP * args.steps},
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"], line["parity"] = cpu_leg_and_parity(grid, coords, lambda: chunks, o, d, dC, dD,
                                                                      dN, cfg)
        except Exception as e:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    del grid, chunks
    torch.cuda.empty_cache()
    if world == 1 and not args.no_extra and cfg["name"] == "cfg3":
        extra = {}
        for name, fn in (("cfg1_reference_case", lambda: bench_cfg1(dev, stream, cpu=not args.no_cpu_baseline)),
                         ("cfg2_image_forward", lambda: bench_cfg2(dev, stream, cpu=not args.no_cpu_baseline)),
                         ("cfg3_hash_lookup", lambda: bench_cfg3_hash(args, dev, stream)),
                         ("cfg4_activation_and_query", lambda: bench_cfg4(dev, stream, cpu=not args.no_cpu_baseline)),
                         ("cfg3_fusion_and_denoise", lambda: bench_fusion(dev, stream, cpu=not args.no_cpu_baseline)),
                         ("cfg3_refine_step", lambda: bench_refine(dev, stream, cpu=not args.no_cpu_baseline))):
            try:
                extra[name] = fn()
            except Exception as e:  # pragma: no cover
                extra[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
            torch.cuda.empty_cache()
        if "cpu_baseline" in line and "error" not in extra.get("cfg3_hash_lookup", {"error": 1}):
            # the reference renders through its own hash BlockMap whatever the GPU lookup mode
            extra["cfg3_hash_lookup"]["cpu_baseline"] = dict(
                line["cpu_baseline"], sample="the main line's CPU leg (the reference looks every block up in its "
                                             "hash BlockMap; the dense index is a GPU-side choice)")
        line["extra_configs"] = extra
    print(json.dumps(line), flush=True)


# ours per step: k_ray_keys_dir, k_march (+ post-march keys), k_forward (+ the previous step's
# deferred zeroing), k_backward_pipe, k_touch_expand, k_active_count / scan / write (+ the
# reduction's kernels for N > 1); the last step's zeroing runs as k_grad_zero_active at the end of
# the timed region; plus 2 CUB radix sorts that only reorder rays
LAUNCHES_PER_STEP = 8
LIBRARY_LAUNCHES_PER_STEP = 10  # 2 CUB radix sorts of 24-bit keys: histogram + scan + 3 onesweep passes each


def make_reducer(args, grid, dev, dist, rank):
    from paper_2305_13220_b200.distributed import PeerGradReducer, reduce_active_grads

    variants = {}
    if dist.get_backend() == "nccl" or args.reduce == "nccl":
        variants["nccl"] = lambda: reduce_active_grads(grid, dev)
    if args.reduce in ("auto", "peer"):  # sync-free peer group (CUDA IPC; gloo host barriers)
        try:
            variants["peer"] = PeerGradReducer(grid, dev).reduce
        except Exception as e:  # pragma: no cover - no IPC / P2P on this system
            log(f"[rank {rank}] peer reduction unavailable: {e}")
    if not variants:  # gloo test hook: host-side collectives
        variants["host"] = lambda: reduce_active_grads(grid, dev)
    if args.reduce == "nccl":
        variants.pop("peer", None)
    return {"variants": variants, "fn": next(iter(variants.values())), "used": next(iter(variants)),
            "calib_ms": {}, "force": args.reduce}


def calibrate_reducer(reducer, step, stream, dev, dist):
    """Time every available reduction over a few steps and keep the fastest (max over ranks)."""
    import torch

    for name, fn in reducer["variants"].items():
        reducer["fn"] = fn
        for _ in range(2):
            step(False)
        torch.cuda.synchronize(dev)
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(3):
            step(False)
        c1.record(stream)
        torch.cuda.synchronize(dev)
        tt = torch.tensor([c0.elapsed_time(c1) / 3], dtype=torch.float64, device=dev)
        _all_reduce(dist, tt, dist.ReduceOp.MAX)
        reducer["calib_ms"][name] = float(tt.item())
    best = min(reducer["calib_ms"], key=reducer["calib_ms"].get)
    if reducer["force"] in reducer["variants"]:
        best = reducer["force"]
    reducer["fn"], reducer["used"] = reducer["variants"][best], best


def _events_ms(stream, fn, reps):
    import torch

    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _cpu_ref_grid(cfg, coords, chunks):
    """The reference grid code (oracle/_ref) holding the same blocks + payload (else the port)."""
    import oracle

    Grid = oracle.RefGrid if oracle.ref_available() else oracle.OracleGrid
    rg = Grid(cfg["h"], 8, cfg["C"], capacity=max(len(coords), 1 << 21))
    rg.allocate_blocks(coords)
    for f, nb, p in chunks:
        rg.set_payload(f, nb, **p)
    return Grid, rg, "reference" if Grid is oracle.RefGrid else "port"


def bench_cfg1(dev, stream, cpu=True):
    """configs[0] (the reference's CPU-runnable case): 5x5x3 m room, 2 cm voxels (R=2 from 24
    ring frames), 4096 rays from the 24 ring poses, fwd+bwd.  GPU: device time per step
    (forward + backward + zeroing, launch-bound at this size); cpu_baseline leg: the reference
    grid code compiled verbatim + the spec renderer (oracle/_ref), all host cores and 1 core."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid
    from fixtures import uniform_floats

    cfg = CFG1
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], device=dev.index)
    g.set_stream(stream)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    coords = g.coords()
    chunks = []
    fill_in_chunks(scene, cfg, coords, lambda f, n, p: (g.set_payload(f, n, **p), chunks.append((f, n, p))))
    o, d = scene.rays(24, 171, seed=0)
    o, d = np.ascontiguousarray(o[:4096]), np.ascontiguousarray(d[:4096])
    u = uniform_floats(7 * 4096, 1).reshape(4096, 7)
    dC, dD, dN = (np.ascontiguousarray(a) for a in (u[:, :3], u[:, 3], u[:, 4:]))
    dev_in = [torch.from_numpy(a).to(dev) for a in (o, d, dC, dD, dN)]
    n = 4096
    outs = {k: torch.empty(s, dtype=torch.float32, device=dev)
            for k, s in (("rgb", (n, 3)), ("depth", (n,)), ("normal", (n, 3)), ("wsum", (n,)))}
    outs["n_samples"] = None
    step, S, beta = cfg["h"] / 2, 64, 2 * cfg["h"]

    def one():
        g.render_forward(dev_in[0], dev_in[1], step, S, beta, out=outs)
        g.render_backward(dev_in[2], dev_in[3], dev_in[4])
        g.grad_zero_active()
        g.join()

    ms = _events_ms(stream, one, 50)
    st = g.render_stats()
    peak, _ = peaks()
    step_bytes = st.valid_samples * STEP_B_SAMPLE + n * STEP_B_RAY
    out = {"blocks": g.block_count(), "rays": n, "valid_samples": int(st.valid_samples),
           "ms_per_step": ms, "samples_per_s": st.valid_samples / (ms * 1e-3),
           "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                        "bytes_model": "SURVEY.md 8(d): 438.8 B/valid sample + 108 B/ray (fwd + bwd)",
                        "achieved": step_bytes / (ms * 1e-3) / 1e9, "frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                        "note": "launch-bound at 4096 rays (10 kernels for 0.25 M samples)"}}
    # launch-bound at this size: the same step captured once into a CUDA graph and replayed
    try:
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            one()
        gms = _events_ms(stream, graph.replay, 50)
        out["cuda_graph"] = {"ms_per_step": gms, "samples_per_s": st.valid_samples / (gms * 1e-3)}
    except Exception as e:  # pragma: no cover
        out["cuda_graph"] = {"error": str(e)[:200]}
    if cpu:
        Grid, rg, kind = _cpu_ref_grid(cfg, coords, chunks)
        res = {}
        for cores in (os.cpu_count() or 1, 1):
            Grid.set_threads(cores)
            best = None
            for _ in range(3):
                t0 = time.perf_counter()
                f = rg.render_forward(o, d, step, S, beta)
                if kind == "reference":
                    rg.render_backward(dC, dD, dN)
                else:
                    rg.render_backward(o, d, step, S, beta, dC, dD, dN)
                dt = time.perf_counter() - t0
                best = dt if best is None else min(best, dt)
            res[cores] = (int(f["n_valid"].sum()) / best, best)
        Grid.set_threads(1)
        allc = os.cpu_count() or 1
        out["cpu_baseline"] = {"value": res[allc][0], "unit": "samples/s", "cores": allc, "kind": kind,
                               "ms_per_step": res[allc][1] * 1e3,
                               "single_core": {"value": res[1][0], "ms_per_step": res[1][1] * 1e3},
                               "sample": "the whole cfg1 step (4096 rays fwd+bwd), best of 3"}
    del g
    return out


def bench_cfg2(dev, stream, cpu=True):
    """configs[1]: 5x5x3 m room, 2 cm voxels (R=2 from 24 ring frames), one full 640x480
    image from camera_for_frame(0), forward only (color/depth/normal).  CPU: the reference grid
    code + spec renderer (oracle/_ref) on the same image, all host cores and 1 core."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG1
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], device=dev.index)
    g.set_stream(stream)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    coords = g.coords()
    chunks = []
    fill_in_chunks(scene, cfg, coords, lambda f, n, p: (g.set_payload(f, n, **p), chunks.append((f, n, p))))
    o, d = scene.image_rays(0)
    od, dd = torch.from_numpy(o).to(dev), torch.from_numpy(d).to(dev)
    n = len(o)
    outs = {k: torch.empty(s, dtype=torch.float32, device=dev)
            for k, s in (("rgb", (n, 3)), ("depth", (n,)), ("normal", (n, 3)), ("wsum", (n,)))}
    outs["n_samples"] = None
    g.set_tuning("records", 0)  # inference: no backward context needed
    g.set_tuning("ray_sort", 0)  # a full image in raster order is coherent already
    ms = _events_ms(stream, lambda: g.render_forward(od, dd, cfg["h"] / 2, 64, 2 * cfg["h"], out=outs), 20)
    st = g.render_stats()
    peak, _ = peaks()
    fwd_bytes = st.valid_samples * FWD_B_SAMPLE + n * FWD_B_RAY
    out = {"blocks": g.block_count(), "rays": n, "valid_samples": int(st.valid_samples),
           "ms_per_image": ms, "rays_per_s": n / (ms * 1e-3),
           "samples_per_s": st.valid_samples / (ms * 1e-3),
           "roofline": {"bound": "hbm", "achieved": fwd_bytes / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                        "frac": fwd_bytes / (ms * 1e-3) / 1e9 / peak,
                        "bytes_model": "SURVEY.md 8(d) forward-only: 182.8 B/valid sample + 80 B/ray"}}
    if cpu:
        Grid, rg, kind = _cpu_ref_grid(cfg, coords, chunks)
        res = {}
        for cores in (os.cpu_count() or 1, 1):
            Grid.set_threads(cores)
            t0 = time.perf_counter()
            f = rg.render_forward(o, d, cfg["h"] / 2, 64, 2 * cfg["h"])
            dt = time.perf_counter() - t0
            res[cores] = (n / dt, int(f["n_valid"].sum()) / dt, dt)
        Grid.set_threads(1)
        allc = os.cpu_count() or 1
        out["cpu_baseline"] = {"value": res[allc][0], "unit": "rays/s", "cores": allc, "kind": kind,
                               "samples_per_s": res[allc][1], "ms_per_image": res[allc][2] * 1e3,
                               "single_core": {"value": res[1][0], "unit": "rays/s", "ms_per_image": res[1][2] * 1e3},
                               "sample": "the whole 640x480 image, forward only"}
    del g
    return out


def bench_cfg3_hash(args, dev, stream, steps=10):
    """The headline cfg3 step with the hash table as the block lookup (SVR_LOOKUP_HASH) instead
    of the dense AABB index: same rays, same grid, every march / forward block lookup and the
    neighbour table go through the open-addressing table (K1)."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG3
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22, device=dev.index)
    g.set_stream(stream)
    g.set_lookup(1)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    fill_in_chunks(scene, cfg, g.coords(), lambda f, n, p: g.set_payload(f, n, **p))
    o, d, dC, dD, dN = (torch.from_numpy(a).to(dev) for a in rays_for_rank(scene, cfg, 0, 1))
    S, step_len, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    g.grad_zero()
    ev = []

    def one():
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        g.render_forward(o, d, step_len, S, beta, out={"n_samples": None})
        e[1].record(stream)
        g.render_backward(dC, dD, dN)
        e[2].record(stream)
        g.grad_zero_active()
        ev.append(e)

    ms = _events_ms(stream, one, steps)
    g.join()
    torch.cuda.synchronize()
    ev = ev[2:]
    st = g.render_stats()
    info = g.info()
    peak, _ = peaks()
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    bwd_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    bwd_bytes = st.valid_samples * BWD_B_SAMPLE + len(o) * BWD_B_RAY
    step_bytes = st.valid_samples * STEP_B_SAMPLE + len(o) * STEP_B_RAY
    out = {"lookup": "hash" if info.lookup_mode == 1 else "dense", "hash_slots": int(info.hash_slots),
           "blocks": int(info.block_count), "rays": len(o), "valid_samples": int(st.valid_samples),
           "ms_per_step": ms, "samples_per_s": st.valid_samples / (ms * 1e-3), "fwd_call_ms": fwd_ms,
           "bwd_ms": bwd_ms,
           "roofline": {"bound": "hbm", "kernel": "k_backward_pipe", "peak": peak, "unit": "GB/s",
                        "achieved": bwd_bytes / (bwd_ms * 1e-3) / 1e9,
                        "frac": bwd_bytes / (bwd_ms * 1e-3) / 1e9 / peak,
                        "step_frac": step_bytes / (ms * 1e-3) / 1e9 / peak}}
    cap = traffic_from_profiles("cfg3_hash", len(o), build_id())
    if cap:
        out["roofline"]["ncu"] = {"file": cap.get("file"), "dram_bytes": cap.get("dram_bytes"),
                                  "l2_hit_pct": cap.get("l2_hit_pct")}
    del g
    return out


def bench_cfg4(dev, stream, n_frames=300, k=256, cpu=True):
    """configs[3]: block activation + hash insert from 300 GT depth frames (640x480) into an
    empty 1 cm grid (R=2), then a k^3 query_sdf_with_gradient sweep over the bounds.  CPU: the
    reference's allocate_for_frames (allocation.cpp:56-83, single thread as written) on the
    same 300 frames -- its coordinate set is also compared with the GPU's (`parity`) -- and its
    query_sdf_with_gradient (grid.cpp:250-261) on a bounded point sample."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG4
    scene = make_scene(cfg)
    cams = scene.cameras(n_frames)
    depth = scene.depth(cams)
    depth_d = torch.from_numpy(depth).to(dev)
    times = []
    for _ in range(3):
        g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22, device=dev.index)
        g.set_stream(stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        rep = g.allocate_for_frames(depth_d, cams, cfg["dilation"])
        e1.record(stream)
        torch.cuda.synchronize()
        times.append((time.perf_counter() - t0, e0.elapsed_time(e1) * 1e-3))
    act_s = min(t[0] for t in times)
    act_dev_s = min(t[1] for t in times)
    coords = g.coords()
    fill_in_chunks(scene, cfg, coords, lambda f, n, p: g.set_payload(f, n, **p))
    info = g.info()
    L = cfg["h"] * 8
    lo = np.array(info.bounds_lo) * L
    hi = (np.array(info.bounds_hi) + 1) * L
    ax = [np.linspace(lo[a], hi[a], k, endpoint=False) + (hi[a] - lo[a]) / (2 * k) for a in range(3)]
    pts = np.stack(np.meshgrid(*ax, indexing="ij"), -1).reshape(-1, 3)
    x = torch.from_numpy(pts).to(dev)
    sdf = torch.empty(len(pts), dtype=torch.float64, device=dev)
    grad = torch.empty((len(pts), 3), dtype=torch.float64, device=dev)
    valid = torch.empty(len(pts), dtype=torch.uint8, device=dev)
    from paper_2305_13220_b200._lib import check

    ms = _events_ms(stream, lambda: check(g._lib.svr_query(g._h, x.data_ptr(), len(pts), sdf.data_ptr(),
                                                           grad.data_ptr(), None, None, valid.data_ptr())), 5)
    peak, _ = peaks()
    C = cfg["C"]
    act_bytes_all = depth.size * ACT_B_PIXEL + rep.blocks_added * (16 + 12 + 512 * (20 + 4 * C))
    q_bytes = len(pts) * QUERY_B_POINT
    out = {"frames": n_frames, "pixels": int(depth.size), "pixels_used": int(rep.pixels_used),
           "blocks": int(rep.blocks_added), "activation_ms": act_s * 1e3, "activation_device_ms": act_dev_s * 1e3,
           "activation_first_ms": times[0][0] * 1e3,
           "activation_note": ("best of 3 fresh grids; the first (activation_first_ms) also pays the driver's "
                               "first-touch mapping of the 7.8 GB of per-block arrays, later grids reuse the "
                               "library's cached device blocks"),
           "pixels_per_s": depth.size / act_s, "blocks_per_s": rep.blocks_added / act_s,
           "query_points": len(pts), "query_valid": int(valid.sum().item()), "query_ms": ms,
           "query_points_per_s": len(pts) / (ms * 1e-3),
           "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                        "bytes_model": "SURVEY.md 8(d) cfg4: 4 B/pixel + per new block 16 + 12 + 512 (20 + 4C) B; "
                                       "query 127 B/point",
                        "activation_achieved": act_bytes_all / act_s / 1e9,
                        "activation_frac": act_bytes_all / act_s / 1e9 / peak,
                        "query_achieved": q_bytes / (ms * 1e-3) / 1e9,
                        "query_frac": q_bytes / (ms * 1e-3) / 1e9 / peak}}
    if cpu:
        import oracle

        Grid = oracle.RefGrid if oracle.ref_available() else oracle.OracleGrid
        kind = "reference" if Grid is oracle.RefGrid else "port"
        rg = Grid(cfg["h"], 8, C, capacity=1 << 22)
        Grid.set_threads(1)
        t0 = time.perf_counter()
        rrep = rg.allocate_frames(depth, cams, cfg["dilation"])
        dt = time.perf_counter() - t0
        rc = rg.coords()
        m21 = 0x1FFFFF
        key = lambda c: np.sort(((c[:, 0].astype(np.int64) & m21) << 42) | ((c[:, 1].astype(np.int64) & m21) << 21)  # noqa: E731
                                | (c[:, 2].astype(np.int64) & m21))
        out["parity"] = {"coordinate_set_equal": bool(len(rc) == len(coords) and np.array_equal(key(rc), key(coords))),
                         "report_equal": bool((rrep.blocks_added, rrep.blocks_requested, rrep.pixels_used) ==
                                              (rep.blocks_added, rep.blocks_requested, rep.pixels_used)),
                         "blocks": int(len(rc)), "oracle": f"{kind} allocate_for_frames on the same 300 frames"}
        out["cpu_baseline"] = {"value": depth.size / dt, "unit": "pixels/s", "cores": 1, "kind": kind,
                               "blocks_per_s": rrep.blocks_added / dt, "activation_ms": dt * 1e3,
                               "sample": "allocate_for_frames over all 300 frames (single thread, as written)"}
        # query sweep on a bounded sample (the reference query is a serial loop)
        fill_in_chunks(scene, cfg, rc, lambda f, n, p: rg.set_payload(f, n, **p))
        sub = pts[:: max(1, len(pts) // (1 << 20))]
        t0 = time.perf_counter()
        q = rg.query(sub)
        dt = time.perf_counter() - t0
        out["cpu_baseline_query"] = {"value": len(sub) / dt, "unit": "points/s", "cores": 1, "kind": kind,
                                     "valid": int(q["valid"].sum()),
                                     "sample": f"every {max(1, len(pts) // (1 << 20))}th point of the sweep "
                                               f"({len(sub)} points) through query_sdf_with_gradient"}
    del g
    return out


def bench_fusion(dev, stream, cpu=True):
    """SURVEY.md 8(f) rank 3 on the cfg3 grid: fuse_all of the 64 activation frames (640x480
    GT depth + rgb + one-hot semantics, mu = L*R) from HBM-resident images, then denoise
    (radius 1, sigma 1 voxel).  CPU: the oracle on all host cores over the first 2 frames."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG3
    scene = make_scene(cfg)
    cams = scene.cameras(cfg["act_frames"])
    depth, rgb, sem = scene.frames(cams)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], device=dev.index)
    g.set_stream(stream)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    mu = 8 * cfg["h"] * cfg["dilation"]
    dd, dr, ds = (torch.from_numpy(a).to(dev) for a in (depth, rgb, sem))
    torch.cuda.synchronize()
    rep = {}

    def fuse():
        rep["r"] = g.fuse_all(dd, cams, mu, rgb=dr, semantic=ds)

    fuse_ms = _events_ms(stream, fuse, 3)
    r = rep["r"]
    den_ms = _events_ms(stream, lambda: g.denoise(1.0, 1), 3)
    mc = {}

    def mesh():
        mc["n"] = g._lib.svr_marching_cubes(g._h, 0.0, ctypes.byref(mc.setdefault("nv", ctypes.c_uint64())),
                                            ctypes.byref(mc.setdefault("nt", ctypes.c_uint64())))

    mc_ms = _events_ms(stream, mesh, 3)
    A, C = g.block_count(), cfg["C"]
    vox = A * 512
    # algorithmic bytes of one denoise: read + write payload float4 + logits, read validity
    den_bytes = vox * (16 + 4 * C) * 2 + A * 64
    # fuse_all: the 32.32 fixed-point sums (4 + C channels) and counts read + written once per
    # launch, the frames read (depth 4 + rgb 12 + semantics 4C per pixel), the finalize pass
    # writing payload + weight + logits + validity
    npx = depth.size
    fuse_bytes = vox * ((4 + C) * 8 + 4) * 2 + npx * (4 + 12 + 4 * C) + vox * (16 + 4 + 4 * C) + A * 64
    peak, _ = peaks()
    out = {"blocks": A, "frames": len(cams), "voxel_frame_pairs": vox * len(cams),
           "associations": int(r.in_view), "integrated": int(r.integrated), "rejected": int(r.rejected),
           "fuse_all_ms": fuse_ms, "voxel_frames_per_s": vox * len(cams) / (fuse_ms * 1e-3),
           "associations_per_s": r.in_view / (fuse_ms * 1e-3),
           "denoise_ms": den_ms, "denoise_voxels_per_s": vox / (den_ms * 1e-3),
           "denoise_GBps_algorithmic": den_bytes / (den_ms * 1e-3) / 1e9,
           "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                        "bytes_model": "fuse_all: sums + counts read and written once, frames read once, finalize "
                                       "writes payload / weight / logits / validity; denoise: payload + logits read "
                                       "and written, validity read",
                        "fuse_achieved": fuse_bytes / (fuse_ms * 1e-3) / 1e9,
                        "fuse_frac": fuse_bytes / (fuse_ms * 1e-3) / 1e9 / peak,
                        "denoise_achieved": den_bytes / (den_ms * 1e-3) / 1e9,
                        "denoise_frac": den_bytes / (den_ms * 1e-3) / 1e9 / peak,
                        "note": "k_fuse is FP64-issue bound (exact Camera::project per voxel-frame pair), "
                                "k_denoise issue / barrier bound (fp64 separable passes)"},
           "marching_cubes_ms": mc_ms, "mesh_vertices": int(mc["nv"].value), "mesh_triangles": int(mc["nt"].value),
           "marching_cubes_cells_per_s": vox / (mc_ms * 1e-3),
           "launches": {"fuse_all": "memset x2 + k_fuse x ceil(64 / batch) + k_fuse_finalize",
                        "denoise": "k_denoise x1",
                        "marching_cubes": "k_mc_count, k_mc_emit, k_mc_heads, k_mc_resolve, k_mc_keep, "
                                          "k_mc_compact, k_mc_attrs + CUB scans / radix sort"}}
    if cpu:
        from oracle import OracleGrid

        og = OracleGrid(cfg["h"], 8, C, capacity=max(A, 1 << 21))
        og.allocate_blocks(g.coords())
        cores = os.cpu_count() or 1
        OracleGrid.set_threads(cores)
        og.fuse_begin(True, True)
        t0 = time.perf_counter()
        og.fuse_frames(depth[:2], cams[:2], mu, rgb=rgb[:2], sem=sem[:2])
        dt = time.perf_counter() - t0
        OracleGrid.set_threads(1)
        out["cpu_baseline"] = {"value": vox * 2 / dt, "unit": "voxel_frames/s", "cores": cores, "kind": "port",
                               "sample": f"fuse_frames over the first 2 frames ({dt:.2f} s)"}
        # marching cubes: the oracle on a contiguous middle slab of 40000 blocks (index order is
        # ascending (z, y, x), so the slab is spatially coherent and crosses the surfaces)
        nb = min(A, 40000)
        b0 = (A - nb) // 2
        p = g.get_payload(b0, nb)
        om = OracleGrid(cfg["h"], 8, C, capacity=max(A, 1 << 21))
        om.allocate_blocks(g.coords()[b0:b0 + nb])
        om.set_payload(0, nb, **p)
        OracleGrid.set_threads(cores)
        t0 = time.perf_counter()
        sm = om.marching_cubes(0.0)
        dt = time.perf_counter() - t0
        OracleGrid.set_threads(1)
        out["cpu_baseline_marching_cubes"] = {"value": nb * 512 / dt, "unit": "cells/s", "cores": cores,
                                              "kind": "port",
                                              "sample": f"blocks [{b0}, {b0 + nb}) -> {len(sm['triangles'])} "
                                                        f"triangles ({dt:.2f} s)"}
    del g
    torch.cuda.empty_cache()
    return out


def bench_refine(dev, stream, steps=20, cpu=True):
    """SURVEY.md 8(f) / SPEC.md:320-327: the full refinement step at the paper's batch (64 images
    x 1024 rays) on the cfg3 grid with device-resident 640x480 frames (rgb, depth prior,
    normal prior): sample batch -> forward -> losses -> backward -> Eikonal -> RMSProp."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid
    from paper_2305_13220_b200.refine import RefineConfig, Refiner, frames_to_device

    cfg = CFG3
    scene = make_scene(cfg)
    cams = scene.cameras(cfg["act_frames"])
    depth, rgb, _, nrm = scene.frames(cams, normals=True)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], device=dev.index)
    g.set_stream(stream)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    fill_in_chunks(scene, cfg, g.coords(), lambda f, n, p: g.set_payload(f, n, **p))
    r, dp, nm = frames_to_device(rgb, depth, nrm, device=dev)
    mu = 8 * cfg["h"] * cfg["dilation"]
    # 256 samples: with R = 2 the allocated shell in front of a surface alone is 2 L = 16 cm =
    # 32 samples at h/2 and rays cross other shells first; 64 would stop most rays short
    ref = Refiner(g, cams, r, dp, nm, step_m=cfg["h"] / 2, beta=2 * cfg["h"], mu=mu,
                  config=RefineConfig(max_samples=256))
    ref.run(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ref.run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    st = ref.step(0, 1, stats=True)
    # the step's sizes for the byte model: re-render the last batch (forward + backward only)
    S, step_m, beta = 256, cfg["h"] / 2, 2 * cfg["h"]
    g.grad_zero()
    g.render_forward(ref.o, ref.d, step_m, S, beta)
    g.render_backward(ref.grads["d_rgb"], ref.grads["d_depth"], ref.grads["d_normal"])
    valid = int(g.render_stats().valid_samples)
    act = int(g.active_mask().sum())
    g.grad_zero()
    peak, _ = peaks()
    step_bytes = valid * STEP_B_SAMPLE + ref.n * STEP_B_RAY + act * 512 * 96
    out = {"rays_per_step": ref.n, "max_samples": 256, "ms_per_step": ms, "rays_per_s": ref.n / (ms * 1e-3),
           "valid_samples": valid, "active_blocks": act,
           "roofline": {"bound": "hbm", "peak": peak, "unit": "GB/s",
                        "bytes_model": "render 438.8 B/valid sample + 108 B/ray; RMSProp 96 B per active voxel "
                                       "(gradient, rms state and payload float4 read + written)",
                        "achieved": step_bytes / (ms * 1e-3) / 1e9, "frac": step_bytes / (ms * 1e-3) / 1e9 / peak},
           "loss": {k: st[k] for k in ("L_c", "L_d", "L_n", "L_eik", "total")},
           "launches_per_step": "k_sample_frame_rays, ray order x2 (+CUB), k_march, k_forward, k_loss_sums, "
                                "k_loss_fit, k_loss_grad, k_backward (S > 64: non-pipelined), k_band_count (+CUB scan), k_band_write, "
                                "k_sample_uniform, k_eik_stats, k_eik_scatter, k_active_*, k_rmsprop"}
    if cpu:  # the oracle's fp64 step on the host cores over 1/16 of the same batch
        from oracle import OracleGrid, render_losses as oracle_losses

        A = g.block_count()
        og = OracleGrid(cfg["h"], 8, cfg["C"], capacity=max(A, 1 << 21))
        og.allocate_blocks(g.coords())
        for f in range(0, A, 16384):
            m = min(16384, A - f)
            og.set_payload(f, m, **g.get_payload(f, m))
        m = ref.n // 16
        host = {k: v[:m].cpu().numpy() for k, v in (("o", ref.o), ("d", ref.d), ("tgt", ref.tgt), ("pd", ref.pd),
                                                      ("pn", ref.pn), ("ci", ref.ci))}
        npts = min(len(ref.pts), ref.cfg.uniform_points + ref.cfg.band_cap) // 16
        pts = ref.pts[:npts].cpu().numpy()
        cores = os.cpu_count() or 1
        OracleGrid.set_threads(cores)
        t0 = time.perf_counter()
        o_out = og.render_forward(host["o"], host["d"], step_m, S, beta)
        o_g, _ = oracle_losses(o_out, host["tgt"], host["pd"], host["pn"], host["ci"], cams)
        gs, gr, active = og.render_backward(host["o"], host["d"], step_m, S, beta, o_g["d_rgb"], o_g["d_depth"],
                                            o_g["d_normal"])
        _, _, egs, eact = og.eikonal(pts, 1.0)
        rms = np.zeros((A, 512, 4), np.float32)
        og.rmsprop(gs + egs, gr, active | eact, 1e-3, 0.9, 1e-8, rms)
        dt = time.perf_counter() - t0
        OracleGrid.set_threads(1)
        out["cpu_baseline"] = {"value": m / dt, "unit": "rays/s", "cores": cores, "kind": "port",
                               "sample": f"{m} rays of the batch (1/16): forward + losses + backward + Eikonal on "
                                         f"{npts} points + RMSProp, fp64 oracle ({dt:.2f} s)"}
    del ref, g
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="skip the CPU timing / parity legs")
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg1/2/4, hash, fusion and refine rows")
    ap.add_argument("--reduce", default="auto", choices=["auto", "peer", "nccl"],
                    help="N > 1 gradient reduction: fused peer-memory kernel, NCCL, or the faster of both")
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS),
                    help="cfg3: 1M rays per GPU (weak scaling, default); cfg5: 8M rays split over the GPUs")
    ap.add_argument("--lookup", default="auto", choices=["auto", "hash"],
                    help="block lookup: dense AABB index when it fits (auto) or the hash table")
    ap.add_argument("--rays-per-pose", type=int, default=None)
    ap.add_argument("--dry-run", action="store_true", help="print the resolved rank / world and exit")
    args = ap.parse_args()
    base = CFG5 if args.workload == "cfg5" else CFG3
    cfg = dict(base, rays_per_pose=args.rays_per_pose or base["rays_per_pose"])
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torch.distributed.run with --gpus ranks
        import socket

        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: one rank per GPU expected")
    if args.dry_run:
        print(json.dumps({"rank": rank, "world": world, "local_rank": local_rank, "impl": args.impl}), flush=True)
        return
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    # test hook (CI on a 1-GPU box): SVR_BENCH_PG=gloo + SVR_BENCH_SAME_GPU=1 run every rank
    # on cuda:0 with host-side collectives, which is safe on one device only because no kernel
    # then waits for another rank's kernel (NCCL kernels would)
    if os.environ.get("SVR_BENCH_SAME_GPU") == "1":
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local_rank)
        backend = os.environ.get("SVR_BENCH_PG", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, cfg, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
