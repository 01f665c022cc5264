"""The refinement loop around the rendering path (SPEC.md:297-327 `backward_step` / `refine`,
PAPER sec. 3.5, Eq. 23), composed from the library's kernels on one device stream:

  K17 batch of images_per_batch x rays_per_image rays from the device-resident frames
  K4/K5 render_forward -> K15 losses (colour L1, depth L2 with the minibatch affine prior
  fit, normal L1) -> K6 render_backward -> K16 band samples (|sdf| < mu/2) + K9 uniform
  samples -> K10 Eikonal (scale lambda_eik) -> K11 RMSProp (lr decayed exponentially to
  lr * gamma over the run), which also zeroes the active gradients.

Frames and every per-step buffer stay in HBM; a step synchronises with the host only for
the band-point count and the Eikonal normaliser (and for the loss stats when asked).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import Camera, check


@dataclass
class RefineConfig:
    """RenderConfig + the sampling choices of this build."""

    rays_per_image: int = 1024
    images_per_batch: int = 64
    lambda_d: float = 0.1
    lambda_n: float = 0.05
    lambda_eik: float = 0.1
    lr: float = 1e-3
    gamma: float = 0.1
    alpha: float = 0.99
    eps: float = 1e-8
    max_samples: int = 64
    uniform_points: int = 16384   # sample_eikonal_points part (b)
    band_cap: int = 65536         # cap on part (a) (surface-band ray samples) per step
    seed: int = 0


class Refiner:
    """refine(grid, frames, config) on a SparseDenseGrid.

    frames: rgb [F,H,W,3], depth prior [F,H,W] (<= 0 invalid) and normal prior [F,H,W,3]
    (camera frame, zeros invalid) as CUDA tensors (or None), cameras: list of Camera.
    step_m: sample spacing (h/2), beta: Laplace scale (2h), mu: truncation (band = mu/2).
    """

    def __init__(self, grid, cameras, rgb, depth=None, normal=None, *, step_m, beta, mu,
                 config: RefineConfig | None = None, group=None):
        import torch
        import torch.distributed as dist

        # data parallel over a process group: each rank draws its own batch, the per-rank
        # means are scaled by 1/world and the voxel gradients summed (distributed.py) before
        # the update, so every replica applies the same step
        self.group = group
        self.world = dist.get_world_size(group) if (group is not None or dist.is_initialized()) else 1
        self.rank = dist.get_rank(group) if self.world > 1 else 0

        self.g = grid
        if self.world > 1:
            # the 1/world scaling of the upstream gradients (torch ops) and the process-group
            # collectives of reduce_active_grads run on torch's current stream: the grid's
            # kernels must be ordered on that same stream
            grid.set_stream(torch.cuda.current_stream(rgb.device))
        self.cfg = config or RefineConfig()
        self.step_m, self.beta, self.mu = step_m, beta, mu
        self.cams = list(cameras)
        self.rgb, self.depth, self.normal = rgb, depth, normal
        dev = rgb.device
        self.dev = dev
        n = self.cfg.rays_per_image * self.cfg.images_per_batch
        self.n = n
        f32 = dict(dtype=torch.float32, device=dev)
        self.o = torch.empty((n, 3), dtype=torch.float64, device=dev)
        self.d = torch.empty((n, 3), dtype=torch.float64, device=dev)
        self.tgt = torch.empty((n, 3), **f32)
        self.pd = torch.empty((n,), **f32)
        self.pn = torch.empty((n, 3), **f32)
        self.ci = torch.empty((n,), dtype=torch.int32, device=dev)
        self.out = {"rgb": torch.empty((n, 3), **f32), "depth": torch.empty((n,), **f32),
                    "normal": torch.empty((n, 3), **f32), "wsum": torch.empty((n,), **f32), "n_samples": None}
        self.grads = {"d_rgb": torch.empty((n, 3), **f32), "d_depth": torch.empty((n,), **f32),
                      "d_normal": torch.empty((n, 3), **f32)}
        self.pts = torch.empty((self.cfg.band_cap + self.cfg.uniform_points, 3), dtype=torch.float64, device=dev)
        self._camarr = (Camera * len(self.cams))(*self.cams)
        self.cams_dev = torch.frombuffer(bytearray(bytes(self._camarr)), dtype=torch.uint8).to(dev)
        # the frames / cameras were uploaded on torch's stream; the grid may run on its own (world 1)
        torch.cuda.synchronize(dev)

    def lr_at(self, i: int, steps: int) -> float:
        """exponential decay to lr * gamma at the final step."""
        return self.cfg.lr * self.cfg.gamma ** (i / max(steps - 1, 1))

    def step(self, i: int, steps: int, stats: bool = False) -> dict | None:
        c, g, lib = self.cfg, self.g, self.g._lib
        ptr = lambda t: t.data_ptr() if t is not None else None  # noqa: E731
        check(lib.svr_sample_frame_rays(
            g._h, self.cams_dev.data_ptr(), len(self.cams), ptr(self.rgb), ptr(self.depth), ptr(self.normal),
            c.images_per_batch, c.rays_per_image, (c.seed * 1000003 + i) * 65599 + self.rank, ptr(self.o),
            ptr(self.d), ptr(self.tgt),
            ptr(self.pd), ptr(self.pn), ptr(self.ci), None))
        g.render_forward(self.o, self.d, self.step_m, c.max_samples, self.beta, out=self.out)
        _, st = g.render_losses(self.out, self.tgt, self.pd if self.depth is not None else None,
                                self.pn if self.normal is not None else None, self.ci, self.cams,
                                c.lambda_d, c.lambda_n, grads=self.grads, stats=stats)
        if self.world > 1:
            for t in self.grads.values():
                t.mul_(1.0 / self.world)
        g.render_backward(self.grads["d_rgb"], self.grads["d_depth"], self.grads["d_normal"])
        nb = ctypes.c_uint64()
        check(lib.svr_band_points(g._h, 0.5 * self.mu, c.band_cap, self.pts.data_ptr(), ctypes.byref(nb)))
        m = min(nb.value, c.band_cap)
        if c.uniform_points:
            check(lib.svr_sample_uniform(g._h, c.uniform_points, (c.seed * 7919 + i) * 65599 + self.rank,
                                         self.pts[m:].data_ptr()))
            m += c.uniform_points
        eik = (0.0, 0)
        if m and c.lambda_eik > 0:
            eik = g.eikonal(self.pts[:m], c.lambda_eik / self.world)
        if self.world > 1:
            from .distributed import reduce_active_grads

            reduce_active_grads(g, self.dev, self.group)
        g.rmsprop_step(self.lr_at(i, steps), c.alpha, c.eps)
        if stats:
            st = dict(st)
            st["L_eik"], st["eik_points"] = eik
            st["total"] += c.lambda_eik * eik[0]
            st["lr"] = self.lr_at(i, steps)
        return st

    def run(self, steps: int, log_every: int = 0) -> list[dict]:
        """The step loop; returns the loss trace (step, L_c, L_d, L_n, L_eik,
        total, lr) at every log_every-th step."""
        trace = []
        for i in range(steps):
            want = bool(log_every) and (i % log_every == 0 or i == steps - 1)
            st = self.step(i, steps, stats=want)
            if want:
                st["step"] = i
                trace.append(st)
        return trace


def frames_to_device(rgb, depth=None, normal=None, device="cuda"):
    """Host frame arrays -> contiguous CUDA tensors (one upload for the whole run)."""
    import torch

    f = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(device)  # noqa: E731
    return f(rgb), f(depth), f(normal)


class NativeRefiner:
    """The same loop run by the library's own C++ host code (svr_refiner_* in include/svr.h):
    frames copied to the device once, every per-step buffer owned by the handle.  Single
    GPU; use Refiner(group=...) for data parallelism."""

    def __init__(self, grid, cameras, rgb, depth=None, normal=None, *, step_m, beta, mu,
                 config: RefineConfig | None = None):
        from ._lib import RefineConfig as CCfg

        c = config or RefineConfig()
        lib = grid._lib
        cc = CCfg()
        lib.svr_refine_config_default(ctypes.byref(cc))
        for f, _ in CCfg._fields_:
            if hasattr(c, f):
                setattr(cc, f, getattr(c, f))
        cc.step, cc.beta, cc.mu = step_m, beta, mu
        self.g, self.lib, self.cfg = grid, lib, c
        arr = (Camera * len(cameras))(*cameras)
        keep = []
        ptr = lambda a: None if a is None else (a.data_ptr() if hasattr(a, "data_ptr") else  # noqa: E731
                                                 (keep.append(np.ascontiguousarray(a, np.float32)) or keep[-1].ctypes.data))
        h = ctypes.c_void_p()
        check(lib.svr_refiner_create(grid._h, ctypes.addressof(arr), len(cameras), ptr(rgb), ptr(depth), ptr(normal),
                                     ctypes.byref(cc), ctypes.byref(h)))
        self._h = h

    def step(self, i: int, steps: int, stats: bool = False) -> dict | None:
        from ._lib import LossStats

        st = LossStats()
        el = ctypes.c_double()
        check(self.lib.svr_refiner_step(self._h, i, steps, ctypes.byref(st) if stats else None, ctypes.byref(el)))
        if not stats:
            return None
        out = {f: getattr(st, f) for f, _ in LossStats._fields_}
        out["L_eik"] = el.value
        out["lr"] = self.cfg.lr * self.cfg.gamma ** (i / max(steps - 1, 1))
        return out

    def run(self, steps: int, log_every: int = 0) -> list[dict]:
        trace = []
        for i in range(steps):
            want = bool(log_every) and (i % log_every == 0 or i == steps - 1)
            st = self.step(i, steps, stats=want)
            if want:
                st["step"] = i
                trace.append(st)
        return trace

    def close(self):
        if self._h:
            self.lib.svr_refiner_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
