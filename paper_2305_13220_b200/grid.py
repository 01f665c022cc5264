"""Python mirror of the reference grid/renderer API over the C-ABI (include/svr.h).

``SparseDenseGrid`` keeps the reference's names and error behaviour
(/root/reference/proj/src/core/grid.hpp:100-223, allocation.hpp:22-29,
grid_io.hpp:14-15, renderer ops of SPEC.md:268-327) so parity tests read like the
reference's own tests.  Array arguments may be numpy arrays (host) or torch tensors
(host or CUDA); CUDA tensors stay on the device and the call is asynchronous on the
grid's stream.  Every numerical result comes from libsvr_b200.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes
from typing import Any

import numpy as np

from . import _lib
from ._lib import AllocReport, Camera, FuseReport, GridInfo, LossStats, RenderStats, check

try:  # torch is plumbing only (device buffers, streams); numpy works without it
    import torch
except Exception:  # pragma: no cover
    torch = None


def _is_tensor(a: Any) -> bool:
    return torch is not None and isinstance(a, torch.Tensor)


def _in(a, dtype, keep: list):
    """Address of a read-only array argument (None -> NULL)."""
    if a is None:
        return None
    if _is_tensor(a):
        want = {np.float64: torch.float64, np.float32: torch.float32, np.int32: torch.int32,
                np.uint32: torch.int32, np.uint8: torch.uint8}[dtype]
        if a.dtype != want or not a.is_contiguous():
            a = a.to(want).contiguous()
        keep.append(a)
        return a.data_ptr()
    arr = np.ascontiguousarray(a, dtype=dtype)
    keep.append(arr)
    return arr.ctypes.data


def _out(shape, dtype, like=None):
    """Allocate an output: a CUDA tensor when `like` is a CUDA tensor, else numpy."""
    if like is not None and _is_tensor(like) and like.is_cuda:
        tdt = {np.float64: torch.float64, np.float32: torch.float32, np.uint32: torch.int32,
               np.uint8: torch.uint8, np.int32: torch.int32}[dtype]
        t = torch.empty(shape, dtype=tdt, device=like.device)
        return t, t.data_ptr()
    arr = np.empty(shape, dtype=dtype)
    return arr, arr.ctypes.data


def camera(fx, fy, cx, cy, width, height, R=None, t=None) -> Camera:
    """svr_camera from intrinsics and a camera-to-world pose (camera.hpp:16-29)."""
    c = Camera()
    c.fx, c.fy, c.cx, c.cy = fx, fy, cx, cy
    c.width, c.height = int(width), int(height)
    R = np.eye(3) if R is None else np.asarray(R, dtype=np.float64).reshape(3, 3)
    t = np.zeros(3) if t is None else np.asarray(t, dtype=np.float64).reshape(3)
    c.R[:] = list(R.reshape(9))
    c.t[:] = list(t)
    return c


class SparseDenseGrid:
    """Device-resident globally-sparse / locally-dense 8^3 voxel-block grid."""

    kInvalidBlock = _lib.SVR_INVALID_BLOCK
    kDefaultCapacity = 1 << 21

    def __init__(self, voxel_size: float, block_res: int = 8, label_channels: int = 1,
                 capacity: int = 0, device: int = 0, _handle=None):
        self._lib = _lib.load()
        if _handle is not None:
            self._h = _handle
        else:
            h = ctypes.c_void_p()
            check(self._lib.svr_grid_create(voxel_size, block_res, label_channels, capacity, device,
                                            ctypes.byref(h)))
            self._h = h
        info = self.info()
        self._voxel_size = info.voxel_size
        self._block_res = info.block_res
        self._label_channels = info.label_channels
        self._capacity = info.capacity
        self.device = info.device

    # --- lifetime ----------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.svr_grid_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @classmethod
    def load(cls, path: str, device: int = 0) -> "SparseDenseGrid":
        """load_grid (grid_io.cpp:83-97): index = record order."""
        lib = _lib.load()
        h = ctypes.c_void_p()
        check(lib.svr_grid_load_sdgv(str(path).encode(), device, ctypes.byref(h)))
        return cls(0.0, _handle=h)

    def save(self, path: str) -> None:
        """save_grid (grid_io.cpp:37-58)."""
        check(self._lib.svr_grid_save_sdgv(self._h, str(path).encode()))

    def set_stream(self, stream) -> None:
        """Launch on a CUDA stream (torch.cuda.Stream or raw handle); None = own stream.

        Torch's legacy default stream (handle 0) maps to cudaStreamLegacy so that device
        inputs produced by torch on it are ordered before the library's kernels."""
        if stream is None:
            check(self._lib.svr_grid_set_stream(self._h, None))
            return
        handle = getattr(stream, "cuda_stream", stream)
        check(self._lib.svr_grid_set_stream(self._h, ctypes.c_void_p(handle if handle else 1)))

    def synchronize(self) -> None:
        check(self._lib.svr_grid_synchronize(self._h))

    def join(self) -> None:
        """Order the handle's stream after its pending internal work (a deferred zeroing; no host wait)."""
        check(self._lib.svr_grid_join(self._h))

    def set_lookup(self, mode: int) -> None:
        check(self._lib.svr_grid_set_lookup(self._h, mode))

    def set_tuning(self, key: str, value: int) -> None:
        check(self._lib.svr_grid_set_tuning(self._h, key.encode(), int(value)))

    # --- metadata (grid.hpp:109-120) -----------------------------------------
    def info(self) -> GridInfo:
        i = GridInfo()
        check(self._lib.svr_grid_get_info(self._h, ctypes.byref(i)))
        return i

    def voxel_size(self) -> float:
        return self._voxel_size

    def block_res(self) -> int:
        return self._block_res

    def label_channels(self) -> int:
        return self._label_channels

    def capacity(self) -> int:
        return self._capacity

    def block_extent(self) -> float:
        return self._voxel_size * self._block_res

    def block_count(self) -> int:
        return int(self.info().block_count)

    def empty(self) -> bool:
        return self.block_count() == 0

    def coords(self) -> np.ndarray:
        n = self.block_count()
        out = np.empty((n, 3), dtype=np.int32)
        if n:
            check(self._lib.svr_grid_coords(self._h, out.ctypes.data))
        return out

    def block_coord(self, i: int) -> tuple[int, int, int]:
        return tuple(int(v) for v in self.coords()[i])

    # --- allocation -------------------------------------------------------------
    def allocate_blocks(self, coords) -> np.ndarray:
        """allocate_block (grid.cpp:88-108) over coords[n][3], in order."""
        keep: list = []
        c = np.ascontiguousarray(coords, dtype=np.int32).reshape(-1, 3)
        idx = np.empty(len(c), dtype=np.uint32)
        check(self._lib.svr_grid_allocate_blocks(self._h, _in(c, np.int32, keep), len(c),
                                                 idx.ctypes.data))
        return idx

    def allocate_block(self, coord) -> int:
        return int(self.allocate_blocks(np.asarray(coord).reshape(1, 3))[0])

    def allocate_for_points(self, points, dilation: int) -> AllocReport:
        """allocate_for_points (allocation.cpp:45-54)."""
        keep: list = []
        pts = points if _is_tensor(points) else np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
        n = pts.shape[0] if pts.ndim > 1 else len(pts) // 3
        rep = AllocReport()
        st = self._lib.svr_grid_activate_points(self._h, _in(pts, np.float64, keep), n, dilation,
                                                ctypes.byref(rep))
        check(st, rep)
        return rep

    def allocate_for_frames(self, depth, cameras, dilation: int, scales=None) -> AllocReport:
        """allocate_for_frames (allocation.cpp:56-83): depth[F][H][W], cameras[F]."""
        keep: list = []
        cams = (Camera * len(cameras))(*cameras)
        sc_ptr, rows, cols = None, 0, 0
        if scales is not None:
            sc = np.ascontiguousarray(scales, dtype=np.float64)
            rows, cols = sc.shape[-2], sc.shape[-1]
            sc_ptr = _in(sc, np.float64, keep)
        rep = AllocReport()
        st = self._lib.svr_grid_activate_depth(self._h, _in(depth, np.float32, keep),
                                               ctypes.addressof(cams), len(cameras), sc_ptr, rows,
                                               cols, dilation, ctypes.byref(rep))
        check(st, rep)
        return rep

    def find(self, coords) -> np.ndarray:
        """find_block (grid.hpp:156) over coords[n][3]."""
        keep: list = []
        c = np.ascontiguousarray(coords, dtype=np.int32).reshape(-1, 3)
        out = np.empty(len(c), dtype=np.uint32)
        if len(c):
            check(self._lib.svr_grid_find(self._h, _in(c, np.int32, keep), len(c), out.ctypes.data))
        return out

    def find_block(self, coord) -> int:
        return int(self.find(np.asarray(coord).reshape(1, 3))[0])

    # --- payload ------------------------------------------------------------
    def set_payload(self, first: int, n: int, sdf=None, weight=None, rgb=None, logits=None) -> None:
        keep: list = []
        check(self._lib.svr_grid_set_payload(
            self._h, first, n, _in(sdf, np.float32, keep), _in(weight, np.float32, keep),
            _in(rgb, np.float32, keep), _in(logits, np.float32, keep)))

    def get_payload(self, first: int = 0, n: int | None = None) -> dict:
        n = self.block_count() - first if n is None else n
        C = self._label_channels
        out = {"sdf": np.empty((n, 512), np.float32), "weight": np.empty((n, 512), np.float32),
               "rgb": np.empty((n, 512, 3), np.float32), "logits": np.empty((n, 512, C), np.float32)}
        if n:
            check(self._lib.svr_grid_get_payload(self._h, first, n, out["sdf"].ctypes.data,
                                                 out["weight"].ctypes.data, out["rgb"].ctypes.data,
                                                 out["logits"].ctypes.data))
        return out

    # --- queries (grid.cpp:157-261) -----------------------------------------
    def query(self, points, logits: bool = False) -> dict:
        keep: list = []
        n = points.shape[0]
        like = points
        sdf, p_sdf = _out((n,), np.float64, like)
        grad, p_grad = _out((n, 3), np.float64, like)
        rgb, p_rgb = _out((n, 3), np.float64, like)
        lg, p_lg = _out((n, self._label_channels), np.float64, like) if logits else (None, None)
        valid, p_valid = _out((n,), np.uint8, like)
        if n:
            check(self._lib.svr_query(self._h, _in(points, np.float64, keep), n, p_sdf, p_grad, p_rgb,
                                      p_lg, p_valid))
        res = {"sdf": sdf, "grad": grad, "rgb": rgb, "valid": valid}
        if logits:
            res["logits"] = lg
        return res

    def query_sdf_with_gradient(self, x) -> tuple[bool, float, np.ndarray]:
        r = self.query(np.asarray(x, dtype=np.float64).reshape(1, 3))
        return bool(r["valid"][0]), float(r["sdf"][0]), r["grad"][0]

    def query_sdf(self, x) -> tuple[bool, float]:
        ok, s, _ = self.query_sdf_with_gradient(x)
        return ok, s

    # --- ray marching (grid.cpp:263-353) -------------------------------------------
    def march(self, origins, dirs, step: float, max_samples: int) -> dict:
        keep: list = []
        n = origins.shape[0]
        counts, pc = _out((n,), np.uint32, origins)
        t, pt = _out((n, max_samples), np.float64, origins)
        delta, pd = _out((n, max_samples), np.float64, origins)
        if n:
            check(self._lib.svr_march(self._h, _in(origins, np.float64, keep),
                                      _in(dirs, np.float64, keep), n, step, max_samples, pc, pt, pd))
        return {"counts": counts, "t": t, "delta": delta}

    def march_ray(self, origin, direction, step: float, max_samples: int):
        r = self.march(np.asarray(origin, np.float64).reshape(1, 3),
                       np.asarray(direction, np.float64).reshape(1, 3), step, max_samples)
        k = int(r["counts"][0])
        return r["t"][0, :k].copy(), r["delta"][0, :k].copy()

    # --- renderer ------------------------------------------
    def render_forward(self, origins, dirs, step: float, max_samples: int, beta: float,
                       out: dict | None = None) -> dict:
        keep: list = []
        n = origins.shape[0]
        if out is None:
            out = {}
            for k, shape in (("rgb", (n, 3)), ("depth", (n,)), ("normal", (n, 3)), ("wsum", (n,))):
                out[k], _ = _out(shape, np.float32, origins)
            out["n_samples"], _ = _out((n,), np.uint32, origins)
        ptr = {k: (v.data_ptr() if _is_tensor(v) else v.ctypes.data) if v is not None else None
               for k, v in out.items()}
        check(self._lib.svr_render_forward(self._h, _in(origins, np.float64, keep),
                                           _in(dirs, np.float64, keep), n, step, max_samples, beta,
                                           ptr.get("rgb"), ptr.get("depth"), ptr.get("normal"),
                                           ptr.get("wsum"), ptr.get("n_samples")))
        self._keep_rays = keep  # device ray buffers must outlive render_backward
        return out

    def render_backward(self, d_rgb, d_depth, d_normal) -> None:
        keep: list = []
        check(self._lib.svr_render_backward(self._h, _in(d_rgb, np.float32, keep),
                                            _in(d_depth, np.float32, keep),
                                            _in(d_normal, np.float32, keep)))
        self._keep_up = keep  # host_async: pinned inputs are read after the call returns

    def render_stats(self) -> RenderStats:
        s = RenderStats()
        check(self._lib.svr_render_get_stats(self._h, ctypes.byref(s)))
        return s

    # --- gradients / active blocks ---------------------------------------------
    def grad_zero(self) -> None:
        check(self._lib.svr_grad_zero(self._h))

    def grad_zero_active(self) -> None:
        check(self._lib.svr_grad_zero_active(self._h))

    def grads(self) -> tuple[np.ndarray, np.ndarray]:
        n = self.block_count()
        gs = np.empty((n, 512), np.float32)
        gr = np.empty((n, 512, 3), np.float32)
        if n:
            check(self._lib.svr_grad_get(self._h, gs.ctypes.data, gr.ctypes.data))
        return gs, gr

    def active_mask(self) -> np.ndarray:
        n = self.block_count()
        m = np.zeros(n, np.uint8)
        if n:
            check(self._lib.svr_active_blocks(self._h, m.ctypes.data, None, None))
        return m

    def active_blocks(self) -> np.ndarray:
        n = self.block_count()
        lst = np.empty(max(n, 1), np.uint32)
        cnt = ctypes.c_uint64()
        check(self._lib.svr_active_blocks(self._h, None, lst.ctypes.data, ctypes.addressof(cnt)))
        return lst[: cnt.value].copy()

    # --- losses / update around the path ------------------------------
    def sample_uniform(self, n: int, seed: int) -> np.ndarray:
        """sample_uniform (grid.cpp:355-370); counter-based device RNG, not mt19937_64."""
        out = np.empty((n, 3), np.float64)
        check(self._lib.svr_sample_uniform(self._h, n, seed, out.ctypes.data if n else None))
        return out

    def eikonal(self, points, scale: float = 1.0) -> tuple[float, int]:
        """Eikonal loss mean (|grad f| - 1)^2 over valid points; adds scale * dL/dsdf to the
        gradient plane.  Returns (loss, n_valid)."""
        keep: list = []
        loss = ctypes.c_double()
        nv = ctypes.c_uint64()
        n = points.shape[0]
        check(self._lib.svr_eikonal(self._h, _in(points, np.float64, keep), n, scale, ctypes.byref(loss),
                                    ctypes.byref(nv)))
        return loss.value, nv.value

    def rmsprop_step(self, lr: float, alpha: float = 0.99, eps: float = 1e-8) -> None:
        """RMSProp on active blocks, then zero their gradients."""
        check(self._lib.svr_rmsprop_step(self._h, lr, alpha, eps))

    # --- refinement losses ------------------------------------------
    def render_losses(self, out: dict, tgt_rgb, prior_depth=None, prior_normal=None, cam_idx=None,
                      cameras=None, lambda_d: float = 0.1, lambda_n: float = 0.05, grads: dict | None = None,
                      stats: bool = True):
        """Upstream gradients (d_rgb, d_depth, d_normal) of L_c + lambda_d L_d + lambda_n L_n for
        render_backward, from a render_forward output dict; see include/svr.h."""
        keep: list = []
        n = out["depth"].shape[0]
        like = out["depth"]
        if grads is None:
            grads = {}
            for k, shape in (("d_rgb", (n, 3)), ("d_depth", (n,)), ("d_normal", (n, 3))):
                grads[k], _ = _out(shape, np.float32, like)
        ptr = {k: (v.data_ptr() if _is_tensor(v) else v.ctypes.data) for k, v in grads.items()}
        cams = (Camera * max(len(cameras), 1))(*cameras) if cameras else None
        st = LossStats()
        check(self._lib.svr_render_losses(
            self._h, n, _in(out["rgb"], np.float32, keep), _in(out["depth"], np.float32, keep),
            _in(out["normal"], np.float32, keep), _in(out["wsum"], np.float32, keep),
            _in(tgt_rgb, np.float32, keep), _in(prior_depth, np.float32, keep),
            _in(prior_normal, np.float32, keep), _in(cam_idx, np.uint32, keep),
            ctypes.addressof(cams) if cams is not None else None, len(cameras) if cameras else 0,
            lambda_d, lambda_n, ptr["d_rgb"], ptr["d_depth"], ptr["d_normal"],
            ctypes.byref(st) if stats else None))
        return grads, ({f: getattr(st, f) for f, _ in LossStats._fields_} if stats else None)

    # --- fusion + de-noising -----------------------------------------
    def fuse_begin(self, color: bool = True, semantic: bool = True) -> None:
        """Open a fusion session (zeroed fixed-point sums); see include/svr.h."""
        check(self._lib.svr_fuse_begin(self._h, (1 if color else 0) | (2 if semantic else 0)))

    def fuse_frames(self, depth, cameras, mu: float, rgb=None, semantic=None, scales=None) -> FuseReport:
        """fuse_frame over depth[F][H][W] (+ rgb[F][H][W][3], semantic[F][H][W][C])."""
        keep: list = []
        cams = (Camera * len(cameras))(*cameras)
        sc_ptr, rows, cols = None, 0, 0
        if scales is not None:
            sc = np.ascontiguousarray(scales, dtype=np.float64)
            rows, cols = sc.shape[-2], sc.shape[-1]
            sc_ptr = _in(sc, np.float64, keep)
        rep = FuseReport()
        check(self._lib.svr_fuse_frames(self._h, _in(depth, np.float32, keep), _in(rgb, np.float32, keep),
                                        _in(semantic, np.float32, keep), ctypes.addressof(cams), len(cameras),
                                        sc_ptr, rows, cols, mu, ctypes.byref(rep)))
        return rep

    def fuse_finalize(self) -> None:
        check(self._lib.svr_fuse_finalize(self._h))

    def fuse_all(self, depth, cameras, mu: float, rgb=None, semantic=None, scales=None) -> FuseReport:
        """fuse_all: begin + every frame + finalize."""
        self.fuse_begin(rgb is not None, semantic is not None)
        rep = self.fuse_frames(depth, cameras, mu, rgb, semantic, scales)
        self.fuse_finalize()
        return rep

    def denoise(self, sigma_vox: float = 1.0, radius: int = 1) -> None:
        """denoise: separable Gaussian over the valid neighbourhood."""
        check(self._lib.svr_denoise(self._h, sigma_vox, radius))

    # --- meshing (meshing.cpp:168-273, mesh_io.cpp:30-68) ----------------------------------
    def marching_cubes(self, iso: float = 0.0) -> dict:
        """marching_cubes -> {vertices, normals, colors [nv,3] f64, labels [nv] i32,
        triangles [nt,3] i32} (the reference's Mesh)."""
        nv, nt = ctypes.c_uint64(), ctypes.c_uint64()
        check(self._lib.svr_marching_cubes(self._h, iso, ctypes.byref(nv), ctypes.byref(nt)))
        m = {"vertices": np.empty((nv.value, 3)), "normals": np.empty((nv.value, 3)),
             "colors": np.empty((nv.value, 3)), "labels": np.empty(nv.value, np.int32),
             "triangles": np.empty((nt.value, 3), np.int32)}
        check(self._lib.svr_mesh_get(self._h, *[m[k].ctypes.data if m[k].size else None for k in
                                               ("vertices", "normals", "colors", "labels", "triangles")]))
        return m

    def save_ply(self, path: str) -> None:
        """export_ply of the last marching_cubes mesh."""
        check(self._lib.svr_mesh_save_ply(self._h, str(path).encode()))

    def save_obj(self, path: str) -> None:
        """export_obj of the last marching_cubes mesh."""
        check(self._lib.svr_mesh_save_obj(self._h, str(path).encode()))

    # device-pointer plumbing for the multi-GPU reduction (paper_2305_13220_b200.distributed)
    def active_set_mask(self, mask) -> None:
        keep: list = []
        check(self._lib.svr_active_set_mask(self._h, _in(mask, np.uint8, keep)))

    def grad_pack(self, blocks, out) -> None:
        keep: list = []
        n = blocks.shape[0]
        check(self._lib.svr_grad_pack(self._h, _in(blocks, np.uint32, keep), n,
                                      out.data_ptr() if _is_tensor(out) else out.ctypes.data))

    def grad_unpack(self, blocks, packed) -> None:
        keep: list = []
        n = blocks.shape[0]
        check(self._lib.svr_grad_unpack(self._h, _in(blocks, np.uint32, keep), n,
                                        _in(packed, np.float32, keep)))
