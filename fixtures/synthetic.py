"""Synthetic analytic-SDF scene fixtures (fixtures/svr_synth.h; host-only, no GPU needed).

Restates the reference's SyntheticScene (proj/src/core/synthetic.cpp:42-192) and the
input recipes of SURVEY.md 8(d): GT depth frames for activation, clamped-SDF payloads,
random-pixel rays from ring poses and U(-1,1) upstream gradients.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int32, c_uint32, c_uint64, c_void_p

import numpy as np

from paper_2305_13220_b200._lib import Camera, SvrError, _ERRORS

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsvr_fixture.so")


class SceneSpec(ctypes.Structure):
    """svr_scene_spec (synthetic.hpp:13-30)."""

    _fields_ = [("room_w", c_double), ("room_d", c_double), ("room_h", c_double),
                ("n_objects", c_int32), ("n_frames", c_int32), ("width", c_int32),
                ("height", c_int32), ("fov_deg", c_double), ("label_channels", c_int32),
                ("texture_amplitude", c_double), ("texture_frequency", c_double),
                ("seed", c_uint64)]


P, _I = c_void_p, c_int32
_PROTOS = {
    "svr_fixture_last_error": (c_char_p, []),
    "svr_scene_spec_default": (None, [POINTER(SceneSpec)]),
    "svr_scene_create": (_I, [POINTER(SceneSpec), POINTER(c_void_p)]),
    "svr_scene_destroy": (None, [c_void_p]),
    "svr_scene_camera": (_I, [c_void_p, c_int32, POINTER(Camera)]),
    "svr_scene_depth": (_I, [c_void_p, P, c_uint32, P, c_int32]),
    "svr_scene_frames": (_I, [c_void_p, P, c_uint32, P, P, P, c_int32, P, c_int32]),
    "svr_scene_sdf": (_I, [c_void_p, P, c_uint64, P]),
    "svr_scene_fill_payload": (_I, [c_void_p, c_double, c_int32, c_int32, c_double, P, c_uint64,
                                    P, P, P, P, c_int32]),
    "svr_scene_rays": (_I, [c_void_p, c_uint32, c_uint32, c_uint64, P, P]),
    "svr_scene_image_rays": (_I, [c_void_p, c_int32, P, P]),
    "svr_uniform_floats": (_I, [c_uint64, c_uint64, c_float, c_float, P]),
}
_lib_handle = None


def load() -> ctypes.CDLL:
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            from . import build

            build.build()
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _lib_handle = lib
    return _lib_handle


def check(status: int) -> None:
    if status:
        msg = (load().svr_fixture_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(status, SvrError)(msg)


class SyntheticScene:
    def __init__(self, **spec):
        self._lib = load()
        s = SceneSpec()
        self._lib.svr_scene_spec_default(ctypes.byref(s))
        for k, v in spec.items():
            if not hasattr(s, k):
                raise TypeError(f"unknown SceneSpec field {k}")
            setattr(s, k, v)
        self.spec = s
        h = ctypes.c_void_p()
        check(self._lib.svr_scene_create(ctypes.byref(s), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h.value:
                self._lib.svr_scene_destroy(self._h)
        except Exception:
            pass

    def camera_for_frame(self, frame: int) -> Camera:
        c = Camera()
        check(self._lib.svr_scene_camera(self._h, frame, ctypes.byref(c)))
        return c

    def cameras(self, n: int | None = None) -> list[Camera]:
        n = self.spec.n_frames if n is None else n
        return [self.camera_for_frame(f) for f in range(n)]

    def depth(self, cams: list[Camera], threads: int = 0) -> np.ndarray:
        arr = (Camera * len(cams))(*cams)
        out = np.empty((len(cams), self.spec.height, self.spec.width), np.float32)
        check(self._lib.svr_scene_depth(self._h, ctypes.addressof(arr), len(cams), out.ctypes.data,
                                        threads))
        return out

    def frames(self, cams: list[Camera], threads: int = 0, label_channels: int | None = None,
               normals: bool = False):
        """(depth[F][H][W], rgb[F][H][W][3], semantic[F][H][W][C]) as generate_dataset renders
        them (synthetic.cpp:318-340): GT z-depth, scene colour at the hit, one-hot hit label;
        with normals=True also the camera-frame normal map [F][H][W][3]."""
        C = self.spec.label_channels if label_channels is None else label_channels
        arr = (Camera * len(cams))(*cams)
        F, H, W = len(cams), self.spec.height, self.spec.width
        depth = np.empty((F, H, W), np.float32)
        rgb = np.empty((F, H, W, 3), np.float32)
        sem = np.empty((F, H, W, C), np.float32)
        nrm = np.empty((F, H, W, 3), np.float32) if normals else None
        check(self._lib.svr_scene_frames(self._h, ctypes.addressof(arr), F, depth.ctypes.data,
                                         rgb.ctypes.data, sem.ctypes.data, C,
                                         nrm.ctypes.data if normals else None, threads))
        return (depth, rgb, sem, nrm) if normals else (depth, rgb, sem)

    def sdf(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64).reshape(-1, 3)
        out = np.empty(len(x), np.float64)
        check(self._lib.svr_scene_sdf(self._h, x.ctypes.data, len(x), out.ctypes.data))
        return out

    def fill_payload(self, voxel_size: float, coords, trunc: float, label_channels: int,
                     block_res: int = 8, threads: int = 0) -> dict:
        c = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
        n, V = len(c), block_res ** 3
        out = {"sdf": np.empty((n, V), np.float32), "weight": np.empty((n, V), np.float32),
               "rgb": np.empty((n, V, 3), np.float32),
               "logits": np.empty((n, V, label_channels), np.float32)}
        check(self._lib.svr_scene_fill_payload(
            self._h, voxel_size, block_res, label_channels, trunc, c.ctypes.data, n,
            out["sdf"].ctypes.data, out["weight"].ctypes.data, out["rgb"].ctypes.data,
            out["logits"].ctypes.data, threads))
        return out

    def rays(self, n_poses: int, rays_per_pose: int, seed: int = 0) -> tuple[np.ndarray, np.ndarray]:
        n = n_poses * rays_per_pose
        o = np.empty((n, 3), np.float64)
        d = np.empty((n, 3), np.float64)
        check(self._lib.svr_scene_rays(self._h, n_poses, rays_per_pose, seed, o.ctypes.data,
                                       d.ctypes.data))
        return o, d

    def image_rays(self, frame: int) -> tuple[np.ndarray, np.ndarray]:
        n = self.spec.width * self.spec.height
        o = np.empty((n, 3), np.float64)
        d = np.empty((n, 3), np.float64)
        check(self._lib.svr_scene_image_rays(self._h, frame, o.ctypes.data, d.ctypes.data))
        return o, d


def uniform_floats(n: int, seed: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    out = np.empty(n, np.float32)
    check(load().svr_uniform_floats(n, seed, lo, hi, out.ctypes.data))
    return out
