"""TEST INFRASTRUCTURE ONLY -- Python handles on the CPU checkers.

* ``OracleGrid``  -> liboracle.so, the C++ restatement (svr_oracle.cpp) of the reference
  grid / march / activation code plus the spec-restated renderer, fp64 throughout.
* ``RefGrid``     -> _ref/libsvr_ref.so, the reference's own sources
  (/root/reference/proj/src/core/{grid,allocation,camera,grid_io,scale_field,parallel}.cpp)
  compiled verbatim against shim/ (see Makefile), plus ref_capi.cpp's renderer on top.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product (paper_2305_13220_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from ctypes import POINTER, c_char_p, c_double, c_float, c_int, c_int32, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsvr_ref.so")
REF_TESTS = os.path.join(HERE, "_ref", "ref_tests")
REF_ROOT = "/root/reference/proj"


def build(ref: bool | None = None) -> None:
    """make liboracle.so (always) and _ref/* (when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_ROOT)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


class Report(ctypes.Structure):
    _fields_ = [("blocks_added", c_uint64), ("blocks_requested", c_uint64),
                ("pixels_used", c_uint64), ("unallocated", c_uint64)]


class OracleError(RuntimeError):
    def __init__(self, code, msg, report=None):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.report = report


P = c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a if shape is None else a.reshape(shape)


class _Base:
    _so = None
    _prefix = ""
    _protos: dict = {}
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            if not os.path.exists(cls._so):
                build()
            lib = ctypes.CDLL(cls._so)
            for name, (res, args) in cls._protos.items():
                fn = getattr(lib, cls._prefix + name)
                fn.restype = res
                fn.argtypes = args
            cls._lib = lib
        return cls._lib

    def _check(self, st, report=None):
        if st:
            msg = getattr(self.lib(), self._prefix + "last_error")().decode()
            raise OracleError(st, msg, report)

    def __del__(self):
        try:
            if self._h.value:
                getattr(self.lib(), self._prefix + "grid_destroy")(self._h)
        except Exception:
            pass

    def block_count(self) -> int:
        return int(getattr(self.lib(), self._prefix + "block_count")(self._h))

    def coords(self) -> np.ndarray:
        out = np.empty((self.block_count(), 3), np.int32)
        getattr(self.lib(), self._prefix + "coords")(self._h, _ptr(out))
        return out

    def allocate_blocks(self, coords) -> np.ndarray:
        c = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
        idx = np.empty(len(c), np.uint32)
        self._check(getattr(self.lib(), self._prefix + "allocate_blocks")(self._h, _ptr(c), len(c), _ptr(idx)))
        return idx

    def allocate_points(self, pts, dilation) -> Report:
        p = _f64(pts, (-1, 3))
        rep = Report()
        st = getattr(self.lib(), self._prefix + "allocate_points")(self._h, _ptr(p), len(p), dilation,
                                                                   ctypes.byref(rep))
        self._check(st, rep)
        return rep

    def allocate_frames(self, depth, cams, dilation, scales=None) -> Report:
        d = np.ascontiguousarray(depth, np.float32)
        arr = (_Cam * len(cams))(*[_Cam.from_any(c) for c in cams])
        sc = None if scales is None else np.ascontiguousarray(scales, np.float64)
        rows, cols = (0, 0) if sc is None else (sc.shape[-2], sc.shape[-1])
        rep = Report()
        st = getattr(self.lib(), self._prefix + "allocate_frames")(
            self._h, _ptr(d), ctypes.addressof(arr), len(cams), _ptr(sc), rows, cols, dilation,
            ctypes.byref(rep))
        self._check(st, rep)
        return rep

    def find(self, coords) -> np.ndarray:
        c = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
        out = np.empty(len(c), np.uint32)
        getattr(self.lib(), self._prefix + "find")(self._h, _ptr(c), len(c), _ptr(out))
        return out

    def set_payload(self, first, n, sdf=None, weight=None, rgb=None, logits=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)  # noqa: E731
        arrs = [f(sdf), f(weight), f(rgb), f(logits)]
        self._check(getattr(self.lib(), self._prefix + "set_payload")(self._h, first, n, *[_ptr(a) for a in arrs]))

    def march(self, o, d, step, max_samples):
        o, d = _f64(o, (-1, 3)), _f64(d, (-1, 3))
        n = len(o)
        counts = np.empty(n, np.uint32)
        t = np.zeros((n, max_samples), np.float64)
        delta = np.zeros((n, max_samples), np.float64)
        getattr(self.lib(), self._prefix + "march")(self._h, _ptr(o), _ptr(d), n, step, max_samples,
                                                    _ptr(counts), _ptr(t), _ptr(delta))
        return {"counts": counts, "t": t, "delta": delta}

    def get_payload(self, first=0, n=None):
        n = self.block_count() - first if n is None else n
        V = self.B ** 3
        out = {"sdf": np.empty((n, V), np.float32), "weight": np.empty((n, V), np.float32),
               "rgb": np.empty((n, V, 3), np.float32), "logits": np.empty((n, V, self.C), np.float32)}
        self._check(getattr(self.lib(), self._prefix + "get_payload")(self._h, first, n, *[_ptr(out[k]) for k in
                                                                     ("sdf", "weight", "rgb", "logits")]))
        return out


    def fuse_begin(self, color=True, semantic=True):
        self._check(getattr(self.lib(), self._prefix + "fuse_begin")(self._h, int(color) | (int(semantic) << 1)))

    def _fuse_args(self, depth, cams, rgb, sem, scales):
        d = np.ascontiguousarray(depth, np.float32)
        f = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)  # noqa: E731
        arr = (_Cam * len(cams))(*[_Cam.from_any(c) for c in cams])
        sc = None if scales is None else np.ascontiguousarray(scales, np.float64)
        rows, cols = (0, 0) if sc is None else (sc.shape[-2], sc.shape[-1])
        keep = (d, f(rgb), f(sem), sc, arr)
        return keep, [_ptr(d), _ptr(keep[1]), _ptr(keep[2]), ctypes.addressof(arr), len(cams), _ptr(sc),
                      rows, cols]

    def marching_cubes(self, iso=0.0) -> dict:
        """marching_cubes -> {vertices, normals, colors [nv,3] f64, labels [nv] i32,
        triangles [nt,3] i32}."""
        nv, nt = c_uint64(), c_uint64()
        self._check(getattr(self.lib(), self._prefix + "marching_cubes")(self._h, iso, ctypes.byref(nv),
                                                                          ctypes.byref(nt)))
        m = {"vertices": np.empty((nv.value, 3)), "normals": np.empty((nv.value, 3)),
             "colors": np.empty((nv.value, 3)), "labels": np.empty(nv.value, np.int32),
             "triangles": np.empty((nt.value, 3), np.int32)}
        getattr(self.lib(), self._prefix + "mesh_get")(self._h, *[_ptr(m[k]) for k in
                                                                  ("vertices", "normals", "colors", "labels",
                                                                   "triangles")])
        return m

    def fuse_finalize(self):
        self._check(getattr(self.lib(), self._prefix + "fuse_finalize")(self._h))

    def save(self, path):
        self._check(getattr(self.lib(), self._prefix + "save_sdgv")(self._h, str(path).encode()))


class _Cam(ctypes.Structure):
    _fields_ = [("fx", c_double), ("fy", c_double), ("cx", c_double), ("cy", c_double),
                ("width", c_int32), ("height", c_int32), ("R", c_double * 9), ("t", c_double * 3)]

    @classmethod
    def from_any(cls, c):
        out = cls()
        for k in ("fx", "fy", "cx", "cy", "width", "height"):
            setattr(out, k, getattr(c, k))
        out.R[:] = list(c.R)
        out.t[:] = list(c.t)
        return out


_COMMON = {
    "last_error": (c_char_p, []),
    "set_threads": (None, [c_int]),
    "grid_destroy": (None, [c_void_p]),
    "block_count": (c_uint64, [c_void_p]),
    "coords": (None, [c_void_p, P]),
    "allocate_blocks": (c_int, [c_void_p, P, c_uint64, P]),
    "allocate_points": (c_int, [c_void_p, P, c_uint64, c_int, POINTER(Report)]),
    "allocate_frames": (c_int, [c_void_p, P, P, c_uint32, P, c_int, c_int, c_int, POINTER(Report)]),
    "find": (None, [c_void_p, P, c_uint64, P]),
    "set_payload": (c_int, [c_void_p, c_uint32, c_uint32, P, P, P, P]),
    "march": (None, [c_void_p, P, P, c_uint64, c_double, c_uint32, P, P, P]),
    "save_sdgv": (c_int, [c_void_p, c_char_p]),
    "load_sdgv": (c_int, [c_char_p, POINTER(c_void_p)]),
    "get_payload": (c_int, [c_void_p, c_uint32, c_uint32, P, P, P, P]),
    "fuse_begin": (c_int, [c_void_p, c_int]),
    "marching_cubes": (c_int, [c_void_p, c_double, POINTER(c_uint64), POINTER(c_uint64)]),
    "mesh_get": (c_int, [c_void_p, P, P, P, P, P]),
    "fuse_finalize": (c_int, [c_void_p]),
}


class FuseReport(ctypes.Structure):
    _fields_ = [("frames", c_uint64), ("in_view", c_uint64), ("integrated", c_uint64),
                ("rejected", c_uint64)]


class OracleGrid(_Base):
    """The restated CPU oracle (svr_oracle.cpp)."""

    _so = ORACLE_SO
    _prefix = "svro_"
    _protos = dict(_COMMON, **{
        "grid_create": (c_int, [c_double, c_int, c_int, c_uint64, POINTER(c_void_p)]),
        "bounds": (c_int, [c_void_p, P, P]),
        "get_payload": (c_int, [c_void_p, c_uint32, c_uint32, P, P, P, P]),
        "query": (None, [c_void_p, P, c_uint64, P, P, P, P, P]),
        "render_forward": (c_int, [c_void_p, P, P, c_uint64, c_double, c_uint32, c_double, P, P, P, P, P, P]),
        "render_backward": (c_int, [c_void_p, P, P, c_uint64, c_double, c_uint32, c_double, P, P, P, P, P, P]),
        "sdf_to_density": (c_double, [c_double, c_double]),
        "eikonal": (c_int, [c_void_p, P, c_uint64, c_double, P, P, POINTER(c_double), POINTER(c_uint64)]),
        "rmsprop": (c_int, [c_void_p, P, P, P, c_float, c_float, c_float, P]),
        "fuse_frames": (c_int, [c_void_p, P, P, P, P, c_uint32, P, c_int, c_int, c_double, POINTER(FuseReport)]),
        "denoise": (c_int, [c_void_p, c_double, c_int]),
        "mc_table": (c_int, [P, P]),
        "fit_depth_affine": (c_int, [P, P, c_uint64, POINTER(c_double), POINTER(c_double)]),
        "render_losses": (c_int, [c_uint64, P, P, P, P, P, P, P, P, P, c_double, c_double, P, P, P, P]),
    })

    def __init__(self, voxel_size=0.015, block_res=8, label_channels=1, capacity=0, _handle=None):
        self.C = label_channels
        self.B = block_res
        if _handle is not None:
            self._h = _handle
            return
        h = c_void_p()
        self._check(self.lib().svro_grid_create(voxel_size, block_res, label_channels, capacity, ctypes.byref(h)))
        self._h = h

    @classmethod
    def load(cls, path, label_channels):
        h = c_void_p()
        st = cls.lib().svro_load_sdgv(str(path).encode(), ctypes.byref(h))
        if st:
            raise OracleError(st, cls.lib().svro_last_error().decode())
        return cls(label_channels=label_channels, _handle=h)

    @classmethod
    def set_threads(cls, n):
        cls.lib().svro_set_threads(n)

    @classmethod
    def density(cls, s, beta):
        return cls.lib().svro_sdf_to_density(s, beta)

    def bounds(self):
        lo = np.zeros(3, np.int32)
        hi = np.zeros(3, np.int32)
        st = self.lib().svro_bounds(self._h, _ptr(lo), _ptr(hi))
        return (lo, hi) if st == 0 else None

    def query(self, x, logits=False):
        x = _f64(x, (-1, 3))
        n = len(x)
        out = {"sdf": np.empty(n), "grad": np.empty((n, 3)), "rgb": np.empty((n, 3)),
               "valid": np.empty(n, np.uint8)}
        lg = np.empty((n, self.C)) if logits else None
        self.lib().svro_query(self._h, _ptr(x), n, _ptr(out["sdf"]), _ptr(out["grad"]), _ptr(out["rgb"]),
                              _ptr(lg), _ptr(out["valid"]))
        if logits:
            out["logits"] = lg
        return out

    def render_forward(self, o, d, step, max_samples, beta):
        o, d = _f64(o, (-1, 3)), _f64(d, (-1, 3))
        n = len(o)
        out = {"rgb": np.empty((n, 3)), "depth": np.empty(n), "normal": np.empty((n, 3)),
               "wsum": np.empty(n), "n_samples": np.empty(n, np.uint32), "n_valid": np.empty(n, np.uint32)}
        self._check(self.lib().svro_render_forward(self._h, _ptr(o), _ptr(d), n, step, max_samples, beta,
                                                   _ptr(out["rgb"]), _ptr(out["depth"]), _ptr(out["normal"]),
                                                   _ptr(out["wsum"]), _ptr(out["n_samples"]),
                                                   _ptr(out["n_valid"])))
        return out

    def grad_buffers(self):
        A, V = self.block_count(), self.B ** 3
        return np.zeros((A, V)), np.zeros((A, V, 3)), np.zeros(A, np.uint8)

    def render_backward(self, o, d, step, max_samples, beta, d_rgb, d_depth, d_normal, out=None):
        """Accumulates into `out` = (grad_sdf, grad_rgb, active) if given, else fresh zeros."""
        o, d = _f64(o, (-1, 3)), _f64(d, (-1, 3))
        n = len(o)
        gs, gr, active = self.grad_buffers() if out is None else out
        up = [_f64(d_rgb, (-1, 3)), _f64(d_depth, (-1,)), _f64(d_normal, (-1, 3))]
        self._check(self.lib().svro_render_backward(
            self._h, _ptr(o), _ptr(d), n, step, max_samples, beta, _ptr(up[0]), _ptr(up[1]),
            _ptr(up[2]), _ptr(gs), _ptr(gr), _ptr(active)))
        return gs, gr, active


def _eikonal(self, x, scale=1.0):
    """(loss, n_valid, grad_sdf[A,V], active[A]) of the restated Eikonal regulariser."""
    x = _f64(x, (-1, 3))
    A, V = self.block_count(), self.B ** 3
    gs = np.zeros((A, V))
    act = np.zeros(A, np.uint8)
    loss, nv = c_double(), c_uint64()
    self._check(self.lib().svro_eikonal(self._h, _ptr(x), len(x), scale, _ptr(gs), _ptr(act),
                                        ctypes.byref(loss), ctypes.byref(nv)))
    return loss.value, nv.value, gs, act


def _rmsprop(self, grad_sdf, grad_rgb, active, lr, alpha, eps, rms_state):
    arrs = [np.ascontiguousarray(grad_sdf, np.float64), np.ascontiguousarray(grad_rgb, np.float64),
            np.ascontiguousarray(active, np.uint8)]
    self._check(self.lib().svro_rmsprop(self._h, *[_ptr(a) for a in arrs], lr, alpha, eps, _ptr(rms_state)))


def _o_fuse_frames(self, depth, cams, mu, rgb=None, sem=None, scales=None) -> FuseReport:
    keep, args = self._fuse_args(depth, cams, rgb, sem, scales)
    rep = FuseReport()
    self._check(self.lib().svro_fuse_frames(self._h, *args, mu, ctypes.byref(rep)))
    del keep
    return rep


def _o_denoise(self, sigma_vox=1.0, radius=1):
    self._check(self.lib().svro_denoise(self._h, sigma_vox, radius))


def fit_depth_affine(t, D):
    """(a, b, singular) of the minibatch depth prior fit."""
    t, D = _f64(t), _f64(D)
    a, b = c_double(), c_double()
    sing = OracleGrid.lib().svro_fit_depth_affine(_ptr(t), _ptr(D), len(t), ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value, bool(sing)


def render_losses(out, tgt_rgb, prior_depth, prior_normal, cam_idx, cams, lambda_d=0.1, lambda_n=0.05):
    """Refinement losses + per-ray upstream gradients, fp64."""
    n = len(out["depth"])
    f = lambda a, dt=np.float32: None if a is None else np.ascontiguousarray(a, dt)  # noqa: E731
    arrs = [_f64(out["rgb"]), _f64(out["depth"]), _f64(out["normal"]), _f64(out["wsum"]),
            f(tgt_rgb), f(prior_depth), f(prior_normal), f(cam_idx, np.uint32)]
    camarr = (_Cam * len(cams))(*[_Cam.from_any(c) for c in cams])
    g = {"d_rgb": np.empty((n, 3)), "d_depth": np.empty(n), "d_normal": np.empty((n, 3))}
    stats = np.empty(10)
    st = OracleGrid.lib().svro_render_losses(n, *[_ptr(a) for a in arrs], ctypes.addressof(camarr), lambda_d,
                                             lambda_n, _ptr(g["d_rgb"]), _ptr(g["d_depth"]), _ptr(g["d_normal"]),
                                             _ptr(stats))
    if st:
        raise OracleError(st, OracleGrid.lib().svro_last_error().decode())
    keys = ("L_c", "L_d", "L_n", "total", "a", "b", "n_c", "n_d", "n_n", "singular")
    return g, dict(zip(keys, stats.tolist()))


OracleGrid.fuse_frames = _o_fuse_frames
OracleGrid.denoise = _o_denoise
OracleGrid.eikonal = _eikonal
OracleGrid.rmsprop = _rmsprop


class RefGrid(_Base):
    """The reference's own grid code compiled verbatim (oracle/_ref/libsvr_ref.so)."""

    _so = REF_SO
    _prefix = "svrr_"
    _protos = dict(_COMMON, **{
        "grid_create": (c_int, [c_double, c_int, c_int, c_uint64, POINTER(c_void_p)]),
        "worker_count": (c_int, []),
        "bounds": (c_int, [c_void_p, P, P]),
        "query": (None, [c_void_p, P, c_uint64, P, P, P, P]),
        "render_forward": (c_int, [c_void_p, P, P, c_uint64, c_double, c_uint32, c_double, P, P, P, P, P]),
        "render_backward": (c_int, [c_void_p, P, P, P]),
        "grad_get": (c_int, [c_void_p, P, P]),
        "fuse_frames": (c_int, [c_void_p, P, P, P, P, c_uint32, P, c_int, c_int, c_double]),
        "mesh_export_ply": (c_int, [c_void_p, c_char_p]),
        "mesh_area": (c_double, [c_void_p]),
        "mesh_export_obj": (c_int, [c_void_p, c_char_p]),
    })

    def export_obj(self, path):
        """export_obj (mesh_io.cpp:155-164) of the last marching_cubes mesh."""
        self._check(self.lib().svrr_mesh_export_obj(self._h, str(path).encode()))

    def export_ply(self, path):
        """export_ply (mesh_io.cpp:30-68) of the last marching_cubes mesh."""
        self._check(self.lib().svrr_mesh_export_ply(self._h, str(path).encode()))

    def fuse_frames(self, depth, cams, mu, rgb=None, sem=None, scales=None):
        keep, args = self._fuse_args(depth, cams, rgb, sem, scales)
        self._check(self.lib().svrr_fuse_frames(self._h, *args, mu))
        del keep

    def __init__(self, voxel_size=0.015, block_res=8, label_channels=1, capacity=0, _handle=None):
        self.C = label_channels
        self.B = block_res
        if _handle is not None:
            self._h = _handle
            return
        h = c_void_p()
        self._check(self.lib().svrr_grid_create(voxel_size, block_res, label_channels, capacity, ctypes.byref(h)))
        self._h = h

    @classmethod
    def load(cls, path, label_channels):
        h = c_void_p()
        st = cls.lib().svrr_load_sdgv(str(path).encode(), ctypes.byref(h))
        if st:
            raise OracleError(st, cls.lib().svrr_last_error().decode())
        return cls(label_channels=label_channels, _handle=h)

    @classmethod
    def set_threads(cls, n):
        cls.lib().svrr_set_threads(n)

    @classmethod
    def worker_count(cls):
        return cls.lib().svrr_worker_count()

    def query(self, x):
        x = _f64(x, (-1, 3))
        n = len(x)
        out = {"sdf": np.empty(n), "grad": np.empty((n, 3)), "rgb": np.empty((n, 3)),
               "valid": np.empty(n, np.uint8)}
        self.lib().svrr_query(self._h, _ptr(x), n, _ptr(out["sdf"]), _ptr(out["grad"]), _ptr(out["rgb"]),
                              _ptr(out["valid"]))
        return out

    def render_forward(self, o, d, step, max_samples, beta):
        o, d = _f64(o, (-1, 3)), _f64(d, (-1, 3))
        n = len(o)
        out = {"rgb": np.empty((n, 3), np.float32), "depth": np.empty(n, np.float32),
               "normal": np.empty((n, 3), np.float32), "wsum": np.empty(n, np.float32),
               "n_valid": np.empty(n, np.uint32)}
        self._check(self.lib().svrr_render_forward(self._h, _ptr(o), _ptr(d), n, step, max_samples, beta,
                                                   _ptr(out["rgb"]), _ptr(out["depth"]), _ptr(out["normal"]),
                                                   _ptr(out["wsum"]), _ptr(out["n_valid"])))
        return out

    def render_backward(self, d_rgb, d_depth, d_normal):
        up = [np.ascontiguousarray(a, np.float32) for a in (d_rgb, d_depth, d_normal)]
        self._check(self.lib().svrr_render_backward(self._h, *[_ptr(a) for a in up]))

    def grads(self):
        A, V = self.block_count(), self.B ** 3
        gs = np.empty((A, V), np.float32)
        gr = np.empty((A, V, 3), np.float32)
        self.lib().svrr_grad_get(self._h, _ptr(gs), _ptr(gr))
        return gs, gr


class RefScene:
    """The reference's own SyntheticScene (synthetic.cpp, compiled verbatim into
    _ref/libsvr_ref.so) behind the interface of fixtures.SyntheticScene: the --impl reference
    bench arm builds every input with it, and tests pin the fixture restatement to it."""

    class Spec(ctypes.Structure):
        _fields_ = [("room_w", c_double), ("room_d", c_double), ("room_h", c_double),
                    ("n_objects", c_int32), ("n_frames", c_int32), ("width", c_int32),
                    ("height", c_int32), ("fov_deg", c_double), ("label_channels", c_int32),
                    ("texture_amplitude", c_double), ("texture_frequency", c_double),
                    ("seed", c_uint64)]

    # synthetic.hpp:13-30 defaults (the fields the harness sets)
    DEFAULTS = dict(room_w=2.4, room_d=2.2, room_h=2.0, n_objects=2, n_frames=24, width=320, height=240,
                    fov_deg=70.0, label_channels=4, texture_amplitude=0.25, texture_frequency=4.0, seed=1)

    _protos = {
        "scene_create": (c_int, [P, POINTER(c_void_p)]),
        "scene_destroy": (None, [c_void_p]),
        "scene_camera": (c_int, [c_void_p, c_int32, P]),
        "scene_frames": (c_int, [c_void_p, P, c_uint32, P, P, P, c_int32, P, c_int32]),
        "scene_sdf": (c_int, [c_void_p, P, c_uint64, P]),
        "scene_fill_payload": (c_int, [c_void_p, c_double, c_int32, c_int32, c_double, P, c_uint64,
                                       P, P, P, P, c_int32]),
        "scene_rays": (c_int, [c_void_p, c_uint32, c_uint32, c_uint64, P, P]),
        "scene_image_rays": (c_int, [c_void_p, c_int32, P, P]),
        "uniform_floats": (c_int, [c_uint64, c_uint64, c_float, c_float, P]),
    }
    _bound = False

    @classmethod
    def lib(cls):
        lib = RefGrid.lib()
        if not cls._bound:
            for name, (res, args) in cls._protos.items():
                fn = getattr(lib, "svrr_" + name)
                fn.restype, fn.argtypes = res, args
            cls._bound = True
        return lib

    def __init__(self, **spec):
        vals = dict(self.DEFAULTS)
        for k, v in spec.items():
            if k not in vals:
                raise TypeError(f"unknown SceneSpec field {k}")
            vals[k] = v
        self.spec = self.Spec(**vals)
        h = c_void_p()
        self._check(self.lib().svrr_scene_create(ctypes.addressof(self.spec), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h.value:
                self.lib().svrr_scene_destroy(self._h)
        except Exception:
            pass

    def _check(self, st):
        if st:
            raise OracleError(st, self.lib().svrr_last_error().decode())

    def camera_for_frame(self, frame: int):
        c = _Cam()  # the svr_camera layout; the product package is never imported here
        self._check(self.lib().svrr_scene_camera(self._h, frame, ctypes.addressof(c)))
        return c

    def cameras(self, n=None):
        n = self.spec.n_frames if n is None else n
        return [self.camera_for_frame(f) for f in range(n)]

    def frames(self, cams, threads=0, label_channels=None, normals=False, what=("depth", "rgb", "sem")):
        C = self.spec.label_channels if label_channels is None else label_channels
        F, H, W = len(cams), self.spec.height, self.spec.width
        arr = (_Cam * F)(*[_Cam.from_any(c) for c in cams])
        out = {"depth": np.empty((F, H, W), np.float32) if "depth" in what else None,
               "rgb": np.empty((F, H, W, 3), np.float32) if "rgb" in what else None,
               "sem": np.empty((F, H, W, C), np.float32) if "sem" in what else None,
               "normal": np.empty((F, H, W, 3), np.float32) if normals else None}
        self._check(self.lib().svrr_scene_frames(self._h, ctypes.addressof(arr), F, _ptr(out["depth"]),
                                                 _ptr(out["rgb"]), _ptr(out["sem"]), C, _ptr(out["normal"]),
                                                 threads))
        res = tuple(out[k] for k in ("depth", "rgb", "sem") if k in what)
        return res + (out["normal"],) if normals else res

    def depth(self, cams, threads=0):
        return self.frames(cams, threads, what=("depth",))[0]

    def sdf(self, x):
        x = _f64(x, (-1, 3))
        out = np.empty(len(x))
        self._check(self.lib().svrr_scene_sdf(self._h, _ptr(x), len(x), _ptr(out)))
        return out

    def fill_payload(self, voxel_size, coords, trunc, label_channels, block_res=8, threads=0):
        c = np.ascontiguousarray(coords, np.int32).reshape(-1, 3)
        n, V = len(c), block_res ** 3
        out = {"sdf": np.empty((n, V), np.float32), "weight": np.empty((n, V), np.float32),
               "rgb": np.empty((n, V, 3), np.float32), "logits": np.empty((n, V, label_channels), np.float32)}
        self._check(self.lib().svrr_scene_fill_payload(self._h, voxel_size, block_res, label_channels, trunc,
                                                       _ptr(c), n, _ptr(out["sdf"]), _ptr(out["weight"]),
                                                       _ptr(out["rgb"]), _ptr(out["logits"]), threads))
        return out

    def rays(self, n_poses, rays_per_pose, seed=0):
        n = n_poses * rays_per_pose
        o, d = np.empty((n, 3)), np.empty((n, 3))
        self._check(self.lib().svrr_scene_rays(self._h, n_poses, rays_per_pose, seed, _ptr(o), _ptr(d)))
        return o, d

    def image_rays(self, frame):
        n = self.spec.width * self.spec.height
        o, d = np.empty((n, 3)), np.empty((n, 3))
        self._check(self.lib().svrr_scene_image_rays(self._h, frame, _ptr(o), _ptr(d)))
        return o, d

    @classmethod
    def uniform_floats(cls, n, seed, lo=-1.0, hi=1.0):
        out = np.empty(n, np.float32)
        cls.lib().svrr_uniform_floats(n, seed, lo, hi, _ptr(out))
        return out
