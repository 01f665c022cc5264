"""ctypes binding of libsvr_b200.so (include/svr.h).

The shared library is built in-tree by ``paper_2305_13220_b200.build.build()`` (called
from ``__graft_entry__.build()``).  Loading fails loudly when it is missing: there is
no CPU fallback for any entry point.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_float, c_int32, c_uint8, c_uint32, c_uint64, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
# SVR_LIB_VARIANT=name loads libsvr_b200.<name>.so instead (side-by-side A/B builds of the
# same sources made by profiles/ab_build.sh; never set by the tests, smoke() or bench runs)
_VARIANT = os.environ.get("SVR_LIB_VARIANT", "")
LIB_PATH = os.path.join(HERE, f"libsvr_b200.{_VARIANT}.so" if _VARIANT else "libsvr_b200.so")

SVR_OK = 0
SVR_ERR_CONFIG = 2
SVR_ERR_DATA = 3
SVR_ERR_DIVERGED = 4
SVR_ERR_CAPACITY = 5
SVR_ERR_CUDA = 6
SVR_INVALID_BLOCK = 0xFFFFFFFF
SVR_LOOKUP_AUTO, SVR_LOOKUP_HASH, SVR_LOOKUP_DENSE = 0, 1, 2


class SvrError(RuntimeError):
    """Base of the status-code exceptions (proj/src/core/errors.hpp:8-31)."""

    code = -1


class ConfigError(SvrError):
    code = SVR_ERR_CONFIG


class DataError(SvrError):
    code = SVR_ERR_DATA


class DivergedError(SvrError):
    code = SVR_ERR_DIVERGED


class CapacityError(SvrError):
    code = SVR_ERR_CAPACITY

    def __init__(self, msg: str, unallocated_blocks: int = 0):
        super().__init__(msg)
        self.unallocated_blocks = unallocated_blocks


class CudaError(SvrError):
    code = SVR_ERR_CUDA


_ERRORS = {c.code: c for c in (ConfigError, DataError, DivergedError, CapacityError, CudaError)}


class Camera(ctypes.Structure):
    """svr_camera: pinhole camera, camera-to-world x_w = R x_c + t (camera.hpp:16-29)."""

    _fields_ = [("fx", c_double), ("fy", c_double), ("cx", c_double), ("cy", c_double),
                ("width", c_int32), ("height", c_int32), ("R", c_double * 9), ("t", c_double * 3)]


class AllocReport(ctypes.Structure):
    _fields_ = [("blocks_added", c_uint64), ("blocks_requested", c_uint64),
                ("pixels_used", c_uint64), ("unallocated", c_uint64)]


class GridInfo(ctypes.Structure):
    _fields_ = [("voxel_size", c_double), ("block_res", c_int32), ("label_channels", c_int32),
                ("capacity", c_uint64), ("block_count", c_uint64), ("hash_slots", c_uint64),
                ("bounds_lo", c_int32 * 3), ("bounds_hi", c_int32 * 3), ("lookup_mode", c_int32),
                ("device", c_int32), ("device_bytes", c_uint64)]


class RenderStats(ctypes.Structure):
    _fields_ = [("rays", c_uint64), ("samples", c_uint64), ("valid_samples", c_uint64)]


class FuseReport(ctypes.Structure):
    _fields_ = [("frames", c_uint64), ("in_view", c_uint64), ("integrated", c_uint64),
                ("rejected", c_uint64)]


class LossStats(ctypes.Structure):
    _fields_ = [("L_c", c_double), ("L_d", c_double), ("L_n", c_double), ("total", c_double),
                ("a", c_double), ("b", c_double), ("n_c", c_uint64), ("n_d", c_uint64), ("n_n", c_uint64),
                ("singular", c_int32)]


class RefineConfig(ctypes.Structure):
    _fields_ = [("rays_per_image", c_uint32), ("images_per_batch", c_uint32), ("lambda_d", c_double),
                ("lambda_n", c_double), ("lambda_eik", c_double), ("lr", c_double), ("gamma", c_double),
                ("alpha", c_double), ("eps", c_double), ("max_samples", c_uint32), ("uniform_points", c_uint32),
                ("band_cap", c_uint32), ("seed", c_uint64), ("step", c_double), ("beta", c_double),
                ("mu", c_double)]


class PeerExport(ctypes.Structure):
    """svr_peer_export: IPC handles of one rank's gradient plane, active flags and phase events."""

    _fields_ = [("grad", ctypes.c_uint8 * 64), ("active", ctypes.c_uint8 * 64), ("ev_done", ctypes.c_uint8 * 64),
                ("ev_reduced", ctypes.c_uint8 * 64), ("n_blocks", c_uint64), ("device", c_int32),
                ("reserved", c_int32)]


SVR_REDUCE_AUTO, SVR_REDUCE_PEER, SVR_REDUCE_NCCL = 0, 1, 2
SVR_REDUCE_PUBLISH, SVR_REDUCE_SUM, SVR_REDUCE_ADOPT = 0, 1, 2

P = c_void_p  # every array argument: host or device address
_I = c_int32

_PROTOS = {
    "svr_last_error": (c_char_p, []),
    "svr_abi_version": (_I, []),
    "svr_device_count": (_I, [POINTER(c_int32)]),
    "svr_grid_create": (_I, [c_double, c_int32, c_int32, c_uint64, c_int32, POINTER(c_void_p)]),
    "svr_grid_destroy": (_I, [c_void_p]),
    "svr_grid_set_stream": (_I, [c_void_p, c_void_p]),
    "svr_grid_synchronize": (_I, [c_void_p]),
    "svr_grid_join": (_I, [c_void_p]),
    "svr_grid_get_info": (_I, [c_void_p, POINTER(GridInfo)]),
    "svr_grid_set_lookup": (_I, [c_void_p, c_int32]),
    "svr_grid_set_tuning": (_I, [c_void_p, c_char_p, ctypes.c_int64]),
    "svr_grid_load_sdgv": (_I, [c_char_p, c_int32, POINTER(c_void_p)]),
    "svr_grid_save_sdgv": (_I, [c_void_p, c_char_p]),
    "svr_grid_allocate_blocks": (_I, [c_void_p, P, c_uint64, P]),
    "svr_grid_activate_points": (_I, [c_void_p, P, c_uint64, c_int32, POINTER(AllocReport)]),
    "svr_grid_activate_depth": (_I, [c_void_p, P, P, c_uint32, P, c_int32, c_int32, c_int32,
                                     POINTER(AllocReport)]),
    "svr_grid_find": (_I, [c_void_p, P, c_uint64, P]),
    "svr_grid_coords": (_I, [c_void_p, P]),
    "svr_grid_set_payload": (_I, [c_void_p, c_uint32, c_uint32, P, P, P, P]),
    "svr_grid_get_payload": (_I, [c_void_p, c_uint32, c_uint32, P, P, P, P]),
    "svr_query": (_I, [c_void_p, P, c_uint64, P, P, P, P, P]),
    "svr_march": (_I, [c_void_p, P, P, c_uint64, c_double, c_uint32, P, P, P]),
    "svr_render_forward": (_I, [c_void_p, P, P, c_uint64, c_double, c_uint32, c_double, P, P, P,
                                P, P]),
    "svr_render_backward": (_I, [c_void_p, P, P, P]),
    "svr_render_get_stats": (_I, [c_void_p, POINTER(RenderStats)]),
    "svr_grad_zero": (_I, [c_void_p]),
    "svr_grad_get": (_I, [c_void_p, P, P]),
    "svr_active_blocks": (_I, [c_void_p, P, P, P]),
    "svr_active_set_mask": (_I, [c_void_p, P]),
    "svr_grad_pack": (_I, [c_void_p, P, c_uint64, P]),
    "svr_grad_unpack": (_I, [c_void_p, P, c_uint64, P]),
    "svr_grad_zero_active": (_I, [c_void_p]),
    "svr_sample_uniform": (_I, [c_void_p, c_uint64, c_uint64, P]),
    "svr_eikonal": (_I, [c_void_p, P, c_uint64, c_double, POINTER(c_double), POINTER(c_uint64)]),
    "svr_rmsprop_step": (_I, [c_void_p, c_float, c_float, c_float]),
    "svr_fuse_begin": (_I, [c_void_p, c_int32]),
    "svr_fuse_frames": (_I, [c_void_p, P, P, P, P, c_uint32, P, c_int32, c_int32, c_double,
                             POINTER(FuseReport)]),
    "svr_fuse_finalize": (_I, [c_void_p]),
    "svr_denoise": (_I, [c_void_p, c_double, c_int32]),
    "svr_grad_ipc_handle": (_I, [c_void_p, P, POINTER(c_uint64)]),
    "svr_grad_plane": (_I, [c_void_p, POINTER(c_void_p), POINTER(c_uint64)]),
    "svr_ipc_open": (_I, [P, c_int32, POINTER(c_void_p)]),
    "svr_ipc_close": (_I, [c_void_p]),
    "svr_grad_peer_allreduce": (_I, [c_void_p, P, c_uint32, c_uint32, P, c_uint64]),
    "svr_reduce_grads": (_I, [P, c_uint32]),
    "svr_reduce_grads_ex": (_I, [P, c_uint32, c_int32]),
    "svr_peer_export_get": (_I, [c_void_p, POINTER(PeerExport)]),
    "svr_peer_group_open": (_I, [c_void_p, P, c_uint32, c_uint32, POINTER(c_void_p)]),
    "svr_peer_reduce_phase": (_I, [c_void_p, c_int32]),
    "svr_peer_group_close": (_I, [c_void_p]),
    "svr_render_losses": (_I, [c_void_p, c_uint64, P, P, P, P, P, P, P, P, P, c_uint32, c_double, c_double,
                               P, P, P, POINTER(LossStats)]),
    "svr_sample_frame_rays": (_I, [c_void_p, P, c_uint32, P, P, P, c_uint32, c_uint32, c_uint64, P, P, P, P, P, P,
                                   P]),
    "svr_band_points": (_I, [c_void_p, c_double, c_uint64, P, POINTER(c_uint64)]),
    "svr_refine_config_default": (None, [POINTER(RefineConfig)]),
    "svr_refiner_create": (_I, [c_void_p, P, c_uint32, P, P, P, POINTER(RefineConfig), POINTER(c_void_p)]),
    "svr_refiner_step": (_I, [c_void_p, c_uint32, c_uint32, POINTER(LossStats), POINTER(c_double)]),
    "svr_refiner_destroy": (_I, [c_void_p]),
    "svr_marching_cubes": (_I, [c_void_p, c_double, POINTER(c_uint64), POINTER(c_uint64)]),
    "svr_mesh_get": (_I, [c_void_p, P, P, P, P, P]),
    "svr_mesh_save_ply": (_I, [c_void_p, c_char_p]),
    "svr_mesh_save_obj": (_I, [c_void_p, c_char_p]),
}

EXPORTED = tuple(_PROTOS)

_lib = None


def load() -> ctypes.CDLL:
    """Load libsvr_b200.so; raises ImportError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, report: AllocReport | None = None) -> None:
    """Raise the exception class mirroring the reference's for a non-zero status."""
    if status == SVR_OK:
        return
    msg = (load().svr_last_error() or b"").decode(errors="replace")
    cls = _ERRORS.get(status, SvrError)
    if cls is CapacityError:
        raise CapacityError(msg, int(report.unallocated) if report is not None else 0)
    raise cls(msg)
