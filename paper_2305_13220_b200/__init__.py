"""B200-native differentiable SDF volume rendering over the sparse-dense voxel-block grid.

Drop-in for the hot path of arXiv 2305.13220's reference (`svrecon`): block activation,
hash lookup, ray-block marching, trilinear SDF/gradient/color interpolation, Laplace
density compositing and the scatter-add backward.  Behind ``SparseDenseGrid`` is the
C-ABI of ``libsvr_b200.so`` (include/svr.h) and hand-written sm_100a kernels.
"""
from ._lib import (CapacityError, ConfigError, CudaError, DataError, DivergedError, SvrError,
                   SVR_INVALID_BLOCK, SVR_LOOKUP_AUTO, SVR_LOOKUP_DENSE, SVR_LOOKUP_HASH)
from .grid import SparseDenseGrid, camera

__all__ = ["SparseDenseGrid", "camera", "SvrError", "ConfigError", "DataError",
           "DivergedError", "CapacityError", "CudaError", "SVR_INVALID_BLOCK", "SVR_LOOKUP_AUTO",
           "SVR_LOOKUP_DENSE", "SVR_LOOKUP_HASH"]
