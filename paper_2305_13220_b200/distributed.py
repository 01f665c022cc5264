"""Multi-GPU active-block gradient reduction (kernels K7/K8).

Rays are sharded across ranks with the grid replicated; after each rank's backward the
voxel gradients must be summed.  Only blocks touched by some rank carry gradient, so:

  1. active mask  u8[A]   -> all_reduce(MAX)      (union of touched blocks)
  2. compaction           -> ascending block list, identical on every rank (K7)
  3. pack  [n,512,4] fp32 -> all_reduce(SUM)      (NCCL over NVLink, K8)
  4. unpack into the gradient planes

``reduce_active_grads`` drives steps 1-4 for a ``SparseDenseGrid`` whose kernels run on
torch's current stream (grid.set_stream), so NCCL and the pack/unpack kernels are
stream-ordered; it reads the active count on the host.  ``PeerGradReducer`` (one process per
GPU) and ``reduce_grads`` (one process, one handle per GPU) do the whole reduction on the
devices with no host synchronisation (csrc/svr_reduce.cu).  The collective sequence itself is ``allreduce_active`` and is backend
agnostic, which lets tests exercise it with gloo on CPU tensors.
"""
from __future__ import annotations

from typing import Protocol

import torch
import torch.distributed as dist


class ActiveGradStore(Protocol):
    """What the collective sequence needs from a gradient holder."""

    def mask_tensor(self) -> torch.Tensor: ...           # u8[A] touched blocks (this rank)
    def set_mask(self, mask: torch.Tensor) -> None: ...  # adopt the union mask
    def active_list(self) -> torch.Tensor: ...           # int32[n] ascending block ids
    def pack(self, blocks: torch.Tensor) -> torch.Tensor: ...        # -> f32[n,512,4]
    def unpack(self, blocks: torch.Tensor, packed: torch.Tensor) -> None: ...


def allreduce_active(store: ActiveGradStore, group=None) -> torch.Tensor:
    mask = store.mask_tensor()
    dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=group)
    store.set_mask(mask)
    blocks = store.active_list()
    if blocks.numel() == 0:
        return blocks
    packed = store.pack(blocks)
    dist.all_reduce(packed, op=dist.ReduceOp.SUM, group=group)
    store.unpack(blocks, packed)
    return blocks


class _GridStore:
    """ActiveGradStore over a device SparseDenseGrid (all buffers stay in HBM)."""

    def __init__(self, grid, device):
        self.grid = grid
        self.device = device

    def mask_tensor(self):
        n = self.grid.block_count()
        m = torch.empty(n, dtype=torch.uint8, device=self.device)
        if n:
            from ._lib import check

            check(self.grid._lib.svr_active_blocks(self.grid._h, m.data_ptr(), None, None))
        return m

    def set_mask(self, mask):
        self.grid.active_set_mask(mask)

    def active_list(self):
        import ctypes

        from ._lib import check

        n = self.grid.block_count()
        lst = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        cnt = ctypes.c_uint64()
        check(self.grid._lib.svr_active_blocks(self.grid._h, None, lst.data_ptr(), ctypes.addressof(cnt)))
        return lst[: cnt.value]

    def pack(self, blocks):
        out = torch.empty((blocks.numel(), 512, 4), dtype=torch.float32, device=self.device)
        self.grid.grad_pack(blocks, out)
        return out

    def unpack(self, blocks, packed):
        self.grid.grad_unpack(blocks, packed)


class PeerGradReducer:
    """The fused alternative to steps 1-4 (K8r, csrc/svr_reduce.cu), free of device
    synchronisation: every rank exports its gradient plane, active flags and two
    interprocess events (CUDA IPC), maps the other ranks', and one reduction is three
    stream-ordered phases on the grid's own stream -- publish (record "done"), sum (wait every
    rank's "done", union of the flags by peer reads, ascending compaction, this rank's 1/world
    slice of the rows summed over all planes in rank order and stored into every plane, record
    "reduced"), adopt (wait every rank's "reduced", take the union active set).  Between the
    phases the ranks meet at a host barrier on a gloo group, so every rank has recorded an
    event before another waits on it; no phase synchronises a device or reads a count on the
    host, so the host keeps queueing work ahead of the GPU.  Construct after the grid has all
    its blocks (the mapped planes must not be reallocated)."""

    def __init__(self, grid, device, group=None):
        import ctypes

        from ._lib import PeerExport, check

        self.grid, self.device, self.group = grid, torch.device(device), group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 8:
            raise ValueError("PeerGradReducer: at most 8 ranks")
        lib = grid._lib
        ex = PeerExport()
        check(lib.svr_peer_export_get(grid._h, ctypes.byref(ex)))
        allx = [None] * self.world
        dist.all_gather_object(allx, bytes(ex), group=group)
        self._exports = (PeerExport * self.world)()
        for q, raw in enumerate(allx):
            ctypes.memmove(ctypes.addressof(self._exports[q]), raw, ctypes.sizeof(PeerExport))
        # host rendezvous between the phases: a CPU-only (gloo) barrier
        self._host = group if dist.get_backend(group) == "gloo" else dist.new_group(backend="gloo")
        self._pg = ctypes.c_void_p()
        check(lib.svr_peer_group_open(grid._h, ctypes.addressof(self._exports), self.world, self.rank,
                                      ctypes.byref(self._pg)))

    def reduce(self) -> None:
        from ._lib import SVR_REDUCE_ADOPT, SVR_REDUCE_PUBLISH, SVR_REDUCE_SUM, check

        lib = self.grid._lib
        check(lib.svr_peer_reduce_phase(self._pg, SVR_REDUCE_PUBLISH))
        dist.barrier(group=self._host)  # every rank recorded "done"
        check(lib.svr_peer_reduce_phase(self._pg, SVR_REDUCE_SUM))
        dist.barrier(group=self._host)  # every rank recorded "reduced"
        check(lib.svr_peer_reduce_phase(self._pg, SVR_REDUCE_ADOPT))

    def close(self):
        if self._pg:
            self.grid._lib.svr_peer_group_close(self._pg)
            self._pg = None


def reduce_grads(grids, mode: str = "auto") -> None:
    """Single process, one SparseDenseGrid replica per device: sum the active-block gradients
    of all handles into every handle (svr_reduce_grads_ex; stream-ordered across the devices
    with peer access, NCCL otherwise or when mode == "nccl")."""
    import ctypes

    from ._lib import SVR_REDUCE_AUTO, SVR_REDUCE_NCCL, SVR_REDUCE_PEER, check

    m = {"auto": SVR_REDUCE_AUTO, "peer": SVR_REDUCE_PEER, "nccl": SVR_REDUCE_NCCL}[mode]
    hs = (ctypes.c_void_p * len(grids))(*[g._h for g in grids])
    check(grids[0]._lib.svr_reduce_grads_ex(ctypes.addressof(hs), len(grids), m))


def reduce_active_grads(grid, device, group=None) -> torch.Tensor:
    """Sum the active-block gradients of `grid` across the process group."""
    return allreduce_active(_GridStore(grid, device), group)
