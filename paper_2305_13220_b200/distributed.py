"""Multi-GPU active-block gradient reduction (kernels K7/K8).

Rays are sharded across ranks with the grid replicated; after each rank's backward the
voxel gradients must be summed.  Only blocks touched by some rank carry gradient, so:

  1. active mask  u8[A]   -> all_reduce(MAX)      (union of touched blocks)
  2. compaction           -> ascending block list, identical on every rank (K7)
  3. pack  [n,512,4] fp32 -> all_reduce(SUM)      (NCCL over NVLink, K8)
  4. unpack into the gradient planes

``reduce_active_grads`` drives steps 1-4 for a ``SparseDenseGrid`` whose kernels run on
torch's current stream (grid.set_stream), so NCCL and the pack/unpack kernels are
stream-ordered.  The collective sequence itself is ``allreduce_active`` and is backend
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
    """The fused alternative to steps 2-4 (K8p): every rank maps the other ranks' gradient
    planes (CUDA IPC over NVLink), and after a barrier each rank reduces its 1/world slice of
    the common active list straight in peer memory -- sum in rank order, store to every
    plane -- so there is no pack buffer, no unpack and no NCCL ring for the 2.4 GB payload.
    Only the u8 mask union still goes through the process group.  Construct after the grid
    has all its blocks (the planes must not be reallocated while mapped)."""

    def __init__(self, grid, device, group=None):
        import ctypes

        from ._lib import check

        self.grid, self.device, self.group = grid, torch.device(device), group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > 8:
            raise ValueError("PeerGradReducer: at most 8 ranks")
        lib = grid._lib
        h = (ctypes.c_uint8 * 64)()
        nbytes = ctypes.c_uint64()
        check(lib.svr_grad_ipc_handle(grid._h, ctypes.addressof(h), ctypes.byref(nbytes)))
        allh = [None] * self.world
        dist.all_gather_object(allh, (bytes(h), nbytes.value), group=group)
        self.ptrs = (ctypes.c_void_p * self.world)()
        self.opened = []
        dev = self.device.index if self.device.index is not None else torch.cuda.current_device()
        for q, (hb, _) in enumerate(allh):
            if q == self.rank:
                continue
            p = ctypes.c_void_p()
            buf = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
            check(lib.svr_ipc_open(ctypes.addressof(buf), dev, ctypes.byref(p)))
            self.ptrs[q] = p.value
            self.opened.append(p)
        self._gloo = dist.get_backend(group) == "gloo"

    def reduce(self) -> torch.Tensor:
        import ctypes

        from ._lib import check

        store = _GridStore(self.grid, self.device)
        mask = store.mask_tensor()
        self.grid.synchronize()  # the mask (and the backward) are complete whatever stream reads them
        if self._gloo:
            m = mask.cpu()
            dist.all_reduce(m, op=dist.ReduceOp.MAX, group=self.group)
            mask = m.to(self.device)
        else:
            dist.all_reduce(mask, op=dist.ReduceOp.MAX, group=self.group)
        store.set_mask(mask)
        blocks = store.active_list()
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)  # every rank's backward is in its plane
        if blocks.numel():
            check(self.grid._lib.svr_grad_peer_allreduce(self.grid._h, ctypes.addressof(self.ptrs), self.world, self.rank,
                                                         blocks.data_ptr(), blocks.numel()))
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)  # every slice is summed into every plane
        return blocks

    def close(self):
        for p in self.opened:
            self.grid._lib.svr_ipc_close(p)
        self.opened = []


def reduce_active_grads(grid, device, group=None) -> torch.Tensor:
    """Sum the active-block gradients of `grid` across the process group."""
    return allreduce_active(_GridStore(grid, device), group)
