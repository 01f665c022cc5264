"""CPU, world_size 2 (gloo): the multi-GPU active-block gradient reduction
(paper_2305_13220_b200.distributed.allreduce_active) on rank-sharded rays.

Each rank renders its contiguous shard of the rays with the CPU oracle; after
mask-union + compaction + pack + all-reduce + unpack every rank must hold the
full-batch gradients and the full-batch active set (fp64 reorder tolerance)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


class OracleStore:
    """ActiveGradStore over CPU tensors holding one rank's oracle gradients."""

    def __init__(self, gs, gr, active):
        self.g = torch.from_numpy(np.concatenate([gs[..., None], gr], -1))  # [A,512,4] f64
        self.mask = torch.from_numpy(active.astype(np.uint8))

    def mask_tensor(self):
        return self.mask.clone()

    def set_mask(self, mask):
        self.mask = mask

    def active_list(self):
        return torch.nonzero(self.mask).flatten().to(torch.int32)

    def pack(self, blocks):
        return self.g[blocks.long()].clone()

    def unpack(self, blocks, packed):
        self.g[blocks.long()] = packed


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from common import scene_case

        from paper_2305_13220_b200.distributed import allreduce_active

        c = scene_case()
        og = c["oracle"]
        n = len(c["o"])
        sl = slice(rank * n // world, (rank + 1) * n // world)
        gs, gr, act = og.render_backward(c["o"][sl], c["d"][sl], c["step"], 64, c["beta"],
                                         c["dC"][sl], c["dD"][sl], c["dN"][sl])
        store = OracleStore(gs, gr, act)
        allreduce_active(store)
        fs, fr, fa = og.render_backward(c["o"], c["d"], c["step"], 64, c["beta"], c["dC"], c["dD"], c["dN"])
        full = np.concatenate([fs[..., None], fr], -1)
        ok_mask = np.array_equal(store.mask.numpy(), fa)
        err = float(np.abs(store.g.numpy() - full).max())
        scale = float(np.abs(full).max())
        shard_only = int(act.sum()) < int(fa.sum())
        result[rank] = (ok_mask, err, scale, shard_only)
    finally:
        dist.destroy_process_group()


def test_allreduce_active_two_ranks():
    world = 2
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), result), nprocs=world, join=True)
    for r in range(world):
        ok_mask, err, scale, shard_only = result[r]
        assert ok_mask, f"rank {r}: union mask != full-batch active set"
        assert err <= 1e-12 * scale, (r, err, scale)
        assert shard_only  # each shard alone touches fewer blocks than the union
