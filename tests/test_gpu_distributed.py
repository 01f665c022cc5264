"""GPU: the multi-GPU active-block reduction's device plumbing (mask read-back into a CUDA
tensor, NCCL all_reduce MAX / SUM, ascending compaction, pack / unpack kernels) on a
single-rank NCCL group -- the only multi-rank shape a one-GPU box can run without ranks
waiting on each other.  The N > 1 arithmetic is covered by tests/test_distributed_gloo.py."""
import os
import socket

import numpy as np
import pytest

from common import gpu_grid_from, scene_case

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_reduce_active_grads_single_rank_nccl():
    import torch
    import torch.distributed as dist

    from paper_2305_13220_b200.distributed import reduce_active_grads

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        case = scene_case()
        g = gpu_grid_from(case)
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        g.set_stream(stream)
        g.grad_zero()
        g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
        g.render_backward(case["dC"], case["dD"], case["dN"])
        gs, gr = g.grads()
        mask = g.active_mask()
        blocks = reduce_active_grads(g, torch.device("cuda", 0))
        torch.cuda.synchronize()
        assert np.array_equal(blocks.cpu().numpy().astype(np.int64), np.nonzero(mask)[0])
        gs2, gr2 = g.grads()
        assert np.array_equal(gs2, gs) and np.array_equal(gr2, gr)  # sum over one rank
        assert np.array_equal(g.active_mask(), mask)
    finally:
        torch.cuda.set_stream(torch.cuda.default_stream())
        dist.destroy_process_group()
