"""GPU: the peer-memory active-block all-reduce.  (1) Emulated ranks: W gradient planes on
one GPU, one kernel launch per rank slice -- every plane ends with the rank-order sum.
(2) The sync-free group (K8r, PeerGradReducer): 2 processes on the one GPU with CUDA IPC
planes, flags and interprocess events, gloo host barriers between the phases; the kernels
only wait on events recorded before the wait (no kernel spins on another), so this is safe
on a single device.  (3) svr_reduce_grads: one process, several handles on the one GPU
(peer path) and the NCCL path on one device."""
import ctypes
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

COORDS = np.array([[x, y, z] for z in range(3) for y in range(3) for x in range(4)], np.int32)


def _rank_grads(rank, A):
    rng = np.random.default_rng(100 + rank)
    rows = np.sort(rng.choice(A, size=A // 2, replace=False)).astype(np.uint32)
    vals = rng.normal(size=(len(rows), 512, 4)).astype(np.float32)
    return rows, vals


def _load(g, rows, vals):
    import torch

    g.set_stream(torch.cuda.current_stream())  # the torch-made device inputs are ordered on it
    g.grad_zero()
    A = g.block_count()
    g.grad_unpack(torch.from_numpy(rows.astype(np.int32)).cuda(), torch.from_numpy(vals).cuda())
    m = np.zeros(A, np.uint8)
    m[rows] = 1
    g.active_set_mask(torch.from_numpy(m).cuda())


def _expected(world, A):
    tot = np.zeros((A, 512, 4), np.float32)
    union = np.zeros(A, bool)
    for r in range(world):
        rows, vals = _rank_grads(r, A)
        tot[rows] += vals  # rank order, float32: the kernel's summation order
        union[rows] = True
    return tot, union


def _plane(g):
    gs, gr = g.grads()
    return np.concatenate([gs[..., None], gr], axis=-1)


@pytest.mark.parametrize("world", [2, 3, 4])
def test_peer_allreduce_emulated_ranks(world):
    from paper_2305_13220_b200 import SparseDenseGrid
    from paper_2305_13220_b200._lib import check

    grids = []
    for r in range(world):
        g = SparseDenseGrid(0.02, 8, 1)
        g.allocate_blocks(COORDS)
        _load(g, *_rank_grads(r, len(COORDS)))
        grids.append(g)
    planes = (ctypes.c_void_p * world)()
    for r, g in enumerate(grids):
        p = ctypes.c_void_p()
        check(g._lib.svr_grad_plane(g._h, ctypes.byref(p), None))
        planes[r] = p.value
    tot, union = _expected(world, len(COORDS))
    rows = np.flatnonzero(union).astype(np.uint32)
    for r, g in enumerate(grids):  # one launch per rank slice, in sequence
        check(g._lib.svr_grad_peer_allreduce(g._h, ctypes.addressof(planes), world, r, rows.ctypes.data, len(rows)))
        g.synchronize()
    for g in grids:
        got = _plane(g)
        assert np.array_equal(got[union], tot[union])
        assert not got[~union].any()


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    from paper_2305_13220_b200 import SparseDenseGrid
    from paper_2305_13220_b200.distributed import PeerGradReducer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = SparseDenseGrid(0.02, 8, 1)
    g.allocate_blocks(COORDS)
    _load(g, *_rank_grads(rank, len(COORDS)))
    red = PeerGradReducer(g, "cuda:0")
    red.reduce()  # stream-ordered, no device synchronisation inside
    np.save(os.path.join(out_dir, f"r{rank}.npy"), _plane(g))
    np.save(os.path.join(out_dir, f"b{rank}.npy"), np.flatnonzero(g.active_mask()))
    red.reduce()  # a second step on the same group (events re-recorded): sums again
    np.save(os.path.join(out_dir, f"s{rank}.npy"), _plane(g))
    red.close()
    dist.barrier()
    dist.destroy_process_group()


def test_peer_allreduce_ipc_two_processes_one_gpu(tmp_path):
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world = 2
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    tot, union = _expected(world, len(COORDS))
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npy")
        assert np.array_equal(got[union], tot[union]), r
        assert not got[~union].any()
        assert np.array_equal(np.load(tmp_path / f"b{r}.npy"), np.flatnonzero(union))
        # second reduction: every plane held the sum, so the new sum is world x that
        assert np.array_equal(np.load(tmp_path / f"s{r}.npy")[union], world * tot[union]), r


def _render_case(lookup=None):
    from common import scene_case

    return scene_case()


@pytest.mark.parametrize("n", [2, 3])
def test_reduce_grads_single_process_handles(n):
    """n replicas, each rendering its contiguous ray shard, summed by svr_reduce_grads (peer
    path, stream-ordered across the handles' own streams): every replica ends with the
    full-batch gradients and the full-batch active set."""
    from common import assert_close, gpu_grid_from, scene_case

    from paper_2305_13220_b200.distributed import reduce_grads

    case = scene_case()
    R = len(case["o"])
    full = gpu_grid_from(case)
    full.grad_zero()
    full.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    full.render_backward(case["dC"], case["dD"], case["dN"])
    gs_ref, gr_ref = full.grads()
    act_ref = full.active_mask()
    grids = []
    for i in range(n):
        a, b = R * i // n, R * (i + 1) // n
        g = gpu_grid_from(case)
        g.grad_zero()
        g.render_forward(case["o"][a:b], case["d"][a:b], case["step"], 64, case["beta"])
        g.render_backward(case["dC"][a:b], case["dD"][a:b], case["dN"][a:b])
        grids.append(g)
    reduce_grads(grids, "peer")
    planes = []
    for g in grids:
        gs, gr = g.grads()
        assert_close(gs, gs_ref, what="grad_sdf")
        assert_close(gr, gr_ref, what="grad_rgb")
        assert np.array_equal(g.active_mask(), act_ref)
        planes.append((gs, gr))
    for gs, gr in planes[1:]:  # rank-order sums: bitwise identical replicas
        assert np.array_equal(gs, planes[0][0]) and np.array_equal(gr, planes[0][1])


def test_reduce_grads_nccl_one_device():
    """The NCCL path (dlopen'ed libnccl, ncclCommInitAll, grouped all-reduces, pack/unpack)
    on the one device: a one-rank sum leaves the gradients and the active set unchanged;
    two handles on one device are refused (NCCL needs one per device)."""
    from common import gpu_grid_from, scene_case

    from paper_2305_13220_b200._lib import ConfigError
    from paper_2305_13220_b200.distributed import reduce_grads

    import torch  # noqa: F401  (the process's NCCL is torch's, as in the bench)

    case = scene_case()
    g = gpu_grid_from(case)
    g.grad_zero()
    g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    g.render_backward(case["dC"], case["dD"], case["dN"])
    gs, gr = g.grads()
    act = g.active_mask()
    reduce_grads([g], "nccl")
    gs2, gr2 = g.grads()
    assert np.array_equal(gs2, gs) and np.array_equal(gr2, gr)
    assert np.array_equal(g.active_mask(), act)
    g2 = gpu_grid_from(case)
    with pytest.raises(ConfigError):
        reduce_grads([g, g2], "nccl")
