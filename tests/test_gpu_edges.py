"""GPU: edge cases of the render path through the C-ABI -- empty batches, an empty grid,
rays that miss the grid, a backward without a forward, and invalid arguments.  The
reference's behaviour for each (SPEC.md:281 rays with no valid sample -> zeros; errors.hpp
status codes) is what the boundary must reproduce."""
import numpy as np
import pytest

from common import gpu_grid_from, scene_case

pytestmark = pytest.mark.gpu


def _grid(C=4, h=0.04):
    from paper_2305_13220_b200 import SparseDenseGrid

    return SparseDenseGrid(h, 8, C)


def test_empty_batch_forward_backward():
    c = scene_case()
    g = gpu_grid_from(c)
    o = np.zeros((0, 3))
    out = g.render_forward(o, o, c["step"], 64, c["beta"])
    assert all(v.shape[0] == 0 for v in out.values())
    g.render_backward(np.zeros((0, 3), np.float32), np.zeros(0, np.float32), np.zeros((0, 3), np.float32))
    gs, gr = g.grads()
    assert not gs.any() and not gr.any()


def test_empty_grid_renders_zeros():
    g = _grid()
    rng = np.random.default_rng(0)
    o = rng.uniform(-1, 1, (100, 3))
    d = rng.normal(size=(100, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    out = g.render_forward(o, d, 0.02, 64, 0.08)
    for k in ("rgb", "depth", "normal", "wsum"):
        assert not out[k].any(), k
    assert not out["n_samples"].any()
    g.render_backward(np.ones((100, 3), np.float32), np.ones(100, np.float32), np.ones((100, 3), np.float32))


def test_rays_that_miss_the_grid_give_zeros_and_no_gradient():
    c = scene_case()
    g = gpu_grid_from(c)
    n = 64
    o = np.tile([[50.0, 50.0, 50.0]], (n, 1))  # far outside, pointing away
    d = np.tile([[1.0, 0.0, 0.0]], (n, 1))
    g.grad_zero()
    out = g.render_forward(o, d, c["step"], 64, c["beta"])
    assert not out["n_samples"].any() and not out["wsum"].any()
    g.render_backward(np.ones((n, 3), np.float32), np.ones(n, np.float32), np.ones((n, 3), np.float32))
    gs, gr = g.grads()
    assert not gs.any() and not gr.any() and not g.active_mask().any()


def test_mixed_batch_matches_the_hitting_rays_alone():
    """Rays with no sample do not disturb their neighbours (sorting puts them last)."""
    c = scene_case()
    g = gpu_grid_from(c)
    n = len(c["o"])
    miss_o = np.tile([[50.0, 50.0, 50.0]], (n, 1))
    o = np.empty((2 * n, 3))
    d = np.empty((2 * n, 3))
    o[0::2], o[1::2] = c["o"], miss_o
    d[0::2], d[1::2] = c["d"], np.tile([[1.0, 0.0, 0.0]], (n, 1))
    both = g.render_forward(o, d, c["step"], 64, c["beta"])
    alone = g.render_forward(c["o"], c["d"], c["step"], 64, c["beta"])
    for k in ("rgb", "depth", "normal", "wsum", "n_samples"):
        assert np.array_equal(both[k][0::2], alone[k]), k
        assert not both[k][1::2].any(), k


def test_backward_without_forward_is_a_data_error():
    from paper_2305_13220_b200 import DataError

    c = scene_case()
    g = gpu_grid_from(c)
    with pytest.raises(DataError):
        g.render_backward(np.zeros((4, 3), np.float32), np.zeros(4, np.float32), np.zeros((4, 3), np.float32))


@pytest.mark.parametrize("kw", [dict(step=0.0), dict(beta=0.0), dict(beta=-1.0), dict(S=0), dict(S=4096)])
def test_invalid_render_arguments_are_config_errors(kw):
    from paper_2305_13220_b200 import ConfigError

    c = scene_case()
    g = gpu_grid_from(c)
    a = dict(step=c["step"], beta=c["beta"], S=64)
    a.update(kw)
    with pytest.raises(ConfigError):
        g.render_forward(c["o"][:8], c["d"][:8], a["step"], a["S"], a["beta"])


def test_active_blocks_device_outputs_stay_stream_ordered():
    """svr_active_blocks with device outputs (count and list) is stream-ordered, no host read of
    the count: the device count and the first `count` list entries match the host form."""
    import ctypes

    import torch

    from common import gpu_grid_from, scene_case

    from paper_2305_13220_b200._lib import check

    c = scene_case()
    g = gpu_grid_from(c)
    g.set_stream(torch.cuda.current_stream())
    g.grad_zero()
    g.render_forward(c["o"], c["d"], c["step"], 64, c["beta"])
    g.render_backward(c["dC"], c["dD"], c["dN"])
    A = g.block_count()
    lst = torch.full((A,), -1, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    check(g._lib.svr_active_blocks(g._h, None, lst.data_ptr(), cnt.data_ptr()))
    torch.cuda.synchronize()
    want = np.flatnonzero(g.active_mask())
    n = int(cnt.item())
    assert n == len(want) and np.array_equal(lst[:n].cpu().numpy(), want)
