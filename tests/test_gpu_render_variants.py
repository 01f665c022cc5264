"""GPU: renderer parity vs the CPU oracle across the paths the default configuration does
not exercise -- partially observed blocks (validity mask), rays longer than one 64-sample
chunk (multi-chunk scans, non-pipelined backward), hash-mode lookups, axis-parallel rays,
and every performance knob (results must not depend on them)."""
import itertools

import numpy as np
import pytest

from common import assert_close, gpu_grid_from, scene_case

pytestmark = pytest.mark.gpu


def _mask_some(case, frac, seed):
    """Copy of a case whose payload has a fraction of unobserved voxels (weight 0)."""
    from oracle import OracleGrid

    rng = np.random.default_rng(seed)
    pay = {k: v.copy() for k, v in case["pay"].items()}
    pay["weight"][rng.uniform(size=pay["weight"].shape) < frac] = 0.0
    og = OracleGrid(case["h"], 8, case["C"])
    og.allocate_blocks(case["coords"])
    og.set_payload(0, len(case["coords"]), **pay)
    c = dict(case)
    c["pay"] = pay
    c["oracle"] = og
    return c


def _check_fwd_bwd(g, case, S):
    g.grad_zero()
    out = g.render_forward(case["o"], case["d"], case["step"], S, case["beta"])
    ref = case["oracle"].render_forward(case["o"], case["d"], case["step"], S, case["beta"])
    assert np.array_equal(out["n_samples"], ref["n_samples"])
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(out[k], ref[k], what=k)
    g.render_backward(case["dC"], case["dD"], case["dN"])
    gs, gr = g.grads()
    os_, or_, act = case["oracle"].render_backward(case["o"], case["d"], case["step"], S, case["beta"],
                                                   case["dC"], case["dD"], case["dN"])
    assert_close(gs, os_, what="grad_sdf")
    assert_close(gr, or_, what="grad_rgb")
    assert np.array_equal(g.active_mask(), act)
    return int(ref["n_samples"].max())


@pytest.mark.parametrize("lookup", [1, 2])
def test_partially_observed_blocks(lookup):
    case = _mask_some(scene_case(), 0.01, 5)
    g = gpu_grid_from(case, lookup)
    _check_fwd_bwd(g, case, 64)
    v = case["oracle"].render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    assert (v["n_valid"] < v["n_samples"]).sum() > 50  # the mask actually bites


@pytest.mark.parametrize("S", [2, 33, 96, 160])
def test_long_and_short_rays(S):
    case = scene_case(h=0.03, dilation=2)
    g = gpu_grid_from(case)
    longest = _check_fwd_bwd(g, case, S)
    assert longest == S  # the cap is reached: multi-chunk path for S > 64


def test_axis_parallel_rays():
    case = dict(scene_case())
    o = case["o"].copy()
    d = case["d"].copy()
    d[::3, 0] = 0.0
    d[1::3, 2] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    case["o"], case["d"] = o, d
    g = gpu_grid_from(case)
    _check_fwd_bwd(g, case, 64)


KNOBS = list(itertools.product([0, 1, 2, 3], [0, 1], [0, 1]))


@pytest.mark.parametrize("ray_sort,records,pipe", KNOBS)
def test_performance_knobs_do_not_change_results(ray_sort, records, pipe):
    case = scene_case()
    g = gpu_grid_from(case)
    g.set_tuning("ray_sort", ray_sort)
    g.set_tuning("records", records)
    g.set_tuning("bwd_pipe", pipe)
    _check_fwd_bwd(g, case, 64)


@pytest.mark.parametrize("bwd_pipe", [1, 0])
def test_scatter_paths_match_oracle(bwd_pipe):
    """Pipelined (cp.async.bulk ring, records <= 64 samples) and plain backward, with invalid
    samples inside the runs (partially observed blocks)."""
    for c in (scene_case(), _mask_some(scene_case(), 0.15, 3)):
        g = gpu_grid_from(c)
        g.set_tuning("bwd_pipe", bwd_pipe)
        _check_fwd_bwd(g, c, 64)


def test_host_async_pipeline_matches_synchronous():
    """host_async: three forward/backward steps with different pinned ray batches issued
    back to back (slots reused), outputs and accumulated gradients equal the synchronous
    path's."""
    import torch

    case = scene_case()
    n = len(case["o"])
    rng = np.random.default_rng(4)
    perms = [rng.permutation(n) for _ in range(3)]
    batches = [{k: np.ascontiguousarray(case[k][p]) for k in ("o", "d", "dC", "dD", "dN")} for p in perms]
    S = 64

    def run(async_mode):
        g = gpu_grid_from(case)
        g.grad_zero()
        g.set_tuning("host_async", int(async_mode))
        outs = []
        for b in batches:
            pin = {k: torch.from_numpy(v).pin_memory() for k, v in b.items()}
            out = {k: torch.empty(s, dtype=torch.float32).pin_memory()
                   for k, s in (("rgb", (n, 3)), ("depth", (n,)), ("normal", (n, 3)), ("wsum", (n,)))}
            out["n_samples"] = torch.empty(n, dtype=torch.int32).pin_memory()
            g.render_forward(pin["o"], pin["d"], case["step"], S, case["beta"], out=out)
            g.render_backward(pin["dC"], pin["dD"], pin["dN"])
            outs.append((out, pin))  # keep the pinned inputs alive until synchronize
        g.synchronize()
        return [{k: v.numpy().copy() for k, v in o.items()} for o, _ in outs], g.grads()

    ref_out, (ref_gs, ref_gr) = run(False)
    out, (gs, gr) = run(True)
    for a, b in zip(out, ref_out):
        for k in a:
            assert np.array_equal(a[k], b[k]), k
    assert_close(gs, ref_gs, what="grad_sdf")
    assert_close(gr, ref_gr, what="grad_rgb")


@pytest.mark.parametrize("S", [8, 33, 100])
@pytest.mark.parametrize("records", [1, 0])
def test_sample_budgets_below_at_and_beyond_one_pass(S, records):
    """The forward's one-pass-ahead t prefetch at budgets below, just above and beyond one
    32-sample pass, with and without records (the backward re-gathers without them)."""
    for c in (scene_case(), _mask_some(scene_case(), 0.15, 3)):
        g = gpu_grid_from(c)
        g.set_tuning("records", records)
        _check_fwd_bwd(g, c, S)


@pytest.mark.parametrize("rays_per_pose", [64, 512])
def test_deferred_zeroing_keeps_results(rays_per_pose):
    """zero_fused: svr_grad_zero_active leaves the zeroing to the next forward's warps (512
    rays: more blocks than the warps take, so it runs as its own kernel; 4096 rays: fused), and
    every other entry point runs it first -- same gradients as the in-order zeroing, step after
    step, and the planes read back zero right after the call."""
    c = scene_case(rays_per_pose=rays_per_pose)
    got = {}
    for za in (0, 1):
        g = gpu_grid_from(c)
        g.set_tuning("zero_fused", za)
        g.grad_zero()
        seq = []
        for it in range(3):
            g.render_forward(c["o"], c["d"], c["step"], 64, c["beta"])
            g.render_backward(c["dC"], c["dD"], c["dN"])
            seq.append(tuple(a.copy() for a in g.grads()))
            g.grad_zero_active()
            if it == 1:  # a read right after the call sees zeros (runs the pending zeroing)
                gs, gr = g.grads()
                assert not gs.any() and not gr.any() and not g.active_mask().any()
        got[za] = seq
    # every step's gradients are the single-step ones: equal to the oracle's (the fp32 atomic
    # order differs run to run, so not bit for bit)
    ogs, ogr, _ = c["oracle"].render_backward(c["o"], c["d"], c["step"], 64, c["beta"], c["dC"], c["dD"], c["dN"])
    for za in (0, 1):
        for gs, gr in got[za]:
            assert_close(gs, ogs, what=f"grad_sdf zero_fused={za}")
            assert_close(gr, ogr, what=f"grad_rgb zero_fused={za}")


def test_small_batches_skip_the_ordering():
    """sort_min_rays: a batch below the threshold renders in caller order -- same outputs
    (bit for bit: the per-ray arithmetic does not depend on the order) and gradients within
    the atomic-order tolerance."""
    c = scene_case()
    res = []
    for smr in (0, 1 << 20):
        g = gpu_grid_from(c)
        g.set_tuning("sort_min_rays", smr)
        g.grad_zero()
        out = g.render_forward(c["o"], c["d"], c["step"], 64, c["beta"])
        g.render_backward(c["dC"], c["dD"], c["dN"])
        res.append((out, g.grads(), g.active_mask()))
    for k in ("rgb", "depth", "normal", "wsum", "n_samples"):
        assert np.array_equal(res[0][0][k], res[1][0][k]), k
    assert_close(res[1][1][0], res[0][1][0], what="grad_sdf")
    assert_close(res[1][1][1], res[0][1][1], what="grad_rgb")
    assert np.array_equal(res[0][2], res[1][2])
