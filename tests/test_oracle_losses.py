"""CPU: the restated refinement losses (PAPER Eq. 12-14/23) -- the
minibatch depth-prior fit against the SPEC's known answers, and the full analytic gradient
(render + losses + render backward) against per-voxel central finite differences."""
import numpy as np
import pytest

from oracle import OracleGrid, fit_depth_affine, render_losses


def test_affine_fit_known_answers():
    rng = np.random.default_rng(0)
    D = rng.uniform(0.5, 4.0, 500)
    a, b, s = fit_depth_affine(D, D)
    assert not s and a == pytest.approx(1.0, abs=1e-12) and b == pytest.approx(0.0, abs=1e-12)
    a, b, s = fit_depth_affine(2.0 * D + 0.3, D)
    assert a == pytest.approx(2.0, abs=1e-10) and b == pytest.approx(0.3, abs=1e-10)
    t = np.full(10, 1.7) + rng.normal(0, 0.01, 10)
    a, b, s = fit_depth_affine(t, np.full(10, 1.5))  # all D equal: fallback
    assert s and a == 1.0 and b == pytest.approx(np.mean(t - 1.5), abs=1e-14)


def test_affine_fit_is_optimal_and_unbiased():
    rng = np.random.default_rng(1)
    D = rng.uniform(0.5, 4.0, 2000)
    sig = 0.02
    t = D + rng.normal(0, sig, D.shape)
    a, b, _ = fit_depth_affine(t, D)
    res = lambda a_, b_: np.mean((t - (a_ * D + b_)) ** 2)  # noqa: E731
    r0 = res(a, b)
    assert r0 == pytest.approx(sig ** 2, rel=0.1)
    for da in (-1e-3, 1e-3):
        for db in (-1e-3, 0.0, 1e-3):
            assert res(a + da, b + db) >= r0
    se = sig / np.sqrt(np.sum((D - D.mean()) ** 2))
    assert abs(a - 1.0) < 3 * se


def _toy(seed=0):
    import sys
    import os

    sys.path.insert(0, os.path.dirname(__file__))
    from common import scene_case

    case = scene_case()
    sc = case["scene"]
    n_poses, rpp = 8, 64
    cams = [sc.camera_for_frame(p) for p in range(n_poses)]
    cam_idx = np.repeat(np.arange(n_poses), rpp).astype(np.uint32)
    og = case["oracle"]
    out = og.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    rng = np.random.default_rng(seed)
    n = len(case["o"])
    tgt = np.clip(out["rgb"] + 0.3 * np.sign(rng.normal(size=(n, 3))), -1, 2).astype(np.float32)
    prior_d = (out["depth"] * 0.9 + 0.05 + rng.normal(0, 0.02, n)).astype(np.float32)
    prior_d[rng.uniform(size=n) < 0.1] = 0.0  # invalid prior pixels
    pn = rng.normal(size=(n, 3))
    pn /= np.linalg.norm(pn, axis=1, keepdims=True)
    pn[rng.uniform(size=n) < 0.1] = 0.0
    # the normal term is 1/|N|-conditioned: keep it to rays that are mostly opaque, where a
    # 1e-4 voxel perturbation stays in the linear regime of the normalisation
    pn[out["wsum"] < 0.5] = 0.0
    return case, cams, cam_idx, out, tgt, prior_d, pn.astype(np.float32)


def test_losses_stats_and_participation():
    case, cams, cam_idx, out, tgt, pd, pn = _toy()
    g, st = render_losses(out, tgt, pd, pn, cam_idx, cams)
    part = out["wsum"] > 0
    assert st["n_c"] == part.sum() > 100
    assert st["n_d"] == (part & (pd > 0)).sum()
    assert not st["singular"] and 0.5 < st["a"] < 1.5
    assert np.all(g["d_rgb"][~part] == 0) and np.all(g["d_depth"][pd <= 0] == 0)
    assert st["L_c"] == pytest.approx(np.abs(out["rgb"][part] - tgt[part]).sum(1).mean(), rel=1e-12)
    assert st["total"] == pytest.approx(st["L_c"] + 0.1 * st["L_d"] + 0.05 * st["L_n"], rel=1e-14)


def test_total_loss_gradient_matches_finite_differences():
    """every accumulated voxel gradient vs central differences of the total
    loss (h = 1e-4) within rel 2e-3."""
    case, cams, cam_idx, out, tgt, pd, pn = _toy(3)
    og = OracleGrid(case["h"], 8, case["C"])
    og.allocate_blocks(case["coords"])
    A = len(case["coords"])
    pay = {k: v.copy() for k, v in case["pay"].items()}
    og.set_payload(0, A, **pay)
    args = (case["o"], case["d"], case["step"], 64, case["beta"])

    def total():
        o = og.render_forward(*args)
        return render_losses(o, tgt, pd, pn, cam_idx, cams)

    g, st = total()
    gs, gr, _ = og.render_backward(*args, g["d_rgb"], g["d_depth"], g["d_normal"])
    eps = 2e-5  # the L1 / normalisation terms are piecewise smooth: keep the step small
    checked = 0
    for plane, grad in (("sdf", gs), ("rgb", gr)):
        flat = np.abs(grad).ravel()
        for fi in np.argsort(-flat)[:12]:
            arr = pay[plane]
            idx = np.unravel_index(fi, arr.shape)
            base = float(arr[idx])
            vals = []
            for sgn in (1, -1):
                arr[idx] = np.float32(base + sgn * eps)
                og.set_payload(0, A, **{plane: arr})
                vals.append((total()[1]["total"], float(arr[idx])))
            arr[idx] = np.float32(base)
            og.set_payload(0, A, **{plane: arr})
            fd = (vals[0][0] - vals[1][0]) / (vals[0][1] - vals[1][1])
            assert fd == pytest.approx(grad[idx], rel=2e-3, abs=1e-3 * flat.max()), (plane, idx)
            checked += 1
    assert checked == 24
