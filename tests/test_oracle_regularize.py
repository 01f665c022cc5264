"""CPU: the restated Eikonal regulariser and RMSProp update
against the SPEC's known answers and finite differences."""
import numpy as np
import pytest

from oracle import OracleGrid


def _linear_grid(a, b, h=1.0 / 64.0):
    """grid filled with theta = a.x + b (test_grid.cpp:207 style), all voxels valid."""
    g = OracleGrid(h, 8, 1)
    g.allocate_points(np.array([[0.05, 0.05, 0.05], [-0.05, 0.02, 0.08]]), 1)
    c = g.coords()
    n = len(c)
    v = np.arange(512)
    lx, ly, lz = v % 8, (v // 8) % 8, v // 64
    X = (c[:, 0:1] * 8 + lx) * h
    Y = (c[:, 1:2] * 8 + ly) * h
    Z = (c[:, 2:3] * 8 + lz) * h
    sdf = (a[0] * X + a[1] * Y + a[2] * Z + b).astype(np.float32)
    g.set_payload(0, n, sdf=sdf, weight=np.ones((n, 512), np.float32),
                  rgb=np.zeros((n, 512, 3), np.float32), logits=np.zeros((n, 512, 1), np.float32))
    return g


def _points(n=3000, seed=1):
    return np.random.default_rng(seed).uniform(-0.05, 0.1, size=(n, 3))


def test_perfect_plane_has_zero_loss():
    n = np.array([2.0, -1.0, 2.0]) / 3.0  # unit normal
    g = _linear_grid(n, 0.1)
    loss, nv, gs, _ = g.eikonal(_points())
    assert nv > 1000
    assert loss < 1e-12  # float32 payload rounding only


def test_doubled_plane_has_unit_loss():
    """theta = 2 (n.x + c) -> |grad f| = 2 -> loss = 1 at every fully valid cell."""
    n = np.array([2.0, -1.0, 2.0]) / 3.0
    g = _linear_grid(2 * n, 0.2)
    loss, nv, _, _ = g.eikonal(_points())
    assert nv > 1000
    assert loss == pytest.approx(1.0, abs=1e-6)


def test_eikonal_gradient_matches_finite_differences():
    """voxel gradient of the loss vs central differences, rel 1e-4."""
    rng = np.random.default_rng(7)
    g = _linear_grid(np.array([0.7, 0.5, -0.4]), 0.05)
    n = g.block_count()
    base = g.get_payload()["sdf"].astype(np.float64)
    sdf = (base + rng.normal(0, 0.002, base.shape)).astype(np.float32)
    g.set_payload(0, n, sdf=sdf)
    x = _points(400, 3)
    loss, nv, gs, _ = g.eikonal(x)
    eps = 1e-4  # |grad f| moves by ~eps * inv_h: keep the higher-order FD error << 1e-4
    for fi in np.argsort(-np.abs(gs).ravel())[:25]:
        b, v = divmod(int(fi), 512)
        sp = sdf.copy()
        sp[b, v] = np.float32(sdf[b, v] + eps)
        up = float(sp[b, v]) - float(sdf[b, v])  # the float32 perturbation actually applied
        g.set_payload(0, n, sdf=sp)
        lp = g.eikonal(x, 0.0)[0]
        sp[b, v] = np.float32(sdf[b, v] - eps)
        dn = float(sp[b, v]) - float(sdf[b, v])
        g.set_payload(0, n, sdf=sp)
        lm = g.eikonal(x, 0.0)[0]
        g.set_payload(0, n, sdf=sdf)
        assert (lp - lm) / (up - dn) == pytest.approx(gs[b, v], rel=1e-4, abs=1e-9 * np.abs(gs).max())


def test_rmsprop_single_step_closed_form():
    g = OracleGrid(0.02, 8, 1)
    g.allocate_blocks(np.array([[0, 0, 0], [3, 0, 0]]))
    A = 2
    sdf = np.full((A, 512), 0.5, np.float32)
    g.set_payload(0, A, sdf=sdf, weight=np.ones((A, 512), np.float32),
                  rgb=np.full((A, 512, 3), 0.25, np.float32), logits=np.zeros((A, 512, 1), np.float32))
    gsdf = np.full((A, 512), 0.1)
    grgb = np.full((A, 512, 3), -0.2)
    active = np.array([1, 0], np.uint8)
    rms = np.zeros((A, 512, 4), np.float32)
    lr, alpha, eps = 1e-2, 0.99, 1e-8
    g.rmsprop(gsdf, grgb, active, lr, alpha, eps, rms)
    p = g.get_payload()
    # first step: v = (1-a) g^2 -> theta -= lr g / (sqrt((1-a)) |g| + eps) = lr sign(g) / sqrt(0.01)
    assert p["sdf"][0, 0] == pytest.approx(0.5 - lr / np.sqrt(1 - alpha), rel=1e-5)
    assert p["rgb"][0, 0, 0] == pytest.approx(0.25 + lr / np.sqrt(1 - alpha), rel=1e-5)
    assert p["sdf"][1, 0] == 0.5  # inactive block untouched
    assert rms[0, 0, 0] == pytest.approx((1 - alpha) * 0.01, rel=1e-5) and rms[1].max() == 0
