"""CPU: the restated renderer oracle against the SPEC's known-answer tests and finite
differences (the reference has no renderer code, so these pin it: SPEC.md:268-319,
SPEC.md:581-584).  Also randomized oracle-vs-compiled-reference checks of the grid path.
"""
import numpy as np
import pytest

import oracle
from oracle import OracleGrid, RefGrid

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference not built")


# --- sdf_to_density ---------------------------------------------
def test_density_known_answers():
    beta = 0.01
    assert OracleGrid.density(0.0, beta) == pytest.approx(1 / (2 * beta), rel=1e-15)
    assert OracleGrid.density(0.01, 0.01) == pytest.approx(18.394, rel=1e-4)  # (1/b) 0.5 e^-1
    assert OracleGrid.density(10.0, beta) < 1e-300
    assert OracleGrid.density(-10.0, beta) == pytest.approx(1 / beta, rel=1e-12)
    s = np.linspace(-0.1, 0.1, 2001)
    a = np.array([OracleGrid.density(v, beta) for v in s])
    assert (np.diff(a) <= 0).all()  # monotone non-increasing


def _block_grid(sdf_value, h=0.02, C=1):
    """2 x 1 x 1 blocks, every voxel valid, constant sdf / rgb."""
    g = OracleGrid(h, 8, C)
    g.allocate_blocks(np.array([[0, 0, 0], [1, 0, 0]]))
    n = 2
    g.set_payload(0, n, sdf=np.full((n, 512), sdf_value, np.float32), weight=np.ones((n, 512), np.float32),
                  rgb=np.full((n, 512, 3), 0.5, np.float32), logits=np.zeros((n, 512, C), np.float32))
    return g


def _axis_rays(n=8, h=0.02):
    L = 8 * h
    y = np.linspace(0.2, 0.8, n) * L
    o = np.stack([np.full(n, -1.0), y, np.full(n, 0.5 * L)], 1)
    d = np.tile([1.0, 0.0, 0.0], (n, 1))
    return o, d


def test_zero_density_gives_zero_weights():
    """alpha == 0 -> all w_k = 0, black/zero outputs."""
    g = _block_grid(1e3)  # far outside: sigma = (1/b) 0.5 exp(-s/b) underflows to 0
    o, d = _axis_rays()
    f = g.render_forward(o, d, 0.01, 64, 0.04)
    assert (f["n_samples"] > 10).all()
    for k in ("rgb", "depth", "normal", "wsum"):
        assert np.abs(f[k]).max() == 0.0, k


def test_opaque_first_sample():
    """first sample opaque (alpha delta >= 20) -> w1 ~ 1, depth ~ t1."""
    g = _block_grid(-1.0)
    o, d = _axis_rays()
    beta = 1e-4  # sigma ~ 1/beta = 1e4, delta = 0.01 -> tau = 100
    f = g.render_forward(o, d, 0.01, 64, beta)
    m = g.march(o, d, 0.01, 64)
    np.testing.assert_allclose(f["wsum"], 1.0, rtol=1e-12)
    np.testing.assert_allclose(f["depth"], m["t"][:, 0], rtol=1e-9)
    np.testing.assert_allclose(f["rgb"], 0.5, rtol=1e-6)


def test_weights_partition_random_fields():
    """0 <= sum w <= 1 for random sdf fields and betas."""
    rng = np.random.default_rng(3)
    for beta in (0.005, 0.02, 0.2):
        g = OracleGrid(0.02, 8, 1)
        g.allocate_points(rng.uniform(-0.2, 0.2, size=(6, 3)), 1)
        n = g.block_count()
        g.set_payload(0, n, sdf=rng.uniform(-0.1, 0.1, (n, 512)).astype(np.float32),
                      weight=np.ones((n, 512), np.float32),
                      rgb=rng.uniform(0, 1, (n, 512, 3)).astype(np.float32),
                      logits=np.zeros((n, 512, 1), np.float32))
        o = rng.uniform(-1, 1, (400, 3))
        d = -o + rng.normal(0, 0.05, (400, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        f = g.render_forward(o, d, 0.01, 64, beta)
        assert (f["wsum"] >= 0).all() and (f["wsum"] <= 1 + 1e-12).all()
        assert (f["n_samples"] > 0).sum() > 100


def _loss(g, o, d, step, S, beta, dC, dD, dN):
    f = g.render_forward(o, d, step, S, beta)
    return float((f["rgb"] * dC).sum() + (f["depth"] * dD).sum() + (f["normal"] * dN).sum())


def test_backward_matches_finite_differences():
    """Per-voxel FD of L = sum dC.C + dD D + dN.N on a 2-block toy, rel 2e-3."""
    rng = np.random.default_rng(11)
    h = 0.02
    g = OracleGrid(h, 8, 1)
    g.allocate_blocks(np.array([[0, 0, 0], [1, 0, 0]]))
    n = 2
    x = (np.arange(512) % 8) * h
    sdf = np.tile((0.12 - x)[None], (n, 1)).astype(np.float32)  # plane crossing in block 0
    sdf[1] -= 8 * h
    sdf += rng.normal(0, 0.002, sdf.shape).astype(np.float32)
    rgb = rng.uniform(0, 1, (n, 512, 3)).astype(np.float32)
    g.set_payload(0, n, sdf=sdf, weight=np.ones((n, 512), np.float32), rgb=rgb,
                  logits=np.zeros((n, 512, 1), np.float32))
    L = 8 * h
    m = 24
    o = np.stack([np.full(m, -0.3), rng.uniform(0.1, 0.9, m) * L, rng.uniform(0.1, 0.9, m) * L], 1)
    d = np.stack([np.ones(m), rng.normal(0, 0.1, m), rng.normal(0, 0.1, m)], 1)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    dC, dD, dN = rng.uniform(-1, 1, (m, 3)), rng.uniform(-1, 1, m), rng.uniform(-1, 1, (m, 3))
    step, S, beta = h / 2, 64, 2 * h
    gs, gr, _ = g.render_backward(o, d, step, S, beta, dC, dD, dN)
    flat = np.argsort(-np.abs(gs).ravel())[:40]
    eps = 1e-3
    checked = 0
    for fi in flat:
        b, v = divmod(int(fi), 512)
        sp = sdf.copy()
        sp[b, v] += eps
        g.set_payload(0, n, sdf=sp)
        lp = _loss(g, o, d, step, S, beta, dC, dD, dN)
        sp[b, v] -= 2 * eps
        g.set_payload(0, n, sdf=sp)
        lm = _loss(g, o, d, step, S, beta, dC, dD, dN)
        g.set_payload(0, n, sdf=sdf)
        fd = (lp - lm) / (2 * eps)
        assert fd == pytest.approx(gs[b, v], rel=2e-3, abs=1e-6 * np.abs(gs).max()), (b, v)
        checked += 1
    assert checked == 40
    # colour is linear in the payload: gradient equals the FD exactly up to rounding
    for fi in np.argsort(-np.abs(gr).ravel())[:10]:
        b, v, c = np.unravel_index(int(fi), gr.shape)
        rp = rgb.copy()
        rp[b, v, c] += 0.25
        g.set_payload(0, n, rgb=rp)
        lp = _loss(g, o, d, step, S, beta, dC, dD, dN)
        g.set_payload(0, n, rgb=rgb)
        l0 = _loss(g, o, d, step, S, beta, dC, dD, dN)
        assert (lp - l0) / 0.25 == pytest.approx(gr[b, v, c], rel=1e-6)


# --- randomized restated-oracle vs compiled-reference (grid path) -------------------
@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_oracle_equals_reference_random_scenes(seed):
    rng = np.random.default_rng(100 + seed)
    h = [0.0125, 0.015, 0.02][seed]
    og, rg = OracleGrid(h, 8, 2), RefGrid(h, 8, 2)
    pts = rng.uniform(-0.7, 0.7, size=(60, 3))
    R = seed % 3
    r1, r2 = og.allocate_points(pts, R), rg.allocate_points(pts, R)
    assert (r1.blocks_added, r1.blocks_requested) == (r2.blocks_added, r2.blocks_requested)
    co, cr = og.coords(), rg.coords()
    assert set(map(tuple, co)) == set(map(tuple, cr))
    # identical per-coordinate payload
    vals = rng.uniform(-1, 1, size=(len(co), 512)).astype(np.float32)
    wts = (rng.uniform(0, 1, size=(len(co), 512)) > 0.03).astype(np.float32)
    og.set_payload(0, len(co), sdf=vals, weight=wts)
    perm = og.find(cr)
    rg.set_payload(0, len(cr), sdf=vals[perm], weight=wts[perm])
    x = rng.uniform(-0.9, 0.9, size=(20000, 3))
    qo, qr = og.query(x), rg.query(x)
    for k in ("sdf", "grad", "rgb", "valid"):
        assert np.array_equal(qo[k], qr[k]), k
    o = rng.uniform(-2.5, 2.5, size=(500, 3))
    d = rng.uniform(-1, 1, size=(500, 3))
    d[::13, 1] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    mo, mr = og.march(o, d, h / 2, 128), rg.march(o, d, h / 2, 128)
    for k in ("counts", "t", "delta"):
        assert np.array_equal(mo[k], mr[k]), k
