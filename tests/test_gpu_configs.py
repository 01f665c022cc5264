"""GPU vs oracle at BASELINE.json's own CPU-runnable configurations:
cfg1 -- 5x5x3 m room, 2 cm voxels, R = 2 activation from 24 ring frames, 4096 rays x <= 64
samples, fwd+bwd; cfg2 -- the same grid, one full 640x480 image, forward only."""
import numpy as np
import pytest

from common import assert_close
from oracle import OracleGrid

pytestmark = pytest.mark.gpu

CFG1 = dict(room_w=5.0, room_d=5.0, room_h=3.0, n_objects=4, seed=1, width=640, height=480, fov_deg=70.0,
            label_channels=4, n_frames=24)
H, R = 0.02, 2


@pytest.fixture(scope="module")
def cfg1():
    from paper_2305_13220_b200 import SparseDenseGrid
    from fixtures import SyntheticScene, uniform_floats

    sc = SyntheticScene(**CFG1)
    cams = sc.cameras()
    depth = sc.depth(cams)
    g = SparseDenseGrid(H, 8, 4)
    g.allocate_for_frames(depth, cams, R)
    og = OracleGrid(H, 8, 4)
    og.allocate_frames(depth, cams, R)
    coords = og.coords()
    assert np.array_equal(g.coords(), coords)  # activation: same blocks, same order
    assert 15000 < len(coords) < 40000
    pay = sc.fill_payload(H, coords, 8 * H * R, 4)
    g.set_payload(0, len(coords), **pay)
    og.set_payload(0, len(coords), **pay)
    o, d = sc.rays(24, 4096 // 24 + 1, seed=0)
    o, d = o[:4096], d[:4096]
    u = uniform_floats(7 * 4096, 1).reshape(4096, 7)
    return {"scene": sc, "g": g, "og": og, "o": o, "d": d, "dC": np.ascontiguousarray(u[:, :3]),
            "dD": np.ascontiguousarray(u[:, 3]), "dN": np.ascontiguousarray(u[:, 4:])}


@pytest.mark.parametrize("lookup", [2, 1], ids=["dense", "hash"])
def test_cfg1_forward_backward(cfg1, lookup):
    g, og = cfg1["g"], cfg1["og"]
    step, beta = H / 2, 2 * H
    g.set_lookup(lookup)
    assert g.info().lookup_mode == lookup
    out = g.render_forward(cfg1["o"], cfg1["d"], step, 64, beta)
    OracleGrid.set_threads(8)
    try:
        ref = og.render_forward(cfg1["o"], cfg1["d"], step, 64, beta)
        g.grad_zero()
        g.render_backward(cfg1["dC"], cfg1["dD"], cfg1["dN"])
        gs, gr, act = og.render_backward(cfg1["o"], cfg1["d"], step, 64, beta, cfg1["dC"], cfg1["dD"], cfg1["dN"])
    finally:
        OracleGrid.set_threads(1)
    assert np.array_equal(out["n_samples"], ref["n_samples"])
    assert ref["n_valid"].sum() > 100_000
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(out[k], ref[k], what=k)
    ggs, ggr = g.grads()
    assert_close(ggs, gs, what="grad_sdf")
    assert_close(ggr, gr, what="grad_rgb")
    assert np.array_equal(g.active_mask(), act)
    g.set_lookup(0)


@pytest.mark.parametrize("lookup", [2, 1], ids=["dense", "hash"])
def test_cfg2_full_image_forward(cfg1, lookup):
    g, og = cfg1["g"], cfg1["og"]
    o, d = cfg1["scene"].image_rays(0)
    assert len(o) == 640 * 480
    step, beta = H / 2, 2 * H
    g.set_lookup(lookup)
    g.set_tuning("records", 0)  # inference
    out = g.render_forward(o, d, step, 64, beta)
    g.set_tuning("records", 1)
    g.set_lookup(0)
    OracleGrid.set_threads(16)
    try:
        ref = og.render_forward(o, d, step, 64, beta)
    finally:
        OracleGrid.set_threads(1)
    assert np.array_equal(out["n_samples"], ref["n_samples"])
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(out[k], ref[k], what=k)
