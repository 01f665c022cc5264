"""CPU: the restated fusion + de-noising module against the SPEC's
known answers and properties, and -- where the reference has code for the
pieces it uses (Camera::project, ScaleField::value, voxel_to_world) -- against the
reference compiled verbatim (oracle/_ref)."""
import numpy as np
import pytest

from oracle import OracleGrid, RefGrid, ref_available
from fixtures import SyntheticScene

H = 0.02  # voxel size of the known-answer grids
LOCAL = (3, 3, 3)
LIDX = LOCAL[0] + 8 * LOCAL[1] + 64 * LOCAL[2]


class _Cam:  # the fields OracleGrid's camera conversion reads
    def __init__(self, t, W=32, Hh=24, f=30.0):
        self.fx = self.fy = f
        self.cx, self.cy = (W - 1) / 2.0, (Hh - 1) / 2.0
        self.width, self.height = W, Hh
        self.R = [1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0]
        self.t = list(t)


def _kat_grid(C=1):
    g = OracleGrid(H, 8, C)
    g.allocate_blocks(np.array([[0, 0, 0]]))
    return g


def _kat_cam():
    """Camera 1 m in front of voxel (3,3,3) of block 0 looking down +z: that voxel has z = 1
    and projects on the principal point."""
    x = np.array(LOCAL) * H
    return _Cam((x[0], x[1], x[2] - 1.0))


def _fuse(g, depths, mu=0.24, rgb=None, sem=None):
    cams = [_kat_cam()] * len(depths)
    d = np.stack([np.full((24, 32), v, np.float32) for v in depths])
    g.fuse_begin(color=rgb is not None, semantic=sem is not None)
    rep = g.fuse_frames(d, cams, mu, rgb=rgb, sem=sem)
    g.fuse_finalize()
    return rep, g.get_payload()


def test_single_observation_is_its_own_mean():
    _, p = _fuse(_kat_grid(), [1.03])
    assert p["sdf"][0, LIDX] == pytest.approx(0.03, abs=1e-6)
    assert p["weight"][0, LIDX] == 1.0


def test_two_observations_average():
    _, p = _fuse(_kat_grid(), [1.02, 1.04])
    assert p["sdf"][0, LIDX] == pytest.approx(0.03, abs=1e-6)
    assert p["weight"][0, LIDX] == 2.0


def test_truncation_and_rejection():
    _, p = _fuse(_kat_grid(), [1.5])  # d = 0.5 > mu -> min(d, mu) = 0.24
    assert p["sdf"][0, LIDX] == pytest.approx(0.24, abs=1e-7)
    rep, p = _fuse(_kat_grid(), [0.5])  # d = -0.5 < -mu -> rejected
    assert p["weight"][0, LIDX] == 0.0
    assert rep.rejected > 0 and rep.integrated + rep.rejected == rep.in_view


def test_zero_frames_leave_every_weight_zero():
    g = _kat_grid()
    g.fuse_begin()
    g.fuse_finalize()
    assert not g.get_payload()["weight"].any()


def test_constant_color_scene_fuses_to_that_color():
    W, Hh = 32, 24
    rgb = np.broadcast_to(np.array([0.3, 0.55, 0.8], np.float32), (2, Hh, W, 3)).copy()
    _, p = _fuse(_kat_grid(), [1.02, 1.07], rgb=rgb)
    seen = p["weight"][0] > 0
    assert seen.sum() > 50
    assert np.array_equal(p["rgb"][0][seen], np.broadcast_to(rgb[0, 0, 0], (int(seen.sum()), 3)))


def test_logits_are_unit_norm():
    W, Hh, C = 32, 24, 3
    sem = np.random.default_rng(0).uniform(0.0, 2.0, (2, Hh, W, C)).astype(np.float32)
    _, p = _fuse(_kat_grid(C), [1.02, 1.07], sem=sem)
    seen = p["weight"][0] > 0
    n = np.linalg.norm(p["logits"][0][seen].astype(np.float64), axis=1)
    assert seen.sum() > 50 and np.allclose(n, 1.0, atol=1e-6)


def test_channel_flags_are_enforced():
    from oracle import OracleError

    g = _kat_grid()
    g.fuse_begin(color=True, semantic=False)
    with pytest.raises(OracleError):
        g.fuse_frames(np.ones((1, 24, 32), np.float32), [_kat_cam()], 0.24)  # rgb missing


def _scene(C=4, n_frames=6, W=48, Hh=36):
    sc = SyntheticScene(n_frames=n_frames, width=W, height=Hh, label_channels=C)
    cams = sc.cameras()
    depth, rgb, sem = sc.frames(cams)
    return sc, cams, depth, rgb, sem


def _scene_grid(depth, cams, h=0.05, C=4, dil=1):
    g = OracleGrid(h, 8, C)
    g.allocate_frames(depth, cams, dil)
    return g


def test_fusion_is_order_independent_and_bounded():
    sc, cams, depth, rgb, sem = _scene()
    mu = 8 * 0.05 * 1
    out = []
    for order in (range(len(cams)), reversed(range(len(cams)))):
        order = list(order)
        g = _scene_grid(depth, cams)
        g.fuse_begin()
        for f in order:  # one frame per call: the sums must not care
            g.fuse_frames(depth[f:f + 1], [cams[f]], mu, rgb=rgb[f:f + 1], sem=sem[f:f + 1])
        g.fuse_finalize()
        out.append(g.get_payload())
    for k in ("sdf", "weight", "rgb", "logits"):
        assert np.array_equal(out[0][k], out[1][k]), k
    seen = out[0]["weight"] > 0
    assert seen.mean() > 0.2
    assert np.abs(out[0]["sdf"][seen]).max() <= mu * (1 + 1e-7)


def test_fused_zero_crossing_near_ground_truth_surface():
    """zero-crossing of the fused SDF within 1 voxel of the GT surface for >= 95%
    of surface-adjacent cells (synthetic room, GT depth, phi = 1)."""
    h = 0.04
    sc, cams, depth, rgb, sem = _scene(n_frames=24, W=96, Hh=72)
    g = _scene_grid(depth, cams, h=h, dil=1)
    OracleGrid.set_threads(8)
    g.fuse_begin(False, False)
    g.fuse_frames(depth, cams, 8 * h)
    g.fuse_finalize()
    OracleGrid.set_threads(1)
    p = g.get_payload()
    coords = g.coords()
    hits = []
    v = np.arange(512)
    loc = np.stack([v % 8, (v // 8) % 8, v // 64], 1)
    for b in range(len(coords)):
        s, w = p["sdf"][b], p["weight"][b]
        for axis, step in ((0, 1), (1, 8), (2, 64)):
            ok = (loc[:, axis] < 7) & (w > 0)
            i = v[ok]
            j = i + step
            m = (w[j] > 0) & (np.sign(s[i]) != np.sign(s[j])) & (s[i] != 0)
            i, j = i[m], j[m]
            t = s[i] / (s[i] - s[j])
            x = (coords[b] * 8 + loc[i]) * h
            x[:, axis] += t * h
            hits.append(x)
    x = np.concatenate(hits)
    assert len(x) > 500
    err = np.abs(sc.sdf(x))
    assert (err < h).mean() >= 0.95


@pytest.mark.skipif(not ref_available(), reason="reference not compiled (oracle/_ref)")
def test_oracle_fusion_matches_reference_primitives_bit_exact():
    """Same association rules evaluated through the reference's own Camera::project,
    ScaleField::value and voxel_to_world (oracle/ref_capi.cpp) -> identical payloads."""
    sc, cams, depth, rgb, sem = _scene()
    rng = np.random.default_rng(3)
    scales = rng.uniform(0.9, 1.1, (len(cams), 4, 5))
    mu = 0.4
    og = _scene_grid(depth, cams)
    rg = RefGrid(0.05, 8, 4)
    rg.allocate_blocks(og.coords())
    for g in (og, rg):
        g.fuse_begin()
        g.fuse_frames(depth, cams, mu, rgb=rgb, sem=sem, scales=scales)
        g.fuse_finalize()
    a, b = og.get_payload(), rg.get_payload()
    assert (a["weight"] > 0).mean() > 0.2
    for k in ("sdf", "weight", "rgb", "logits"):
        assert np.array_equal(a[k], b[k]), k


# ---- denoise -----------------------------------------------------------
def _dense_grid(C=2, nb=(2, 2, 2), valid=None, seed=0):
    """All blocks of an nb box allocated; payload random; validity from `valid` (bool
    [X][Y][Z] over the voxel lattice) or all valid."""
    g = OracleGrid(0.05, 8, C)
    cs = np.array([[x, y, z] for z in range(nb[2]) for y in range(nb[1]) for x in range(nb[0])], np.int32)
    g.allocate_blocks(cs)
    A = len(cs)
    rng = np.random.default_rng(seed)
    sdf = rng.normal(0, 1, (A, 512)).astype(np.float32)
    rgb = rng.uniform(0, 1, (A, 512, 3)).astype(np.float32)
    lg = rng.normal(0, 1, (A, 512, C)).astype(np.float32)
    w = np.ones((A, 512), np.float32)
    if valid is not None:
        v = np.arange(512)
        for b, c in enumerate(cs):
            w[b] = valid[c[0] * 8 + v % 8, c[1] * 8 + (v // 8) % 8, c[2] * 8 + v // 64]
    g.set_payload(0, A, sdf=sdf, weight=w, rgb=rgb, logits=lg)
    return g, cs


def _to_dense(g, cs, key, nb=(2, 2, 2)):
    p = g.get_payload()[key]
    p = p.reshape(len(cs), 512, -1)
    out = np.zeros((nb[0] * 8, nb[1] * 8, nb[2] * 8, p.shape[-1]))
    v = np.arange(512)
    for b, c in enumerate(cs):
        out[c[0] * 8 + v % 8, c[1] * 8 + (v // 8) % 8, c[2] * 8 + v // 64] = p[b]
    return out


def test_denoise_radius_zero_is_identity():
    g, cs = _dense_grid()
    before = g.get_payload()
    g.denoise(1.0, 0)
    after = g.get_payload()
    for k in before:
        assert np.array_equal(before[k], after[k]), k


def test_denoise_constant_field_unchanged():
    g, cs = _dense_grid(C=1)
    A = len(cs)
    g.set_payload(0, A, sdf=np.full((A, 512), 0.37, np.float32), rgb=np.full((A, 512, 3), 0.2, np.float32),
                  logits=np.full((A, 512, 1), -1.5, np.float32))
    g.denoise(1.0, 2)
    p = g.get_payload()
    assert (p["sdf"] == np.float32(0.37)).all() and (p["rgb"] == np.float32(0.2)).all()
    assert (p["logits"] == np.float32(-1.5)).all()


def test_denoise_impulse_matches_dense_convolution():
    """impulse, radius 1, sigma 1 -> the 3^3 Gaussian stencil (renormalised),
    vs a dense-array convolution within 1e-6."""
    g, cs = _dense_grid(C=1)
    A = len(cs)
    sdf = np.zeros((A, 512), np.float32)
    c = (7, 8, 9)  # lattice voxel straddling block faces
    b = [i for i, cc in enumerate(cs) if tuple(cc) == (c[0] // 8, c[1] // 8, c[2] // 8)][0]
    sdf[b, c[0] % 8 + 8 * (c[1] % 8) + 64 * (c[2] % 8)] = 1.0
    g.set_payload(0, A, sdf=sdf)
    g.denoise(1.0, 1)
    out = _to_dense(g, cs, "sdf")[..., 0]
    d = np.arange(-1, 2)
    k3 = np.exp(-(d[:, None, None] ** 2 + d[None, :, None] ** 2 + d[None, None, :] ** 2) / 2.0)
    k3 /= k3.sum()
    want = np.zeros_like(out)
    want[c[0] - 1:c[0] + 2, c[1] - 1:c[1] + 2, c[2] - 1:c[2] + 2] = k3
    assert np.abs(out - want).max() < 1e-6


def test_denoise_with_holes_matches_direct_masked_sum():
    """Validity-restricted, renormalised Gaussian vs a direct numpy masked sum (radius 2,
    sigma 0.8); invalid voxels keep their value; min/max bounds preserved."""
    rng = np.random.default_rng(5)
    valid = rng.uniform(size=(16, 16, 16)) > 0.3
    g, cs = _dense_grid(C=2, valid=valid)
    before = {k: _to_dense(g, cs, k) for k in ("sdf", "rgb", "logits")}
    g.denoise(0.8, 2)
    r, s = 2, 0.8
    d = np.arange(-r, r + 1)
    gw = np.exp(-(d ** 2) / (2 * s * s))
    for k in ("sdf", "rgb", "logits"):
        x = before[k]
        out = _to_dense(g, cs, k)
        pad = np.pad(x * valid[..., None], ((r, r), (r, r), (r, r), (0, 0)))
        pv = np.pad(valid.astype(np.float64), r)
        num = np.zeros_like(x)
        den = np.zeros(valid.shape)
        for i, a in enumerate(d):
            for j, bb in enumerate(d):
                for l, cc in enumerate(d):
                    w = gw[i] * gw[j] * gw[l]
                    sl = (slice(r + a, r + a + 16), slice(r + bb, r + bb + 16), slice(r + cc, r + cc + 16))
                    num += w * pad[sl]
                    den += w * pv[sl]
        want = np.where(valid[..., None], num / np.maximum(den, 1e-300)[..., None], x)
        assert np.abs(out - want).max() <= 1e-6 * max(1.0, np.abs(want).max()), k
        assert np.array_equal(out[~valid], x[~valid]), k
        assert out[valid].min() >= x[valid].min() - 1e-6 and out[valid].max() <= x[valid].max() + 1e-6
