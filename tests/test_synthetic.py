"""CPU: synthetic fixture generator (restates proj/src/core/synthetic.cpp:42-192)."""
import numpy as np
import pytest

from fixtures import SyntheticScene, uniform_floats


@pytest.fixture(scope="module")
def scene():
    return SyntheticScene(room_w=2.4, room_d=2.2, room_h=2.0, n_objects=4, width=64, height=48, n_frames=12)


def test_ring_cameras_are_orthonormal(scene):
    for f in range(12):
        c = scene.camera_for_frame(f)
        R = np.array(c.R).reshape(3, 3)
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-12
        assert abs(np.linalg.det(R) - 1) < 1e-12
        assert c.cx == (64 - 1) / 2 and c.cy == (48 - 1) / 2


def test_depth_hits_the_surface(scene):
    cams = scene.cameras()
    depth = scene.depth(cams)
    assert depth.shape == (12, 48, 64) and (depth > 0).all()
    # unprojected GT depth lies on the zero level set of the analytic sdf
    c = cams[3]
    R, t = np.array(c.R).reshape(3, 3), np.array(c.t)
    ys, xs = np.mgrid[0:48:7, 0:64:9]
    d = depth[3, ys, xs].astype(np.float64)
    xc = np.stack([(xs - c.cx) / c.fx * d, (ys - c.cy) / c.fy * d, d], -1).reshape(-1, 3)
    pw = xc @ R.T + t
    assert np.abs(scene.sdf(pw)).max() < 2e-6  # float32 depth rounding


def test_payload_is_truncated_and_valid(scene):
    coords = np.array([[0, 0, -8], [-3, 2, 1], [5, -5, 5]], np.int32)
    p = scene.fill_payload(0.02, coords, 0.32, 4)
    assert np.abs(p["sdf"]).max() <= 0.32 + 1e-7
    assert (p["weight"] == 1).all()
    assert ((p["rgb"] >= 0) & (p["rgb"] <= 1)).all()
    assert np.array_equal(p["logits"].sum(-1), np.ones((3, 512)))


def test_rays_are_unit_and_deterministic(scene):
    o1, d1 = scene.rays(4, 100, seed=0)
    o2, d2 = scene.rays(4, 100, seed=0)
    assert np.array_equal(d1, d2) and np.array_equal(o1, o2)
    np.testing.assert_allclose(np.linalg.norm(d1, axis=1), 1.0, rtol=1e-15)
    u = uniform_floats(1000, 1)
    assert u.min() >= -1 and u.max() < 1 and abs(u.mean()) < 0.1


import oracle  # noqa: E402

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


@needs_ref
@pytest.mark.parametrize("spec", [
    dict(room_w=2.4, room_d=2.2, room_h=2.0, n_objects=4, width=64, height=48, n_frames=12),
    # the bench's cfg3 scene (11 x 11 x 3 m, 640 x 480, 64 ring poses) on a frame subset
    dict(room_w=11.0, room_d=11.0, room_h=3.0, n_objects=4, width=640, height=480, n_frames=64, seed=1),
    dict(room_w=5.0, room_d=5.0, room_h=3.0, n_objects=3, width=96, height=80, n_frames=24, seed=7,
         texture_amplitude=0.4, texture_frequency=2.5, fov_deg=60.0, label_channels=6),
])
def test_fixture_equals_reference_generator(spec):
    """fixtures/synthetic.cpp restates proj/src/core/synthetic.cpp:42-192; the reference's own
    SyntheticScene (compiled verbatim into oracle/_ref) must give the same cameras, GT frames,
    payloads, rays and upstream gradients bit for bit (SURVEY.md 8(d) input recipes)."""
    fx, ref = SyntheticScene(**spec), oracle.RefScene(**spec)
    frames = [0, 1, spec["n_frames"] // 2, spec["n_frames"] - 1]
    cf, cr = fx.cameras(spec["n_frames"]), ref.cameras(spec["n_frames"])
    assert all(bytes(a) == bytes(b) for a, b in zip(cf, cr))
    sub_f, sub_r = [cf[i] for i in frames], [cr[i] for i in frames]
    C = spec.get("label_channels", 4)
    a = fx.frames(sub_f, normals=True)
    b = ref.frames(sub_r, normals=True)
    for x, y, name in zip(a, b, ("depth", "rgb", "sem", "normal")):
        assert np.array_equal(x, y), name
    assert a[2].shape[-1] == C
    o1, d1 = fx.rays(8, 512, seed=0)
    o2, d2 = ref.rays(8, 512, seed=0)
    assert np.array_equal(o1, o2) and np.array_equal(d1, d2)
    oi, di = fx.image_rays(3)
    oj, dj = ref.image_rays(3)
    assert np.array_equal(oi, oj) and np.array_equal(di, dj)
    rng = np.random.default_rng(0)
    half = np.array([spec["room_w"], spec["room_d"], spec["room_h"]]) / 2
    h = 0.02
    coords = np.unique(np.floor(rng.uniform(-half, half, size=(300, 3)) / (8 * h)).astype(np.int32), axis=0)
    p, q = fx.fill_payload(h, coords, 8 * h * 2, C), ref.fill_payload(h, coords, 8 * h * 2, C)
    for k in p:
        assert np.array_equal(p[k], q[k]), k
    pts = rng.uniform(-half, half, size=(4096, 3))
    assert np.array_equal(fx.sdf(pts), ref.sdf(pts))
    assert np.array_equal(uniform_floats(7000, 1), oracle.RefScene.uniform_floats(7000, 1))
