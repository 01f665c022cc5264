"""CPU: synthetic fixture generator (restates proj/src/core/synthetic.cpp:42-192)."""
import numpy as np
import pytest

from paper_2305_13220_b200.synthetic import SyntheticScene, uniform_floats


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
