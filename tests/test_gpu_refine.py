"""GPU: the refinement loop pieces -- batch sampling from device frames
(K17) vs the host Camera::ray_direction restatement, Eikonal band points (K16) vs the oracle,
and the composed Refiner reducing the losses and the geometric error of the extracted mesh."""
import numpy as np
import pytest

from common import gpu_grid_from, scene_case

pytestmark = pytest.mark.gpu


def _frames(n=6, W=64, H=48, C=4):
    from fixtures import SyntheticScene

    sc = SyntheticScene(n_frames=n, width=W, height=H, label_channels=C)
    cams = sc.cameras()
    depth, rgb, sem, nrm = sc.frames(cams, normals=True)
    return sc, cams, depth, rgb, nrm


def test_sample_frame_rays_match_host_camera_rays():
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid
    from paper_2305_13220_b200._lib import Camera, check
    from paper_2305_13220_b200.refine import frames_to_device

    sc, cams, depth, rgb, nrm = _frames()
    g = SparseDenseGrid(0.05, 8, 1)
    r, dp, nm = frames_to_device(rgb, depth, nrm)
    ipb, rpi = 5, 300
    n = ipb * rpi
    o = np.empty((n, 3)), np.empty((n, 3))
    outs = {"o": np.empty((n, 3)), "d": np.empty((n, 3)), "t": np.empty((n, 3), np.float32),
            "pd": np.empty(n, np.float32), "pn": np.empty((n, 3), np.float32),
            "ci": np.empty(n, np.uint32), "px": np.empty(n, np.uint32)}
    arr = (Camera * len(cams))(*cams)
    import ctypes

    check(g._lib.svr_sample_frame_rays(g._h, ctypes.addressof(arr), len(cams), r.data_ptr(), dp.data_ptr(),
                                       nm.data_ptr(), ipb, rpi, 42, *[outs[k].ctypes.data for k in
                                                                       ("o", "d", "t", "pd", "pn", "ci", "px")]))
    W, H = 64, 48
    f = outs["px"] // (W * H)
    p = outs["px"] % (W * H)
    assert np.array_equal(f, outs["ci"])
    assert len(np.unique(f)) > 1 and np.all(f == np.repeat(f[::rpi], rpi))  # one frame per image slot
    for fr in np.unique(f):
        ho, hd = sc.image_rays(int(fr))
        m = f == fr
        assert np.array_equal(outs["o"][m], ho[p[m]]) and np.array_equal(outs["d"][m], hd[p[m]])
    flat = lambda a, k: a.reshape(-1, k)  # noqa: E731
    assert np.array_equal(outs["t"], flat(rgb, 3)[outs["px"]])
    assert np.array_equal(outs["pd"], depth.reshape(-1)[outs["px"]])
    assert np.array_equal(outs["pn"], flat(nrm, 3)[outs["px"]])


def test_band_points_match_oracle():
    import ctypes

    case = scene_case()
    g = gpu_grid_from(case)
    g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    band = 0.05
    cap = 200000
    pts = np.empty((cap, 3))
    nb = ctypes.c_uint64()
    from paper_2305_13220_b200._lib import check

    check(g._lib.svr_band_points(g._h, band, cap, pts.ctypes.data, ctypes.byref(nb)))
    got = pts[:nb.value]
    # oracle: every marched sample, fp64 sdf, same band
    m = case["oracle"].march(case["o"], case["d"], case["step"], 64)
    mask = np.arange(64)[None, :] < m["counts"][:, None]
    x = case["o"][:, None, :] + m["t"][:, :, None] * case["d"][:, None, :]
    q = case["oracle"].query(x[mask])
    keep = (q["valid"] == 1) & (np.abs(q["sdf"]) < band)
    want = x[mask][keep]
    assert len(want) > 1000
    assert abs(len(got) - len(want)) <= max(2, 0.002 * len(want))  # fp32 vs fp64 sdf at the edge
    if len(got) == len(want):
        assert np.array_equal(got, want)


def test_refiner_reduces_losses_and_surface_error():
    """Fused-from-distorted-depth initialisation -> refine with GT colour, the distorted depth
    prior (the per-batch affine fit absorbs the scale) and GT normals: the losses fall and the
    extracted mesh moves toward the GT surface."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid
    from paper_2305_13220_b200.refine import RefineConfig, Refiner, frames_to_device

    sc, cams, depth, rgb, nrm = _frames(n=16, W=96, H=72)
    h = 0.04
    g = SparseDenseGrid(h, 8, 4)
    g.allocate_for_frames(depth, cams, 1)
    rng = np.random.default_rng(0)
    scale = 1.0 + 0.08 * np.sin(np.linspace(0, 3, depth.shape[2]))[None, None, :]
    bad = (depth * scale * (1 + 0.02 * rng.normal(size=depth.shape))).astype(np.float32)
    mu = 8 * h
    g.fuse_all(bad, cams, mu, rgb=rgb)

    def surface_err():
        m = g.marching_cubes(0.0)
        return float(np.mean(np.abs(sc.sdf(m["vertices"])))) if len(m["vertices"]) else 1.0

    e0 = surface_err()
    r, dp, nm = frames_to_device(rgb, bad, nrm)
    cfg = RefineConfig(rays_per_image=512, images_per_batch=16, lr=2e-3, uniform_points=4096, band_cap=16384)
    ref = Refiner(g, cams, r, dp, nm, step_m=h / 2, beta=2 * h, mu=mu, config=cfg)
    trace = ref.run(120, log_every=20)
    torch.cuda.synchronize()
    e1 = surface_err()
    first, last = trace[0], trace[-1]
    assert last["L_c"] < 0.8 * first["L_c"]
    assert last["total"] < first["total"]
    assert e1 < e0, (e0, e1)


def test_native_refiner_matches_python_refiner():
    """svr_refiner_* (C++ host loop) == refine.Refiner (Python host loop) step for step."""
    import torch

    from paper_2305_13220_b200 import SparseDenseGrid
    from paper_2305_13220_b200.refine import NativeRefiner, RefineConfig, Refiner, frames_to_device

    sc, cams, depth, rgb, nrm = _frames(n=8, W=64, H=48)
    h = 0.04
    cfg = RefineConfig(rays_per_image=256, images_per_batch=8, uniform_points=2048, band_cap=8192)
    grids, traces = [], []
    for native in (False, True):
        g = SparseDenseGrid(h, 8, 4)
        g.allocate_for_frames(depth, cams, 1)
        g.fuse_all(depth, cams, 8 * h, rgb=rgb)
        r, dp, nm = frames_to_device(rgb, depth, nrm)
        kw = dict(step_m=h / 2, beta=2 * h, mu=8 * h, config=cfg)
        ref = NativeRefiner(g, cams, r, dp, nm, **kw) if native else Refiner(g, cams, r, dp, nm, **kw)
        traces.append(ref.run(6, log_every=1))
        torch.cuda.synchronize()
        grids.append(g.get_payload())
    for a, b in zip(*traces):
        for k in ("L_c", "L_d", "L_n", "n_c", "n_d", "n_n"):
            assert a[k] == pytest.approx(b[k], rel=1e-4), (a["step"], k)
    for k in ("sdf", "rgb"):
        d = np.abs(grids[0][k] - grids[1][k])
        assert d.max() < 1e-3, k  # atomic-order differences only
        assert (d > 1e-6).mean() < 0.01, k
