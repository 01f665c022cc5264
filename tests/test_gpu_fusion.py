"""GPU: fusion (K12) and de-noising (K13) vs the CPU oracle, bit-exact (SURVEY.md 8(f)
rank 3).  Both sides evaluate the same fp64 association arithmetic with
explicit round-to-nearest ops and 32.32 fixed-point sums, so every payload word agrees."""
import numpy as np
import pytest

from oracle import OracleGrid
from fixtures import SyntheticScene

pytestmark = pytest.mark.gpu


def _case(C=4, n_frames=10, W=80, Hh=60, h=0.05, dil=1, seed=0):
    sc = SyntheticScene(n_frames=n_frames, width=W, height=Hh, label_channels=max(C, 4), seed=seed)
    cams = sc.cameras()
    depth, rgb, sem = sc.frames(cams, label_channels=max(C, 4))
    sem = np.ascontiguousarray(sem[..., :C])
    og = OracleGrid(h, 8, C)
    og.allocate_frames(depth, cams, dil)
    return sc, cams, depth, rgb, sem, og


def _gpu_grid(og, h, C):
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(h, 8, C)
    idx = g.allocate_blocks(og.coords())
    assert np.array_equal(idx, np.arange(og.block_count(), dtype=np.uint32))
    return g


def _same(a, b, keys=("sdf", "weight", "rgb", "logits")):
    for k in keys:
        assert a[k].shape == b[k].shape, k
        bad = a[k].view(np.uint32) != b[k].view(np.uint32)
        assert not bad.any(), f"{k}: {int(bad.sum())} words differ"


@pytest.mark.parametrize("C", [4, 11])  # register-resident logit sums / generic HBM path
def test_fuse_matches_oracle_bit_exact(C):
    sc, cams, depth, rgb, sem, og = _case(C=C)
    g = _gpu_grid(og, 0.05, C)
    mu = 0.4
    for grid in (og, g):
        grid.fuse_begin(True, True)
    ro = og.fuse_frames(depth, cams, mu, rgb=rgb, sem=sem)
    rg = g.fuse_frames(depth, cams, mu, rgb=rgb, semantic=sem)
    assert (rg.frames, rg.in_view, rg.integrated, rg.rejected) == (ro.frames, ro.in_view, ro.integrated,
                                                                    ro.rejected)
    assert rg.integrated > 10000 and rg.rejected > 0
    og.fuse_finalize()
    g.fuse_finalize()
    _same(g.get_payload(), og.get_payload())


def test_fuse_with_scale_fields_and_split_calls():
    sc, cams, depth, rgb, sem, og = _case(C=4, n_frames=8)
    g = _gpu_grid(og, 0.05, 4)
    scales = np.random.default_rng(1).uniform(0.85, 1.15, (len(cams), 5, 7))
    og.fuse_begin(True, False)
    og.fuse_frames(depth, cams, 0.3, rgb=rgb, scales=scales)
    og.fuse_finalize()
    g.fuse_begin(True, False)
    for f0 in (0, 3, 5):  # frames in uneven batches
        f1 = {0: 3, 3: 5, 5: 8}[f0]
        g.fuse_frames(depth[f0:f1], cams[f0:f1], 0.3, rgb=rgb[f0:f1], scales=scales[f0:f1])
    g.fuse_finalize()
    _same(g.get_payload(), og.get_payload())


def test_fuse_order_independent_on_gpu():
    sc, cams, depth, rgb, sem, og = _case(C=4, n_frames=6)
    outs = []
    for order in (list(range(6)), [5, 2, 0, 4, 1, 3]):
        g = _gpu_grid(og, 0.05, 4)
        g.fuse_begin(True, True)
        for f in order:
            g.fuse_frames(depth[f:f + 1], [cams[f]], 0.4, rgb=rgb[f:f + 1], semantic=sem[f:f + 1])
        g.fuse_finalize()
        outs.append(g.get_payload())
    _same(outs[0], outs[1])


def test_fuse_then_render_sees_fused_validity():
    """finalize rebuilds validity: the renderer and query see exactly the fused voxels."""
    sc, cams, depth, rgb, sem, og = _case(C=4, n_frames=8)
    g = _gpu_grid(og, 0.05, 4)
    og.fuse_begin(True, True)
    og.fuse_frames(depth, cams, 0.4, rgb=rgb, sem=sem)
    og.fuse_finalize()
    g.fuse_all(depth, cams, 0.4, rgb=rgb, semantic=sem)
    x = og.coords()[:200].astype(np.float64) * 8 * 0.05 + 0.17
    q, qo = g.query(x), og.query(x)
    assert np.array_equal(q["valid"], qo["valid"]) and q["valid"].any()
    assert np.array_equal(q["sdf"], qo["sdf"])


def test_zero_frames_and_late_blocks():
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(0.05, 8, 2)
    g.allocate_blocks(np.array([[0, 0, 0]]))
    g.fuse_begin(False, False)
    g.allocate_blocks(np.array([[1, 0, 0]]))  # joins the open session with zero sums
    g.fuse_finalize()
    assert not g.get_payload()["weight"].any()


@pytest.mark.parametrize("radius,sigma", [(1, 1.0), (2, 0.7), (4, 1.5), (0, 1.0)])
def test_denoise_matches_oracle_bit_exact(radius, sigma):
    sc, cams, depth, rgb, sem, og = _case(C=5, n_frames=8)
    g = _gpu_grid(og, 0.05, 5)
    og.fuse_begin(True, True)
    og.fuse_frames(depth, cams, 0.4, rgb=rgb, sem=sem)
    og.fuse_finalize()
    g.fuse_all(depth, cams, 0.4, rgb=rgb, semantic=sem)
    OracleGrid.set_threads(8)
    og.denoise(sigma, radius)
    OracleGrid.set_threads(1)
    g.denoise(sigma, radius)
    _same(g.get_payload(), og.get_payload())


def test_fuse_denoise_hash_lookup_mode():
    """the same fusion + denoise through the hash lookup (no dense AABB index)."""
    sc, cams, depth, rgb, sem, og = _case(C=4, n_frames=6)
    g = _gpu_grid(og, 0.05, 4)
    g.set_lookup(1)
    og.fuse_begin(True, True)
    og.fuse_frames(depth, cams, 0.4, rgb=rgb, sem=sem)
    og.fuse_finalize()
    og.denoise(1.0, 2)
    g.fuse_all(depth, cams, 0.4, rgb=rgb, semantic=sem)
    g.denoise(1.0, 2)
    _same(g.get_payload(), og.get_payload())
