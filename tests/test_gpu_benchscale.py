"""GPU vs oracle on the BENCHMARK's own workload (BASELINE.json configs[2] / [3]):

* cfg3 -- the bench's grid (290k blocks from 64 ring frames, 1 cm voxels, R = 2) and the first
  65,536 of the bench's 1,048,576 rays, forward + backward, in both lookup modes (dense AABB
  index and the hash table): sample counts and active-block set bit-exact, rgb / depth /
  normal / wsum and both gradient planes within |gpu - oracle| <= 1e-4 |oracle| + 1e-6
  max|oracle|;
* cfg4 -- activation from the 300 GT depth frames: the coordinate list equals the restated
  oracle's (same ascending packed-key order) and, as a set, the compiled reference's
  allocate_for_frames (allocation.cpp:56-83); the reports agree.

The whole 1M-ray step is compared with the oracle by bench.py itself (its `parity` object).
"""
import numpy as np
import pytest

from common import assert_close

pytestmark = pytest.mark.gpu

N_RAYS = 65536


@pytest.fixture(scope="module")
def cfg3():
    import oracle
    from fixtures.workloads import CFG3, activation_frames, fill_in_chunks, make_scene, rays_for_rank
    from oracle import OracleGrid
    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG3
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    coords = g.coords()
    og = OracleGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    assert np.array_equal(og.allocate_blocks(coords), np.arange(len(coords), dtype=np.uint32))

    def sink(f, n, p):
        g.set_payload(f, n, **p)
        og.set_payload(f, n, **p)

    fill_in_chunks(scene, cfg, coords, sink)
    rays = rays_for_rank(scene, cfg, 0, 1)
    o, d, dC, dD, dN = (a[:N_RAYS] for a in rays)
    S, step, beta = cfg["max_samples"], cfg["h"] / 2, 2 * cfg["h"]
    OracleGrid.set_threads(16)
    try:
        ref = og.render_forward(o, d, step, S, beta)
        gs, gr, act = og.render_backward(o, d, step, S, beta, dC, dD, dN)
    finally:
        OracleGrid.set_threads(1)
    del og
    assert 250_000 < len(coords) < 350_000
    return {"g": g, "o_all": rays[0], "d_all": rays[1], "o": o, "d": d, "dC": dC, "dD": dD, "dN": dN, "S": S, "step": step, "beta": beta,
            "ref": ref, "gs": gs, "gr": gr, "act": act, "oracle_mod": oracle}


@pytest.mark.parametrize("lookup", [2, 1], ids=["dense", "hash"])
def test_bench_grid_ray_subset_matches_oracle(cfg3, lookup):
    c = cfg3
    g = c["g"]
    g.set_lookup(lookup)
    assert g.info().lookup_mode == lookup
    g.grad_zero()
    out = g.render_forward(c["o"], c["d"], c["step"], c["S"], c["beta"])
    g.render_backward(c["dC"], c["dD"], c["dN"])
    ref = c["ref"]
    assert np.array_equal(out["n_samples"], ref["n_samples"])
    assert int(ref["n_valid"].sum()) > 3_000_000
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(out[k], ref[k], what=k)
    gs, gr = g.grads()
    assert np.array_equal(g.active_mask(), c["act"])
    assert_close(gs, c["gs"], what="grad_sdf")
    assert_close(gr, c["gr"], what="grad_rgb")
    g.set_lookup(0)


def test_bench_rays_march_same_in_both_lookup_modes(cfg3):
    """All 1,048,576 bench rays: the hash-mode march (superblock distances, block-distance
    bricks near the blocks, hash probes nowhere) emits the same counts and t values, bit for
    bit, as the dense-index march -- both are the reference's march_ray (grid.cpp:337-353),
    which the 65,536-ray subset above checks against the oracle directly."""
    c = cfg3
    g = c["g"]
    S, step = c["S"], c["step"]
    try:
        for a in range(0, len(c["o_all"]), 1 << 18):
            o, d = c["o_all"][a:a + (1 << 18)], c["d_all"][a:a + (1 << 18)]
            g.set_lookup(2)
            md = g.march(o, d, step, S)
            g.set_lookup(1)
            mh = g.march(o, d, step, S)
            assert np.array_equal(md["counts"], mh["counts"])
            valid = np.arange(S)[None, :] < md["counts"][:, None]
            assert np.array_equal(md["t"][valid].view(np.uint64), mh["t"][valid].view(np.uint64))
    finally:
        g.set_lookup(0)


def test_cfg4_activation_matches_reference():
    """300 GT depth frames (640x480) -> 290k blocks: same coordinate list as the restated
    oracle (ascending packed-key order within the call), same set and report as the compiled
    reference, whose indices follow its std::unordered_set iteration order."""
    import oracle
    from fixtures.workloads import CFG4, make_scene
    from oracle import OracleGrid
    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG4
    scene = make_scene(cfg)
    cams = scene.cameras(cfg["act_frames"])
    depth = scene.depth(cams)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    rep = g.allocate_for_frames(depth, cams, cfg["dilation"])
    coords = g.coords()
    og = OracleGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    orep = og.allocate_frames(depth, cams, cfg["dilation"])
    assert np.array_equal(coords, og.coords())
    assert (rep.blocks_added, rep.blocks_requested, rep.pixels_used) == \
        (orep.blocks_added, orep.blocks_requested, orep.pixels_used)
    assert 250_000 < len(coords) < 350_000
    if oracle.ref_available():
        rg = oracle.RefGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
        rrep = rg.allocate_frames(depth, cams, cfg["dilation"])
        rc = rg.coords()
        key = lambda c: np.sort(((c[:, 0].astype(np.int64) & 0x1FFFFF) << 42)  # noqa: E731
                                | ((c[:, 1].astype(np.int64) & 0x1FFFFF) << 21) | (c[:, 2].astype(np.int64) & 0x1FFFFF))
        assert np.array_equal(key(rc), key(coords))
        assert (rrep.blocks_added, rrep.blocks_requested, rrep.pixels_used) == \
            (rep.blocks_added, rep.blocks_requested, rep.pixels_used)
