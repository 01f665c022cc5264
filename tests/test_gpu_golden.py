"""GPU: libsvr_b200.so against the golden vectors produced by the REFERENCE's own code
(tests/golden/make_golden.py).  These run on the GPU box, where /root/reference is absent.
Hash / activation / query / march / SDGV are bit-exact; rendering uses the fp32 tolerance
of tests/common.py against the spec-restated renderer on the reference grid API."""
import os

import numpy as np
import pytest

from common import assert_close

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


def canonical(coords):
    c = np.asarray(coords, np.int64)
    return c[np.lexsort((c[:, 0], c[:, 1], c[:, 2]))].astype(np.int32)


def cams_from(rows):
    from paper_2305_13220_b200 import camera

    return [camera(r[0], r[1], r[2], r[3], int(r[4]), int(r[5]), np.array(r[6:15]), np.array(r[15:18]))
            for r in rows]


def test_hash_golden():
    from paper_2305_13220_b200 import SparseDenseGrid

    z = gold("hash.npz")
    g = SparseDenseGrid(0.015, 8, 2, capacity=1 << 16)
    assert np.array_equal(g.allocate_blocks(z["coords"]), z["idx"])
    assert np.array_equal(g.find(z["coords"]), z["found"])
    assert np.array_equal(g.find(z["far"]), z["far_found"])


@pytest.mark.parametrize("R", [0, 1, 2])
def test_activation_points_golden(R):
    from paper_2305_13220_b200 import SparseDenseGrid

    z = gold("activation.npz")
    g = SparseDenseGrid(0.015, 8, 2)
    rep = g.allocate_for_points(z["points"], R)
    assert np.array_equal(canonical(g.coords()), z[f"points_R{R}_coords"])
    assert [rep.blocks_added, rep.blocks_requested, rep.pixels_used] == list(z[f"points_R{R}_report"])


@pytest.mark.parametrize("R,use_scales", [(0, False), (0, True), (1, False), (1, True)])
def test_activation_frames_golden(R, use_scales):
    from paper_2305_13220_b200 import SparseDenseGrid

    z = gold("activation.npz")
    g = SparseDenseGrid(0.04, 8, 2)
    rep = g.allocate_for_frames(z["depth"], cams_from(z["cams"]), R,
                                scales=z["scales"] if use_scales else None)
    key = f"frames_R{R}_s{int(use_scales)}"
    assert np.array_equal(canonical(g.coords()), z[key + "_coords"])
    assert [rep.blocks_added, rep.blocks_requested, rep.pixels_used] == list(z[key + "_report"])


@pytest.mark.parametrize("lookup", [1, 2])
def test_query_golden(lookup):
    from paper_2305_13220_b200 import SparseDenseGrid

    z = gold("query.npz")
    g = SparseDenseGrid(float(z["h"]), 8, int(z["C"]))
    g.allocate_blocks(z["coords"])
    g.set_payload(0, len(z["coords"]), z["pay_sdf"], z["pay_weight"], z["pay_rgb"], z["pay_logits"])
    g.set_lookup(lookup)
    q = g.query(z["x"])
    for k in ("sdf", "grad", "rgb", "valid"):
        assert np.array_equal(q[k], z["q_" + k]), k


@pytest.mark.parametrize("lookup", [1, 2])
def test_march_golden(lookup):
    from paper_2305_13220_b200 import SparseDenseGrid

    z = gold("march.npz")
    for s in range(10):
        g = SparseDenseGrid(0.015, 8, 2)
        g.allocate_blocks(z[f"s{s}_coords"])
        g.set_lookup(lookup)
        m = g.march(z[f"s{s}_o"], z[f"s{s}_d"], 0.008, 96)
        assert np.array_equal(m["counts"], z[f"s{s}_counts"]), s
        for r in range(len(m["counts"])):
            k = int(m["counts"][r])
            assert np.array_equal(m["t"][r, :k], z[f"s{s}_t"][r, :k])
            assert np.array_equal(m["delta"][r, :k], z[f"s{s}_delta"][r, :k])


def test_render_golden():
    from paper_2305_13220_b200 import SparseDenseGrid
    from fixtures import SyntheticScene

    z = gold("render.npz")
    h = float(z["h"])
    sc = SyntheticScene(room_w=2.4, room_d=2.2, room_h=2.0, n_objects=2, width=48, height=36, n_frames=6)
    g = SparseDenseGrid(h, 8, 4)
    g.allocate_blocks(z["coords"])
    g.set_payload(0, len(z["coords"]), **sc.fill_payload(h, z["coords"], 8 * h, 4))
    g.grad_zero()
    f = g.render_forward(z["o"], z["d"], h / 2, 64, 2 * h)
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(f[k], z[k], what=k)
    g.render_backward(z["dC"], z["dD"], z["dN"])
    gs, gr = g.grads()
    idx = g.find(z["grad_blocks"])
    assert_close(gs[idx], z["grad_sdf"], what="grad_sdf")
    assert_close(gr[idx], z["grad_rgb"], what="grad_rgb")


def test_sdgv_reference_file_roundtrip(tmp_path):
    from paper_2305_13220_b200 import SparseDenseGrid

    src = os.path.join(GOLD, "ref_small.sdgv")
    g = SparseDenseGrid.load(src)
    out = tmp_path / "g.sdgv"
    g.save(out)
    assert open(src, "rb").read() == open(out, "rb").read()
