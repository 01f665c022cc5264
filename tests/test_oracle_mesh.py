"""CPU: the restated marching cubes (oracle/svr_oracle.cpp) against the reference's own
marching_cubes compiled verbatim (oracle/_ref), word for word."""
import numpy as np
import pytest

from mesh_cases import all_cases_payload, sphere_payload
from oracle import OracleGrid, RefGrid, ref_available

pytestmark = pytest.mark.skipif(not ref_available(), reason="reference not compiled (oracle/_ref)")


def _pair(h, B=8, C=2):
    return OracleGrid(h, B, C), RefGrid(h, B, C)


def _same(a, b):
    for k in ("vertices", "normals", "colors", "labels", "triangles"):
        assert a[k].shape == b[k].shape, k
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("r,h,holes,iso,B", [(0.5, 0.015, 0.0, 0.0, 8), (0.2, 0.02, 0.05, 0.0, 8),
                                             (0.15, 0.02, 0.3, 0.01, 8), (0.06, 0.02, 0.0, 0.0, 4)])
def test_sphere_mesh_matches_reference(r, h, holes, iso, B):
    og, rg = _pair(h, B)
    cs, pay = sphere_payload(og, r, h, holes=holes, B=B)
    rg.allocate_blocks(cs)
    rg.set_payload(0, len(cs), **pay)
    a, b = og.marching_cubes(iso), rg.marching_cubes(iso)
    assert len(a["triangles"]) > 50
    _same(a, b)


def test_all_256_cases_match_reference():
    og, rg = _pair(0.05)
    cs, pay = all_cases_payload()
    for g in (og, rg):
        g.allocate_blocks(cs)
        g.set_payload(0, len(cs), **pay)
    a, b = og.marching_cubes(0.0), rg.marching_cubes(0.0)
    assert len(a["triangles"]) > 500
    _same(a, b)


def test_case_table_shape():
    lib = OracleGrid.lib()
    cnt = np.zeros(256, np.int32)
    tri = np.zeros(256 * 16 * 3, np.int32)
    lib.svro_mc_table(cnt.ctypes.data, tri.ctypes.data)
    assert cnt[0] == 0 and cnt[255] == 0 and cnt.max() == 5
    single = [1 << c for c in range(8)]  # one inside corner: one triangle cutting it off
    assert all(cnt[c] == 1 for c in single) and all(cnt[255 - c] == 1 for c in single)


def test_empty_grid_and_positive_field():
    og, rg = _pair(0.02)
    assert len(og.marching_cubes(0.0)["vertices"]) == 0
    og.allocate_points(np.array([[0.05, 0.05, 0.05]]), 1)
    A = og.block_count()
    og.set_payload(0, A, sdf=np.full((A, 512), 0.5, np.float32), weight=np.ones((A, 512), np.float32))
    m = og.marching_cubes(0.0)
    assert len(m["vertices"]) == 0 and len(m["triangles"]) == 0


from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402


@settings(max_examples=20, deadline=None, suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 2 ** 31 - 1), nb=st.integers(1, 30), holes=st.sampled_from([0.0, 0.1]),
       iso=st.sampled_from([0.0, 0.015]))
def test_random_grids_match_reference(seed, nb, holes, iso):
    rng = np.random.default_rng(seed)
    h = 0.02
    coords = np.unique(rng.integers(-2, 3, size=(nb, 3)), axis=0).astype(np.int32)
    A = len(coords)
    v = np.arange(512)
    X = (coords[:, None, :] * 8 + np.stack([v % 8, (v // 8) % 8, v // 64], 1)[None]) * h
    pay = {"sdf": (np.sin(9 * X[..., 0]) * 0.05 + X[..., 2] - 0.01 + rng.normal(0, 0.003, (A, 512))).astype(np.float32),
           "weight": (rng.uniform(size=(A, 512)) >= holes).astype(np.float32),
           "rgb": rng.uniform(0, 1, (A, 512, 3)).astype(np.float32),
           "logits": rng.normal(size=(A, 512, 2)).astype(np.float32)}
    og, rg = _pair(h)
    for g in (og, rg):
        g.allocate_blocks(coords)
        g.set_payload(0, A, **pay)
    _same(og.marching_cubes(iso), rg.marching_cubes(iso))
