"""GPU: marching cubes (K14) vs the CPU oracle and the reference's own marching_cubes /
export_ply (oracle/_ref), word for word and byte for byte, plus the
reference's meshing known answers (proj/tests/test_meshing.cpp:44-99) on the GPU mesh."""
import os

import numpy as np
import pytest

from mesh_cases import all_cases_payload, fibonacci_sphere, sphere_payload
from oracle import OracleGrid, RefGrid, ref_available

pytestmark = pytest.mark.gpu


def _gpu_from(og, pay, h, C=2):
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(h, 8, C)
    idx = g.allocate_blocks(og.coords())
    assert np.array_equal(idx, np.arange(og.block_count(), dtype=np.uint32))
    g.set_payload(0, og.block_count(), **pay)
    return g


def _same(a, b):
    for k in ("vertices", "normals", "colors", "labels", "triangles"):
        assert a[k].shape == b[k].shape, (k, a[k].shape, b[k].shape)
        bad = a[k] != b[k]
        assert not bad.any(), f"{k}: {int(bad.sum())} entries differ"


@pytest.mark.parametrize("r,h,holes,iso", [(0.5, 0.015, 0.0, 0.0), (0.2, 0.02, 0.05, 0.0),
                                           (0.15, 0.02, 0.3, 0.01)])
def test_sphere_mesh_matches_oracle(r, h, holes, iso):
    og = OracleGrid(h, 8, 2)
    cs, pay = sphere_payload(og, r, h, holes=holes)
    g = _gpu_from(og, pay, h)
    _same(g.marching_cubes(iso), og.marching_cubes(iso))


@pytest.mark.parametrize("lookup", [1, 2])  # hash / dense AABB index
def test_all_256_cases_match_oracle(lookup):
    og = OracleGrid(0.05, 8, 2)
    cs, pay = all_cases_payload()
    og.allocate_blocks(cs)
    og.set_payload(0, len(cs), **pay)
    g = _gpu_from(og, pay, 0.05)
    g.set_lookup(lookup)
    _same(g.marching_cubes(0.0), og.marching_cubes(0.0))


def test_fused_scene_mesh_matches_oracle():
    """fusion -> marching cubes on a synthetic room: the inference output path end to end."""
    from fixtures import SyntheticScene

    sc = SyntheticScene(n_frames=12, width=96, height=72, label_channels=4)
    cams = sc.cameras()
    depth, rgb, sem = sc.frames(cams)
    og = OracleGrid(0.04, 8, 4)
    og.allocate_frames(depth, cams, 1)
    og.fuse_begin()
    og.fuse_frames(depth, cams, 0.32, rgb=rgb, sem=sem)
    og.fuse_finalize()
    og.denoise(1.0, 1)
    p = og.get_payload()
    g = _gpu_from(og, p, 0.04, C=4)
    a, b = g.marching_cubes(0.0), og.marching_cubes(0.0)
    assert len(b["triangles"]) > 2000
    _same(a, b)


@pytest.mark.skipif(not ref_available(), reason="reference not compiled (oracle/_ref)")
def test_ply_and_obj_bytes_match_reference_export(tmp_path):
    og = OracleGrid(0.02, 8, 2)
    cs, pay = sphere_payload(og, 0.15, 0.02, holes=0.02)
    g = _gpu_from(og, pay, 0.02)
    rg = RefGrid(0.02, 8, 2)
    rg.allocate_blocks(cs)
    rg.set_payload(0, len(cs), **pay)
    g.marching_cubes(0.0)
    rg.marching_cubes(0.0)
    g.save_ply(tmp_path / "gpu.ply")
    rg.export_ply(tmp_path / "ref.ply")
    a, b = (tmp_path / "gpu.ply").read_bytes(), (tmp_path / "ref.ply").read_bytes()
    assert len(a) > 10000 and a == b
    g.save_obj(tmp_path / "gpu.obj")
    rg.export_obj(tmp_path / "ref.obj")
    a, b = (tmp_path / "gpu.obj").read_bytes(), (tmp_path / "ref.obj").read_bytes()
    assert len(a) > 10000 and a == b


def _sphere_gpu(r, voxel):
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(voxel, 8, 2)
    g.allocate_for_points(fibonacci_sphere(np.zeros(3), r, 6000), 1)
    cs = g.coords()
    v = np.arange(512)
    X = (cs[:, None, :] * 8 + np.stack([v % 8, (v // 8) % 8, v // 64], 1)[None]) * voxel
    g.set_payload(0, len(cs), sdf=(np.linalg.norm(X, axis=2) - r).astype(np.float32),
                  weight=np.ones((len(cs), 512), np.float32))
    return g


def test_reference_kat_sphere_within_half_voxel():
    """test_meshing.cpp:44-55."""
    r, voxel = 0.5, 0.015
    m = _sphere_gpu(r, voxel).marching_cubes(0.0)
    V, T = m["vertices"], m["triangles"]
    assert len(V) > 1000
    assert (np.abs(np.linalg.norm(V, axis=1) - r) < voxel / 2).all()
    e1, e2 = V[T[:, 1]] - V[T[:, 0]], V[T[:, 2]] - V[T[:, 0]]
    area = 0.5 * np.linalg.norm(np.cross(e1, e2), axis=1).sum()
    assert area == pytest.approx(4 * np.pi * r * r, rel=0.05)
    idx = np.arange(0, len(V), 97)
    assert (np.sum(m["normals"][idx] * V[idx] / np.linalg.norm(V[idx], axis=1)[:, None], 1) > 0.9).all()


def test_reference_kat_plane_and_empty():
    """test_meshing.cpp:57-82."""
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(0.02, 8, 2)
    g.allocate_for_points(np.array([[0.05, 0.05, 0.05]]), 1)
    A = g.block_count()
    g.set_payload(0, A, sdf=np.full((A, 512), 0.5, np.float32), weight=np.ones((A, 512), np.float32))
    m = g.marching_cubes(0.0)
    assert len(m["vertices"]) == 0 and len(m["triangles"]) == 0
    g = SparseDenseGrid(0.02, 8, 2)
    xs = np.arange(-0.1, 0.25 + 1e-9, 0.05)
    g.allocate_for_points(np.array([[x, y, 0.08] for x in xs for y in xs]), 1)
    n = np.array([0.3, -0.2, 0.93])
    n /= np.linalg.norm(n)
    cs = g.coords()
    v = np.arange(512)
    X = (cs[:, None, :] * 8 + np.stack([v % 8, (v // 8) % 8, v // 64], 1)[None]) * 0.02
    g.set_payload(0, len(cs), sdf=(X @ n - 0.07).astype(np.float32), weight=np.ones((len(cs), 512), np.float32))
    m = g.marching_cubes(0.0)
    assert len(m["vertices"]) and (np.abs(m["vertices"] @ n - 0.07) < 1e-6).all()


def test_reference_kat_vertices_on_iso_level():
    """test_meshing.cpp:84-99: query_sdf at every 7th vertex ~ 0, indices in range, no
    repeated corners."""
    g = _sphere_gpu(0.2, 0.02)
    m = g.marching_cubes(0.0)
    q = g.query(m["vertices"][::7])
    assert q["valid"].all() and (np.abs(q["sdf"]) < 1e-6).all()
    T = m["triangles"]
    assert (T[:, 0] != T[:, 1]).all() and (T[:, 1] != T[:, 2]).all()
    assert T.min() >= 0 and T.max() < len(m["vertices"])
