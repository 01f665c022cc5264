"""CPU: bench.py's host-side ray sharding: weak scaling gives every rank its
own full shard; strong scaling (cfg5) splits one fixed global ray set contiguously, so the
shards of any world size concatenate to the 1-rank set."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _cfg(**kw):
    return dict(bench.CFG3, room=(5.0, 5.0, 3.0), h=0.02, ray_poses=4, rays_per_pose=64, **kw)


def test_strong_shards_concatenate_to_the_global_set():
    cfg = _cfg(strong=True, name="cfg5")
    scene = bench.make_scene(cfg)
    full = bench.rays_for_rank(scene, cfg, 0, 1)
    for world in (2, 4):
        parts = [bench.rays_for_rank(scene, cfg, r, world) for r in range(world)]
        for k in range(5):
            assert np.array_equal(np.concatenate([p[k] for p in parts]), full[k])


def test_weak_shards_keep_the_per_rank_size():
    cfg = _cfg(name="cfg3")
    scene = bench.make_scene(cfg)
    a = bench.rays_for_rank(scene, cfg, 0, 1)
    b = bench.rays_for_rank(scene, cfg, 1, 2)
    assert a[0].shape == b[0].shape == (4 * 64, 3)


def test_traffic_lookup_is_keyed_by_workload_and_size():
    assert bench.traffic_from_profiles("cfg3", 1 << 20).get("k_backward_pipe", 0) > 0
    assert bench.traffic_from_profiles("cfg3", 12345) == {}
    assert bench.traffic_from_profiles("nope", 1 << 20) == {}
