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


def test_traffic_lookup_is_keyed_by_workload_size_and_build(tmp_path):
    """roofline.traffic comes from an ncu capture of THIS build only (kernel-source hash)."""
    import json

    bid = bench.build_id()
    entry = {"workload": "cfg3", "rays_per_gpu": 1 << 20, "build_id": bid, "file": "x",
             "dram_bytes": {"k_backward_pipe": 123}}
    stale = dict(entry, build_id="0" * 16, dram_bytes={"k_backward_pipe": 999})
    p = tmp_path / "t.json"
    p.write_text(json.dumps({"captures": [stale, entry]}))
    assert bench.traffic_from_profiles("cfg3", 1 << 20, bid, p)["dram_bytes"]["k_backward_pipe"] == 123
    assert bench.traffic_from_profiles("cfg3", 12345, bid, p) == {}
    assert bench.traffic_from_profiles("nope", 1 << 20, bid, p) == {}
    p.write_text(json.dumps({"captures": [stale]}))
    assert bench.traffic_from_profiles("cfg3", 1 << 20, bid, p) == {}


def test_both_arms_report_the_same_config():
    """The reference arm and ours build `config` with the same function and inputs."""
    a = bench.workload_config(bench.CFG3, 290481, 1 << 20, 64135704, 1)
    b = bench.workload_config(dict(bench.CFG3), 290481, 1 << 20, 64135704, 1)
    assert a == b and a["rays_per_gpu"] == 1 << 20 and "workload" in a


def test_gpus_flag_relaunches_under_torchrun():
    """--gpus N outside torchrun re-launches N ranks; a WORLD_SIZE that disagrees aborts."""
    import json
    import subprocess

    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(x["rank"] for x in lines) == [0, 1] and all(x["world"] == 2 for x in lines)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run"],
                       capture_output=True, text=True, env=dict(env, WORLD_SIZE="1", RANK="0"), timeout=300)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
