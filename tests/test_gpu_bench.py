"""GPU: bench.py keeps the driver's JSON contract (one line, the keys the round-end run
reads), for our arm and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "4", "--warmup", "3", "--no-extra", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] >= 3 and d["value"] > 1e9
    assert d["config"]["workload"].startswith("cfg3")
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] <= 1.5 and r["peak"] > 1000 and r["unit"] == "GB/s"
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and d["clocks"]["samples"] >= 1


def test_reference_arm_contract():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_cfg5_strong_scaling_line():
    """--workload cfg5 (BASELINE configs[4]): total rays fixed, scaling "strong"; traffic is
    only reported for a captured (workload, rays per GPU) pair, so null at this reduced size."""
    d = _run("--workload", "cfg5", "--rays-per-pose", "4096", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    assert d["scaling"] == "strong" and d["config"]["workload"].startswith("cfg5")
    assert d["config"]["rays_per_gpu"] == 64 * 4096 and d["roofline"]["traffic"] is None
    assert "extra_configs" not in d


@pytest.mark.parametrize("workload,rpp", [("cfg3", 2048), ("cfg5", 4096)])
def test_two_rank_line_on_one_gpu(workload, rpp):
    """The N > 1 path of bench.py under torchrun: two ranks with host-side (gloo) collectives on
    cuda:0 -- safe on one device because no kernel waits for another rank's kernel.  Every rank
    must run the same number of steps (a divergent count would hang a collective)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, SVR_BENCH_PG="gloo", SVR_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--workload", workload, "--rays-per-pose", str(rpp), "--steps", "3",
                        "--warmup", "3", "--no-extra", "--no-cpu-baseline", "--reduce", "peer"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["build"]["grad_reduction"]["used"] == "peer"
    assert d["scaling"] == ("strong" if workload == "cfg5" else "weak")
