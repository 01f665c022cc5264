"""GPU: randomized parity sweep (hypothesis) -- random sparse block sets with partially
observed blocks, random payloads and rays from inside and outside the grid, every
render-path output against the oracle (counts / t bit-exact, values within tolerance)."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from common import assert_close
from oracle import OracleGrid

pytestmark = pytest.mark.gpu


@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 2 ** 31 - 1), h=st.sampled_from([0.01, 0.02, 0.05]),
       nb=st.integers(1, 60), holes=st.sampled_from([0.0, 0.1, 0.5]), S=st.sampled_from([16, 64, 96]))
def test_render_path_random_grids(seed, h, nb, holes, S):
    from paper_2305_13220_b200 import SparseDenseGrid

    rng = np.random.default_rng(seed)
    # clustered random blocks so rays cross contiguous runs and gaps
    centre = rng.integers(-3, 3, size=3)
    coords = np.unique(centre + rng.integers(-3, 4, size=(nb, 3)), axis=0).astype(np.int32)
    A = len(coords)
    v = np.arange(512)
    X = (coords[:, None, :] * 8 + np.stack([v % 8, (v // 8) % 8, v // 64], 1)[None]) * h
    pay = {"sdf": (np.sin(X[..., 0] * 7) * 0.03 + np.cos(X[..., 1] * 5) * 0.02 + X[..., 2] * 0.1
                   + rng.normal(0, 0.005, (A, 512))).astype(np.float32),
           "weight": (rng.uniform(size=(A, 512)) >= holes).astype(np.float32),
           "rgb": rng.uniform(0, 1, (A, 512, 3)).astype(np.float32),
           "logits": np.zeros((A, 512, 1), np.float32)}
    og = OracleGrid(h, 8, 1)
    og.allocate_blocks(coords)
    og.set_payload(0, A, **pay)
    g = SparseDenseGrid(h, 8, 1)
    g.allocate_blocks(coords)
    g.set_payload(0, A, **pay)
    n = 300
    L = 8 * h
    o = (centre + rng.uniform(-5, 5, size=(n, 3))) * L
    tgt = (coords[rng.integers(0, A, n)] + rng.uniform(0, 1, (n, 3))) * L
    d = tgt - o
    d[: n // 10, 1:] = 0.0  # axis-parallel
    d[: n // 10, 0] += (d[: n // 10, 0] == 0)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    step, beta = h / 2, 2 * h
    m, mo = g.march(o, d, step, S), og.march(o, d, step, S)
    assert np.array_equal(m["counts"], mo["counts"])
    mask = np.arange(S)[None, :] < m["counts"][:, None]
    assert np.array_equal(m["t"][mask], mo["t"][mask])
    out = g.render_forward(o, d, step, S, beta)
    ref = og.render_forward(o, d, step, S, beta)
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(out[k], ref[k], what=k)
    u = rng.uniform(-1, 1, (n, 7))
    g.grad_zero()
    g.render_backward(u[:, :3], u[:, 3], u[:, 4:])
    gs, gr = g.grads()
    ogs, ogr, act = og.render_backward(o, d, step, S, beta, u[:, :3], u[:, 3], u[:, 4:])
    assert_close(gs, ogs, what="grad_sdf")
    assert_close(gr, ogr, what="grad_rgb")
    assert np.array_equal(g.active_mask(), act)


@settings(max_examples=15, deadline=None, suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 2 ** 31 - 1), nb=st.integers(1, 40), holes=st.sampled_from([0.0, 0.05, 0.3]),
       iso=st.sampled_from([0.0, 0.01, -0.02]))
def test_marching_cubes_random_grids(seed, nb, holes, iso):
    from paper_2305_13220_b200 import SparseDenseGrid

    rng = np.random.default_rng(seed)
    h = 0.02
    coords = np.unique(rng.integers(-2, 3, size=(nb, 3)), axis=0).astype(np.int32)
    A = len(coords)
    v = np.arange(512)
    X = (coords[:, None, :] * 8 + np.stack([v % 8, (v // 8) % 8, v // 64], 1)[None]) * h
    c = rng.uniform(-0.1, 0.1, 3)
    pay = {"sdf": (np.linalg.norm(X - c, axis=2) - rng.uniform(0.05, 0.2)
                   + rng.normal(0, 0.002, (A, 512))).astype(np.float32),
           "weight": (rng.uniform(size=(A, 512)) >= holes).astype(np.float32),
           "rgb": rng.uniform(-0.1, 1.1, (A, 512, 3)).astype(np.float32),
           "logits": rng.normal(size=(A, 512, 3)).astype(np.float32)}
    og = OracleGrid(h, 8, 3)
    og.allocate_blocks(coords)
    og.set_payload(0, A, **pay)
    g = SparseDenseGrid(h, 8, 3)
    g.allocate_blocks(coords)
    g.set_payload(0, A, **pay)
    a, b = g.marching_cubes(iso), og.marching_cubes(iso)
    for k in b:
        assert np.array_equal(a[k], b[k]), k
