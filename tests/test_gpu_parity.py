"""GPU parity: libsvr_b200.so (through the C-ABI) vs the CPU oracle on identical inputs.

Integer / index / fp64-decision outputs are compared bit-exactly; fp32 rendering outputs
and gradients within the tolerance stated in tests/common.py (RTOL=1e-4 relative plus an
atomic-order floor of 1e-6 x max|oracle|).
"""
import numpy as np
import pytest

from common import assert_close, gpu_grid_from, scene_case
from oracle import OracleGrid

pytestmark = pytest.mark.gpu

LOOKUPS = [1, 2]  # SVR_LOOKUP_HASH, SVR_LOOKUP_DENSE


@pytest.fixture(scope="module")
def case():
    return scene_case()


def test_hash_insert_find_roundtrip():
    """test_grid.cpp:33 at 1e5 coords in [-4000,4000]^3 plus 1000 far misses."""
    from paper_2305_13220_b200 import SparseDenseGrid

    rng = np.random.default_rng(42)
    coords = rng.integers(-4000, 4001, size=(100000, 3), dtype=np.int32)
    g = SparseDenseGrid(0.015, 8, 2, capacity=200000)
    og = OracleGrid(0.015, 8, 2, capacity=200000)
    idx = g.allocate_blocks(coords)
    oidx = og.allocate_blocks(coords)
    assert np.array_equal(idx, oidx)
    assert np.array_equal(g.coords(), og.coords())
    assert np.array_equal(g.find(coords), oidx)
    far = rng.integers(10000, 20001, size=(1000, 3), dtype=np.int32)
    assert (g.find(far) == 0xFFFFFFFF).all()


def test_activation_points_matches_oracle():
    from paper_2305_13220_b200 import SparseDenseGrid

    rng = np.random.default_rng(1)
    pts = rng.uniform(-0.5, 0.5, size=(2000, 3))
    for R in (0, 1, 2):
        g = SparseDenseGrid(0.015, 8, 2)
        og = OracleGrid(0.015, 8, 2)
        r = g.allocate_for_points(pts, R)
        ro = og.allocate_points(pts, R)
        assert (r.blocks_added, r.blocks_requested, r.pixels_used) == \
               (ro.blocks_added, ro.blocks_requested, ro.pixels_used)
        assert np.array_equal(g.coords(), og.coords())  # same deterministic order
        again = g.allocate_for_points(pts, R)  # idempotent (test_grid.cpp:76)
        assert again.blocks_added == 0 and g.block_count() == og.block_count()


def test_activation_capacity_error():
    """test_grid.cpp:89: capacity 10, 20 distinct blocks -> 10 allocated, 10 unallocated."""
    from paper_2305_13220_b200 import CapacityError, SparseDenseGrid

    g = SparseDenseGrid(0.015, 8, 2, capacity=10)
    pts = np.array([[0.13 * i, 0.0, 0.0] for i in range(20)])
    with pytest.raises(CapacityError) as e:
        g.allocate_for_points(pts, 0)
    assert e.value.unallocated_blocks == 10
    assert g.block_count() == 10


def test_activation_depth_matches_oracle(case):
    from paper_2305_13220_b200 import SparseDenseGrid

    g = SparseDenseGrid(case["h"], 8, case["C"])
    r = g.allocate_for_frames(case["depth"], case["cams"], 1)
    og = OracleGrid(case["h"], 8, case["C"])
    ro = og.allocate_frames(case["depth"], case["cams"], 1)
    assert (r.blocks_added, r.blocks_requested, r.pixels_used) == \
           (ro.blocks_added, ro.blocks_requested, ro.pixels_used)
    assert np.array_equal(g.coords(), og.coords())


@pytest.mark.parametrize("lookup", LOOKUPS)
def test_query_bit_exact(case, lookup):
    g = gpu_grid_from(case, lookup)
    rng = np.random.default_rng(7)
    x = rng.uniform(-1.3, 1.3, size=(20000, 3))
    q = g.query(x, logits=True)
    qo = case["oracle"].query(x, logits=True)
    assert q["valid"].sum() > 1000
    for k in ("sdf", "grad", "rgb", "logits", "valid"):
        assert np.array_equal(q[k], qo[k]), k


@pytest.mark.parametrize("lookup", LOOKUPS)
def test_march_bit_exact(case, lookup):
    g = gpu_grid_from(case, lookup)
    m = g.march(case["o"], case["d"], case["step"], 64)
    mo = case["oracle"].march(case["o"], case["d"], case["step"], 64)
    assert np.array_equal(m["counts"], mo["counts"])
    for r in range(len(m["counts"])):
        k = int(m["counts"][r])
        assert np.array_equal(m["t"][r, :k], mo["t"][r, :k])
        assert np.array_equal(m["delta"][r, :k], mo["delta"][r, :k])


@pytest.mark.parametrize("lookup", LOOKUPS)
def test_render_forward_matches_oracle(case, lookup):
    g = gpu_grid_from(case, lookup)
    out = g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    ref = case["oracle"].render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    assert np.array_equal(out["n_samples"], ref["n_samples"])
    for k in ("rgb", "depth", "normal", "wsum"):
        assert_close(out[k], ref[k], what=k)


@pytest.mark.parametrize("lookup", LOOKUPS)
def test_render_backward_matches_oracle(case, lookup):
    g = gpu_grid_from(case, lookup)
    g.grad_zero()
    g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    g.render_backward(case["dC"], case["dD"], case["dN"])
    gs, gr = g.grads()
    os_, or_, act = case["oracle"].render_backward(case["o"], case["d"], case["step"], 64, case["beta"],
                                                   case["dC"], case["dD"], case["dN"])
    assert_close(gs, os_, what="grad_sdf")
    assert_close(gr, or_, what="grad_rgb")
    assert np.array_equal(g.active_mask(), act)
    assert np.array_equal(g.active_blocks(), np.nonzero(act)[0].astype(np.uint32))


def test_grad_zero_active_and_pack_roundtrip(case):
    import torch

    g = gpu_grid_from(case)
    g.set_stream(torch.cuda.current_stream())
    g.grad_zero()
    g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    g.render_backward(case["dC"], case["dD"], case["dN"])
    gs, gr = g.grads()
    blocks = torch.from_numpy(g.active_blocks().astype(np.int32)).cuda()
    packed = torch.empty((blocks.numel(), 512, 4), dtype=torch.float32, device="cuda")
    g.grad_pack(blocks, packed)
    g.synchronize()
    b = blocks.cpu().numpy()
    p = packed.cpu().numpy()
    assert np.array_equal(p[..., 0], gs[b])
    assert np.array_equal(p[..., 1:], gr[b])
    g.grad_zero_active()
    gs2, gr2 = g.grads()
    assert not gs2.any() and not gr2.any() and not g.active_mask().any()
    g.grad_unpack(blocks, packed)
    g.synchronize()
    gs3, gr3 = g.grads()
    assert np.array_equal(gs3, gs) and np.array_equal(gr3, gr)


def test_sdgv_roundtrip_with_oracle(case, tmp_path):
    from paper_2305_13220_b200 import SparseDenseGrid

    g = gpu_grid_from(case)
    path = tmp_path / "g.sdgv"
    g.save(path)
    og = OracleGrid.load(path, case["C"])
    assert np.array_equal(og.coords(), case["coords"])
    p = og.get_payload()
    for k in ("sdf", "weight", "rgb", "logits"):
        assert np.array_equal(p[k], case["pay"][k]), k
    path2 = tmp_path / "o.sdgv"
    case["oracle"].save(path2)
    g2 = SparseDenseGrid.load(path2)
    assert np.array_equal(g2.coords(), case["coords"])
    p2 = g2.get_payload()
    for k in ("sdf", "weight", "rgb", "logits"):
        assert np.array_equal(p2[k], case["pay"][k]), k


def test_device_resident_path_matches_host_path(case):
    import torch

    g = gpu_grid_from(case)
    g.set_stream(torch.cuda.current_stream())  # order after torch's H2D copies
    host = g.render_forward(case["o"], case["d"], case["step"], 64, case["beta"])
    o = torch.from_numpy(case["o"]).cuda()
    d = torch.from_numpy(case["d"]).cuda()
    dev = g.render_forward(o, d, case["step"], 64, case["beta"])
    g.synchronize()
    for k in ("rgb", "depth", "normal", "wsum"):
        assert np.array_equal(dev[k].cpu().numpy(), host[k]), k


@pytest.mark.parametrize("lookup", LOOKUPS)
def test_march_bit_exact_random_rays_with_degenerate_directions(case, lookup):
    """200k rays from random origins (inside and outside the AABB) with random and nearly
    axis-parallel directions (components down to 1e-300) -- counts, t, delta bit-exact."""
    rng = np.random.default_rng(99)
    n = 200_000
    o = rng.uniform(-2.0, 2.0, size=(n, 3))
    d = rng.normal(size=(n, 3))
    k = n // 8
    for j, tiny in enumerate((1e-9, 1e-17, 1e-200, 1e-300)):
        sl = slice(j * k, (j + 1) * k)
        d[sl, j % 3] = tiny * np.sign(d[sl, j % 3])
    d[4 * k:5 * k, 1] = 0.0
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    g = gpu_grid_from(case, lookup)
    m = g.march(o, d, case["step"], 48)
    OracleGrid.set_threads(8)
    try:
        mo = case["oracle"].march(o, d, case["step"], 48)
    finally:
        OracleGrid.set_threads(1)
    assert np.array_equal(m["counts"], mo["counts"])
    mask = np.arange(48)[None, :] < m["counts"][:, None]
    assert np.array_equal(m["t"][mask], mo["t"][mask])
    assert np.array_equal(m["delta"][mask], mo["delta"][mask])
    assert mask.sum() > 500_000


@pytest.mark.parametrize("jump,lookup", [(1, 2), (0, 2), (1, 1)])
def test_march_empty_space_jumps_bit_exact(jump, lookup):
    """Sparse block clusters inside a 96^3-block AABB, so most of each ray's walk crosses
    wide empty space where the march jumps -- over the block-distance field (dense index) or
    the 8^3-superblock distance field (hash mode): counts, t and delta must equal the oracle's
    step-by-step walk bit for bit (random rays, rays through exact block corners / along block
    edges, axis-parallel and diagonal rays)."""
    from paper_2305_13220_b200 import SparseDenseGrid

    h = 0.01
    L = 8 * h
    rng = np.random.default_rng(21)
    centres = rng.integers(0, 96, size=(40, 3))
    cl = np.concatenate([c + rng.integers(-2, 3, size=(30, 3)) for c in centres])
    cl = np.concatenate([cl, [[0, 0, 0], [95, 95, 95]]])  # pin the AABB
    coords = np.unique(cl, axis=0).astype(np.int32)
    og = OracleGrid(h, 8, 1)
    og.allocate_blocks(coords)
    A = len(coords)
    og.set_payload(0, A, weight=np.ones((A, 512), np.float32))
    g = SparseDenseGrid(h, 8, 1)
    g.allocate_blocks(coords)
    g.set_payload(0, A, weight=np.ones((A, 512), np.float32))
    g.set_lookup(lookup)  # 2: dense AABB index + block distances; 1: hash + superblock distances
    g.set_tuning("march_jump", jump)
    n = 60_000
    o = rng.uniform(-0.5, 96 * L + 0.5, size=(n, 3))
    d = rng.normal(size=(n, 3))
    k = n // 10
    o[:k] = rng.integers(0, 97, size=(k, 3)) * L  # exact block corners
    d[k:2 * k] = [1.0, 1.0, 1.0]                   # diagonals through corners
    o[k:2 * k] = rng.integers(0, 97, size=(k, 3)) * L
    d[2 * k:3 * k] = [1.0, 1.0, 0.0]
    d[3 * k:4 * k, 1:] = 0.0                       # axis-parallel
    d[3 * k:4 * k, 0] = np.sign(d[3 * k:4 * k, 0]) + (d[3 * k:4 * k, 0] == 0)
    o[4 * k:5 * k, 2] = rng.integers(0, 97, size=k) * L  # rays in block face planes
    d[4 * k:5 * k, 2] = 0.0
    tgt = (coords[rng.integers(0, A, size=n - 5 * k)] + rng.uniform(0, 1, size=(n - 5 * k, 3))) * L
    d[5 * k:] = tgt - o[5 * k:]  # the rest aim at allocated blocks across empty space
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    m = g.march(o, d, h / 2, 64)
    OracleGrid.set_threads(8)
    try:
        mo = og.march(o, d, h / 2, 64)
    finally:
        OracleGrid.set_threads(1)
    assert np.array_equal(m["counts"], mo["counts"])
    mask = np.arange(64)[None, :] < m["counts"][:, None]
    assert np.array_equal(m["t"][mask], mo["t"][mask])
    assert np.array_equal(m["delta"][mask], mo["delta"][mask])
    assert (m["counts"] > 0).sum() > n // 3


@pytest.mark.parametrize("far", [None, 5000], ids=["bricks", "superblocks-only"])
def test_march_hash_mode_jump_structures_exact(far):
    """Hash mode's three march paths give the same samples bit for bit: block-distance bricks
    near the blocks (superblock grid <= 2^26), the superblock distance field alone (a far block
    makes the superblock grid 625^3 > 2^26: no bricks), and the plain per-block hash probe walk
    (march_jump = 0, the reference's march_intervals restated; bit-exact with the oracle in
    test_march_bit_exact)."""
    from paper_2305_13220_b200 import SparseDenseGrid

    h = 0.01
    L = 8 * h
    rng = np.random.default_rng(5)
    centres = rng.integers(0, 64, size=(30, 3))
    cl = np.concatenate([c + rng.integers(-2, 3, size=(25, 3)) for c in centres])
    if far is not None:
        cl = np.concatenate([cl, [[far, far, far]]])
    coords = np.unique(cl, axis=0).astype(np.int32)
    A = len(coords)
    g = SparseDenseGrid(h, 8, 1)
    g.allocate_blocks(coords)
    g.set_payload(0, A, weight=np.ones((A, 512), np.float32))
    g.set_lookup(1)
    assert g.info().lookup_mode == 1
    n = 20_000
    o = rng.uniform(-0.5, 64 * L + 0.5, size=(n, 3))
    tgt = (coords[rng.integers(0, A, size=n)] + rng.uniform(0, 1, size=(n, 3))) * L
    d = tgt - o
    d[: n // 10, 1:] = 0.0  # axis-parallel
    d[: n // 10, 0] = np.where(d[: n // 10, 0] >= 0, 1.0, -1.0)
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    g.set_tuning("march_jump", 1)
    mj = g.march(o, d, h / 2, 64)
    g.set_tuning("march_jump", 0)
    mp = g.march(o, d, h / 2, 64)
    assert np.array_equal(mj["counts"], mp["counts"])
    mask = np.arange(64)[None, :] < mj["counts"][:, None]
    assert np.array_equal(mj["t"][mask].view(np.uint64), mp["t"][mask].view(np.uint64))
    assert np.array_equal(mj["delta"][mask].view(np.uint64), mp["delta"][mask].view(np.uint64))
    assert (mj["counts"] > 0).sum() > n // 2


def test_march_hash_mode_isolated_blocks_exact():
    """3375 isolated blocks, one per 3-superblock cell: the bricks (27 per occupied superblock)
    would outweigh the blocks, so hash mode keeps the superblock field alone -- the march must
    still equal the plain hash-probe walk bit for bit."""
    from paper_2305_13220_b200 import SparseDenseGrid

    h = 0.01
    L = 8 * h
    rng = np.random.default_rng(9)
    ax = np.arange(15) * 24
    coords = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), -1).reshape(-1, 3).astype(np.int32)
    A = len(coords)
    g = SparseDenseGrid(h, 8, 1)
    g.allocate_blocks(coords)
    g.set_payload(0, A, weight=np.ones((A, 512), np.float32))
    g.set_lookup(1)
    n = 20_000
    o = rng.uniform(-0.5, 15 * 24 * L, size=(n, 3))
    tgt = (coords[rng.integers(0, A, size=n)] + rng.uniform(0, 1, size=(n, 3))) * L
    d = tgt - o
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    g.set_tuning("march_jump", 1)
    mj = g.march(o, d, h / 2, 64)
    g.set_tuning("march_jump", 0)
    mp = g.march(o, d, h / 2, 64)
    assert np.array_equal(mj["counts"], mp["counts"])
    mask = np.arange(64)[None, :] < mj["counts"][:, None]
    assert np.array_equal(mj["t"][mask].view(np.uint64), mp["t"][mask].view(np.uint64))
    assert (mj["counts"] > 0).sum() > n // 2
