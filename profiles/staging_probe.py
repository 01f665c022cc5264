"""How much would staging block payloads in shared memory reuse?  (north_star's "stage block
payloads through shared memory or TMA when rays in a tile share blocks".)

On the cfg3 workload: march all 1M rays on the GPU (svr_march), order them as the forward
does (Morton key of the block of the first sample), and for windows of W consecutive rays
(the rays a CTA / an SM has in flight) count
  * corner reads  = 8 per valid-candidate sample (what the forward gathers),
  * distinct voxels and distinct 8^3 blocks the window touches (the corners' blocks),
  * staged bytes  = distinct blocks x 8 KB (a whole-block stage of the float4 payload).
usage: python profiles/staging_probe.py [rays]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def spread3(v):
    v = v & 0x3FF
    v = (v | (v << 16)) & 0x030000FF
    v = (v | (v << 8)) & 0x0300F00F
    v = (v | (v << 4)) & 0x030C30C3
    v = (v | (v << 2)) & 0x09249249
    return v


def main(nrays=1 << 20):
    from fixtures.workloads import CFG3, activation_frames, fill_in_chunks, make_scene, rays_for_rank
    from paper_2305_13220_b200 import SparseDenseGrid

    cfg = CFG3
    scene = make_scene(cfg)
    cams, depth = activation_frames(scene, cfg)
    g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22)
    g.allocate_for_frames(depth, cams, cfg["dilation"])
    fill_in_chunks(scene, cfg, g.coords(), lambda f, n, p: g.set_payload(f, n, **p))
    o, d = rays_for_rank(scene, cfg, 0, 1)[:2]
    o, d = o[:nrays], d[:nrays]
    h = cfg["h"]
    m = g.march(o, d, h / 2, cfg["max_samples"])
    cnt, t = m["counts"], m["t"]
    S = t.shape[1]
    k = np.arange(S)[None, :]
    valid = k < cnt[:, None]
    x = o[:, None, :] + t[:, :, None] * d[:, None, :]          # [R, S, 3]
    base = np.floor(x / h).astype(np.int64)                    # cell base voxel
    blk = base >> 3
    info = g.info()
    lo = np.array(info.bounds_lo)
    first = blk[:, 0, :] - lo
    key = (spread3(first[:, 0]) | (spread3(first[:, 1]) << 1) | (spread3(first[:, 2]) << 2)).astype(np.int64)
    key[cnt == 0] = 1 << 40
    order = np.argsort(key, kind="stable")
    print(f"{nrays} rays, {int(valid.sum())} samples, {len(g.coords())} blocks")
    for W in (32, 256, 1024, 4096):
        reads = vox = blocks = 0
        nwin = 0
        for w0 in range(0, min(nrays, 1 << 18), W):
            ids = order[w0:w0 + W]
            v = valid[ids]
            b = base[ids][v]                                      # [n, 3]
            corners = (b[:, None, :] + np.array([[i & 1, (i >> 1) & 1, i >> 2] for i in range(8)])[None]).reshape(-1, 3)
            reads += len(corners)
            ck = (corners[:, 0] + (1 << 20)) | ((corners[:, 1] + (1 << 20)) << 21) | ((corners[:, 2] + (1 << 20)) << 42)
            vox += len(np.unique(ck))
            cb = corners >> 3
            bk = (cb[:, 0] + (1 << 20)) | ((cb[:, 1] + (1 << 20)) << 21) | ((cb[:, 2] + (1 << 20)) << 42)
            blocks += len(np.unique(bk))
            nwin += 1
        print(f"W={W:5d}: corner reads / distinct voxels = {reads / vox:5.2f}; distinct blocks per window "
              f"{blocks / nwin:8.1f} -> whole-block stage {blocks / nwin * 8192 / 1024:8.1f} KB "
              f"(vs {reads / nwin * 16 / 1024:7.1f} KB gathered, {vox / nwin * 16 / 1024:7.1f} KB distinct)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 20)
