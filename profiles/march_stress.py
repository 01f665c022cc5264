"""Randomised march stress (not part of the test suite): sparse block clusters in large AABBs
(negative coordinates included), both lookup modes (dense block-distance jumps, hash-mode
superblock jumps) and odd sample budgets; counts / t / delta must equal the oracle bit for bit.
usage: python profiles/march_stress.py [scenes] [rays per scene]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(scenes=6, n=150_000):
    from oracle import OracleGrid
    from paper_2305_13220_b200 import SparseDenseGrid

    bad = 0
    for seed in range(scenes):
        rng = np.random.default_rng(1000 + seed)
        h = [0.01, 0.02, 0.0175][seed % 3]
        L = 8 * h
        ext = int(rng.integers(40, 160))
        off = rng.integers(-200, 50, size=3)
        centres = rng.integers(0, ext, size=(int(rng.integers(5, 60)), 3))
        cl = np.concatenate([c + rng.integers(-3, 4, size=(25, 3)) for c in centres]) + off
        coords = np.unique(cl, axis=0).astype(np.int32)
        A = len(coords)
        og = OracleGrid(h, 8, 1)
        og.allocate_blocks(coords)
        og.set_payload(0, A, weight=np.ones((A, 512), np.float32))
        o = (rng.uniform(-2, ext + 2, size=(n, 3)) + off) * L
        tgt = (coords[rng.integers(0, A, size=n)] + rng.uniform(0, 1, size=(n, 3))) * L
        d = tgt - o
        k = n // 8
        d[:k] = rng.normal(size=(k, 3))
        d[k:2 * k, rng.integers(0, 3)] = 0.0
        o[2 * k:3 * k] = (rng.integers(0, ext, size=(k, 3)) + off) * L
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        S = [64, 37, 128][seed % 3]
        OracleGrid.set_threads(os.cpu_count() or 1)
        mo = og.march(o, d, h / 2, S)
        OracleGrid.set_threads(1)
        for lookup in (2, 1):
            g = SparseDenseGrid(h, 8, 1)
            g.allocate_blocks(coords)
            g.set_payload(0, A, weight=np.ones((A, 512), np.float32))
            try:
                g.set_lookup(lookup)
            except Exception:
                continue  # AABB too large for the dense index
            m = g.march(o, d, h / 2, S)
            mask = np.arange(S)[None, :] < m["counts"][:, None]
            ok = (np.array_equal(m["counts"], mo["counts"]) and np.array_equal(m["t"][mask], mo["t"][mask])
                  and np.array_equal(m["delta"][mask], mo["delta"][mask]))
            bad += not ok
            print(f"scene {seed}: {A} blocks, extent {ext}, S {S}, lookup {lookup}: "
                  f"{'ok' if ok else 'MISMATCH'} ({int((m['counts'] > 0).sum())} rays with samples)", flush=True)
    print("all bit-exact" if bad == 0 else f"{bad} mismatching runs")
    return bad


if __name__ == "__main__":
    sys.exit(main(*[int(a) for a in sys.argv[1:]]))
