"""cfg4 activation cost breakdown on the GPU: fresh-grid allocate_for_frames (cold), a repeat
call on the populated grid (keys + dilation + filter, no new blocks), and the raw cost of the
device allocation and zeroing the new blocks need (cudaMalloc / memset of the same bytes).
usage: python profiles/activation_probe.py [frames]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(n_frames=300):
    import torch

    from fixtures.workloads import CFG4
    from fixtures.workloads import make_scene
    from paper_2305_13220_b200 import SparseDenseGrid

    dev = torch.device("cuda:0")
    cfg = CFG4
    scene = make_scene(cfg)
    cams = scene.cameras(n_frames)
    depth_d = torch.from_numpy(scene.depth(cams)).to(dev)
    torch.cuda.synchronize()

    def timed(fn):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        return time.perf_counter() - t0, r

    for i in range(3):
        g = SparseDenseGrid(cfg["h"], 8, cfg["C"], capacity=1 << 22, device=0)
        dt, rep = timed(lambda: g.allocate_for_frames(depth_d, cams, cfg["dilation"]))
        print(f"fresh grid {i}: {dt * 1e3:.2f} ms, {rep.blocks_added} blocks")
        dt2, rep2 = timed(lambda: g.allocate_for_frames(depth_d, cams, cfg["dilation"]))
        print(f"  repeat on populated grid: {dt2 * 1e3:.2f} ms ({rep2.blocks_added} added)")
        nb = rep.blocks_added
        del g
    per_block = 16 + 512 * (16 + 4 + 4 * cfg["C"] + 16) + 64 + 4 + 1 + 8
    nbytes = nb * per_block
    from cuda.bindings import runtime as cudart

    for i in range(2):
        t0 = time.perf_counter()
        err, ptr = cudart.cudaMalloc(nbytes)
        t1 = time.perf_counter()
        cudart.cudaFree(ptr)
        print(f"cudaMalloc of {nbytes / 1e9:.2f} GB: {(t1 - t0) * 1e3:.2f} ms ({err})")
    x = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for i in range(2):
        dt, _ = timed(lambda: x.zero_())
        print(f"zero {nbytes / 1e9:.2f} GB: {dt * 1e3:.2f} ms")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 300)
