"""Time the cfg3 refinement step (bench.py's cfg3_refine_step row without its CPU leg)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda:0")
stream = torch.cuda.Stream(dev)
torch.cuda.set_stream(stream)
out = bench.bench_refine(dev, stream, steps=int(sys.argv[1]) if len(sys.argv) > 1 else 20, cpu=False)
print(json.dumps({k: out[k] for k in ("ms_per_step", "valid_samples", "active_blocks")} | {"frac": out["roofline"]["frac"]}))
