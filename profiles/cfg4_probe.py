"""cfg4 activation + query timing alone (bench.py's cfg4 row without its CPU legs), twice in one
process.  usage: python profiles/cfg4_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.Stream(dev)
for _ in range(2):
    r = bench.bench_cfg4(dev, stream, cpu=False)
    print(json.dumps({k: r[k] for k in ("activation_ms", "activation_device_ms", "activation_first_ms", "query_ms")}))
