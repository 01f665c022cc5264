"""Host-only build of fixtures/libsvr_fixture.so (the synthetic-scene input generator).

Test / bench fixture infrastructure: it makes INPUTS (scenes, GT depth frames, payloads,
rays, upstream gradients) and is never linked into the product library.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "synthetic.cpp")
HDRS = [os.path.join(HERE, "svr_synth.h"), os.path.join(ROOT, "include", "svr.h")]
OUT = os.path.join(HERE, "libsvr_fixture.so")
# -ffp-contract=off: the reference build has no FMA (proj/CMakeLists.txt:9-11), and the
# fixture is pinned bit for bit to the reference generator compiled that way
FLAGS = ["-O3", "-std=c++17", "-fPIC", "-shared", "-ffp-contract=off", "-Wl,--exclude-libs,ALL", "-Wl,-Bsymbolic"]


def build(force: bool = False) -> str:
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(p) <= t for p in [SRC, *HDRS, __file__]):
            return OUT
    cmd = [os.environ.get("CXX", "g++"), *FLAGS, "-I" + HERE, "-I" + os.path.join(ROOT, "include"), SRC,
           "-o", OUT + ".tmp", "-lpthread"]
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force=True))
