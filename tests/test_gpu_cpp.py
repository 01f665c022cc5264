"""GPU: the C++ host mirror (include/svr.hpp) running the reference's test_grid.cpp
scenarios against libsvr_b200.so, compiled with g++ and linked to the in-tree library."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_mirror_scenarios(tmp_path):
    lib_dir = os.path.join(ROOT, "paper_2305_13220_b200")
    exe = tmp_path / "test_svr_hpp"
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "test_svr_hpp.cpp"), "-o", str(exe),
                    "-L", lib_dir, "-l:libsvr_b200.so", f"-Wl,-rpath,{lib_dir}"], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
