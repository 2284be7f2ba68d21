"""The multi-GPU setup step through the C-ABI: sogk_grid_create_dense_broadcast
over a real NCCL communicator -- the grid every rank ends up with equals the root's payload and
builds the identical VDB.  (One GPU per call here: a one-rank communicator exercises the same
NCCL path; bench.py's two-rank run on one device covers the sharded sampling path.)"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_nccl_broadcast_helper(tmp_path):
    exe = tmp_path / "nccl_bcast_test"
    lib = os.path.join(ROOT, "paper_2404_10272_b200", "_lib")
    cmd = ["g++", "-std=c++17", "-O1", os.path.join(ROOT, "tests", "native", "nccl_bcast_test.cpp"),
           "-I", os.path.join(ROOT, "include"), "-I/usr/local/cuda/include", "-L", lib, "-lsogk",
           "-lnccl", f"-Wl,-rpath,{lib}", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0 and "nccl.h" in r.stderr:
        pytest.skip("nccl.h not available")
    assert r.returncode == 0, r.stderr
    env = dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0])
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "\nOK:" in "\n" + out.stdout, out.stdout
