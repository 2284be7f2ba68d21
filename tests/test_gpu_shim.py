"""The C++ drop-in shim (include/sogk_sog.hpp) against the unmodified reference:
oracle/_ref/shim_test compares sog::gpu with sog::run_sampler / build_sparse bit for bit."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "shim_test")


@pytest.mark.gpu
def test_cpp_shim_is_bit_exact_vs_reference():
    if not os.path.exists(EXE):
        pytest.skip("oracle/_ref/shim_test not built (needs the reference headers at build time)")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.startswith("OK")
