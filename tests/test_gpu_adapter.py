"""The drop-in adapter (include/solidfv_gpu.hpp) compiled against the reference's own headers
and sources (tests/cpp/Makefile) and run on the device: the reference's gmres_solve with the
GPU J.v operator and preconditioner, gpu::run_steps against run_steps, bitwise residuals with
boundary functions and a body force (tests/cpp/test_adapter.cpp lists the checks)."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

BIN = os.path.join(os.path.dirname(__file__), "cpp", "_bin", "test_adapter")


def test_adapter_against_reference():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_bin/test_adapter not built (make -C tests/cpp where the reference is present)")
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "FAIL" not in p.stdout
