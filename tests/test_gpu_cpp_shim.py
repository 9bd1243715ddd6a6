"""The reference's own C++ types (wamrec::ScanGeometry, wamrec::SystemMatrix
from the unmodified headers) drive the B200 path through include/wamgpu.hpp:
tests/cpp/shim_test.cpp, built by oracle/Makefile into oracle/_ref/shim_test."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_test")

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_test not built (needs /root/reference at build time)")
def test_reference_types_drive_the_gpu_path():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0 and "SHIM OK" in r.stdout
