"""Runs the C++ parity tests of the drop-in library (tests/cpp/test_shim.cpp,
built by __graft_entry__.build()) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "paper_2512_16615_b200", "build", "tests", "test_shim")


@pytest.mark.gpu
def test_cpp_shim_suite():
    if not os.path.exists(EXE):
        pytest.fail(f"{EXE} not built: run __graft_entry__.build()")
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
