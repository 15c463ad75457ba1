"""The drop-in proof: the reference's own run_with<Engine> / ImsDriver /
RunContext (compiled from its unmodified headers into
oracle/_ref/test_reference_adapter) drive gomix::GpuParallelEngine and compare
it with the reference's ParallelEngine (tests/cpp/test_reference_adapter.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_reference_adapter")


@pytest.mark.gpu
def test_reference_run_with_drives_the_gpu_engine():
    if not os.path.exists(BIN):
        pytest.skip("adapter test binary not built (needs the reference headers at build time)")
    res = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "FAIL" not in res.stdout
    assert res.stdout.count("PASS") >= 20
