"""Runs the C++ drop-in parity test (tests/cpp/dropin_test.cpp): dtwgpu::build_matrix /
dtwgpu::kmedoids vs the unmodified reference dtwclust::build_matrix / kmedoids, same
signatures, bit-identical results, same exception types."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin", "dropin_test")


@pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in test binary not built "
                    "(needs /root/reference headers at build time)")
def test_cpp_dropin_matches_reference():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
