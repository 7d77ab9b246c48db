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
@pytest.mark.parametrize("devices", [None, "0,0"])
def test_cpp_dropin_matches_reference(devices):
    """devices "0,0": the drop-in's context drives two device contexts (on the one GPU
    here, separate GPUs on a node): slots and restarts split over them, same results."""
    env = dict(os.environ)
    if devices:
        env["DTWGPU_DEVICES"] = devices
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=600, env=env)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "FAIL" not in out.stdout
