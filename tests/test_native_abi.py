"""CPU tests of the C-ABI library: it loads, exports every symbol include/dtwgpu.h
declares, and fails loudly (no CPU fallback) when no CUDA device is visible."""
import ctypes
import os
import re

import pytest

from paper_2307_04904_b200 import _native, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "dtwgpu.h")).read()
    return sorted(set(re.findall(r"\b(dtwg_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    for name in header_symbols():
        assert hasattr(L, name), name


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    L = _native.lib()
    h = ctypes.c_void_p()
    assert L.dtwg_create(0, ctypes.byref(h)) == 101  # DTWG_NO_DEVICE
    with pytest.raises(api.DeviceError):
        api.Engine(0)


def test_python_validation_mirrors_reference_order():
    # These checks run on the host before any device work (pairwise.hpp:65-67).
    U = api.WarpWindow.unlimited()
    with pytest.raises(api.EmptyDatasetError):
        api.build_matrix([], U, 1)
    with pytest.raises(api.InvalidArgumentsError):
        api.build_matrix([api.TimeSeries("a", [1.0])], U, 0)
    with pytest.raises(api.InvalidSeriesError):
        api.build_matrix([api.TimeSeries("a", [1.0]), api.TimeSeries("a", [2.0])], U, 1)
    with pytest.raises(api.InvalidSeriesError):
        api.build_matrix([api.TimeSeries("a", [float("nan")])], U, 1)


def test_warp_window_semantics():
    w = api.WarpWindow.banded(3)
    assert w.feasible_for(5, 2) and not api.WarpWindow.banded(2).feasible_for(5, 2)
    assert api.WarpWindow.unlimited().effective(4, 9) == 9 and w.effective(4, 9) == 3


def test_distance_matrix_semantics():
    m = api.DistanceMatrix.from_condensed(3, [1.0, 2.0, 3.0])
    assert m.distance(0, 2) == 2.0 and m.distance(2, 1) == 3.0 and m.distance(1, 1) == 0.0
    with pytest.raises(api.IndexOutOfRangeError):
        m.distance(0, 3)
    with pytest.raises(api.DistanceMatrixInvalidError):
        api.DistanceMatrix.from_condensed(3, [1.0, -2.0, 3.0])
    with pytest.raises(api.DistanceMatrixInvalidError):
        api.DistanceMatrix.from_condensed(3, [1.0, 2.0])
