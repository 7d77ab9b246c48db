"""ctypes binding of libdtwgpu.so (include/dtwgpu.h).

The CUDA library is the product: there is no CPU fallback. If the shared object is
missing or no CUDA device is visible, every entry point raises -- loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# DTWGPU_LIB: load an alternative build (kernel-variant experiments in tools/).
LIB_PATH = os.environ.get("DTWGPU_LIB") or os.path.join(HERE, "libdtwgpu.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_u8 = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_vp = C.c_void_p
OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64, C.c_double)

# Every symbol include/dtwgpu.h declares (checked by tests/test_native_abi.py).
EXPORTS = [
    "dtwg_create", "dtwg_destroy", "dtwg_last_error", "dtwg_last_error_pair", "dtwg_set_stream",
    "dtwg_synchronize", "dtwg_build_matrix", "dtwg_upload_series", "dtwg_fill_slots",
    "dtwg_count_cells", "dtwg_last_fill_ms", "dtwg_launch_count", "dtwg_last_plan",
    "dtwg_adopt_condensed", "dtwg_download_condensed", "dtwg_download_range", "dtwg_kmedoids", "dtwg_km_nearest_update",
    "dtwg_km_assign", "dtwg_km_update", "dtwg_force_kernel", "dtwg_measure_cell_peak", "dtwg_km_stats", "dtwg_silhouette",
    "dtwg_create_multi", "dtwg_device_count", "dtwg_visible_devices",
    "dtwg_exchange_export", "dtwg_exchange_open", "dtwg_exchange_fill", "dtwg_exchange_complete",
    "dtwg_exchange_close",
    # host-side data path (csrc/host_io.cpp)
    "dtwg_io_last_error", "dtwg_io_last_file", "dtwg_free", "dtwg_save_matrix_text",
    "dtwg_load_matrix_text", "dtwg_save_matrix_binary", "dtwg_load_matrix_binary",
    "dtwg_ingest_csv", "dtwg_dataset_size", "dtwg_dataset_samples", "dtwg_dataset_offsets",
    "dtwg_dataset_id", "dtwg_dataset_free", "dtwg_z_normalize",
]
_HOST_INT = ("dtwg_create_multi", "dtwg_device_count", "dtwg_visible_devices",
             "dtwg_exchange_export", "dtwg_exchange_open", "dtwg_exchange_fill",
             "dtwg_exchange_complete", "dtwg_exchange_close", "dtwg_save_matrix_text", "dtwg_load_matrix_text", "dtwg_save_matrix_binary",
             "dtwg_load_matrix_binary", "dtwg_ingest_csv", "dtwg_z_normalize")


class NativeMissingError(RuntimeError):
    pass


def build() -> None:
    import subprocess
    subprocess.run(["make", "-s", "-j4", "-C", os.path.join(HERE, "csrc")], check=True)


@lru_cache(None)
def lib() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise NativeMissingError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    L.dtwg_create.argtypes = [C.c_int, P(_vp)]
    L.dtwg_create.restype = C.c_int
    L.dtwg_destroy.argtypes = [_vp]
    L.dtwg_destroy.restype = None
    L.dtwg_last_error.argtypes = [_vp]
    L.dtwg_last_error.restype = C.c_char_p
    L.dtwg_last_error_pair.argtypes = [_vp, P(_i64), P(_i64)]
    L.dtwg_last_error_pair.restype = None
    L.dtwg_set_stream.argtypes = [_vp, _vp]
    L.dtwg_synchronize.argtypes = [_vp]
    L.dtwg_build_matrix.argtypes = [_vp, _dp, _ip, _i64, _i64, C.c_int, C.c_uint, C.c_int, _vp,
                                    P(C.c_uint64)]
    L.dtwg_upload_series.argtypes = [_vp, _dp, _ip, _i64]
    L.dtwg_fill_slots.argtypes = [_vp, _i64, C.c_int, C.c_int, _i64, _i64, _vp]
    L.dtwg_count_cells.argtypes = [_vp, _i64, C.c_int, _i64, _i64, P(C.c_uint64)]
    L.dtwg_last_fill_ms.argtypes = [_vp, P(C.c_float)]
    L.dtwg_launch_count.argtypes = [_vp]
    L.dtwg_launch_count.restype = C.c_uint64
    L.dtwg_last_plan.argtypes = [_vp]
    L.dtwg_last_plan.restype = C.c_char_p
    L.dtwg_adopt_condensed.argtypes = [_vp, _vp, _i64, C.c_int]
    L.dtwg_download_condensed.argtypes = [_vp, _dp]
    L.dtwg_download_range.argtypes = [_vp, _i64, _i64, _vp]
    L.dtwg_kmedoids.argtypes = [_vp, _i64, _i64, _i64, C.c_uint64, _i64, _i64, OBSERVER, _vp,
                                _ip, _ip, P(C.c_double), P(_i64)]
    L.dtwg_km_nearest_update.argtypes = [_vp, _i64, _u8, _dp]
    L.dtwg_km_assign.argtypes = [_vp, _ip, _i64, _ip, _dp]
    L.dtwg_km_update.argtypes = [_vp, _ip, _i64, _ip, _ip]
    L.dtwg_force_kernel.argtypes = [_vp, C.c_int, C.c_int, C.c_int]
    L.dtwg_measure_cell_peak.argtypes = [_vp, C.c_int, P(C.c_double)]
    L.dtwg_km_stats.argtypes = [_vp, _dp, C.c_int]
    L.dtwg_silhouette.argtypes = [_vp, _ip, _i64, _ip, _i64, _dp, P(C.c_double)]
    L.dtwg_create_multi.argtypes = [P(C.c_int), C.c_int, P(_vp)]
    L.dtwg_device_count.argtypes = [_vp]
    L.dtwg_visible_devices.argtypes = []
    L.dtwg_exchange_export.argtypes = [_vp, _i64, C.c_char_p]
    L.dtwg_exchange_open.argtypes = [_vp, C.c_char_p, C.c_int, C.c_int]
    L.dtwg_exchange_fill.argtypes = [_vp, _i64, C.c_int, C.c_int, _i64, _i64]
    L.dtwg_exchange_complete.argtypes = [_vp]
    L.dtwg_exchange_close.argtypes = [_vp]
    L.dtwg_io_last_error.argtypes = [P(_i64), P(_i64)]
    L.dtwg_io_last_error.restype = C.c_char_p
    L.dtwg_io_last_file.argtypes = []
    L.dtwg_io_last_file.restype = C.c_char_p
    L.dtwg_free.argtypes = [_vp]
    L.dtwg_free.restype = None
    L.dtwg_save_matrix_text.argtypes = [_vp, _i64, C.c_char_p, C.c_int]
    L.dtwg_load_matrix_text.argtypes = [C.c_char_p, C.c_int, P(_i64), P(_vp)]
    L.dtwg_save_matrix_binary.argtypes = [_vp, _i64, C.c_char_p]
    L.dtwg_load_matrix_binary.argtypes = [C.c_char_p, P(_i64), P(_vp)]
    L.dtwg_ingest_csv.argtypes = [P(C.c_char_p), _i64, C.c_int, C.c_int, C.c_int, P(_vp)]
    L.dtwg_dataset_size.argtypes = [_vp]
    L.dtwg_dataset_size.restype = _i64
    L.dtwg_dataset_samples.argtypes = [_vp]
    L.dtwg_dataset_samples.restype = P(C.c_double)
    L.dtwg_dataset_offsets.argtypes = [_vp]
    L.dtwg_dataset_offsets.restype = P(_i64)
    L.dtwg_dataset_id.argtypes = [_vp, _i64]
    L.dtwg_dataset_id.restype = C.c_char_p
    L.dtwg_dataset_free.argtypes = [_vp]
    L.dtwg_dataset_free.restype = None
    L.dtwg_z_normalize.argtypes = [_vp, _vp, _i64, C.c_int]
    for name in _HOST_INT:
        getattr(L, name).restype = C.c_int
    for name in EXPORTS:
        fn = getattr(L, name)
        if fn.restype is C.c_int or name in ("dtwg_set_stream", "dtwg_synchronize",
                                              "dtwg_build_matrix", "dtwg_upload_series",
                                              "dtwg_fill_slots", "dtwg_count_cells",
                                              "dtwg_last_fill_ms", "dtwg_adopt_condensed",
                                              "dtwg_download_condensed", "dtwg_download_range", "dtwg_kmedoids",
                                              "dtwg_km_nearest_update", "dtwg_km_assign",
                                              "dtwg_km_update", "dtwg_force_kernel",
                                              "dtwg_measure_cell_peak", "dtwg_km_stats",
                                              "dtwg_silhouette"):
            fn.restype = C.c_int
    return L
