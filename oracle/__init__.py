"""TEST INFRASTRUCTURE ONLY -- the parity checkers.

ctypes bindings for
  * liboracle.so            -- oracle/dtw_oracle.c, a C restatement of the reference hot path;
  * _ref/libdtwclust_ref.so -- the reference's own headers compiled in place (oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package. The product (paper_2307_04904_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdtwclust_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
OBSERVER = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_int64, C.c_double)


def build() -> None:
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE], check=True)


@lru_cache(None)
def lib():
    if not os.path.exists(ORACLE_SO):
        build()
    L = C.CDLL(ORACLE_SO)
    L.oracle_dtw.argtypes = [_dp, _i64, _dp, _i64, _i64, C.c_void_p]
    L.oracle_dtw.restype = C.c_double
    L.oracle_dtw_brute_force.argtypes = [_dp, _i64, _dp, _i64, _i64]
    L.oracle_dtw_brute_force.restype = C.c_double
    L.oracle_build_condensed.argtypes = [_dp, _ip, _i64, _i64, C.c_int, _i64, _i64, _dp]
    L.oracle_build_condensed.restype = None
    L.oracle_pair_cells.argtypes = [_i64, _i64, _i64]
    L.oracle_pair_cells.restype = _i64
    L.oracle_pair_window.argtypes = [_i64, _i64, _i64, C.c_int]
    L.oracle_pair_window.restype = _i64
    L.oracle_first_infeasible.argtypes = [_ip, _i64, _i64, C.POINTER(_i64), C.POINTER(_i64)]
    L.oracle_first_infeasible.restype = C.c_int
    L.oracle_condensed_pair.argtypes = [_i64, _i64, C.POINTER(_i64), C.POINTER(_i64)]
    L.oracle_assign.argtypes = [_dp, _i64, _ip, _i64, _ip]
    L.oracle_assignment_cost.argtypes = [_dp, _i64, _ip]
    L.oracle_assignment_cost.restype = C.c_double
    L.oracle_update.argtypes = [_dp, _i64, _ip, _i64, _ip, _ip]
    L.oracle_kmedoids.argtypes = [_dp, _i64, _i64, _i64, _i64, C.c_uint64, OBSERVER, C.c_void_p,
                                  _ip, _ip, C.POINTER(C.c_double)]
    L.oracle_kmedoids.restype = C.c_int
    L.oracle_kmedoids_range.argtypes = [_dp, _i64, _i64, _i64, _i64, C.c_uint64, _i64, _i64,
                                        OBSERVER, C.c_void_p, _ip, _ip, C.POINTER(C.c_double),
                                        C.POINTER(_i64)]
    L.oracle_kmedoids_range.restype = C.c_int
    L.oracle_silhouette.argtypes = [_dp, _i64, _ip, _i64, _ip, _i64, _dp, C.POINTER(C.c_double)]
    L.oracle_silhouette.restype = C.c_int
    L.oracle_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
    L.oracle_splitmix_next.restype = C.c_uint64
    return L


def have_ref() -> bool:
    return os.path.exists(REF_SO)


@lru_cache(None)
def ref():
    if not os.path.exists(REF_SO):
        raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
    L = C.CDLL(REF_SO)
    L.ref_last_error.restype = C.c_char_p
    L.ref_last_pair.argtypes = [C.POINTER(_i64), C.POINTER(_i64)]
    L.ref_build_condensed.argtypes = [_dp, _ip, _i64, _i64, C.c_int, C.c_uint, _dp,
                                      C.POINTER(C.c_uint64)]
    L.ref_build_condensed.restype = C.c_int
    L.ref_build_condensed_ids.argtypes = [_dp, _ip, _i64, C.POINTER(C.c_char_p), _i64, C.c_int,
                                          C.c_uint, _dp, C.POINTER(C.c_uint64)]
    L.ref_build_condensed_ids.restype = C.c_int
    L.ref_dtw.argtypes = [_dp, _i64, _dp, _i64, _i64, C.POINTER(C.c_double)]
    L.ref_dtw.restype = C.c_int
    L.ref_dtw_brute_force.argtypes = [_dp, _i64, _dp, _i64, _i64, C.POINTER(C.c_double)]
    L.ref_dtw_brute_force.restype = C.c_int
    L.ref_kmedoids.argtypes = [_dp, _i64, _i64, _i64, _i64, C.c_uint64, OBSERVER, C.c_void_p,
                               _ip, _ip, C.POINTER(C.c_double)]
    L.ref_kmedoids.restype = C.c_int
    L.ref_sweep.argtypes = [_dp, _i64, _ip, _i64, _ip, C.POINTER(C.c_double), _ip]
    L.ref_sweep.restype = C.c_int
    L.ref_silhouette.argtypes = [_dp, _i64, _ip, _i64, _ip, _i64, _dp, C.POINTER(C.c_double)]
    L.ref_silhouette.restype = C.c_int
    L.ref_free.argtypes = [C.c_void_p]
    L.ref_free.restype = None
    L.ref_save_matrix.argtypes = [_dp, _i64, C.c_char_p]
    L.ref_save_matrix.restype = C.c_int
    L.ref_load_matrix.argtypes = [C.c_char_p, C.POINTER(_i64), C.POINTER(C.c_void_p)]
    L.ref_load_matrix.restype = C.c_int
    L.ref_ingest.argtypes = [C.POINTER(C.c_char_p), _i64, C.c_int, C.c_int, C.POINTER(_i64),
                             C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
    L.ref_ingest.restype = C.c_int
    L.ref_z_normalize.argtypes = [_dp, _ip, _i64]
    L.ref_z_normalize.restype = C.c_int
    return L


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64a(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ---------------------------------------------------------------- restatement
def dtw(x, y, half_width: int = -1) -> float:
    x, y = _f64(x), _f64(y)
    return lib().oracle_dtw(x, len(x), y, len(y), half_width, None)


def dtw_brute_force(x, y, half_width: int = -1) -> float:
    x, y = _f64(x), _f64(y)
    return lib().oracle_dtw_brute_force(x, len(x), y, len(y), half_width)


def build_condensed(samples, offsets, half_width=-1, auto_widen=False, slot_begin=0,
                    slot_end=None) -> np.ndarray:
    samples, offsets = _f64(samples), _i64a(offsets)
    p = len(offsets) - 1
    total = p * (p - 1) // 2
    if slot_end is None:
        slot_end = total
    out = np.empty(max(slot_end - slot_begin, 0), dtype=np.float64)
    if slot_end > slot_begin:
        lib().oracle_build_condensed(samples, offsets, p, half_width, int(auto_widen), slot_begin,
                                     slot_end, out)
    return out


def pair_cells(n, m, hw) -> int:
    return lib().oracle_pair_cells(n, m, hw)


def first_infeasible(offsets, half_width):
    i, j = _i64(), _i64()
    offsets = _i64a(offsets)
    if lib().oracle_first_infeasible(offsets, len(offsets) - 1, half_width, C.byref(i), C.byref(j)):
        return int(i.value), int(j.value)
    return None


def assign(D, p, medoids):
    out = np.empty(p, dtype=np.int64)
    lib().oracle_assign(_f64(D), p, _i64a(medoids), len(medoids), out)
    return out


def assignment_cost(D, p, assignment) -> float:
    return lib().oracle_assignment_cost(_f64(D), p, _i64a(assignment))


def update(D, p, medoids, assignment):
    out = np.empty(len(medoids), dtype=np.int64)
    lib().oracle_update(_f64(D), p, _i64a(medoids), len(medoids), _i64a(assignment), out)
    return out


def kmedoids(D, p, k, restarts=10, max_iterations=100, seed=0, observer=None):
    med = np.empty(max(k, 1), dtype=np.int64)
    asg = np.empty(p, dtype=np.int64)
    cost = C.c_double()
    cb = OBSERVER((lambda u, r, it, c: observer(r, it, c)) if observer else (lambda *a: None))
    rc = lib().oracle_kmedoids(_f64(D), p, k, restarts, max_iterations, seed, cb, None, med, asg,
                               C.byref(cost))
    if rc:
        raise RuntimeError(f"oracle_kmedoids error code {rc}")
    return med[:k], asg, cost.value


def kmedoids_range(D, p, k, restarts, max_iterations, seed, rb, re):
    """Restarts [rb, re) only; returns (medoids, assignment, cost, best_restart)."""
    med = np.empty(max(k, 1), dtype=np.int64)
    asg = np.empty(p, dtype=np.int64)
    cost = C.c_double()
    br = _i64(-1)
    rc = lib().oracle_kmedoids_range(_f64(D), p, k, restarts, max_iterations, seed, rb, re,
                                     OBSERVER(lambda *a: None), None, med, asg, C.byref(cost),
                                     C.byref(br))
    if rc:
        raise RuntimeError(f"oracle_kmedoids_range error code {rc}")
    return med[:k], asg, cost.value, int(br.value)


def silhouette(D, p, medoids, assignment):
    """validation.hpp:30-79 restated; returns (per-series silhouettes, mean)."""
    asg = _i64a(assignment)
    out = np.zeros(max(p, 1), dtype=np.float64)
    mean = C.c_double()
    rc = lib().oracle_silhouette(_f64(D), p, _i64a(medoids), len(medoids), asg, len(asg), out,
                                 C.byref(mean))
    if rc:
        raise RuntimeError(f"oracle_silhouette error code {rc}")
    return out[:p], mean.value


# ---------------------------------------------------------------- reference itself
class RefError(Exception):
    def __init__(self, code, message, pair=None):
        super().__init__(message)
        self.code = code
        self.pair = pair


def _ref_check(rc):
    if rc:
        i, j = _i64(), _i64()
        ref().ref_last_pair(C.byref(i), C.byref(j))
        pair = (int(i.value), int(j.value)) if i.value >= 0 else None
        raise RefError(rc, ref().ref_last_error().decode(), pair)


def ref_build_condensed(samples, offsets, half_width=-1, auto_widen=False, workers=1,
                        ids=None):
    samples, offsets = _f64(samples), _i64a(offsets)
    p = len(offsets) - 1
    out = np.empty(max(p * (p - 1) // 2, 1), dtype=np.float64)
    ev = C.c_uint64()
    if ids is None:
        rc = ref().ref_build_condensed(samples, offsets, p, half_width, int(auto_widen), workers,
                                       out, C.byref(ev))
    else:
        arr = (C.c_char_p * p)(*[s.encode() for s in ids])
        rc = ref().ref_build_condensed_ids(samples, offsets, p, arr, half_width, int(auto_widen),
                                           workers, out, C.byref(ev))
    _ref_check(rc)
    return out[: p * (p - 1) // 2], int(ev.value)


def ref_dtw(x, y, half_width=-1) -> float:
    x, y = _f64(x), _f64(y)
    v = C.c_double()
    _ref_check(ref().ref_dtw(x, len(x), y, len(y), half_width, C.byref(v)))
    return v.value


def ref_dtw_brute_force(x, y, half_width=-1) -> float:
    x, y = _f64(x), _f64(y)
    v = C.c_double()
    _ref_check(ref().ref_dtw_brute_force(x, len(x), y, len(y), half_width, C.byref(v)))
    return v.value


def ref_kmedoids(D, p, k, restarts=10, max_iterations=100, seed=0, observer=None):
    med = np.empty(max(k, 1), dtype=np.int64)
    asg = np.empty(p, dtype=np.int64)
    cost = C.c_double()
    cb = OBSERVER((lambda u, r, it, c: observer(r, it, c)) if observer else (lambda *a: None))
    _ref_check(ref().ref_kmedoids(_f64(D), p, k, restarts, max_iterations, seed, cb, None, med,
                                  asg, C.byref(cost)))
    return med[:k], asg, cost.value


def ref_sweep(D, p, medoids):
    k = len(medoids)
    asg = np.empty(p, dtype=np.int64)
    upd = np.empty(k, dtype=np.int64)
    cost = C.c_double()
    _ref_check(ref().ref_sweep(_f64(D), p, _i64a(medoids), k, asg, C.byref(cost), upd))
    return asg, cost.value, upd


def ref_silhouette(D, p, medoids, assignment):
    asg = _i64a(assignment)
    out = np.zeros(max(p, 1), dtype=np.float64)
    mean = C.c_double()
    _ref_check(ref().ref_silhouette(_f64(D), p, _i64a(medoids), len(medoids), asg, len(asg), out,
                                    C.byref(mean)))
    return out[:p], mean.value


# ---------------------------------------------------------------- host I/O (reference)
def _ref_take(ptr, n, dtype):
    try:
        if n == 0:
            return np.zeros(0, dtype=dtype)
        ct = C.c_double if dtype == np.float64 else C.c_int64
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()
    finally:
        ref().ref_free(ptr)


def ref_save_matrix(D, p, path):
    """dtwclust::save_matrix (distance_matrix.hpp:104-122)."""
    _ref_check(ref().ref_save_matrix(_f64(D), p, os.fsencode(path)))


def ref_load_matrix(path):
    """dtwclust::load_matrix (distance_matrix.hpp:127-192) -> (p, condensed)."""
    p, buf = _i64(), C.c_void_p()
    _ref_check(ref().ref_load_matrix(os.fsencode(path), C.byref(p), C.byref(buf)))
    n = int(p.value) * (int(p.value) - 1) // 2
    return int(p.value), _ref_take(buf, n, np.float64)


def ref_ingest(paths, label_column=False, delimiter=None):
    """dtwclust::ingest (csv.hpp:55-106) -> (samples, offsets, ids)."""
    enc = [os.fsencode(x) for x in paths]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    p, smp, off, ids = _i64(), C.c_void_p(), C.c_void_p(), C.c_void_p()
    _ref_check(ref().ref_ingest(arr, len(enc), int(label_column),
                                0 if delimiter is None else ord(delimiter), C.byref(p),
                                C.byref(smp), C.byref(off), C.byref(ids)))
    n = int(p.value)
    offsets = _ref_take(off, n + 1, np.int64)
    samples = _ref_take(smp, int(offsets[-1]), np.float64)
    try:
        text = C.cast(ids, C.c_char_p).value.decode()
    finally:
        ref().ref_free(ids)
    return samples, offsets, text.split("\n")[:n]


def ref_z_normalize(samples, offsets):
    """dtwclust::detail::z_normalize (runner.hpp:82-95), returns a normalised copy."""
    out = _f64(samples).copy()
    _ref_check(ref().ref_z_normalize(out, _i64a(offsets), len(offsets) - 1))
    return out
