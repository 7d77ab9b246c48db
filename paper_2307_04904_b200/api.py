"""Host-side mirror of the reference's hot-path interface, backed by libdtwgpu.so.

Same names, argument meaning and error behaviour as the reference's C++ entry points
(namespace dtwclust), so code and tests written against those read the same here:

  TimeSeries / validate / validate_dataset     time_series.hpp:13-45
  WarpWindow                                   warp_window.hpp:13-47
  BuildStats / build_matrix                    pairwise.hpp:21-23, 62-127
  DistanceMatrix                               distance_matrix.hpp:20-78
  KMedoidsConfig / kmedoids                    kmedoids.hpp:15-20, 148-189
  ClusterResult / assign_to_medoids /
  assignment_cost                              cluster_result.hpp:27-72
  Error + subclasses (codes = ErrorCode)       errors.hpp:11-176

Every distance and every sweep runs on the GPU through the C-ABI; there is no CPU
fallback (a missing library or device raises).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from . import _native

FP64 = 0
FP32 = 1


# ----------------------------------------------------------------------------- errors
class Error(RuntimeError):
    code = 0

    def __init__(self, message: str = ""):
        super().__init__(message)


class InvalidArgumentsError(Error):
    code = 2


class InvalidSeriesError(Error):
    code = 5

    def __init__(self, id_: str, message: str):
        super().__init__(f"series '{id_}': {message}")
        self.id = id_


class EmptyDatasetError(Error):
    code = 7

    def __init__(self, message: str = "dataset contains no series"):
        super().__init__(message)


class BandInfeasibleError(Error):
    code = 8

    def __init__(self, message: str, pair_i: int = -1, pair_j: int = -1):
        super().__init__(message)
        self.pair_i = pair_i
        self.pair_j = pair_j

    def has_pair(self) -> bool:
        return self.pair_i >= 0


class KOutOfRangeError(Error):
    code = 10


class DistanceMatrixInvalidError(Error):
    code = 11


class IndexOutOfRangeError(Error):
    code = 12

    def __init__(self, index: int, p: int):
        super().__init__(f"index {index} is outside [0, {p})")


class SingleClusterUndefinedError(Error):
    code = 13

    def __init__(self, message: str = "silhouette scores are undefined for a single cluster; "
                                      "request k >= 2"):
        super().__init__(message)


class DeviceError(Error):
    code = 100


_BY_CODE = {2: InvalidArgumentsError, 7: EmptyDatasetError, 10: KOutOfRangeError,
            11: DistanceMatrixInvalidError, 13: SingleClusterUndefinedError}


# ----------------------------------------------------------------------------- engine
class Engine:
    """One dtwg_ctx (device buffers, stream, resident series and matrix) on one GPU."""

    def __init__(self, device: int = 0, devices: Optional[Sequence[int]] = None):
        """devices: drive several GPUs from this one context (dtwg_create_multi): builds
        split the slots over them, k-medoids splits the restarts; results are identical."""
        self.L = _native.lib()
        h = C.c_void_p()
        if devices:
            arr = (C.c_int * len(devices))(*devices)
            rc = self.L.dtwg_create_multi(arr, len(devices), C.byref(h))
            device = int(devices[0])
        else:
            rc = self.L.dtwg_create(device, C.byref(h))
        if rc != 0:
            raise DeviceError(f"dtwg_create(device={device}) failed with code {rc}: no CUDA "
                              "device visible (there is no CPU fallback)")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.L.dtwg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- error translation ---------------------------------------------------------
    def check(self, rc: int) -> None:
        if rc == 0:
            return
        msg = self.L.dtwg_last_error(self.h).decode()
        if rc == 8:
            i, j = C.c_int64(), C.c_int64()
            self.L.dtwg_last_error_pair(self.h, C.byref(i), C.byref(j))
            raise BandInfeasibleError(msg, int(i.value), int(j.value))
        if rc == 5:
            raise InvalidSeriesError(msg.split(":")[0].replace("series ", "").strip("'#"),
                                     msg.split(": ", 1)[-1])
        if rc == 12:
            e = IndexOutOfRangeError(-1, -1)
            e.args = (msg,)
            raise e
        cls = _BY_CODE.get(rc)
        if cls is not None:
            raise cls(msg)
        raise DeviceError(f"[code {rc}] {msg}")

    # -- low level -----------------------------------------------------------------
    def set_stream(self, stream_ptr: int) -> None:
        self.check(self.L.dtwg_set_stream(self.h, C.c_void_p(stream_ptr) if stream_ptr else None))

    def synchronize(self) -> None:
        self.check(self.L.dtwg_synchronize(self.h))

    def upload(self, samples: np.ndarray, offsets: np.ndarray) -> None:
        samples = np.ascontiguousarray(samples, dtype=np.float64)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.check(self.L.dtwg_upload_series(self.h, samples, offsets, len(offsets) - 1))

    def fill_slots(self, half_width: int, auto_widen: bool, precision: int, slot_begin: int,
                   slot_end: int, d_out: int = 0) -> None:
        self.check(self.L.dtwg_fill_slots(self.h, half_width, int(auto_widen), precision,
                                          slot_begin, slot_end,
                                          C.c_void_p(d_out) if d_out else None))

    def count_cells(self, half_width: int, auto_widen: bool, slot_begin: int,
                    slot_end: int) -> int:
        v = C.c_uint64()
        self.check(self.L.dtwg_count_cells(self.h, half_width, int(auto_widen), slot_begin,
                                           slot_end, C.byref(v)))
        return int(v.value)

    def last_fill_ms(self) -> float:
        v = C.c_float()
        self.check(self.L.dtwg_last_fill_ms(self.h, C.byref(v)))
        return float(v.value)

    def launch_count(self) -> int:
        return int(self.L.dtwg_launch_count(self.h))

    def force_kernel(self, family: int = -1, G: int = 0, R: int = 0) -> None:
        """Tests/diagnostics: pin the kernel family/(G, R); family < 0 = cost model."""
        self.check(self.L.dtwg_force_kernel(self.h, family, G, R))

    def measure_cell_peak(self, precision: int = FP64) -> float:
        """Cells/s ceiling of the bare cell body on this GPU (roofline denominator)."""
        v = C.c_double()
        self.check(self.L.dtwg_measure_cell_peak(self.h, precision, C.byref(v)))
        return float(v.value)

    def km_stats(self, reset: bool = False) -> dict:
        """Sweep count and device time / algorithmic bytes of the k-medoids kernels."""
        out = np.zeros(8, dtype=np.float64)
        self.check(self.L.dtwg_km_stats(self.h, out, int(reset)))
        return {"sweeps": int(out[0]), "assign_ms": out[1], "assign_bytes": out[2],
                "update_ms": out[3], "update_bytes": out[4], "prep_ms": out[5],
                "cluster_layout": {0: None, 1: "fp64", 2: "fp32"}.get(int(out[6])),
                "layout_ms": out[7]}

    def last_plan(self) -> str:
        return self.L.dtwg_last_plan(self.h).decode()

    def build_condensed(self, samples, offsets, half_width=-1, auto_widen=False, workers=1,
                        precision=FP64) -> np.ndarray:
        samples = np.ascontiguousarray(samples, dtype=np.float64)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        p = len(offsets) - 1
        total = max(p * (p - 1) // 2, 0)
        out = np.empty(max(total, 1), dtype=np.float64)
        ev = C.c_uint64()
        self.check(self.L.dtwg_build_matrix(self.h, samples, offsets, p, half_width,
                                            int(auto_widen), workers, precision,
                                            out.ctypes.data_as(C.c_void_p), C.byref(ev)))
        self._last_evaluations = int(ev.value)
        return out[:total]

    # -- fused fill + all-gather over peer memory (include/dtwgpu.h, dtwg_exchange_*) --
    def exchange_export(self, p: int) -> bytes:
        buf = C.create_string_buffer(64)
        self.check(self.L.dtwg_exchange_export(self.h, p, buf))
        return buf.raw

    def exchange_open(self, handles, rank: int) -> None:
        blob = b"".join(handles)
        self.check(self.L.dtwg_exchange_open(self.h, blob, len(handles), rank))

    def exchange_fill(self, half_width: int, auto_widen: bool, precision: int, b: int,
                      e: int) -> None:
        self.check(self.L.dtwg_exchange_fill(self.h, half_width, int(auto_widen), precision, b, e))

    def exchange_complete(self) -> None:
        self.check(self.L.dtwg_exchange_complete(self.h))

    def exchange_close(self) -> None:
        self.check(self.L.dtwg_exchange_close(self.h))

    def adopt(self, condensed, p: int, on_device_ptr: int = 0) -> None:
        if on_device_ptr:
            self.check(self.L.dtwg_adopt_condensed(self.h, C.c_void_p(on_device_ptr), p, 1))
        else:
            cond = np.ascontiguousarray(condensed, dtype=np.float64)
            self.check(self.L.dtwg_adopt_condensed(
                self.h, cond.ctypes.data_as(C.c_void_p) if cond.size else None, p, 0))

    def download(self, p: int) -> np.ndarray:
        out = np.empty(max(p * (p - 1) // 2, 1), dtype=np.float64)
        self.check(self.L.dtwg_download_condensed(self.h, out))
        return out[: p * (p - 1) // 2]

    def download_range(self, b: int, e: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Slots [b, e) of the resident matrix (a rank's own slice during an exchange)."""
        if out is None:
            out = np.empty(max(e - b, 1), dtype=np.float64)
        self.check(self.L.dtwg_download_range(self.h, b, e, C.c_void_p(out.ctypes.data)))
        return out[: e - b]

    def kmedoids(self, p, k, restarts, max_iterations, seed, restart_begin=0, restart_end=None,
                 observer=None):
        if restart_end is None:
            restart_end = restarts
        med = np.empty(max(k, 1), dtype=np.int64)
        asg = np.empty(max(p, 1), dtype=np.int64)
        cost = C.c_double()
        best_r = C.c_int64(-1)
        errors = []

        def _obs(_u, r, it, c):
            try:
                observer(int(r), int(it), float(c))
            except Exception as e:  # surface after the native call returns
                errors.append(e)

        cb = _native.OBSERVER(_obs if observer else (lambda *a: None))
        self.check(self.L.dtwg_kmedoids(self.h, k, restarts, max_iterations, seed & (2**64 - 1),
                                        restart_begin, restart_end, cb, None, med, asg,
                                        C.byref(cost), C.byref(best_r)))
        if errors:
            raise errors[0]
        return med[:k].copy(), asg[:p].copy(), float(cost.value), int(best_r.value)

    def silhouette(self, medoids, assignment):
        medoids = np.ascontiguousarray(medoids, dtype=np.int64)
        assignment = np.ascontiguousarray(assignment, dtype=np.int64)
        out = np.zeros(max(len(assignment), 1), dtype=np.float64)
        mean = C.c_double()
        self.check(self.L.dtwg_silhouette(self.h, medoids, len(medoids), assignment,
                                          len(assignment), out, C.byref(mean)))
        return out[: len(assignment)], float(mean.value)

    def km_assign(self, medoids):
        medoids = np.ascontiguousarray(medoids, dtype=np.int64)
        p = self._p_resident
        asg = np.empty(p, dtype=np.int64)
        dist = np.empty(p, dtype=np.float64)
        self.check(self.L.dtwg_km_assign(self.h, medoids, len(medoids), asg, dist))
        return asg, dist

    def km_update(self, medoids, assignment):
        medoids = np.ascontiguousarray(medoids, dtype=np.int64)
        out = np.empty(len(medoids), dtype=np.int64)
        self.check(self.L.dtwg_km_update(self.h, medoids, len(medoids),
                                         np.ascontiguousarray(assignment, dtype=np.int64), out))
        return out

    def km_nearest_update(self, current, chosen, nearest):
        chosen = np.ascontiguousarray(chosen, dtype=np.uint8)
        nearest = np.ascontiguousarray(nearest, dtype=np.float64).copy()
        self.check(self.L.dtwg_km_nearest_update(self.h, current, chosen, nearest))
        return nearest


_ENGINES: dict = {}


def engine(device: int = 0, devices: Optional[Sequence[int]] = None) -> Engine:
    """Process-wide engine per device, or per device list (one context over several GPUs:
    builds split the slots, k-medoids the restarts -- dtwg_create_multi)."""
    key = tuple(int(d) for d in devices) if devices else device
    e = _ENGINES.get(key)
    if e is None or e.h is None:
        e = Engine(device, devices=list(key) if devices else None)
        e.multi = bool(devices) and len(key) > 1
        _ENGINES[key] = e
    return e


# ----------------------------------------------------------------------------- types
@dataclass
class TimeSeries:
    id: str
    samples: np.ndarray

    def __post_init__(self):
        self.samples = np.asarray(self.samples, dtype=np.float64).reshape(-1)

    def length(self) -> int:
        return int(self.samples.shape[0])

    def __eq__(self, other):
        return (isinstance(other, TimeSeries) and self.id == other.id and
                np.array_equal(self.samples, other.samples))


def validate(series: TimeSeries) -> None:
    """time_series.hpp:24-33."""
    if series.length() == 0:
        raise InvalidSeriesError(series.id, "series is empty")
    if not np.all(np.isfinite(series.samples)):
        raise InvalidSeriesError(series.id, "series contains a non-finite sample")


def validate_dataset(dataset: Sequence[TimeSeries]) -> None:
    """time_series.hpp:36-45: each series in order, then id uniqueness."""
    seen = set()
    for s in dataset:
        validate(s)
        if s.id in seen:
            raise InvalidSeriesError(s.id, "duplicate id in dataset")
        seen.add(s.id)


class WarpWindow:
    """warp_window.hpp:13-47 (Sakoe-Chiba band or unlimited)."""

    def __init__(self, half_width: Optional[int]):
        self._hw = half_width

    @staticmethod
    def unlimited() -> "WarpWindow":
        return WarpWindow(None)

    @staticmethod
    def banded(half_width: int) -> "WarpWindow":
        if half_width < 0:
            raise InvalidArgumentsError("half_width must be >= 0")
        return WarpWindow(int(half_width))

    def is_unlimited(self) -> bool:
        return self._hw is None

    def half_width(self) -> int:
        if self._hw is None:
            raise ValueError("unlimited window has no half-width")
        return self._hw

    def feasible_for(self, n: int, m: int) -> bool:
        return self._hw is None or self._hw >= abs(n - m)

    def effective(self, n: int, m: int) -> int:
        return self._hw if self._hw is not None else max(n, m)

    def describe(self) -> str:
        return "unlimited" if self._hw is None else str(self._hw)

    @property
    def native(self) -> int:
        return -1 if self._hw is None else self._hw

    def __eq__(self, other):
        return isinstance(other, WarpWindow) and self._hw == other._hw

    def __repr__(self):
        return f"WarpWindow({self.describe()})"


@dataclass
class BuildStats:
    evaluations: int = 0


def condensed_size(p: int) -> int:
    return p * (p - 1) // 2


class DistanceMatrix:
    """distance_matrix.hpp:20-78: condensed upper triangle, row-major, p(p-1)/2 values.

    A matrix produced by build_matrix also stays resident on the GPU (its engine), so
    kmedoids over it needs no upload.
    """

    def __init__(self, p: int):
        if p == 0:
            raise DistanceMatrixInvalidError("matrix needs at least one series")
        self._p = int(p)
        self._values = np.zeros(condensed_size(p), dtype=np.float64)
        self._engine: Optional[Engine] = None

    @staticmethod
    def from_condensed(p: int, values) -> "DistanceMatrix":
        m = DistanceMatrix(p)
        values = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
        if values.shape[0] != condensed_size(p):
            raise DistanceMatrixInvalidError(
                f"condensed storage holds {values.shape[0]} values, expected {condensed_size(p)}")
        if values.size and not np.all(np.isfinite(values) & (values >= 0.0)):
            raise DistanceMatrixInvalidError("entries must be finite and non-negative")
        m._values = values
        return m

    def size(self) -> int:
        return self._p

    def _offset(self, i: int, j: int) -> int:
        if i > j:
            i, j = j, i
        return i * (2 * self._p - i - 1) // 2 + (j - i - 1)

    def distance(self, i: int, j: int) -> float:
        for t in (i, j):
            if t < 0 or t >= self._p:
                raise IndexOutOfRangeError(t, self._p)
        if i == j:
            return 0.0
        return float(self._values[self._offset(i, j)])

    def condensed(self) -> np.ndarray:
        return self._values

    def square(self) -> np.ndarray:
        p = self._p
        sq = np.zeros((p, p), dtype=np.float64)
        iu = np.triu_indices(p, 1)
        sq[iu] = self._values
        sq.T[iu] = self._values
        return sq

    def __eq__(self, other):
        return (isinstance(other, DistanceMatrix) and self._p == other._p and
                np.array_equal(self._values, other._values))


def _pack(dataset: Sequence[TimeSeries]):
    lens = np.array([s.length() for s in dataset], dtype=np.int64)
    offsets = np.zeros(len(dataset) + 1, dtype=np.int64)
    np.cumsum(lens, out=offsets[1:])
    samples = (np.concatenate([s.samples for s in dataset]) if len(dataset)
               else np.zeros(0, dtype=np.float64))
    return np.ascontiguousarray(samples, dtype=np.float64), offsets


def build_matrix(dataset: Sequence[TimeSeries], w: WarpWindow, workers: int,
                 stats: Optional[BuildStats] = None, auto_widen: bool = False, *,
                 precision: int = FP64, device: int = 0,
                 devices: Optional[Sequence[int]] = None) -> DistanceMatrix:
    """pairwise.hpp:62-127 on the GPU. `workers` is validated (>= 1) as the reference does.

    Validation order follows the reference: EmptyDataset, InvalidArguments (workers),
    InvalidSeries (validate_dataset, ids included), then the first band-infeasible pair.
    """
    if len(dataset) == 0:
        raise EmptyDatasetError()
    if workers == 0:
        raise InvalidArgumentsError("workers must be >= 1")
    validate_dataset(dataset)
    samples, offsets = _pack(dataset)
    eng = engine(device, devices)
    cond = eng.build_condensed(samples, offsets, w.native, auto_widen, max(int(workers), 1),
                               precision)
    if stats is not None:
        stats.evaluations = eng._last_evaluations
    return _wrap(cond, len(dataset), eng)


def _wrap(cond: np.ndarray, p: int, eng: Engine) -> DistanceMatrix:
    m = DistanceMatrix(p)
    m._values = cond
    m._engine = eng
    if not getattr(eng, "multi", False):  # a multi-device build leaves only slices resident
        eng._resident_matrix = m
        eng._p_resident = p
    return m


def dtw_distance(x: TimeSeries, y: TimeSeries, w: WarpWindow, *, device: int = 0) -> float:
    """dtw.hpp:40-75 for one pair on the GPU: validate both series, then the band's
    feasibility (BandInfeasibleError without a pair), then the bit-identical distance."""
    validate(x)
    validate(y)
    n, m = len(x.samples), len(y.samples)
    if not w.feasible_for(n, m):
        raise BandInfeasibleError(
            f"half-width {w.half_width()} is narrower than the length gap of {abs(n - m)} "
            f"(lengths {n} and {m})")
    samples = np.concatenate([np.asarray(x.samples, np.float64), np.asarray(y.samples, np.float64)])
    offsets = np.array([0, n, n + m], dtype=np.int64)
    return float(engine(device).build_condensed(samples, offsets, w.native, False, 1, FP64)[0])


def build_matrix_packed(samples: np.ndarray, offsets: np.ndarray, w: WarpWindow,
                        auto_widen: bool = False, *, precision: int = FP64,
                        device: int = 0, devices: Optional[Sequence[int]] = None
                        ) -> DistanceMatrix:
    """build_matrix over an already-packed CSR dataset (ids implicit and unique)."""
    eng = engine(device, devices)
    p = len(offsets) - 1
    if p <= 0:
        raise EmptyDatasetError()
    cond = eng.build_condensed(samples, offsets, w.native, auto_widen, 1, precision)
    return _wrap(cond, p, eng)


# ----------------------------------------------------------------------------- k-medoids
@dataclass
class KMedoidsConfig:
    k: int = 1
    restarts: int = 10
    max_iterations: int = 100
    seed: int = 0


@dataclass
class ClusterResult:
    medoids: list = field(default_factory=list)
    assignment: list = field(default_factory=list)
    total_cost: float = 0.0
    certificate: str = "local_heuristic"
    nodes_explored: int = 0

    def __eq__(self, other):
        return (isinstance(other, ClusterResult) and list(self.medoids) == list(other.medoids)
                and list(self.assignment) == list(other.assignment)
                and self.total_cost == other.total_cost and self.certificate == other.certificate
                and self.nodes_explored == other.nodes_explored)


IterationObserver = Callable[[int, int, float], None]


def _resident(source: DistanceMatrix, device: int = 0,
              devices: Optional[Sequence[int]] = None) -> Engine:
    eng = engine(device, devices) if devices else (source._engine or engine(device))
    if getattr(eng, "_resident_matrix", None) is not source:
        eng.adopt(source.condensed(), source.size())
        eng._resident_matrix = source
        eng._p_resident = source.size()
        source._engine = eng
    return eng


def kmedoids(source: DistanceMatrix, config: KMedoidsConfig,
             observer: Optional[IterationObserver] = None, *, device: int = 0,
             devices: Optional[Sequence[int]] = None,
             restart_range: Optional[tuple] = None) -> ClusterResult:
    """kmedoids.hpp:148-189 with the distance sweeps on the GPU."""
    p = source.size()
    if config.k < 1 or config.k > p:
        raise KOutOfRangeError(f"k={config.k} is outside [1, p] with p={p}")
    if config.restarts < 1:
        raise InvalidArgumentsError("restarts must be >= 1")
    if config.max_iterations < 1:
        raise InvalidArgumentsError("max_iterations must be >= 1")
    eng = _resident(source, device, devices)
    rb, re = restart_range if restart_range else (0, config.restarts)
    med, asg, cost, best_r = eng.kmedoids(p, config.k, config.restarts, config.max_iterations,
                                          config.seed, rb, re, observer)
    res = ClusterResult([int(v) for v in med], [int(v) for v in asg], cost)
    res.best_restart = best_r
    return res


def assign_to_medoids(source: DistanceMatrix, medoids) -> list:
    """cluster_result.hpp:40-61 on the GPU."""
    eng = _resident(source)
    asg, _ = eng.km_assign(medoids)
    return [int(v) for v in asg]


def assignment_cost(source: DistanceMatrix, assignment) -> float:
    """cluster_result.hpp:65-72: ascending-j sequential sum."""
    total = 0.0
    for j, a in enumerate(assignment):
        total += source.distance(j, int(a))
    return total


def update_medoids(source: DistanceMatrix, medoids, assignment) -> list:
    """kmedoids.hpp:84-139 (detail::update_medoids) on the GPU."""
    eng = _resident(source)
    return [int(v) for v in eng.km_update(medoids, assignment)]


# ----------------------------------------------------------------------------- scores
@dataclass
class ScoreReport:
    """validation.hpp:20-24."""
    silhouette: list = field(default_factory=list)
    mean_silhouette: float = 0.0
    elbow: list = field(default_factory=list)


def silhouette_scores(distances: DistanceMatrix, result: ClusterResult) -> ScoreReport:
    """validation.hpp:30-79 over the GPU-resident matrix, bit-identical to the reference."""
    eng = _resident(distances)
    sil, mean = eng.silhouette(result.medoids, result.assignment)
    return ScoreReport([float(v) for v in sil], mean)
