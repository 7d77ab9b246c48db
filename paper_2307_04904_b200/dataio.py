"""Host-side data path either side of the fill, over libdtwgpu.so.

Mirrors the reference's I/O entry points with the same formats, results and errors:

* ``save_matrix`` / ``load_matrix``    -- distance_matrix.hpp:104-192 (text, byte-identical,
  rows formatted / parsed by several host threads),
* ``save_matrix_binary`` / ``load_matrix_binary`` -- a binary sidecar (condensed doubles),
* ``ingest`` / ``ingest_packed``       -- csv.hpp:55-106 (one series per CSV row),
* ``z_normalize`` / ``z_normalize_packed`` -- runner.hpp:82-95 (bit-identical).

None of these needs a GPU; they run in csrc/host_io.cpp.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from . import _native
from .api import (DistanceMatrix, DistanceMatrixInvalidError, EmptyDatasetError, Error,
                  InvalidArgumentsError, InvalidSeriesError, TimeSeries, condensed_size)


class IoFailureError(Error):
    code = 3


class ParseFailureError(Error):
    code = 4

    def __init__(self, message: str, file: str = "", line: int = -1, column: int = -1):
        super().__init__(message)
        self.file, self.line, self.column = file, line, column


class EmptySeriesError(Error):
    code = 6

    def __init__(self, message: str, line: int = -1):
        super().__init__(message)
        self.line = line


class FormatViolationError(Error):
    code = 9

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}")
        self.line = line


def _check(rc: int) -> None:
    if rc == 0:
        return
    L = _native.lib()
    line, col = C.c_int64(), C.c_int64()
    msg = L.dtwg_io_last_error(C.byref(line), C.byref(col)).decode()
    where = L.dtwg_io_last_file().decode()
    if rc == 3:
        raise IoFailureError(msg)
    if rc == 4:
        raise ParseFailureError(msg, where, int(line.value), int(col.value))
    if rc == 5:
        prefix = f"series '{where}': "
        raise InvalidSeriesError(where, msg[len(prefix):] if msg.startswith(prefix) else msg)
    if rc == 6:
        raise EmptySeriesError(msg, int(line.value))
    if rc == 7:
        raise EmptyDatasetError()
    if rc == 9:
        raise FormatViolationError(int(line.value), msg)
    if rc == 11:
        raise DistanceMatrixInvalidError(msg)
    raise InvalidArgumentsError(f"[code {rc}] {msg}")


def _path(path) -> bytes:
    return os.fsencode(os.fspath(path))


def _take(ptr: C.c_void_p, n: int) -> np.ndarray:
    """Copies n doubles out of a library-allocated buffer and frees it."""
    L = _native.lib()
    try:
        if n == 0:
            return np.zeros(0)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(n,)).copy()
    finally:
        L.dtwg_free(ptr)


# ----------------------------------------------------------------------------- matrices
def save_matrix(m: DistanceMatrix, path, threads: int = 0) -> None:
    """distance_matrix.hpp:104-122: `p=<count>`, p rows of p values, literal 0 diagonal."""
    cond = np.ascontiguousarray(m.condensed(), dtype=np.float64)
    _check(_native.lib().dtwg_save_matrix_text(cond.ctypes.data, m.size(), _path(path), threads))


def load_matrix(path, threads: int = 0) -> DistanceMatrix:
    """distance_matrix.hpp:127-192, the reference's checks and first error."""
    p, buf = C.c_int64(), C.c_void_p()
    _check(_native.lib().dtwg_load_matrix_text(_path(path), threads, C.byref(p), C.byref(buf)))
    return DistanceMatrix.from_condensed(int(p.value), _take(buf, condensed_size(int(p.value))))


def save_matrix_binary(m: DistanceMatrix, path) -> None:
    cond = np.ascontiguousarray(m.condensed(), dtype=np.float64)
    _check(_native.lib().dtwg_save_matrix_binary(cond.ctypes.data, m.size(), _path(path)))


def load_matrix_binary(path) -> DistanceMatrix:
    p, buf = C.c_int64(), C.c_void_p()
    _check(_native.lib().dtwg_load_matrix_binary(_path(path), C.byref(p), C.byref(buf)))
    return DistanceMatrix.from_condensed(int(p.value), _take(buf, condensed_size(int(p.value))))


# ----------------------------------------------------------------------------- ingest
@dataclass
class CsvFormat:
    """csv.hpp:18-23."""
    label_column: bool = False
    delimiter: Optional[str] = None  # None: ',' (tab for .tsv files)


@dataclass
class PackedDataset:
    """Series i is samples[offsets[i]:offsets[i+1]], id ids[i] -- the fill's input layout."""
    samples: np.ndarray
    offsets: np.ndarray
    ids: List[str]

    @property
    def p(self) -> int:
        return len(self.ids)

    def to_series(self) -> List[TimeSeries]:
        return [TimeSeries(self.ids[i], self.samples[self.offsets[i]:self.offsets[i + 1]].copy())
                for i in range(self.p)]


def ingest_packed(paths: Sequence, fmt: CsvFormat = CsvFormat(), normalize: bool = False,
                  threads: int = 0) -> PackedDataset:
    """csv.hpp:55-106 (+ runner.hpp:82-95 when normalize), packed for the fill."""
    L = _native.lib()
    enc = [_path(p) for p in paths]
    arr = (C.c_char_p * max(len(enc), 1))(*enc)
    delim = 0 if fmt.delimiter is None else ord(fmt.delimiter)
    ds = C.c_void_p()
    _check(L.dtwg_ingest_csv(arr, len(enc), int(fmt.label_column), delim, threads, C.byref(ds)))
    try:
        p = int(L.dtwg_dataset_size(ds))
        off = np.ctypeslib.as_array(L.dtwg_dataset_offsets(ds), shape=(p + 1,)).copy()
        n = int(off[-1])
        smp = (np.ctypeslib.as_array(L.dtwg_dataset_samples(ds), shape=(n,)).copy() if n
               else np.zeros(0))
        ids = [L.dtwg_dataset_id(ds, i).decode() for i in range(p)]
    finally:
        L.dtwg_dataset_free(ds)
    if normalize:
        z_normalize_packed(smp, off, threads)
    return PackedDataset(smp, off, ids)


def ingest(paths: Sequence, fmt: CsvFormat = CsvFormat(), threads: int = 0) -> List[TimeSeries]:
    """csv.hpp:55-106: one TimeSeries per row, ids `<file name>:<row>`."""
    return ingest_packed(paths, fmt, False, threads).to_series()


def z_normalize_packed(samples: np.ndarray, offsets: np.ndarray, threads: int = 0) -> None:
    """runner.hpp:82-95 in place (population std; constant series become zeros)."""
    if samples.dtype != np.float64 or not samples.flags.c_contiguous:
        raise InvalidArgumentsError("samples must be a contiguous float64 array")
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    _check(_native.lib().dtwg_z_normalize(samples.ctypes.data, off.ctypes.data,
                                          len(off) - 1, threads))


def z_normalize(dataset: List[TimeSeries], threads: int = 0) -> None:
    """runner.hpp:82-95 on a list of TimeSeries, in place."""
    if not dataset:
        return
    lens = [len(s.samples) for s in dataset]
    off = np.zeros(len(dataset) + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    smp = np.concatenate([np.asarray(s.samples, dtype=np.float64) for s in dataset])
    z_normalize_packed(smp, off, threads)
    for i, s in enumerate(dataset):
        s.samples = smp[off[i]:off[i + 1]].copy()
