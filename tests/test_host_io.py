"""CPU tests of the host-side data path (csrc/host_io.cpp) against
the UNMODIFIED reference (oracle/_ref): matrix text files byte-identical, loads and
ingests with the same values, ids and first error (type, message, line/column), and
z-normalisation bit-identical. No GPU needed."""
import os

import numpy as np
import pytest

import oracle
from paper_2307_04904_b200 import api, dataio
from tests.helpers import ScalarRng, assert_bitwise, random_condensed

needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="oracle/_ref not built")


def write(path, text, mode="w"):
    with open(path, mode) as f:
        f.write(text)
    return str(path)


# ---------------------------------------------------------------- matrix text / binary
@needs_ref
@pytest.mark.parametrize("p,threads", [(1, 1), (2, 1), (7, 3), (64, 8), (301, 0)])
@pytest.mark.parametrize("block", [None, "4096"])
def test_save_matrix_byte_identical_and_round_trip(tmp_path, monkeypatch, p, threads, block):
    if block:
        monkeypatch.setenv("DTWGPU_IO_BLOCK", block)
    D = random_condensed(ScalarRng(p), p, 0.0, 1e6) if p > 1 else np.zeros(0)
    if p > 3:
        D[::5] = np.round(D[::5])  # integral values print without a fraction
        D[1] = 0.0
    m = api.DistanceMatrix.from_condensed(p, D)
    a, b = tmp_path / "gpu.txt", tmp_path / "ref.txt"
    dataio.save_matrix(m, a, threads)
    oracle.ref_save_matrix(D, p, str(b))
    assert a.read_bytes() == b.read_bytes()
    assert_bitwise(dataio.load_matrix(b, threads).condensed(), D)
    q, D2 = oracle.ref_load_matrix(str(a))
    assert q == p
    assert_bitwise(D2, D)
    dataio.save_matrix_binary(m, tmp_path / "m.bin")
    assert_bitwise(dataio.load_matrix_binary(tmp_path / "m.bin").condensed(), D)


BAD_MATRICES = {
    "empty": "",
    "no_header": "3\n",
    "header_zero": "p=0\n",
    "header_text": "p=abc\n",
    "header_space": "p=2 \n0,1\n1,0\n",
    "few_rows": "p=3\n0,1,2\n1,0,3\n",
    "many_cells": "p=2\n0,1,5\n1,0\n",
    "few_cells": "p=2\n0\n1,0\n",
    "bad_token": "p=2\n0,1e\n1e,0\n",
    "empty_token": "p=3\n0,,2\n1,0,3\n2,3,0\n",
    "diag": "p=2\n1,1\n1,0\n",
    "negative": "p=2\n0,-1\n-1,0\n",
    "inf": "p=2\n0,inf\ninf,0\n",
    "nan": "p=2\n0,nan\nnan,0\n",
    "asym": "p=3\n0,1,2\n1,0,3\n2,4,0\n",
    "asym_before_value_error": "p=3\n0,1,2\n1,0,3\n5,3,-1\n",
    "value_error_before_asym": "p=3\n0,1,2\n1,0,-3\n7,3,0\n",
    "trailing": "p=2\n0,1\n1,0\nx\n",
    "trailing_cr": "p=2\n0,1\n1,0\n\r\n",
    "trailing_empty_then_text": "p=2\n0,1\n1,0\n\nx\n",
    "crlf_ok": "p=2\r\n0,1.5\r\n1.5,0\r\n",
    "no_final_newline_ok": "p=2\n0,2\n2,0",
    "late_bad_row": "p=4\n0,1,2,3\n1,0,4,5\n2,4,0,6\n3,5,6,x\n",
}


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD_MATRICES))
@pytest.mark.parametrize("threads,block", [(1, None), (4, None), (3, "16")])
def test_load_matrix_errors_match_reference(tmp_path, monkeypatch, name, threads, block):
    """block: the streaming reader's text block (DTWGPU_IO_BLOCK); 16 bytes puts line and
    block boundaries everywhere."""
    if block:
        monkeypatch.setenv("DTWGPU_IO_BLOCK", block)
    path = write(tmp_path / f"{name}.txt", BAD_MATRICES[name], "w" if "\r" not in
                 BAD_MATRICES[name] else "w")
    with open(path, "wb") as f:
        f.write(BAD_MATRICES[name].encode())
    try:
        q, want = oracle.ref_load_matrix(path)
        ref_err = None
    except oracle.RefError as e:
        ref_err = e
    if ref_err is None:
        got = dataio.load_matrix(path, threads)
        assert got.size() == q
        assert_bitwise(got.condensed(), want)
        return
    with pytest.raises(api.Error) as ei:
        dataio.load_matrix(path, threads)
    assert ei.value.code == ref_err.code, (str(ei.value), str(ref_err))
    assert str(ei.value) == str(ref_err)


def test_missing_files_raise_io_failure(tmp_path):
    with pytest.raises(dataio.IoFailureError):
        dataio.load_matrix(tmp_path / "nope.txt")
    with pytest.raises(dataio.IoFailureError):
        dataio.ingest([tmp_path / "nope.csv"])
    with pytest.raises(dataio.FormatViolationError):
        dataio.load_matrix_binary(write(tmp_path / "x.bin", "DTWGMAT0"))


# ---------------------------------------------------------------- ingest
def _ingest_pair(paths, label=False, delim=None, threads=0):
    try:
        want = oracle.ref_ingest([str(p) for p in paths], label, delim)
        ref_err = None
    except oracle.RefError as e:
        want, ref_err = None, e
    fmt = dataio.CsvFormat(label, delim)
    if ref_err is not None:
        with pytest.raises(api.Error) as ei:
            dataio.ingest_packed(paths, fmt, threads=threads)
        assert ei.value.code == ref_err.code, (str(ei.value), str(ref_err))
        assert str(ei.value) == str(ref_err)
        return None
    got = dataio.ingest_packed(paths, fmt, threads=threads)
    assert_bitwise(got.samples, want[0])
    np.testing.assert_array_equal(got.offsets, want[1])
    assert got.ids == want[2]
    return got


CSV_CASES = {
    "ragged": ("a.csv", "1,2,3\n4.5,5e-3\n+7, 8 ,\t9\t,,\n-1e300,2\n"),
    "crlf": ("b.csv", "1,2\r\n3,4\r\n"),
    "tsv": ("c.tsv", "1\t2\t3\n4\t5\n"),
    "empty_cell": ("d.csv", "1,2\n3,,4\n"),
    "not_numeric": ("e.csv", "1,2\n3,x4\n"),
    "empty_row": ("f.csv", "1,2\n\n3,4\n"),
    "nan": ("g.csv", "1,2\n3,nan\n"),
    "inf": ("h.csv", "1,2\ninf,4\n"),
    "hex": ("i.csv", "0x10,2\n"),
    "only_commas": ("j.csv", "1\n,,,\n"),
    "spaces_cell": ("k.csv", "1,  ,2\n"),
}


@needs_ref
@pytest.mark.parametrize("case", sorted(CSV_CASES))
@pytest.mark.parametrize("threads", [1, 3])
def test_ingest_matches_reference(tmp_path, case, threads):
    name, text = CSV_CASES[case]
    path = tmp_path / name
    path.write_bytes(text.encode())
    _ingest_pair([path], threads=threads)


@needs_ref
def test_ingest_label_column_delimiter_and_duplicate_names(tmp_path):
    (tmp_path / "x").mkdir()
    (tmp_path / "y").mkdir()
    a = tmp_path / "x" / "train.csv"
    b = tmp_path / "y" / "train.csv"
    a.write_text("1,0.5,0.25\n2,3,4,5\n")
    b.write_text("1;7;8\n3;9\n")
    _ingest_pair([a], label=True)
    _ingest_pair([b], label=True, delim=";")
    got = _ingest_pair([a, b, a], label=True)
    assert got is None or got.ids[-1].endswith("#3:2")
    lab = tmp_path / "lab.csv"
    lab.write_text("1,2\n5\n")
    _ingest_pair([lab], label=True)  # second row has only a label -> EmptySeries
    empty = tmp_path / "empty.csv"
    empty.write_text("")
    _ingest_pair([empty])  # EmptyDataset


@needs_ref
def test_ingest_large_file_parallel(tmp_path):
    rng = np.random.default_rng(5)
    rows = [rng.normal(size=int(rng.integers(5, 60))) for _ in range(6000)]
    text = "\n".join(",".join(repr(float(v)) for v in r) for r in rows) + "\n"
    path = tmp_path / "big.csv"
    path.write_text(text)
    got = _ingest_pair([path], threads=8)
    assert got.p == 6000
    # an error deep in the file: the first one in file order is reported
    lines = text.splitlines()
    lines[4500] = lines[4500] + ",x"
    lines[5200] = ""
    bad = tmp_path / "bad.csv"
    bad.write_text("\n".join(lines) + "\n")
    _ingest_pair([bad], threads=8)


# ---------------------------------------------------------------- z-normalisation
@needs_ref
def test_z_normalize_bit_identical():
    rng = np.random.default_rng(9)
    rows = [rng.normal(size=int(n)) * 10 ** rng.uniform(-3, 3) + rng.uniform(-1e3, 1e3)
            for n in rng.integers(1, 300, size=200)]
    rows[3] = np.full(17, 2.5)   # constant -> zeros
    rows[4] = np.array([7.0])    # single sample -> zero
    off = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum([len(r) for r in rows], out=off[1:])
    smp = np.concatenate(rows)
    want = oracle.ref_z_normalize(smp, off)
    got = smp.copy()
    dataio.z_normalize_packed(got, off, threads=4)
    assert_bitwise(got, want)
    series = [api.TimeSeries(f"s{i}", r.copy()) for i, r in enumerate(rows)]
    dataio.z_normalize(series)
    assert_bitwise(np.concatenate([s.samples for s in series]), want)


def test_generators_match_native_z_normalize():
    """The synthetic configs' z-normalisation (generators.py) equals runner.hpp's."""
    from paper_2307_04904_b200 import generators as gen
    rng = gen.SplitMix64(2307049042)
    raw = np.cumsum(rng.gaussian(3 * 500).reshape(3, 500), axis=1)
    want = gen.z_normalize_rows(raw)
    got = raw.reshape(-1).copy()
    dataio.z_normalize_packed(got, np.array([0, 500, 1000, 1500], dtype=np.int64))
    assert_bitwise(got, want.reshape(-1))


@needs_ref
def test_large_matrix_text_threaded_identical(tmp_path):
    """p = 1500 (2.25 M cells, ~40 MB of text): byte-identical with 1 and 16 threads and
    with the reference, and loads back bit-exactly (timings printed)."""
    import time
    p = 1500
    D = random_condensed(ScalarRng(7), p, 0.0, 1e4)
    m = api.DistanceMatrix.from_condensed(p, D)
    t0 = time.perf_counter()
    oracle.ref_save_matrix(D, p, str(tmp_path / "ref.txt"))
    t_ref = time.perf_counter() - t0
    dataio.save_matrix(m, tmp_path / "one.txt", threads=1)
    t0 = time.perf_counter()
    dataio.save_matrix(m, tmp_path / "many.txt", threads=16)
    t_ours = time.perf_counter() - t0
    ref = (tmp_path / "ref.txt").read_bytes()
    assert (tmp_path / "one.txt").read_bytes() == ref
    assert (tmp_path / "many.txt").read_bytes() == ref
    t0 = time.perf_counter()
    back = dataio.load_matrix(tmp_path / "many.txt", threads=16)
    t_load = time.perf_counter() - t0
    t0 = time.perf_counter()
    q, D2 = oracle.ref_load_matrix(str(tmp_path / "ref.txt"))
    t_ref_load = time.perf_counter() - t0
    assert_bitwise(back.condensed(), D)
    assert_bitwise(D2, D)
    print(f"save: ours {t_ours:.3f}s vs reference {t_ref:.3f}s; load: ours {t_load:.3f}s vs "
          f"reference {t_ref_load:.3f}s")
    # (timings depend on the cores this container grants; printed, not asserted)
