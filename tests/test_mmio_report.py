"""Matrix Market files and the CLI report schema (paper_2601_04112_b200/mmio.py, report.py)
against the compiled reference's own mmio.hpp (oracle/_ref)."""
import ctypes as C
import os

import numpy as np
import pytest

from oracle import refbind
from paper_2601_04112_b200 import abi, configs, lsamgdd, mmio, report


@pytest.fixture(scope="module")
def ref():
    try:
        return refbind.reference()
    except (FileNotFoundError, OSError):
        pytest.skip("oracle/_ref not built")


def test_mm_write_is_byte_identical_and_reads_back(ref, tmp_path):
    cfg = configs.config("c2", 12)
    mine, theirs = str(tmp_path / "mine.mtx"), str(tmp_path / "ref.mtx")
    mmio.mm_write(mine, cfg.g_rowptr, cfg.g_cols, cfg.g_vals, cfg.n)
    g = abi.csr_struct(cfg.g_rowptr, cfg.g_cols, cfg.g_vals, cfg.n)
    err = C.create_string_buffer(512)
    abi.check(ref.fn("mm_write")(C.byref(g), theirs.encode(), err, C.c_size_t(512)), err)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    rp, ci, va, nc = mmio.mm_read(mine)
    assert nc == cfg.n and np.array_equal(rp, cfg.g_rowptr) and np.array_equal(ci, cfg.g_cols)
    assert np.array_equal(va, cfg.g_vals)  # %.17g round-trips the bits
    # the reference reads my file into the same CSR
    sizes = (C.c_int64 * 3)()
    abi.check(ref.fn("mm_read")(mine.encode(), sizes, None, None, None, err, C.c_size_t(512)), err)
    off, col, val = np.empty(sizes[0] + 1, np.int64), np.empty(sizes[2], np.int64), np.empty(sizes[2])
    abi.check(ref.fn("mm_read")(mine.encode(), sizes, abi.ptr(off), abi.ptr(col), abi.ptr(val), err, C.c_size_t(512)), err)
    assert np.array_equal(off, cfg.g_rowptr) and np.array_equal(col, cfg.g_cols) and np.array_equal(val, cfg.g_vals)


def test_mm_vector_and_symmetric_and_errors(ref, tmp_path):
    v = configs.mt19937_64_uniform(7, 50)
    mine, theirs = str(tmp_path / "v.mtx"), str(tmp_path / "vr.mtx")
    mmio.mm_write_vector(mine, v)
    err = C.create_string_buffer(512)
    abi.check(ref.fn("mm_write_vector")(abi.ptr(v), C.c_int64(50), theirs.encode(), err, C.c_size_t(512)), err)
    assert open(mine, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(mmio.mm_read_vector(theirs), v)
    sym = tmp_path / "s.mtx"
    sym.write_text("%%MatrixMarket matrix coordinate real symmetric\n% comment\n3 3 3\n1 1 2.0\n2 1 -1.0\n3 3 0.0\n")
    rp, ci, va, nc = mmio.mm_read(str(sym))
    assert rp.tolist() == [0, 2, 3, 3] and ci.tolist() == [0, 1, 0] and va.tolist() == [2.0, -1.0, -1.0]
    bad = tmp_path / "b.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(lsamgdd.FormatError, match="outside 2x2"):
        mmio.mm_read(str(bad))
    bad.write_text("%%MatrixMarket matrix coordinate complex general\n1 1 0\n")
    with pytest.raises(lsamgdd.FormatError, match="unsupported field"):
        mmio.mm_read(str(bad))
    with pytest.raises(lsamgdd.FormatError, match="cannot open"):
        mmio.mm_read(str(tmp_path / "missing.mtx"))


def test_report_schema_numbers():
    assert report.csv_num(float("nan")) == "nan" and report.csv_num(float("inf")) == "inf"
    assert report.csv_num(-float("inf")) == "-inf" and report.csv_num(0.1) == "0.10000000000000001"
    assert report.CSV_HEADER.split(",") == ["value", "iterations", "rho", "iters_to_tenth", "op_complexity", "levels",
                                            "setup_s", "solve_s"]
    doc = {"iterations": 7, "rho": 0.5, "iters_to_tenth": 3.3, "op_complexity": 1.25, "levels": 3, "setup_s": 0.5, "solve_s": 0.25}
    assert report.csv_row(1e-3, doc) == "0.001,7,0.5,3.2999999999999998,1.25,3,0.5,0.25"
