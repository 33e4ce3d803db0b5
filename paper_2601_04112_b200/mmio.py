"""Matrix Market exchange files in the reference's dialect (mmio.hpp:62-160):
real coordinate (general; symmetric accepted on read) matrices and real
array vectors, 1-based on disk, values written with 17 significant digits so
a read-back reproduces the bits. Read errors raise ``FormatError`` with the
reference's messages. The same files feed the CPU reference (mm_read /
load_system, problems.hpp:191-218) and the B200 path.
"""
from __future__ import annotations

import numpy as np

from .lsamgdd import FormatError


def _data_lines(f):
    for line in f:
        s = line.strip()
        if not s or s.startswith("%"):
            continue
        yield line


def _header(f, path: str):
    first = f.readline()
    if not first:
        raise FormatError(f"{path}: empty file")
    tok = first.split()
    tok += [""] * (5 - len(tok))
    banner, obj, fmt, field, sym = [t.lower() for t in tok[:5]]
    if banner != "%%matrixmarket":
        raise FormatError(f"{path}: missing MatrixMarket banner")
    if obj != "matrix":
        raise FormatError(f"{path}: unsupported object '{obj}'")
    if field != "real":
        raise FormatError(f"{path}: unsupported field '{field}' (only real is supported)")
    return fmt, sym


def mm_write(path: str, rowptr: np.ndarray, cols: np.ndarray, vals: np.ndarray, n_cols: int) -> None:
    """mm_write (mmio.hpp:108-121): "%zu %zu %.17g" per stored entry, row by row."""
    n_rows = rowptr.shape[0] - 1
    rows = np.repeat(np.arange(1, n_rows + 1, dtype=np.int64), np.diff(rowptr))
    with open(path, "w") as out:
        out.write("%%MatrixMarket matrix coordinate real general\n")
        out.write(f"{n_rows} {n_cols} {cols.shape[0]}\n")
        chunk = 1 << 20
        for a in range(0, cols.shape[0], chunk):
            b = min(cols.shape[0], a + chunk)
            out.write("".join("%d %d %.17g\n" % (r, c + 1, v) for r, c, v in zip(rows[a:b], cols[a:b], vals[a:b])))


def mm_read(path: str):
    """mm_read (mmio.hpp:62-106) -> (rowptr, cols, vals, n_cols) as csr_from_triplets builds it
    (sparse.hpp:79-108: duplicates summed in file order, exact-zero sums dropped, columns ascending)."""
    try:
        f = open(path)
    except OSError:
        raise FormatError(f"{path}: cannot open file")
    with f:
        fmt, sym = _header(f, path)
        if fmt != "coordinate":
            raise FormatError(f"{path}: expected coordinate format, got '{fmt}'")
        if sym not in ("general", "symmetric"):
            raise FormatError(f"{path}: unsupported symmetry '{sym}'")
        lines = _data_lines(f)
        size = next(lines, None)
        if size is None:
            raise FormatError(f"{path}: missing size line")
        try:
            n_rows, n_cols, entries = (int(t) for t in size.split()[:3])
            assert n_rows >= 0 and n_cols >= 0 and entries >= 0
        except Exception:
            raise FormatError(f"{path}: malformed size line '{size.rstrip()}'")
        ri, ci, vv = [], [], []
        for k in range(entries):
            line = next(lines, None)
            if line is None:
                raise FormatError(f"{path}: expected {entries} entries, got {k}")
            t = line.split()
            try:
                i, j, v = int(t[0]), int(t[1]), float(t[2])
            except Exception:
                raise FormatError(f"{path}: malformed entry '{line.rstrip()}'")
            if i < 1 or i > n_rows or j < 1 or j > n_cols:
                raise FormatError(f"{path}: entry index ({i}, {j}) outside {n_rows}x{n_cols}")
            ri.append(i - 1); ci.append(j - 1); vv.append(v)
            if sym == "symmetric" and i != j:
                ri.append(j - 1); ci.append(i - 1); vv.append(v)
    ri, ci, vv = np.array(ri, dtype=np.int64), np.array(ci, dtype=np.int64), np.array(vv, dtype=np.float64)
    order = np.lexsort((np.arange(ri.shape[0]), ci, ri))  # stable by (row, col), file order inside duplicates
    ri, ci, vv = ri[order], ci[order], vv[order]
    keys = ri * max(n_cols, 1) + ci
    first = np.ones(keys.shape[0], dtype=bool)
    first[1:] = keys[1:] != keys[:-1]
    starts = np.flatnonzero(first)
    sums = np.empty(starts.shape[0])
    ends = np.append(starts[1:], keys.shape[0])
    for q, (a, b) in enumerate(zip(starts, ends)):  # sequential sums keep the reference's rounding
        s = 0.0
        for v in vv[a:b]:
            s += v
        sums[q] = s
    keep = sums != 0.0
    r, c, v = ri[starts][keep], ci[starts][keep], sums[keep]
    rowptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(rowptr, r + 1, 1)
    return np.cumsum(rowptr), c, v, n_cols


def mm_write_vector(path: str, v: np.ndarray) -> None:
    """mm_write_vector (mmio.hpp:149-160)."""
    with open(path, "w") as out:
        out.write("%%MatrixMarket matrix array real general\n")
        out.write(f"{v.shape[0]} 1\n")
        out.write("".join("%.17g\n" % x for x in v))


def mm_read_vector(path: str) -> np.ndarray:
    """mm_read_vector (mmio.hpp:123-147)."""
    try:
        f = open(path)
    except OSError:
        raise FormatError(f"{path}: cannot open file")
    with f:
        fmt, sym = _header(f, path)
        if fmt != "array":
            raise FormatError(f"{path}: expected array format for a vector, got '{fmt}'")
        if sym != "general":
            raise FormatError(f"{path}: unsupported symmetry '{sym}' for a vector")
        lines = _data_lines(f)
        size = next(lines, None)
        if size is None:
            raise FormatError(f"{path}: missing size line")
        t = size.split()
        try:
            rows, cols = int(t[0]), int(t[1])
            assert rows >= 0 and cols == 1
        except Exception:
            raise FormatError(f"{path}: a vector must have one column")
        out = np.empty(rows)
        for i in range(rows):
            line = next(lines, None)
            if line is None:
                raise FormatError(f"{path}: expected {rows} values, got {i}")
            try:
                out[i] = float(line.split()[0])
            except Exception:
                raise FormatError(f"{path}: malformed value '{line.rstrip()}'")
    return out


def write_config(prefix: str, cfg) -> dict:
    """Dump a configs.ConfigInput as the file set the reference ingests (G, rhs, partition)."""
    paths = {"G": prefix + "_G.mtx", "rhs": prefix + "_rhs.mtx", "partition": prefix + "_partition.txt"}
    mm_write(paths["G"], cfg.g_rowptr, cfg.g_cols, cfg.g_vals, cfg.n)
    mm_write_vector(paths["rhs"], cfg.rhs)
    if cfg.level0_partition is not None:
        with open(paths["partition"], "w") as out:
            out.write(f"{cfg.level0_partition.shape[0]} {int(cfg.level0_n_aggregates)}\n")
            out.write("".join("%d\n" % a for a in cfg.level0_partition))
    return paths
