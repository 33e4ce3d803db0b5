"""ctypes mirror of include/lsamgdd_b200.h (the C ABI structs and codes).

Shared by the product wrapper (``paper_2601_04112_b200.lsamgdd``) and the
test-side bindings of the oracle libraries; it holds only type layouts.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

OK = 0
STATUS_NAMES = {
    1: "Error",
    2: "IndexError",
    3: "DimError",
    4: "InputError",
    5: "FormatError",
    6: "SplittingError",
    7: "EigError",
    8: "SetupError",
    9: "IndefiniteError",
    10: "SizeError",
    64: "CudaError",
    65: "OutOfMemoryError",
}

HOST, DEVICE = 0, 1
RAS, RAST, ASM = 0, 1, 2
EXPORT_A, EXPORT_G, EXPORT_P, EXPORT_PARTITION, EXPORT_GAMMA, EXPORT_COLORS, EXPORT_SPECTRA, EXPORT_MULTIPLICITY = range(8)


class Csr(C.Structure):
    _fields_ = [
        ("n_rows", C.c_int64),
        ("n_cols", C.c_int64),
        ("nnz", C.c_int64),
        ("row_offsets", C.c_void_p),
        ("col_indices", C.c_void_p),
        ("values", C.c_void_p),
        ("memory", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Params(C.Structure):
    _fields_ = [
        ("max_levels", C.c_uint64),
        ("coarse_size", C.c_uint64),
        ("aggregation_passes", C.c_uint64),
        ("kappa", C.c_double),
        ("must_keep", C.c_double),
        ("n_ratios", C.c_uint64),
        ("coarsening_ratios", C.c_uint64 * 8),
        ("pre_sweeps", C.c_uint64),
        ("post_sweeps", C.c_uint64),
        ("gevp_variant", C.c_int32),
        ("keep_spectra", C.c_int32),
        ("level0_partition", C.c_void_p),
        ("level0_n_aggregates", C.c_int64),
        ("level0_overlap", C.c_int32),
        ("device", C.c_int32),
        ("thresh_override", C.c_double),
        ("level0_max_modes", C.c_uint64),
        ("probe_levels", C.c_uint64),
        ("level_offset", C.c_uint64),
        ("reserved", C.c_uint64 * 2),
    ]


class LevelSummary(C.Structure):
    _fields_ = [
        ("level", C.c_uint64),
        ("dim", C.c_uint64),
        ("nnz", C.c_uint64),
        ("n_aggregates", C.c_uint64),
        ("k_c", C.c_uint64),
        ("n_mult", C.c_uint64),
        ("thresh", C.c_double),
        ("modes_kept", C.c_uint64),
    ]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_uint64),
        ("converged", C.c_int32),
        ("reserved", C.c_int32),
        ("avg_conv_factor", C.c_double),
        ("iters_to_tenth", C.c_double),
        ("operator_complexity", C.c_double),
        ("setup_seconds", C.c_double),
        ("solve_seconds", C.c_double),
        ("residual_history", C.c_void_p),
        ("history_capacity", C.c_uint64),
        ("history_len", C.c_uint64),
    ]


class KernelStats(C.Structure):
    _fields_ = [
        ("schwarz_ms", C.c_double),
        ("schwarz_bytes", C.c_double),
        ("schwarz_launches", C.c_int64),
        ("spmv_ms", C.c_double),
        ("spmv_bytes", C.c_double),
        ("spmv_launches", C.c_int64),
        ("total_launches", C.c_int64),
    ]


def default_params(**over) -> Params:
    """LevelParams defaults (hierarchy.hpp:19-30) plus extension overrides."""
    p = Params()
    p.max_levels = 25
    p.coarse_size = 400
    p.aggregation_passes = 1
    p.kappa = 50.0
    p.must_keep = 5.0
    p.n_ratios = 2
    p.coarsening_ratios[0] = 2
    p.coarsening_ratios[1] = 3
    p.pre_sweeps = 1
    p.post_sweeps = 1
    p.gevp_variant = 0
    p.keep_spectra = 0
    p.level0_partition = None
    p.level0_n_aggregates = 0
    p.level0_overlap = 1
    p.device = 0
    p.thresh_override = 0.0
    p.level0_max_modes = 0
    p.probe_levels = 0
    p.level_offset = 0
    for k, v in over.items():
        if k == "coarsening_ratios":
            p.n_ratios = len(v)
            for i, r in enumerate(v):
                p.coarsening_ratios[i] = int(r)
        else:
            setattr(p, k, v)
    return p


def ptr(a: np.ndarray | None) -> C.c_void_p | None:
    if a is None:
        return None
    return C.c_void_p(a.ctypes.data)


def csr_struct(rowptr: np.ndarray, cols: np.ndarray, vals: np.ndarray, n_cols: int) -> Csr:
    g = Csr()
    g.n_rows = rowptr.shape[0] - 1
    g.n_cols = n_cols
    g.nnz = cols.shape[0]
    g.row_offsets = rowptr.ctypes.data
    g.col_indices = cols.ctypes.data
    g.values = vals.ctypes.data
    g.memory = HOST
    return g


class LsamgddError(RuntimeError):
    """Raised for a non-zero status; ``name`` is the reference class name."""

    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.name}: {msg}")


def check(status: int, err: C.Array | None = None) -> None:
    if status != OK:
        msg = err.value.decode(errors="replace") if err is not None else ""
        raise LsamgddError(status, msg)
