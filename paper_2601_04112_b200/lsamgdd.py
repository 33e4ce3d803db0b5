"""Python host mirror of the reference's lsamgdd API over the B200 C ABI.

Same names, argument meaning and error classes as the reference header
library (``/root/reference/proj/include/lsamgdd``): ``LevelParams``
(hierarchy.hpp:19-30), ``setup`` (:106), ``vcycle`` (:205/:229), ``apply``
(smoother.hpp:65), ``pcg`` with the factored operator Gᵀ(G·)
(krylov.hpp:42-92, lsamgdd_cli.cpp:137-142), ``operator_complexity`` (:257),
and host mirrors of ``Hierarchy.levels[l].{A,G,P,topology,thresh}`` and
``summary``. All compute runs in ``liblsamgdd_b200.so`` on the GPU; there is
no CPU fallback — without the built library or a B200 every call raises.
"""
from __future__ import annotations

import ctypes as C
import weakref
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import abi

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblsamgdd_b200.so")
_lib: Optional[C.CDLL] = None
_ERRLEN = 1024


def library() -> C.CDLL:
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        lib = C.CDLL(_LIB_PATH)
        lib.lsamgdd_device_available.restype = C.c_int32
        lib.lsamgdd_abi_version.restype = C.c_int32
        _lib = lib
    return _lib


# ---- error classes (errors.hpp:11-69) ------------------------------------------------


class Error(RuntimeError):
    """Base of all lsamgdd errors; ``name()`` matches the reference."""

    def name(self) -> str:
        return type(self).__name__


class IndexError(Error):  # noqa: A001 - mirrors lsamgdd::IndexError
    pass


class DimError(Error):
    pass


class InputError(Error):
    pass


class FormatError(Error):
    pass


class SplittingError(Error):
    pass


class EigError(Error):
    pass


class SetupError(Error):
    pass


class IndefiniteError(Error):
    pass


class SizeError(Error):
    pass


class CudaError(Error):
    pass


_BY_STATUS = {1: Error, 2: IndexError, 3: DimError, 4: InputError, 5: FormatError, 6: SplittingError, 7: EigError,
              8: SetupError, 9: IndefiniteError, 10: SizeError, 64: CudaError, 65: CudaError}


def _check(status: int, err=None) -> None:
    if status != 0:
        msg = err.value.decode(errors="replace") if err is not None else ""
        raise _BY_STATUS.get(status, Error)(msg)


# ---- parameters -------------------------------------------------------------------------


@dataclass
class LevelParams:
    """LevelParams (hierarchy.hpp:19-30) plus the opt-in config extensions."""

    max_levels: int = 25
    coarse_size: int = 400
    aggregation_passes: int = 1
    kappa: float = 50.0
    must_keep: float = 5.0
    coarsening_ratios: Sequence[int] = (2, 3)
    pre_sweeps: int = 1
    post_sweeps: int = 1
    gevp_variant: int = 0  # 0 SchurReduced, 1 WeightedLhs
    keep_spectra: bool = False
    # extensions; defaults reproduce the reference
    level0_partition: Optional[np.ndarray] = None
    level0_n_aggregates: int = 0
    level0_overlap: int = 1
    thresh_override: float = 0.0
    level0_max_modes: int = 0
    device: int = 0
    probe_levels: int = 0  # > 0: build that many fine levels and stop (stage-wise parity / timing at full size)
    level_offset: int = 0  # > 0: the factor is that level of a hierarchy whose finer levels were built elsewhere

    def to_abi(self) -> tuple[abi.Params, Optional[np.ndarray]]:
        keep = None
        kw = dict(
            max_levels=self.max_levels, coarse_size=self.coarse_size, aggregation_passes=self.aggregation_passes,
            kappa=float(self.kappa), must_keep=float(self.must_keep), coarsening_ratios=list(self.coarsening_ratios),
            pre_sweeps=self.pre_sweeps, post_sweeps=self.post_sweeps, gevp_variant=self.gevp_variant,
            keep_spectra=1 if self.keep_spectra else 0, level0_overlap=self.level0_overlap,
            thresh_override=float(self.thresh_override), level0_max_modes=self.level0_max_modes, device=self.device,
            probe_levels=int(self.probe_levels), level_offset=int(self.level_offset),
        )
        if self.level0_partition is not None:
            keep = np.ascontiguousarray(self.level0_partition, dtype=np.int64)
            kw["level0_partition"] = keep.ctypes.data
            kw["level0_n_aggregates"] = int(self.level0_n_aggregates)
        return abi.default_params(**kw), keep


def params_for(cfg, **over) -> LevelParams:
    """LevelParams of a configs.ConfigInput (partition + config hooks)."""
    kw = dict(cfg.params)
    kw.update(over)
    if cfg.level0_partition is not None:
        kw.setdefault("level0_partition", cfg.level0_partition)
        kw.setdefault("level0_n_aggregates", cfg.level0_n_aggregates)
    return LevelParams(**kw)


# ---- CSR ----------------------------------------------------------------------------------


@dataclass
class SparseMatrix:
    """Host CSR mirror (sparse.hpp:28-72)."""

    n_rows: int
    n_cols: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_indices.shape[0])

    @classmethod
    def from_arrays(cls, rowptr, cols, vals, n_cols: int) -> "SparseMatrix":
        return cls(int(len(rowptr) - 1), int(n_cols), np.ascontiguousarray(rowptr, dtype=np.int64),
                   np.ascontiguousarray(cols, dtype=np.int64), np.ascontiguousarray(vals, dtype=np.float64))

    def to_abi(self) -> abi.Csr:
        return abi.csr_struct(self.row_offsets, self.col_indices, self.values, self.n_cols)

    def todense(self) -> np.ndarray:
        d = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_offsets))
        d[rows, self.col_indices] = self.values
        return d


class DeviceSparseMatrix:
    """Device-resident CSR written by the on-device generator
    (lsamgdd_generate_stencil_rows); owns the device arrays. Accepted by
    :func:`setup` and :func:`pcg` in place of a host :class:`SparseMatrix`."""

    def __init__(self, owner: C.c_void_p, csr: abi.Csr):
        self._owner = owner
        self._csr = csr
        self.n_rows, self.n_cols, self.nnz = int(csr.n_rows), int(csr.n_cols), int(csr.nnz)

    def to_abi(self) -> abi.Csr:
        if not self._owner:
            raise InputError("generated matrix was closed")
        return self._csr

    def to_host(self) -> SparseMatrix:
        off = np.empty(self.n_rows + 1, dtype=np.int64)
        col = np.empty(self.nnz, dtype=np.int64)
        val = np.empty(self.nnz, dtype=np.float64)
        err = C.create_string_buffer(_ERRLEN)
        _check(library().lsamgdd_generated_export(self._owner, abi.ptr(off), abi.ptr(col), abi.ptr(val), err,
                                                  C.c_size_t(_ERRLEN)), err)
        return SparseMatrix(self.n_rows, self.n_cols, off, col, val)

    def close(self) -> None:
        if self._owner:
            library().lsamgdd_generated_destroy(self._owner)
            self._owner = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def generate_stencil_rows(grid, offsets: np.ndarray, coefs: np.ndarray, device: int = 0) -> DeviceSparseMatrix:
    """lsamgdd_generate_stencil_rows: the constant-coefficient grid factor of
    BASELINE configs 2, 3, 5 written on the device (configs.config_stencil)."""
    g = (C.c_int64 * 3)(*[int(v) for v in grid])
    offsets = np.ascontiguousarray(offsets, dtype=np.int32)
    coefs = np.ascontiguousarray(coefs, dtype=np.float64)
    if offsets.ndim != 3 or offsets.shape[2] != 3 or coefs.shape != offsets.shape[:2]:
        raise DimError("generate_stencil_rows: offsets must be [rows][entries][3] and coefs [rows][entries]")
    owner = C.c_void_p()
    csr = abi.Csr()
    err = C.create_string_buffer(_ERRLEN)
    lib = library()
    _check(lib.lsamgdd_generate_stencil_rows(g, C.c_int32(coefs.shape[0]), C.c_int32(coefs.shape[1]), abi.ptr(offsets),
                                             abi.ptr(coefs), C.c_int32(device), C.byref(owner), C.byref(csr), err,
                                             C.c_size_t(_ERRLEN)), err)
    return DeviceSparseMatrix(owner, csr)


def _as_sparse(g):
    if isinstance(g, (SparseMatrix, DeviceSparseMatrix)):
        return g
    if hasattr(g, "g_rowptr"):
        return SparseMatrix.from_arrays(g.g_rowptr, g.g_cols, g.g_vals, g.n)
    if hasattr(g, "indptr"):  # scipy.sparse.csr_matrix
        return SparseMatrix.from_arrays(g.indptr, g.indices, g.data, g.shape[1])
    rowptr, cols, vals, ncols = g
    return SparseMatrix.from_arrays(rowptr, cols, vals, ncols)


# ---- hierarchy ----------------------------------------------------------------------------


@dataclass
class LevelSummary:
    level: int
    dim: int
    nnz: int
    n_aggregates: int
    k_c: int
    n_mult: int
    thresh: float
    modes_kept: int


@dataclass
class AggregateTopology:
    omega: list
    gamma: list
    colors: np.ndarray
    n_colors: int
    n_nodes: int
    multiplicity_max: int = 0

    def n_aggregates(self) -> int:
        return len(self.omega)

    def subdomain(self, i: int) -> np.ndarray:
        return np.concatenate([self.omega[i], self.gamma[i]])

    def pou_mask(self, i: int) -> np.ndarray:
        return np.concatenate([np.ones(len(self.omega[i]), np.uint8), np.zeros(len(self.gamma[i]), np.uint8)])


class Level:
    """Lazy host mirror of one device level (hierarchy.hpp:46-51)."""

    def __init__(self, h: "Hierarchy", index: int):
        # weak: a strong reference would close a cycle (hierarchy -> levels -> hierarchy) and keep the
        # device memory of a dropped hierarchy alive until the cycle collector happens to run
        self._href = weakref.ref(h)
        self.index = index
        self._cache: dict = {}

    @property
    def _h(self) -> "Hierarchy":
        h = self._href()
        if h is None:
            raise InputError("the hierarchy of this level was released")
        return h

    def _csr(self, what: int) -> SparseMatrix:
        if what not in self._cache:
            self._cache[what] = self._h._export_csr(self.index, what)
        return self._cache[what]

    @property
    def A(self) -> SparseMatrix:
        return self._csr(abi.EXPORT_A)

    @property
    def G(self) -> SparseMatrix:
        return self._csr(abi.EXPORT_G)

    @property
    def P(self) -> SparseMatrix:
        return self._csr(abi.EXPORT_P)

    @property
    def has_interpolation(self) -> bool:
        return self.index + 1 < self._h.num_levels

    @property
    def thresh(self) -> float:
        return self._h.summary[self.index].thresh if self.has_interpolation else 0.0

    @property
    def topology(self) -> AggregateTopology:
        if "topo" not in self._cache:
            part, nagg = self._h._export_vec(self.index, abi.EXPORT_PARTITION)
            g0, g1 = self._h._export_offsets(self.index, abi.EXPORT_GAMMA)
            colors, ncol = self._h._export_vec(self.index, abi.EXPORT_COLORS)
            order = np.argsort(part, kind="stable")
            bounds = np.searchsorted(part[order], np.arange(nagg + 1))
            omega = [order[bounds[i]:bounds[i + 1]] for i in range(nagg)]
            gamma = [g1[g0[i]:g0[i + 1]] for i in range(nagg)]
            self._cache["topo"] = AggregateTopology(omega, gamma, colors, ncol, len(part),
                                                    self._h.summary[self.index].n_mult)
        return self._cache["topo"]

    def spectra(self) -> list:
        off, vals = self._h._export_offsets(self.index, abi.EXPORT_SPECTRA, with_vals=True)
        return [vals[off[i]:off[i + 1]] for i in range(len(off) - 1)]

    def multiplicity(self) -> np.ndarray:
        return self._h._export_vec(self.index, abi.EXPORT_MULTIPLICITY)[0]


class Hierarchy:
    """Immutable device hierarchy; safe to share across concurrent solves."""

    def __init__(self, handle: C.c_void_p, g: SparseMatrix, params: LevelParams):
        self._handle = handle
        self._g = g
        self.params = params
        lib = library()
        n = C.c_int64()
        _check(lib.lsamgdd_num_levels(handle, C.byref(n)))
        self.num_levels = n.value
        self.levels = [Level(self, l) for l in range(self.num_levels)]
        self.summary = []
        for l in range(self.num_levels):
            s = abi.LevelSummary()
            _check(lib.lsamgdd_get_level_summary(handle, C.c_int64(l), C.byref(s)))
            self.summary.append(LevelSummary(*(getattr(s, f) for f, _ in abi.LevelSummary._fields_)))

    @property
    def handle(self) -> C.c_void_p:
        return self._handle

    def close(self) -> None:
        if self._handle:
            library().lsamgdd_destroy(self._handle)
            self._handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _sizes(self, level: int, what: int):
        sizes = (C.c_int64 * 3)()
        _check(library().lsamgdd_level_export(self._handle, C.c_int64(level), C.c_int32(what), sizes, None, None, None))
        return sizes[0], sizes[1], sizes[2]

    def _export_csr(self, level: int, what: int) -> SparseMatrix:
        r, c, nnz = self._sizes(level, what)
        off = np.empty(r + 1, np.int64)
        col = np.empty(nnz, np.int64)
        val = np.empty(nnz)
        sizes = (C.c_int64 * 3)()
        _check(library().lsamgdd_level_export(self._handle, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(off),
                                              abi.ptr(col), abi.ptr(val)))
        return SparseMatrix(r, c, off, col, val)

    def _export_vec(self, level: int, what: int):
        s0, s1, _ = self._sizes(level, what)
        out = np.empty(s0, np.int64)
        sizes = (C.c_int64 * 3)()
        _check(library().lsamgdd_level_export(self._handle, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(out),
                                              None, None))
        return out, s1

    def _export_offsets(self, level: int, what: int, with_vals: bool = False):
        s0, s1, _ = self._sizes(level, what)
        off = np.empty(s0 + 1, np.int64)
        idx = np.empty(s1, np.int64)
        vals = np.empty(s1)
        sizes = (C.c_int64 * 3)()
        _check(library().lsamgdd_level_export(self._handle, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(off),
                                              None if with_vals else abi.ptr(idx), abi.ptr(vals) if with_vals else None))
        return (off, vals) if with_vals else (off, idx)

    def timings(self) -> list[tuple[str, float]]:
        names = (C.c_char_p * 64)()
        ms = (C.c_double * 64)()
        cnt = C.c_int64()
        _check(library().lsamgdd_setup_timings(self._handle, names, ms, C.c_int64(64), C.byref(cnt)))
        return [(names[i].decode(), ms[i]) for i in range(min(cnt.value, 64))]


def setup(g0, params: Optional[LevelParams] = None) -> Hierarchy:
    """setup(g0, params) — hierarchy.hpp:106."""
    params = params or LevelParams()
    g = _as_sparse(g0)
    p, keep = params.to_abi()
    csr = g.to_abi()
    h = C.c_void_p()
    err = C.create_string_buffer(_ERRLEN)
    _check(library().lsamgdd_setup(C.byref(csr), C.byref(p), C.byref(h), err, C.c_size_t(_ERRLEN)), err)
    del keep
    return Hierarchy(h, g, params)


def _vec_call(fn, h: Hierarchy, args: list, x: np.ndarray, nout: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty(nout)
    err = C.create_string_buffer(_ERRLEN)
    _check(fn(h.handle, *args, abi.ptr(x), abi.ptr(out), C.c_int32(abi.HOST), err, C.c_size_t(_ERRLEN)), err)
    return out


def vcycle(h: Hierarchy, r: np.ndarray, level: int = 0) -> np.ndarray:
    """vcycle(h, level, r) — hierarchy.hpp:205/229."""
    if level < 0 or level >= h.num_levels:
        raise IndexError("vcycle: level out of range")
    n = h.summary[level].dim
    if len(r) != n:
        raise DimError("vcycle: residual length mismatch")
    return _vec_call(library().lsamgdd_vcycle, h, [C.c_int64(level)], r, n)


RAS, RAST, ASM = abi.RAS, abi.RAST, abi.ASM


def apply(h: Hierarchy, level: int, r: np.ndarray, mode: int = RAS) -> np.ndarray:
    """apply(smoother of level, r, mode) — smoother.hpp:65."""
    if level < 0 or level + 1 >= h.num_levels:
        raise IndexError("schwarz: level has no smoother")
    n = h.summary[level].dim
    if len(r) != n:
        raise DimError(f"schwarz apply: vector length {len(r)} does not match system size {n}")
    return _vec_call(library().lsamgdd_schwarz_apply, h, [C.c_int64(level), C.c_int32(mode)], r, n)


def level_spmv(h: Hierarchy, level: int, what: str, x: np.ndarray, transpose: bool = False) -> np.ndarray:
    """spmv / spmv_transpose (sparse.hpp:110,125) with A_l, G_l or P_l."""
    w = {"A": 0, "G": 1, "P": 2}[what]
    lev = h.levels[level]
    if w == 0:
        nout = lev.A.n_rows
    elif w == 1:
        nout = lev.G.n_cols if transpose else lev.G.n_rows
    else:
        nout = h.summary[level + 1].dim if transpose else h.summary[level].dim
    return _vec_call(library().lsamgdd_level_spmv, h, [C.c_int64(level), C.c_int32(w), C.c_int32(1 if transpose else 0)],
                     x, nout)


@dataclass
class SolveReport:
    """SolveReport (krylov.hpp:24-33)."""

    iterations: int = 0
    residual_history: np.ndarray = field(default_factory=lambda: np.zeros(0))
    converged: bool = False
    avg_conv_factor: float = 0.0
    iters_to_tenth: float = 0.0
    operator_complexity: float = 0.0
    setup_seconds: float = 0.0
    solve_seconds: float = 0.0


def pcg(h: Hierarchy, b: np.ndarray, tol: float = 1e-8, maxit: int = 1000, g0=None, stats: bool = False):
    """pcg(apply_a = Gᵀ(G·), apply_b = vcycle(h,·), b, tol, maxit) — krylov.hpp:42-92.

    ``g0`` defaults to the factor the hierarchy was built from. Returns
    ``(x, SolveReport)`` (plus kernel stats when ``stats``).
    """
    lib = library()
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty_like(b)
    hist = np.empty(int(maxit) + 2)
    rep = abi.Report()
    rep.residual_history = hist.ctypes.data
    rep.history_capacity = hist.shape[0]
    err = C.create_string_buffer(_ERRLEN)
    if stats:
        ks = abi.KernelStats()
        st = lib.lsamgdd_profile_pcg(h.handle, abi.ptr(b), C.c_double(tol), C.c_uint64(maxit), abi.ptr(x),
                                     C.c_int32(abi.HOST), C.byref(rep), C.byref(ks), err, C.c_size_t(_ERRLEN))
    else:
        gs = None
        if g0 is not None:
            gsp = _as_sparse(g0)
            gs = gsp.to_abi()
        st = lib.lsamgdd_pcg(h.handle, C.byref(gs) if gs is not None else None, abi.ptr(b), C.c_double(tol),
                             C.c_uint64(maxit), abi.ptr(x), C.c_int32(abi.HOST), C.byref(rep), err, C.c_size_t(_ERRLEN))
    _check(st, err)
    report = SolveReport(rep.iterations, hist[: rep.history_len].copy(), bool(rep.converged), rep.avg_conv_factor,
                         rep.iters_to_tenth, rep.operator_complexity, rep.setup_seconds, rep.solve_seconds)
    if stats:
        return x, report, {f: getattr(ks, f) for f, _ in abi.KernelStats._fields_}
    return x, report


def operator_complexity(h: Hierarchy) -> float:
    """operator_complexity(h) — hierarchy.hpp:257."""
    v = C.c_double()
    _check(library().lsamgdd_operator_complexity(h.handle, C.byref(v)))
    return v.value


def device_available() -> bool:
    return bool(library().lsamgdd_device_available())
