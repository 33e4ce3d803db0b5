"""ctypes bindings of the two CPU checkers — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline/reference arm. Two libraries share one Python surface:

* ``oracle/_ref/libref_lsamgdd.so`` — the unmodified reference headers behind
  ``ref_harness.cpp`` (built here by ``oracle/Makefile``; the .so travels).
* ``oracle/liboracle_lsamgdd.so`` — the plain-C restatement
  ``lsamgdd_oracle.c``, pinned against the former and the reference's
  golden vectors.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2601_04112_b200 import abi

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libref_lsamgdd.so")
ORACLE_LIB = os.path.join(HERE, "liboracle_lsamgdd.so")

_ERRLEN = 512


class CpuChecker:
    """One of the CPU implementations behind a uniform surface."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
        self.lib = C.CDLL(path)
        self.prefix = prefix
        self.path = path

    def fn(self, name: str):
        return getattr(self.lib, f"{self.prefix}_{name}")

    # --- hierarchy ---
    def setup(self, cfg_or_csr, params: abi.Params, plain: bool = False):
        return CpuHierarchy(self, cfg_or_csr, params, plain)

    # --- unit-level ---
    def sym_eig(self, a: np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        n = a.shape[0]
        vals = np.empty(n)
        vecs = np.empty((n, n))
        err = C.create_string_buffer(_ERRLEN)
        st = self.fn("sym_eig")(C.c_int64(n), abi.ptr(a), abi.ptr(vals), abi.ptr(vecs), err, C.c_size_t(_ERRLEN))
        abi.check(st, err)
        return vals, vecs

    def spsd_gevp(self, l: np.ndarray, b: np.ndarray, tau: float = 1e-10):
        l = np.ascontiguousarray(l, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        n = l.shape[0]
        vals = np.empty(n)
        vecs = np.empty(n * n)
        k = C.c_int64()
        disc = C.c_int64()
        err = C.create_string_buffer(_ERRLEN)
        st = self.fn("spsd_gevp")(C.c_int64(n), abi.ptr(l), abi.ptr(b), C.c_double(tau), abi.ptr(vals),
                                  abi.ptr(vecs), C.byref(k), C.byref(disc), err, C.c_size_t(_ERRLEN))
        abi.check(st, err)
        kk = k.value
        return vals[:kk].copy(), vecs[: n * kk].reshape(n, kk).copy(), disc.value

    def pseudo_inverse(self, a: np.ndarray, tau: float = 1e-10):
        a = np.ascontiguousarray(a, dtype=np.float64)
        n = a.shape[0]
        out = np.empty((n, n))
        err = C.create_string_buffer(_ERRLEN)
        st = self.fn("pseudo_inverse")(C.c_int64(n), abi.ptr(a), C.c_double(tau), abi.ptr(out), err, C.c_size_t(_ERRLEN))
        abi.check(st, err)
        return out

    def standard_aggregation(self, rowptr, cols, vals):
        n = rowptr.shape[0] - 1
        g = abi.csr_struct(rowptr, cols, vals, n)
        out = np.empty(n, dtype=np.int64)
        nagg = C.c_int64()
        err = C.create_string_buffer(_ERRLEN)
        st = self.fn("standard_aggregation")(C.byref(g), abi.ptr(out), C.byref(nagg), err, C.c_size_t(_ERRLEN))
        abi.check(st, err)
        return out, nagg.value

    def eigen_threshold(self, kappa: float, kc: int, n_mult: int) -> float:
        out = C.c_double()
        err = C.create_string_buffer(_ERRLEN)
        st = self.fn("eigen_threshold")(C.c_double(kappa), C.c_int64(kc), C.c_int64(n_mult), C.byref(out), err,
                                        C.c_size_t(_ERRLEN))
        abi.check(st, err)
        return out.value

    def uniform(self, seed: int, n: int, lo: float = -1.0, hi: float = 1.0):
        out = np.empty(n)
        self.fn("uniform")(C.c_uint64(seed), C.c_double(lo), C.c_double(hi), C.c_int64(n), abi.ptr(out))
        return out


class CpuHierarchy:
    def __init__(self, chk: CpuChecker, cfg_or_csr, params: abi.Params, plain: bool):
        self.chk = chk
        if isinstance(cfg_or_csr, tuple):
            rowptr, cols, vals, ncols = cfg_or_csr
        else:
            rowptr, cols, vals, ncols = cfg_or_csr.g_rowptr, cfg_or_csr.g_cols, cfg_or_csr.g_vals, cfg_or_csr.n
        self._keep = (rowptr, cols, vals)
        self.g = abi.csr_struct(rowptr, cols, vals, ncols)
        self.n = ncols
        self.params = params
        self.h = C.c_void_p()
        err = C.create_string_buffer(_ERRLEN)
        st = chk.fn("setup")(C.byref(self.g), C.byref(params), C.c_int32(1 if plain else 0), C.byref(self.h), err,
                             C.c_size_t(_ERRLEN))
        abi.check(st, err)

    def __del__(self):
        if getattr(self, "h", None) and self.h.value:
            self.chk.fn("destroy")(self.h)
            self.h = None

    @property
    def num_levels(self) -> int:
        v = C.c_int64()
        self.chk.fn("num_levels")(self.h, C.byref(v))
        return v.value

    def summary(self, level: int) -> dict:
        s = abi.LevelSummary()
        abi.check(self.chk.fn("level_summary")(self.h, C.c_int64(level), C.byref(s)))
        return {f: getattr(s, f) for f, _ in abi.LevelSummary._fields_}

    def operator_complexity(self) -> float:
        v = C.c_double()
        self.chk.fn("operator_complexity")(self.h, C.byref(v))
        return v.value

    def export(self, level: int, what: int):
        sizes = (C.c_int64 * 3)()
        abi.check(self.chk.fn("level_export")(self.h, C.c_int64(level), C.c_int32(what), sizes, None, None, None))
        s0, s1, s2 = sizes[0], sizes[1], sizes[2]
        if what in (abi.EXPORT_A, abi.EXPORT_G, abi.EXPORT_P):
            i0 = np.empty(s0 + 1, dtype=np.int64)
            i1 = np.empty(s2, dtype=np.int64)
            v = np.empty(s2)
            abi.check(self.chk.fn("level_export")(self.h, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(i0),
                                                  abi.ptr(i1), abi.ptr(v)))
            return i0, i1, v, (s0, s1)
        if what in (abi.EXPORT_PARTITION, abi.EXPORT_COLORS, abi.EXPORT_MULTIPLICITY):
            i0 = np.empty(s0, dtype=np.int64)
            abi.check(self.chk.fn("level_export")(self.h, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(i0), None,
                                                  None))
            return i0, s1
        if what == abi.EXPORT_GAMMA:
            i0 = np.empty(s0 + 1, dtype=np.int64)
            i1 = np.empty(s1, dtype=np.int64)
            abi.check(self.chk.fn("level_export")(self.h, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(i0),
                                                  abi.ptr(i1), None))
            return i0, i1
        if what == abi.EXPORT_SPECTRA:
            i0 = np.empty(s0 + 1, dtype=np.int64)
            v = np.empty(s1)
            abi.check(self.chk.fn("level_export")(self.h, C.c_int64(level), C.c_int32(what), sizes, abi.ptr(i0), None,
                                                  abi.ptr(v)))
            return i0, v
        raise ValueError(what)

    def _vec_call(self, name, *args, nout):
        out = np.empty(nout)
        err = C.create_string_buffer(_ERRLEN)
        st = self.chk.fn(name)(self.h, *args, abi.ptr(out), err, C.c_size_t(_ERRLEN))
        abi.check(st, err)
        return out

    def level_dim(self, level: int) -> int:
        return self.export(level, abi.EXPORT_A)[3][0]

    def vcycle(self, r: np.ndarray, level: int = 0) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        return self._vec_call("vcycle", C.c_int64(level), abi.ptr(r), nout=r.shape[0])

    def schwarz_apply(self, r: np.ndarray, level: int, mode: int) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        return self._vec_call("schwarz_apply", C.c_int64(level), C.c_int32(mode), abi.ptr(r), nout=r.shape[0])

    def spmv(self, x: np.ndarray, level: int, what: int, transpose: bool, nout: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self._vec_call("level_spmv", C.c_int64(level), C.c_int32(what), C.c_int32(1 if transpose else 0),
                              abi.ptr(x), nout=nout)

    def pcg(self, b: np.ndarray, tol: float = 1e-8, maxit: int = 1000):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(self.n)
        hist = np.empty(maxit + 2)
        rep = abi.Report()
        rep.residual_history = hist.ctypes.data
        rep.history_capacity = hist.shape[0]
        err = C.create_string_buffer(_ERRLEN)
        st = self.chk.fn("pcg")(self.h, None, abi.ptr(b), C.c_double(tol), C.c_uint64(maxit), abi.ptr(x), C.byref(rep),
                                err, C.c_size_t(_ERRLEN))
        abi.check(st, err)
        return x, {
            "iterations": rep.iterations,
            "converged": bool(rep.converged),
            "avg_conv_factor": rep.avg_conv_factor,
            "iters_to_tenth": rep.iters_to_tenth,
            "operator_complexity": rep.operator_complexity,
            "solve_seconds": rep.solve_seconds,
            "residual_history": hist[: rep.history_len].copy(),
        }

    def timings(self) -> list[tuple[str, float]]:
        names = (C.c_char_p * 64)()
        secs = (C.c_double * 64)()
        cnt = C.c_int64()
        self.chk.fn("setup_timings")(self.h, names, secs, C.c_int64(64), C.byref(cnt))
        return [(names[i].decode(), secs[i]) for i in range(min(cnt.value, 64))]


def reference() -> CpuChecker:
    return CpuChecker(REF_LIB, "ref")


def oracle() -> CpuChecker:
    return CpuChecker(ORACLE_LIB, "oracle")


def params_for(cfg, **over) -> abi.Params:
    kw = dict(cfg.params)
    kw.update(over)
    if cfg.level0_partition is not None:
        kw["level0_partition"] = cfg.level0_partition.ctypes.data
        kw["level0_n_aggregates"] = cfg.level0_n_aggregates
    return abi.default_params(**kw)
