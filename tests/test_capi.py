"""The C-ABI library (no GPU needed): it loads, exports every entry point
include/lsamgdd_b200.h declares, validates setup inputs with the reference's
error classes on the host, and refuses to compute without a B200 (no CPU
fallback)."""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2601_04112_b200 import abi, configs, lsamgdd

from . import _cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols() -> list[str]:
    text = open(os.path.join(ROOT, "include", "lsamgdd_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lsamgdd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = lsamgdd.library()
    names = _declared_symbols()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert lib.lsamgdd_abi_version() == 1


def test_library_is_sm100a_only():
    so = open(lsamgdd._LIB_PATH, "rb").read()
    assert b"sm_100a" in so or b"sm_100" in so


def test_params_default_matches_levelparams():
    lib = lsamgdd.library()
    p = abi.Params()
    lib.lsamgdd_params_default(C.byref(p))
    q = abi.default_params()
    for f, _ in abi.Params._fields_:
        if f in ("coarsening_ratios", "reserved"):
            assert list(getattr(p, f)) == list(getattr(q, f))
        else:
            assert getattr(p, f) == getattr(q, f), f


@pytest.mark.parametrize("kw,name", [
    (dict(max_levels=1), "InputError"),
    (dict(coarse_size=0), "InputError"),
    (dict(kappa=1.0), "InputError"),
    (dict(must_keep=1.0), "InputError"),
    (dict(coarsening_ratios=(1,)), "InputError"),
    (dict(aggregation_passes=0), "InputError"),
])
def test_setup_validation_errors(kw, name):
    g = _cases.chain_factor(12, shift=0.5)
    with pytest.raises(lsamgdd.Error) as e:
        lsamgdd.setup(g, lsamgdd.LevelParams(**kw))
    assert e.value.name() == name


def test_empty_factor_is_input_error():
    g = (np.zeros(1, np.int64), np.zeros(0, np.int64), np.zeros(0), 5)
    with pytest.raises(lsamgdd.InputError):
        lsamgdd.setup(g)


def test_no_cpu_fallback_without_device():
    if lsamgdd.device_available():
        pytest.skip("a B200 is visible")
    cfg = configs.config("c1", 16)
    with pytest.raises(lsamgdd.CudaError):
        lsamgdd.setup(cfg, lsamgdd.params_for(cfg))


def test_uniform_entry_point_matches_generator():
    lib = lsamgdd.library()
    out = np.empty(1000)
    lib.lsamgdd_uniform(C.c_uint64(3), C.c_double(-1.0), C.c_double(1.0), C.c_int64(1000), abi.ptr(out))
    assert np.array_equal(out, configs.mt19937_64_uniform(3, 1000))
