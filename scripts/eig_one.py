"""One dense eigensolve on one device path (for ncu): eig_one.py n path"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2601_04112_b200 import abi, lsamgdd

n, path = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(n)
a = rng.uniform(-1, 1, (n, n))
a[np.abs(a) < 0.3] = 0.0
a = a @ a.T
gv, gV = np.empty(n), np.empty((n, n))
err = C.create_string_buffer(512)
st = lsamgdd.library().lsamgdd_dense_sym_eig(C.c_int64(n), abi.ptr(np.ascontiguousarray(a)), abi.ptr(gv), abi.ptr(gV),
                                             C.c_int32(path), err, C.c_size_t(512))
print("status", st, err.value)
