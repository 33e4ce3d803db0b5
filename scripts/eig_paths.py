"""Times dense eigensolves on chosen device paths: eig_paths.py n path [path...]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2601_04112_b200 import abi, lsamgdd

lib = lsamgdd.library()
n = int(sys.argv[1])
rng = np.random.default_rng(n)
a = rng.uniform(-1, 1, (n, n))
a[np.abs(a) < 0.3] = 0.0
a = a @ a.T
for path in [int(x) for x in sys.argv[2:]]:
    gv, gV = np.empty(n), np.empty((n, n))
    err = C.create_string_buffer(512)
    for rep in range(2):
        t0 = time.perf_counter()
        st = lib.lsamgdd_dense_sym_eig(C.c_int64(n), abi.ptr(np.ascontiguousarray(a)), abi.ptr(gv), abi.ptr(gV), C.c_int32(path), err, C.c_size_t(512))
        dt = time.perf_counter() - t0
    print(f"n={n} path={path} status={st} {dt * 1e3:.2f} ms", flush=True)
