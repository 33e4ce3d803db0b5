"""One device eigensolve (for ncu): python scripts/eig_one.py N PATH."""
import sys, time, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import abi, lsamgdd
n, path = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(n)
a = rng.uniform(-1, 1, (n, n)); a[np.abs(a) < 0.3] = 0; a = a @ a.T
gv, gV = np.empty(n), np.empty((n, n)); err = C.create_string_buffer(512)
t = time.time()
st = lsamgdd.library().lsamgdd_dense_sym_eig(C.c_int64(n), abi.ptr(a), abi.ptr(gv), abi.ptr(gV), C.c_int32(path), err, C.c_size_t(512))
print("n", n, "path", path, "status", st, "time %.3f s" % (time.time() - t))
if len(sys.argv) > 3:
    from oracle import refbind
    vals, vecs = refbind.oracle().sym_eig(a)
    print("exact", np.array_equal(gv, vals), np.array_equal(gV, vecs))
