"""Time the device Jacobi eigensolver (test hook) at several sizes, with the
per-phase cycle counters (LSB_EIG_PROF) and a bit-exact check vs the oracle."""
import os, sys, time, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import abi, lsamgdd
from oracle import refbind
orc = refbind.oracle()
lib = lsamgdd.library()
sizes = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [100, 240, 400, 550]
check = os.environ.get("CHECK", "1") == "1"
for n in sizes:
    rng = np.random.default_rng(n)
    a = rng.uniform(-1, 1, (n, n)); a[np.abs(a) < 0.3] = 0; a = a @ a.T
    gv, gV = np.empty(n), np.empty((n, n)); err = C.create_string_buffer(512)
    t = time.time(); st = lib.lsamgdd_dense_sym_eig(C.c_int64(n), abi.ptr(a), abi.ptr(gv), abi.ptr(gV), C.c_int32(2), err, C.c_size_t(512)); tg = time.time() - t
    msg = ""
    if check:
        t = time.time(); vals, vecs = orc.sym_eig(a); to = time.time() - t
        msg = "exact %s %s cpu %.3fs" % (np.array_equal(gv, vals), np.array_equal(gV, vecs), to)
    print(n, "st", st, "gpu %.3fs" % tg, msg, flush=True)
