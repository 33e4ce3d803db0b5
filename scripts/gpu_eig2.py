import os, sys, time, ctypes as C, numpy as np, subprocess
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import abi, lsamgdd
from oracle import refbind
orc = refbind.oracle()
lib = lsamgdd.library()
for n in [64, 150, 400, 700, 1300]:
    rng = np.random.default_rng(n)
    a = rng.uniform(-1,1,(n,n)); a[np.abs(a)<0.3]=0; a = a@a.T
    t=time.time(); vals, vecs = orc.sym_eig(a); to=time.time()-t
    gv, gV = np.empty(n), np.empty((n,n)); err = C.create_string_buffer(512)
    t=time.time(); st = lib.lsamgdd_dense_sym_eig(C.c_int64(n), abi.ptr(a), abi.ptr(gv), abi.ptr(gV), C.c_int32(2), err, C.c_size_t(512)); tg=time.time()-t
    print(n, os.environ.get("LSB_EIG_SPLIT","1"), "st", st, "exact", np.array_equal(gv, vals), np.array_equal(gV, vecs), "cpu %.3fs gpu %.3fs" % (to, tg), flush=True)
