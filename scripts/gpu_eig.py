import sys, time, ctypes as C, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2601_04112_b200 import abi, lsamgdd
from oracle import refbind
orc = refbind.oracle()
lib = lsamgdd.library()
for n, path in [(7,0),(30,0),(30,1),(64,1),(64,2),(150,2),(333,2),(400,2),(700,2),(1300,2)]:
    rng = np.random.default_rng(n)
    a = rng.uniform(-1,1,(n,n)); a[np.abs(a)<0.3]=0; a = a@a.T
    t=time.time(); vals, vecs = orc.sym_eig(a); to=time.time()-t
    gv, gV = np.empty(n), np.empty((n,n)); err = C.create_string_buffer(512)
    t=time.time(); st = lib.lsamgdd_dense_sym_eig(C.c_int64(n), abi.ptr(a), abi.ptr(gv), abi.ptr(gV), C.c_int32(path), err, C.c_size_t(512)); tg=time.time()-t
    print(n, path, "st", st, err.value, "vals exact", np.array_equal(gv, vals), "vecs exact", np.array_equal(gV, vecs), "maxdiff %.2e" % np.abs(gv-vals).max(), "cpu %.3fs gpu %.3fs" % (to, tg), flush=True)
