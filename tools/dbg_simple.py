import ctypes as C, sys
sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200 import _native as N
from paper_1410_4054_b200.device import context_for
for side in (1024, 2048):
    ctx = pk.ExecutionContext(128, 256, device=0)
    dm, _ = pk.convdiff2d(side, device=True, context=ctx)
    dc = context_for(ctx)
    lib = N.lib()
    f = lib.pk_debug_bench
    f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
    for kind in (2, 3, 8):
        us = C.c_double()
        N.check(f(dc.handle, dm.handle, kind, 20, C.byref(us)))
        n, nnz = dm.n_rows, dm.nnz
        b = 12 * nnz + 4 * (n + 1) + (16 * n if kind == 0 else 32 * n)
        print(side, kind, round(us.value, 2), "us", round(b / us.value / 1e3), "GB/s")
