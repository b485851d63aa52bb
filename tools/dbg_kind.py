"""Run one pk_debug_bench kind once (ncu target)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200 import _native as N
from paper_1410_4054_b200.device import context_for
kind = int(sys.argv[1]); side = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
ctx = pk.ExecutionContext(128, 256, device=0)
dm, _ = pk.convdiff2d(side, device=True, context=ctx)
f = N.lib().pk_debug_bench
f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
us = C.c_double()
N.check(f(context_for(ctx).handle, dm.handle, kind, 2, C.byref(us)))
print(kind, us.value)
