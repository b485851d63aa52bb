"""Where the public call's host time goes (C2, 20 iterations, pinned b):
cProfile of 10 calls, plus the native pk_solve share."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_1410_4054_b200 as pk  # noqa: E402
from paper_1410_4054_b200 import _native as N  # noqa: E402

ctx = pk.ExecutionContext(128, 256, device=0)
a, b0 = pk.convdiff2d(1024)
b = pk.host_array(a.n_rows)
b[:] = b0
cfg = pk.SolverConfig(fixed_iterations=20, max_iterations=20)
for _ in range(3):
    pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
lib = N.lib()
orig = lib.pk_solve
acc = [0.0]


def timed(*args):
    t0 = time.perf_counter()
    r = orig(*args)
    acc[0] += time.perf_counter() - t0
    return r


lib.pk_solve = timed
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    r = pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
pr.disable()
wall = (time.perf_counter() - t0) / 10
print(f"call {wall * 1e3:.3f} ms; native pk_solve {acc[0] / 10 * 1e3:.3f} ms; loop {r.loop_seconds * 1e3:.3f} ms")
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
