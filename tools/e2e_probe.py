"""Where the e2e call's fixed cost goes (C2 system, public API, pinned b)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1410_4054_b200 as pk  # noqa: E402

ctx = pk.ExecutionContext(128, 256, device=0)
a, b0 = pk.convdiff2d(1024)
b = pk.host_array(a.n_rows)
b[:] = b0


def med(f, reps=7):
    ws = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ws.append(time.perf_counter() - t0)
    return statistics.median(ws) * 1e3


for it in (1, 20, 200):
    cfg = pk.SolverConfig(fixed_iterations=it, max_iterations=it)
    pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
    r = pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
    print(f"iters {it}: call {med(lambda: pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)):.3f} ms, "
          f"loop {r.loop_seconds * 1e3:.3f} ms")
hb = torch.from_numpy(b)
db = torch.empty(a.n_rows, dtype=torch.float64, device="cuda")
hx = torch.empty(a.n_rows, dtype=torch.float64, pin_memory=True)
print(f"H2D 8 MB pinned {med(lambda: db.copy_(hb, non_blocking=True)):.3f} ms; "
      f"D2H 8 MB pinned {med(lambda: hx.copy_(db, non_blocking=True)):.3f} ms")
pg = torch.from_numpy(np.array(b0))
print(f"H2D 8 MB pageable {med(lambda: db.copy_(pg)):.3f} ms")
