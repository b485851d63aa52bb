"""Probe: is "plain SpMV sweep + separate ordered fold over materialised
contributions" cheaper than the fused engine kernel?  C2 matrix (n = 1M),
128x256 geometry.  Each kernel is timed alone with CUDA events, with an L2
flush (256 MB write) before every rep so the numbers look like in-loop ones."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk  # noqa: E402
from paper_1410_4054_b200 import fused  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = pk.ExecutionContext(128, 256, device=0)
dm, _ = pk.convdiff2d(side, device=True, context=ctx)
n = dm.n_rows
g = torch.Generator(device="cuda").manual_seed(1)
V = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(8)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def t(fn, reps=20, do_flush=True):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        if do_flush:
            flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return round(tot / reps * 1e3, 2)


bc = 12 * dm.nnz + 4 * (n + 1)
res = {"n": n}
for fl in (True, False):
    k = "flush" if fl else "warm"
    r = {}
    r["spmv_plain"] = t(lambda: fused.spmv(dm, V[0], ctx), do_flush=fl)
    r["spmv_fused4"] = t(lambda: fused.spmv_fused(dm, V[0], ("input", "result", V[1], V[2]), ctx), do_flush=fl)
    r["spmv_fused2"] = t(lambda: fused.spmv_fused(dm, V[0], ("input", "result"), ctx), do_flush=fl)
    r["stage1_4col"] = t(lambda: fused.reduce_stage1([V[3], V[4], V[5], V[6]], ctx), do_flush=fl)
    r["stage1_2col"] = t(lambda: fused.reduce_stage1([V[3], V[4]], ctx), do_flush=fl)
    r["stage1_1col"] = t(lambda: fused.reduce_stage1([V[3]], ctx), do_flush=fl)
    r["dot"] = t(lambda: fused.dot(V[3], V[4], ctx), do_flush=fl)
    r["torch_copy"] = t(lambda: V[6].copy_(V[7]), do_flush=fl)
    res[k] = r
print(json.dumps(res))
