"""Engine micro-benchmark: CUDA-event time of single kernel-level launches on
the C2 matrix (n = 1M) for several PK_ENGINE_FLAGS (fresh process each)."""
import os
import subprocess
import sys

CHILD = r'''
import sys, torch, json
sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200 import fused
side = int(sys.argv[1]); geom = tuple(int(v) for v in sys.argv[2].split("x"))
ctx = pk.ExecutionContext(*geom, device=0)
dm, _ = pk.convdiff2d(side, device=True, context=ctx)
n = dm.n_rows
g = torch.Generator(device="cuda").manual_seed(1)
V = [torch.rand(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(8)]
def t(fn, reps=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3
bc = 12 * dm.nnz + 4 * (n + 1)
res = {}
us = t(lambda: fused.spmv_fused(dm, V[0], ("input", "result", V[1]), ctx)); res["spmv3"] = (round(us, 2), round((bc + 32 * n) / us / 1e3))
us = t(lambda: fused.spmv_fused(dm, V[0], ("result",), ctx)); res["spmv1"] = (round(us, 2), round((bc + 16 * n) / us / 1e3))
us = t(lambda: fused.fused_cg_vector_update(V[2], V[3], V[4], V[5], 0.5, 0.25, ctx)); res["cgupd"] = (round(us, 2), round(56 * n / us / 1e3))
us = t(lambda: fused.dot(V[0], V[1], ctx)); res["dot"] = (round(us, 2), round(16 * n / us / 1e3))
us = t(lambda: V[6].copy_(V[7])); res["torch_copy"] = (round(us, 2), round(16 * n / us / 1e3))
print(json.dumps(res))
'''

if __name__ == "__main__":
    for spec in sys.argv[1:] or ["1024:128x256:0"]:
        side, geom, flags = spec.split(":")
        env = dict(os.environ, PK_ENGINE_FLAGS=flags)
        out = subprocess.run([sys.executable, "-c", CHILD, side, geom], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr.strip()[-600:]
        print(f"{spec} {line}", flush=True)
