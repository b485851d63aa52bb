import sys, time, statistics
sys.path.insert(0, ".")
import torch
import paper_1410_4054_b200 as pk
ctx = pk.ExecutionContext(128, 256, device=0)
a, b = pk.convdiff2d(1024)
for it in (1, 8, 200):
    cfg = pk.SolverConfig(fixed_iterations=it, max_iterations=it)
    pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
    ws = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
        ws.append(time.perf_counter() - t0)
    print(it, "wall_ms", round(statistics.median(ws) * 1e3, 3), "loop_ms", round(r.loop_seconds * 1e3, 3))
cfg = pk.SolverConfig(fixed_iterations=200, max_iterations=200, loop_mode="host")
pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
torch.cuda.synchronize(); t0 = time.perf_counter(); r = pk.bicgstab_pipelined(a, b, config=cfg, context=ctx)
print("host200 wall_ms", round((time.perf_counter() - t0) * 1e3, 3), "loop_ms", round(r.loop_seconds * 1e3, 3))
