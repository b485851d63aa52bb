"""Debug helper: per-op kernel parity report at several geometries."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200 import fused
from oracle import pk_oracle as orc

rng = np.random.default_rng(5)
a, _ = pk.convdiff2d(40)
n = a.n_rows
V = {k: rng.standard_normal(n) for k in "p w x r ap s as r0 v b0 b1 b2 b3".split()}
dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
h = lambda t: t.cpu().numpy()

def rep(name, d, o):
    d, o = np.asarray(d), np.asarray(o)
    if d.shape != o.shape:
        print(f"  {name}: SHAPE {d.shape} vs {o.shape}"); return
    bad = np.flatnonzero(d.ravel().view(np.uint64) != o.ravel().view(np.uint64))
    if bad.size:
        i = bad[0]
        print(f"  {name}: {bad.size} mismatches, first {i}: {d.ravel()[i]!r} vs {o.ravel()[i]!r}")
    else:
        print(f"  {name}: ok")

for geom in [(4, 8), (2, 4), (8, 32), (128, 256), (1, 4096)]:
    ctx = pk.ExecutionContext(*geom)
    print(geom)
    rep("stage1", h(fused.reduce_stage1(dev(V["x"]), ctx)), orc.stage1(V["x"], *geom))
    rep("stage1x2", h(fused.reduce_stage1([dev(V["x"]), dev(V["r"])], ctx)), orc.stage1(np.stack([V["x"], V["r"]], 1), *geom))
    q, part = fused.spmv_fused(a, dev(V["p"]), ("input",), ctx)
    oq, op_ = orc.spmv_fused(a, V["p"], ("input",), geom)
    rep("spmv q", h(q), oq); rep("spmv part1", h(part), op_)
    q, part = fused.spmv_fused(a, dev(V["p"]), ("input", "result"), ctx)
    oq, op_ = orc.spmv_fused(a, V["p"], ("input", "result"), geom)
    rep("spmv part2", h(part), op_)
    x, r, p = dev(V["x"]), dev(V["r"]), dev(V["p"])
    part = fused.fused_cg_vector_update(x, r, p, dev(V["ap"]), 0.37, -0.8, ctx)
    ox, orr, opp = V["x"].copy(), V["r"].copy(), V["p"].copy()
    opart = orc.cg_update(ox, orr, opp, V["ap"], 0.37, -0.8, geom)
    rep("cg x", h(x), ox); rep("cg part", h(part), opart)
    for nb in (1, 2, 3, 4):
        basis = [V[f"b{j}"] for j in range(nb)]
        g = h(fused.fused_gs_stage1([dev(b) for b in basis], dev(V["v"]), ctx))
        rep(f"gs1 nb={nb}", g, orc.gs_stage1(basis, V["v"], geom))
        w = dev(V["v"]); ow = V["v"].copy()
        c, npart = fused.fused_gs_update(w, [dev(b) for b in basis], dev(orc.gs_stage1(basis, V["v"], geom)), ctx)
        oc, onp = orc.gs_update(ow, basis, orc.gs_stage1(basis, V["v"], geom), geom)
        rep(f"gsu c nb={nb}", h(c), oc); rep(f"gsu v nb={nb}", h(w), ow); rep(f"gsu part nb={nb}", h(npart), onp)
    print("  dot", fused.dot(dev(V["x"]), dev(V["r"]), ctx) == orc.dot(V["x"], V["r"], geom))
