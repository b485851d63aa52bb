"""Debug: per-CTA %globaltimer stamps of the BULK engine (libpk_b200_trace.so,
built with -DPK_BULK_TRACE) for one K_B launch of the C2 loop.  Prints a
summary of the per-CTA timeline (ns relative to the earliest CTA start)."""
import ctypes, json, os, sys
os.environ.setdefault("PK_LIB_VARIANT", "trace")
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1410_4054_b200 as pk
from paper_1410_4054_b200 import _native
from paper_1410_4054_b200.solvers import solve_resident
side = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
ctx = pk.ExecutionContext(128, 256, device=0)
dm, b = pk.convdiff2d(side, device=True, context=ctx)
b = torch.from_numpy(b).cuda()
cfg = pk.SolverConfig(fixed_iterations=3, max_iterations=3, loop_mode="host")
solve_resident("bicgstab", dm, b, config=cfg, context=ctx)
torch.cuda.synchronize()
buf = torch.zeros(1024 * 32 * 64, dtype=torch.int64, device="cuda")
lib = ctypes.CDLL(str(_native.LIB_PATH))
lib.pk_debug_bulk_trace(ctypes.c_void_p(buf.data_ptr()))
cfg1 = pk.SolverConfig(fixed_iterations=1, max_iterations=1, loop_mode="host")
solve_resident("bicgstab", dm, b, config=cfg1, context=ctx)
torch.cuda.synchronize()
lib.pk_debug_bulk_trace(ctypes.c_void_p(0))
fin = buf[1024 * 32: 1024 * 32 + 2].cpu().numpy()
t = buf[: 1024 * 32].view(1024, 32).cpu().numpy()
# the last bulk launch overwrote the buffer: ApNext (2nd SpMV) -- report it
t0 = t[:, 0].min()
def st(x):
    x = x.astype(np.float64)
    return {"min": round(float(x.min()), 1), "p50": round(float(np.median(x)), 1), "max": round(float(x.max()), 1)}
out = {"start": st(t[:, 0] - t0), "first_issue": st(t[:, 4] - t0), "fold_end": st(t[:, 1] - t0),
       "tree_end": st(t[:, 2] - t0)}
for j in range(8):
    out[f"chunk{j}_full"] = st(t[:, 5 + 2 * j] - t0)
    out[f"chunk{j}_computed"] = st(t[:, 21 + j] - t0)
    out[f"chunk{j}_end"] = st(t[:, 6 + 2 * j] - t0)
out["finalizer_start"] = float(fin[0] - t0)
out["finalizer_end"] = float(fin[1] - t0)
sm = t[:, 3]
out["ctas_per_sm"] = np.bincount(sm.astype(np.int64)).tolist()[:8]
out["distinct_sms"] = int(len(set(sm.tolist())))
print(json.dumps(out))
