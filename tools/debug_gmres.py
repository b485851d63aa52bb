"""Debug helper: GMRES history on the device vs the oracle, first mismatch."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_1410_4054_b200 as pk
from oracle import pk_oracle as orc

a, b = pk.gen_poisson2d(1)
for fixed in (1, 2, 3, 5):
    cfg = pk.SolverConfig(fixed_iterations=fixed, max_iterations=fixed)
    r = pk.gmres_pipelined(a, b, config=cfg)
    o = orc.gmres_pipelined(a, b, fixed=fixed, max_iterations=fixed)
    print(fixed, "dev", r.residual_history[:6], r.termination)
    print(fixed, "orc", o["history"][:6], o["termination"])
    print("  x maxdiff", np.abs(r.x - o["x"]).max(), "true", r.true_final_residual, o["true_final_residual"])
