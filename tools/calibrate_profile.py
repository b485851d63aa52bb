"""Calibrate the reference's cost model on this B200 and price the classical
vs pipelined CG / BiCGStab iterations across sizes; also report the measured
per-iteration times of both drivers for the same systems (fixed 30
iterations, loop wall time).  Writes profiles/<tag>/b200.profile + JSON."""
import json
import sys
from pathlib import Path

sys.path.insert(0, ".")
import paper_1410_4054_b200 as pk  # noqa: E402

out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/calib")
out.mkdir(parents=True, exist_ok=True)
prof = pk.calibrate_b200(0)
prof.to_file(out / "b200.profile")
lb = pk.latency_barrier(prof)
rows = []
for method in ("cg", "bicgstab"):
    cl, pl = pk.SOLVERS[(method, "classical")], pk.SOLVERS[(method, "pipelined")]
    for k in (1, 2, 3, 4, 5, 6):
        a, b = pk.gen_poisson2d(k)
        pred = pk.speedup_curve((cl, pl), [(f"poisson2d:{k}", a, b)], prof, iterations=30)[0]
        cfg = pk.SolverConfig(fixed_iterations=30, max_iterations=30)
        meas = [s(a, b, config=cfg).loop_seconds / 30 for s in (cl, pl)]
        rows.append({"method": method, "system": f"poisson2d:{k}", "n": a.n_rows,
                     "predicted_classical_us": round(pred["classical_s"] * 1e6, 2),
                     "predicted_pipelined_us": round(pred["pipelined_s"] * 1e6, 2),
                     "predicted_ratio": round(pred["ratio"], 2),
                     "measured_classical_us": round(meas[0] * 1e6, 2), "measured_pipelined_us": round(meas[1] * 1e6, 2),
                     "measured_ratio": round(meas[0] / meas[1], 2)})
res = {"profile": {k: getattr(prof, k) for k in ("launch_latency", "transfer_latency", "bandwidth",
                                                 "transfer_bandwidth")},
       "latency_barrier_bytes": lb.nbytes, "latency_barrier_doubles": lb.real64_count, "curve": rows}
(out / "calibration.json").write_text(json.dumps(res, indent=1))
print(json.dumps(res))
