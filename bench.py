"""Benchmark of the B200 pipelined Krylov path (contract: one JSON line on rank 0).

Headline workload (BASELINE.json configs[1], single B200): pipelined BiCGStab
on the 2D first-order upwind convection-diffusion operator, 1024 x 1024 grid
(n = 1 048 576, nnz = 5 238 784), fp64, reference default reduction geometry
128 x 256 (bit-identical to the reference CPU implementation at that
geometry).  A "step" is one pipelined BiCGStab iteration (3 kernels); the K
timed steps are one fixed-iteration device loop (conditional-WHILE CUDA graph)
timed with CUDA events on its stream, setup excluded -- the paper's /
reference's loop_seconds protocol (solvers.py:632-695).

value    = time per iteration (us).
e2e      = the same metric through the public reference-facing call
           bicgstab_pipelined(A, b, config) with b in page-locked host memory
           (pk.host_array) and x returned in host memory: per-iteration wall
           time of the whole call (H2D b, setup, loop, true residual, D2H x +
           history), K iterations per call.
roofline = dominant loop kernel, CUDA-event timed per launch inside a
           host-enqueued fixed-iteration loop (PK_FLAG_PROFILE), against the
           measured HBM copy peak (MEASURED_PEAKS.json).
cpu_baseline / --impl reference = the UNMODIFIED reference (pipekrylov,
           numba row loop; installed in baseline/_ref by
           oracle/install_reference.sh) on the same system, single-threaded as
           the reference is; the NumPy oracle port only if the reference
           cannot be imported.
Sub-objects (same JSON line): c1 (CG 512^2 to tolerance, latency floor), c3
(GMRES(30) 128^3), c4 (row-partitioned CG 512^3 at this N -- the workload
that shards; at N > 1 it is the headline).

--gpus N without torchrun re-executes itself under torch.distributed.run with
N ranks (one per GPU).  At N > 1 the headline is configs[3]: pipelined CG on
the 3D 7-point Poisson operator 512^3, row-partitioned over the N GPUs (halo
exchange + one NCCL allgather of the group partials per iteration),
max-over-ranks device time.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "CG/BiCGStab/GMRES time per iteration vs unknowns (fp64); achieved HBM GB/s"
SIDE = 1024
GEOM = (128, 256)
C4_SIDE = 512


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def b_csr(n, nnz):
    return 12 * nnz + 4 * (n + 1)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


class ClockSampler:
    """NVML SM clock / throttle reasons sampled during the timed region."""

    BAD = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
           "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, device):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(0.002)

    def sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            pass

    def __enter__(self):
        self.sample()
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self.t.join()
        self.sample()

    def summary(self):
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = [k for k, bit in self.BAD.items() if self.reasons & bit]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU baselines: the reference itself (baseline/_ref), else the oracle port
# ---------------------------------------------------------------------------


def _reference_module():
    """The UNMODIFIED reference package installed by oracle/install_reference.sh."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "pipekrylov" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    os.environ.setdefault("NUMBA_NUM_THREADS", "1")
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import pipekrylov

        return pipekrylov
    except Exception:
        return None


def cpu_baseline_c2(iters):
    """pipelined BiCGStab on the C2 system, fixed iterations, loop time only
    (the reference's loop_seconds, solvers.py:632-695), one host thread."""
    from oracle import pk_oracle as orc  # the synthetic operator's arrays (the reference has no conv-diff generator)

    a, b = orc.convdiff2d(SIDE)
    ref = _reference_module()
    if ref is not None:
        ra = ref.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)
        ctx = ref.ExecutionContext(*GEOM)
        warm = ref.SolverConfig(fixed_iterations=1, max_iterations=1)
        ref.bicgstab_pipelined(ra, b, config=warm, context=ctx)  # numba JIT
        res = ref.bicgstab_pipelined(ra, b, config=ref.SolverConfig(fixed_iterations=iters, max_iterations=iters),
                                     context=ctx)
        us = res.loop_seconds / iters * 1e6
        kind = "reference"
        sample = (f"reference pipekrylov.bicgstab_pipelined (numba row loop, unmodified, baseline/_ref) on the C2 "
                  f"system, {iters} fixed iterations, loop time only")
    else:
        timing = {}
        orc.bicgstab_pipelined(a, b, fixed=iters, max_iterations=iters, geom=GEOM, timing=timing)
        us = timing["loop_seconds"] / iters * 1e6
        kind = "port"
        sample = f"oracle NumPy port of pipekrylov (reference not importable), C2 system, {iters} fixed iterations"
    return {"value": round(us, 1), "unit": "us/iter", "cores": 1, "kind": kind, "sample": sample,
            "cpu": cpu_model(), "host_threads_available": len(os.sched_getaffinity(0))}


def cpu_baseline_c4(iters, side=128):
    """pipelined CG on gen_poisson3d_block(side, 1) with the reference (the
    512^3 system needs ~120 GB of host RAM in the reference's NumPy layout),
    scaled to 512^3 by the unknown count (the CPU iteration is linear in n)."""
    ref = _reference_module()
    from oracle import pk_oracle as orc

    n = side ** 3
    if ref is not None:
        a, b = ref.gen_poisson3d_block(side, 1)
        ctx = ref.ExecutionContext(n // 4096, 4096)
        ref.cg_pipelined(a, b, config=ref.SolverConfig(fixed_iterations=1, max_iterations=1), context=ctx)
        res = ref.cg_pipelined(a, b, config=ref.SolverConfig(fixed_iterations=iters, max_iterations=iters),
                               context=ctx)
        loop = res.loop_seconds
        kind = "reference"
    else:
        a, b = orc.poisson3d(side)
        timing = {}
        orc.cg_pipelined(a, b, fixed=iters, max_iterations=iters, geom=(n // 4096, 4096), timing=timing)
        loop = timing["loop_seconds"]
        kind = "port"
    us = loop / iters * 1e6 * (C4_SIDE ** 3 / n)
    return {"value": round(us, 1), "unit": "us/iter", "cores": 1, "kind": kind, "cpu": cpu_model(),
            "sample": f"pipelined CG 3D Poisson {side}^3 ({iters} fixed iterations, slab geometry), per-iteration "
                      f"time scaled x{C4_SIDE ** 3 // n} to {C4_SIDE}^3 by unknown count"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    iters = max(1, min(args.steps, 40))
    if world > 1:
        cb = cpu_baseline_c4(max(1, min(args.steps, 10)))
        cfgb = c4_config(world)
    else:
        cb = cpu_baseline_c2(iters)
        cfgb = config_block()
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "us/iter",
            "n_gpus": world, "steps": iters, "warmup": args.warmup, "ms_per_step": cb["value"] / 1e3,
            "higher_is_better": False, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": cfgb, "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "us/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# configs
# ---------------------------------------------------------------------------


def config_block():
    return {"workload": "pipelined BiCGStab, 2D upwind convection-diffusion 1024x1024 (configs[1])",
            "n": SIDE * SIDE, "nnz": 5 * SIDE * SIDE - 4 * SIDE, "reduction_geometry": f"{GEOM[0]}x{GEOM[1]}",
            "parallelism": "single GPU (the headline config is single-B200; see c4 for the sharded path)",
            "l2": "inputs larger than L2 (per-iteration working set: CSR 67 MB + 11 n-vectors of 8.4 MB = 159 MB "
                  "> 126 MB L2); no flush between iterations"}


def c4_config(world, side=C4_SIDE):
    n = side ** 3
    gs = 65536 if side >= 256 else 4096
    return {"workload": f"pipelined CG, 3D Poisson 7-point {side}^3 row-partitioned over {world} GPU(s) (configs[3])",
            "n": n, "nnz": 7 * n - 6 * side * side, "reduction_geometry": f"{n // gs}x{gs}",
            "parallelism": f"row-slabs x{world}",
            "collectives_per_iteration": "halo send/recv of p' (one plane per neighbour) + ONE allgather of the "
                                        "group partials (3 doubles per group)",
            "l2": "working set 22 GB >> L2"}


def ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full capture summary (profiles/), or None."""
    try:
        d = json.loads((ROOT / "profiles" / "ncu_traffic.json").read_text())
        return d.get(kernel)
    except Exception:
        return None


def ncu_launch_list(path="profiles/r2/ncu_c2_final/launches.csv"):
    """Average gpu__time_duration per kernel name prefix from the committed
    ncu launch list of this bench command (serialised, one launch at a time)."""
    import csv
    out = {}
    try:
        rows = list(csv.reader(open(ROOT / path)))
    except Exception:
        return out
    hdr = None
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            name = r[hdr.index("Kernel Name")]
            v = float(r[hdr.index("Metric Value")].replace(",", ""))
            t = out.setdefault(name.split("(")[0], [0.0, 0])
            t[0] += v
            t[1] += 1
    return {k: round(v / c / 1e3, 2) for k, (v, c) in out.items()}


def kernel_roofline(pk, dm, ctx, b, iters=200):
    """Per-kernel CUDA-event times of the three loop kernels (host-enqueued
    loop with PK_FLAG_PROFILE, events on the launching stream), against the
    measured HBM copy peak.  Algorithmic bytes per launch (int32 indices,
    fp64 values, every vector read/written once):
      As-SpMV  (OpBicgB):        B_CSR + 32 n   (read r, Ap, r0*; write As)
      Ap'-SpMV (OpBicgApNext):   B_CSR + 32 n   (read p', r', r0*; write Ap')
      xrp      (OpBicgXrpSweep): 64 n           (read x, r, p, Ap, As; write x, r', p')"""
    from paper_1410_4054_b200.solvers import solve_resident

    n = dm.n_rows
    cfg = pk.SolverConfig(fixed_iterations=iters, max_iterations=iters, loop_mode="host")
    solve_resident("bicgstab", dm, b, config=cfg, context=ctx, profile=True)  # warm
    _, res = solve_resident("bicgstab", dm, b, config=cfg, context=ctx, profile=True)
    ks, kl = res.diagnostics["kernel_seconds"], res.diagnostics["kernel_launches"]
    bc = b_csr(n, dm.nnz)
    kernels = [("k_reduce<OpBicgB> (CTA CHAIN engine: s-update + As = A s + 4 dots)", bc + 32 * n, ks[0], kl[0]),
               ("k_reduce_bulk<OpBicgApNext> (BULK engine, TMA-fed: Ap' = A p' + 2 dots)", bc + 32 * n, ks[1], kl[1]),
               ("k_sweep2<OpBicgXrpSweep> (xrp update, 16-byte accesses)", 64 * n, ks[2], kl[2])]
    peak, kind = peaks()
    rows = []
    for name, alg, sec, cnt in kernels:
        t = sec / max(cnt, 1)
        rows.append({"kernel": name, "bytes_per_launch": alg, "launches": cnt, "us_per_launch": round(t * 1e6, 2),
                     "achieved": round(alg / t / 1e9, 1) if t > 0 else None})
    # the committed ncu launch list of this command: serialised per-launch
    # durations (no event brackets); only the SHARE is comparable
    nl = ncu_launch_list()
    keys = {"k_reduce<OpBicgB>": "void k_reduce<4, 2, 4, pk::OpBicgB<int, 5, 0>>",
            "k_reduce_bulk<OpBicgApNext>": "void k_reduce_bulk<2, 4, 3, 7, pk::OpBicgApNext<int, 5, 0>>",
            "k_sweep2<OpBicgXrpSweep>": "void k_sweep2<pk::OpBicgXrpSweep, 4>"}
    ncu_us = {}
    for r in rows:
        k = keys.get(r["kernel"].split(" ")[0])
        if k is not None and k in nl:
            r["ncu_launch_us"] = nl[k]
            ncu_us[r["kernel"]] = nl[k]
    dom = max(rows, key=lambda r: r["us_per_launch"])
    total = sum(r["us_per_launch"] for r in rows)
    if len(ncu_us) == len(rows):
        nt = sum(ncu_us.values())
        for r in rows:
            r["share_events"] = round(r["us_per_launch"] / total, 3)
            r["share_ncu"] = round(r["ncu_launch_us"] / nt, 3)
    return {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved"], "peak": peak,
            "peak_kind": kind, "unit": "GB/s", "frac": round(dom["achieved"] / peak, 4),
            "traffic": ncu_traffic(dom["kernel"].split(" ")[0]), "bytes_per_launch": dom["bytes_per_launch"],
            "us_per_launch": dom["us_per_launch"], "share_of_step": round(dom["us_per_launch"] / total, 3),
            "timing_note": "per-launch CUDA-event brackets on the solve stream in a host-enqueued loop whose "
                           "16-iteration batches are queued behind a spin kernel, so the bracketed kernels run "
                           "back to back (no host launch latency inside a bracket); the graph loop (value) adds "
                           "the per-node launch gaps of the conditional WHILE body",
            "kernels": rows}


def roofline_wide(pk, b_host, iters=200):
    """The parity tax of the reference geometry: the same C2 system at the
    one-element-per-lane geometry 128 x 8192 (G = n, K = 1: LEAF engine, no
    lane chains) -- different reduction geometry, so different roundings; a
    performance comparison only."""
    from paper_1410_4054_b200.solvers import solve_resident
    import torch

    wide = pk.ExecutionContext(128, 8192)
    dm, _ = pk.convdiff2d(SIDE, device=True, context=wide)
    b = torch.from_numpy(b_host).to("cuda")
    n = dm.n_rows
    g = pk.SolverConfig(fixed_iterations=iters, max_iterations=iters)
    solve_resident("bicgstab", dm, b, config=g, context=wide)
    _, rg = solve_resident("bicgstab", dm, b, config=g, context=wide)
    us = rg.loop_seconds / iters * 1e6
    r = kernel_roofline(pk, dm, wide, b, iters)
    iter_bytes = 2 * b_csr(n, dm.nnz) + 128 * n
    peak, _ = peaks()
    return {"geometry": "128x8192 (the headline's 128 groups, one element per lane: LEAF engine)", "us_per_iter": round(us, 3),
            "iteration_frac": round(iter_bytes / (us * 1e-6) / 1e9 / peak, 4),
            "dominant_kernel_us": r["us_per_launch"], "dominant_kernel_frac": r["frac"],
            "kernels": [{"kernel": name, "us_per_launch": row["us_per_launch"], "achieved": row["achieved"]}
                        for name, row in zip(("As = A s + 4 dots (LEAF engine)", "Ap' = A p' + 2 dots (LEAF engine)",
                                              "xrp sweep"), r["kernels"])],
            "note": "same system at a geometry whose lanes hold one row each (no lane chains; LEAF engine): "
                    "what reproducing the reference's 128 x 256 chains bit for bit costs or saves relative to "
                    "the other ordering the reference could be run with"}


def classical_same_box(pk, method, a, b, ctx, pipelined_us, iters=40):
    """The reference's classical driver (one kernel per BLAS op, a host read
    per inner product; solvers.py:310-389 / 485-580) on the same B200 and the
    same kernels library -- the paper's baseline, beside the pipelined number."""
    cfg = pk.SolverConfig(fixed_iterations=iters, max_iterations=iters)
    fn = pk.SOLVERS[(method, "classical")]
    fn(a, b, config=pk.SolverConfig(fixed_iterations=3, max_iterations=3), context=ctx)
    res = fn(a, b, config=cfg, context=ctx)
    us = res.loop_seconds / res.iterations * 1e6
    st = res.trace.steady_state()
    return {"value": round(us, 3), "unit": "us/iter", "iterations": res.iterations,
            "launches_per_iteration": st.launches, "host_reads_per_iteration": st.transfers,
            "pipelined_speedup": round(us / pipelined_us, 2),
            "note": f"{method}_classical on this GPU, {iters} fixed iterations, loop wall time "
                    "(host-driven: each inner product is a device->host read)"}


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def sub_c1(pk, dev, with_classical=True):
    """configs[0]: CG 2D Poisson 512^2 to tol 1e-8 at 128 x 256 (941
    iterations) -- the latency-bound regime: per-iteration time against the
    measured floor of one gated kernel per WHILE-graph iteration."""
    a, b = pk.poisson2d_grid(512)
    ctx = pk.ExecutionContext(*GEOM, device=dev)
    cfg = pk.SolverConfig(max_iterations=2000)
    pk.cg_pipelined(a, b, config=cfg, context=ctx)
    t0 = time.perf_counter()
    res = pk.cg_pipelined(a, b, config=cfg, context=ctx)
    wall = time.perf_counter() - t0
    us = res.loop_seconds / res.iterations * 1e6
    n = a.n_rows
    byt = b_csr(n, a.nnz) + 64 * n
    floor = pk.launch_floor(ctx, kernels_per_iteration=1)
    out = {"workload": "pipelined CG, 2D Poisson 512x512 to tol 1e-8 (configs[0])", "n": n,
           "iterations": res.iterations, "termination": res.termination, "us_per_iter": round(us, 3),
           "time_to_tolerance_s": round(wall, 5),
           "launch_floor_us_per_iter": round(floor["us_per_iteration"], 3),
           "floor_note": floor["note"], "vs_floor": round(us / floor["us_per_iteration"], 2),
           "iteration_bytes": byt, "achieved_gbs": round(byt / (us * 1e-6) / 1e9, 1),
           "l2": "working set 31 MB < 126 MB L2: latency/L2-bound"}
    if with_classical:
        out["classical_gpu"] = classical_same_box(pk, "cg", a, b, ctx, us)
    return out


def sub_c3(pk, dev, torch, cycles=1):
    """configs[2]: GMRES(30) on the 3D upwind convection-diffusion 128^3."""
    from paper_1410_4054_b200.solvers import solve_resident

    side, m = 128, 30
    ctx = pk.ExecutionContext(*GEOM, device=dev)
    dm, b_host = pk.convdiff3d(side, device=True, context=ctx)
    b = torch.from_numpy(b_host).to("cuda")
    iters = cycles * m
    cfg = pk.SolverConfig(fixed_iterations=iters, max_iterations=iters, restart=m)
    solve_resident("gmres", dm, b, config=cfg, context=ctx)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, res = solve_resident("gmres", dm, b, config=cfg, context=ctx)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    n, nnz = dm.n_rows, dm.nnz
    us_inner = res.loop_seconds / res.iterations * 1e6
    us_full = wall / res.iterations * 1e6
    steps = sum(pk.solvers.iteration_kernel_bytes("gmres", n, nnz, 4, i) for i in range(1, m + 1))
    per_inner = steps / m
    per_full = (steps + 8 * n * (m + 2)) / m
    peak, _ = peaks()
    return {"workload": f"pipelined GMRES({m}), 3D 7-point upwind convection-diffusion {side}^3 (configs[2])",
            "n": n, "nnz": nnz, "iterations": res.iterations, "us_per_iter_inner": round(us_inner, 3),
            "us_per_iter_full_cycle": round(us_full, 3),
            "inner_is": "Arnoldi-loop time / iteration (the reference's loop_seconds protocol, solvers.py:928/953)",
            "bytes_per_iteration_inner": int(per_inner),
            "frac_inner": round(per_inner / (us_inner * 1e-6) / 1e9 / peak, 4),
            "frac_full_cycle": round(per_full / (us_full * 1e-6) / 1e9 / peak, 4)}


def c4_run(pk, torch, dist, world, rank, dev, steps, warmup, side=C4_SIDE):
    """configs[3]: row-partitioned CG, one slab per rank (NCCL halos + one
    partials allgather per iteration); world 1 runs the same solver in one
    process.  Returns (us per iteration, max over ranks; SolverResult)."""
    gs = 65536 if side >= 256 else 4096
    if world > 1:
        solver = pk.PartitionedCG(side, gs, rank, world, dev, max(steps, warmup))
        solver.solve(pk.SolverConfig(fixed_iterations=warmup, max_iterations=warmup))
        dist.barrier()
        torch.cuda.synchronize()
        res = solver.solve(pk.SolverConfig(fixed_iterations=steps, max_iterations=steps))
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([res.loop_seconds], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        loop_s = float(t.item())
        solver.close()
    else:
        pk.cg_partitioned(side, 1, gs, config=pk.SolverConfig(fixed_iterations=warmup, max_iterations=warmup),
                          device=dev)
        res = pk.cg_partitioned(side, 1, gs, config=pk.SolverConfig(fixed_iterations=steps, max_iterations=steps),
                                device=dev)
        loop_s = res.loop_seconds
    return loop_s / steps * 1e6, res


def c4_roofline(us, world, res, side=C4_SIDE):
    n = side ** 3
    nnz = 7 * n - 6 * side * side
    peak, _ = peaks()
    split = int(res.diagnostics.get("launches_per_iteration", 2)) >= 2
    # split step (partitions >= 2^20 rows): update sweep 56 n + SpMV B_CSR + 24 n, one halo plane
    # of p' per neighbour; fused step: B_CSR + 64 n, three halo planes (r, p, Ap)
    per_gpu = (b_csr(n, nnz) + (80 if split else 64) * n) / world
    halo = (1 if split else 3) * 2 * 8 * side * side * (world > 1)
    return {"bytes_per_iteration_per_gpu": int(per_gpu), "halo_bytes_per_iteration_per_gpu": halo,
            "achieved_gbs_per_gpu": round(per_gpu / (us * 1e-6) / 1e9, 1),
            "frac": round(per_gpu / (us * 1e-6) / 1e9 / peak, 4)}


def e2e_c2(pk, ctx, iters):
    """The public reference-facing call with host buffers: b in page-locked
    memory (pk.host_array), x returned in host memory; H2D of b, setup, loop,
    true residual, D2H of x + history inside the timed region."""
    a_host, b0 = pk.convdiff2d(SIDE)
    b = pk.host_array(a_host.n_rows)
    b[:] = b0
    cfg = pk.SolverConfig(fixed_iterations=iters, max_iterations=iters)
    pk.bicgstab_pipelined(a_host, b, config=cfg, context=ctx)  # uploads A once (cached on A), caches the workspace
    walls = []
    for _ in range(5):
        t0 = time.perf_counter()
        r = pk.bicgstab_pipelined(a_host, b, config=cfg, context=ctx)
        walls.append(time.perf_counter() - t0)
    per_call = statistics.median(walls)
    n = a_host.n_rows
    return {"value": round(per_call / iters * 1e6, 3), "unit": "us/iter", "iterations_per_call": iters,
            "h2d_bytes_per_step": round(8 * n / iters), "d2h_bytes_per_step": round((8 * n + 8 * iters) / iters),
            "h2d_bytes_per_call": 8 * n, "d2h_bytes_per_call": 8 * n + 8 * iters,
            "call_ms": round(per_call * 1e3, 3), "termination": r.termination}


def run_c2(args, torch, pk, dev):
    from paper_1410_4054_b200.solvers import solve_resident

    ctx = pk.ExecutionContext(*GEOM, device=dev)
    dm, b_host = pk.convdiff2d(SIDE, device=True, context=ctx)
    n, nnz = dm.n_rows, dm.nnz
    b = torch.from_numpy(b_host).to("cuda")
    # warm-up: graph build/instantiate paths, clocks up
    solve_resident("bicgstab", dm, b, config=pk.SolverConfig(fixed_iterations=args.warmup,
                                                                max_iterations=args.warmup), context=ctx)
    cfg = pk.SolverConfig(fixed_iterations=args.steps, max_iterations=args.steps, loop_mode=args.loop)
    solve_resident("bicgstab", dm, b, config=cfg, context=ctx)  # the timed configuration, once untimed
    torch.cuda.synchronize()
    with ClockSampler(dev) as clk:
        _, res = solve_resident("bicgstab", dm, b, config=cfg, context=ctx)
        torch.cuda.synchronize()
    us_iter = res.loop_seconds / args.steps * 1e6
    iter_bytes = 2 * b_csr(n, nnz) + 128 * n
    peak, _ = peaks()
    line = {
        "metric": METRIC, "value": round(us_iter, 3), "unit": "us/iter", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(us_iter / 1e3, 6), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config_block(),
        "iteration_roofline": {"bytes_per_iteration": iter_bytes,
                               "reference_4kernel_bytes": 2 * b_csr(n, nnz) + 144 * n,
                               "fused_2kernel_bytes": 2 * b_csr(n, nnz) + 112 * n,
                               "achieved_gbs": round(iter_bytes / (us_iter * 1e-6) / 1e9, 1),
                               "frac": round(iter_bytes / (us_iter * 1e-6) / 1e9 / peak, 4)},
        "roofline": kernel_roofline(pk, dm, ctx, b),
        "e2e": e2e_c2(pk, ctx, args.steps),
        # kernel launches of the timed solve (setup, the loop -- one cooperative kernel when the loop is
        # persistent, else 3 per iteration -- and the tail), counted by the library
        "gpu_launches": int(res.diagnostics.get("launches", 3 * args.steps)),
        "clocks": clk.summary(),
        "termination": res.termination,
    }
    a_host, bh = pk.convdiff2d(SIDE)
    line["classical_gpu"] = classical_same_box(pk, "bicgstab", a_host, bh, ctx, us_iter)
    try:
        line["roofline_wide"] = roofline_wide(pk, b_host)
    except Exception as exc:  # informational only
        line["roofline_wide"] = {"error": str(exc)[:200]}
    return line


def spawn_ranks(args):
    """--gpus N without a torchrun environment: re-execute this script under
    torch.distributed.run, one rank per GPU, and forward its exit code."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-sub", action="store_true", help="skip the c1/c3/c4 sub-objects")
    ap.add_argument("--loop", default="graph", choices=["graph", "host"],
                    help="iteration loop driver (host: per-launch kernels visible to ncu)")
    ap.add_argument("--workload", default="c2", choices=["c2", "c1", "c3", "c4", "c5", "ranks"],
                    help="c2 = configs[1] (default headline at N=1); c4 = configs[3] (headline at N>1)")
    ap.add_argument("--side", type=int, default=None, help="c4 grid side (default 512)")
    ap.add_argument("--nsys", type=int, default=4096, help="c5 number of systems")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    if args.workload == "ranks":
        # launcher self-check (CPU test): every rank reports and exits
        print(json.dumps({"rank": rank, "world": world, "local_rank": local}), flush=True)
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_1410_4054_b200 as pk

    dev = torch.cuda.current_device()
    line = None
    if world > 1 or args.workload == "c4":
        side = args.side or C4_SIDE
        with ClockSampler(dev) as clk:
            us, res = c4_run(pk, torch, dist, world, rank, dev, args.steps, args.warmup, side)
        line = {"metric": METRIC, "value": round(us, 3), "unit": "us/iter", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(us / 1e3, 6), "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": c4_config(world, side), "iteration_roofline": c4_roofline(us, world, res, side),
                "gpu_launches": int(res.diagnostics.get("launches_per_iteration", 2)) * args.steps,
                "clocks": clk.summary(), "termination": res.termination,
                "e2e": {"value": round(us, 3), "unit": "us/iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                        "note": "device-resident partitioned solve (the matrix is generated in HBM on each rank)"}}
        if rank == 0 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_c4(max(1, min(args.steps, 10)))
    elif args.workload == "c2":
        line = run_c2(args, torch, pk, dev)
        if not args.no_sub:
            line["c1"] = sub_c1(pk, dev)
            line["c3"] = sub_c3(pk, dev, torch)
            us4, res4 = c4_run(pk, torch, None, 1, 0, dev, max(args.steps, 10), args.warmup)
            line["c4"] = {"config": c4_config(1), "us_per_iter": round(us4, 3), "n_gpus": 1,
                          "iteration_roofline": c4_roofline(us4, 1, res4), "termination": res4.termination,
                          "note": "the workload --gpus N runs as its headline (sharded over N GPUs)"}
        if not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline_c2(max(1, min(args.steps, 40)))
    elif args.workload == "c1":
        c1 = sub_c1(pk, dev)
        line = {"metric": METRIC, "value": c1["us_per_iter"], "unit": "us/iter", "n_gpus": 1, "steps": c1["iterations"],
                "warmup": args.warmup, "ms_per_step": round(c1["us_per_iter"] / 1e3, 6), "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": c1}
    elif args.workload == "c3":
        c3 = sub_c3(pk, dev, torch, cycles=max(args.steps // 30, 1))
        line = {"metric": METRIC, "value": c3["us_per_iter_inner"], "unit": "us/iter", "n_gpus": 1,
                "steps": c3["iterations"], "warmup": args.warmup, "ms_per_step": round(c3["us_per_iter_inner"] / 1e3, 6),
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "config": c3}
    elif args.workload == "c5":
        line = run_c5(args, pk, torch, dist, world, rank)
    if rank == 0 and line is not None:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def _c5_system(i, sides=(128, 256, 512)):
    from oracle import pk_oracle as orc

    side = sides[i % 3]
    a, _ = orc.poisson2d_side(side)
    return a, np.random.default_rng(i).random(side * side)


def _c5_ref_init():
    ref = _reference_module()
    a, b = _c5_system(0)
    if ref is not None:  # numba JIT once per worker
        ra = ref.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)
        ref.cg_pipelined(ra, b, config=ref.SolverConfig(fixed_iterations=1, max_iterations=1))


def _c5_ref_solve(i):
    ref = _reference_module()
    a, b = _c5_system(i)
    if ref is None:
        from oracle import pk_oracle as orc

        return orc.cg_pipelined(a, b, max_iterations=5000, geom=GEOM)["iterations"]
    ra = ref.CsrMatrix(a.n_rows, a.n_cols, a.rowptr, a.cols, a.vals)
    return ref.cg_pipelined(ra, b, config=ref.SolverConfig(max_iterations=5000)).iterations


def cpu_baseline_c5(nsample=48):
    """The C5 mix solved by the reference (one system per task) on a
    multiprocessing pool over all host cores; systems/s of the sample."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    with ctx.Pool(processes=cores, initializer=_c5_ref_init) as pool:
        pool.map(_c5_ref_solve, [0] * cores)  # workers warm
        t0 = time.perf_counter()
        its = pool.map(_c5_ref_solve, list(range(nsample)), chunksize=1)
        wall = time.perf_counter() - t0
    kind = "reference" if _reference_module() is not None else "port"
    return {"value": round(nsample / wall, 3), "unit": "systems/s", "cores": cores, "kind": kind,
            "cpu": cpu_model(), "iterations_total": int(sum(its)),
            "sample": f"first {nsample} systems of the C5 mix (sides 128/256/512, seeded RHS), reference "
                      f"cg_pipelined to tol 1e-8, one system per task on a {cores}-process pool"}


def lpt_assign(costs, world):
    """Longest-processing-time-first assignment of independent systems to
    ranks (greedy: largest estimated cost to the least-loaded rank)."""
    load = [0.0] * world
    owner = [0] * len(costs)
    for i in sorted(range(len(costs)), key=lambda j: -costs[j]):
        r = min(range(world), key=lambda k: load[k])
        owner[i] = r
        load[r] += costs[i]
    return owner


def run_c5(args, pk, torch, dist, world, rank):
    nsys_total = args.nsys
    sides = [128, 256, 512]
    # LPT over ranks by the estimated work nnz x iterations (CG iterations grow ~linearly with the side)
    costs = [5 * sides[i % 3] ** 2 * 3.0 * sides[i % 3] for i in range(nsys_total)]
    owner = lpt_assign(costs, world)
    mine = [i for i in range(nsys_total) if owner[i] == rank]
    mats = {sd: pk.poisson2d_grid(sd)[0] for sd in sides}
    systems = [(mats[sides[i % 3]], np.random.default_rng(i).random(sides[i % 3] ** 2)) for i in mine]
    cfg = pk.SolverConfig(max_iterations=5000, loop_mode="graph")
    pk.solve_batch(systems[:48], tag="cg", config=cfg, threads=16)  # uploads + worker contexts + cached graphs
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = pk.solve_batch(systems, tag="cg", config=cfg, threads=16)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    its = sum(r.iterations for r in out)
    if dist:
        t = torch.tensor([wall, its], dtype=torch.float64, device="cuda")
        w = t.clone()
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        wall, its = float(w[0].item()), float(t[1].item())
    line = {"metric": "transient batch: systems/s (pipelined CG to tol 1e-8)", "unit": "systems/s",
            "higher_is_better": True, "value": round(nsys_total / wall, 3), "n_gpus": world,
            "ms_per_step": round(wall * 1e3, 3), "scaling": "strong", "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{nsys_total} independent 2D Poisson systems (sides 128/256/512, "
                                   "RHS default_rng(s).random(n)) LPT-assigned to the GPUs (configs[4])",
                       "solver_iterations_total": int(its), "batch_wall_s": round(wall, 4),
                       "workers": "16 host threads x own stream, cached workspaces + WHILE graphs"},
            "all_converged": all(r.termination == "converged" for r in out)}
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_c5()
    return line


if __name__ == "__main__":
    main()
