"""The reference's launch/transfer cost model, calibrated on B200
(execmodel.py:42-107, 225-278).

``DeviceProfile`` / ``latency_barrier`` / ``predict_iteration_time`` /
``speedup_curve`` keep the reference's semantics (additive, no overlap:
launches x launch latency + transfers x transfer latency + kernel bytes /
bandwidth + transfer bytes / link bandwidth).  ``calibrate_b200`` measures
the four figures on the current GPU with the library's own kernels, so the
model prices a trace with B200 numbers instead of the reference's generic
accelerator (8 us, 200 GB/s, 8 GB/s):

* launch_latency: back-to-back stream launches of a 32-element
  ``pk_vec_update`` (CUDA events over 400 launches);
* transfer_latency: an 8-byte device-to-host read after a kernel
  (``tensor.item()``, wall clock, median of 200);
* bandwidth: ``pk_vec_update`` COPY of 2 x 1 GiB (read + write bytes / time);
* transfer_bandwidth: 512 MiB pinned host -> device copy.

Traces recorded by the B200 drivers count real launches (a pipelined
iteration is 1-3 graph-resident launches, a classical one 8-20 launches plus
2-7 host reads), so ``speedup_curve`` over (classical, pipelined) reproduces
the paper's latency-regime argument with measured constants.
"""

from __future__ import annotations

import math
import statistics
import time
from dataclasses import dataclass
from pathlib import Path

from .linalg import ExecutionContext, PhaseRecord

_FIELDS = ("launch_latency", "transfer_latency", "bandwidth", "transfer_bandwidth")


@dataclass(frozen=True)
class DeviceProfile:
    """Latency (s) and bandwidth (B/s) figures of the modelled device;
    defaults are the reference's generic accelerator (execmodel.py:42-60)."""

    launch_latency: float = 8e-6
    transfer_latency: float = 8e-6
    bandwidth: float = 200e9
    transfer_bandwidth: float = 8e9

    def __post_init__(self):
        for name in _FIELDS:
            v = getattr(self, name)
            if not (isinstance(v, (int, float)) and math.isfinite(v) and v > 0):
                raise ValueError(f"{name} must be a finite positive number, got {v!r}")

    @classmethod
    def from_file(cls, path) -> "DeviceProfile":
        """``key = value`` lines, ``#`` comments (execmodel.py:62-87)."""
        values: dict[str, float] = {}
        for lineno, raw in enumerate(Path(path).read_text().splitlines(), start=1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            key, sep, text = line.partition("=")
            if not sep:
                raise ValueError(f"{path}: line {lineno}: expected 'key = value', got {raw!r}")
            key = key.strip()
            if key not in _FIELDS:
                raise ValueError(f"{path}: line {lineno}: unknown profile key {key!r} "
                                 f"(expected one of: {', '.join(sorted(_FIELDS))})")
            try:
                values[key] = float(text.strip())
            except ValueError:
                raise ValueError(f"{path}: line {lineno}: bad number {text.strip()!r}") from None
        return cls(**values)

    def to_file(self, path) -> None:
        Path(path).write_text("".join(f"{k} = {getattr(self, k)!r}\n" for k in _FIELDS))


@dataclass(frozen=True)
class LatencyBarrier:
    """Data volume whose streaming time equals one launch latency."""

    nbytes: float
    real64_count: float


def latency_barrier(profile: DeviceProfile | None = None) -> LatencyBarrier:
    """Bytes (and float64 values) movable in one launch latency (execmodel.py:98-107)."""
    p = profile or DeviceProfile()
    nbytes = p.launch_latency * p.bandwidth
    return LatencyBarrier(nbytes=nbytes, real64_count=nbytes / 8)


def predict_iteration_time(record: PhaseRecord, profile: DeviceProfile | None = None) -> float:
    """Modelled seconds of one phase record (execmodel.py:225-236)."""
    p = profile or DeviceProfile()
    return (record.launches * p.launch_latency + record.transfers * p.transfer_latency
            + record.bytes_kernel / p.bandwidth + record.bytes_transfer / p.transfer_bandwidth)


def speedup_curve(solver_pair, systems, profile: DeviceProfile | None = None, iterations: int = 30,
                  context: ExecutionContext | None = None) -> list[dict]:
    """Predicted per-iteration time of (classical, pipelined) over systems
    (execmodel.py:239-278): fixed iterations, steady-state record priced."""
    from .solvers import SolverConfig

    p = profile or DeviceProfile()
    cfg = SolverConfig(fixed_iterations=iterations, max_iterations=max(iterations, 1))
    rows = []
    for label, a, b in systems:
        times = [predict_iteration_time(s(a, b, config=cfg, context=context).trace.steady_state(), p)
                 for s in solver_pair]
        rows.append({"label": label, "size": a.n_rows, "classical_s": times[0], "pipelined_s": times[1],
                     "ratio": times[0] / times[1]})
    return rows


def calibrate_b200(device: int = 0) -> DeviceProfile:
    """Measure the four profile figures on ``cuda:device`` with the
    library's kernels (see the module docstring)."""
    import ctypes as C

    import torch

    from . import _native as N
    from .device import context_for

    ctx = ExecutionContext(device=device)
    dc = context_for(ctx)
    dev = torch.device("cuda", device)
    stream = torch.cuda.current_stream(dev)
    dc.set_stream(stream)
    lib = N.lib()

    def vec(kind, n, y, x):
        N.check(lib.pk_vec_update(dc.handle, kind, n, C.c_void_p(y.data_ptr()), C.c_void_p(x.data_ptr()), None,
                                  1.0, 0.0), "calibration kernel")

    def timed(fn, reps):
        for _ in range(5):
            fn()
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1) * 1e-3 / reps

    small = torch.zeros(32, dtype=torch.float64, device=dev)
    small2 = torch.zeros(32, dtype=torch.float64, device=dev)
    launch = timed(lambda: vec(N.VEC_COPY, 32, small, small2), 400)

    reads = []
    for _ in range(200):
        vec(N.VEC_COPY, 32, small, small2)
        t0 = time.perf_counter()
        small[0].item()
        reads.append(time.perf_counter() - t0)
    transfer = statistics.median(reads)

    n = 1 << 27  # 1 GiB per vector
    big_x = torch.empty(n, dtype=torch.float64, device=dev).fill_(1.0)
    big_y = torch.empty_like(big_x)
    bw = 16 * n / timed(lambda: vec(N.VEC_COPY, n, big_y, big_x), 10)
    del big_x, big_y

    host = torch.empty(1 << 26, dtype=torch.float64).pin_memory()
    devbuf = torch.empty(1 << 26, dtype=torch.float64, device=dev)
    link = 8 * (1 << 26) / timed(lambda: devbuf.copy_(host, non_blocking=True), 5)
    return DeviceProfile(launch_latency=launch, transfer_latency=transfer, bandwidth=bw, transfer_bandwidth=link)
