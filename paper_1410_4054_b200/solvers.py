"""Pipelined Krylov drivers on B200 behind the reference's solver API.

Drop-in for ``pipekrylov.SOLVERS[(method, "pipelined")]`` (reference
__init__.py:81-88; solvers.py:395-469, 583-712, 865-1008): same signature
``solver(a, b, x0=None, config=None, context=None, debug=False)``, same
``SolverResult`` fields, same ``ValueError`` validation, and bit-identical
numbers at the same ``ExecutionContext`` geometry.  The loop itself runs in
libpk_b200.so: CG and BiCGStab as a conditional-WHILE CUDA graph with all
scalar recurrences finalized on the device, GMRES(m) with one host round trip
per restart cycle for the triangular solve (done here in NumPy, exactly as
the reference does it).

``solve(A, b, tag, tol, maxiter)`` is the north-star convenience entry.
"""

from __future__ import annotations

import ctypes as C
import math
import sys
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .device import DeviceMatrix, context_for, device_matrix
from .linalg import CHECK, FINISH, ITERATION, SETUP, CsrMatrix, ExecutionContext, ExecutionTrace, PhaseRecord, as_vector

CONVERGED = "converged"
MAX_ITER = "max_iter"
BREAKDOWN = "breakdown"
LUCKY_BREAKDOWN = "lucky_breakdown"
CLASSICAL_GS = "classical_gs"
MODIFIED_GS = "modified_gs"
DEFAULT_BREAKDOWN_TOLERANCE = 1e-30


class BreakdownError(RuntimeError):
    """A recurrence divisor vanished (errors.py:6-18)."""

    def __init__(self, kind: str, message: str = ""):
        self.kind = kind
        super().__init__(message or f"breakdown: {kind}")


class LuckyBreakdown(Exception):
    """The GMRES candidate basis vector has (numerically) zero norm (errors.py:21-27)."""

    def __init__(self, norm: float):
        self.norm = norm
        super().__init__(f"candidate basis vector has norm {norm!r}")


@dataclass(frozen=True)
class SolverConfig:
    """Driver knobs (solvers.py:104-145) plus ``loop_mode``: "graph" (CUDA
    graph with a device-side WHILE condition, default) or "host"."""

    tolerance: float = 1e-8
    max_iterations: int = 500
    restart: int = 30
    orthogonalization: str = CLASSICAL_GS
    breakdown_tolerance: float = DEFAULT_BREAKDOWN_TOLERANCE
    fixed_iterations: int | None = None
    loop_mode: str = "graph"

    def __post_init__(self):
        if not (self.tolerance > 0):
            raise ValueError("tolerance must be positive")
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.restart < 1:
            raise ValueError("restart must be at least 1")
        if self.orthogonalization not in (CLASSICAL_GS, MODIFIED_GS):
            raise ValueError(f"unknown orthogonalization {self.orthogonalization!r}")
        if not (self.breakdown_tolerance > 0):
            raise ValueError("breakdown_tolerance must be positive")
        if self.fixed_iterations is not None and self.fixed_iterations < 1:
            raise ValueError("fixed_iterations must be at least 1 when set")
        if self.loop_mode not in ("graph", "host"):
            raise ValueError(f"unknown loop_mode {self.loop_mode!r}")

    @property
    def fixed(self) -> bool:
        return self.fixed_iterations is not None

    def iteration_limit(self) -> int:
        return self.fixed_iterations if self.fixed else self.max_iterations

    def loop_breakdown_tolerance(self) -> float:
        return 0.0 if self.fixed else self.breakdown_tolerance

    @classmethod
    def coerce(cls, cfg) -> "SolverConfig":
        if cfg is None:
            return cls()
        if isinstance(cfg, cls):
            return cfg
        # the reference's SolverConfig (same field names)
        return cls(tolerance=cfg.tolerance, max_iterations=cfg.max_iterations, restart=cfg.restart,
                   orthogonalization=cfg.orthogonalization, breakdown_tolerance=cfg.breakdown_tolerance,
                   fixed_iterations=cfg.fixed_iterations)


@dataclass
class SolverResult:
    """Outcome of one run (solvers.py:148-171)."""

    x: np.ndarray
    residual_history: list
    true_final_residual: float
    iterations: int
    termination: str
    trace: ExecutionTrace
    breakdown_kind: str | None = None
    loop_seconds: float = 0.0
    diagnostics: dict = field(default_factory=dict)

    @property
    def converged(self) -> bool:
        return self.termination == CONVERGED


class UpperTriangular:
    """Dense upper-triangular matrix filled column by column (solvers.py:174-202)."""

    def __init__(self, order: int):
        if order < 0:
            raise ValueError("order must be non-negative")
        self.order = order
        self.data = np.zeros((order, order))

    def set(self, row: int, col: int, value: float) -> None:
        if not (0 <= row <= col < self.order):
            raise ValueError(f"entry ({row}, {col}) is not in the upper triangle")
        self.data[row, col] = value

    def get(self, row: int, col: int) -> float:
        if not (0 <= row <= col < self.order):
            raise ValueError(f"entry ({row}, {col}) is not in the upper triangle")
        return float(self.data[row, col])

    def leading(self, k: int) -> "UpperTriangular":
        if not (0 <= k <= self.order):
            raise ValueError(f"leading block size {k} out of range")
        out = UpperTriangular(k)
        out.data[:] = self.data[:k, :k]
        return out

    def entry_count(self) -> int:
        return self.order * (self.order + 1) // 2


def solve_upper_triangular(r: UpperTriangular, rhs, breakdown_tolerance: float = DEFAULT_BREAKDOWN_TOLERANCE):
    """Host back substitution with NumPy's dot, as the reference does
    (solvers.py:205-218), so the BLAS summation order is identical."""
    rhs = as_vector(rhs, n=r.order, name="rhs")
    eta = np.zeros(r.order)
    for i in range(r.order - 1, -1, -1):
        d = r.data[i, i]
        if abs(d) < breakdown_tolerance:
            raise BreakdownError("singular_R", f"zero diagonal at position {i}")
        eta[i] = (rhs[i] - float(np.dot(r.data[i, i + 1:], eta[i + 1:]))) / d
    return eta


@N.TRISOLVE_FN
def _trisolve_cb(user, k, rptr, ld, xiptr, btol, etaptr):
    """Called by libpk_b200 once per GMRES cycle (solvers.py:971-978)."""
    try:
        rfull = np.ctypeslib.as_array(rptr, shape=(ld * ld,)).reshape(ld, ld)
        xi = np.ctypeslib.as_array(xiptr, shape=(k,)).copy()
        tri = UpperTriangular(k)
        tri.data[:] = rfull[:k, :k]
        eta = solve_upper_triangular(tri, xi, btol)
        out = np.ctypeslib.as_array(etaptr, shape=(k,))
        out[:] = eta
        return 0
    except BreakdownError:
        return 1


class _Diagnostics:
    """The reference's debug=True side computations (solvers.py:417-467,
    606-673, 895-997), evaluated with NumPy on host copies of the device
    vectors the native loop hands over one iteration at a time -- the same
    np.dot / np.linalg.norm / matmul calls on bit-identical vectors."""

    def __init__(self, method: str):
        self.method = method
        if method == "cg":
            self.diag = {"rr_direct": [], "beta": []}
        elif method == "bicgstab":
            self.diag = {"s_dot_r0star": [], "s_norm": [], "identity_rr": [], "direct_rr": []}
        else:
            self.diag = {"ortho_offdiag": []}
        self.r0star = None
        self.error = None

    def __call__(self, user, event, it, v0, v1, n, scal, nscal):
        try:
            a0 = np.ctypeslib.as_array(v0, shape=(n,)).copy() if v0 and event != N.DBG_GMRES_CYCLE else None
            sc = [float(scal[i]) for i in range(nscal)]
            d = self.diag
            if event == N.DBG_CG_SETUP or event == N.DBG_CG_ITER:
                d["rr_direct"].append(float(np.dot(a0, a0)))
                if sc:
                    d["beta"].append(sc[0])
            elif event == N.DBG_BICG_SETUP:
                self.r0star = a0
                d["r0star_norm"] = float(np.linalg.norm(a0))
            elif event == N.DBG_BICG_S:
                ap = np.ctypeslib.as_array(v1, shape=(n,))
                s_vec = a0 - sc[0] * ap  # fused.py:177, s = r - alpha Ap
                d["s_dot_r0star"].append(float(np.dot(s_vec, self.r0star)))
                d["s_norm"].append(float(np.linalg.norm(s_vec)))
            elif event == N.DBG_BICG_XRP:
                d["identity_rr"].append(sc[0])
                d["direct_rr"].append(float(np.dot(a0, a0)))
            elif event == N.DBG_GMRES_CYCLE:
                k = int(sc[0])
                v = np.ctypeslib.as_array(v0, shape=(k * n,)).reshape(k, n)
                vmat = np.stack([v[j].copy() for j in range(k)], axis=1)
                gram = vmat.T @ vmat
                d["ortho_offdiag"].append(float(np.abs(gram - np.eye(k)).max()))
            return 0
        except Exception as exc:  # surfaced after the native call returns
            self.error = exc
            return 1


def _prepare(a, b, x0):
    """Validation of solvers.py:259-269 (ValueError on misuse)."""
    if isinstance(a, DeviceMatrix):
        n_rows, n_cols = a.n_rows, a.n_cols
    else:
        a = CsrMatrix.coerce(a)
        n_rows, n_cols = a.n_rows, a.n_cols
    if n_rows != n_cols:
        raise ValueError(f"matrix must be square, got {n_rows} x {n_cols}")
    b = np.ascontiguousarray(as_vector(b, n=n_rows, name="b"), dtype=np.float64)
    x0 = None if x0 is None else np.ascontiguousarray(as_vector(x0, n=n_rows, name="x0"), dtype=np.float64)
    return a, b, x0


_PINNED: dict[int, list] = {}  # n -> page-locked float64 arrays (their owners)
_PINNED_KEEP = 4


def _host_empty(n: int) -> np.ndarray:
    """float64 host buffer for a solution: page-locked when a CUDA device is
    present (the device->host copy of x then runs at full DMA speed), else a
    plain NumPy array.  Page-locked arrays are recycled: one is handed out
    again only when nothing but this pool references it (no result, no view
    of it is alive) -- a fresh page-locked allocation costs ~0.3 ms."""
    try:
        import torch

        if not torch.cuda.is_available():
            return np.empty(n)
    except Exception:
        return np.empty(n)
    pool = _PINNED.setdefault(n, [])
    for i in range(len(pool)):
        if sys.getrefcount(pool[i]) == 2:  # the pool's reference + getrefcount's argument
            return pool[i]
    arr = torch.empty(max(n, 1), dtype=torch.float64, pin_memory=True).numpy()
    if n != arr.shape[0]:
        arr = np.empty(0)
    if len(pool) < _PINNED_KEEP:
        pool.append(arr)
    return arr


def host_array(n: int) -> np.ndarray:
    """A float64 host vector in page-locked memory, for right-hand sides that
    are streamed to the device every solve (full-speed DMA); see _host_empty."""
    return _host_empty(n)


def _native_config(cfg: SolverConfig) -> N.PkConfig:
    return N.PkConfig(
        tolerance=cfg.tolerance, max_iterations=cfg.max_iterations, restart=cfg.restart,
        breakdown_tolerance=cfg.breakdown_tolerance,
        fixed_iterations=cfg.fixed_iterations if cfg.fixed else 0,
        loop_mode=N.LOOP_GRAPH if cfg.loop_mode == "graph" else N.LOOP_HOST, flags=0)


def iteration_kernel_bytes(method: str, n: int, nnz: int, launches: int, step: int = 1) -> int:
    """Algorithmic HBM bytes of one iteration's kernels as the library issues
    them (int32 indices, fp64 values, every vector read/written once per
    kernel, a gathered vector counted once): B_CSR = 12 nnz + 4 (n + 1).

    CG: 1 kernel (OpCgFused) B_CSR + 64 n; 2 kernels (update sweep 56 n +
    OpCgApNext B_CSR + 24 n).  BiCGStab: 2 kernels (OpBicgB B_CSR + 32 n +
    OpBicgA B_CSR + 80 n); 3 kernels (OpBicgB + xrp sweep 64 n + OpBicgApNext
    B_CSR + 32 n).  GMRES step i: SpMV B_CSR + 16 n, multi-dot 8 n (i - 1)
    (i >= 3), GS update 8 n (i - 1) + 16 n (i >= 2), normalize 24 n."""
    bcsr = 12 * nnz + 4 * (n + 1)
    if method == "cg":
        return bcsr + 64 * n if launches <= 1 else bcsr + 80 * n
    if method == "bicgstab":
        return 2 * bcsr + (112 * n if launches <= 2 else 128 * n)
    i = step
    total = bcsr + 16 * n + 24 * n
    if i >= 2:
        total += 8 * n * (i - 1) + 16 * n
    if i >= 3:
        total += 8 * n * (i - 1)
    return total


def _trace_from(res: N.PkResult, method: str, n: int, restart: int, nnz: int = 0) -> ExecutionTrace:
    """ExecutionTrace filled with the launches/transfers really issued and
    the algorithmic bytes of those kernels (so the cost model prices both
    sides with the same terms; execmodel.py:227-278).

    GMRES step i of a cycle launches SpMV+normalize (i=1), SpMV+update+
    normalize (i=2) or SpMV+multi-dot+update+normalize (i>=3)."""
    tr = ExecutionTrace()
    tr.add_phase(SETUP, res.setup_launches, res.setup_transfers, bytes_kernel=(12 * nnz + 48 * n) if nnz else 0,
                 bytes_transfer=8 * 2 * n)
    # one record per iteration (the reference's trace layout); the per-step
    # values repeat with period 1 (CG, BiCGStab) or the restart (GMRES)
    period = restart if method == "gmres" else 1
    proto = []
    for step in range(1, min(period, max(res.iterations, 1)) + 1):
        launches = (2 if step == 1 else (3 if step == 2 else 4)) if method == "gmres" else res.launches_per_iteration
        kb = iteration_kernel_bytes(method, n, nnz, launches, step) if nnz else 0
        proto.append((int(launches), int(res.transfers_per_iteration), int(kb)))
    tr.phases.extend(PhaseRecord(ITERATION, *proto[i % period]) for i in range(res.iterations))
    for _ in range(res.check_phases):
        tr.add_phase(CHECK, 1, 1, bytes_kernel=(12 * nnz + 24 * n) if nnz else 0, bytes_transfer=8)
    tr.add_phase(FINISH, res.finish_launches, res.finish_transfers,
                 bytes_kernel=(12 * nnz + 24 * n) if nnz else 0, bytes_transfer=8 * (n + res.iterations))
    return tr


def _run(method: str, a, b, x0, config, context, debug):
    cfg = SolverConfig.coerce(config)
    if method == "gmres" and cfg.orthogonalization != CLASSICAL_GS:
        raise ValueError("pipelined GMRES supports classical Gram-Schmidt only")
    a, b, x0 = _prepare(a, b, x0)
    ctx = ExecutionContext.coerce(context)
    dc = context_for(ctx)
    dm = device_matrix(a, ctx)
    n = dm.n_rows
    limit = cfg.iteration_limit()
    x = _host_empty(n)
    hist = np.empty(max(limit, 1))
    res = N.PkResult()
    ncfg = _native_config(cfg)
    dp = C.POINTER(C.c_double)
    dc.reset_stream()
    dbg = _Diagnostics(method) if debug else None
    hook = N.DEBUG_FN(dbg) if debug else None
    if debug:
        N.check(N.lib().pk_ctx_set_debug(dc.handle, hook, None))
    try:
        rc = N.lib().pk_solve(
            dc.handle, dm.handle, N.METHODS[method], b.ctypes.data_as(dp),
            x0.ctypes.data_as(dp) if x0 is not None else None, C.byref(ncfg), _trisolve_cb, None,
            x.ctypes.data_as(dp), hist.ctypes.data_as(dp), len(hist), C.byref(res))
    finally:
        if debug:
            N.lib().pk_ctx_set_debug(dc.handle, N.DEBUG_FN(), None)
    if dbg is not None and dbg.error is not None:
        raise dbg.error
    N.check(rc, f"{method}_pipelined")
    trace = _trace_from(res, method, n, cfg.restart, dm.nnz)
    diag = dbg.diag if debug else {}
    return SolverResult(
        x=x,
        residual_history=hist[: res.iterations].tolist(),
        true_final_residual=float(res.true_final_residual),
        iterations=int(res.iterations),
        termination=N.TERM_NAMES[res.termination],
        trace=trace,
        breakdown_kind=N.KIND_NAMES[res.breakdown_kind],
        loop_seconds=float(res.loop_seconds),
        diagnostics=diag,
    )


def cg_pipelined(a, b, x0=None, config=None, context=None, debug=False) -> SolverResult:
    """Pipelined CG (solvers.py:395-469): below 2^20 rows ONE fused kernel per
    iteration (the vector update folded into the SpMV by recompute-at-gather),
    above it the update sweep + a one-gather SpMV (2 kernels, faster when
    bandwidth-bound); the stage-2 reduction and alpha/beta/convergence are
    finalized on the device either way."""
    return _run("cg", a, b, x0, config, context, debug)


def bicgstab_pipelined(a, b, x0=None, config=None, context=None, debug=False) -> SolverResult:
    """Pipelined BiCGStab (solvers.py:583-712): the s-update folded into the
    As-SpMV; below 2^20 rows the xrp update is also folded into the next
    iteration's Ap-SpMV (2 kernels per iteration), above it runs as a lean
    elementwise sweep before a one-gather Ap-SpMV (3 kernels; faster on B200).
    The reference emulates 4 launches + 1 transfer."""
    return _run("bicgstab", a, b, x0, config, context, debug)


def gmres_pipelined(a, b, x0=None, config=None, context=None, debug=False) -> SolverResult:
    """Pipelined GMRES(m) with fused classical Gram-Schmidt (solvers.py:865-1008)."""
    return _run("gmres", a, b, x0, config, context, debug)


SOLVERS = {
    ("cg", "pipelined"): cg_pipelined,
    ("bicgstab", "pipelined"): bicgstab_pipelined,
    ("gmres", "pipelined"): gmres_pipelined,
}


def solve(A, b, tag=("cg", "pipelined"), tol: float = 1e-8, maxiter: int = 500, x0=None, context=None,
          restart: int = 30, fixed_iterations: int | None = None) -> SolverResult:
    """North-star entry: ``SOLVERS[tag](A, b, x0, SolverConfig(tol, maxiter), context)``.

    ``tag`` is a (method, variant) pair or a bare method name."""
    if isinstance(tag, str):
        tag = (tag, "pipelined")
    if tuple(tag) not in SOLVERS:
        raise ValueError(f"unknown solver {tag!r}; the B200 path implements {sorted(SOLVERS)}")
    cfg = SolverConfig(tolerance=tol, max_iterations=maxiter, restart=restart, fixed_iterations=fixed_iterations)
    return SOLVERS[tuple(tag)](A, b, x0=x0, config=cfg, context=context)


def solve_resident(method: str, a, b, x0=None, config=None, context=None, profile: bool = False):
    """HBM-resident solve: ``a`` a DeviceMatrix (or CsrMatrix, uploaded once),
    ``b``/``x0`` float64 CUDA tensors; returns (x tensor, SolverResult without
    a host copy of x).  No host<->device vector traffic besides the history --
    the entry the benchmark times (pk_solve_device).

    ``profile=True`` (needs ``loop_mode="host"``) brackets every loop kernel
    with CUDA events; the per-kernel times land in
    ``diagnostics["kernel_seconds"]`` / ``["kernel_launches"]``."""
    import torch

    cfg = SolverConfig.coerce(config)
    if method == "gmres" and cfg.orthogonalization != CLASSICAL_GS:
        raise ValueError("pipelined GMRES supports classical Gram-Schmidt only")
    ctx = ExecutionContext.coerce(context)
    dc = context_for(ctx)
    dm = device_matrix(a, ctx)
    n = dm.n_rows
    if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dtype == torch.float64 and b.shape == (n,)):
        raise ValueError("b must be a float64 CUDA tensor of length n")
    b = b.contiguous()
    x = torch.empty_like(b)
    hist = np.empty(max(cfg.iteration_limit(), 1))
    res = N.PkResult()
    ncfg = _native_config(cfg)
    if profile:
        if cfg.loop_mode != "host":
            raise ValueError("kernel profiling needs loop_mode='host'")
        ncfg.flags = N.FLAG_PROFILE
    x0p = None
    if x0 is not None:
        x0 = x0.contiguous()
        x0p = C.c_void_p(x0.data_ptr())
    dc.reset_stream()
    N.check(N.lib().pk_solve_device(
        dc.handle, dm.handle, N.METHODS[method], C.c_void_p(b.data_ptr()), x0p, C.byref(ncfg), _trisolve_cb,
        None, C.c_void_p(x.data_ptr()), hist.ctypes.data_as(C.POINTER(C.c_double)), len(hist), C.byref(res)),
        f"{method}_pipelined")
    result = SolverResult(
        x=None, residual_history=[float(v) for v in hist[: res.iterations]],
        true_final_residual=float(res.true_final_residual), iterations=int(res.iterations),
        termination=N.TERM_NAMES[res.termination], trace=_trace_from(res, method, n, cfg.restart, dm.nnz),
        breakdown_kind=N.KIND_NAMES[res.breakdown_kind], loop_seconds=float(res.loop_seconds),
        diagnostics={"launches": res.total_launches, "launches_per_iteration": res.launches_per_iteration,
                     "kernel_seconds": [float(v) for v in res.kernel_seconds],
                     "kernel_launches": [int(v) for v in res.kernel_launches]})
    return x, result


def solve_batch(systems, tag=("cg", "pipelined"), config=None, context=None, threads: int = 16):
    """Transient batch (BASELINE configs[4]): independent systems ``[(A, b)]``
    or ``[(A, b, x0)]`` solved with the same driver and config, no
    communication.  ``threads`` host workers (each with its own CUDA stream)
    overlap the device-resident solves; every result is bit-identical to
    ``SOLVERS[tag](A, b, x0, config, context)`` on its own.  Matrices are
    uploaded once per object.  Returns a list of :class:`SolverResult`."""
    if isinstance(tag, str):
        tag = (tag, "pipelined")
    if tuple(tag) not in SOLVERS:
        raise ValueError(f"unknown solver {tag!r}; the B200 path implements {sorted(SOLVERS)}")
    if tag[1] != "pipelined":
        # the batch runs the native pipelined drivers; a classical tag would
        # silently get different rounding and a different trace
        raise ValueError(f"solve_batch runs the pipelined drivers only, got {tag!r}")
    method = tag[0]
    cfg = SolverConfig.coerce(config)
    if method == "gmres" and cfg.orthogonalization != CLASSICAL_GS:
        raise ValueError("pipelined GMRES supports classical Gram-Schmidt only")
    ctx = ExecutionContext.coerce(context)
    dc = context_for(ctx)
    systems = list(systems)
    nsys = len(systems)
    mats, bs, x0s, xs, hists = [], [], [], [], []
    limit = cfg.iteration_limit()
    for item in systems:
        a, b = item[0], item[1]
        x0 = item[2] if len(item) > 2 else None
        a, b, x0 = _prepare(a, b, x0)
        dm = device_matrix(a, ctx)
        mats.append(dm)
        bs.append(b)
        x0s.append(x0)
        xs.append(np.empty(dm.n_rows))
        hists.append(np.empty(max(limit, 1)))
    P = C.c_void_p
    dp = lambda v: C.cast(v.ctypes.data, P) if v is not None else None
    mat_arr = (P * max(nsys, 1))(*[m.handle for m in mats])
    b_arr = (P * max(nsys, 1))(*[dp(v) for v in bs])
    x0_arr = (P * max(nsys, 1))(*[dp(v) for v in x0s])
    x_arr = (P * max(nsys, 1))(*[dp(v) for v in xs])
    h_arr = (P * max(nsys, 1))(*[dp(v) for v in hists])
    res = (N.PkResult * max(nsys, 1))()
    ncfg = _native_config(cfg)
    dc.reset_stream()
    N.check(N.lib().pk_solve_batch(dc.handle, nsys, mat_arr, N.METHODS[method], b_arr, x0_arr, C.byref(ncfg),
                                   _trisolve_cb, None, x_arr, h_arr, max(limit, 1), res, int(threads)),
            f"{method}_pipelined batch")
    out = []
    for i in range(nsys):
        r = res[i]
        out.append(SolverResult(
            x=xs[i], residual_history=[float(v) for v in hists[i][: r.iterations]],
            true_final_residual=float(r.true_final_residual), iterations=int(r.iterations),
            termination=N.TERM_NAMES[r.termination], trace=_trace_from(r, method, mats[i].n_rows, cfg.restart, mats[i].nnz),
            breakdown_kind=N.KIND_NAMES[r.breakdown_kind], loop_seconds=float(r.loop_seconds), diagnostics={}))
    return out


def launch_floor(context=None, kernels_per_iteration: int = 1, grid: int = 0, iterations: int = 2000) -> dict:
    """Measured floor of the device-resident loop: microseconds per iteration
    of a conditional-WHILE graph with `kernels_per_iteration` empty gated
    full-width kernels (ticket + WHILE-condition protocol of the solvers)."""
    ctx = ExecutionContext.coerce(context)
    dc = context_for(ctx)
    us = C.c_double()
    N.check(N.lib().pk_launch_floor(dc.handle, int(kernels_per_iteration), int(grid), int(iterations),
                                    C.byref(us)), "pk_launch_floor")
    return {"us_per_iteration": us.value, "kernels_per_iteration": kernels_per_iteration,
            "note": f"{kernels_per_iteration} empty gated kernel(s) of {grid or '4 x SM'} CTAs per iteration in the "
                    "unrolled conditional-WHILE graph, ticket + condition as in the solver finalizers"}
