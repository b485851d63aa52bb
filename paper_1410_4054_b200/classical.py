"""Classical (unfused) CG, BiCGStab and GMRES(m) on B200 -- the paper's baseline.

Same drivers as the reference's ``SOLVERS[(method, "classical")]``
(solvers.py:310-389, 485-580, 725-858): one kernel per BLAS operation and a
host round trip per inner product (the scalar recurrences run here, in
Python binary64, exactly as the reference writes them).  Every kernel is a
libpk_b200.so launch -- ``pk_spmv`` (linalg.py:373-380), ``pk_dot``
(two-stage reduction at the context geometry, linalg.py:351-365) and
``pk_vec_update`` (axpy / axpy2 / xpay / scale / add_scaled / the BiCGStab
p update / copy, linalg.py:403-457, solvers.py:277-280, 477-482) -- so the
results are bit-identical to the reference's classical drivers at the same
``ExecutionContext``; there is no CPU fallback.

Running both formulations on the same B200 reproduces the paper's central
comparison (PAPER.md: pipelined >= 2-3x faster in the latency regime): the
classical loop issues 6 (CG) / 13 (BiCGStab) launches and 2 / 7 host reads per
iteration, the pipelined one 1-3 graph-resident launches and none.
"""

from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np
import torch

from . import _native as N
from .device import context_for, device_matrix
from .linalg import FINISH, ITERATION, SETUP, ExecutionContext, ExecutionTrace
from .solvers import (BREAKDOWN, CONVERGED, LUCKY_BREAKDOWN, MAX_ITER, MODIFIED_GS, BreakdownError, SolverConfig,
                      SolverResult, UpperTriangular, _prepare, solve_upper_triangular)


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


class _Device:
    """Kernel-per-operation BLAS on one context, with the reference's trace
    bookkeeping (real launches: a dot is stage 1 + stage 2, then one read)."""

    def __init__(self, a, ctx: ExecutionContext, trace: ExecutionTrace):
        self.ctx = ctx
        self.dc = context_for(ctx)
        self.dm = device_matrix(a, ctx)
        self.n = self.dm.n_rows
        self.dev = torch.device("cuda", ctx.device)
        self.trace = trace
        self.stream = torch.cuda.current_stream(self.dev)
        self.dc.set_stream(self.stream)
        self.lib = N.lib()
        self._tot = torch.empty(1, dtype=torch.float64, device=self.dev)

    def empty(self):
        return torch.empty(self.n, dtype=torch.float64, device=self.dev)

    def upload(self, v: np.ndarray):
        t = self.empty()
        t.copy_(torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)))
        return t

    def spmv(self, p):
        q = self.empty()
        N.check(self.lib.pk_spmv(self.dc.handle, self.dm.handle, _p(p), _p(q)), "spmv")
        self.trace.record_launch(8 * (2 * self.dm.nnz + 2 * self.n + 1))
        return q

    def dot(self, x, y) -> float:
        N.check(self.lib.pk_dot(self.dc.handle, self.n, _p(x), _p(y), _p(self._tot)), "dot")
        self.trace.record_launch(16 * self.n)
        self.trace.record_launch()
        self.trace.record_transfer(8)
        return float(self._tot.item())

    def vec(self, kind, y, x=None, z=None, alpha=0.0, beta=0.0):
        N.check(self.lib.pk_vec_update(self.dc.handle, kind, self.n, _p(y), _p(x), _p(z), float(alpha),
                                       float(beta)), "vector update")
        self.trace.record_launch(8 * 3 * self.n)
        return y

    # linalg.py / solvers.py helpers by name
    def axpy(self, y, alpha, x):
        return self.vec(N.VEC_AXPY, y, x, None, alpha)

    def axpy2(self, y, alpha, x, beta, z):
        return self.vec(N.VEC_AXPY2, y, x, z, alpha, beta)

    def xpay(self, y, x, beta):
        return self.vec(N.VEC_XPAY, y, x, None, 0.0, beta)

    def scale(self, y, alpha):
        return self.vec(N.VEC_SCALE, y, None, None, alpha)

    def add_scaled(self, x, alpha, z):
        return self.vec(N.VEC_ADD_SCALED, self.empty(), x, z, alpha)

    def copy(self, v):
        return self.vec(N.VEC_COPY, self.empty(), v)

    def bicg_p(self, p, r, beta, omega, ap):
        return self.vec(N.VEC_BICG_P, p, r, ap, beta, omega)


def _begin(a, b, x0, config, context):
    cfg = SolverConfig.coerce(config)
    a, b, x0 = _prepare(a, b, x0)
    ctx = ExecutionContext.coerce(context)
    trace = ExecutionTrace()
    d = _Device(a, ctx, trace)
    x = d.upload(x0) if x0 is not None else torch.zeros(d.n, dtype=torch.float64, device=d.dev)
    return cfg, d, d.upload(b), x, trace


def _result(d, b, x, trace, history, termination, kind, loop_seconds, diag):
    """solvers.py:283-302: the true residual is part of FINISH."""
    with trace.phase(FINISH):
        q = d.spmv(x)
        res = d.add_scaled(b, -1.0, q)
        true_norm = math.sqrt(d.dot(res, res))
        xh = x.cpu().numpy()
        trace.record_transfer(8 * d.n)
    return SolverResult(x=xh, residual_history=history, true_final_residual=true_norm, iterations=len(history),
                        termination=termination, trace=trace, breakdown_kind=kind, loop_seconds=loop_seconds,
                        diagnostics=diag)


def cg_classical(a, b, x0=None, config=None, context=None, debug=False) -> SolverResult:
    """Conjugate Gradient, one kernel per BLAS operation (solvers.py:310-389)."""
    cfg, d, b, x, trace = _begin(a, b, x0, config, context)
    btol = cfg.loop_breakdown_tolerance()
    diag: dict = {"rr_direct": [], "beta": []} if debug else {}
    with trace.phase(SETUP):
        norm_b = math.sqrt(d.dot(b, b))
        scale_ = norm_b if norm_b > 0 else 1.0
        q0 = d.spmv(x)
        r = d.add_scaled(b, -1.0, q0)
        p = d.copy(r)
        rr = d.dot(r, r)
    if debug:
        diag["rr_direct"].append(float(torch.dot(r, r)))
    history: list[float] = []
    termination, kind = MAX_ITER, None
    entry = math.sqrt(rr) / scale_
    if entry <= cfg.tolerance and (not cfg.fixed or rr == 0.0):
        return _result(d, b, x, trace, history, CONVERGED, kind, 0.0, diag)
    t0 = time.perf_counter()
    for _ in range(cfg.iteration_limit()):
        with trace.phase(ITERATION):
            q = d.spmv(p)
            pap = d.dot(p, q)
            if abs(pap) < btol:
                termination, kind = BREAKDOWN, "pAp"
                break
            if pap == 0.0:  # ZeroDivisionError in the reference (fixed mode)
                termination, kind = BREAKDOWN, "pAp"
                break
            alpha = rr / pap
            d.axpy(x, alpha, p)
            d.axpy(r, -alpha, q)
            rr_new = d.dot(r, r)
            if debug:
                diag["rr_direct"].append(float(torch.dot(r, r)))
            monitored = math.sqrt(rr_new) / scale_
            history.append(monitored)
            if not math.isfinite(monitored):
                termination, kind = BREAKDOWN, "divergence"
                break
            if not cfg.fixed and monitored <= cfg.tolerance:
                termination = CONVERGED
                break
            beta = rr_new / rr
            if debug:
                diag["beta"].append(float(beta))
            d.xpay(p, r, beta)
            rr = rr_new
    torch.cuda.synchronize(d.dev)
    loop_seconds = time.perf_counter() - t0
    return _result(d, b, x, trace, history, termination, kind, loop_seconds, diag)


def bicgstab_classical(a, b, x0=None, config=None, context=None, debug=False) -> SolverResult:
    """BiCGStab, one kernel per BLAS operation (solvers.py:485-580); the
    direction coefficient through beta = -<As, r0*> / <Ap, r0*>."""
    cfg, d, b, x, trace = _begin(a, b, x0, config, context)
    btol = cfg.loop_breakdown_tolerance()
    diag: dict = {"s_dot_r0star": [], "s_norm": [], "direct_rr": []} if debug else {}
    with trace.phase(SETUP):
        norm_b = math.sqrt(d.dot(b, b))
        scale_ = norm_b if norm_b > 0 else 1.0
        q0 = d.spmv(x)
        r = d.add_scaled(b, -1.0, q0)
        r0star = d.copy(r)
        p = d.copy(r)
        rr = d.dot(r, r)
        rho = d.dot(r, r0star)
    if debug:
        diag["r0star_norm"] = float(torch.linalg.norm(r0star))
    history: list[float] = []
    termination, kind = MAX_ITER, None
    entry = math.sqrt(rr) / scale_
    if entry <= cfg.tolerance and (not cfg.fixed or rr == 0.0):
        return _result(d, b, x, trace, history, CONVERGED, kind, 0.0, diag)
    t0 = time.perf_counter()
    for _ in range(cfg.iteration_limit()):
        with trace.phase(ITERATION):
            ap = d.spmv(p)
            apr = d.dot(ap, r0star)
            if abs(apr) < btol or apr == 0.0:
                termination, kind = BREAKDOWN, "Apr0star"
                break
            alpha = rho / apr
            s = d.add_scaled(r, -alpha, ap)
            ss = d.dot(s, s)
            if debug:
                diag["s_dot_r0star"].append(float(torch.dot(s, r0star)))
                diag["s_norm"].append(float(torch.linalg.norm(s)))
            monitored_s = math.sqrt(ss) / scale_
            if not cfg.fixed and monitored_s <= cfg.tolerance:
                d.axpy(x, alpha, p)
                history.append(monitored_s)
                termination = CONVERGED
                break
            as_ = d.spmv(s)
            ass = d.dot(as_, s)
            asas = d.dot(as_, as_)
            asr = d.dot(as_, r0star)
            if asas < btol or asas == 0.0:
                termination, kind = BREAKDOWN, "AsAs"
                break
            omega = ass / asas
            d.axpy2(x, alpha, p, omega, s)
            r = d.add_scaled(s, -omega, as_)
            rho_new = d.dot(r, r0star)
            rr = d.dot(r, r)
            if debug:
                diag["direct_rr"].append(float(rr))
            monitored = math.sqrt(rr) / scale_
            history.append(monitored)
            if not math.isfinite(monitored):
                termination, kind = BREAKDOWN, "divergence"
                break
            if not cfg.fixed and monitored <= cfg.tolerance:
                termination = CONVERGED
                break
            if abs(rho_new) < btol:
                termination, kind = BREAKDOWN, "rho"
                break
            if abs(omega) < btol:
                termination, kind = BREAKDOWN, "omega"
                break
            beta = -asr / apr
            d.bicg_p(p, r, beta, omega, ap)
            rho = rho_new
    torch.cuda.synchronize(d.dev)
    loop_seconds = time.perf_counter() - t0
    return _result(d, b, x, trace, history, termination, kind, loop_seconds, diag)


def orthogonalize_mgs(d: _Device, basis, v) -> np.ndarray:
    """Modified Gram-Schmidt sweep (solvers.py:221-237)."""
    coeffs = np.zeros(len(basis))
    for j, q in enumerate(basis):
        coeffs[j] = d.dot(q, v)
        d.axpy(v, -coeffs[j], q)
    return coeffs


def _orthogonalize_cgs(d: _Device, basis, v) -> np.ndarray:
    """Classical Gram-Schmidt against the unmodified v (solvers.py:240-251)."""
    coeffs = np.zeros(len(basis))
    for j, q in enumerate(basis):
        coeffs[j] = d.dot(q, v)
    for j, q in enumerate(basis):
        d.axpy(v, -coeffs[j], q)
    return coeffs


def gmres_classical(a, b, x0=None, config=None, context=None, debug=False) -> SolverResult:
    """Restarted GMRES on a QR of the Krylov directions (solvers.py:725-858):
    CGS or MGS per the config, xi_i projections, host triangular solve."""
    cfg, d, b, x, trace = _begin(a, b, x0, config, context)
    btol = cfg.loop_breakdown_tolerance()
    diag: dict = {"ortho_offdiag": []} if debug else {}
    m = cfg.restart
    history: list[float] = []
    termination, kind = MAX_ITER, None
    limit = cfg.iteration_limit()
    total = 0
    norm_b = None
    scale_ = 1.0
    loop_seconds = 0.0
    done = False
    while not done and total < limit:
        with trace.phase(SETUP):
            if norm_b is None:
                norm_b = math.sqrt(d.dot(b, b))
                scale_ = norm_b if norm_b > 0 else 1.0
            q0 = d.spmv(x)
            r = d.add_scaled(b, -1.0, q0)
            rho = math.sqrt(d.dot(r, r))
            start_ok = rho > 0 and not (not cfg.fixed and rho / scale_ <= cfg.tolerance)
            if start_ok:
                d.scale(r, 1.0 / rho)
        if not start_ok:
            termination = CONVERGED
            break
        basis: list = []
        rmat = UpperTriangular(m)
        xi: list[float] = []
        est2 = 1.0
        lucky = False
        converged_in_cycle = False
        t0 = time.perf_counter()
        while len(basis) < m and total < limit:
            i = len(basis) + 1
            with trace.phase(ITERATION):
                v_in = basis[-1] if basis else r
                w = d.spmv(v_in)
                if cfg.orthogonalization == MODIFIED_GS:
                    coeffs = orthogonalize_mgs(d, basis, w)
                else:
                    coeffs = _orthogonalize_cgs(d, basis, w)
                for j, c in enumerate(coeffs):
                    rmat.set(j, i - 1, float(c))
                nrm = math.sqrt(d.dot(w, w))
                if nrm < btol:
                    lucky = True
                    break
                if nrm == 0.0:  # ZeroDivisionError in the reference (fixed mode)
                    lucky = True
                    break
                rmat.set(i - 1, i - 1, nrm)
                d.scale(w, 1.0 / nrm)
                basis.append(w)
                xi_i = d.dot(r, w)
                xi.append(xi_i)
                d.axpy(r, -xi_i, w)
                est2 = max(est2 - xi_i * xi_i, 0.0)
                monitored = rho * math.sqrt(est2) / scale_
                history.append(monitored)
                total += 1
                if not math.isfinite(monitored):
                    termination, kind = BREAKDOWN, "divergence"
                    done = True
                    break
                if not cfg.fixed and monitored <= cfg.tolerance:
                    converged_in_cycle = True
                    break
        torch.cuda.synchronize(d.dev)
        loop_seconds += time.perf_counter() - t0
        k = len(basis)
        gate_true = None
        if k > 0 and termination != BREAKDOWN:
            with trace.phase(FINISH):
                try:
                    eta = solve_upper_triangular(rmat.leading(k), np.asarray(xi), cfg.breakdown_tolerance)
                except BreakdownError as err:
                    termination, kind = BREAKDOWN, err.kind
                    done = True
                    eta = None
                if eta is not None:
                    # update = eta0 r; update += coeff v; x += rho update (NumPy order)
                    update = d.copy(r)
                    d.scale(update, eta[0])
                    for idx in range(1, k + 1):
                        coeff = (eta[idx] if idx < k else 0.0) + eta[0] * xi[idx - 1]
                        d.axpy(update, coeff, basis[idx - 1])
                    d.axpy(x, rho, update)
                    if converged_in_cycle or lucky:
                        q = d.spmv(x)
                        res = d.add_scaled(b, -1.0, q)
                        gate_true = math.sqrt(d.dot(res, res))
        if debug and k > 0:
            vmat = torch.stack(basis, dim=1)
            gram = vmat.T @ vmat
            diag["ortho_offdiag"].append(float((gram - torch.eye(k, dtype=gram.dtype, device=gram.device)).abs().max()))
        if termination == BREAKDOWN:
            pass
        elif converged_in_cycle or lucky:
            if gate_true is not None and gate_true <= cfg.tolerance * scale_:
                termination = CONVERGED
                done = True
            elif lucky and k == 0:
                termination = LUCKY_BREAKDOWN
                done = True
    return _result(d, b, x, trace, history, termination, kind, loop_seconds, diag)
