"""Kernel-level entry points on CUDA tensors -- the B200 counterparts of the
reference's emulated fused kernels (pipekrylov/fused.py) and reductions
(pipekrylov/linalg.py:323-380).

Vectors are float64 CUDA ``torch.Tensor``s (torch is only the device-memory
plumbing; all arithmetic happens in libpk_b200.so).  Each call is one (or,
where the reference finalizes a scalar in-kernel, two) kernel launch on the
current torch stream.  Partials come back as (n_groups, n_quantities)
tensors, bit-identical to the reference's ``WorkgroupPartials.data``.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from .device import DeviceMatrix, context_for, device_matrix
from .linalg import ExecutionContext
from .solvers import BreakdownError, LuckyBreakdown

WITH_INPUT = "input"
WITH_RESULT = "result"


class FusedReductionRequest:
    """Inner products accumulated alongside a fused SpMV (fused.py:55-83):
    each quantity is "input" (<q,p>), "result" (<q,q>) or a fixed vector w
    (<q,w>, here a float64 CUDA tensor); 1 to 4 quantities per kernel."""

    MAX_QUANTITIES = 4

    def __init__(self, quantities):
        quantities = tuple(quantities)
        if not 1 <= len(quantities) <= self.MAX_QUANTITIES:
            raise ValueError(f"request must carry 1 to {self.MAX_QUANTITIES} quantities, got {len(quantities)}")
        for q in quantities:
            if isinstance(q, str) and q not in (WITH_INPUT, WITH_RESULT):
                raise ValueError(f"unknown quantity kind {q!r}")
        self.quantities = quantities

    def __len__(self) -> int:
        return len(self.quantities)

    def __iter__(self):
        return iter(self.quantities)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() else None


def _dc(ctx, like=None):
    ctx = ExecutionContext.coerce(ctx)
    dc = context_for(ctx)
    dc.set_stream(torch.cuda.current_stream(ctx.device))
    return ctx, dc


def _vec(t, n, name):
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or t.dim() != 1:
        raise ValueError(f"{name} must be a 1-D float64 CUDA tensor")
    if t.shape[0] != n:
        raise ValueError(f"{name} has length {t.shape[0]}, expected {n}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _partials(ctx, nq, device):
    return torch.empty((ctx.n_groups, nq), dtype=torch.float64, device=device)


def spmv_csr(a, p, ctx=None):
    """q = A p (spmv_csr, linalg.py:373-380)."""
    ctx, dc = _dc(ctx)
    dm = device_matrix(a, ctx)
    p = _vec(p, dm.n_cols, "p")
    q = torch.empty(dm.n_rows, dtype=torch.float64, device=p.device)
    N.check(N.lib().pk_spmv(dc.handle, dm.handle, _ptr(p), _ptr(q)))
    return q


def spmv_fused(a, p, quantities, ctx=None):
    """q = A p plus stage-1 partials of 1-4 dots (fused.py:86-120).

    ``quantities`` entries: "input" (<q,p>), "result" (<q,q>) or a CUDA
    vector w (<q,w>)."""
    ctx, dc = _dc(ctx)
    dm = device_matrix(a, ctx)
    p = _vec(p, dm.n_cols, "p")
    quantities = tuple(FusedReductionRequest(quantities))
    if WITH_INPUT in [q for q in quantities if isinstance(q, str)] and dm.n_rows != dm.n_cols:
        raise ValueError("result-with-input dot needs a square matrix")
    kinds = (C.c_int32 * 4)()
    ws = (C.c_void_p * 4)()
    keep = []
    for i, qk in enumerate(quantities):
        if isinstance(qk, str):
            if qk not in (WITH_INPUT, WITH_RESULT):
                raise ValueError(f"unknown quantity kind {qk!r}")
            kinds[i] = N.DOT_INPUT if qk == WITH_INPUT else N.DOT_RESULT
        else:
            w = _vec(qk, dm.n_rows, "fixed dot vector")
            keep.append(w)
            kinds[i] = N.DOT_VECTOR
            ws[i] = w.data_ptr()
    q = torch.empty(dm.n_rows, dtype=torch.float64, device=p.device)
    part = _partials(ctx, len(quantities), p.device)
    N.check(N.lib().pk_spmv_fused(dc.handle, dm.handle, _ptr(p), _ptr(q), len(quantities), kinds, ws,
                                  _ptr(part)))
    return q, part


def reduce_stage1(columns, ctx=None):
    """Stage-1 partials of one or several contribution streams (linalg.py:323-337)."""
    ctx, dc = _dc(ctx)
    if isinstance(columns, torch.Tensor) and columns.dim() == 1:
        columns = [columns]
    elif isinstance(columns, torch.Tensor):
        columns = [columns[:, j].contiguous() for j in range(columns.shape[1])]
    cols = [c.contiguous() for c in columns]
    n = cols[0].shape[0]
    for c in cols:
        _vec(c, n, "contribution column")
    arr = (C.c_void_p * len(cols))(*[c.data_ptr() if c.numel() else None for c in cols])
    part = _partials(ctx, len(cols), cols[0].device)
    N.check(N.lib().pk_reduce_stage1(dc.handle, n, len(cols), arr, _ptr(part)))
    return part


def reduce_stage2(partials, ctx=None):
    """Serial sum over groups, on the device (linalg.py:311-320, 340-348)."""
    ctx, dc = _dc(ctx)
    part = partials.contiguous()
    if part.dim() != 2 or part.shape[0] != ctx.n_groups:
        raise ValueError("partials must be (n_groups, n_quantities)")
    out = torch.empty(part.shape[1], dtype=torch.float64, device=part.device)
    N.check(N.lib().pk_reduce_stage2(dc.handle, part.shape[1], _ptr(part), _ptr(out)))
    return out


def dot(x, y, ctx=None) -> float:
    """Two-stage inner product (linalg.py:351-365)."""
    ctx, dc = _dc(ctx)
    n = x.shape[0]
    _vec(x, n, "x"), _vec(y, n, "y")
    out = torch.empty(1, dtype=torch.float64, device=x.device)
    N.check(N.lib().pk_dot(dc.handle, n, _ptr(x), _ptr(y), _ptr(out)))
    return float(out.item())


def fused_cg_vector_update(x, r, p, Ap, alpha, beta, ctx=None):
    """x += a p; r -= a Ap; p = b p + r; <r,r> partials (fused.py:123-151)."""
    ctx, dc = _dc(ctx)
    n = x.shape[0]
    for t, nm in ((x, "x"), (r, "r"), (p, "p"), (Ap, "Ap")):
        _vec(t, n, nm)
    part = _partials(ctx, 1, x.device)
    N.check(N.lib().pk_cg_update(dc.handle, n, _ptr(x), _ptr(r), _ptr(p), _ptr(Ap), float(alpha), float(beta),
                                 _ptr(part)))
    return part


def fused_bicgstab_s_update(r, Ap, rr0_partials, Apr0_partials, ctx=None, breakdown_tolerance=1e-30):
    """alpha finalized on the device; s = r - alpha Ap; <s,s> (fused.py:154-182)."""
    ctx, dc = _dc(ctx)
    n = r.shape[0]
    _vec(r, n, "r"), _vec(Ap, n, "Ap")
    s = torch.empty_like(r)
    part = _partials(ctx, 1, r.device)
    alpha = torch.empty(1, dtype=torch.float64, device=r.device)
    flag = torch.zeros(1, dtype=torch.int32, device=r.device)
    N.check(N.lib().pk_bicg_s_update(dc.handle, n, _ptr(r), _ptr(Ap), _ptr(rr0_partials.contiguous()),
                                     _ptr(Apr0_partials.contiguous()), float(breakdown_tolerance), _ptr(s),
                                     _ptr(part), _ptr(alpha), _ptr(flag)))
    if int(flag.item()):
        raise BreakdownError("Apr0star")
    return s, part, float(alpha.item())


def fused_bicgstab_xrp_update(x, r, p, s, Ap, As, alpha, omega, beta, r0star, ctx=None):
    """x += a p + w s; r = s - w As; p = b (p - w Ap) + r; <r,r0*> (fused.py:185-219)."""
    ctx, dc = _dc(ctx)
    n = x.shape[0]
    for t, nm in ((x, "x"), (r, "r"), (p, "p"), (s, "s"), (Ap, "Ap"), (As, "As"), (r0star, "r0star")):
        _vec(t, n, nm)
    part = _partials(ctx, 1, x.device)
    N.check(N.lib().pk_bicg_xrp_update(dc.handle, n, _ptr(x), _ptr(r), _ptr(p), _ptr(s), _ptr(Ap), _ptr(As),
                                       float(alpha), float(omega), float(beta), _ptr(r0star), _ptr(part)))
    return part


def _basis_array(basis, n):
    for b in basis:
        _vec(b, n, "basis vector")
    return (C.c_void_p * max(len(basis), 1))(*[b.data_ptr() for b in basis])


def fused_gs_stage1(basis, v, ctx=None):
    """Partials of <b_j, v> for every basis vector, one launch (fused.py:222-243)."""
    ctx, dc = _dc(ctx)
    n = v.shape[0]
    _vec(v, n, "v")
    part = _partials(ctx, len(basis), v.device)
    if basis:
        N.check(N.lib().pk_gs_stage1(dc.handle, n, len(basis), _basis_array(basis, n), _ptr(v), _ptr(part)))
    return part


def fused_gs_update(v, basis, partials, ctx=None):
    """coeffs = stage2(partials); v -= sum_j c_j b_j; <v,v> partials (fused.py:246-277)."""
    ctx, dc = _dc(ctx)
    n = v.shape[0]
    _vec(v, n, "v")
    if len(basis) != partials.shape[1]:
        raise ValueError(f"{len(basis)} basis vectors but partials carry {partials.shape[1]} quantities")
    coeffs = torch.zeros(max(len(basis), 1), dtype=torch.float64, device=v.device)
    npart = _partials(ctx, 1, v.device)
    N.check(N.lib().pk_gs_update(dc.handle, n, _ptr(v), len(basis), _basis_array(basis, n),
                                 _ptr(partials.contiguous()), _ptr(coeffs), _ptr(npart)))
    return coeffs[: len(basis)], npart


def fused_gs_normalize(v, norm_partials, r, ctx=None, breakdown_tolerance=1e-30):
    """||v|| finalized on the device; v *= 1/||v||; <r,v> partials (fused.py:280-305)."""
    ctx, dc = _dc(ctx)
    n = v.shape[0]
    _vec(v, n, "v"), _vec(r, n, "r")
    norm = torch.empty(1, dtype=torch.float64, device=v.device)
    flag = torch.zeros(1, dtype=torch.int32, device=v.device)
    part = _partials(ctx, 1, v.device)
    N.check(N.lib().pk_gs_normalize(dc.handle, n, _ptr(v), _ptr(norm_partials.contiguous()), _ptr(r),
                                    float(breakdown_tolerance), _ptr(norm), _ptr(flag), _ptr(part)))
    if int(flag.item()):
        raise LuckyBreakdown(float(norm.item()))
    return float(norm.item()), part


spmv = spmv_csr
