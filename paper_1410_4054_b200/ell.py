"""ELLPACK storage and its SpMV on B200.

Mirrors the reference's ``EllMatrix`` / ``csr_to_ell`` / ``ell_to_csr`` /
``spmv_ell`` (linalg.py:179-246, 383-390): ``width`` slots per row stored
column-major (slot k of row i at ``i + k * n_rows``), padded slots holding the
sentinel column ``n_cols`` and value 0.  That layout is what a thread-per-row
GPU kernel wants: slot k of 32 consecutive rows is 32 consecutive words, so
every load of ``k_spmv_ell`` is coalesced without relying on L1 reuse.  The
kernel skips padded slots instead of multiplying by zero, so the row sums are
bit-identical to the CSR product (the reference's ELL = CSR contract,
test_linalg.py:119-137).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .device import context_for
from .linalg import CsrMatrix, ExecutionContext


@dataclass(frozen=True, eq=False)
class EllMatrix:
    """ELLPACK matrix (linalg.py:179-218): validated like the reference."""

    n_rows: int
    n_cols: int
    width: int
    col_indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "col_indices", np.asarray(self.col_indices, dtype=np.int64))
        object.__setattr__(self, "values", np.asarray(self.values, dtype=np.float64))
        if min(self.n_rows, self.n_cols, self.width) < 0:
            raise ValueError("matrix dimensions must be non-negative")
        total = self.n_rows * self.width
        if self.col_indices.shape != (total,) or self.values.shape != (total,):
            raise ValueError(f"col_indices and values must have {total} entries")
        if total:
            if self.col_indices.min() < 0 or self.col_indices.max() > self.n_cols:
                raise ValueError("column index out of range")
            if np.any(self.values[self.col_indices == self.n_cols] != 0.0):
                raise ValueError("padded slots must store value 0")

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    @property
    def nnz(self) -> int:
        return int(np.count_nonzero(self.col_indices != self.n_cols))


def csr_to_ell(a: CsrMatrix) -> EllMatrix:
    """CSR -> ELLPACK with width = the longest row (linalg.py:221-232);
    vectorised: entry e of row i goes to slot (e - row_offsets[i])."""
    a = CsrMatrix.coerce(a)
    counts = a.row_nnz()
    width = int(counts.max()) if a.n_rows else 0
    cols = np.full(a.n_rows * width, a.n_cols, dtype=np.int64)
    vals = np.zeros(a.n_rows * width)
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), counts)
    slot = np.arange(a.nnz, dtype=np.int64) - a.row_offsets[rows]
    cols[rows + slot * a.n_rows] = a.col_indices
    vals[rows + slot * a.n_rows] = a.values
    return EllMatrix(a.n_rows, a.n_cols, width, cols, vals)


def ell_to_csr(e: EllMatrix) -> CsrMatrix:
    """Drop the padding and rebuild canonical CSR (linalg.py:235-246)."""
    grid_cols = e.col_indices.reshape(e.width, e.n_rows).T  # [row][slot]
    grid_vals = e.values.reshape(e.width, e.n_rows).T
    keep = grid_cols != e.n_cols
    offsets = np.zeros(e.n_rows + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=offsets[1:])
    return CsrMatrix(e.n_rows, e.n_cols, offsets, grid_cols[keep], grid_vals[keep])


class DeviceEll:
    """HBM copy of an EllMatrix on one context's device (pk_ell handle)."""

    def __init__(self, e: EllMatrix, ctx: ExecutionContext):
        self.dc = context_for(ctx)
        self.n_rows, self.n_cols, self.width = e.n_rows, e.n_cols, e.width
        h = C.c_void_p()
        cols = np.ascontiguousarray(e.col_indices, dtype=np.int64)
        vals = np.ascontiguousarray(e.values, dtype=np.float64)
        N.check(N.lib().pk_ell_upload(self.dc.handle, e.n_rows, e.n_cols, e.width, cols.ctypes.data_as(C.c_void_p),
                                      vals.ctypes.data_as(C.c_void_p), C.byref(h)), "ell upload")
        self.handle = h

    def __del__(self):
        try:  # may run at interpreter shutdown, after the module globals are gone
            h = getattr(self, "handle", None)
            if h is not None and h.value:
                N.lib().pk_ell_destroy(h)
                self.handle = None
        except Exception:
            pass


_CACHE: "weakref.WeakKeyDictionary[EllMatrix, dict]" = weakref.WeakKeyDictionary()


def device_ell(e: EllMatrix, ctx: ExecutionContext | None = None) -> DeviceEll:
    ctx = ExecutionContext.coerce(ctx)
    per = _CACHE.setdefault(e, {})
    if ctx.device not in per:
        per[ctx.device] = DeviceEll(e, ctx)
    return per[ctx.device]


def spmv_ell(e: EllMatrix, p, ctx: ExecutionContext | None = None):
    """q = A p on the device from ELLPACK storage (linalg.py:383-390); ``p`` a
    float64 CUDA tensor of length n_cols; returns a new CUDA tensor."""
    ctx = ExecutionContext.coerce(ctx)
    de = device_ell(e, ctx)
    if not (isinstance(p, torch.Tensor) and p.is_cuda and p.dtype == torch.float64 and p.dim() == 1
            and p.shape[0] == e.n_cols and p.is_contiguous()):
        raise ValueError(f"p must be a contiguous 1-D float64 CUDA tensor of length {e.n_cols}")
    q = torch.empty(e.n_rows, dtype=torch.float64, device=p.device)
    de.dc.set_stream(torch.cuda.current_stream(p.device))
    N.check(N.lib().pk_spmv_ell(de.dc.handle, de.handle, C.c_void_p(p.data_ptr()) if p.numel() else None,
                                C.c_void_p(q.data_ptr()) if q.numel() else None), "spmv_ell")
    return q
