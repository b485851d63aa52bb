"""Device handles: reduction contexts and HBM-resident matrices.

A :class:`DeviceContext` wraps one ``pk_ctx`` (device + stream + geometry);
contexts are cached per (device, n_groups, group_size) and per host thread
(``pk_ctx`` is not shared across threads, include/pipekrylov_b200.h).  A
:class:`DeviceMatrix` wraps one ``pk_mat`` (CSR in HBM: int32 row offsets and
columns when nnz < 2^31, float64 values).
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native as N
from .linalg import CsrMatrix, ExecutionContext

_tls = threading.local()


class DeviceContext:
    def __init__(self, device: int = 0, n_groups: int = 128, group_size: int = 256):
        self.device = int(device)
        self.n_groups = int(n_groups)
        self.group_size = int(group_size)
        h = C.c_void_p()
        N.check(N.lib().pk_ctx_create(self.device, self.n_groups, self.group_size, C.byref(h)), "pk_ctx_create")
        self.handle = h

    def set_stream(self, stream) -> None:
        """Run kernel-level entries on ``stream``: a torch.cuda.Stream or a raw
        cudaStream_t int (0 = the legacy default stream, torch's default)."""
        ptr = getattr(stream, "cuda_stream", stream)
        N.check(N.lib().pk_ctx_set_stream(self.handle, C.c_void_p(int(ptr)) if ptr else None))

    def reset_stream(self) -> None:
        """Back to the context's private non-blocking stream."""
        N.check(N.lib().pk_ctx_reset_stream(self.handle))

    def synchronize(self) -> None:
        N.check(N.lib().pk_ctx_synchronize(self.handle))

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib().pk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def context_for(ctx: ExecutionContext | None) -> DeviceContext:
    """Cached DeviceContext for an ExecutionContext (per host thread)."""
    ctx = ExecutionContext.coerce(ctx)
    cache = getattr(_tls, "contexts", None)
    if cache is None:
        cache = _tls.contexts = {}
    key = (ctx.device, ctx.n_groups, ctx.group_size)
    dc = cache.get(key)
    if dc is None:
        dc = cache[key] = DeviceContext(*key)
    return dc


class DeviceMatrix:
    """A CSR matrix resident in HBM (``pk_mat``)."""

    def __init__(self, handle, device: int):
        self.handle = handle
        self.device = device
        n_rows, n_cols, nnz, mx = (C.c_int64() for _ in range(4))
        N.check(N.lib().pk_csr_info(handle, C.byref(n_rows), C.byref(n_cols), C.byref(nnz), C.byref(mx)))
        self.n_rows, self.n_cols, self.nnz, self.max_row_nnz = n_rows.value, n_cols.value, nnz.value, mx.value

    @classmethod
    def upload(cls, dc: DeviceContext, a: CsrMatrix) -> "DeviceMatrix":
        h = C.c_void_p()
        offs = np.ascontiguousarray(a.row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(a.col_indices, dtype=np.int64)
        vals = np.ascontiguousarray(a.values, dtype=np.float64)
        N.check(N.lib().pk_csr_upload(
            dc.handle, a.n_rows, a.n_cols,
            offs.ctypes.data_as(C.POINTER(C.c_int64)),
            cols.ctypes.data_as(C.POINTER(C.c_int64)),
            vals.ctypes.data_as(C.POINTER(C.c_double)), C.byref(h)), "pk_csr_upload")
        return cls(h, dc.device)

    @classmethod
    def generate(cls, dc: DeviceContext, family: str, dims, coef=()) -> "DeviceMatrix":
        """Build a stencil matrix directly in HBM (see generators.py)."""
        if family not in N.GEN:
            raise ValueError(f"unknown generator family {family!r}")
        d = np.ascontiguousarray(dims, dtype=np.int64)
        cf = np.ascontiguousarray(coef if len(coef) else [0.0], dtype=np.float64)
        h = C.c_void_p()
        N.check(N.lib().pk_csr_generate(
            dc.handle, N.GEN[family], d.ctypes.data_as(C.POINTER(C.c_int64)), len(d),
            cf.ctypes.data_as(C.POINTER(C.c_double)), len(coef), C.byref(h)), "pk_csr_generate")
        return cls(h, dc.device)

    FORMATS = {"csr": N.FMT_CSR, "sell32": N.FMT_SELL32}

    @property
    def format(self) -> str:
        f = C.c_int32()
        N.check(N.lib().pk_mat_get_format(self.handle, C.byref(f), None))
        return {v: k for k, v in self.FORMATS.items()}[f.value]

    @property
    def stored_entries(self) -> int:
        f, e = C.c_int32(), C.c_int64()
        N.check(N.lib().pk_mat_get_format(self.handle, C.byref(f), C.byref(e)))
        return e.value

    def set_format(self, fmt: str, context=None) -> "DeviceMatrix":
        """Storage the kernels walk: "csr" or "sell32" (an additional SELL-32
        copy, slot-major 32-row slices; bit-identical results)."""
        if fmt not in self.FORMATS:
            raise ValueError(f"unknown matrix format {fmt!r}; expected one of {sorted(self.FORMATS)}")
        dc = context_for(ExecutionContext(device=self.device) if context is None else context)
        N.check(N.lib().pk_mat_set_format(dc.handle, self.handle, self.FORMATS[fmt]), "pk_mat_set_format")
        return self

    def download(self, dc: DeviceContext) -> CsrMatrix:
        offs = np.empty(self.n_rows + 1, dtype=np.int64)
        cols = np.empty(self.nnz, dtype=np.int64)
        vals = np.empty(self.nnz, dtype=np.float64)
        N.check(N.lib().pk_csr_download(
            dc.handle, self.handle, offs.ctypes.data_as(C.POINTER(C.c_int64)),
            cols.ctypes.data_as(C.POINTER(C.c_int64)), vals.ctypes.data_as(C.POINTER(C.c_double))))
        return CsrMatrix(self.n_rows, self.n_cols, offs, cols, vals)

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib().pk_mat_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def device_matrix(a, ctx: ExecutionContext | None = None) -> DeviceMatrix:
    """HBM copy of a CsrMatrix, uploaded once per device and cached on it.
    A DeviceMatrix passes through unchanged."""
    if isinstance(a, DeviceMatrix):
        return a
    a = CsrMatrix.coerce(a)
    ctx = ExecutionContext.coerce(ctx)
    dm = a._device_cache.get(ctx.device)
    if dm is None:
        dm = DeviceMatrix.upload(context_for(ctx), a)
        a._device_cache[ctx.device] = dm
    return dm
