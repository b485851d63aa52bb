"""Benchmark systems of the hot path.

Poisson families follow the reference generators exactly (io.py:201-275):
``gen_poisson2d(k)`` is the 5-point 4/-1 Laplacian on a (2**(k+3)-1)^2 grid,
``gen_poisson3d_block(n, 1)`` the 7-point Laplacian scaled by the 2x block
(values 12/-2).  ``poisson2d_grid(side)`` frees the side length (the C1
config is 512 x 512, not a reference level).

The convection-diffusion families are defined by this project (the reference
has none; BASELINE.json configs 2 and 3 name them): first-order upwind
discretisation of -Lap(u) + c . grad(u) on the unit square/cube, scaled by
h^2 with h = 1/(side+1):

  2D: diag 4 + h (cx + cy); west -1 - h cx; south -1 - h cy; east, north -1
  3D: diag 6 + h ((cx + cy) + cz); west/south/down -1 - h c; others -1

Every family exists twice: on the host (NumPy CsrMatrix, what a reference
user passes in) and in HBM (``device=True``: built by a CUDA kernel with the
same values, bit-identical arrays; needed for 512^3 where the host copy would
take ~100 GB).  The right-hand side is all ones, as in the reference.
"""

from __future__ import annotations

import numpy as np

from .linalg import CsrMatrix

__all__ = ["gen_poisson2d", "gen_poisson3d_block", "poisson2d_grid", "poisson3d_grid", "convdiff2d",
           "convdiff3d", "stencil_coefficients"]


def stencil_coefficients(family: str, side: int, c=(1.0, 1.0, 1.0)):
    """(diag, [(axis, step, value)]) for a family; the single source of the
    values for the host and the device generators."""
    if family == "poisson2d":
        return 4.0, [(ax, st, -1.0) for ax in (0, 1) for st in (-1, 1)]
    if family == "poisson3d":
        return 12.0, [(ax, st, -2.0) for ax in (0, 1, 2) for st in (-1, 1)]
    h = 1.0 / (side + 1)
    if family == "convdiff2d":
        cx, cy = float(c[0]), float(c[1])
        return 4.0 + h * (cx + cy), [(0, -1, -1.0 - h * cx), (0, 1, -1.0), (1, -1, -1.0 - h * cy), (1, 1, -1.0)]
    if family == "convdiff3d":
        cx, cy, cz = (float(v) for v in c[:3])
        return 6.0 + h * (cx + cy + cz), [(0, -1, -1.0 - h * cx), (0, 1, -1.0), (1, -1, -1.0 - h * cy),
                                          (1, 1, -1.0), (2, -1, -1.0 - h * cz), (2, 1, -1.0)]
    raise ValueError(f"unknown generator family {family!r}")


def _assemble(dims, diag, faces) -> CsrMatrix:
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64)
    strides = np.cumprod((1,) + tuple(dims[:-1]))
    rows, cols, vals = [idx], [idx], [np.full(n, diag)]
    for axis, step, val in faces:
        coord = (idx // strides[axis]) % dims[axis]
        keep = (coord + step >= 0) & (coord + step < dims[axis])
        r = idx[keep]
        rows.append(r)
        cols.append(r + step * strides[axis])
        vals.append(np.full(r.size, val))
    return CsrMatrix.from_coo(n, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))


def _device(family, dims, coef, context):
    from .device import DeviceMatrix, context_for
    from .linalg import ExecutionContext

    ctx = ExecutionContext.coerce(context)
    return DeviceMatrix.generate(context_for(ctx), family, dims, coef)


def poisson2d_grid(side: int, device: bool = False, context=None):
    if side < 1:
        raise ValueError("side must be at least 1")
    if device:
        return _device("poisson2d", (side, side), (4.0, -1.0), context), np.ones(side * side)
    diag, faces = stencil_coefficients("poisson2d", side)
    return _assemble((side, side), diag, faces), np.ones(side * side)


def gen_poisson2d(k: int, device: bool = False, context=None):
    """Reference level k (io.py:201-229): side 2**(k+3) - 1."""
    if k < 1:
        raise ValueError("level k must be at least 1")
    return poisson2d_grid(2 ** (k + 3) - 1, device=device, context=context)


def poisson3d_grid(side: int, device: bool = False, context=None):
    """== gen_poisson3d_block(side, 1) (io.py:232-275): values 12 / -2."""
    if side < 1:
        raise ValueError("grid dimension n must be at least 1")
    if device:
        return _device("poisson3d", (side, side, side), (12.0, -2.0), context), np.ones(side ** 3)
    diag, faces = stencil_coefficients("poisson3d", side)
    return _assemble((side, side, side), diag, faces), np.ones(side ** 3)


def _block_expand(scalar: CsrMatrix, block: int) -> CsrMatrix:
    """Kronecker product of a scalar CSR operator with the SPD block
    B = I + ones(block, block) / block (io.py:232-275): scalar entry (i, j, v)
    becomes the block-row entries (i b + s, j b + t, v * B[s, t]).  Every
    block row keeps the scalar row's column order (neighbour j ascending,
    then t), which is the canonical order from_coo would produce; no
    duplicates arise, so no value is summed."""
    b = int(block)
    bmat = np.eye(b) + np.ones((b, b)) / b
    offs, cols, vals = scalar.row_offsets, scalar.col_indices, scalar.values
    n = scalar.n_rows
    rowlen = np.diff(offs)
    row_of = np.repeat(np.arange(n, dtype=np.int64), rowlen)
    k_of = np.arange(offs[-1], dtype=np.int64) - offs[row_of]
    t = np.arange(b, dtype=np.int64)
    out_cols = np.empty(int(offs[-1]) * b * b, dtype=np.int64)
    out_vals = np.empty(int(offs[-1]) * b * b)
    for s in range(b):
        # block row (i, s) starts at offs[i] b^2 + s rowlen_i b; entry k, column t at + k b + t
        base = offs[row_of] * b * b + s * rowlen[row_of] * b + k_of * b
        pos = base[:, None] + t[None, :]
        out_cols[pos] = cols[:, None] * b + t[None, :]
        out_vals[pos] = vals[:, None] * bmat[s][None, :]
    out_offs = np.zeros(n * b + 1, dtype=np.int64)
    np.cumsum(np.repeat(rowlen * b, b), out=out_offs[1:])
    return CsrMatrix(n * b, n * b, out_offs, out_cols, out_vals)


def gen_poisson3d_block(n: int, block: int, device: bool = False, context=None):
    """Seven-point Laplacian (6 / -1) on an n^3 grid, every entry times the
    block I + ones(block, block)/block (io.py:232-275); block == 1 gives the
    12 / -2 operator of the C4 config (also generated directly in HBM with
    ``device=True``)."""
    if n < 1:
        raise ValueError("grid dimension n must be at least 1")
    if block < 1:
        raise ValueError("block size must be at least 1")
    if block == 1:
        return poisson3d_grid(n, device=device, context=context)
    faces = [(ax, st, -1.0) for ax in (0, 1, 2) for st in (-1, 1)]
    a = _block_expand(_assemble((n, n, n), 6.0, faces), block)
    if device:
        from .device import device_matrix
        from .linalg import ExecutionContext

        return device_matrix(a, ExecutionContext.coerce(context)), np.ones(n ** 3 * block)
    return a, np.ones(n ** 3 * block)


def convdiff2d(side: int, c=(1.0, 1.0), device: bool = False, context=None):
    if side < 1:
        raise ValueError("side must be at least 1")
    if device:
        return _device("convdiff2d", (side, side), tuple(float(v) for v in c[:2]), context), np.ones(side * side)
    diag, faces = stencil_coefficients("convdiff2d", side, c)
    return _assemble((side, side), diag, faces), np.ones(side * side)


def convdiff3d(side: int, c=(1.0, 1.0, 1.0), device: bool = False, context=None):
    if side < 1:
        raise ValueError("side must be at least 1")
    if device:
        return (_device("convdiff3d", (side, side, side), tuple(float(v) for v in c[:3]), context),
                np.ones(side ** 3))
    diag, faces = stencil_coefficients("convdiff3d", side, c)
    return _assemble((side, side, side), diag, faces), np.ones(side ** 3)
