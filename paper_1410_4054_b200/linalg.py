"""Host-side data types of the hot path: CSR matrix, reduction geometry and
the launch/transfer trace.

These mirror the reference's public types so reference-style code runs
unchanged:

* :class:`CsrMatrix`       -- pipekrylov/linalg.py:71-176 (canonical CSR,
  validation raising ``ValueError``, ``from_coo`` summing duplicates).
* :class:`ExecutionContext` -- pipekrylov/execmodel.py:188-219 (reduction
  geometry ``n_groups x group_size``; the geometry fixes every rounded
  result).  Extended with ``device`` (CUDA ordinal).
* :class:`ExecutionTrace` / :class:`PhaseRecord` -- execmodel.py:110-185, here
  filled with the launches and host<->device transfers the B200 path really
  performed.

Matrices are immutable; the first solve on a device uploads the CSR arrays to
HBM (int32 columns, float64 values) and caches the device copy on the object.
"""

from __future__ import annotations

from contextlib import contextmanager
from dataclasses import dataclass, field, replace

import numpy as np

SETUP, ITERATION, FINISH, CHECK = "setup", "iteration", "finish", "check"


def as_vector(x, n: int | None = None, name: str = "vector") -> np.ndarray:
    """1-D float64 view/copy of ``x`` with an optional length check (linalg.py:53-60)."""
    v = np.asarray(x, dtype=np.float64)
    if v.ndim != 1:
        raise ValueError(f"{name} must be one-dimensional, got shape {v.shape}")
    if n is not None and v.shape[0] != n:
        raise ValueError(f"{name} has length {v.shape[0]}, expected {n}")
    return v


class CsrMatrix:
    """Canonical CSR matrix (strictly increasing columns per row).

    Same constructor, attributes and validation as the reference
    (linalg.py:71-111).  Arrays are stored as int64/float64 and never
    mutated."""

    __slots__ = ("n_rows", "n_cols", "row_offsets", "col_indices", "values", "_device_cache", "__weakref__")

    def __init__(self, n_rows, n_cols, row_offsets, col_indices, values):
        n_rows, n_cols = int(n_rows), int(n_cols)
        # private copies: freezing them must not make the caller's arrays
        # read-only, and later edits of the caller's buffers must not desync
        # the cached HBM copy (the reference keeps its own arrays too)
        offs = np.array(row_offsets, dtype=np.int64, copy=True)
        cols = np.array(col_indices, dtype=np.int64, copy=True)
        vals = np.array(values, dtype=np.float64, copy=True)
        if n_rows < 0 or n_cols < 0:
            raise ValueError("matrix dimensions must be non-negative")
        if offs.ndim != 1 or offs.shape[0] != n_rows + 1:
            raise ValueError(f"row_offsets must have {n_rows + 1} entries")
        if offs[0] != 0:
            raise ValueError("row_offsets must start at 0")
        steps = np.diff(offs)
        if np.any(steps < 0):
            raise ValueError("row_offsets must be non-decreasing")
        nnz = int(offs[-1])
        if cols.shape != (nnz,) or vals.shape != (nnz,):
            raise ValueError("col_indices and values must match row_offsets[-1] entries")
        if nnz and (cols.min() < 0 or cols.max() >= n_cols):
            raise ValueError("column index out of range")
        if nnz > 1:
            # a non-increasing step is only allowed where a new row starts
            first_of_row = np.zeros(nnz, dtype=bool)
            starts = offs[:-1][steps > 0]
            first_of_row[starts] = True
            bad = (np.diff(cols) <= 0) & ~first_of_row[1:]
            if bad.any():
                raise ValueError("column indices must be strictly increasing within each row")
        for name, arr in (("row_offsets", offs), ("col_indices", cols), ("values", vals)):
            arr.flags.writeable = False
            object.__setattr__(self, name, arr)
        object.__setattr__(self, "n_rows", n_rows)
        object.__setattr__(self, "n_cols", n_cols)
        object.__setattr__(self, "_device_cache", {})

    def __setattr__(self, key, value):
        raise AttributeError("CsrMatrix is immutable")

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    def row_nnz(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    @classmethod
    def from_coo(cls, n_rows, n_cols, rows, cols, values) -> "CsrMatrix":
        """Triplets -> canonical CSR; duplicates summed (linalg.py:121-145)."""
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        values = np.asarray(values, dtype=np.float64)
        if rows.ndim != 1 or not (rows.shape == cols.shape == values.shape):
            raise ValueError("rows, cols and values must be 1-D and equally long")
        if rows.size:
            if rows.min() < 0 or rows.max() >= n_rows:
                raise ValueError("row index out of range")
            if cols.min() < 0 or cols.max() >= n_cols:
                raise ValueError("column index out of range")
        order = np.lexsort((cols, rows))
        rows, cols, values = rows[order], cols[order], values[order]
        if rows.size:
            new = np.ones(rows.size, dtype=bool)
            new[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
            heads = np.flatnonzero(new)
            values = np.add.reduceat(values, heads)
            rows, cols = rows[heads], cols[heads]
        offsets = np.zeros(n_rows + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=n_rows), out=offsets[1:])
        return cls(n_rows, n_cols, offsets, cols, values)

    @classmethod
    def from_dense(cls, a) -> "CsrMatrix":
        a = np.asarray(a, dtype=np.float64)
        if a.ndim != 2:
            raise ValueError("dense input must be two-dimensional")
        r, c = np.nonzero(a)
        return cls.from_coo(a.shape[0], a.shape[1], r, c, a[r, c])

    @classmethod
    def identity(cls, n: int) -> "CsrMatrix":
        return cls(n, n, np.arange(n + 1), np.arange(n), np.ones(n))

    @classmethod
    def coerce(cls, a) -> "CsrMatrix":
        """Accept this class or any object with the reference CsrMatrix fields."""
        if isinstance(a, cls):
            return a
        needed = ("n_rows", "n_cols", "row_offsets", "col_indices", "values")
        if all(hasattr(a, k) for k in needed):
            return cls(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values)
        raise ValueError("A must be a CsrMatrix")

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n_rows, self.n_cols))
        rows = np.repeat(np.arange(self.n_rows), self.row_nnz())
        out[rows, self.col_indices] = self.values
        return out

    def equals(self, other) -> bool:
        return (self.shape == other.shape
                and np.array_equal(self.row_offsets, other.row_offsets)
                and np.array_equal(self.col_indices, other.col_indices)
                and np.array_equal(self.values, other.values))


@dataclass(frozen=True)
class WorkgroupPartials:
    """Per-group partial sums, shape (n_groups, n_quantities) (linalg.py:254-286)."""

    data: np.ndarray

    def __post_init__(self):
        d = np.asarray(self.data, dtype=np.float64)
        if d.ndim != 2:
            raise ValueError("partials must be two-dimensional (n_groups, n_quantities)")
        object.__setattr__(self, "data", d)

    @property
    def n_groups(self) -> int:
        return self.data.shape[0]

    @property
    def n_quantities(self) -> int:
        return self.data.shape[1]

    @property
    def nbytes(self) -> int:
        return self.data.size * 8

    @classmethod
    def stack(cls, parts) -> "WorkgroupPartials":
        if not parts:
            raise ValueError("need at least one partials block")
        if len({p.n_groups for p in parts}) > 1:
            raise ValueError("partials blocks disagree on n_groups")
        return cls(np.hstack([p.data for p in parts]))


@dataclass
class PhaseRecord:
    """Launch/transfer counters of one phase (execmodel.py:110-118)."""

    label: str
    launches: int = 0
    transfers: int = 0
    bytes_kernel: int = 0
    bytes_transfer: int = 0


class ExecutionTrace:
    """Phases of one solve with the launches/transfers the device path issued."""

    def __init__(self):
        self.phases: list[PhaseRecord] = []
        self._open: PhaseRecord | None = None

    def begin_phase(self, label: str) -> PhaseRecord:
        if self._open is not None:
            raise RuntimeError(f"phase {self._open.label!r} is still open")
        rec = PhaseRecord(label)
        self.phases.append(rec)
        self._open = rec
        return rec

    def end_phase(self) -> None:
        if self._open is None:
            raise RuntimeError("no phase is open")
        self._open = None

    @contextmanager
    def phase(self, label: str):
        self.begin_phase(label)
        try:
            yield
        finally:
            self.end_phase()

    def add_phase(self, label: str, launches: int = 0, transfers: int = 0, bytes_kernel: int = 0,
                  bytes_transfer: int = 0) -> PhaseRecord:
        rec = PhaseRecord(label, int(launches), int(transfers), int(bytes_kernel), int(bytes_transfer))
        self.phases.append(rec)
        return rec

    def record_launch(self, nbytes: int = 0) -> None:
        if self._open is None:
            raise RuntimeError("record_launch outside an open phase")
        self._open.launches += 1
        self._open.bytes_kernel += int(nbytes)

    def record_transfer(self, nbytes: int = 0) -> None:
        if self._open is None:
            raise RuntimeError("record_transfer outside an open phase")
        self._open.transfers += 1
        self._open.bytes_transfer += int(nbytes)

    @property
    def iterations(self) -> list[PhaseRecord]:
        return [p for p in self.phases if p.label == ITERATION]

    def totals(self) -> PhaseRecord:
        t = PhaseRecord("total")
        for p in self.phases:
            t.launches += p.launches
            t.transfers += p.transfers
            t.bytes_kernel += p.bytes_kernel
            t.bytes_transfer += p.bytes_transfer
        return t

    def steady_state(self) -> PhaseRecord:
        it = self.iterations
        if not it:
            raise ValueError("trace has no iteration phases")
        return it[1] if len(it) > 1 else it[0]


@dataclass
class ExecutionContext:
    """Reduction geometry (execmodel.py:188-207) plus the CUDA device ordinal.

    ``n_groups`` workgroups of ``group_size`` (power of two) lanes define the
    stage-1 schedule; the B200 kernels reproduce it exactly, so results are
    bit-identical to the reference run with the same geometry."""

    n_groups: int = 128
    group_size: int = 256
    trace: ExecutionTrace | None = None
    device: int = 0

    def __post_init__(self):
        if self.n_groups < 1:
            raise ValueError(f"n_groups must be >= 1, got {self.n_groups}")
        if self.group_size < 1 or (self.group_size & (self.group_size - 1)) != 0:
            raise ValueError(f"group_size must be a positive power of two, got {self.group_size}")

    def with_trace(self, trace: ExecutionTrace) -> "ExecutionContext":
        return replace(self, trace=trace)

    @classmethod
    def coerce(cls, ctx) -> "ExecutionContext":
        if ctx is None:
            return cls()
        if isinstance(ctx, cls):
            return ctx
        # the reference's ExecutionContext (same field names)
        return cls(n_groups=int(ctx.n_groups), group_size=int(ctx.group_size))

    @classmethod
    def one_per_lane(cls, n: int, group_size: int = 1024, device: int = 0) -> "ExecutionContext":
        """Wide geometry: G >= n so every lane holds at most one element and
        each group is a contiguous row tile (fastest on B200)."""
        return cls(n_groups=max(1, -(-int(n) // group_size)), group_size=group_size, device=device)


DEFAULT_CONTEXT = ExecutionContext()
