"""Matrix Market ingestion and the unstructured random family -- the data
formats on the caller's side of the solve path.

Same contract as the reference's ``pipekrylov.io`` (io.py:36-199, 278-343):

* ``read_matrix_market(path)``: coordinate format, ``real`` / ``integer`` /
  ``pattern`` fields, ``general`` / ``symmetric`` symmetry; symmetric storage
  is expanded (off-diagonal entries mirrored), duplicates are summed by
  ``CsrMatrix.from_coo`` (``np.add.reduceat`` in sorted order, the
  reference's canonicalisation, linalg.py:121-145), malformed input raises
  ``MatrixMarketError`` (a ``ValueError``) carrying the 1-based file line.
* ``write_matrix_market``: general real, 17 significant digits, so a
  write/read cycle is bitwise.
* ``gen_random_rowwise(n, k, seed)``: the reference's strictly diagonally
  dominant random family with exactly k distinct columns per row, drawn from
  the same ``default_rng(seed)`` stream in the same order, so the arrays are
  identical to the reference's.
* ``gen_system(spec)``: ``poisson2d:<k>``, ``poisson3d:<n>,<block>``,
  ``random:<n>,<k>[,<seed>]``.

Parsing is host work before the matrix is uploaded once to HBM; the solve
itself runs on the device (thread-per-row SpMV, rows of any length in
passes of kSlots entries).
"""

from __future__ import annotations

import numpy as np

from .generators import gen_poisson2d, gen_poisson3d_block
from .linalg import CsrMatrix

FIELDS = ("real", "integer", "pattern")
SYMMETRIES = ("general", "symmetric")


class MatrixMarketError(ValueError):
    """Malformed Matrix Market input; ``line`` is the 1-based offending line
    (errors.py MatrixMarketError)."""

    def __init__(self, message: str, line: int | None = None):
        self.line = line
        super().__init__(message if line is None else f"line {line}: {message}")


def _content(raw: str) -> str:
    # '%' starts a comment anywhere on a line (np.loadtxt(comments="%") in the reference)
    return raw.split("%", 1)[0].strip()


def read_matrix_market(path) -> CsrMatrix:
    """Coordinate Matrix Market file -> canonical CSR (io.py:36-142)."""
    with open(path, "r", encoding="ascii", errors="replace") as f:
        lines = f.read().splitlines()
    if not lines:
        raise MatrixMarketError("empty file", 1)
    head = lines[0].strip().split()
    if len(head) != 5 or head[0] != "%%MatrixMarket":
        raise MatrixMarketError("header must read '%%MatrixMarket matrix coordinate <field> <symmetry>'", 1)
    obj, fmt, field, symmetry = (t.lower() for t in head[1:])
    if obj != "matrix":
        raise MatrixMarketError(f"unsupported object {obj!r}", 1)
    if fmt != "coordinate":
        raise MatrixMarketError(f"unsupported format {fmt!r} (only coordinate)", 1)
    if field not in FIELDS:
        raise MatrixMarketError(f"unsupported field {field!r}", 1)
    if symmetry not in SYMMETRIES:
        raise MatrixMarketError(f"unsupported symmetry {symmetry!r}", 1)

    # size line: first line after the header that is neither blank nor a comment
    pos = 1
    while pos < len(lines) and (not lines[pos].strip() or lines[pos].strip().startswith("%")):
        pos += 1
    if pos >= len(lines):
        raise MatrixMarketError("missing size line", pos + 1)
    size_no = pos + 1
    parts = lines[pos].split()
    if len(parts) != 3:
        raise MatrixMarketError("size line must read 'rows cols nnz'", size_no)
    try:
        n_rows, n_cols, nnz = (int(p) for p in parts)
    except ValueError:
        raise MatrixMarketError("size line must hold three integers", size_no) from None
    if min(n_rows, n_cols, nnz) < 0:
        raise MatrixMarketError("size line entries must be non-negative", size_no)
    if symmetry == "symmetric" and n_rows != n_cols:
        raise MatrixMarketError("symmetric matrices must be square", size_no)

    want = 2 if field == "pattern" else 3
    entries, where = [], []
    for k in range(pos + 1, len(lines)):
        body = _content(lines[k])
        if not body:
            continue
        tok = body.split()
        if len(tok) != want:
            raise MatrixMarketError(f"entries must have {want} columns for field {field!r}", k + 1)
        try:
            entries.append([float(t) for t in tok])
        except ValueError:
            raise MatrixMarketError("malformed entry", k + 1) from None
        where.append(k + 1)
    if len(entries) != nnz:
        raise MatrixMarketError(f"expected {nnz} entries, found {len(entries)}")
    data = np.asarray(entries, dtype=np.float64).reshape(nnz, want)

    rows_f, cols_f = data[:, 0], data[:, 1]
    rows, cols = rows_f.astype(np.int64), cols_f.astype(np.int64)
    for bad, msg in (((rows != rows_f) | (cols != cols_f), "indices must be integers"),
                     ((rows < 1) | (rows > n_rows) | (cols < 1) | (cols > n_cols),
                      f"index out of range for a {n_rows} x {n_cols} matrix")):
        if bad.any():
            raise MatrixMarketError(msg, where[int(np.flatnonzero(bad)[0])])
    rows -= 1
    cols -= 1
    values = np.ones(nnz) if field == "pattern" else data[:, 2].copy()
    if symmetry == "symmetric":
        above = rows < cols
        if above.any():
            raise MatrixMarketError("symmetric entries must lie on or below the diagonal",
                                    where[int(np.flatnonzero(above)[0])])
        off = rows != cols
        rows, cols, values = (np.concatenate([rows, cols[off]]), np.concatenate([cols, rows[off]]),
                              np.concatenate([values, values[off]]))
    return CsrMatrix.from_coo(n_rows, n_cols, rows, cols, values)


def write_matrix_market(path, a: CsrMatrix, comment: str | None = None) -> None:
    """General real coordinate file, values with 17 significant digits
    (io.py:175-198): write -> read reproduces the matrix bitwise."""
    if not isinstance(a, CsrMatrix):
        raise TypeError("write_matrix_market expects a CsrMatrix")
    rows = np.repeat(np.arange(a.n_rows, dtype=np.int64), a.row_nnz()) + 1
    out = ["%%MatrixMarket matrix coordinate real general"]
    if comment:
        out += [f"% {ln}" for ln in comment.splitlines()]
    out.append(f"{a.n_rows} {a.n_cols} {a.nnz}")
    out += [f"{r} {c + 1} {v:.17g}" for r, c, v in zip(rows, a.col_indices, a.values)]
    with open(path, "w", encoding="ascii", newline="\n") as f:
        f.write("\n".join(out) + "\n")


def gen_random_rowwise(n: int, nnz_per_row: int, seed: int = 0):
    """Random strictly diagonally dominant system with exactly ``nnz_per_row``
    distinct columns per row, diagonal included (io.py:278-316): diagonal
    value ``nnz_per_row``, off-diagonals in (-1, 0); b = ones.  Draws from
    ``default_rng(seed)`` in the reference's order, so the arrays match."""
    if n < 1:
        raise ValueError("n must be at least 1")
    if not 1 <= nnz_per_row <= n:
        raise ValueError("nnz_per_row must lie in [1, n]")
    rng = np.random.default_rng(seed)
    k = nnz_per_row
    cols = np.empty((n, k), dtype=np.int64)
    vals = np.empty((n, k))
    for i in range(n):
        if k > n // 2:  # dense rows: a sorted prefix of a permutation
            c = np.sort(rng.permutation(n)[:k].astype(np.int64))
        else:  # sparse rows: redraw until the k columns are distinct
            c = np.unique(rng.integers(0, n, size=k))
            while c.size != k:
                c = np.unique(rng.integers(0, n, size=k))
        if i not in c:
            c[0] = i
            c.sort()
        v = -(1.0 - rng.random(k))
        v[c == i] = float(k)
        cols[i], vals[i] = c, v
    rows = np.repeat(np.arange(n, dtype=np.int64), k)
    return CsrMatrix.from_coo(n, n, rows, cols.ravel(), vals.ravel()), np.ones(n)


def gen_system(spec: str):
    """``family:args`` -> (matrix, rhs, normalised label) (io.py:319-352)."""
    family, _, argstr = spec.partition(":")
    args = [p.strip() for p in argstr.split(",") if p.strip()] if argstr else []
    try:
        if family == "poisson2d":
            (k,) = (int(p) for p in args)
            a, b = gen_poisson2d(k)
            return a, b, f"poisson2d:{k}"
        if family == "poisson3d":
            n, block = (int(p) for p in args)
            a, b = gen_poisson3d_block(n, block)
            return a, b, f"poisson3d:{n},{block}"
        if family == "random":
            n, k, seed = (int(args[0]), int(args[1]), 0) if len(args) == 2 else (int(p) for p in args)
            a, b = gen_random_rowwise(n, k, seed)
            return a, b, f"random:{n},{k},{seed}"
    except ValueError as exc:
        raise ValueError(f"bad generator spec {spec!r}: {exc}") from None
    raise ValueError(f"unknown generator family {family!r}")
