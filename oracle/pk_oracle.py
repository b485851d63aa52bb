"""CPU oracle for the pipelined Krylov hot path -- TEST INFRASTRUCTURE ONLY.

This module is a NumPy restatement of the reference package ``pipekrylov``
(arXiv 1410.4054 emulation, mounted read-only at /root/reference during
development; absent on the GPU box).  It exists so that the CUDA product path
in ``paper_1410_4054_b200`` can be checked bit-for-bit against the
reference's arithmetic on machines where the reference cannot be imported.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import it, and only as the checker (or as the timed CPU port).  The
product never calls into this file.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference and
stores its outputs under ``tests/golden/*.npz``; ``tests/test_oracle.py``
asserts this module reproduces every stored array bitwise.  When the reference
is importable (this development container) the same tests also diff the
oracle against the live reference on freshly generated cases.

Arithmetic contract (restated from the reference; every op is IEEE binary64,
round to nearest, never fused):

* SpMV row:   acc = 0.0; acc = acc + val[k] * x[col[k]]  in stored order
              (_spmvkernels.py:12-18).
* stage 1:    lane t = serial sum (from 0.0) of c[t], c[t+G], c[t+2G], ...
              with G = n_groups * group_size, then a halving tree inside each
              group of group_size lanes (linalg.py:289-308).
* stage 2:    serial left-to-right sum over groups (linalg.py:311-320).
"""

from __future__ import annotations

import math
import time

import numpy as np

DEFAULT_N_GROUPS = 128  # execmodel.py:199
DEFAULT_GROUP_SIZE = 256  # execmodel.py:200
DEFAULT_BTOL = 1e-30  # fused.py:49

CONVERGED, MAX_ITER, BREAKDOWN, LUCKY_BREAKDOWN = (
    "converged", "max_iter", "breakdown", "lucky_breakdown")  # solvers.py:95-98


class Csr:
    """Plain CSR triple (int64 offsets/columns, float64 values)."""

    def __init__(self, n_rows, n_cols, rowptr, cols, vals):
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self.rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self._slots = None

    @property
    def nnz(self):
        return int(self.rowptr[-1])

    def slots(self):
        """Per-slot (rows, entry index) lists: slot s holds the s-th entry of
        every row that has more than s entries.  Lets the row loop run
        vectorised over rows while keeping each row's left-to-right order."""
        if self._slots is None:
            counts = np.diff(self.rowptr)
            width = int(counts.max()) if counts.size else 0
            out = []
            for s in range(width):
                rows = np.flatnonzero(counts > s)
                out.append((rows, self.rowptr[rows] + s))
            self._slots = out
        return self._slots


def as_csr(a) -> Csr:
    if isinstance(a, Csr):
        return a
    # duck-type the reference CsrMatrix / the product's CsrMatrix
    return Csr(a.n_rows, a.n_cols, a.row_offsets, a.col_indices, a.values)


# ---------------------------------------------------------------------------
# core arithmetic
# ---------------------------------------------------------------------------


def csr_spmv(a, x):
    """Row-sequential product, no FMA (_spmvkernels.py:12-18)."""
    a = as_csr(a)
    x = np.asarray(x, dtype=np.float64)
    acc = np.zeros(a.n_rows)
    for rows, idx in a.slots():
        acc[rows] = acc[rows] + a.vals[idx] * x[a.cols[idx]]
    return acc


def ell_spmv(n_rows, n_cols, width, cols, vals, x):
    """ELLPACK product (_spmvkernels.py:21-34): slot k of row i at
    i + k n_rows, sentinel column n_cols skipped (not multiplied by 0), slots
    in order -- vectorised over rows, sequential over slots."""
    x = np.asarray(x, dtype=np.float64)
    acc = np.zeros(n_rows)
    rows = np.arange(n_rows)
    for k in range(width):
        c = np.asarray(cols[k * n_rows:(k + 1) * n_rows])
        live = c < n_cols
        r = rows[live]
        acc[r] = acc[r] + np.asarray(vals[k * n_rows:(k + 1) * n_rows])[live] * x[c[live]]
    return acc


def stage1(contrib, n_groups=DEFAULT_N_GROUPS, group_size=DEFAULT_GROUP_SIZE):
    """Grid-stride lanes + per-group halving tree (linalg.py:289-308).

    ``contrib`` is (n,) or (n, nq); returns (n_groups, nq)."""
    c = np.asarray(contrib, dtype=np.float64)
    if c.ndim == 1:
        c = c[:, None]
    n, nq = c.shape
    span = n_groups * group_size
    lanes = np.zeros((span, nq))
    for k0 in range(0, n, span):
        seg = c[k0:k0 + span]
        lanes[: seg.shape[0]] = lanes[: seg.shape[0]] + seg
    tree = lanes.reshape(n_groups, group_size, nq)
    width = group_size
    while width > 1:
        width //= 2
        tree = tree[:, :width] + tree[:, width: 2 * width]
    return np.ascontiguousarray(tree[:, 0])


def stage2(partials):
    """Serial sum over groups per quantity (linalg.py:311-320)."""
    p = np.asarray(partials, dtype=np.float64)
    if p.ndim == 1:
        p = p[:, None]
    out = np.zeros(p.shape[1])
    for q in range(p.shape[1]):
        tot = 0.0
        for v in p[:, q].tolist():
            tot += v
        out[q] = tot
    return out


def dot(x, y, geom):
    """Two-stage inner product (linalg.py:351-365)."""
    return float(stage2(stage1(np.asarray(x) * np.asarray(y), *geom))[0])


# ---------------------------------------------------------------------------
# fused ops (fused.py)
# ---------------------------------------------------------------------------


def spmv_fused(a, p, kinds, geom):
    """q = A p plus stage-1 partials for each requested dot (fused.py:86-120).

    ``kinds`` entries: "input" (q*p), "result" (q*q) or a vector w (q*w)."""
    q = csr_spmv(a, p)
    cols = []
    for kind in kinds:
        if isinstance(kind, str):
            cols.append(q * p if kind == "input" else q * q)
        else:
            cols.append(q * np.asarray(kind))
    return q, stage1(np.stack(cols, axis=1), *geom)


def cg_update(x, r, p, ap, alpha, beta, geom):
    """In place x+=a p, r-=a Ap, p=b p + r; returns <r,r> partials (fused.py:123-151)."""
    x += alpha * p
    r -= alpha * ap
    p *= beta
    p += r
    return stage1(r * r, *geom)


def bicg_s_update(r, ap, rr0_part, apr_part, geom, btol):
    """alpha from partials, s = r - alpha Ap (fused.py:154-182).

    Returns (s, ss partials, alpha) or raises ``Breakdown``."""
    rho = stage2(rr0_part)[0]
    den = stage2(apr_part)[0]
    if abs(den) < btol:
        raise Breakdown("Apr0star")
    with np.errstate(all="ignore"):
        alpha = rho / den
        s = r - alpha * ap
    return s, stage1(s * s, *geom), float(alpha)


def bicg_xrp_update(x, r, p, s, ap, as_, alpha, omega, beta, r0s, geom):
    """x+=a p+w s; r=s-w As; p=b(p-w Ap)+r; <r,r0*> partials (fused.py:185-219)."""
    x += alpha * p + omega * s
    r[:] = s - omega * as_
    p -= omega * ap
    p *= beta
    p += r
    return stage1(r * r0s, *geom)


def gs_stage1(basis, v, geom):
    """Partials of <b_j, v> for all j (fused.py:222-243)."""
    n = np.asarray(v).shape[0]
    if not basis:
        return np.zeros((geom[0], 0))
    return stage1(np.stack([b * v for b in basis], axis=1), *geom)


def gs_update(v, basis, partials, geom):
    """coeffs = stage2; v -= sum_j c_j b_j (accumulated from 0.0); <v,v> partials
    (fused.py:246-277)."""
    coeffs = stage2(partials) if partials.shape[1] else np.zeros(0)
    if basis:
        acc = np.zeros(v.shape[0])
        for c, b in zip(coeffs, basis):
            acc += c * b
        v -= acc
    return coeffs, stage1(v * v, *geom)


def gs_normalize(v, norm_part, r, geom, btol):
    """||v|| = sqrt(stage2); v *= 1/||v||; <r,v> partials (fused.py:280-305)."""
    nrm = math.sqrt(stage2(norm_part)[0])
    if nrm < btol or nrm == 0.0:
        # nrm == 0.0 with btol == 0 (fixed mode) is a ZeroDivisionError in
        # the reference (fused.py:300); treated as a lucky breakdown here.
        raise Lucky(nrm)
    v *= 1.0 / nrm
    return nrm, stage1(r * v, *geom)


class Breakdown(Exception):
    def __init__(self, kind):
        super().__init__(kind)
        self.kind = kind


class Lucky(Exception):
    pass


def solve_upper_triangular(rmat, rhs, btol):
    """Back substitution with np.dot (solvers.py:205-218); raises Breakdown."""
    k = rmat.shape[0]
    eta = np.zeros(k)
    for i in range(k - 1, -1, -1):
        d = rmat[i, i]
        if abs(d) < btol:
            raise Breakdown("singular_R")
        eta[i] = (rhs[i] - float(np.dot(rmat[i, i + 1:], eta[i + 1:]))) / d
    return eta


# ---------------------------------------------------------------------------
# drivers (solvers.py)
# ---------------------------------------------------------------------------


def _true_residual(a, b, x, geom):
    q = csr_spmv(a, x)
    res = b + (-1.0) * q
    return math.sqrt(dot(res, res, geom))


def _finish(a, b, x, geom, history, term, kind):
    return {
        "x": x,
        "history": list(history),
        "iterations": len(history),
        "termination": term,
        "breakdown_kind": kind,
        "true_final_residual": _true_residual(a, b, x, geom),
    }


def _setup(a, b, x0):
    a = as_csr(a)
    b = np.array(b, dtype=np.float64)
    x = np.zeros(a.n_rows) if x0 is None else np.array(x0, dtype=np.float64)
    return a, b, x


def cg_pipelined(a, b, x0=None, tol=1e-8, max_iterations=500, fixed=None,
                 geom=(DEFAULT_N_GROUPS, DEFAULT_GROUP_SIZE), btol=DEFAULT_BTOL, timing=None):
    """Restatement of solvers.cg_pipelined (solvers.py:395-469)."""
    a, b, x = _setup(a, b, x0)
    lbt = 0.0 if fixed else btol  # solvers.py:141-145
    limit = fixed if fixed else max_iterations
    norm_b = math.sqrt(dot(b, b, geom))
    scale = norm_b if norm_b > 0 else 1.0
    r = b + (-1.0) * csr_spmv(a, x)
    p = r.copy()
    ap, pq = spmv_fused(a, p, ("input", "result"), geom)
    rr_part = stage1(r * r, *geom)
    rr, pap, apap = stage2(np.hstack([rr_part, pq])).tolist()
    hist = []
    if math.sqrt(rr) / scale <= tol and (not fixed or rr == 0.0):
        return _finish(a, b, x, geom, hist, CONVERGED, None)
    if abs(pap) < lbt or pap == 0.0:
        return _finish(a, b, x, geom, hist, BREAKDOWN, "pAp")
    alpha = rr / pap
    beta = alpha * alpha * apap / rr - 1.0
    term, kind = MAX_ITER, None
    t0 = time.perf_counter()  # loop_seconds protocol, solvers.py:444/468
    for _ in range(limit):
        rr_part = cg_update(x, r, p, ap, alpha, beta, geom)
        ap, pq = spmv_fused(a, p, ("input", "result"), geom)
        rr, pap, apap = stage2(np.hstack([rr_part, pq])).tolist()
        mon = math.sqrt(rr) / scale
        hist.append(mon)
        if not math.isfinite(mon):
            term, kind = BREAKDOWN, "divergence"
            break
        if mon <= tol and (not fixed or rr == 0.0):
            term = CONVERGED
            break
        if abs(pap) < lbt or pap == 0.0:
            # pap == 0.0 in fixed mode raises ZeroDivisionError in the
            # reference; the B200 path reports it as a pAp breakdown.
            term, kind = BREAKDOWN, "pAp"
            break
        alpha = rr / pap
        beta = alpha * alpha * apap / rr - 1.0
    if timing is not None:
        timing["loop_seconds"] = time.perf_counter() - t0
    return _finish(a, b, x, geom, hist, term, kind)


def bicgstab_pipelined(a, b, x0=None, tol=1e-8, max_iterations=500, fixed=None,
                       geom=(DEFAULT_N_GROUPS, DEFAULT_GROUP_SIZE), btol=DEFAULT_BTOL, timing=None):
    """Restatement of solvers.bicgstab_pipelined (solvers.py:583-712)."""
    a, b, x = _setup(a, b, x0)
    lbt = 0.0 if fixed else btol
    limit = fixed if fixed else max_iterations
    norm_b = math.sqrt(dot(b, b, geom))
    scale = norm_b if norm_b > 0 else 1.0
    r = b + (-1.0) * csr_spmv(a, x)
    r0s = r.copy()
    p = r.copy()
    rr = dot(r, r, geom)
    rr0_part = stage1(r * r0s, *geom)
    hist = []
    if math.sqrt(rr) / scale <= tol and (not fixed or rr == 0.0):
        return _finish(a, b, x, geom, hist, CONVERGED, None)
    term, kind, half = MAX_ITER, None, None
    it = 0
    t0 = time.perf_counter()  # solvers.py:632/695
    while it < limit:
        it += 1
        confirm = False
        ap, apr_part = spmv_fused(a, p, (r0s,), geom)
        try:
            s, ss_part, alpha = bicg_s_update(r, ap, rr0_part, apr_part, geom, lbt)
        except Breakdown as e:
            term, kind = BREAKDOWN, e.kind
            break
        as_, tri = spmv_fused(a, s, ("input", "result", r0s), geom)
        ss, ass, asas, asr, apr = stage2(np.hstack([ss_part, tri, apr_part])).tolist()
        mon_s = math.sqrt(ss) / scale
        if not fixed and mon_s <= tol:
            half = alpha
            hist.append(mon_s)
            term = CONVERGED
            break
        if asas < lbt or asas == 0.0:
            # asas == 0.0 (fixed mode) is a ZeroDivisionError crash in the
            # reference; the B200 path reports an AsAs breakdown instead.
            term, kind = BREAKDOWN, "AsAs"
            break
        if apr == 0.0:
            # same for -asr / apr (solvers.py:664)
            term, kind = BREAKDOWN, "Apr0star"
            break
        omega = ass / asas
        beta = -asr / apr
        ident = ss - 2.0 * omega * ass + omega * omega * asas
        clamped = ident < 0.0
        rr = max(ident, 0.0)
        rr0_part = bicg_xrp_update(x, r, p, s, ap, as_, alpha, omega, beta, r0s, geom)
        mon = math.sqrt(rr) / scale
        hist.append(mon)
        if not math.isfinite(mon):
            term, kind = BREAKDOWN, "divergence"
            break
        if not fixed and mon <= tol:
            if clamped:
                confirm = True
            else:
                term = CONVERGED
                break
        if confirm and _true_residual(a, b, x, geom) <= tol * scale:
            term = CONVERGED
            break
    if timing is not None:
        timing["loop_seconds"] = time.perf_counter() - t0
    if half is not None:
        x += half * p
    return _finish(a, b, x, geom, hist, term, kind)


def gmres_pipelined(a, b, x0=None, tol=1e-8, max_iterations=500, fixed=None, restart=30,
                    geom=(DEFAULT_N_GROUPS, DEFAULT_GROUP_SIZE), btol=DEFAULT_BTOL, timing=None):
    """Restatement of solvers.gmres_pipelined (solvers.py:865-1008)."""
    a, b, x = _setup(a, b, x0)
    lbt = 0.0 if fixed else btol
    limit = fixed if fixed else max_iterations
    m = restart
    hist = []
    term, kind = MAX_ITER, None
    total = 0
    scale = None
    done = False
    while not done and total < limit:
        if scale is None:
            nb = math.sqrt(dot(b, b, geom))
            scale = nb if nb > 0 else 1.0
        r = b + (-1.0) * csr_spmv(a, x)
        rho = math.sqrt(dot(r, r, geom))
        if not (rho > 0 and not (not fixed and rho / scale <= tol)):
            term = CONVERGED
            break
        r *= 1.0 / rho
        basis, xi_parts = [], []
        rmat = np.zeros((m, m))
        lucky = False
        t0 = time.perf_counter()  # inner loop only, solvers.py:928/953
        while len(basis) < m and total < limit:
            i = len(basis) + 1
            if i == 1:
                w, norm_part = spmv_fused(a, r, ("result",), geom)
            else:
                w, last = spmv_fused(a, basis[-1], ("input",), geom)
                older = gs_stage1(basis[:-1], w, geom)
                coeffs, norm_part = gs_update(w, basis, np.hstack([older, last]), geom)
                rmat[: i - 1, i - 1] = coeffs
            try:
                nrm, xi_part = gs_normalize(w, norm_part, r, geom, lbt)
            except Lucky:
                lucky = True
                break
            rmat[i - 1, i - 1] = nrm
            basis.append(w)
            xi_parts.append(xi_part)
            total += 1
        if timing is not None:
            timing["loop_seconds"] = timing.get("loop_seconds", 0.0) + time.perf_counter() - t0
        k = len(basis)
        conv_at = None
        gate = None
        if k > 0:
            xi = stage2(np.hstack(xi_parts))
            est2 = 1.0
            for idx, xv in enumerate(xi.tolist()):
                est2 = max(est2 - xv * xv, 0.0)
                mon = rho * math.sqrt(est2) / scale
                hist.append(mon)
                if not fixed and conv_at is None and mon <= tol:
                    conv_at = idx + 1
            ks = conv_at if conv_at is not None else k
            try:
                eta = solve_upper_triangular(rmat[:ks, :ks], xi[:ks], btol)
            except Breakdown as e:
                term, kind, done, eta = BREAKDOWN, e.kind, True, None
            if eta is not None:
                upd = eta[0] * r
                for idx in range(1, ks):
                    upd += eta[idx] * basis[idx - 1]
                x += rho * upd
                if conv_at is not None or lucky:
                    gate = _true_residual(a, b, x, geom)
            with np.errstate(all="ignore"):
                if not math.isfinite(float(np.sum(np.asarray(xi) ** 2))):
                    term, kind, done = BREAKDOWN, "divergence", True
        if term == BREAKDOWN:
            pass
        elif conv_at is not None or lucky:
            if gate is not None and gate <= tol * scale:
                term, done = CONVERGED, True
            elif lucky and k == 0:
                term, done = LUCKY_BREAKDOWN, True
    return _finish(a, b, x, geom, hist, term, kind)


SOLVERS = {"cg": cg_pipelined, "bicgstab": bicgstab_pipelined, "gmres": gmres_pipelined}


# ---------------------------------------------------------------------------
# classical drivers (solvers.py:310-389, 485-580, 725-858): one BLAS op per
# step, scalars on the host.  NumPy expression order of linalg.py:403-457.
# ---------------------------------------------------------------------------


def cg_classical(a, b, x0=None, tol=1e-8, max_iterations=500, fixed=None,
                 geom=(DEFAULT_N_GROUPS, DEFAULT_GROUP_SIZE), btol=DEFAULT_BTOL, timing=None):
    """Restatement of solvers.cg_classical (solvers.py:310-389)."""
    a, b, x = _setup(a, b, x0)
    lbt = 0.0 if fixed else btol
    limit = fixed if fixed else max_iterations
    norm_b = math.sqrt(dot(b, b, geom))
    scale = norm_b if norm_b > 0 else 1.0
    r = b + (-1.0) * csr_spmv(a, x)  # add_scaled (linalg.py:451-457)
    p = r.copy()
    rr = dot(r, r, geom)
    hist = []
    term, kind = MAX_ITER, None
    if math.sqrt(rr) / scale <= tol and (not fixed or rr == 0.0):
        return _finish(a, b, x, geom, hist, CONVERGED, None)
    t0 = time.perf_counter()
    for _ in range(limit):
        q = csr_spmv(a, p)
        pap = dot(p, q, geom)
        if abs(pap) < lbt or pap == 0.0:  # pap == 0: ZeroDivisionError in the reference
            term, kind = BREAKDOWN, "pAp"
            break
        alpha = rr / pap
        x += alpha * p  # axpy (linalg.py:403-411)
        r += (-alpha) * q
        rr_new = dot(r, r, geom)
        mon = math.sqrt(rr_new) / scale
        hist.append(mon)
        if not math.isfinite(mon):
            term, kind = BREAKDOWN, "divergence"
            break
        if not fixed and mon <= tol:
            term = CONVERGED
            break
        beta = rr_new / rr
        p *= beta  # xpay (linalg.py:428-438): y *= beta; y += x
        p += r
        rr = rr_new
    if timing is not None:
        timing["loop_seconds"] = time.perf_counter() - t0
    return _finish(a, b, x, geom, hist, term, kind)


def bicgstab_classical(a, b, x0=None, tol=1e-8, max_iterations=500, fixed=None,
                       geom=(DEFAULT_N_GROUPS, DEFAULT_GROUP_SIZE), btol=DEFAULT_BTOL, timing=None):
    """Restatement of solvers.bicgstab_classical (solvers.py:485-580)."""
    a, b, x = _setup(a, b, x0)
    lbt = 0.0 if fixed else btol
    limit = fixed if fixed else max_iterations
    norm_b = math.sqrt(dot(b, b, geom))
    scale = norm_b if norm_b > 0 else 1.0
    r = b + (-1.0) * csr_spmv(a, x)
    r0s = r.copy()
    p = r.copy()
    rr = dot(r, r, geom)
    rho = dot(r, r0s, geom)
    hist = []
    term, kind = MAX_ITER, None
    if math.sqrt(rr) / scale <= tol and (not fixed or rr == 0.0):
        return _finish(a, b, x, geom, hist, CONVERGED, None)
    t0 = time.perf_counter()
    for _ in range(limit):
        ap = csr_spmv(a, p)
        apr = dot(ap, r0s, geom)
        if abs(apr) < lbt or apr == 0.0:
            term, kind = BREAKDOWN, "Apr0star"
            break
        alpha = rho / apr
        s = r + (-alpha) * ap
        ss = dot(s, s, geom)
        mon_s = math.sqrt(ss) / scale
        if not fixed and mon_s <= tol:
            x += alpha * p
            hist.append(mon_s)
            term = CONVERGED
            break
        as_ = csr_spmv(a, s)
        ass = dot(as_, s, geom)
        asas = dot(as_, as_, geom)
        asr = dot(as_, r0s, geom)
        if asas < lbt or asas == 0.0:
            term, kind = BREAKDOWN, "AsAs"
            break
        omega = ass / asas
        x += alpha * p + omega * s  # axpy2 (linalg.py:414-425)
        r = s + (-omega) * as_
        rho_new = dot(r, r0s, geom)
        rr = dot(r, r, geom)
        mon = math.sqrt(rr) / scale
        hist.append(mon)
        if not math.isfinite(mon):
            term, kind = BREAKDOWN, "divergence"
            break
        if not fixed and mon <= tol:
            term = CONVERGED
            break
        if abs(rho_new) < lbt:
            term, kind = BREAKDOWN, "rho"
            break
        if abs(omega) < lbt:
            term, kind = BREAKDOWN, "omega"
            break
        beta = -asr / apr
        p -= omega * ap  # _bicgstab_p_update (solvers.py:477-482)
        p *= beta
        p += r
        rho = rho_new
    if timing is not None:
        timing["loop_seconds"] = time.perf_counter() - t0
    return _finish(a, b, x, geom, hist, term, kind)


def gmres_classical(a, b, x0=None, tol=1e-8, max_iterations=500, fixed=None, restart=30, mgs=False,
                    geom=(DEFAULT_N_GROUPS, DEFAULT_GROUP_SIZE), btol=DEFAULT_BTOL, timing=None):
    """Restatement of solvers.gmres_classical (solvers.py:725-858), CGS
    (solvers.py:240-251) or MGS (solvers.py:221-237)."""
    a, b, x = _setup(a, b, x0)
    lbt = 0.0 if fixed else btol
    limit = fixed if fixed else max_iterations
    m = restart
    hist = []
    term, kind = MAX_ITER, None
    total = 0
    norm_b = None
    scale = 1.0
    done = False
    while not done and total < limit:
        if norm_b is None:
            norm_b = math.sqrt(dot(b, b, geom))
            scale = norm_b if norm_b > 0 else 1.0
        r = b + (-1.0) * csr_spmv(a, x)
        rho = math.sqrt(dot(r, r, geom))
        start_ok = rho > 0 and not (not fixed and rho / scale <= tol)
        if not start_ok:
            term = CONVERGED
            break
        r *= 1.0 / rho  # scale (linalg.py:441-448)
        basis, xi = [], []
        rmat = np.zeros((m, m))
        est2 = 1.0
        lucky = conv = False
        t0 = time.perf_counter()
        while len(basis) < m and total < limit:
            i = len(basis) + 1
            w = csr_spmv(a, basis[-1] if basis else r)
            coeffs = np.zeros(len(basis))
            if mgs:
                for j, q in enumerate(basis):
                    coeffs[j] = dot(q, w, geom)
                    w += (-coeffs[j]) * q
            else:
                for j, q in enumerate(basis):
                    coeffs[j] = dot(q, w, geom)
                for j, q in enumerate(basis):
                    w += (-coeffs[j]) * q
            for j, c in enumerate(coeffs):
                rmat[j, i - 1] = float(c)
            nrm = math.sqrt(dot(w, w, geom))
            if nrm < lbt or nrm == 0.0:
                lucky = True
                break
            rmat[i - 1, i - 1] = nrm
            w *= 1.0 / nrm
            basis.append(w)
            xi_i = dot(r, w, geom)
            xi.append(xi_i)
            r += (-xi_i) * w
            est2 = max(est2 - xi_i * xi_i, 0.0)
            mon = rho * math.sqrt(est2) / scale
            hist.append(mon)
            total += 1
            if not math.isfinite(mon):
                term, kind, done = BREAKDOWN, "divergence", True
                break
            if not fixed and mon <= tol:
                conv = True
                break
        if timing is not None:
            timing["loop_seconds"] = timing.get("loop_seconds", 0.0) + time.perf_counter() - t0
        k = len(basis)
        gate = None
        if k > 0 and term != BREAKDOWN:
            try:
                eta = solve_upper_triangular(rmat[:k, :k], np.asarray(xi), btol)
            except Breakdown as e:
                term, kind, done, eta = BREAKDOWN, e.kind, True, None
            if eta is not None:
                upd = eta[0] * r
                for idx in range(1, k + 1):
                    coeff = (eta[idx] if idx < k else 0.0) + eta[0] * xi[idx - 1]
                    upd += coeff * basis[idx - 1]
                x += rho * upd
                if conv or lucky:
                    gate = _true_residual(a, b, x, geom)
        if term == BREAKDOWN:
            pass
        elif conv or lucky:
            if gate is not None and gate <= tol * scale:
                term, done = CONVERGED, True
            elif lucky and k == 0:
                term, done = LUCKY_BREAKDOWN, True
    return _finish(a, b, x, geom, hist, term, kind)


CLASSICAL = {"cg": cg_classical, "bicgstab": bicgstab_classical, "gmres": gmres_classical}



# ---------------------------------------------------------------------------
# generators (io.py:201-275 for the Poisson families; convection-diffusion
# families are defined by this project)
# ---------------------------------------------------------------------------


def _stencil_csr(dims, diag, offsets):
    """Canonical CSR of a constant-coefficient stencil on a box grid, x
    fastest.  ``offsets`` = [(axis, step, value)], boundary neighbours
    dropped.  Columns come out strictly increasing per row."""
    dims = tuple(int(d) for d in dims)
    n = int(np.prod(dims))
    idx = np.arange(n, dtype=np.int64)
    coord = []
    stride = 1
    strides = []
    for d in dims:
        coord.append((idx // stride) % d)
        strides.append(stride)
        stride *= d
    entries = [(0, np.ones(n, dtype=bool), diag)]
    for axis, step, val in offsets:
        c = coord[axis]
        mask = (c + step >= 0) & (c + step < dims[axis])
        entries.append((step * strides[axis], mask, val))
    entries.sort(key=lambda e: e[0])
    counts = np.zeros(n, dtype=np.int64)
    for _, mask, _ in entries:
        counts += mask
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    cols = np.empty(int(rowptr[-1]), dtype=np.int64)
    vals = np.empty(int(rowptr[-1]))
    fill = rowptr[:-1].copy()
    for off, mask, val in entries:
        rows = idx[mask]
        cols[fill[rows]] = rows + off
        vals[fill[rows]] = val
        fill[rows] += 1
    return Csr(n, n, rowptr, cols, vals)


def poisson2d_side(side):
    """5-point 4/-1 Laplacian on side x side (io.py:201-229 with free side)."""
    return _stencil_csr((side, side), 4.0,
                        [(0, -1, -1.0), (0, 1, -1.0), (1, -1, -1.0), (1, 1, -1.0)]), np.ones(side * side)


def poisson2d(k):
    """Reference level k: side 2**(k+3)-1 (io.py:201-214)."""
    return poisson2d_side(2 ** (k + 3) - 1)


def poisson3d(side, diag=12.0, off=-2.0):
    """7-point Laplacian; defaults equal gen_poisson3d_block(side, 1)
    (io.py:232-275: (6/-1) * (1 + 1/1) = 12/-2)."""
    offs = [(ax, st, off) for ax in range(3) for st in (-1, 1)]
    return _stencil_csr((side, side, side), diag, offs), np.ones(side ** 3)


def convdiff2d(side, cx=1.0, cy=1.0):
    """First-order upwind convection-diffusion, h^2-scaled:
    diag 4 + h(cx+cy), west -1 - h cx, south -1 - h cy, east/north -1."""
    h = 1.0 / (side + 1)
    offs = [(0, -1, -1.0 - h * cx), (0, 1, -1.0), (1, -1, -1.0 - h * cy), (1, 1, -1.0)]
    return _stencil_csr((side, side), 4.0 + h * (cx + cy), offs), np.ones(side * side)


def convdiff3d(side, cx=1.0, cy=1.0, cz=1.0):
    """3D analogue of convdiff2d: diag 6 + h(cx+cy+cz), upwind minus faces."""
    h = 1.0 / (side + 1)
    offs = [(0, -1, -1.0 - h * cx), (0, 1, -1.0), (1, -1, -1.0 - h * cy), (1, 1, -1.0),
            (2, -1, -1.0 - h * cz), (2, 1, -1.0)]
    return _stencil_csr((side, side, side), 6.0 + h * (cx + cy + cz), offs), np.ones(side ** 3)


def poisson3d_block(side, block):
    """gen_poisson3d_block(side, block) restated (io.py:232-275): COO triplets
    of the 6/-1 Laplacian times I + ones/block, then lexicographic sort by
    (row, column) -- the canonical order CsrMatrix.from_coo produces
    (linalg.py:121-145); the triplets are unique so nothing is summed."""
    lap = poisson3d(side, 6.0, -1.0)[0]
    b = int(block)
    bmat = np.eye(b) + np.ones((b, b)) / b
    lrow = np.repeat(np.arange(lap.n_rows, dtype=np.int64), np.diff(lap.rowptr))
    st = np.arange(b * b, dtype=np.int64)
    rows = (np.repeat(lrow * b, b * b) + np.tile(st // b, lrow.size))
    cols = (np.repeat(lap.cols * b, b * b) + np.tile(st % b, lrow.size))
    vals = np.repeat(lap.vals, b * b) * np.tile(bmat.ravel(), lrow.size)
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    n = lap.n_rows * b
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rowptr[1:])
    return Csr(n, n, rowptr, cols, vals), np.ones(n)
