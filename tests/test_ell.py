"""ELLPACK storage + SpMV (paper_1410_4054_b200.ell; linalg.py:179-246,
_spmvkernels.py:21-34): the reference's ELL = CSR bitwise contract
(test_linalg.py:119-137), on the oracle (CPU) and on the B200 kernel (gpu)."""

import numpy as np
import pytest

from oracle import pk_oracle as orc
from paper_1410_4054_b200 import CsrMatrix
from paper_1410_4054_b200.ell import EllMatrix, csr_to_ell, ell_to_csr
from paper_1410_4054_b200.mmio import gen_random_rowwise
from tests import golden_data as gd


def ragged(seed=4, n=700, m=650):
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((n, m))
    d[rng.random((n, m)) > 0.02] = 0.0
    d[5] = 0.0                    # empty row
    d[9, :300] = rng.standard_normal(300)  # one long row
    return CsrMatrix.from_dense(d)


def test_round_trip_and_layout():
    a = ragged()
    e = csr_to_ell(a)
    assert e.width == int(a.row_nnz().max()) and e.nnz == a.nnz
    assert ell_to_csr(e).equals(a)
    # slot k of row i lives at i + k n_rows; padding = sentinel n_cols, value 0
    i = 9
    lo, hi = a.row_offsets[i], a.row_offsets[i + 1]
    assert np.array_equal(e.col_indices[i + np.arange(hi - lo) * a.n_rows], a.col_indices[lo:hi])
    assert np.all(e.col_indices[5 + np.arange(e.width) * a.n_rows] == a.n_cols)


def test_validation():
    with pytest.raises(ValueError):
        EllMatrix(2, 2, 1, [0, 3], [1.0, 1.0])      # column out of range
    with pytest.raises(ValueError):
        EllMatrix(2, 2, 1, [0, 2], [1.0, 1.0])      # padded slot with a value
    with pytest.raises(ValueError):
        EllMatrix(2, 2, 2, [0, 1], [1.0, 1.0])      # wrong entry count


def test_oracle_ell_equals_golden_csr_product():
    """ELL product of the golden matrix == the reference's own spmv_csr
    output stored in the fixtures (bitwise)."""
    f = gd.fused()
    n, m, rp, cols, vals = gd.csr_arrays(f, "A")
    e = csr_to_ell(CsrMatrix(n, m, rp, cols, vals))
    q = orc.ell_spmv(e.n_rows, e.n_cols, e.width, e.col_indices, e.values, f["vec/x"])
    assert np.array_equal(q.view(np.int64), f["g0/spmv_plain"].view(np.int64))


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["ragged", "random5", "random40", "convdiff"])
def test_gpu_ell_spmv_equals_csr(which):
    import torch

    import paper_1410_4054_b200 as pk

    if which == "ragged":
        a = ragged()
    elif which == "convdiff":
        a, _ = pk.convdiff2d(300)
    else:
        a, _ = gen_random_rowwise(5000, int(which[6:]), seed=1)
    x = np.random.default_rng(3).standard_normal(a.n_cols)
    xd = torch.from_numpy(x).cuda()
    q_ell = pk.spmv_ell(csr_to_ell(a), xd).cpu().numpy()
    ref = orc.csr_spmv(a, x)
    assert np.array_equal(q_ell.view(np.int64), ref.view(np.int64))
    from paper_1410_4054_b200 import fused
    q_csr = fused.spmv(a, xd).cpu().numpy()
    assert np.array_equal(q_ell.view(np.int64), q_csr.view(np.int64))
