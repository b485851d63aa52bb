"""Matrix Market ingestion + unstructured random family (paper_1410_4054_b200.mmio).

Behaviour follows the reference's io tests (test_io.py:33-170, 208-241);
arrays are pinned to the reference's own generator output stored in the
golden fixtures, and diffed live against the reference when importable."""

import importlib
import sys

import numpy as np
import pytest

from paper_1410_4054_b200 import CsrMatrix
from paper_1410_4054_b200.mmio import (MatrixMarketError, gen_random_rowwise, gen_system, read_matrix_market,
                                       write_matrix_market)
from tests import golden_data as gd
from tests.conftest import REFERENCE_SRC, reference_available


def write_mm(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_read_general_real(tmp_path):
    p = write_mm(tmp_path, "%%MatrixMarket matrix coordinate real general\n% a comment\n\n2 3 3\n"
                           "1 1 4.5\n2 3 -1.0\n1 2 2.0\n")
    a = read_matrix_market(p)
    assert a.shape == (2, 3)
    assert np.array_equal(a.to_dense(), [[4.5, 2.0, 0.0], [0.0, 0.0, -1.0]])


def test_read_symmetric_expands_off_diagonals(tmp_path):
    p = write_mm(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2.0\n2 1 5.0\n2 2 3.0\n")
    a = read_matrix_market(p)
    assert a.nnz == 4 and np.array_equal(a.to_dense(), [[2.0, 5.0], [5.0, 3.0]])


def test_read_pattern_and_integer_fields(tmp_path):
    a = read_matrix_market(write_mm(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 1\n2 1\n"))
    assert np.array_equal(a.to_dense(), [[1.0, 0.0], [1.0, 0.0]])
    b = read_matrix_market(write_mm(tmp_path, "%%MatrixMarket matrix coordinate integer general\n1 2 1\n1 2 7\n",
                                    "i.mtx"))
    assert np.array_equal(b.to_dense(), [[0.0, 7.0]])


def test_read_sums_duplicate_entries(tmp_path):
    a = read_matrix_market(write_mm(tmp_path, "%%MatrixMarket matrix coordinate real general\n2 2 3\n"
                                              "1 1 1.5\n1 1 2.25\n2 2 1.0\n"))
    assert a.nnz == 2 and a.to_dense()[0, 0] == 3.75


@pytest.mark.parametrize("header", [
    "%%MatrixMarket matrix array real general",
    "%%MatrixMarket vector coordinate real general",
    "%%MatrixMarket matrix coordinate complex general",
    "%%MatrixMarket matrix coordinate real hermitian",
    "not a matrix market file",
])
def test_read_rejects_unsupported_headers(tmp_path, header):
    with pytest.raises(MatrixMarketError) as info:
        read_matrix_market(write_mm(tmp_path, header + "\n1 1 1\n1 1 1.0\n"))
    assert info.value.line == 1 and isinstance(info.value, ValueError)


def test_read_reports_line_of_bad_entry(tmp_path):
    p = write_mm(tmp_path, "%%MatrixMarket matrix coordinate real general\n% padding comment\n2 2 2\n"
                           "1 1 1.0\n3 1 2.0\n")
    with pytest.raises(MatrixMarketError) as info:
        read_matrix_market(p)
    assert info.value.line == 5 and "line 5" in str(info.value)


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix coordinate real general\n1 1 1\n1.5 1 2.0\n",       # fractional index
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n1 2 3.0\n",       # above the diagonal
    "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n",  # entry count
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n",           # malformed value
    "%%MatrixMarket matrix coordinate real general\n2 2\n",                     # size line
])
def test_read_rejects_malformed(tmp_path, text):
    with pytest.raises(MatrixMarketError):
        read_matrix_market(write_mm(tmp_path, text))


def test_write_read_round_trip_is_bitwise(tmp_path):
    rng = np.random.default_rng(2)
    dense = rng.standard_normal((7, 5))
    dense[rng.random((7, 5)) > 0.4] = 0.0
    a = CsrMatrix.from_dense(dense)
    write_matrix_market(tmp_path / "r.mtx", a, comment="written by the test suite")
    back = read_matrix_market(tmp_path / "r.mtx")
    assert back.equals(a)
    write_matrix_market(tmp_path / "r2.mtx", back)
    assert (tmp_path / "r2.mtx").read_text().splitlines()[2:] == (tmp_path / "r.mtx").read_text().splitlines()[3:]


def test_random_rowwise_matches_reference_arrays():
    """golden cg_random/A = the reference's gen_random_rowwise(2000, 5, seed=3)."""
    a, b = gen_random_rowwise(2000, 5, seed=3)
    _, _, rp, cols, vals = gd.csr_arrays(gd.solvers(), "cg_random/A")
    assert np.array_equal(a.row_offsets, rp) and np.array_equal(a.col_indices, cols)
    assert np.array_equal(a.values.view(np.int64), vals.view(np.int64))
    assert np.array_equal(b, np.ones(2000))
    assert np.array_equal(a.row_nnz(), np.full(2000, 5))


def test_random_rowwise_validation_and_specs():
    with pytest.raises(ValueError):
        gen_random_rowwise(0, 1)
    with pytest.raises(ValueError):
        gen_random_rowwise(5, 6)
    _, _, label = gen_system("random:50,4")
    assert label == "random:50,4,0"
    _, _, label = gen_system("poisson2d:1")
    assert label == "poisson2d:1"
    with pytest.raises(ValueError):
        gen_system("nope:1")


@pytest.mark.reference
def test_against_live_reference(tmp_path):
    if not reference_available():
        pytest.skip("reference not importable here")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    ref = importlib.import_module("pipekrylov")
    for n, k, seed in ((40, 30, 1), (300, 7, 9)):  # dense and sparse sampling
        ra, _ = ref.gen_random_rowwise(n, k, seed)
        oa, _ = gen_random_rowwise(n, k, seed)
        assert np.array_equal(ra.row_offsets, oa.row_offsets) and np.array_equal(ra.col_indices, oa.col_indices)
        assert np.array_equal(ra.values, oa.values)
        p = tmp_path / f"r{n}.mtx"
        ref.write_matrix_market(p, ra)
        assert read_matrix_market(p).equals(oa)
    sym = write_mm(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 2\n3 1 0.1\n3 3 1e-3\n"
                             "2 2 7 % inline\n", "s.mtx")
    r, o = ref.read_matrix_market(sym), read_matrix_market(sym)
    assert np.array_equal(r.to_dense(), o.to_dense())
