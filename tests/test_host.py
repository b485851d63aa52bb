"""CPU-only checks: the C-ABI library loads and exports what the header
declares, host-side types validate like the reference, host generators equal
the oracle, and the device code is compiled without FP contraction."""

import re
import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_1410_4054_b200 as pk
from paper_1410_4054_b200 import _native as N
from oracle import pk_oracle as orc

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "pipekrylov_b200.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int)\s+(pk_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = N.lib()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(N.exported_symbols()) == declared
    assert lib.pk_abi_version() == 1


def test_no_gpu_fails_loudly_without_fallback():
    count = __import__("ctypes").c_int()
    if N.lib().pk_device_count(__import__("ctypes").byref(count)) == 0 and count.value > 0:
        pytest.skip("a GPU is present")
    a, b = pk.gen_poisson2d(1)
    with pytest.raises(N.NativeError):
        pk.cg_pipelined(a, b)


def test_csr_validation_matches_reference_rules():
    with pytest.raises(ValueError):
        pk.CsrMatrix(2, 2, [0, 1], [0], [1.0])  # wrong offsets length
    with pytest.raises(ValueError):
        pk.CsrMatrix(2, 2, [1, 1, 2], [0, 1], [1.0, 1.0])  # offsets start
    with pytest.raises(ValueError):
        pk.CsrMatrix(2, 2, [0, 2, 1], [0, 1], [1.0, 1.0])  # decreasing
    with pytest.raises(ValueError):
        pk.CsrMatrix(2, 2, [0, 1, 2], [0, 2], [1.0, 1.0])  # column range
    with pytest.raises(ValueError):
        pk.CsrMatrix(1, 3, [0, 2], [1, 1], [1.0, 1.0])  # not strictly increasing
    m = pk.CsrMatrix(2, 3, [0, 2, 4], [1, 2, 0, 1], [1.0, 2.0, 3.0, 4.0])  # reset at row start ok
    assert m.nnz == 4 and m.shape == (2, 3)
    dup = pk.CsrMatrix.from_coo(2, 2, [0, 0, 1], [1, 1, 0], [1.0, 2.0, 5.0])
    assert dup.nnz == 2 and dup.values.tolist() == [3.0, 5.0]
    with pytest.raises(AttributeError):
        m.n_rows = 5


def test_solver_config_validation():
    cfg = pk.SolverConfig()
    assert cfg.tolerance == 1e-8 and cfg.max_iterations == 500 and cfg.restart == 30
    for bad in ({"tolerance": 0.0}, {"max_iterations": 0}, {"restart": 0}, {"orthogonalization": "x"},
                {"breakdown_tolerance": 0.0}, {"fixed_iterations": 0}, {"loop_mode": "x"}):
        with pytest.raises(ValueError):
            pk.SolverConfig(**bad)
    f = pk.SolverConfig(fixed_iterations=7)
    assert f.fixed and f.iteration_limit() == 7 and f.loop_breakdown_tolerance() == 0.0


def test_execution_context_validation():
    with pytest.raises(ValueError):
        pk.ExecutionContext(n_groups=0)
    with pytest.raises(ValueError):
        pk.ExecutionContext(group_size=24)
    c = pk.ExecutionContext.one_per_lane(1_000_000, 4096)
    assert c.n_groups * c.group_size >= 1_000_000 and c.group_size == 4096


def test_solver_input_validation_before_device():
    spd = pk.CsrMatrix.from_dense([[4.0, 1.0], [1.0, 3.0]])
    with pytest.raises(ValueError):
        pk.cg_pipelined(pk.CsrMatrix.from_dense([[1.0, 2.0]]), [1.0])
    with pytest.raises(ValueError):
        pk.cg_pipelined(spd, [1.0, 2.0, 3.0])
    with pytest.raises(ValueError):
        pk.cg_pipelined(spd, [1.0, 2.0], x0=[1.0])
    with pytest.raises(ValueError):
        pk.gmres_pipelined(spd, [1.0, 2.0], config=pk.SolverConfig(orthogonalization=pk.MODIFIED_GS))
    with pytest.raises(ValueError):
        pk.solve(spd, [1.0, 2.0], tag=("cg", "sideways"))


def test_upper_triangular_solve_matches_reference_oracle():
    r = pk.UpperTriangular(2)
    r.set(0, 0, 2.0)
    r.set(0, 1, 1.0)
    r.set(1, 1, 4.0)
    assert np.array_equal(pk.solve_upper_triangular(r, [4.0, 8.0]), [1.0, 2.0])
    s = pk.UpperTriangular(2)
    s.set(0, 0, 1.0)
    with pytest.raises(pk.BreakdownError):
        pk.solve_upper_triangular(s, [1.0, 1.0])


@pytest.mark.parametrize("k", [1, 2, 3])
def test_host_poisson2d_equals_oracle(k):
    a, b = pk.gen_poisson2d(k)
    o, ob = orc.poisson2d(k)
    assert np.array_equal(a.row_offsets, o.rowptr) and np.array_equal(a.col_indices, o.cols)
    assert np.array_equal(a.values.view(np.uint64), o.vals.view(np.uint64)) and np.array_equal(b, ob)


@pytest.mark.parametrize("fam,side", [("convdiff2d", 9), ("convdiff2d", 33), ("convdiff3d", 6), ("convdiff3d", 11)])
def test_host_convdiff_equals_oracle(fam, side):
    a, _ = getattr(pk, fam)(side)
    o, _ = getattr(orc, fam)(side)
    assert np.array_equal(a.row_offsets, o.rowptr) and np.array_equal(a.col_indices, o.cols)
    assert np.array_equal(a.values.view(np.uint64), o.vals.view(np.uint64))


def test_host_poisson3d_equals_oracle():
    a, _ = pk.gen_poisson3d_block(7, 1)
    o, _ = orc.poisson3d(7)
    assert np.array_equal(a.col_indices, o.cols) and np.array_equal(a.values, o.vals)


@pytest.mark.skipif(shutil.which("nvcc") is None and not Path("/usr/local/cuda/bin/nvcc").exists(),
                    reason="nvcc not available")
def test_device_code_has_no_fp_contraction(tmp_path):
    """-fmad=false + explicit __d*_rn intrinsics: the PTX holds no fma.rn.f64
    (ptxas later expands div/sqrt into DFMA sequences, which are exact)."""
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    out = tmp_path / "pk.ptx"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-fmad=false", "-ptx",
                    f"-I{ROOT / 'include'}", f"-I{ROOT / 'paper_1410_4054_b200' / 'csrc'}",
                    str(ROOT / "paper_1410_4054_b200" / "csrc" / "pk_capi.cu"), "-o", str(out)], check=True,
                   capture_output=True)
    ptx = out.read_text()
    assert "fma.rn.f64" not in ptx
    assert ptx.count("add.rn.f64") > 100


@pytest.mark.parametrize("side,block", [(3, 2), (4, 3), (5, 1), (2, 5)])
def test_host_poisson3d_block_equals_oracle(side, block):
    """gen_poisson3d_block(n, block > 1) (io.py:232-275) vs the oracle's COO restatement."""
    a, b = pk.gen_poisson3d_block(side, block)
    oa, ob = orc.poisson3d_block(side, block)
    assert a.n_rows == oa.n_rows == side ** 3 * block
    assert np.array_equal(a.row_offsets, oa.rowptr) and np.array_equal(a.col_indices, oa.cols)
    assert np.array_equal(a.values.view(np.int64), oa.vals.view(np.int64))
    assert np.array_equal(b, ob)
