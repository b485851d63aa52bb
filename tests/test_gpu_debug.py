"""debug=True diagnostics (solvers.py:417-467, 606-673, 895-997) on the B200.

Every list the reference's drivers fill with debug=True -- CG rr_direct /
beta, BiCGStab s_dot_r0star / s_norm / identity_rr / direct_rr / r0star_norm,
GMRES ortho_offdiag -- must equal the reference's (tests/golden/
make_debug_golden.py) bit for bit, and the run itself must be unchanged by the
diagnostics.  Plus the reference's acceptance criterion 3 (recurrence
oracles, test_acceptance.py:151-178) evaluated on the B200 diagnostics."""

import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
GOLD = Path(__file__).resolve().parent / "golden"
NOISE_FLOOR = 1e-12  # test_acceptance.py:43


@pytest.fixture(scope="module")
def pk():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1410_4054_b200 as pk

    return pk


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


CASES = json.loads((GOLD / "debug_manifest.json").read_text())["cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_debug_diagnostics_match_reference(pk, case):
    store = np.load(GOLD / "debug_golden.npz")
    name = case["name"]
    a = pk.CsrMatrix(case["shape"][0], case["shape"][1], store[f"{name}/rowptr"], store[f"{name}/cols"],
                     store[f"{name}/vals"])
    b = store[f"{name}/b"]
    cfg = pk.SolverConfig(**case["config"])
    ctx = pk.ExecutionContext(*case["geom"])
    solver = pk.SOLVERS[(case["method"], "pipelined")]
    res = solver(a, b, config=cfg, context=ctx, debug=True)
    plain = solver(a, b, config=cfg, context=ctx)
    assert res.iterations == case["iterations"] == plain.iterations
    assert np.array_equal(bits(res.x), bits(plain.x))
    assert np.array_equal(bits(res.residual_history), bits(plain.residual_history))
    assert sorted(k for k, v in res.diagnostics.items() if isinstance(v, list)) == case["lists"]
    for key in case["lists"]:
        assert np.array_equal(bits(res.diagnostics[key]), bits(store[f"{name}/{key}"])), key
    for key, val in case["scalars"].items():
        assert res.diagnostics[key] == val, key


def test_acceptance_criterion_3_recurrence_oracles(pk):
    """test_acceptance.py:151-178 on the B200 diagnostics."""
    a, b = pk.gen_poisson2d(1)
    cfg = pk.SolverConfig(fixed_iterations=30, max_iterations=30)
    cg = pk.cg_pipelined(a, b, config=cfg, debug=True)
    rr, beta = cg.diagnostics["rr_direct"], cg.diagnostics["beta"]
    beta_gap = max(abs(beta[i] - rr[i + 1] / rr[i]) / abs(rr[i + 1] / rr[i]) for i in range(30))
    st = pk.bicgstab_pipelined(a, b, config=cfg, debug=True)
    d = st.diagnostics
    orth_gap = max(abs(sr) / (sn * d["r0star_norm"]) for sr, sn in zip(d["s_dot_r0star"], d["s_norm"]) if sn > 0)
    identity, direct = np.array(d["identity_rr"]), np.array(d["direct_rr"])
    above = direct > NOISE_FLOOR
    identity_gap = float((np.abs(identity - direct)[above] / direct[above]).max())
    assert beta_gap <= 1e-10 and orth_gap <= 1e-8 and identity_gap <= 1e-8
