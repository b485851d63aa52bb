"""The reference's own test suites, run against the B200 drivers.

The unmodified reference tests (pkg/tests/test_solvers.py, test_acceptance.py,
copied to baseline/_ref_tests by oracle/install_reference.sh) are executed in
a subprocess with tests/ref_shim.py swapping the reference's driver functions
for this package's.  Expected outcome: every solver test passes; the only
failures allowed are the documented trace deviations (the B200
records its real launches/transfers, e.g. CG 1 launch + 0 transfers per
iteration instead of the emulator's 2 + 1)."""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
REF_TESTS = ROOT / "baseline" / "_ref_tests"

# reference tests whose assertion is on the emulator's launch / transfer
# accounting or byte pricing, not on results (documented deviation)
TRACE_ONLY = {
    "test_acceptance.py::test_criterion_1_launch_and_transfer_counts",
    "test_acceptance.py::test_criterion_4_cost_model_arithmetic",
}


def run_suite(files):
    if not (REF / "pipekrylov").exists() or not REF_TESTS.exists():
        pytest.skip("reference suite not installed (oracle/install_reference.sh)")
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT)])
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_refsuite")
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "tests.ref_shim", "-rA",
           "--rootdir", str(REF_TESTS), *[str(REF_TESTS / f) for f in files]]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=str(ROOT), timeout=1500)
    text = out.stdout + out.stderr
    failed = set()
    for m in re.finditer(r"^FAILED (\S+)", text, re.M):
        failed.add(m.group(1).split("/")[-1].split(" ")[0])
    passed = len(re.findall(r"^PASSED ", text, re.M))
    return out.returncode, failed, passed, text


def test_reference_solver_suite_against_b200():
    rc, failed, passed, text = run_suite(["test_solvers.py"])
    print(text[-3000:])
    assert not failed, failed
    assert passed > 30 and rc == 0


def test_reference_acceptance_suite_against_b200():
    rc, failed, passed, text = run_suite(["test_acceptance.py"])
    print(text[-4000:])
    unexpected = {f for f in failed if f.split("[")[0] not in TRACE_ONLY}
    assert not unexpected, unexpected
    assert passed >= 5
