"""pytest plugin: run the reference's OWN solver tests against the B200 drivers.

Loaded with ``-p tests.ref_shim`` by tests/test_gpu_reference_suite.py when
the reference's test files are available (baseline/_ref_tests, copied there by
oracle/install_reference.sh).  Before any test module is imported it replaces
the driver functions in the reference package's namespaces with this
package's, so ``from pipekrylov.solvers import cg_pipelined`` inside the
reference's tests binds the B200 implementation:

* the pipelined drivers -> libpk_b200 device loops (solvers.py here);
* the classical drivers -> the reference loops on B200 kernels (classical.py).

Everything else the tests import (CsrMatrix, SolverConfig, generators, the
cost model, ...) stays the reference's own; the B200 drivers accept the
reference's objects (CsrMatrix / SolverConfig / ExecutionContext are coerced).
"""

import pipekrylov
import pipekrylov.solvers as ref_solvers

import paper_1410_4054_b200 as b200

_DRIVERS = ("cg_pipelined", "bicgstab_pipelined", "gmres_pipelined",
            "cg_classical", "bicgstab_classical", "gmres_classical")


def pytest_configure(config):
    for name in _DRIVERS:
        fn = getattr(b200, name)
        setattr(ref_solvers, name, fn)
        setattr(pipekrylov, name, fn)
    for (method, variant) in list(pipekrylov.SOLVERS):
        pipekrylov.SOLVERS[(method, variant)] = getattr(b200, f"{method}_{variant}")
