"""B200-native pipelined Krylov solvers (CG, BiCGStab, GMRES(m); CSR, fp64).

A drop-in for the pipelined solve path of the reference package
``pipekrylov`` (arXiv 1410.4054): the same driver names and signatures, the
same result/config/context/trace types, bit-identical results at the same
reduction geometry -- computed by hand-written sm_100a kernels in
libpk_b200.so (C ABI in include/pipekrylov_b200.h), with no CPU fallback.
"""

from .device import DeviceContext, DeviceMatrix, context_for, device_matrix
from .generators import (
    convdiff2d,
    convdiff3d,
    gen_poisson2d,
    gen_poisson3d_block,
    poisson2d_grid,
    poisson3d_grid,
)
from .partition import PartitionedCG, cg_partitioned, slab_geometry
from .linalg import (
    DEFAULT_CONTEXT,
    CsrMatrix,
    ExecutionContext,
    ExecutionTrace,
    PhaseRecord,
    WorkgroupPartials,
    as_vector,
)
from .solvers import (
    BREAKDOWN,
    CLASSICAL_GS,
    CONVERGED,
    DEFAULT_BREAKDOWN_TOLERANCE,
    LUCKY_BREAKDOWN,
    LuckyBreakdown,
    MAX_ITER,
    MODIFIED_GS,
    SOLVERS,
    BreakdownError,
    SolverConfig,
    SolverResult,
    UpperTriangular,
    bicgstab_pipelined,
    cg_pipelined,
    gmres_pipelined,
    host_array,
    launch_floor,
    solve,
    solve_batch,
    solve_upper_triangular,
)

from .mmio import MatrixMarketError, gen_random_rowwise, gen_system, read_matrix_market, write_matrix_market  # noqa: E402
from .ell import EllMatrix, csr_to_ell, ell_to_csr, spmv_ell  # noqa: E402
from .execmodel import DeviceProfile, LatencyBarrier, calibrate_b200, latency_barrier, predict_iteration_time, speedup_curve  # noqa: E402,E501
from .fused import (  # noqa: E402  kernel-level ops on CUDA tensors (fused.py / linalg.py mirrors)
    FusedReductionRequest,
    dot,
    fused_bicgstab_s_update,
    fused_bicgstab_xrp_update,
    fused_cg_vector_update,
    fused_gs_normalize,
    fused_gs_stage1,
    fused_gs_update,
    reduce_stage1,
    reduce_stage2,
    spmv_csr,
    spmv_fused,
)
from .classical import bicgstab_classical, cg_classical, gmres_classical, orthogonalize_mgs  # noqa: E402

# the reference's classical drivers (solvers.py:310-389, 485-580, 725-858) on
# the same B200 kernels: SOLVERS[(method, "classical")], as in the reference
SOLVERS.update({
    ("cg", "classical"): cg_classical,
    ("bicgstab", "classical"): bicgstab_classical,
    ("gmres", "classical"): gmres_classical,
})

__version__ = "0.1.0"

__all__ = [
    "BREAKDOWN", "CLASSICAL_GS", "CONVERGED", "DEFAULT_BREAKDOWN_TOLERANCE", "DEFAULT_CONTEXT",
    "LUCKY_BREAKDOWN", "MAX_ITER", "MODIFIED_GS", "PartitionedCG", "SOLVERS", "BreakdownError", "CsrMatrix",
    "DeviceContext", "DeviceMatrix", "ExecutionContext", "ExecutionTrace", "PhaseRecord", "SolverConfig",
    "SolverResult", "UpperTriangular", "WorkgroupPartials", "as_vector", "bicgstab_classical", "bicgstab_pipelined",
    "cg_classical", "gmres_classical", "orthogonalize_mgs", "MatrixMarketError", "gen_random_rowwise",
    "gen_system", "read_matrix_market", "write_matrix_market", "EllMatrix", "csr_to_ell", "ell_to_csr", "spmv_ell",
    "DeviceProfile", "LatencyBarrier", "calibrate_b200", "latency_barrier", "predict_iteration_time", "speedup_curve",
    "cg_partitioned", "cg_pipelined", "context_for", "convdiff2d", "convdiff3d", "device_matrix", "gen_poisson2d",
    "gen_poisson3d_block", "gmres_pipelined", "poisson2d_grid", "poisson3d_grid", "solve", "solve_batch",
    "slab_geometry", "solve_upper_triangular", "__version__", "LuckyBreakdown", "FusedReductionRequest", "dot",
    "fused_bicgstab_s_update", "fused_bicgstab_xrp_update", "fused_cg_vector_update", "fused_gs_normalize",
    "fused_gs_stage1", "fused_gs_update", "reduce_stage1", "reduce_stage2", "spmv_csr", "spmv_fused", "host_array", "launch_floor",
]
