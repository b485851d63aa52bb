/*
 * pipekrylov_b200 -- C ABI of the B200-native pipelined Krylov hot path.
 *
 * This is the drop-in boundary for the reference package `pipekrylov`
 * (arXiv 1410.4054 emulation).  The reference is pure Python and has no FFI
 * of its own; each entry point below replaces one reference interface, cited
 * as file:line under /root/reference/pkg/src/pipekrylov/.  The Python mirror
 * (paper_1410_4054_b200/) binds these with ctypes; INTEGRATION.md shows the
 * binding a reference maintainer would add.
 *
 * Conventions
 *   - Every function returns PK_OK (0) or a PK_ERR_* code; pk_last_error()
 *     returns a thread-local message.  No C++ exception crosses the ABI.
 *   - PK_ERR_INVALID maps to the reference's ValueError (solvers.py:259-269,
 *     linalg.py:53-111); numerical breakdowns never surface as errors, they
 *     are reported in pk_result.termination / breakdown_kind
 *     (solvers.py:95-98, errors.py:6-27).
 *   - "host" pointers are ordinary CPU memory owned by the caller;
 *     "device" pointers are CUDA global memory on the context's device
 *     (e.g. torch.Tensor.data_ptr()).  Kernel-level entries run on the
 *     context's stream and do not synchronize.
 *   - All arithmetic is IEEE binary64 without contraction; results are
 *     bit-identical to the reference at the same reduction geometry.
 */
#ifndef PIPEKRYLOV_B200_H
#define PIPEKRYLOV_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PK_ABI_VERSION 1

/* status codes */
#define PK_OK 0
#define PK_ERR_INVALID 1     /* bad argument -> ValueError */
#define PK_ERR_CUDA 2        /* CUDA runtime failure */
#define PK_ERR_NOMEM 3       /* device allocation failed */
#define PK_ERR_UNSUPPORTED 4 /* valid but not implemented on this path */

/* termination (solvers.py:95-98) */
#define PK_TERM_CONVERGED 0
#define PK_TERM_MAX_ITER 1
#define PK_TERM_BREAKDOWN 2
#define PK_TERM_LUCKY_BREAKDOWN 3

/* breakdown kinds (errors.py:6-27, solvers.py) */
#define PK_BK_NONE 0
#define PK_BK_PAP 1
#define PK_BK_APR0STAR 2
#define PK_BK_ASAS 3
#define PK_BK_DIVERGENCE 4
#define PK_BK_SINGULAR_R 5

/* methods (keys of SOLVERS, __init__.py:81-88, pipelined variants) */
#define PK_METHOD_CG 0
#define PK_METHOD_BICGSTAB 1
#define PK_METHOD_GMRES 2

/* spmv_fused quantity kinds (fused.py:51-83) */
#define PK_DOT_INPUT 0  /* <Ap, p>  "input"  */
#define PK_DOT_RESULT 1 /* <Ap, Ap> "result" */
#define PK_DOT_VECTOR 2 /* <Ap, w>  fixed vector */

/* device-side generator families (io.py:201-275 + DESIGN.md "Inputs") */
#define PK_GEN_POISSON2D 0  /* dims {nx, ny}; coef {diag, off}         */
#define PK_GEN_POISSON3D 1  /* dims {nx, ny, nz}; coef {diag, off}     */
#define PK_GEN_CONVDIFF2D 2 /* dims {side, side}; coef {cx, cy}         */
#define PK_GEN_CONVDIFF3D 3 /* dims {side, side, side}; coef {cx,cy,cz} */

/* loop drivers */
#define PK_LOOP_GRAPH 0 /* CUDA graph with a conditional WHILE node (default) */
#define PK_LOOP_HOST 1  /* host-enqueued launches, device-side stop flag       */

typedef struct pk_ctx pk_ctx; /* device + stream + reduction geometry */
typedef struct pk_mat pk_mat; /* device-resident CSR matrix           */
typedef struct pk_dcg pk_dcg; /* row-partitioned CG solver (C4)       */
typedef struct pk_ell pk_ell; /* device-resident ELLPACK matrix       */

/* SolverConfig (solvers.py:104-145).  fixed_iterations <= 0 means None. */
typedef struct pk_config {
  double tolerance;
  int64_t max_iterations;
  int64_t restart;
  double breakdown_tolerance;
  int64_t fixed_iterations;
  int32_t loop_mode;
  int32_t flags;                /* PK_FLAG_* */
} pk_config;

/* pk_config.flags */
#define PK_FLAG_PROFILE 1 /* PK_LOOP_HOST only: CUDA-event time of every loop
                             kernel, returned in pk_result.kernel_* (bench) */

/* SolverResult (solvers.py:148-171) plus real launch/transfer counts for
 * the ExecutionTrace (execmodel.py:110-185). */
typedef struct pk_result {
  int64_t iterations;
  int32_t termination;
  int32_t breakdown_kind;
  double true_final_residual;
  double loop_seconds;          /* CUDA-event time of the iteration loop(s) */
  int64_t setup_launches;
  int64_t setup_transfers;
  int64_t launches_per_iteration; /* steady state; GMRES: step >= 2 */
  int64_t transfers_per_iteration;
  int64_t finish_launches;
  int64_t finish_transfers;
  int64_t total_launches;
  int64_t total_transfers;
  int64_t cycles;               /* GMRES restart cycles */
  int64_t check_phases;         /* BiCGStab true-residual confirmations */
  /* PK_FLAG_PROFILE: per loop-kernel slot (CG: 0 = fused step; BiCGStab:
   * 0 = As-SpMV, 1 = xrp+Ap-SpMV) summed event time and launch count */
  double kernel_seconds[4];
  int64_t kernel_launches[4];
} pk_result;

/* GMRES host triangular solve R eta = xi (solvers.py:205-218).  R is the
 * leading k x k block, row major with leading dimension ld.  Return 0 on
 * success, 1 for a singular diagonal (BreakdownError "singular_R"). */
typedef int (*pk_trisolve_fn)(void* user, int64_t k, const double* R, int64_t ld,
                              const double* xi, double breakdown_tolerance, double* eta);

/* Per-iteration diagnostics (the reference's debug=True side computations,
 * solvers.py:417-467, 606-673, 895-997).  Registered on a context with
 * pk_ctx_set_debug; while set, solves on that context run their loop from the
 * host one iteration at a time (same kernels, same bits) and call the hook
 * with HOST copies of the vectors the reference inspects:
 *   PK_DBG_CG_SETUP   v0 = r after setup; scal = {beta} if the loop runs
 *   PK_DBG_CG_ITER    v0 = r after the update; scal = {beta} unless stopping
 *   PK_DBG_BICG_SETUP v0 = r0*
 *   PK_DBG_BICG_S     v0 = r, v1 = Ap, scal = {alpha} (s = r - alpha Ap)
 *   PK_DBG_BICG_XRP   v0 = r after the xrp update; scal = {identity}
 *   PK_DBG_GMRES_CYCLE v0 = the cycle's k basis vectors, row-major k x n;
 *                     scal = {k}
 * Return 0 to continue.  The hook runs on the solving host thread. */
typedef int (*pk_debug_fn)(void* user, int32_t event, int64_t iteration, const double* v0,
                           const double* v1, int64_t n, const double* scal, int32_t nscal);
#define PK_DBG_CG_SETUP 1
#define PK_DBG_CG_ITER 2
#define PK_DBG_BICG_SETUP 3
#define PK_DBG_BICG_S 4
#define PK_DBG_BICG_XRP 5
#define PK_DBG_GMRES_CYCLE 6

/* ---- library ---------------------------------------------------------- */
const char* pk_last_error(void);
int pk_abi_version(void);
int pk_device_count(int* count);

/* ExecutionContext (execmodel.py:188-207): n_groups >= 1, group_size a
 * power of two.  Creates a non-blocking stream on `device`. */
int pk_ctx_create(int device, int64_t n_groups, int64_t group_size, pk_ctx** out);
int pk_ctx_destroy(pk_ctx* ctx);
/* hook NULL: back to device-resident loops without diagnostics */
int pk_ctx_set_debug(pk_ctx* ctx, pk_debug_fn hook, void* user);
/* Run kernel-level entries on `stream` (a cudaStream_t; NULL is the legacy
 * default stream, as everywhere in CUDA).  pk_ctx_reset_stream restores the
 * context's private non-blocking stream. */
int pk_ctx_set_stream(pk_ctx* ctx, void* stream);
int pk_ctx_reset_stream(pk_ctx* ctx);
int pk_ctx_synchronize(pk_ctx* ctx);
int pk_ctx_geometry(const pk_ctx* ctx, int64_t* n_groups, int64_t* group_size);

/* ---- matrices (CsrMatrix, linalg.py:71-176) --------------------------- */
/* Host CSR upload with the reference's canonical-form validation
 * (linalg.py:86-111): int64 offsets/columns are narrowed to int32 on the
 * device (offsets stay 64-bit when nnz >= 2^31). */
int pk_csr_upload(pk_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_offsets,
                  const int64_t* col_indices, const double* values, pk_mat** out);
/* Build a stencil matrix directly in HBM (gen_poisson2d / gen_poisson3d_block
 * io.py:201-275 and the convection-diffusion families). */
int pk_csr_generate(pk_ctx* ctx, int32_t family, const int64_t* dims, int32_t ndims,
                    const double* coef, int32_t ncoef, pk_mat** out);
/* Rows [row_lo, row_hi) of a generator family with columns stored as
 * (global column - col_base) and n_cols_local columns: the local block of a
 * row partition with halo. */
int pk_csr_generate_rows(pk_ctx* ctx, int32_t family, const int64_t* dims, int32_t ndims,
                         const double* coef, int32_t ncoef, int64_t row_lo, int64_t row_hi,
                         int64_t col_base, int64_t n_cols_local, pk_mat** out);
int pk_csr_info(const pk_mat* mat, int64_t* n_rows, int64_t* n_cols, int64_t* nnz,
                int64_t* max_row_nnz);
/* Copy the CSR arrays back to host (generator-equality tests). */
int pk_csr_download(pk_ctx* ctx, const pk_mat* mat, int64_t* row_offsets, int64_t* col_indices,
                    double* values);
int pk_mat_destroy(pk_mat* mat);

/* Storage the kernels walk (the CSR arrays always stay resident):
 *   PK_FMT_CSR     row_offsets / columns / values (thread-per-row walk);
 *   PK_FMT_SELL32  an additional SELL-32 copy: 32-row slices, slot-major,
 *                  padded to the slice's longest row (column -1), so a warp's
 *                  32 rows read every slot as one coalesced segment.  Same
 *                  entries in the same order: bit-identical results.
 * New matrices get the context default (SELL-32 unless PK_SELL=0).
 * Replaces nothing in the reference (its CsrMatrix is CSR only,
 * linalg.py:71-176); it is the GPU layout of the same matrix. */
#define PK_FMT_CSR 0
#define PK_FMT_SELL32 1
int pk_mat_set_format(pk_ctx* ctx, pk_mat* mat, int32_t format);
int pk_mat_get_format(const pk_mat* mat, int32_t* format, int64_t* stored_entries);

/* ---- kernel-level entries (device pointers; fused.py / linalg.py) ------ */
/* spmv_csr (linalg.py:373-380). */
int pk_spmv(pk_ctx* ctx, const pk_mat* a, const double* p, double* q);
/* spmv_fused (fused.py:86-120): q = A p and stage-1 partials of nq (1..4)
 * dots; kinds[i] in PK_DOT_*; w[i] a device vector for PK_DOT_VECTOR.
 * partials is device (n_groups x nq), row major. */
int pk_spmv_fused(pk_ctx* ctx, const pk_mat* a, const double* p, double* q, int32_t nq,
                  const int32_t* kinds, const double* const* w, double* partials);
/* reduce_stage1 (linalg.py:323-337) of nq contribution columns, each a
 * device vector of length n; partials (n_groups x nq). */
int pk_reduce_stage1(pk_ctx* ctx, int64_t n, int32_t nq, const double* const* columns,
                     double* partials);
/* reduce_stage2 (linalg.py:340-348): serial sum over groups on the device;
 * totals is device [nq]. */
int pk_reduce_stage2(pk_ctx* ctx, int32_t nq, const double* partials, double* totals);
/* dot (linalg.py:351-365): total written to device *total. */
int pk_dot(pk_ctx* ctx, int64_t n, const double* x, const double* y, double* total);
/* ELLPACK (linalg.py:179-246): width slots per row, column-major (slot k
 * of row i at i + k n_rows), padded slots carry the sentinel column n_cols
 * and value 0.  pk_ell_upload validates like EllMatrix.__post_init__
 * (linalg.py:193-208) and stores int32 columns + fp64 values in HBM. */
int pk_ell_upload(pk_ctx* ctx, int64_t n_rows, int64_t n_cols, int64_t width, const int64_t* col_indices,
                  const double* values, pk_ell** out);
int pk_ell_destroy(pk_ell* ell);
/* spmv_ell (linalg.py:383-390, _spmvkernels.py:21-34): thread per row,
 * coalesced slot loads, padded slots skipped -> bit-identical to pk_spmv on
 * the same matrix in CSR form. */
int pk_spmv_ell(pk_ctx* ctx, const pk_ell* a, const double* p, double* q);

/* Classical-driver vector updates, one launch each (linalg.py:403-457,
 * solvers.py:277-280, 477-482), IEEE mul/add with no contraction, in the
 * NumPy expression order of the reference:
 *   PK_VEC_AXPY        y = y + (alpha x)                     axpy
 *   PK_VEC_AXPY2       y = y + ((alpha x) + (beta z))        axpy2
 *   PK_VEC_XPAY        y = (y beta) + x                      xpay
 *   PK_VEC_SCALE       y = y alpha                           scale
 *   PK_VEC_ADD_SCALED  y = x + (alpha z)    (y a fresh output) add_scaled
 *   PK_VEC_BICG_P      y = ((y - (beta z)) alpha) + x        _bicgstab_p_update
 *   PK_VEC_COPY        y = x                                 _device_copy
 * Unused vector arguments may be NULL. */
enum {
  PK_VEC_AXPY = 0,
  PK_VEC_AXPY2 = 1,
  PK_VEC_XPAY = 2,
  PK_VEC_SCALE = 3,
  PK_VEC_ADD_SCALED = 4,
  PK_VEC_BICG_P = 5,
  PK_VEC_COPY = 6
};
int pk_vec_update(pk_ctx* ctx, int32_t kind, int64_t n, double* y, const double* x, const double* z,
                  double alpha, double beta);
/* fused_cg_vector_update (fused.py:123-151). */
int pk_cg_update(pk_ctx* ctx, int64_t n, double* x, double* r, double* p, const double* ap,
                 double alpha, double beta, double* partials);
/* fused_bicgstab_s_update (fused.py:154-182): alpha finalized from the two
 * partials blocks on the device.  *breakdown (device int) = 1 when
 * |<Ap,r0*>| < btol, in which case s is not written.  alpha_out device. */
int pk_bicg_s_update(pk_ctx* ctx, int64_t n, const double* r, const double* ap,
                     const double* rr0_partials, const double* apr_partials, double btol,
                     double* s, double* partials, double* alpha_out, int32_t* breakdown);
/* fused_bicgstab_xrp_update (fused.py:185-219). */
int pk_bicg_xrp_update(pk_ctx* ctx, int64_t n, double* x, double* r, double* p, const double* s,
                       const double* ap, const double* as, double alpha, double omega,
                       double beta, const double* r0star, double* partials);
/* fused_gs_stage1 (fused.py:222-243): partials (n_groups x nb) of <b_j, v>. */
int pk_gs_stage1(pk_ctx* ctx, int64_t n, int32_t nb, const double* const* basis, const double* v,
                 double* partials);
/* fused_gs_update (fused.py:246-277): coeffs (device [nb]) finalized from
 * partials (n_groups x nb); v -= sum_j c_j b_j; norm partials (n_groups). */
int pk_gs_update(pk_ctx* ctx, int64_t n, double* v, int32_t nb, const double* const* basis,
                 const double* partials, double* coeffs, double* norm_partials);
/* fused_gs_normalize (fused.py:280-305): *norm_out (device) = ||v||,
 * *lucky (device int) = 1 when ||v|| < btol (v untouched). */
int pk_gs_normalize(pk_ctx* ctx, int64_t n, double* v, const double* norm_partials,
                    const double* r, double btol, double* norm_out, int32_t* lucky,
                    double* partials);

/* ---- solver-level entry (host buffers) -------------------------------- */
/* SOLVERS[(method, "pipelined")](a, b, x0, config, context)
 * (solvers.py:395-469, 583-712, 865-1008).  b, x0 (nullable), x_out: host
 * [n].  hist_out: host, capacity hist_cap (>= iteration limit).  For GMRES,
 * trisolve (nullable) computes eta on the host exactly as the reference
 * does (NumPy np.dot); NULL uses a serial dot. */
int pk_solve(pk_ctx* ctx, const pk_mat* a, int32_t method, const double* b, const double* x0,
             const pk_config* config, pk_trisolve_fn trisolve, void* trisolve_user,
             double* x_out, double* hist_out, int64_t hist_cap, pk_result* result);

/* Same as pk_solve but b, x0 and x_out are device pointers (HBM-resident
 * benchmarking; no host<->device copies of vectors). */
int pk_solve_device(pk_ctx* ctx, const pk_mat* a, int32_t method, const double* b,
                    const double* x0, const pk_config* config, pk_trisolve_fn trisolve,
                    void* trisolve_user, double* x_out, double* hist_out, int64_t hist_cap,
                    pk_result* result);

/* Transient batch (BASELINE configs[4]): nsys independent
 * systems solved with the same method/config, each bit-identical to its own
 * pk_solve.  mats[i] / b[i] / x0[i] (x0 nullable, or x0[i] NULL) per system,
 * host vectors; x_out[i] / hist_out[i] host (nullable); results[nsys].
 * `nthreads` host workers, each with its own stream, share the device of ctx.
 * `trisolve` as for pk_solve (it may be called from several workers). */
int pk_solve_batch(pk_ctx* ctx, int64_t nsys, const pk_mat* const* mats, int32_t method,
                   const double* const* b, const double* const* x0, const pk_config* config,
                   pk_trisolve_fn trisolve, void* trisolve_user, double* const* x_out,
                   double* const* hist_out, int64_t hist_cap, pk_result* results, int32_t nthreads);

/* Launch floor of the device-resident loops: time per iteration of a
 * conditional-WHILE graph holding `kernels_per_iteration` empty gated kernels
 * of `grid` CTAs (<= 0: 4 per SM), each CTA taking a ticket and the last one
 * advancing the iteration / setting the WHILE condition as a finalizer does.
 * Best of 3 runs of `iterations`.  No reference counterpart (the reference
 * models this as DeviceProfile.launch_latency, execmodel.py:42-107). */
int pk_launch_floor(pk_ctx* ctx, int32_t kernels_per_iteration, int32_t grid, int64_t iterations,
                    double* us_per_iteration);

/* ---- row-partitioned CG (BASELINE configs[3]) -------- */
/* gen_poisson3d_block(side, 1) split into `world` group-aligned z-slabs; per
 * iteration one halo exchange (r, p, Ap; one plane per neighbour), the fused
 * CG kernel on the local rows, ONE allgather of the group partials and the
 * same serial stage 2 on every rank: bit-identical to cg_pipelined on one
 * device at the geometry n_groups x group_size (which must equal n).
 * comm NULL: all `world` partitions inside this process on ctx's device
 * (halo = device copies); otherwise an ncclComm_t from pk_nccl_comm_create
 * and this process owns partition `rank`.  b: host right-hand side (global
 * for comm NULL, the own rows otherwise; NULL = ones); x_out likewise. */
int pk_nccl_unique_id(void* out /* 128 bytes */);
int pk_nccl_comm_create(int device, const void* unique_id, int nranks, int rank, void** comm);
int pk_nccl_comm_destroy(void* comm);
int pk_dcg_create(pk_ctx* ctx, int64_t side, int64_t n_groups, int64_t group_size, int32_t world,
                  int32_t rank, void* comm, int64_t hist_cap, pk_dcg** out);
int pk_dcg_solve(pk_dcg* dcg, const double* b, const pk_config* config, double* x_out, double* hist_out,
                 int64_t hist_cap, pk_result* result);
int pk_dcg_destroy(pk_dcg* dcg);

/* ---- diagnostics (no reference counterpart) --------------------------- */
/* Engine self-benchmark on `a` (int32 CSR): device time per launch (us) of
 * `reps` launches of a reference kernel (kind 0: plain thread-per-row SpMV,
 * 1: BiCGStab-shaped fused row without the ordered fold) or of the engine
 * (2: As-SpMV with 4 ordered dots; 3, 9: engine row order without the fold;
 * 4: grid-stride rows; 6-8: engine kernel with explicit grids).  Used by
 * tools/dbg_simple.py to bound what the ordered fold costs. */
int pk_debug_bench(pk_ctx* ctx, const pk_mat* a, int kind, int reps, double* us_out);

#ifdef __cplusplus
}
#endif

#endif /* PIPEKRYLOV_B200_H */
