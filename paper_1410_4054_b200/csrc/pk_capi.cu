// C ABI of the B200-native pipelined Krylov path: contexts, matrices,
// kernel-level entries (fused.py / linalg.py mirrors) and the solver-level
// drivers (solvers.py pipelined variants) with device-resident loops.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo
//        -fmad=false -Xcompiler -fPIC,-ffp-contract=off -shared
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "pipekrylov_b200.h"
#include "pk_bulk.cuh"
#include "pk_kernels.cuh"
#include "pk_reduce.cuh"
#include "pk_state.cuh"

using namespace pk;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define PK_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess) {                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? PK_ERR_NOMEM : PK_ERR_CUDA,            \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                     \
    }                                                                                      \
  } while (0)

#define PK_TRY(...)              \
  do {                           \
    int rc_ = (__VA_ARGS__);     \
    if (rc_ != PK_OK) return rc_; \
  } while (0)

// Kernel launch, with the programmatic-dependent-launch attribute when pdl.
template <typename... KArgs, typename... Args>
static cudaError_t launch_k(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  if (!pdl) {
    kern<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// objects
// ---------------------------------------------------------------------------

struct pk_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int32_t ng = 128;
  int32_t gs = 256;
  int sm_count = 148;
  SolveState* scratch = nullptr;  // kernel-level finalizer state
  int32_t* scratch_flag = nullptr;
  double* scratch_d = nullptr;
  double* spill = nullptr;        // engine CHAIN spill, spill_cap doubles
  size_t spill_cap = 0;
  unsigned* gtick = nullptr;      // per-group tickets [ng] + global ticket
  unsigned* ticket = nullptr;
  std::vector<pk_ctx*> workers;   // pk_solve_batch worker contexts (kept across calls)
  void* ws_cache = nullptr;       // cached solver workspaces (pk_solvers.inc WsCache)
  void (*ws_cache_free)(pk_ctx*) = nullptr;
  bool ws_cache_on = true;        // PK_WS_CACHE=0 disables the workspace / graph cache
  bool lane_spmv = true;          // PK_LANE_SPMV=0: SpMV operators on the CTA / warp CHAIN engines instead
  int lane_spmv_maxk = 8;         // PK_LANE_SPMV_MAXK: longest lane chain (K) sent to the pipelined lane engine
                                  // (measured: CG 512^2, K = 8: 19.2 -> 17.7 us/iter; K = 32 (C2): 83 -> 101, so
                                  // long chains stay on the CTA engine)
  bool gs_split = false;          // PK_GS_SPLIT=1: 16-byte update sweep + LANE-engine dot instead of the fused update
                                  // (measured GMRES(30) 128^3: 219 vs 214 us/iter fused; off)
  bool lane_engine = true;        // PK_LANE=0: elementwise reductions on the CTA engine instead of engine_lane
  int gs_chunk = 16;              // PK_GS_CHUNK: basis vectors per Gram-Schmidt update pass (4..32; 16 measured best, GMRES(30) 128^3)
  pk_debug_fn dbg = nullptr;      // per-iteration diagnostics hook (pk_ctx_set_debug)
  void* dbg_user = nullptr;
  bool pdl = false;               // PK_PDL=1: programmatic stream serialization (measured slower, off)
  int mat_mink = 0;               // two-phase SpMV engine for CHAIN chains K >= mat_mink (PK_MAT_MINK=9 to try; 0 = off:
                                  // measured slower than the fused engine on C2, profiles/ENGINE_EXPERIMENTS.md)
  double* mat = nullptr;          // its contribution buffer, mat_cap doubles
  size_t mat_cap = 0;
  bool mat_discard = true;
  bool sweep_one_batch = false;   // PK_SWEEP_ONEBATCH: elementwise sweeps with one V-row batch per thread
  bool staged = true;             // PK_STAGE=0: off (only in -DPK_STAGED_ENGINE builds: the cp.async-staged
                                  // CHAIN engine, measured slower; compiling it in also slows the default engine)
  int sell_mode = 2;              // PK_SELL: 0 never / 1 always / 2 auto -- new matrices get a SELL-32 copy the kernels
                                  // walk when n >= 2^19 and nnz >= 12 n and the VEC pre-pass is off (measured: random
                                  // 16/row, n = 1M: CG 344 -> 260 us/iter; VEC 216); stencils (5-7/row) stay on CSR
  bool sweep_scalar = false;      // PK_SWEEP_SCALAR=1: scalar grid-stride sweeps instead of the 16-byte k_sweep2
  int tile_mink = 0;              // PK_TILE_MINK: shortest lane chain (K) sent to the TILE engine (0 = off; experimental)
  int vec_min_avg = 12;           // PK_VEC_MINAVG: matrices with >= this many entries per row on average take the VEC
                                  // row-sum pre-pass (0 = off).  Measured (CG / BiCGStab us/iter, VEC vs SELL-32 vs
                                  // thread-per-row): 16/row n = 1M 216 / 254 / 338, 454 / 571 / 726; 40/row n = 200k
                                  // 116 / 256 / 165; 400/row n = 20k 90 / 409 / 155
  double* vecbuf = nullptr;       // its row sums, vec_cap doubles
  size_t vec_cap = 0;
  bool mdq = false;               // PK_MDQ=1: GMRES multi-dots by k_multidot_q (quantity-parallel; measured slower:
                                  // GMRES(30) 128^3 multi-dot 98.5 vs 89.3 us, 64^3 51.4 vs 40.5 on the LANE engine)
  bool persist = true;            // PK_PERSIST=0: BiCGStab split-body loop as the WHILE graph instead of one persistent
                                  // cooperative kernel (measured: C2 75.6 vs 76.7 us/iter, 2048^2 221.2 vs 234.8)
  bool bulk = true;               // PK_BULK=0: SpMV operators on long lane chains use the CTA CHAIN engine instead of
                                  // the TMA-fed BULK engine (pk_bulk.cuh)
  bool bulk_pdl = false;          // PK_BULK_PDL=1: BULK kernels launch programmatically (their CSR prologue overlaps
                                  // the previous kernel's tail; measured slower on C2: 94.5 vs 82.3 us/iter -- the
                                  // waiting CTAs hold the registers / shared memory the previous kernel's last wave needs)
  int bulk_mink = 9;              // PK_BULK_MINK: shortest lane chain (K) sent to the BULK engine
  int bulk_maxk = 32;             // PK_BULK_MAXK: longest (measured slower on GMRES 128^3 K = 64, CG 256^3 K = 512)
  int bulk_maxq = 2;              // PK_BULK_MAXQ: operators with at most this many dot quantities (C2: Ap' = A p' + 2
                                  // dots 35.3-36.8 vs 37.3-38.0 us; As = A s + 4 dots 44.1-45.7 vs 42.7-43.8)
  bool warp_k1 = true;            // PK_WARP_K1: n <= G systems on the warp chain engine (vs LEAF)        // PK_MAT_DISCARD=0: keep consumed lines in L2 (write-back on eviction)
};

struct pk_mat {
  uint64_t uid = 0;            // unique per matrix object (workspace-cache key)
  int device = 0;
  int64_t n_rows = 0, n_cols = 0, nnz = 0, max_row = 0;
  int64_t blk_max = -1;        // most entries in an aligned 32-row block (BULK engine slots)
  bool vec_rows = false;       // long rows: SpMV row sums by the VEC pre-pass (k_rowsum_warp)
  bool row64 = false;
  void* rowptr = nullptr;
  int32_t* cols = nullptr;
  double* vals = nullptr;
  // SELL-32 copy (pk_mat_set_format(PK_FMT_SELL32)); the kernels walk it
  // instead of the CSR arrays when `sell` is set
  bool sell = false;
  int64_t sell_nnz = 0;        // padded entries
  void* sell_ptr = nullptr;    // RowT [n_slices + 1]
  int32_t* sell_cols = nullptr;
  double* sell_vals = nullptr;
};

struct pk_ell {
  int device = 0;
  int64_t n_rows = 0, n_cols = 0, width = 0;
  int32_t* cols = nullptr;  // [width][n_rows], sentinel n_cols on padded slots
  double* vals = nullptr;
};

static int apply_default_format(pk_ctx* c, pk_mat* m);

static int set_device(int dev) {
  PK_CUDA(cudaSetDevice(dev));
  return PK_OK;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// Programmatic dependent launch: every loop kernel lets its successor's CTAs
// launch as soon as all of its own CTAs are resident (they then occupy the
// slots the partially filled last wave and the finalizer tail leave idle),
// and waits for its predecessor's completion + memory flush before touching
// anything.  Both are no-ops for launches without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <int NQ, int U, int MINB, class Op>
__global__ void __launch_bounds__(kThreads, MINB)
    k_reduce(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part, int ld,
             int col0, int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip, int fin, int fin_arg) {
  extern __shared__ double smem[];
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  bool last;
#ifdef PK_STAGED_ENGINE
  if constexpr (Op::kSpmv) {
    if (geo.staged)
      last = engine_chain_staged<NQ, U>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
    else
      last = engine_run<NQ, U>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
  } else {
    last = engine_run<NQ, U>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
  }
#else
  last = engine_run<NQ, U>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
#endif
  if (last && fin != FIN_NONE && st && threadIdx.x < 32) {
    // warp 0 of the last CTA; the engine's staging memory is free now
    const Geom g2 = geo;
    finalize(st, fin, fin_arg, ing, smem, (int)(engine_smem_bytes(g2, NQ, U) / sizeof(double)));
  }
}

#ifndef PK_LANE_D_WIDE
#define PK_LANE_D_WIDE 4
#endif
#ifndef PK_LANE_D_LIGHT
#define PK_LANE_D_LIGHT 16  // chunks in flight per lane for items of <= 2 doubles (dots, normalize)
#endif

// LANE engine kernel (elementwise operators on CHAIN geometries): one thread
// per reduction lane, D chunks of loads in flight (pk_reduce.cuh engine_lane).
template <int NQ, int D, class Op>
__global__ void __launch_bounds__(kLaneThreads)
    k_reduce_lane(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part,
                  int ld, int col0, int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip, int fin,
                  int fin_arg, int smem_d) {
  extern __shared__ double smem[];
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  const bool last = engine_lane<NQ, D>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
  if (last && fin != FIN_NONE && st && threadIdx.x < 32) finalize(st, fin, fin_arg, ing, smem, smem_d);
}

#ifndef PK_LANE_P
#define PK_LANE_P 2
#endif

// Software-pipelined LANE engine for SpMV operators (engine_lane_spmv).
template <int NQ, int P, class Op>
__global__ void __launch_bounds__(kLaneThreads, 1)
    k_reduce_lane_spmv(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part,
                       int ld, int col0, int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip,
                       int fin, int fin_arg, int smem_d) {
  extern __shared__ double smem[];
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  const bool last =
      engine_lane_spmv<NQ, P>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
  if (last && fin != FIN_NONE && st && threadIdx.x < 32) finalize(st, fin, fin_arg, ing, smem, smem_d);
}

constexpr int kWarpStage2Doubles = 1024;  // stage-2 staging of the warp engine's finalizer

#ifndef PK_BULK_W
#define PK_BULK_W 4
#endif
#ifndef PK_BULK_MINB
#define PK_BULK_MINB 7
#endif
#ifndef PK_BULK_R
#define PK_BULK_R 3  // data slots (chunks in flight) per row warp
#endif

#ifdef PK_BULK_TRACE
extern "C" int pk_debug_bulk_trace(void* dev_buf) {
  unsigned long long* p = (unsigned long long*)dev_buf;
  return cudaMemcpyToSymbol(g_bulk_trace, &p, sizeof(p)) == cudaSuccess ? PK_OK : PK_ERR_CUDA;
}
#endif

// BULK CHAIN engine (pk_bulk.cuh): one CTA per 32-lane unit, warp 0 = TMA
// producer + ordered fold, warps 1..W = rows from shared memory.
template <int NQ, int W, int R, int MINB, class Op>
__global__ void __launch_bounds__(32 * (W + 1), MINB)
    k_reduce_bulk(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part,
                  int ld, int col0, int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip, int fin,
                  int fin_arg, const __grid_constant__ BulkCfg bc, int smem_d) {
  extern __shared__ __align__(128) unsigned char bsm[];
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  Op op = op0;
  // the CTA's first chunks are requested before the wait for the previous
  // kernel (they depend on the matrix only); the gate, the scalars and every
  // vector after it
  auto sync = [&]() -> bool {
    pdl_wait();
    pdl_trigger();
    if (bc.pdl) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // L1 may hold lines from before the wait
    if (skip && *(volatile const int32_t*)skip) return false;
    const GateVals gv = gate_load(st, gate);
    op.scalars(sp);
    return gate_eval(st, gate, ing, gv);
  };
  const bool last =
      engine_bulk<NQ, W, R>(geo, op, bsm, bc, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket, sync);
  if (last && fin != FIN_NONE && st) {
    PK_BTA((size_t)1024 * 32);
    finalize(st, fin, fin_arg, ing, reinterpret_cast<double*>(bsm + bc.base), smem_d);
    PK_BTA((size_t)1024 * 32 + 1);
  }
}

// One warp per CTA, one unit per warp (CHAIN mapping with group_size >= 32).
template <int NQ, int R, class Op>
__global__ void __launch_bounds__(32, 8)
    k_reduce_warp(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part,
                  int ld, int col0, int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip, int fin,
                  int fin_arg) {
  extern __shared__ double smem[];
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  bool last = engine_warp_chain<NQ, R>(geo, op, smem, part, ld, col0, nstore, scr, st ? &st->ticket : scr.ticket);
  if (last && fin != FIN_NONE && st) finalize(st, fin, fin_arg, ing, smem, kWarpStage2Doubles);
}

#ifdef PK_MAT_ENGINE  // experimental two-phase engine (measured slower on C2), compiled out by default
// ---------------------------------------------------------------------------
// two-phase ("materialised") engine for SpMV operators on long lane chains
// ---------------------------------------------------------------------------
//
// Phase 1 (k_mat_rows): plain grid-stride thread-per-row code -- the SpMV row,
// the operator's vector outputs and its NQ dot contributions c_q[row], which
// are stored to a contribution buffer cb[q][n] (coalesced).  No shared
// memory, no barrier: full occupancy, the row code runs at streaming speed.
// Phase 2 (k_mat_fold): thread = lane t of [0, G); it folds its chain
// cb[q][t], cb[q][t+G], ... serially in chunk order (linalg.py:300-303;
// rows past n add +0.0, which cannot change a sum that starts at +0.0), with
// UF chunks x NQ quantities of loads in flight; a warp's loads are 32
// consecutive doubles.  Lane values go to the spill buffer, the CTA that
// completes a group runs its halving tree (group_tree, linalg.py:304-307),
// the CTA completing the last group runs the finalizer.
// The buffer (8 B x nq x n) is written and read back within two launches and
// mostly served by L2.  Same IEEE operations on the same operands, in the
// same order, as the fused engine: bit-identical partials.
template <int NQ, class Op>
__global__ void __launch_bounds__(256, 4)
    k_mat_rows(int64_t n, const __grid_constant__ Op op0, ScalarPtrs sp, double* __restrict__ cb, int nstore,
               SolveState* st, int gate, const int32_t* skip) {
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n; row += stride) {
    double c[NQ];
    row_contrib<NQ>(op, (uint32_t)row, c);
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q < nstore) cb[(int64_t)q * n + row] = c[q];
  }
}

// quantities of one lane chain are folded by NQP (power of two >= NQ)
// different threads: a CTA covers kMatLanes(NQ) = 256 / NQP lanes
__host__ __device__ constexpr int mat_nqp(int nq) { return nq <= 1 ? 1 : nq <= 2 ? 2 : 4; }
__host__ __device__ constexpr int mat_lanes(int nq) { return kThreads / mat_nqp(nq); }

template <int NQ>
__global__ void __launch_bounds__(kThreads, 4)
    k_mat_fold(const __grid_constant__ Geom geo, const double* __restrict__ cb, double* part, int ld, int col0,
               int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip, int fin, int fin_arg,
               int smem_d, int discard) {
  extern __shared__ double smem[];
  __shared__ int s_flag;
  __shared__ int s_last;
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  if (st && !gate_open(st, gate, ing)) return;
  constexpr int LPB = mat_lanes(NQ);
  const int tid = threadIdx.x;
  const int q = tid / LPB;  // the quantity this thread folds
  const int64_t n = geo.n, G = geo.G, K = geo.K;
  const int64_t lid0 = (int64_t)blockIdx.x * LPB;
  const int nl = (int)((G - lid0) < LPB ? (G - lid0) : LPB);
  const int64_t l = lid0 + tid % LPB;
  if (tid == 0) s_last = 0;
  if (tid % LPB < nl && q < nstore) {
    // full rounds (every row < n): UF loads issued back to back (volatile
    // asm keeps them together), then the ordered adds
    constexpr int UF = 16;
    double acc = 0.0;
    const double* pq = cb + (int64_t)q * n + l;
    const int64_t Kf = n / G;  // chunks whose rows are all < n
    int64_t k = 0;
    for (; k + UF <= Kf; k += UF) {
      double v[UF];
#pragma unroll
      for (int u = 0; u < UF; ++u) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v[u]) : "l"(pq + (k + u) * G));
#pragma unroll
      for (int u = 0; u < UF; ++u) acc = add_rn(acc, v[u]);
      if (discard) {
        // the lines just consumed are dead: drop them from L2 without a
        // write-back (lane 16 j owns the 128-B line of lanes 16 j .. 16 j + 15)
        __syncwarp();
        if ((l & 15) == 0) {
#pragma unroll
          for (int u = 0; u < UF; ++u) asm volatile("discard.global.L2 [%0], 128;" ::"l"(pq + (k + u) * G) : "memory");
        }
      }
    }
    for (; k < K; ++k) acc = add_rn(acc, k * G + l < n ? __ldg(pq + k * G) : 0.0);
    scr.spill[(int64_t)q * G + l] = acc;
  }
  __syncthreads();
  int ncomplete = 0;
  double* tail = smem;
  if (geo.gs >= LPB) {
    const int g = (int)(lid0 / geo.gs);
    if (tid == 0) {
      const unsigned per = (unsigned)(geo.gs / LPB);
      unsigned tk = ticket_add(scr.gtick + g, 1u);
      int last = (tk == per - 1);
      if (last) {
        scr.gtick[g] = 0u;
        acquire_fence();
      }
      s_flag = last;
    }
    __syncthreads();
    if (s_flag) {
      group_tree<NQ>(geo, g, scr.spill, tail, part, ld, col0, nstore);
      ncomplete = 1;
    }
  } else {
    const int g0 = (int)(lid0 / geo.gs);
    int g1 = (int)((lid0 + nl + geo.gs - 1) / geo.gs);
    if (g1 > geo.n_groups) g1 = geo.n_groups;
    for (int g = g0; g < g1; ++g) group_tree<NQ>(geo, g, scr.spill, tail, part, ld, col0, nstore);
    ncomplete = g1 - g0;
  }
  if (ncomplete > 0) {
    __syncthreads();
    if (tid == 0) {
      unsigned* ticket = st ? &st->ticket : scr.ticket;
      unsigned tk = ticket_add(ticket, (unsigned)ncomplete);
      if (tk + (unsigned)ncomplete == (unsigned)geo.n_groups) {
        *ticket = 0u;
        acquire_fence();
        s_last = 1;
      }
    }
  }
  __syncthreads();
  if (s_last && fin != FIN_NONE && st && tid < 32) finalize(st, fin, fin_arg, ing, smem, smem_d);
}

#endif  // PK_MAT_ENGINE

#ifdef PK_TILE_ENGINE  // experimental (measured 3-4x slower than the CTA engine on C2), compiled out by default
// ---------------------------------------------------------------------------
// TILE engine: rows at streaming speed, each group folded by the CTA that
// completes it (SpMV operators on CHAIN geometries, group_size % 256 == 0)
// ---------------------------------------------------------------------------
//
// The work is cut into tiles of 256 consecutive rows: tile (g, k, s) = rows
// k G + g gs + 256 s + [0, 256) -- the chunk-k rows of lanes [256 s, 256 s +
// 256) of group g.  A persistent grid walks the tiles in GROUP-MAJOR order
// (t = (g K + k) sub + s), one row per thread with the lean thread-per-row
// code (row_contrib, the same arithmetic as every other engine), and stores
// the NQ contributions to the contribution buffer cb[q][row].  After each
// tile the CTA bumps the group's tile counter (release); the CTA completing
// the group's K * sub-th tile (acquire) folds the group at once: thread l
// sums lane l's chain cb[q][l], cb[q][l + G], ... in chunk order
// (linalg.py:300-303; rows past n add +0.0 like in the fused engines), the
// CTA runs the group's halving tree (linalg.py:304-307) and takes the global
// ticket; the CTA completing the last group runs the finalizer.
//
// No CTA ever waits for another (no grid barrier: safe under concurrent
// launches), rows run at full occupancy with no staging and no per-batch
// barrier, and -- group-major -- a group's contributions are folded about
// one wave after they were written, so they are read back from L2 and then
// discarded there (discard.global.L2: no write-back).  Same operations, same
// operands, same order as the fused engines: bit-identical partials.
#ifndef PK_TILE_MINB
#define PK_TILE_MINB 4
#endif
template <int NQ, class Op>
__global__ void __launch_bounds__(256, PK_TILE_MINB)
    k_reduce_tiles(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part,
                   int ld, int col0, int nstore, Scratch scr, SolveState* st, int gate, const int32_t* skip, int fin,
                   int fin_arg, double* __restrict__ cb, int smem_d, int discard) {
  extern __shared__ double smem[];
  __shared__ int s_fold;
  __shared__ int s_last;
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  const int tid = threadIdx.x;
  const int64_t n = geo.n, G = geo.G, K = geo.K;
  const int sub = geo.gs / 256;  // tiles per (group, chunk)
  const int64_t per_g = K * sub;
  const int64_t T = per_g * geo.n_groups;
  unsigned* ticket = st ? &st->ticket : scr.ticket;
  if (tid == 0) s_last = 0;
  for (int64_t t = blockIdx.x; t < T; t += gridDim.x) {
    const int g = (int)(t / per_g);
    const int64_t rem = t - (int64_t)g * per_g;
    const int64_t k = rem / sub;
    const int s = (int)(rem - k * sub);
    const int64_t row = k * G + (int64_t)g * geo.gs + 256 * s + tid;
    if (row < n) {
      double c[NQ];
      row_contrib<NQ>(op, (uint32_t)row, c);
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) cb[(int64_t)q * n + row] = c[q];
    }
    __syncthreads();
    if (tid == 0) {
#ifdef PK_TILE_RELAXED
      const unsigned tk = atomicAdd(scr.gtick + g, 1u);  // experiment only: no release ordering
#else
      const unsigned tk = ticket_add(scr.gtick + g, 1u);
#endif
      const int f = tk == (unsigned)(per_g - 1);
      if (f) {
        scr.gtick[g] = 0u;
        acquire_fence();
      }
      s_fold = f;
    }
    __syncthreads();
    if (!s_fold) continue;
    // ---- fold group g: lanes g gs + 256 j + tid, chunk order ----
    double v[NQ];
    for (int j = 0; j < sub; ++j) {
      const int64_t lane = (int64_t)g * geo.gs + 256 * j + tid;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double acc = 0.0;
        if (q < nstore) {
          const double* pq = cb + (int64_t)q * n + lane;
          constexpr int UF = 16;
          int64_t kk = 0;
          for (; kk < K; kk += UF) {
            double x[UF];
#pragma unroll
            for (int u = 0; u < UF; ++u) {
              const int64_t r = (kk + u) * G + lane;
              x[u] = (kk + u < K && r < n) ? __ldcg(pq + (kk + u) * G) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < UF; ++u)
              if (kk + u < K) acc = add_rn(acc, x[u]);
          }
        }
        v[q] = acc;
        if (sub > 1 && q < nstore) scr.spill[(int64_t)q * G + lane] = acc;
      }
    }
    if (discard) {
      // the group's contribution lines are dead: drop them from L2 without a
      // write-back (thread 16 i owns the 128-B line of lanes 16 i .. 16 i + 15)
      __syncthreads();
      if ((tid & 15) == 0) {
        for (int j = 0; j < sub; ++j)
          for (int q = 0; q < nstore; ++q)
            for (int64_t kk = 0; kk < K; ++kk) {
              const int64_t r = kk * G + (int64_t)g * geo.gs + 256 * j + tid;
              if (r + 15 < n) asm volatile("discard.global.L2 [%0], 128;" ::"l"(cb + (int64_t)q * n + r) : "memory");
            }
      }
    }
    if (sub == 1) {
      // the group's 256 lanes are this CTA's threads: halving tree directly
      block_tree<NQ>(v, smem, 256);
      if (tid == 0 && part) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nstore) part[(int64_t)g * ld + col0 + q] = v[q];
      }
      __syncthreads();
    } else {
      __syncthreads();  // the spill was written by this CTA's threads
      group_tree<NQ>(geo, g, scr.spill, smem, part, ld, col0, nstore);
    }
    if (tid == 0) {
      const unsigned tk = ticket_add(ticket, 1u);
      if (tk + 1u == (unsigned)geo.n_groups) {
        *ticket = 0u;
        acquire_fence();
        s_last = 1;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_last && fin != FIN_NONE && st && tid < 32) finalize(st, fin, fin_arg, ing, smem, smem_d);
}

#endif  // PK_TILE_ENGINE

// ---------------------------------------------------------------------------
// VEC row sums: sub-warp-cooperative SpMV rows for long-row matrices
// ---------------------------------------------------------------------------
//
// CSR-adaptive handling of long rows (avg >= vec_min_avg entries): instead of
// one thread walking a 40- or 400-entry row kSlots entries per dependent
// round trip, L = 2^lg lanes (4..32, from the average row length) own a row
// and walk it 4 L entries per round: lane i loads entries c0 + u L + i (u <
// 4; coalesced columns / values), issues the 4 gathers, and parks the
// products in a per-warp tile; the row's first lane then adds the round's
// products in stored order -- acc = ((0 + v0 x0) + v1 x1) + ..., exactly the
// thread-per-row sum (_spmvkernels.py:12-18).  One pair of dependent round
// trips per 4 L entries instead of per kSlots.  The sums go to a buffer; the
// fused operator then runs as an elementwise operator (OpPre) on any
// reduction engine.  Same IEEE operations in the same order: bit-identical.
constexpr int kVecWarps = 8;
constexpr int kVecU = 4;  // entries per lane per round
template <class Op>
__global__ void __launch_bounds__(32 * kVecWarps)
    k_rowsum_warp(int64_t n, const __grid_constant__ Op op0, ScalarPtrs sp, double* __restrict__ qout,
                  SolveState* st, int gate, const int32_t* skip, int lg) {
  __shared__ double tile[kVecWarps][kVecU * 32];
  pdl_wait();
  pdl_trigger();
  if (skip && *(volatile const int32_t*)skip) return;
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  Op op = op0;
  op.scalars(sp);
  if (!gate_eval(st, gate, ing, gv)) return;
  using RowT = typename Op::RowT;
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int L = 1 << lg, li = lane & (L - 1), sub = lane >> lg;  // lane i of row `sub` of the warp
  const int RE = kVecU * L;                                         // entries per row per round
  double* T = tile[wl] + sub * RE;
  const int rpw = 32 >> lg;
  const int64_t nblk = (n + rpw - 1) / rpw;
  for (int64_t blk = (int64_t)blockIdx.x * kVecWarps + wl; blk < nblk; blk += (int64_t)gridDim.x * kVecWarps) {
    const int64_t row = blk * rpw + sub;
    RowT b = 0, e = 0;
    if (row < n) {
      b = __ldg(op.A.rp + row);
      e = __ldg(op.A.rp + row + 1);
    }
    const int len = (int)(e - b);
    int mx = len;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    double acc = 0.0;
    for (int c0 = 0; c0 < mx; c0 += RE) {
      int32_t col[kVecU];
      double val[kVecU];
      bool ok[kVecU];
#pragma unroll
      for (int u = 0; u < kVecU; ++u) {
        const RowT k = b + c0 + u * L + li;
        ok[u] = k < e;
        col[u] = ok[u] ? __ldg(op.A.ci + k) : 0;
        val[u] = ok[u] ? __ldg(op.A.va + k) : 0.0;
      }
      typename Op::Gat g[kVecU];
#pragma unroll
      for (int u = 0; u < kVecU; ++u) op.gload((uint32_t)col[u], g[u]);
#pragma unroll
      for (int u = 0; u < kVecU; ++u) T[u * L + li] = ok[u] ? mul_rn(val[u], op.gval(g[u])) : 0.0;
      __syncwarp();
      if (li == 0) {
        const int cnt = len - c0 < RE ? len - c0 : RE;
        for (int j = 0; j < cnt; ++j) acc = add_rn(acc, T[j]);
      }
      __syncwarp();
    }
    if (li == 0 && row < n) qout[row] = acc;
  }
}

// The fused operator with its SpMV row sum taken from the VEC buffer: an
// elementwise operator for the reduction engines (kSpmv = false).
template <class Op>
struct OpPre {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = Op::kMinBlocks;
  Op in;
  const double* q;
  struct Item { typename Op::Item it; double q; };
  __device__ __forceinline__ void load(uint32_t row, Item& t) const {
    in.load(row, t.it);
    t.q = __ldg(q + row);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& t, double (&c)[M]) const {
    in.compute(row, t.it, t.q, c);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) { in.scalars(sp); }
};

template <class Op>
__global__ void __launch_bounds__(256, 4) k_sweep(int64_t n, Op op, ScalarPtrs sp, SolveState* st, int gate) {
  pdl_wait();
  pdl_trigger();
  const GateVals gv = gate_load(st, gate & 0xff);
  op.scalars(sp);
  if (!gate_eval(st, gate & 0xff, (gate & GATE_IN_GRAPH) != 0, gv)) return;
  sweep_rows(n, op);
}

// Vectorised elementwise sweep (operators with load2/compute2: two adjacent
// rows through 16-byte loads and stores).  Every thread owns UP row pairs
// p, p + T, ..., all loads of a thread issued before its first compute (pair
// indices are clamped, so every load is unconditional and the batch stays
// together); the grid is sized so each thread runs exactly one batch.
// Vectorised elementwise sweep rows (operators with load2/compute2: two
// adjacent rows through 16-byte loads and stores).  Every thread owns UP row
// pairs p, p + T, ..., all loads of a thread issued before its first compute
// (pair indices are clamped, so every load is unconditional and the batch
// stays together).
template <class Op, int UP>
__device__ __forceinline__ void sweep2_rows(int64_t n, const Op& op) {
  const int64_t np = n >> 1;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p0 < np; p0 += T * UP) {
    typename Op::Item2 it[UP];
#pragma unroll
    for (int u = 0; u < UP; ++u) {
      const int64_t pu = p0 + u * T;
      op.load2((uint32_t)(2 * (pu < np ? pu : np - 1)), it[u]);
    }
#pragma unroll
    for (int u = 0; u < UP; ++u)
      if (p0 + u * T < np) op.compute2((uint32_t)(2 * (p0 + u * T)), it[u]);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    typename Op::Item it;
    double c[1];
    op.load((uint32_t)(n - 1), it);
    op.compute((uint32_t)(n - 1), it, c);
  }
}

// the grid is sized so each thread runs exactly one batch
template <class Op, int UP>
__global__ void __launch_bounds__(256) k_sweep2(int64_t n, Op op, ScalarPtrs sp, SolveState* st, int gate) {
  pdl_wait();
  pdl_trigger();
  const GateVals gv = gate_load(st, gate & 0xff);
  op.scalars(sp);
  if (!gate_eval(st, gate & 0xff, (gate & GATE_IN_GRAPH) != 0, gv)) return;
  sweep2_rows<Op, UP>(n, op);
}

template <class Op, class = void>
struct RowsPerThreadDev { static constexpr int value = 2; };
template <class Op>
struct RowsPerThreadDev<Op, std::void_t<decltype(Op::kRowsPerThread)>> { static constexpr int value = Op::kRowsPerThread; };

// ---------------------------------------------------------------------------
// Persistent cooperative BiCGStab loop (PK_PERSIST=1)
// ---------------------------------------------------------------------------
//
// The split BiCGStab body -- As = A s + 4 dots (finalizer FIN_BICG_TAIL), the
// xrp sweep, Ap' = A p' + 2 dots (FIN_BICG_ALPHA) -- as phases of ONE
// co-resident grid separated by grid barriers instead of three kernel
// launches per iteration: the phases are the same engine / sweep device code
// (same operations, same order: the same bits).  A barrier publishes the
// phase's writes (release add, acquire spin) and invalidates L1 (the phases
// read vectors through the non-coherent path).  The loop runs while the
// state says RUNNING, exactly the gates of the graph body.
#ifndef PK_BAR_SLEEP_NS
#define PK_BAR_SLEEP_NS 32
#endif
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    ++gen;
    const unsigned target = gen * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    while (v < target) {
      // back off: ~600 CTAs polling one L2 line would compete with the
      // phase's last CTAs (group trees, finalizer) for that L2 slice
      __nanosleep(PK_BAR_SLEEP_NS);
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}

template <class OB, class OX, class OA>
__global__ void __launch_bounds__(kThreads, 4)
    k_bicg_persist(const __grid_constant__ Geom geo, const __grid_constant__ OB ob0, const __grid_constant__ OX ox0,
                   const __grid_constant__ OA oa0, ScalarPtrs spb, ScalarPtrs spx, ScalarPtrs spa, double* p_quad,
                   double* p_pair, Scratch scr, SolveState* st, unsigned* bar, int smem_d) {
  extern __shared__ double smem[];
  unsigned gen = 0;
  for (;;) {
    if (*(volatile const int32_t*)&st->status != RUNNING) break;
    {
      OB op = ob0;
      op.scalars(spb);
      const bool last = engine_run<4, RowsPerThreadDev<OB>::value>(geo, op, smem, p_quad, 4, 0, 4, scr, &st->ticket);
      if (last && threadIdx.x < 32) finalize(st, FIN_BICG_TAIL, 0, false, smem, smem_d);
    }
    grid_barrier(bar, gen);
    if (*(volatile const int32_t*)&st->status != RUNNING) break;
    {
      OX op = ox0;
      op.scalars(spx);
      sweep2_rows<OX, 2>(geo.n, op);
    }
    grid_barrier(bar, gen);
    {
      OA op = oa0;
      op.scalars(spa);
      const bool last = engine_run<2, RowsPerThreadDev<OA>::value>(geo, op, smem, p_pair, 2, 0, 2, scr, &st->ticket);
      if (last && threadIdx.x < 32) finalize(st, FIN_BICG_ALPHA, 1, false, smem, smem_d);
    }
    grid_barrier(bar, gen);
  }
}

// Profiling aid (PK_FLAG_PROFILE host loops): hold the stream for `cycles`
// SM clocks so the host enqueues the whole batch behind it; the per-kernel
// event brackets then time back-to-back kernels, not the host's launch rate.
__global__ void k_spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
}

// Persistent cooperative CG loop (fused body on the pipelined lane engine,
// short lane chains -- C1): one phase per iteration (OpCgFused + FIN_CG_FUSED)
// and a grid barrier instead of one WHILE-graph kernel node per iteration.
// The lane engine maps lanes to CTAs one to one (grid = G / T, co-resident at
// one CTA per SM); same device code, same bits.
template <class Op>
__global__ void __launch_bounds__(kLaneThreads, 1)
    k_cg_persist(const __grid_constant__ Geom geo, const __grid_constant__ Op op0, ScalarPtrs sp, double* part,
                 Scratch scr, SolveState* st, unsigned* bar, int smem_d) {
  extern __shared__ double smem[];
  unsigned gen = 0;
  for (;;) {
    if (*(volatile const int32_t*)&st->status != RUNNING) break;
    Op op = op0;
    op.scalars(sp);
    const bool last = engine_lane_spmv<3, PK_LANE_P>(geo, op, smem, part, 3, 0, 3, scr, &st->ticket);
    if (last && threadIdx.x < 32) finalize(st, FIN_CG_FUSED, 0, false, smem, smem_d);
    grid_barrier(bar, gen);
  }
}

__global__ void k_finalize(SolveState* st, int fin, int arg) {
  __shared__ double buf[1024];
  finalize(st, fin, arg, false, buf, 1024);
}

// totals[q] = serial sum of column q (reduce_stage2 / in-kernel finalize)
__global__ void k_stage2(const double* part, int ng, int ld, int nq, double* out) {
  for (int q = threadIdx.x; q < nq; q += blockDim.x) out[q] = stage2_col(part, ng, ld, q);
}

__global__ void k_bicg_alpha(const double* rr0p, const double* aprp, int ng, double btol,
                             double* alpha_out, int32_t* bd) {
  __shared__ double t[2];
  if (threadIdx.x == 0) t[0] = stage2_col(rr0p, ng, 1, 0);
  if (threadIdx.x == 1) t[1] = stage2_col(aprp, ng, 1, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (fabs(t[1]) < btol) {
      *bd = 1;
    } else {
      *bd = 0;
      *alpha_out = div_rn(t[0], t[1]);
    }
  }
}

__global__ void k_norm_fin(const double* part, int ng, double btol, double* norm_out, double* inv_out,
                           int32_t* lucky) {
  if (threadIdx.x == 0) {
    double nrm = __dsqrt_rn(stage2_col(part, ng, 1, 0));
    *norm_out = nrm;
    if (nrm < btol || nrm == 0.0) {
      *lucky = 1;
    } else {
      *lucky = 0;
      *inv_out = div_rn(1.0, nrm);
    }
  }
}

// y = y + alpha x with alpha from device memory (axpy, linalg.py:403-411)
__global__ void k_axpy_dev(int64_t n, double* y, const double* x, const double* alpha) {
  double a = *alpha;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = add_rn(y[i], mul_rn(a, x[i]));
}

// y = y * s (scale, linalg.py:440-447), s host value
__global__ void k_scale(int64_t n, double* y, double s) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = mul_rn(y[i], s);
}

// GMRES iterate update (solvers.py:981-984):
//   u = eta0 r; u = u + eta_k V_{k-1} (k = 1..ks-1); x = x + rho u
__global__ void k_gmres_x(int64_t n, double* x, const double* r, const double* V, int64_t ldv,
                          const double* eta, int ks, double rho) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double u = mul_rn(eta[0], r[i]);
    for (int k = 1; k < ks; ++k) u = add_rn(u, mul_rn(eta[k], V[(int64_t)(k - 1) * ldv + i]));
    x[i] = add_rn(x[i], mul_rn(rho, u));
  }
}

__global__ void k_fill_i32(int32_t* p, int32_t v) { *p = v; }

// ---------------------------------------------------------------------------
// device-side generators
// ---------------------------------------------------------------------------

struct StencilSpec {
  int64_t row_lo;     // first global row generated (local row i = global row_lo + i)
  int64_t col_base;   // stored column = global column - col_base
  int32_t nent;
  int64_t off[8];     // column offset, sorted ascending
  int32_t axis[8];    // -1 for the diagonal
  int32_t step[8];
  double val[8];
  int64_t dim[3];
  int64_t stride[3];
};

__device__ __forceinline__ bool stencil_valid(const StencilSpec& s, int64_t row, int e) {
  int ax = s.axis[e];
  if (ax < 0) return true;
  int64_t c = (row / s.stride[ax]) % s.dim[ax];
  int64_t t = c + s.step[e];
  return t >= 0 && t < s.dim[ax];
}

__global__ void k_gen_count(int64_t n, StencilSpec s, int64_t* counts) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int e = 0; e < s.nent; ++e) c += stencil_valid(s, s.row_lo + i, e);
    counts[i] = c;
  }
}

template <typename RowT>
__global__ void k_gen_fill(int64_t n, StencilSpec s, const RowT* rowptr, int32_t* cols, double* vals) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    RowT k = rowptr[i];
    const int64_t gi = s.row_lo + i;
    for (int e = 0; e < s.nent; ++e) {
      if (stencil_valid(s, gi, e)) {
        cols[k] = (int32_t)(gi + s.off[e] - s.col_base);
        vals[k] = s.val[e];
        ++k;
      }
    }
  }
}

// exclusive scan of row counts (single pass per block + block sums); simple
// three-kernel decoupled scan, run once per generated matrix.
__global__ void k_scan_block(const int64_t* in, int64_t* out, int64_t n, int64_t* block_sums) {
  __shared__ int64_t s[1024];
  int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  int64_t v = i < n ? in[i] : 0;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {
    int64_t t = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
    __syncthreads();
    s[threadIdx.x] += t;
    __syncthreads();
  }
  if (i < n) out[i] = s[threadIdx.x];  // inclusive
  if (threadIdx.x == 1023) block_sums[blockIdx.x] = s[1023];
}

__global__ void k_scan_add(int64_t* out, int64_t n, const int64_t* block_prefix) {
  int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  if (i < n && blockIdx.x > 0) out[i] += block_prefix[blockIdx.x - 1];
}

template <typename RowT>
__global__ void k_rowptr_from_incl(const int64_t* incl, int64_t n, RowT* rowptr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    rowptr[i] = (RowT)(i == 0 ? 0 : incl[i - 1]);
}

__global__ void k_rowptr_widen(const int32_t* rp32, int64_t n, int64_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rp32[i];
}

__global__ void k_row_max(const int64_t* counts, int64_t n, unsigned long long* mx) {
  unsigned long long m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)counts[i]);
  // block maximum first: same-address 64-bit atomics serialise in one L2
  // slice (one per warp cost ~400 us at 1M rows), so one atomic per block
  __shared__ unsigned long long wm[32];
  for (int s = 16; s >= 1; s >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, s));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0ull;
    for (int s = 16; s >= 1; s >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, s));
    if (threadIdx.x == 0) atomicMax(mx, m);
  }
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------

// Scratch of the engine (CHAIN spill + per-group tickets), sized for nq
// quantities.  Must be called outside stream capture (it may reallocate).
static int64_t min_units(const pk_ctx* c) { return (int64_t)c->sm_count * 4; }

// single-chunk lanes on the warp engine instead of LEAF when at least a
// quarter of the G <= 2^20 lanes hold a row (CG 128^2 at 128 x 256: 22 -> 16.8
// us/iter, C5 108 -> 118 systems/s); sparser lane sets keep LEAF, whose
// zero-fill unit skips the empty groups (n = 225: 12.5 vs 16.5 us/iter).
// PK_WARP_K1=0 turns it off.
static bool warp_k1(const pk_ctx* c, const Geom& geo) {
  // (gs <= 1024: the warp engine's group tree walks gs / 32 leaves per lane
  // serially -- a 65536-lane group would take milliseconds; LEAF splits it)
  return c->warp_k1 && geo.G <= (int64_t)1 << 20 && 4 * geo.n >= geo.G && geo.gs <= 1024;
}

static bool mat_applies(const pk_ctx* c, const Geom& geo) {
#ifdef PK_MAT_ENGINE
  return c->mat_mink > 0 && !geo.leaf && geo.K >= c->mat_mink;
#else
  (void)c;
  (void)geo;
  return false;  // two-phase engine not compiled in
#endif
}

// TILE engine (k_reduce_tiles): CHAIN geometries with whole 256-lane tiles
static bool tiles_apply(const pk_ctx* c, const Geom& geo) {
  return c->tile_mink > 0 && !geo.leaf && geo.gs >= 256 && geo.gs % 256 == 0 && geo.K >= c->tile_mink;
}

// L2 discard of consumed contribution lines: only when every warp's 32-lane
// segment is whole 128-B lines (n and G multiples of 32)
static int mat_discard(const pk_ctx* c, const Geom& geo) {
  return c->mat_discard && geo.n % 32 == 0 && geo.G % 32 == 0 ? 1 : 0;
}

// Cached solver workspaces hold instantiated graphs whose kernel parameters
// point into the context's scratch (spill, contribution and VEC buffers):
// whenever one of those buffers is reallocated the cache is dropped, so no
// cached graph can ever launch with a freed pointer.
static void scratch_moved(pk_ctx* c) {
  if (c->ws_cache_free) c->ws_cache_free(c);
}

static int ensure_scratch(pk_ctx* c, int64_t n, int nq) {
  Geom geo = make_geom(n, c->ng, c->gs, min_units(c));
  if (mat_applies(c, geo) || tiles_apply(c, geo)) {
    // SpMV operators carry at most 4 quantities
    const size_t mneed = (size_t)n * (size_t)std::min(std::max(nq, 1), 4);
    if (mneed > c->mat_cap) {
      PK_CUDA(cudaStreamSynchronize(c->stream));
      scratch_moved(c);
      if (c->mat) cudaFree(c->mat);
      c->mat = nullptr;
      c->mat_cap = 0;
      PK_CUDA(cudaMalloc(&c->mat, mneed * sizeof(double)));
      c->mat_cap = mneed;
    }
  }
  const bool k1 = geo.leaf && geo.K == 1 && warp_k1(c, geo);
  if (geo.leaf && geo.logf == 0 && !k1) return PK_OK;
  size_t need = geo.leaf && !k1 ? (size_t)geo.units * 32 * (size_t)std::max(nq, 1)
                                : (size_t)geo.G * (size_t)std::max(nq, 1);
  if (need <= c->spill_cap) return PK_OK;
  PK_CUDA(cudaStreamSynchronize(c->stream));
  scratch_moved(c);
  if (c->spill) cudaFree(c->spill);
  c->spill = nullptr;
  c->spill_cap = 0;
  PK_CUDA(cudaMalloc(&c->spill, need * sizeof(double)));
  c->spill_cap = need;
  return PK_OK;
}

// the VEC pre-pass buffer (n doubles) for a long-row matrix; outside any
// graph capture (solver set-up, kernel-level entries)
static int ensure_vec(pk_ctx* c, const pk_mat* a) {
  if (!a || !a->vec_rows || (size_t)a->n_rows <= c->vec_cap) return PK_OK;
  PK_CUDA(cudaStreamSynchronize(c->stream));
  scratch_moved(c);
  if (c->vecbuf) cudaFree(c->vecbuf);
  c->vecbuf = nullptr;
  c->vec_cap = 0;
  PK_CUDA(cudaMalloc(&c->vecbuf, (size_t)a->n_rows * sizeof(double)));
  c->vec_cap = (size_t)a->n_rows;
  return PK_OK;
}

static Scratch scratch_of(const pk_ctx* c) { return Scratch{c->spill, c->gtick, c->ticket}; }

// Raise a kernel's dynamic shared-memory limit when a launch needs more than
// the default 48 KB minus its static shared memory (the finalizer's 8 KB
// stage-2 staging buffer lives there).  The attribute is per device, so the
// granted size is tracked per (device, kernel), under a lock (pk_solve_batch
// workers launch concurrently), and is only ever raised.
static std::mutex g_smem_mu;
static std::map<std::pair<int, const void*>, size_t> g_smem_granted;

template <class K>
static int allow_dynamic_smem(K kern, size_t dyn) {
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_smem_mu);
  size_t& granted = g_smem_granted[{dev, (const void*)kern}];
  if (dyn <= granted) return PK_OK;
  cudaFuncAttributes fa;
  PK_CUDA(cudaFuncGetAttributes(&fa, kern));
  if (dyn + fa.sharedSizeBytes > 48 * 1024)
    PK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  granted = dyn;
  return PK_OK;
}

template <class K>
static int engine_grid(const pk_ctx* c, K kern, size_t smem, int64_t units, int threads = kThreads) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
  int64_t cap = (int64_t)c->sm_count * occ;
  return (int)std::max<int64_t>(1, std::min<int64_t>(units, cap));
}

static int grid_elem(const pk_ctx* c, int64_t n, int block) {
  int64_t want = (n + block - 1) / block;
  int64_t cap = (int64_t)c->sm_count * 16;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
}

// U = rows per thread per batch (chunks per batch = 8 U).
template <class Op, class = void>
struct RowsPerThread { static constexpr int value = 2; };
template <class Op>
struct RowsPerThread<Op, std::void_t<decltype(Op::kRowsPerThread)>> { static constexpr int value = Op::kRowsPerThread; };

template <class Op, class = void>
struct WarpRows { static constexpr int value = 4; };
template <class Op>
struct WarpRows<Op, std::void_t<decltype(Op::kWarpRows)>> { static constexpr int value = Op::kWarpRows; };

template <int NQ, class Op, int U = (NQ <= 4 ? RowsPerThread<Op>::value : 1)>
static int launch_reduce(pk_ctx* c, cudaStream_t s, int64_t n, const Op& op, ScalarPtrs sp,
                         double* part, int ld, int col0, SolveState* st = nullptr, int gate = GATE_NONE,
                         const int32_t* skip = nullptr, int fin = FIN_NONE, int fin_arg = 0,
                         int nstore = NQ) {
  Geom geo = make_geom(n, c->ng, c->gs, min_units(c));
  if (!geo.leaf && (size_t)geo.G * (size_t)nstore > c->spill_cap)
    return fail(PK_ERR_INVALID, "engine scratch not sized (ensure_scratch)");
  if (geo.leaf && geo.logf > 0 && (size_t)geo.units * 32 * NQ > c->spill_cap)
    return fail(PK_ERR_INVALID, "engine scratch not sized (ensure_scratch)");
  if constexpr (Op::kSpmv) {
    if constexpr (!std::decay_t<decltype(op.A)>::kSell && std::is_same<typename Op::RowT, int32_t>::value) {
      if (op.A.vec && c->vecbuf && c->vec_cap >= (size_t)n) {
        // long rows: warp-cooperative row sums, then the operator as an
        // elementwise reduction over them
        auto kv = k_rowsum_warp<Op>;
        const int64_t rpb = (int64_t)(32 >> op.A.vec) * kVecWarps;  // rows per CTA pass
        const int grid = engine_grid(c, kv, 0, (n + rpb - 1) / rpb, 32 * kVecWarps);
        cudaError_t e = launch_k(c->pdl, kv, dim3((unsigned)grid), dim3(32 * kVecWarps), 0, s, n, op, sp, c->vecbuf,
                                 st, gate, skip, (int)op.A.vec);
        if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("VEC row-sum launch: ") + cudaGetErrorString(e));
        OpPre<Op> pre{op, c->vecbuf};
        return launch_reduce<NQ>(c, s, n, pre, sp, part, ld, col0, st, gate, skip, fin, fin_arg, nstore);
      }
    }
  }
#ifdef PK_MAT_ENGINE
  if constexpr (Op::kSpmv && NQ <= 4) {
    if (mat_applies(c, geo) && c->mat_cap >= (size_t)n * (size_t)nstore) {
      auto kr = k_mat_rows<NQ, Op>;
      cudaError_t e = launch_k(c->pdl, kr, dim3(engine_grid(c, kr, 0, (n + 255) / 256, 256)), dim3(256), 0, s, n,
                               op, sp, c->mat, nstore, st, gate, skip);
      if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("two-phase rows launch: ") + cudaGetErrorString(e));
      const int fd = (int)std::max<size_t>(engine_tail_doubles(geo, NQ), 1024);
      auto kf = k_mat_fold<NQ>;
      PK_TRY(allow_dynamic_smem(kf, (size_t)fd * sizeof(double)));
      e = launch_k(c->pdl, kf, dim3((unsigned)((geo.G + mat_lanes(NQ) - 1) / mat_lanes(NQ))), dim3(kThreads),
                   (size_t)fd * sizeof(double), s, geo, (const double*)c->mat, part, ld, col0, nstore, scratch_of(c),
                   st, gate, skip, fin, fin_arg, fd, mat_discard(c, geo));
      if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("two-phase fold launch: ") + cudaGetErrorString(e));
      return PK_OK;
    }
  }
#endif
  if constexpr (!Op::kSpmv) {
    if (c->lane_engine && !geo.leaf && geo.gs >= 32 && geo.K >= 2) {
      // elementwise operator on a CHAIN geometry: thread = lane, in-register
      // chain fold, no staging (engine_lane)
      // chunks of loads in flight per thread, by the bytes a row loads: light
      // rows (dots, normalize, updates) need many chunks to cover a latency,
      // wide ones (multi-dot, Gram-Schmidt) few (registers)
      constexpr size_t IB = sizeof(typename Op::Item);
      constexpr int D = IB <= 16 ? PK_LANE_D_LIGHT : (IB <= 32 ? 16 : (IB <= 64 ? 8 : (IB <= 160 ? PK_LANE_D_WIDE : 2)));
      const int T = lane_cta_threads(geo);
      const int sd = (int)std::max<size_t>(std::max<size_t>(engine_tail_doubles(geo, NQ), (size_t)NQ * T), 1024);
      auto kl = k_reduce_lane<NQ, D, Op>;
      PK_TRY(allow_dynamic_smem(kl, (size_t)sd * sizeof(double)));
      cudaError_t e = launch_k(c->pdl, kl, dim3((unsigned)((geo.G + T - 1) / T)), dim3(T), (size_t)sd * sizeof(double),
                               s, geo, op, sp, part, ld, col0, nstore, scratch_of(c), st, gate, skip, fin, fin_arg, sd);
      if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("lane engine launch: ") + cudaGetErrorString(e));
      return PK_OK;
    }
  }
#ifdef PK_TILE_ENGINE
  if constexpr (Op::kSpmv && NQ <= 4) {
    if (tiles_apply(c, geo) && c->mat && c->mat_cap >= (size_t)n * (size_t)nstore) {
      auto kt = k_reduce_tiles<NQ, Op>;
      const size_t tail = geo.gs > 256 ? engine_tail_doubles(geo, NQ) : (size_t)NQ * 256;
      const int sd = (int)std::max<size_t>(tail, 1024);
      PK_TRY(allow_dynamic_smem(kt, (size_t)sd * sizeof(double)));
      const int64_t tiles = geo.K * (geo.gs / 256) * geo.n_groups;
      const int grid = engine_grid(c, kt, (size_t)sd * sizeof(double), tiles, 256);
      cudaError_t e = launch_k(c->pdl, kt, dim3((unsigned)grid), dim3(256), (size_t)sd * sizeof(double), s, geo, op, sp,
                               part, ld, col0, nstore, scratch_of(c), st, gate, skip, fin, fin_arg, c->mat, sd,
                               mat_discard(c, geo));
      if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("tile engine launch: ") + cudaGetErrorString(e));
      return PK_OK;
    }
  }
#endif
  if constexpr (Op::kSpmv && NQ <= 2) {
    if constexpr (!std::decay_t<decltype(op.A)>::kSell && std::is_same<typename Op::RowT, int32_t>::value) {
      if (c->bulk && !geo.leaf && geo.gs >= 32 && geo.gs <= 1024 && geo.K >= c->bulk_mink && geo.K <= c->bulk_maxk &&
          NQ <= c->bulk_maxq &&
          op.A.blk >= 0) {
        constexpr int W = PK_BULK_W, R = PK_BULK_R;
        BulkCfg bc = bulk_cfg<NQ, W, R, Op>(op.A.blk);
        const bool pdl = c->pdl || c->bulk_pdl;
        bc.pdl = pdl ? 1 : 0;
        const size_t tail = std::max(warp_chain_smem_bytes(geo, NQ), (size_t)kWarpStage2Doubles * sizeof(double));
        const size_t smem = std::max((size_t)bc.total, (size_t)bc.base + tail);
        if (smem <= 100 * 1024 && op.A.maxr <= Op::kSlots) {
          auto kb = k_reduce_bulk<NQ, W, R, PK_BULK_MINB, Op>;
          PK_TRY(allow_dynamic_smem(kb, smem));
          const int smem_d = (int)((smem - bc.base) / sizeof(double));
          cudaError_t e = launch_k(pdl, kb, dim3((unsigned)geo.units), dim3(32 * (W + 1)), smem, s, geo, op, sp,
                                   part, ld, col0, nstore, scratch_of(c), st, gate, skip, fin, fin_arg, bc, smem_d);
          if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("bulk engine launch: ") + cudaGetErrorString(e));
          return PK_OK;
        }
      }
    }
  }
  if constexpr (Op::kSpmv && NQ <= 4) {
    if (c->lane_spmv && !geo.leaf && geo.gs >= 32 && geo.K >= 2 && geo.K <= c->lane_spmv_maxk) {
      const int T = lane_cta_threads(geo);
      const int sd = (int)std::max<size_t>(std::max<size_t>(engine_tail_doubles(geo, NQ), (size_t)NQ * T), 1024);
      auto kl = k_reduce_lane_spmv<NQ, PK_LANE_P, Op>;
      PK_TRY(allow_dynamic_smem(kl, (size_t)sd * sizeof(double)));
      cudaError_t e = launch_k(c->pdl, kl, dim3((unsigned)((geo.G + T - 1) / T)), dim3(T), (size_t)sd * sizeof(double),
                               s, geo, op, sp, part, ld, col0, nstore, scratch_of(c), st, gate, skip, fin, fin_arg, sd);
      if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("lane SpMV engine launch: ") + cudaGetErrorString(e));
      return PK_OK;
    }
  }
  if constexpr (NQ <= 4) {
  // single-chunk lanes (n <= G) also go to the warp engine when the context
  // allows it (PK_WARP_K1): one warp per 32 lanes, no leaf stacks or splits
  const bool k1 = geo.leaf && geo.K == 1 && warp_k1(c, geo);
  const Geom gw = k1 ? make_geom(n, c->ng, c->gs, min_units(c), true) : geo;
  if (k1 && (size_t)gw.G * (size_t)nstore > c->spill_cap)
    return fail(PK_ERR_INVALID, "engine scratch not sized (ensure_scratch)");
  if (!gw.leaf && gw.gs >= 32 && gw.gs <= 1024 && gw.K >= (k1 ? 1 : 2) && gw.K <= 8) {
    const Geom& geo = gw;
    // warp-per-unit chain engine (no shared staging, no CTA barrier): wins
    // for short chains (small, latency-bound systems, e.g. CG 512^2: 20.6 vs
    // 26.8 us/iter); long chains keep the CTA engine (C2: 44.7 vs 63.8 us)
    constexpr int R = WarpRows<Op>::value;
    const size_t wsm = std::max(warp_chain_smem_bytes(geo, NQ), (size_t)kWarpStage2Doubles * sizeof(double));
    auto kw = k_reduce_warp<NQ, R, Op>;
    PK_TRY(allow_dynamic_smem(kw, wsm));
    // grid-stride over the units, capped at the context's SM budget (batch
    // workers run many small solves side by side)
    const int wgrid = engine_grid(c, kw, wsm, geo.units, 32);
    cudaError_t e = launch_k(c->pdl, kw, dim3((unsigned)wgrid), dim3(32), wsm, s, geo, op, sp, part, ld, col0,
                             nstore, scratch_of(c), st, gate, skip, fin, fin_arg);
    if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("warp engine launch: ") + cudaGetErrorString(e));
    return PK_OK;
  }
  }
  size_t smem = engine_smem_bytes(geo, NQ, U);
#ifdef PK_STAGED_ENGINE
  if constexpr (Op::kSpmv) {
    if (c->staged && !geo.leaf && geo.gs >= 32) {
      geo.staged = 1;
      smem += staged_extra_bytes(U, Op::kSlots);
    }
  }
#endif
  constexpr int MINB = NQ > 8 ? 1 : (NQ > 4 ? 2 : Op::kMinBlocks);
  auto kern = k_reduce<NQ, U, MINB, Op>;
  if (smem > 200 * 1024) return fail(PK_ERR_UNSUPPORTED, "reduction geometry needs too much shared memory");
  PK_TRY(allow_dynamic_smem(kern, smem));
  const int grid = engine_grid(c, kern, smem, geo.units);
  cudaError_t e = launch_k(c->pdl, kern, dim3(grid), dim3(kThreads), smem, s, geo, op, sp, part, ld, col0, nstore,
                           scratch_of(c), st, gate, skip, fin, fin_arg);
  if (e != cudaSuccess)
    return fail(PK_ERR_CUDA, std::string("engine launch (nq=") + std::to_string(NQ) + ", smem=" +
                                 std::to_string(smem) + ", grid=" + std::to_string(grid) + ", leaf=" +
                                 std::to_string(geo.leaf) + "): " + cudaGetErrorString(e));
  return PK_OK;
}

template <class Op, class = void>
struct HasVec2 : std::false_type {};
template <class Op>
struct HasVec2<Op, std::void_t<typename Op::Item2>> : std::true_type {};

template <class Op, class = void>
struct SweepPairs { static constexpr int value = 0; };
template <class Op>
struct SweepPairs<Op, std::void_t<decltype(Op::kPairs)>> { static constexpr int value = Op::kPairs; };

#ifndef PK_SWEEP_PAIRS
#define PK_SWEEP_PAIRS 4
#endif
constexpr int kSweepPairs = PK_SWEEP_PAIRS;  // row pairs per thread of k_sweep2 (2 x 16 B per stream in flight)

template <class Op>
static int launch_sweep(pk_ctx* c, cudaStream_t s, int64_t n, const Op& op, ScalarPtrs sp = ScalarPtrs{},
                        SolveState* st = nullptr, int gate = GATE_NONE) {
  if constexpr (Op::kSpmv) {
    if constexpr (!std::decay_t<decltype(op.A)>::kSell && std::is_same<typename Op::RowT, int32_t>::value) {
      if (op.A.vec && c->vecbuf && c->vec_cap >= (size_t)n) {
        auto kv = k_rowsum_warp<Op>;
        const int64_t rpb = (int64_t)(32 >> op.A.vec) * kVecWarps;
        const int grid = engine_grid(c, kv, 0, (n + rpb - 1) / rpb, 32 * kVecWarps);
        PK_CUDA(launch_k(c->pdl, kv, dim3((unsigned)grid), dim3(32 * kVecWarps), 0, s, n, op, sp, c->vecbuf, st, gate,
                         (const int32_t*)nullptr, (int)op.A.vec));
        return launch_sweep(c, s, n, OpPre<Op>{op, c->vecbuf}, sp, st, gate);
      }
    }
  }
  if constexpr (HasVec2<Op>::value) {
    if (!c->sweep_scalar && op.aligned16()) {
      constexpr int UP = SweepPairs<Op>::value > 0 ? SweepPairs<Op>::value : kSweepPairs;
      const int64_t np = n >> 1;
      const int64_t grid = std::max<int64_t>(1, (np + 256 * UP - 1) / (256 * UP));
      PK_CUDA(launch_k(c->pdl, k_sweep2<Op, UP>, dim3((unsigned)grid), dim3(256), 0, s, n, op, sp, st, gate));
      return PK_OK;
    }
  }
  auto kern = k_sweep<Op>;
  // sweep_one_batch: one CTA per 256 x PK_SWEEP_V rows (several waves), so
  // every thread's rows are a single batch of loads in flight; otherwise the
  // grid is capped at the resident CTAs and threads loop
  int64_t grid = engine_grid(c, kern, 0, (n + 255) / 256, 256);
  if (c->sweep_one_batch && !Op::kSpmv) grid = std::max<int64_t>(1, (n + 256 * PK_SWEEP_V - 1) / (256 * PK_SWEEP_V));
  PK_CUDA(launch_k(c->pdl, kern, dim3((unsigned)grid), dim3(256), 0, s, n, op, sp, st, gate));
  return PK_OK;
}

template <typename RowT, bool SELL = false>
static Csr<RowT, SELL> csr_of(const pk_mat* a) {
  Csr<RowT, SELL> A{(const RowT*)a->rowptr, a->cols, a->vals};
  A.blk = (int32_t)std::min<int64_t>(a->blk_max, INT32_MAX);
  A.maxr = (int32_t)std::min<int64_t>(a->max_row, INT32_MAX);
  // VEC pre-pass lanes per row (log2): about a quarter of the average row length, 4..32
  if (a->vec_rows) {
    const int64_t avg = a->nnz / std::max<int64_t>(a->n_rows, 1);
    A.vec = avg >= 96 ? 5 : (avg >= 48 ? 4 : (avg >= 24 ? 3 : 2));
  }
  if constexpr (SELL) {
    A.sp = (const RowT*)a->sell_ptr;
    A.sc = a->sell_cols;
    A.sv = a->sell_vals;
  }
  return A;
}

// nnz slots per lane per pass of the SpMV tile loop: 5 (2-D 5-point rows) or
// 7 (3-D 7-point and anything longer; longer rows take several passes).
static inline bool wide_rows(const pk_mat* a) { return a->max_row > 5; }

// SpMV with NQ fused dots; dispatch on the row index type and slot count.
template <int NQ, typename RowT, int S, bool SELL = false>
static int spmv_fused_t(pk_ctx* c, cudaStream_t s, const pk_mat* a, const double* p, double* q,
                        const int32_t* kinds, const double* const* w, double* part, int ld, int col0,
                        SolveState* st, int gate, int fin, int fin_arg) {
  OpSpmvFused<RowT, NQ, S, SELL> op{};
  op.A = csr_of<RowT, SELL>(a);
  op.p = p;
  op.q = q;
  for (int k = 0; k < 4; ++k) { op.kind[k] = PK_DOT_RESULT; op.w[k] = nullptr; }
  for (int k = 0; k < NQ; ++k) { op.kind[k] = kinds[k]; op.w[k] = w ? w[k] : nullptr; }
  if constexpr (NQ == 0) {
    return launch_sweep(c, s, a->n_rows, op, ScalarPtrs{}, st, gate);
  } else {
    return launch_reduce<NQ>(c, s, a->n_rows, op, ScalarPtrs{}, part, ld, col0, st, gate, nullptr, fin, fin_arg);
  }
}

template <int NQ>
static int spmv_fused_dispatch(pk_ctx* c, cudaStream_t s, const pk_mat* a, const double* p, double* q,
                               const int32_t* kinds, const double* const* w, double* part, int ld, int col0,
                               SolveState* st = nullptr, int gate = GATE_NONE, int fin = FIN_NONE,
                               int fin_arg = 0) {
  if (a->row64) {
    if (wide_rows(a)) return spmv_fused_t<NQ, int64_t, 7>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    return spmv_fused_t<NQ, int64_t, 5>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
  }
  if (a->sell) {
    if (wide_rows(a)) return spmv_fused_t<NQ, int32_t, 7, true>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    return spmv_fused_t<NQ, int32_t, 5, true>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
  }
  if (wide_rows(a)) return spmv_fused_t<NQ, int32_t, 7>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
  return spmv_fused_t<NQ, int32_t, 5>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
}

static int spmv_fused_any(pk_ctx* c, cudaStream_t s, const pk_mat* a, const double* p, double* q, int nq,
                          const int32_t* kinds, const double* const* w, double* part, int ld, int col0,
                          SolveState* st = nullptr, int gate = GATE_NONE, int fin = FIN_NONE, int fin_arg = 0) {
  switch (nq) {
    case 0: return spmv_fused_dispatch<0>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    case 1: return spmv_fused_dispatch<1>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    case 2: return spmv_fused_dispatch<2>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    case 3: return spmv_fused_dispatch<3>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    case 4: return spmv_fused_dispatch<4>(c, s, a, p, q, kinds, w, part, ld, col0, st, gate, fin, fin_arg);
    default: return fail(PK_ERR_INVALID, "spmv_fused carries 1 to 4 quantities");
  }
}

template <typename RowT, int S, bool SELL = false>
static int residual_t(pk_ctx* c, cudaStream_t s, const pk_mat* a, const double* x, const double* b, double* r,
                      double* copy1, double* copy2, double* part, SolveState* st, int gate, int fin, int fin_arg,
                      int ld, int col0) {
  OpResidual<RowT, S, SELL> op{};
  op.A = csr_of<RowT, SELL>(a);
  op.x = x;
  op.b = b;
  op.r = r;
  op.copy1 = copy1;
  op.copy2 = copy2;
  return launch_reduce<1>(c, s, a->n_rows, op, ScalarPtrs{}, part, ld, col0, st, gate, nullptr, fin, fin_arg);
}

// r = b - A x (+ copies) with <r,r> partials (column col0 of a ld-wide array).
static int residual_any(pk_ctx* c, cudaStream_t s, const pk_mat* a, const double* x, const double* b,
                        double* r, double* copy1, double* copy2, double* part, SolveState* st = nullptr,
                        int gate = GATE_NONE, int fin = FIN_NONE, int fin_arg = 0, int ld = 1, int col0 = 0) {
  if (a->row64) {
    if (wide_rows(a)) return residual_t<int64_t, 7>(c, s, a, x, b, r, copy1, copy2, part, st, gate, fin, fin_arg, ld, col0);
    return residual_t<int64_t, 5>(c, s, a, x, b, r, copy1, copy2, part, st, gate, fin, fin_arg, ld, col0);
  }
  if (a->sell) {
    if (wide_rows(a)) return residual_t<int32_t, 7, true>(c, s, a, x, b, r, copy1, copy2, part, st, gate, fin, fin_arg, ld, col0);
    return residual_t<int32_t, 5, true>(c, s, a, x, b, r, copy1, copy2, part, st, gate, fin, fin_arg, ld, col0);
  }
  if (wide_rows(a)) return residual_t<int32_t, 7>(c, s, a, x, b, r, copy1, copy2, part, st, gate, fin, fin_arg, ld, col0);
  return residual_t<int32_t, 5>(c, s, a, x, b, r, copy1, copy2, part, st, gate, fin, fin_arg, ld, col0);
}

static int dot_partials(pk_ctx* c, cudaStream_t s, int64_t n, const double* x, const double* y,
                        double* part, SolveState* st = nullptr, int gate = GATE_NONE, int fin = FIN_NONE,
                        int fin_arg = 0) {
  OpDot op{x, y};
  return launch_reduce<1>(c, s, n, op, ScalarPtrs{}, part, 1, 0, st, gate, nullptr, fin, fin_arg);
}

template <int NB>
static int multidot_t(pk_ctx* c, cudaStream_t s, int64_t n, int nb, const double* const* basis,
                      const double* v, double* part, int ld, int col0, SolveState* st, int gate, int fin,
                      int fin_arg) {
  OpMultiDot<NB> op{};
  op.v = v;
  op.nb = nb;
  for (int j = 0; j < NB; ++j) op.b[j] = j < nb ? basis[j] : nullptr;
  return launch_reduce<NB>(c, s, n, op, ScalarPtrs{}, part, ld, col0, st, gate, nullptr, fin, fin_arg, nb);
}

// Largest NB whose shared-memory footprint fits for this geometry.
static int multidot_nb_cap(const pk_ctx* c, int64_t n) {
  Geom geo = make_geom(n, c->ng, c->gs);
  // at most 16 quantities per pass: wider passes need so much staging smem
  // (and registers) that only 1-2 CTAs fit per SM; re-reading v per pass is
  // cheaper than that loss of occupancy (GMRES(30) 128^3: measured)
  const char* ev = getenv("PK_MULTIDOT_CAP");
  const int top = ev ? atoi(ev) : 16;
  for (int nb : {32, 16, 8, 4, 2, 1}) {
    if (nb <= top && engine_smem_bytes(geo, nb, 1) <= 192 * 1024) return nb;
  }
  return 1;
}

// <b_j, v> partials for nb vectors, in passes of at most the smem cap.
// ---------------------------------------------------------------------------
// MDQ multi-dot: quantity-parallel Gram-Schmidt coefficients
// ---------------------------------------------------------------------------
//
// c_j = <v_j, w> for the nb basis vectors of a classical Gram-Schmidt step
// (fused.py:222-243).  The LANE engine gives one thread a lane and ALL nb
// quantities (nb + 1 loads per chunk, ~200 registers, 32768 threads for the
// whole GPU); here a warp owns one (32-lane unit, quantity) pair: thread =
// (lane, q) folds lane t's chain of v_q[row] * w[row] products in chunk
// order with 16 chunks of loads in flight (the reference order,
// linalg.py:300-303 -- exactly OpMultiDot's products and adds), the 8 warps
// of a CTA are 8 quantities of the same 32 lanes (w is read from DRAM once,
// then hits L1).  Lane values -> spill; the CTA that completes a group (all
// its units and quantity blocks) runs the group's halving trees, 8
// quantities at a time; the CTA completing the last group finalizes.
struct MdqPtrs {
  const double* p[32];
};
constexpr int kMdqD = 16;
__global__ void __launch_bounds__(256)
    k_multidot_q(const __grid_constant__ Geom geo, const double* __restrict__ w, const __grid_constant__ MdqPtrs bp,
                 int nb, double* part, int ld, int col0, Scratch scr, SolveState* st, int gate, int fin, int fin_arg,
                 int smem_d) {
  extern __shared__ double smem[];
  __shared__ int s_flag;
  __shared__ int s_last;
  pdl_wait();
  pdl_trigger();
  const bool ing = (gate & GATE_IN_GRAPH) != 0;
  gate &= 0xff;
  const GateVals gv = gate_load(st, gate);
  if (!gate_eval(st, gate, ing, gv)) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nqb = (nb + 7) >> 3;
  const int64_t unit = blockIdx.x / nqb;
  const int qb = (int)(blockIdx.x - unit * nqb);
  const int q = qb * 8 + warp;
  const int64_t t = unit * 32 + lane;  // lane id (< G: the units tile [0, G))
  const int64_t n = geo.n, G = geo.G, K = geo.K;
  if (tid == 0) s_last = 0;
  if (q < nb) {
    const double* __restrict__ v = bp.p[q];
    double acc = 0.0;
    for (int64_t k0 = 0; k0 < K; k0 += kMdqD) {
      double a[kMdqD], b[kMdqD];
#pragma unroll
      for (int d = 0; d < kMdqD; ++d) {
        const int64_t row = (k0 + d) * G + t;
        const int64_t rc = row < n ? row : t;  // clamped: every load unconditional
        a[d] = __ldg(v + rc);
        b[d] = __ldg(w + rc);
      }
#pragma unroll
      for (int d = 0; d < kMdqD; ++d)
        if (k0 + d < K && (k0 + d) * G + t < n) acc = add_rn(acc, mul_rn(a[d], b[d]));
    }
    scr.spill[(int64_t)q * G + t] = acc;
  }
  __syncthreads();
  const int g = (int)(unit * 32 / geo.gs);
  if (tid == 0) {
    const unsigned per = (unsigned)(geo.gs / 32) * (unsigned)nqb;
    const unsigned tk = ticket_add(scr.gtick + g, 1u);
    const int last = tk == per - 1;
    if (last) {
      scr.gtick[g] = 0u;
      acquire_fence();
    }
    s_flag = last;
  }
  __syncthreads();
  if (s_flag) {
    for (int q0 = 0; q0 < nb; q0 += 8)
      group_tree<8>(geo, g, scr.spill + (int64_t)q0 * G, smem, part, ld, col0 + q0, nb - q0 < 8 ? nb - q0 : 8);
    if (tid == 0) {
      unsigned* ticket = st ? &st->ticket : scr.ticket;
      const unsigned tk = ticket_add(ticket, 1u);
      if (tk + 1u == (unsigned)geo.n_groups) {
        *ticket = 0u;
        acquire_fence();
        s_last = 1;
      }
    }
  }
  __syncthreads();
  if (s_last && fin != FIN_NONE && st && tid < 32) finalize(st, fin, fin_arg, ing, smem, smem_d);
}

static int multidot_any(pk_ctx* c, cudaStream_t s, int64_t n, int nb, const double* const* basis,
                        const double* v, double* part, int ld, int col0, SolveState* st = nullptr,
                        int gate = GATE_NONE, int fin = FIN_NONE, int fin_arg = 0) {
  {
    const Geom geo = make_geom(n, c->ng, c->gs, min_units(c));
    if (c->mdq && nb >= 1 && nb <= 32 && !geo.leaf && geo.gs >= 32 && geo.K >= 2 &&
        (size_t)geo.G * (size_t)nb <= c->spill_cap) {
      MdqPtrs bp{};
      for (int j = 0; j < nb; ++j) bp.p[j] = basis[j];
      const int sd = (int)std::max<size_t>(engine_tail_doubles(geo, 8), 1024);
      PK_TRY(allow_dynamic_smem(k_multidot_q, (size_t)sd * sizeof(double)));
      const int64_t grid = geo.units * ((nb + 7) / 8);
      cudaError_t e = launch_k(c->pdl, k_multidot_q, dim3((unsigned)grid), dim3(256), (size_t)sd * sizeof(double), s,
                               geo, v, bp, nb, part, ld, col0, scratch_of(c), st, gate, fin, fin_arg, sd);
      if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("MDQ multi-dot launch: ") + cudaGetErrorString(e));
      return PK_OK;
    }
  }
  int cap = multidot_nb_cap(c, n);
  int done = 0;
  while (done < nb) {
    int todo = std::min(nb - done, cap);
    bool last = done + todo == nb;
    int f = last ? fin : FIN_NONE;
    int rc;
    if (todo <= 1) rc = multidot_t<1>(c, s, n, todo, basis + done, v, part, ld, col0 + done, st, gate, f, fin_arg);
    else if (todo <= 2) rc = multidot_t<2>(c, s, n, todo, basis + done, v, part, ld, col0 + done, st, gate, f, fin_arg);
    else if (todo <= 4) rc = multidot_t<4>(c, s, n, todo, basis + done, v, part, ld, col0 + done, st, gate, f, fin_arg);
    else if (todo <= 8) rc = multidot_t<8>(c, s, n, todo, basis + done, v, part, ld, col0 + done, st, gate, f, fin_arg);
    else if (todo <= 16) rc = multidot_t<16>(c, s, n, todo, basis + done, v, part, ld, col0 + done, st, gate, f, fin_arg);
    else rc = multidot_t<32>(c, s, n, todo, basis + done, v, part, ld, col0 + done, st, gate, f, fin_arg);
    PK_TRY(rc);
    done += todo;
  }
  return PK_OK;
}

template <int NB>
static int gs_update_t(pk_ctx* c, cudaStream_t s, int64_t n, double* v, int nb, const double* const* basis,
                       const double* coef_dev, const double* acc_in, double* part, SolveState* st, int gate, int fin,
                       int fin_arg) {
  OpGsUpdate<NB> op{};
  op.v = v;
  op.nb = nb;
  op.coef = coef_dev;
  op.acc_in = acc_in;
  for (int j = 0; j < NB; ++j) op.b[j] = j < nb ? basis[j] : nullptr;
  ScalarPtrs sp{coef_dev, nullptr, nullptr, nullptr};
  return launch_reduce<1>(c, s, n, op, sp, part, 1, 0, st, gate, nullptr, fin, fin_arg);
}

template <int NB>
static int gs_acc_t(pk_ctx* c, cudaStream_t s, int64_t n, int nb, const double* const* basis, const double* coef_dev,
                    const double* acc_in, double* acc_out, SolveState* st, int gate) {
  OpGsAcc<NB> op{};
  op.nb = nb;
  op.coef = coef_dev;
  op.acc_in = acc_in;
  op.acc_out = acc_out;
  for (int j = 0; j < NB; ++j) op.b[j] = j < nb ? basis[j] : nullptr;
  return launch_sweep(c, s, n, op, ScalarPtrs{}, st, gate);
}

template <int NB>
static int gs_sweep_t(pk_ctx* c, cudaStream_t s, int64_t n, double* v, int nb, const double* const* basis,
                      const double* coef_dev, const double* acc_in, SolveState* st, int gate) {
  OpGsSweep<NB> op{};
  op.v = v;
  op.nb = nb;
  op.coef = coef_dev;
  op.acc_in = acc_in;
  for (int j = 0; j < NB; ++j) op.b[j] = j < nb ? basis[j] : nullptr;
  return launch_sweep(c, s, n, op, ScalarPtrs{coef_dev, nullptr, nullptr, nullptr}, st, gate);
}

// the lane / CTA CHAIN engines apply (K >= 2): the split update's dot runs on
// the LANE engine; one-element-per-lane geometries keep the fused update
static bool geo_is_leaf(const pk_ctx* c, int64_t n) {
  return make_geom(n, c->ng, c->gs, min_units(c)).leaf != 0;
}

// Gram-Schmidt update over nb basis vectors: chunks of gs_chunk (<= 32)
// vectors accumulate through `acc` (an n-vector; needed only when nb >
// gs_chunk), the last chunk subtracts the sum from v and emits the <v,v>
// partials.  Same rounding sequence for any chunking.
constexpr int kGsChunk = 32;  // largest chunk (the accumulator is allocated for restart - 1 > gs_chunk)

static int gs_update_any(pk_ctx* c, cudaStream_t s, int64_t n, double* v, int nb, const double* const* basis,
                         const double* coef_dev, double* part, SolveState* st = nullptr, int gate = GATE_NONE,
                         int fin = FIN_NONE, int fin_arg = 0, double* acc = nullptr) {
  int j0 = 0;
  const double* acc_in = nullptr;
  const int ch = acc ? c->gs_chunk : kGsChunk;
  while (nb - j0 > ch) {
    if (!acc) return fail(PK_ERR_INVALID, "Gram-Schmidt update over more than 32 vectors needs an accumulator");
    int rc;
    if (ch <= 4) rc = gs_acc_t<4>(c, s, n, ch, basis + j0, coef_dev + j0, acc_in, acc, st, gate);
    else if (ch <= 8) rc = gs_acc_t<8>(c, s, n, ch, basis + j0, coef_dev + j0, acc_in, acc, st, gate);
    else if (ch <= 16) rc = gs_acc_t<16>(c, s, n, ch, basis + j0, coef_dev + j0, acc_in, acc, st, gate);
    else rc = gs_acc_t<32>(c, s, n, ch, basis + j0, coef_dev + j0, acc_in, acc, st, gate);
    PK_TRY(rc);
    acc_in = acc;
    j0 += ch;
  }
  const int r = nb - j0;
  const double* const* bb = basis + j0;
  const double* cd = coef_dev + j0;
  if (c->gs_split && !geo_is_leaf(c, n)) {
    // elementwise update through 16-byte accesses, then the <v,v> partials
    int rc;
    if (r <= 2) rc = gs_sweep_t<2>(c, s, n, v, r, bb, cd, acc_in, st, gate);
    else if (r <= 4) rc = gs_sweep_t<4>(c, s, n, v, r, bb, cd, acc_in, st, gate);
    else if (r <= 8) rc = gs_sweep_t<8>(c, s, n, v, r, bb, cd, acc_in, st, gate);
    else if (r <= 16) rc = gs_sweep_t<16>(c, s, n, v, r, bb, cd, acc_in, st, gate);
    else rc = gs_sweep_t<32>(c, s, n, v, r, bb, cd, acc_in, st, gate);
    PK_TRY(rc);
    return dot_partials(c, s, n, v, v, part, st, gate, fin, fin_arg);
  }
  if (r <= 1) return gs_update_t<1>(c, s, n, v, r, bb, cd, acc_in, part, st, gate, fin, fin_arg);
  if (r <= 2) return gs_update_t<2>(c, s, n, v, r, bb, cd, acc_in, part, st, gate, fin, fin_arg);
  if (r <= 4) return gs_update_t<4>(c, s, n, v, r, bb, cd, acc_in, part, st, gate, fin, fin_arg);
  if (r <= 8) return gs_update_t<8>(c, s, n, v, r, bb, cd, acc_in, part, st, gate, fin, fin_arg);
  if (r <= 16) return gs_update_t<16>(c, s, n, v, r, bb, cd, acc_in, part, st, gate, fin, fin_arg);
  return gs_update_t<32>(c, s, n, v, r, bb, cd, acc_in, part, st, gate, fin, fin_arg);
}

// ---------------------------------------------------------------------------
// library / contexts
// ---------------------------------------------------------------------------

extern "C" const char* pk_last_error(void) { return g_err.c_str(); }
extern "C" int pk_abi_version(void) { return PK_ABI_VERSION; }

extern "C" int pk_device_count(int* count) {
  if (!count) return fail(PK_ERR_INVALID, "count is NULL");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(PK_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  return PK_OK;
}

extern "C" int pk_ctx_create(int device, int64_t n_groups, int64_t group_size, pk_ctx** out) {
  if (!out) return fail(PK_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (n_groups < 1) return fail(PK_ERR_INVALID, "n_groups must be >= 1, got " + std::to_string(n_groups));
  if (group_size < 1 || (group_size & (group_size - 1)) != 0)
    return fail(PK_ERR_INVALID, "group_size must be a positive power of two, got " + std::to_string(group_size));
  if (n_groups > (1ll << 30) || group_size > (1ll << 30))
    return fail(PK_ERR_UNSUPPORTED, "geometry too large for the device path");
  PK_TRY(set_device(device));
  pk_ctx* c = new pk_ctx();
  c->device = device;
  c->ng = (int32_t)n_groups;
  c->gs = (int32_t)group_size;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) == cudaSuccess) c->sm_count = prop.multiProcessorCount;
  cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaMalloc(&c->scratch, sizeof(SolveState));
  if (e == cudaSuccess) e = cudaMalloc(&c->scratch_flag, 64 * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMalloc(&c->scratch_d, 64 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&c->gtick, ((size_t)n_groups + 1) * sizeof(unsigned));
  if (e == cudaSuccess) e = cudaMemset(c->gtick, 0, ((size_t)n_groups + 1) * sizeof(unsigned));
  if (e == cudaSuccess) c->ticket = c->gtick + n_groups;
  if (e != cudaSuccess) {
    pk_ctx_destroy(c);
    return fail(PK_ERR_CUDA, std::string("context allocation: ") + cudaGetErrorString(e));
  }
  c->stream = c->own;
  if (const char* e2 = getenv("PK_PDL")) c->pdl = atoi(e2) != 0;
  if (const char* e3 = getenv("PK_MAT_MINK")) c->mat_mink = atoi(e3);
  if (const char* e4 = getenv("PK_MAT_DISCARD")) c->mat_discard = atoi(e4) != 0;
  if (const char* e5 = getenv("PK_WARP_K1")) c->warp_k1 = atoi(e5) != 0;
  if (const char* e6 = getenv("PK_SWEEP_ONEBATCH")) c->sweep_one_batch = atoi(e6) != 0;
  if (const char* e7 = getenv("PK_SWEEP_SCALAR")) c->sweep_scalar = atoi(e7) != 0;
  if (const char* e8 = getenv("PK_SELL")) c->sell_mode = atoi(e8);
  if (const char* e9 = getenv("PK_STAGE")) c->staged = atoi(e9) != 0;
  if (const char* e10 = getenv("PK_WS_CACHE")) c->ws_cache_on = atoi(e10) != 0;
  if (const char* e12 = getenv("PK_LANE")) c->lane_engine = atoi(e12) != 0;
  if (const char* e19 = getenv("PK_TILE_MINK")) c->tile_mink = atoi(e19);
  if (const char* e23 = getenv("PK_VEC_MINAVG")) c->vec_min_avg = atoi(e23);
  if (const char* e24 = getenv("PK_MDQ")) c->mdq = atoi(e24) != 0;
  if (const char* e16 = getenv("PK_BULK")) c->bulk = atoi(e16) != 0;
  if (const char* e21 = getenv("PK_BULK_PDL")) c->bulk_pdl = atoi(e21) != 0;
  if (const char* e22 = getenv("PK_BULK_MAXQ")) c->bulk_maxq = atoi(e22);
  if (const char* e20 = getenv("PK_BULK_MAXK")) c->bulk_maxk = atoi(e20);
  if (const char* e17 = getenv("PK_BULK_MINK")) c->bulk_mink = std::max(2, atoi(e17));
  if (const char* e15 = getenv("PK_GS_SPLIT")) c->gs_split = atoi(e15) != 0;
  if (const char* e13 = getenv("PK_LANE_SPMV")) c->lane_spmv = atoi(e13) != 0;
  if (const char* e14 = getenv("PK_LANE_SPMV_MAXK")) c->lane_spmv_maxk = atoi(e14);
  if (const char* e11 = getenv("PK_GS_CHUNK")) c->gs_chunk = std::max(4, std::min(32, atoi(e11)));
  // keep freed workspace memory in the stream-ordered pool between solves
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = c;
  return PK_OK;
}

extern "C" int pk_ctx_destroy(pk_ctx* c) {
  if (!c) return PK_OK;
  for (pk_ctx* w : c->workers) pk_ctx_destroy(w);
  c->workers.clear();
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->own) cudaStreamSynchronize(c->own);
  if (c->ws_cache_free) c->ws_cache_free(c);
  if (c->scratch) cudaFree(c->scratch);
  if (c->scratch_flag) cudaFree(c->scratch_flag);
  if (c->scratch_d) cudaFree(c->scratch_d);
  if (c->gtick) cudaFree(c->gtick);
  if (c->spill) cudaFree(c->spill);
  if (c->mat) cudaFree(c->mat);
  if (c->vecbuf) cudaFree(c->vecbuf);
  if (c->own) cudaStreamDestroy(c->own);
  delete c;
  return PK_OK;
}

extern "C" int pk_ctx_set_debug(pk_ctx* c, pk_debug_fn hook, void* user) {
  if (!c) return fail(PK_ERR_INVALID, "ctx is NULL");
  c->dbg = hook;
  c->dbg_user = user;
  return PK_OK;
}

extern "C" int pk_ctx_set_stream(pk_ctx* c, void* stream) {
  if (!c) return fail(PK_ERR_INVALID, "ctx is NULL");
  c->stream = (cudaStream_t)stream;  // NULL: legacy default stream
  return PK_OK;
}

extern "C" int pk_ctx_reset_stream(pk_ctx* c) {
  if (!c) return fail(PK_ERR_INVALID, "ctx is NULL");
  c->stream = c->own;
  return PK_OK;
}

extern "C" int pk_ctx_synchronize(pk_ctx* c) {
  if (!c) return fail(PK_ERR_INVALID, "ctx is NULL");
  PK_CUDA(cudaStreamSynchronize(c->stream));
  return PK_OK;
}

extern "C" int pk_ctx_geometry(const pk_ctx* c, int64_t* ng, int64_t* gs) {
  if (!c) return fail(PK_ERR_INVALID, "ctx is NULL");
  if (ng) *ng = c->ng;
  if (gs) *gs = c->gs;
  return PK_OK;
}

// ---------------------------------------------------------------------------
// matrices
// ---------------------------------------------------------------------------

static std::atomic<uint64_t> g_mat_uid{1};

static int alloc_mat(pk_ctx* c, int64_t n_rows, int64_t n_cols, int64_t nnz, pk_mat** out) {
  pk_mat* m = new pk_mat();
  m->uid = g_mat_uid.fetch_add(1);
  m->device = c->device;
  m->n_rows = n_rows;
  m->n_cols = n_cols;
  m->nnz = nnz;
  m->row64 = nnz >= (1ll << 31) - 1;
  size_t rsz = (size_t)(n_rows + 1) * (m->row64 ? 8 : 4);
  // pad arrays so vectorised/bulk loads may read a little past the end
  cudaError_t e = cudaMalloc(&m->rowptr, rsz + 512);  // bulk row slices read up to 34 entries
  if (e == cudaSuccess) e = cudaMalloc(&m->cols, (size_t)nnz * 4 + 64);
  if (e == cudaSuccess) e = cudaMalloc(&m->vals, (size_t)nnz * 8 + 64);
  if (e != cudaSuccess) {
    pk_mat_destroy(m);
    return fail(e == cudaErrorMemoryAllocation ? PK_ERR_NOMEM : PK_ERR_CUDA,
                std::string("matrix allocation: ") + cudaGetErrorString(e));
  }
  *out = m;
  return PK_OK;
}

extern "C" int pk_csr_upload(pk_ctx* c, int64_t n_rows, int64_t n_cols, const int64_t* offs, const int64_t* cols,
                             const double* vals, pk_mat** out) {
  if (!c || !out || !offs) return fail(PK_ERR_INVALID, "NULL argument");
  *out = nullptr;
  // canonical-form validation, linalg.py:86-111
  if (n_rows < 0 || n_cols < 0) return fail(PK_ERR_INVALID, "matrix dimensions must be non-negative");
  if (n_rows >= (1ll << 31) - 1 || n_cols >= (1ll << 31) - 1)
    return fail(PK_ERR_UNSUPPORTED, "device path indexes rows and columns with int32");
  if (offs[0] != 0) return fail(PK_ERR_INVALID, "row_offsets must start at 0");
  int64_t max_row = 0;
  for (int64_t i = 0; i < n_rows; ++i) {
    int64_t d = offs[i + 1] - offs[i];
    if (d < 0) return fail(PK_ERR_INVALID, "row_offsets must be non-decreasing");
    max_row = std::max(max_row, d);
  }
  int64_t nnz = offs[n_rows];
  if (nnz > 0 && (!cols || !vals)) return fail(PK_ERR_INVALID, "NULL column/value array");
  for (int64_t i = 0; i < n_rows; ++i) {
    for (int64_t k = offs[i]; k < offs[i + 1]; ++k) {
      if (cols[k] < 0 || cols[k] >= n_cols) return fail(PK_ERR_INVALID, "column index out of range");
      if (k > offs[i] && cols[k] <= cols[k - 1])
        return fail(PK_ERR_INVALID, "column indices must be strictly increasing within each row");
    }
  }
  PK_TRY(set_device(c->device));
  pk_mat* m = nullptr;
  PK_TRY(alloc_mat(c, n_rows, n_cols, nnz, &m));
  m->max_row = max_row;
  std::vector<int32_t> c32((size_t)nnz);
  for (int64_t k = 0; k < nnz; ++k) c32[k] = (int32_t)cols[k];
  cudaError_t e = cudaSuccess;
  if (m->row64) {
    e = cudaMemcpy(m->rowptr, offs, (size_t)(n_rows + 1) * 8, cudaMemcpyHostToDevice);
  } else {
    std::vector<int32_t> r32((size_t)n_rows + 1);
    for (int64_t i = 0; i <= n_rows; ++i) r32[i] = (int32_t)offs[i];
    e = cudaMemcpy(m->rowptr, r32.data(), r32.size() * 4, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && nnz) e = cudaMemcpy(m->cols, c32.data(), (size_t)nnz * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && nnz) e = cudaMemcpy(m->vals, vals, (size_t)nnz * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    pk_mat_destroy(m);
    return fail(PK_ERR_CUDA, std::string("matrix upload: ") + cudaGetErrorString(e));
  }
  int rcf = apply_default_format(c, m);
  if (rcf != PK_OK && rcf != PK_ERR_UNSUPPORTED) {
    pk_mat_destroy(m);
    return rcf;
  }
  *out = m;
  return PK_OK;
}

static int gen_stencil(pk_ctx* c, int32_t family, const int64_t* dims, int32_t ndims, const double* coef,
                       int32_t ncoef, int64_t row_lo, int64_t row_hi, int64_t col_base, int64_t n_cols_local,
                       pk_mat** out);

extern "C" int pk_csr_generate(pk_ctx* c, int32_t family, const int64_t* dims, int32_t ndims, const double* coef,
                               int32_t ncoef, pk_mat** out) {
  return gen_stencil(c, family, dims, ndims, coef, ncoef, 0, -1, 0, -1, out);
}

extern "C" int pk_csr_generate_rows(pk_ctx* c, int32_t family, const int64_t* dims, int32_t ndims,
                                    const double* coef, int32_t ncoef, int64_t row_lo, int64_t row_hi,
                                    int64_t col_base, int64_t n_cols_local, pk_mat** out) {
  if (row_lo < 0 || row_hi < row_lo) return fail(PK_ERR_INVALID, "bad row range");
  return gen_stencil(c, family, dims, ndims, coef, ncoef, row_lo, row_hi, col_base, n_cols_local, out);
}

// Rows [row_lo, row_hi) of a stencil family (row_hi < 0: all rows), columns
// stored as global - col_base, matrix n_cols = n_cols_local (< 0: n).
static int gen_stencil(pk_ctx* c, int32_t family, const int64_t* dims, int32_t ndims, const double* coef,
                       int32_t ncoef, int64_t row_lo, int64_t row_hi, int64_t col_base, int64_t n_cols_local,
                       pk_mat** out) {
  if (!c || !out || !dims) return fail(PK_ERR_INVALID, "NULL argument");
  *out = nullptr;
  StencilSpec sp{};
  int nd = (family == PK_GEN_POISSON2D || family == PK_GEN_CONVDIFF2D) ? 2 : 3;
  if (family < 0 || family > 3) return fail(PK_ERR_INVALID, "unknown generator family");
  if (ndims != nd) return fail(PK_ERR_INVALID, "wrong number of grid dimensions");
  int64_t n = 1;
  for (int d = 0; d < nd; ++d) {
    if (dims[d] < 1) return fail(PK_ERR_INVALID, "grid dimensions must be >= 1");
    sp.dim[d] = dims[d];
    sp.stride[d] = n;
    n *= dims[d];
  }
  if (n >= (1ll << 31) - 1) return fail(PK_ERR_UNSUPPORTED, "grid too large for int32 row indices");
  if (row_hi < 0) row_hi = n;
  if (row_hi > n || row_lo > row_hi) return fail(PK_ERR_INVALID, "row range outside the grid");
  const int64_t n_global = n;
  const int64_t ncols = n_cols_local < 0 ? n_global : n_cols_local;
  sp.row_lo = row_lo;
  sp.col_base = col_base;
  n = row_hi - row_lo;  // rows generated
  // per-direction values: {axis, step, value}
  double diag = 0.0;
  double lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
  if (family == PK_GEN_POISSON2D || family == PK_GEN_POISSON3D) {
    double dv = nd == 2 ? 4.0 : 12.0, ov = nd == 2 ? -1.0 : -2.0;
    if (ncoef >= 2) { dv = coef[0]; ov = coef[1]; }
    diag = dv;
    for (int d = 0; d < nd; ++d) lo[d] = hi[d] = ov;
  } else {
    if (nd == 2 && dims[0] != dims[1]) return fail(PK_ERR_INVALID, "convection-diffusion grids are square");
    if (nd == 3 && (dims[0] != dims[1] || dims[1] != dims[2]))
      return fail(PK_ERR_INVALID, "convection-diffusion grids are cubic");
    double cvel[3] = {1.0, 1.0, 1.0};
    for (int d = 0; d < nd && d < ncoef; ++d) cvel[d] = coef[d];
    volatile double h = 1.0 / (double)(dims[0] + 1);
    // same expression trees as oracle.convdiff{2,3}d, no contraction
    volatile double csum = nd == 2 ? cvel[0] + cvel[1] : (cvel[0] + cvel[1]) + cvel[2];
    volatile double hc = h * csum;
    diag = (nd == 2 ? 4.0 : 6.0) + hc;
    for (int d = 0; d < nd; ++d) {
      volatile double t = h * cvel[d];
      lo[d] = -1.0 - t;
      hi[d] = -1.0;
    }
  }
  // entries sorted by column offset: -stride[nd-1] ... +stride[nd-1]
  int e = 0;
  for (int d = nd - 1; d >= 0; --d) { sp.off[e] = -sp.stride[d]; sp.axis[e] = d; sp.step[e] = -1; sp.val[e] = lo[d]; ++e; }
  sp.off[e] = 0; sp.axis[e] = -1; sp.step[e] = 0; sp.val[e] = diag; ++e;
  for (int d = 0; d < nd; ++d) { sp.off[e] = sp.stride[d]; sp.axis[e] = d; sp.step[e] = 1; sp.val[e] = hi[d]; ++e; }
  sp.nent = e;

  PK_TRY(set_device(c->device));
  cudaStream_t s = c->stream;
  int64_t* counts = nullptr;
  int64_t* incl = nullptr;
  int64_t nblk = (n + 1023) / 1024;
  int64_t* bsum = nullptr;
  int64_t* bsum_incl = nullptr;
  unsigned long long* dmax = nullptr;
  PK_CUDA(cudaMalloc(&counts, n * 8));
  PK_CUDA(cudaMalloc(&incl, n * 8));
  PK_CUDA(cudaMalloc(&bsum, nblk * 8));
  PK_CUDA(cudaMalloc(&bsum_incl, nblk * 8));
  PK_CUDA(cudaMalloc(&dmax, 8));
  PK_CUDA(cudaMemsetAsync(dmax, 0, 8, s));
  int g = grid_elem(c, n, 256);
  k_gen_count<<<g, 256, 0, s>>>(n, sp, counts);
  k_row_max<<<std::min(g, c->sm_count * 2), 256, 0, s>>>(counts, n, dmax);
  k_scan_block<<<(unsigned)nblk, 1024, 0, s>>>(counts, incl, n, bsum);
  // scan block sums on the host (nblk <= 2M)
  std::vector<int64_t> hb((size_t)nblk);
  PK_CUDA(cudaMemcpyAsync(hb.data(), bsum, nblk * 8, cudaMemcpyDeviceToHost, s));
  unsigned long long hmax = 0;
  PK_CUDA(cudaMemcpyAsync(&hmax, dmax, 8, cudaMemcpyDeviceToHost, s));
  PK_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 1; i < nblk; ++i) hb[i] += hb[i - 1];
  int64_t nnz = nblk ? hb[nblk - 1] : 0;
  PK_CUDA(cudaMemcpyAsync(bsum_incl, hb.data(), nblk * 8, cudaMemcpyHostToDevice, s));
  k_scan_add<<<(unsigned)nblk, 1024, 0, s>>>(incl, n, bsum_incl);
  pk_mat* m = nullptr;
  int rc = alloc_mat(c, n, ncols, nnz, &m);
  if (rc == PK_OK) {
    m->max_row = (int64_t)hmax;
    if (m->row64) {
      k_rowptr_from_incl<int64_t><<<g, 256, 0, s>>>(incl, n, (int64_t*)m->rowptr);
      k_gen_fill<int64_t><<<g, 256, 0, s>>>(n, sp, (const int64_t*)m->rowptr, m->cols, m->vals);
    } else {
      k_rowptr_from_incl<int32_t><<<g, 256, 0, s>>>(incl, n, (int32_t*)m->rowptr);
      k_gen_fill<int32_t><<<g, 256, 0, s>>>(n, sp, (const int32_t*)m->rowptr, m->cols, m->vals);
    }
  }
  cudaError_t ce = cudaStreamSynchronize(s);
  cudaFree(counts);
  cudaFree(incl);
  cudaFree(bsum);
  cudaFree(bsum_incl);
  cudaFree(dmax);
  if (rc != PK_OK) return rc;
  if (ce != cudaSuccess) {
    pk_mat_destroy(m);
    return fail(PK_ERR_CUDA, std::string("generator: ") + cudaGetErrorString(ce));
  }
  int rcf = apply_default_format(c, m);
  if (rcf != PK_OK && rcf != PK_ERR_UNSUPPORTED) {
    pk_mat_destroy(m);
    return rcf;
  }
  *out = m;
  return PK_OK;
}

extern "C" int pk_csr_info(const pk_mat* m, int64_t* n_rows, int64_t* n_cols, int64_t* nnz, int64_t* max_row) {
  if (!m) return fail(PK_ERR_INVALID, "mat is NULL");
  if (n_rows) *n_rows = m->n_rows;
  if (n_cols) *n_cols = m->n_cols;
  if (nnz) *nnz = m->nnz;
  if (max_row) *max_row = m->max_row;
  return PK_OK;
}

extern "C" int pk_csr_download(pk_ctx* c, const pk_mat* m, int64_t* offs, int64_t* cols, double* vals) {
  if (!c || !m) return fail(PK_ERR_INVALID, "NULL argument");
  PK_TRY(set_device(m->device));
  if (offs) {
    if (m->row64) {
      PK_CUDA(cudaMemcpy(offs, m->rowptr, (size_t)(m->n_rows + 1) * 8, cudaMemcpyDeviceToHost));
    } else {
      std::vector<int32_t> r((size_t)m->n_rows + 1);
      PK_CUDA(cudaMemcpy(r.data(), m->rowptr, r.size() * 4, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < r.size(); ++i) offs[i] = r[i];
    }
  }
  if (cols && m->nnz) {
    std::vector<int32_t> cc((size_t)m->nnz);
    PK_CUDA(cudaMemcpy(cc.data(), m->cols, cc.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < cc.size(); ++i) cols[i] = cc[i];
  }
  if (vals && m->nnz) PK_CUDA(cudaMemcpy(vals, m->vals, (size_t)m->nnz * 8, cudaMemcpyDeviceToHost));
  return PK_OK;
}

// ---- SELL-32 layout ---------------------------------------------------------

// width (longest row) of every 32-row slice, times 32 = the slice's padded entries
template <typename RowT>
__global__ void k_sell_width(int64_t n, const RowT* __restrict__ rp, int64_t* __restrict__ slice_entries) {
  const int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // blockDim multiple of 32
  const int64_t len = row < n ? (int64_t)(rp[row + 1] - rp[row]) : 0;
  unsigned long long w = (unsigned long long)len;
  for (int o = 16; o >= 1; o >>= 1) w = max(w, __shfl_xor_sync(0xffffffffu, w, o));
  if ((threadIdx.x & 31) == 0 && row < n) slice_entries[row >> 5] = (int64_t)w * 32;
}

template <typename RowT>
__global__ void k_sell_ptr(int64_t nsl, const int64_t* __restrict__ incl, RowT* __restrict__ sp) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nsl; i += (int64_t)gridDim.x * blockDim.x)
    sp[i] = (RowT)(i == 0 ? 0 : incl[i - 1]);
}

// thread per row: slot j of row 32 s + l -> sp[s] + 32 j + l (coalesced stores)
template <typename RowT>
__global__ void k_sell_fill(int64_t n, const RowT* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ va, const RowT* __restrict__ sp, int32_t* __restrict__ sc,
                            double* __restrict__ sv) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    const RowT b = rp[row], len = rp[row + 1] - b;
    const RowT s0 = sp[row >> 5], w = (sp[(row >> 5) + 1] - s0) >> 5;
    const RowT base = s0 + (RowT)(row & 31);
    for (RowT j = 0; j < w; ++j) {
      sc[base + 32 * j] = j < len ? ci[b + j] : -1;
      sv[base + 32 * j] = j < len ? va[b + j] : 0.0;
    }
  }
}

static void free_sell(pk_mat* m) {
  if (m->sell_ptr) cudaFree(m->sell_ptr);
  if (m->sell_cols) cudaFree(m->sell_cols);
  if (m->sell_vals) cudaFree(m->sell_vals);
  m->sell_ptr = nullptr;
  m->sell_cols = nullptr;
  m->sell_vals = nullptr;
  m->sell = false;
  m->sell_nnz = 0;
}

template <typename RowT>
static int build_sell_t(pk_ctx* c, pk_mat* m) {
  cudaStream_t s = c->stream;
  const int64_t n = m->n_rows, nsl = (n + 31) / 32;
  const RowT* rp = (const RowT*)m->rowptr;
  int64_t *ent = nullptr, *incl = nullptr, *bsum = nullptr, *bsum_incl = nullptr;
  const int64_t nblk = (nsl + 1023) / 1024;
  PK_CUDA(cudaMalloc(&ent, std::max<int64_t>(nsl, 1) * 8));
  PK_CUDA(cudaMalloc(&incl, std::max<int64_t>(nsl, 1) * 8));
  PK_CUDA(cudaMalloc(&bsum, std::max<int64_t>(nblk, 1) * 8));
  PK_CUDA(cudaMalloc(&bsum_incl, std::max<int64_t>(nblk, 1) * 8));
  k_sell_width<RowT><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(n, rp, ent);
  k_scan_block<<<(unsigned)nblk, 1024, 0, s>>>(ent, incl, nsl, bsum);
  std::vector<int64_t> hb((size_t)nblk);
  PK_CUDA(cudaMemcpyAsync(hb.data(), bsum, nblk * 8, cudaMemcpyDeviceToHost, s));
  PK_CUDA(cudaStreamSynchronize(s));
  for (int64_t i = 1; i < nblk; ++i) hb[i] += hb[i - 1];
  const int64_t total = nblk ? hb[nblk - 1] : 0;
  int rc = PK_OK;
  if (!m->row64 && total >= (1ll << 31) - 1) rc = fail(PK_ERR_UNSUPPORTED, "padded SELL-32 entries overflow int32");
  if (rc == PK_OK) {
    PK_CUDA(cudaMemcpyAsync(bsum_incl, hb.data(), nblk * 8, cudaMemcpyHostToDevice, s));
    k_scan_add<<<(unsigned)nblk, 1024, 0, s>>>(incl, nsl, bsum_incl);
    cudaError_t e = cudaMalloc(&m->sell_ptr, (size_t)(nsl + 1) * sizeof(RowT) + 64);
    if (e == cudaSuccess) e = cudaMalloc(&m->sell_cols, (size_t)total * 4 + 64);
    if (e == cudaSuccess) e = cudaMalloc(&m->sell_vals, (size_t)total * 8 + 64);
    if (e != cudaSuccess) {
      rc = fail(e == cudaErrorMemoryAllocation ? PK_ERR_NOMEM : PK_ERR_CUDA,
                std::string("SELL-32 allocation: ") + cudaGetErrorString(e));
    } else {
      const int g = grid_elem(c, nsl + 1, 256);
      k_sell_ptr<RowT><<<g, 256, 0, s>>>(nsl, incl, (RowT*)m->sell_ptr);
      k_sell_fill<RowT><<<grid_elem(c, n, 256), 256, 0, s>>>(n, rp, m->cols, m->vals, (const RowT*)m->sell_ptr,
                                                             m->sell_cols, m->sell_vals);
      e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) rc = fail(PK_ERR_CUDA, std::string("SELL-32 build: ") + cudaGetErrorString(e));
    }
  }
  cudaStreamSynchronize(s);
  cudaFree(ent);
  cudaFree(incl);
  cudaFree(bsum);
  cudaFree(bsum_incl);
  if (rc != PK_OK) {
    free_sell(m);
    return rc;
  }
  m->sell_nnz = total;
  m->sell = true;
  return PK_OK;
}

extern "C" int pk_mat_set_format(pk_ctx* c, pk_mat* m, int32_t format) {
  if (!c || !m) return fail(PK_ERR_INVALID, "NULL argument");
  if (format != PK_FMT_CSR && format != PK_FMT_SELL32) return fail(PK_ERR_INVALID, "unknown matrix format");
  PK_TRY(set_device(m->device));
  // a format change gives the matrix a new identity: cached solver
  // workspaces (keyed by it) hold graphs that walk the old arrays
  if (format == PK_FMT_CSR) {
    if (m->sell) {
      PK_CUDA(cudaStreamSynchronize(c->stream));
      free_sell(m);
      m->uid = g_mat_uid.fetch_add(1);
    }
    return PK_OK;
  }
  if (m->sell || m->n_rows == 0) return PK_OK;
  if (m->row64) return fail(PK_ERR_UNSUPPORTED, "SELL-32 needs nnz < 2^31 (32-bit offsets)");
  PK_TRY(build_sell_t<int32_t>(c, m));
  m->uid = g_mat_uid.fetch_add(1);
  return PK_OK;
}

extern "C" int pk_mat_get_format(const pk_mat* m, int32_t* format, int64_t* stored_entries) {
  if (!m || !format) return fail(PK_ERR_INVALID, "NULL argument");
  *format = m->sell ? PK_FMT_SELL32 : PK_FMT_CSR;
  if (stored_entries) *stored_entries = m->sell ? m->sell_nnz : m->nnz;
  return PK_OK;
}

// the context's default format for new matrices (PK_SELL env, see pk_ctx)
// most entries in an aligned 32-row block [32 b, 32 b + 32) -- a BULK engine
// chunk (pk_bulk.cuh); atomicMax over the blocks
template <typename RowT>
__global__ void k_blk_max(int64_t n, const RowT* __restrict__ rp, unsigned long long* mx) {
  const int64_t nb = (n + 31) / 32;
  unsigned long long m = 0;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = (b + 1) * 32 < n ? (b + 1) * 32 : n;
    const unsigned long long d = (unsigned long long)(rp[e] - rp[b * 32]);
    m = d > m ? d : m;
  }
  if (m) atomicMax(mx, m);
}

static int compute_blk_max(pk_ctx* c, pk_mat* m) {
  if (m->n_rows == 0) {
    m->blk_max = 0;
    return PK_OK;
  }
  unsigned long long* d = nullptr;
  PK_CUDA(cudaMalloc(&d, 8));
  cudaError_t e = cudaMemsetAsync(d, 0, 8, c->stream);
  const int64_t nb = (m->n_rows + 31) / 32;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((nb + 255) / 256, (int64_t)c->sm_count * 8));
  if (e == cudaSuccess) {
    if (m->row64) k_blk_max<int64_t><<<g, 256, 0, c->stream>>>(m->n_rows, (const int64_t*)m->rowptr, d);
    else k_blk_max<int32_t><<<g, 256, 0, c->stream>>>(m->n_rows, (const int32_t*)m->rowptr, d);
    e = cudaGetLastError();
  }
  unsigned long long h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(PK_ERR_CUDA, std::string("block scan: ") + cudaGetErrorString(e));
  m->blk_max = (int64_t)h;
  return PK_OK;
}

static int apply_default_format(pk_ctx* c, pk_mat* m) {
  PK_TRY(compute_blk_max(c, m));
  m->vec_rows = c->vec_min_avg > 0 && !m->row64 && m->n_rows > 0 && m->nnz >= (int64_t)c->vec_min_avg * m->n_rows;
  if (m->vec_rows) return PK_OK;  // long rows: CSR + VEC pre-pass rather than SELL-32
  const bool want = c->sell_mode == 1 ||
                    (c->sell_mode == 2 && m->n_rows >= (int64_t(1) << 19) && m->nnz >= 12 * m->n_rows && !m->row64);
  return want ? pk_mat_set_format(c, m, PK_FMT_SELL32) : PK_OK;
}

extern "C" int pk_mat_destroy(pk_mat* m) {
  if (!m) return PK_OK;
  cudaSetDevice(m->device);
  free_sell(m);
  if (m->rowptr) cudaFree(m->rowptr);
  if (m->cols) cudaFree(m->cols);
  if (m->vals) cudaFree(m->vals);
  delete m;
  return PK_OK;
}

// ---------------------------------------------------------------------------
// kernel-level entries
// ---------------------------------------------------------------------------

#define PK_CHECK_CTX(c) \
  do { if (!(c)) return fail(PK_ERR_INVALID, "ctx is NULL"); PK_TRY(set_device((c)->device)); } while (0)

extern "C" int pk_spmv(pk_ctx* c, const pk_mat* a, const double* p, double* q) {
  PK_CHECK_CTX(c);
  if (!a || (!p && a->n_cols) || (!q && a->n_rows)) return fail(PK_ERR_INVALID, "NULL argument");
  if (a->n_rows == 0) return PK_OK;
  PK_TRY(ensure_vec(c, a));
  return spmv_fused_any(c, c->stream, a, p, q, 0, nullptr, nullptr, nullptr, 0, 0);
}

// ELLPACK SpMV (_spmvkernels.py:21-34): thread per row; slot k of the 32
// rows of a warp is 32 consecutive words (coalesced, no L1 reuse needed);
// EU slots' loads issued before their ordered adds; padded slots skipped.
__global__ void __launch_bounds__(256) k_spmv_ell(int64_t n, int64_t n_cols, int64_t width,
                                                  const int32_t* __restrict__ cols,
                                                  const double* __restrict__ vals, const double* __restrict__ p,
                                                  double* __restrict__ q) {
  constexpr int EU = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double acc = 0.0;
    int64_t k = 0;
    for (; k + EU <= width; k += EU) {
      int32_t c[EU];
      double v[EU], x[EU];
#pragma unroll
      for (int u = 0; u < EU; ++u) {
        c[u] = __ldg(cols + (k + u) * n + i);
        v[u] = __ldg(vals + (k + u) * n + i);
      }
#pragma unroll
      for (int u = 0; u < EU; ++u) x[u] = c[u] < n_cols ? __ldg(p + c[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < EU; ++u)
        if (c[u] < n_cols) acc = add_rn(acc, mul_rn(v[u], x[u]));
    }
    for (; k < width; ++k) {
      const int32_t c = __ldg(cols + k * n + i);
      if (c < n_cols) acc = add_rn(acc, mul_rn(__ldg(vals + k * n + i), __ldg(p + c)));
    }
    q[i] = acc;
  }
}

extern "C" int pk_ell_upload(pk_ctx* c, int64_t n_rows, int64_t n_cols, int64_t width, const int64_t* cols,
                             const double* vals, pk_ell** out) {
  if (!c || !out) return fail(PK_ERR_INVALID, "NULL argument");
  *out = nullptr;
  if (n_rows < 0 || n_cols < 0 || width < 0) return fail(PK_ERR_INVALID, "matrix dimensions must be non-negative");
  if (n_rows >= (1ll << 31) - 1 || n_cols >= (1ll << 31) - 1)
    return fail(PK_ERR_UNSUPPORTED, "device path indexes rows and columns with int32");
  const int64_t total = n_rows * width;
  if (total && (!cols || !vals)) return fail(PK_ERR_INVALID, "NULL argument");
  std::vector<int32_t> c32((size_t)total);
  for (int64_t t = 0; t < total; ++t) {
    if (cols[t] < 0 || cols[t] > n_cols) return fail(PK_ERR_INVALID, "column index out of range");
    if (cols[t] == n_cols && vals[t] != 0.0) return fail(PK_ERR_INVALID, "padded slots must store value 0");
    c32[(size_t)t] = (int32_t)cols[t];
  }
  PK_TRY(set_device(c->device));
  pk_ell* e = new pk_ell();
  e->device = c->device;
  e->n_rows = n_rows;
  e->n_cols = n_cols;
  e->width = width;
  cudaError_t err = cudaSuccess;
  if (total) {
    err = cudaMalloc(&e->cols, (size_t)total * sizeof(int32_t));
    if (err == cudaSuccess) err = cudaMalloc(&e->vals, (size_t)total * sizeof(double));
    if (err == cudaSuccess) err = cudaMemcpy(e->cols, c32.data(), (size_t)total * sizeof(int32_t), cudaMemcpyHostToDevice);
    if (err == cudaSuccess) err = cudaMemcpy(e->vals, vals, (size_t)total * sizeof(double), cudaMemcpyHostToDevice);
  }
  if (err != cudaSuccess) {
    pk_ell_destroy(e);
    return fail(PK_ERR_CUDA, std::string("ELL upload: ") + cudaGetErrorString(err));
  }
  *out = e;
  return PK_OK;
}

extern "C" int pk_ell_destroy(pk_ell* e) {
  if (!e) return PK_OK;
  cudaSetDevice(e->device);
  if (e->cols) cudaFree(e->cols);
  if (e->vals) cudaFree(e->vals);
  delete e;
  return PK_OK;
}

extern "C" int pk_spmv_ell(pk_ctx* c, const pk_ell* a, const double* p, double* q) {
  PK_CHECK_CTX(c);
  if (!a || (!p && a->n_cols) || (!q && a->n_rows)) return fail(PK_ERR_INVALID, "NULL argument");
  if (a->n_rows == 0) return PK_OK;
  k_spmv_ell<<<grid_elem(c, a->n_rows, 256), 256, 0, c->stream>>>(a->n_rows, a->n_cols, a->width, a->cols, a->vals,
                                                                  p, q);
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

extern "C" int pk_spmv_fused(pk_ctx* c, const pk_mat* a, const double* p, double* q, int32_t nq,
                             const int32_t* kinds, const double* const* w, double* partials) {
  PK_CHECK_CTX(c);
  if (!a || !kinds || !partials) return fail(PK_ERR_INVALID, "NULL argument");
  if (nq < 1 || nq > 4) return fail(PK_ERR_INVALID, "request must carry 1 to 4 quantities, got " + std::to_string(nq));
  for (int k = 0; k < nq; ++k) {
    if (kinds[k] < 0 || kinds[k] > 2) return fail(PK_ERR_INVALID, "unknown quantity kind");
    if (kinds[k] == PK_DOT_INPUT && a->n_rows != a->n_cols)
      return fail(PK_ERR_INVALID, "result-with-input dot needs a square matrix");
    if (kinds[k] == PK_DOT_VECTOR && (!w || !w[k])) return fail(PK_ERR_INVALID, "missing fixed dot vector");
  }
  PK_TRY(ensure_scratch(c, a->n_rows, nq));
  PK_TRY(ensure_vec(c, a));
  return spmv_fused_any(c, c->stream, a, p, q, nq, kinds, w, partials, nq, 0);
}

extern "C" int pk_reduce_stage1(pk_ctx* c, int64_t n, int32_t nq, const double* const* columns, double* partials) {
  PK_CHECK_CTX(c);
  if (!columns || !partials || n < 0) return fail(PK_ERR_INVALID, "bad argument");
  PK_TRY(ensure_scratch(c, n, 4));
  // one launch per block of up to 4 columns (stacking never reorders, test_linalg.py:198-207)
  for (int q0 = 0; q0 < nq; q0 += 4) {
    int k = std::min(4, nq - q0);
    int rc;
    switch (k) {
      case 1: { OpColumns<1> op{}; op.col[0] = columns[q0]; rc = launch_reduce<1>(c, c->stream, n, op, ScalarPtrs{}, partials, nq, q0); break; }
      case 2: { OpColumns<2> op{}; for (int j = 0; j < 2; ++j) op.col[j] = columns[q0 + j]; rc = launch_reduce<2>(c, c->stream, n, op, ScalarPtrs{}, partials, nq, q0); break; }
      case 3: { OpColumns<3> op{}; for (int j = 0; j < 3; ++j) op.col[j] = columns[q0 + j]; rc = launch_reduce<3>(c, c->stream, n, op, ScalarPtrs{}, partials, nq, q0); break; }
      default: { OpColumns<4> op{}; for (int j = 0; j < 4; ++j) op.col[j] = columns[q0 + j]; rc = launch_reduce<4>(c, c->stream, n, op, ScalarPtrs{}, partials, nq, q0); break; }
    }
    PK_TRY(rc);
  }
  return PK_OK;
}

extern "C" int pk_reduce_stage2(pk_ctx* c, int32_t nq, const double* partials, double* totals) {
  PK_CHECK_CTX(c);
  if (!partials || !totals || nq < 0) return fail(PK_ERR_INVALID, "bad argument");
  if (nq == 0) return PK_OK;
  k_stage2<<<1, 32, 0, c->stream>>>(partials, c->ng, nq, nq, totals);
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

// Classical-driver BLAS-1 updates (linalg.py:403-457): one grid-stride
// elementwise kernel, V elements per thread in flight, the NumPy expression
// order with explicit round-to-nearest operations.
template <int KIND>
__global__ void __launch_bounds__(256) k_vec_update(int64_t n, double* __restrict__ y, const double* __restrict__ x,
                                                    const double* __restrict__ z, double alpha, double beta) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double out;
    if constexpr (KIND == PK_VEC_AXPY) out = add_rn(y[i], mul_rn(alpha, x[i]));
    else if constexpr (KIND == PK_VEC_AXPY2) out = add_rn(y[i], add_rn(mul_rn(alpha, x[i]), mul_rn(beta, z[i])));
    else if constexpr (KIND == PK_VEC_XPAY) out = add_rn(mul_rn(y[i], beta), x[i]);
    else if constexpr (KIND == PK_VEC_SCALE) out = mul_rn(y[i], alpha);
    else if constexpr (KIND == PK_VEC_ADD_SCALED) out = add_rn(x[i], mul_rn(alpha, z[i]));
    else if constexpr (KIND == PK_VEC_BICG_P) out = add_rn(mul_rn(sub_rn(y[i], mul_rn(beta, z[i])), alpha), x[i]);
    else out = x[i];
    y[i] = out;
  }
}

extern "C" int pk_vec_update(pk_ctx* c, int32_t kind, int64_t n, double* y, const double* x, const double* z,
                             double alpha, double beta) {
  PK_CHECK_CTX(c);
  if (n < 0 || (n > 0 && !y)) return fail(PK_ERR_INVALID, "bad argument");
  const bool need_x = kind == PK_VEC_AXPY || kind == PK_VEC_AXPY2 || kind == PK_VEC_XPAY ||
                      kind == PK_VEC_ADD_SCALED || kind == PK_VEC_BICG_P || kind == PK_VEC_COPY;
  const bool need_z = kind == PK_VEC_AXPY2 || kind == PK_VEC_ADD_SCALED || kind == PK_VEC_BICG_P;
  if (kind < PK_VEC_AXPY || kind > PK_VEC_COPY) return fail(PK_ERR_INVALID, "unknown vector update kind");
  if (n > 0 && ((need_x && !x) || (need_z && !z))) return fail(PK_ERR_INVALID, "missing vector argument");
  if (n == 0) return PK_OK;
  const dim3 grid((unsigned)grid_elem(c, n, 256)), block(256);
  cudaStream_t s = c->stream;
  switch (kind) {
    case PK_VEC_AXPY: k_vec_update<PK_VEC_AXPY><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
    case PK_VEC_AXPY2: k_vec_update<PK_VEC_AXPY2><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
    case PK_VEC_XPAY: k_vec_update<PK_VEC_XPAY><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
    case PK_VEC_SCALE: k_vec_update<PK_VEC_SCALE><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
    case PK_VEC_ADD_SCALED: k_vec_update<PK_VEC_ADD_SCALED><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
    case PK_VEC_BICG_P: k_vec_update<PK_VEC_BICG_P><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
    default: k_vec_update<PK_VEC_COPY><<<grid, block, 0, s>>>(n, y, x, z, alpha, beta); break;
  }
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}

extern "C" int pk_dot(pk_ctx* c, int64_t n, const double* x, const double* y, double* total) {
  PK_CHECK_CTX(c);
  if (!total || n < 0) return fail(PK_ERR_INVALID, "bad argument");
  PK_TRY(ensure_scratch(c, n, 1));
  double* part = nullptr;
  PK_CUDA(cudaMallocAsync(&part, (size_t)c->ng * 8, c->stream));
  int rc = dot_partials(c, c->stream, n, x, y, part);
  if (rc == PK_OK) {
    k_stage2<<<1, 32, 0, c->stream>>>(part, c->ng, 1, 1, total);
    if (cudaGetLastError() != cudaSuccess) rc = fail(PK_ERR_CUDA, "stage2 launch failed");
  }
  cudaFreeAsync(part, c->stream);
  return rc;
}

extern "C" int pk_cg_update(pk_ctx* c, int64_t n, double* x, double* r, double* p, const double* ap, double alpha,
                            double beta, double* partials) {
  PK_CHECK_CTX(c);
  if (!partials || n < 0) return fail(PK_ERR_INVALID, "bad argument");
  PK_TRY(ensure_scratch(c, n, 1));
  OpCgUpdate op{x, r, p, ap, alpha, beta};
  return launch_reduce<1>(c, c->stream, n, op, ScalarPtrs{}, partials, 1, 0);
}

extern "C" int pk_bicg_s_update(pk_ctx* c, int64_t n, const double* r, const double* ap, const double* rr0p,
                                const double* aprp, double btol, double* s, double* partials, double* alpha_out,
                                int32_t* breakdown) {
  PK_CHECK_CTX(c);
  if (!rr0p || !aprp || !partials || !alpha_out || !breakdown) return fail(PK_ERR_INVALID, "NULL argument");
  PK_TRY(ensure_scratch(c, n, 1));
  k_bicg_alpha<<<1, 32, 0, c->stream>>>(rr0p, aprp, c->ng, btol, alpha_out, breakdown);
  PK_CUDA(cudaGetLastError());
  OpBicgS op{r, ap, s, 0.0};
  ScalarPtrs sp{alpha_out, nullptr, nullptr, nullptr};
  return launch_reduce<1>(c, c->stream, n, op, sp, partials, 1, 0, nullptr, GATE_NONE, breakdown);
}

extern "C" int pk_bicg_xrp_update(pk_ctx* c, int64_t n, double* x, double* r, double* p, const double* s,
                                  const double* ap, const double* as, double alpha, double omega, double beta,
                                  const double* r0star, double* partials) {
  PK_CHECK_CTX(c);
  if (!partials || n < 0) return fail(PK_ERR_INVALID, "bad argument");
  PK_TRY(ensure_scratch(c, n, 1));
  OpBicgXrp op{x, r, p, s, ap, as, r0star, alpha, omega, beta};
  return launch_reduce<1>(c, c->stream, n, op, ScalarPtrs{}, partials, 1, 0);
}

extern "C" int pk_gs_stage1(pk_ctx* c, int64_t n, int32_t nb, const double* const* basis, const double* v,
                            double* partials) {
  PK_CHECK_CTX(c);
  if (nb < 0 || (nb > 0 && (!basis || !partials))) return fail(PK_ERR_INVALID, "bad argument");
  if (nb == 0) return PK_OK;
  PK_TRY(ensure_scratch(c, n, multidot_nb_cap(c, n)));  // padded NB <= cap
  return multidot_any(c, c->stream, n, nb, basis, v, partials, nb, 0);
}

extern "C" int pk_gs_update(pk_ctx* c, int64_t n, double* v, int32_t nb, const double* const* basis,
                            const double* partials, double* coeffs, double* norm_partials) {
  PK_CHECK_CTX(c);
  if (nb < 0 || !norm_partials || (nb > 0 && (!basis || !partials || !coeffs)))
    return fail(PK_ERR_INVALID, "bad argument");
  PK_TRY(ensure_scratch(c, n, 1));
  if (nb > 0) {
    k_stage2<<<1, 32, 0, c->stream>>>(partials, c->ng, nb, nb, coeffs);
    PK_CUDA(cudaGetLastError());
  }
  double* acc = nullptr;
  if (nb > c->gs_chunk) PK_CUDA(cudaMallocAsync(&acc, (size_t)std::max<int64_t>(n, 1) * 8, c->stream));
  int rc = gs_update_any(c, c->stream, n, v, nb, basis, coeffs, norm_partials, nullptr, GATE_NONE, FIN_NONE, 0, acc);
  if (acc) cudaFreeAsync(acc, c->stream);
  return rc;
}

extern "C" int pk_gs_normalize(pk_ctx* c, int64_t n, double* v, const double* norm_partials, const double* r,
                               double btol, double* norm_out, int32_t* lucky, double* partials) {
  PK_CHECK_CTX(c);
  if (!norm_partials || !norm_out || !lucky || !partials) return fail(PK_ERR_INVALID, "NULL argument");
  double* inv = c->scratch_d;
  PK_TRY(ensure_scratch(c, n, 1));
  k_norm_fin<<<1, 32, 0, c->stream>>>(norm_partials, c->ng, btol, norm_out, inv, lucky);
  PK_CUDA(cudaGetLastError());
  OpNormalize op{v, r, 0.0};
  ScalarPtrs sp{inv, nullptr, nullptr, nullptr};
  return launch_reduce<1>(c, c->stream, n, op, sp, partials, 1, 0, nullptr, GATE_NONE, lucky);
}

#include "pk_solvers.inc"
#include "pk_dist.inc"

// ---------------------------------------------------------------------------
// engine experiments (not part of the public header): simple reference
// kernels timed on the device, to bound what the staged engine should reach
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(256) k_dbg_spmv_simple(int64_t n, const int32_t* __restrict__ rp,
                                                         const int32_t* __restrict__ ci,
                                                         const double* __restrict__ va,
                                                         const double* __restrict__ p, double* __restrict__ q) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n; row += (int64_t)gridDim.x * blockDim.x) {
    int b = __ldg(rp + row), e = __ldg(rp + row + 1);
    double acc = 0.0;
    for (int k = b; k < e; ++k) acc = add_rn(acc, mul_rn(__ldg(va + k), __ldg(p + __ldg(ci + k))));
    q[row] = acc;
  }
}

// K_B-shaped: s = r - a Ap recomputed at every gathered column; As and four
// contribution streams written out (no ordered reduction)
__global__ void __launch_bounds__(256) k_dbg_bicgb_simple(int64_t n, const int32_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci,
                                                          const double* __restrict__ va,
                                                          const double* __restrict__ r,
                                                          const double* __restrict__ ap,
                                                          const double* __restrict__ r0, double alpha,
                                                          double* __restrict__ as, double* __restrict__ cc) {
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n; row += (int64_t)gridDim.x * blockDim.x) {
    int b = __ldg(rp + row), e = __ldg(rp + row + 1);
    double acc = 0.0;
    for (int k = b; k < e; ++k) {
      uint32_t c = (uint32_t)__ldg(ci + k);
      acc = add_rn(acc, mul_rn(__ldg(va + k), sub_rn(__ldg(r + c), mul_rn(alpha, __ldg(ap + c)))));
    }
    double s = sub_rn(__ldg(r + row), mul_rn(alpha, __ldg(ap + row)));
    as[row] = acc;
    cc[row] = mul_rn(s, s) + mul_rn(acc, s) + mul_rn(acc, acc) + mul_rn(acc, __ldg(r0 + row));
  }
}

// engine row order (CHAIN units x chunk batches, U rows per thread) with the
// ordered fold removed: contributions are only summed per thread
template <int NQ, int U, class Op, bool kCopy = false>
__global__ void __launch_bounds__(256, 4) k_dbg_order(Geom geo, const __grid_constant__ Op op0, double* sink) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  Op opl = op0;
  if (kCopy) opl.scalars(ScalarPtrs{});
  const Op& op = kCopy ? opl : op0;
  constexpr int B = kWarps * U;
  double keep = 0.0;
  for (int64_t unit = blockIdx.x; unit < geo.units; unit += gridDim.x) {
    const int64_t lid0 = unit * 32;
    for (int64_t k0 = 0; k0 < geo.K; k0 += B) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t row = (k0 + warp + kWarps * u) * geo.G + lid0 + lane;
        double c[NQ];
        if (k0 + warp + kWarps * u < geo.K && row < geo.n) {
          row_contrib<NQ>(op, (uint32_t)row, c);
#pragma unroll
          for (int q = 0; q < NQ; ++q) keep = add_rn(keep, c[q]);
        }
      }
    }
  }
  if (keep == 12345.678) sink[0] = keep;
}

// the same operator on a plain grid-stride thread-per-row loop
template <int NQ, class Op>
__global__ void __launch_bounds__(256, 4) k_dbg_gridstride(int64_t n, Op op, double* sink) {
  double keep = 0.0;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n; row += (int64_t)gridDim.x * blockDim.x) {
    double c[NQ];
    row_contrib<NQ>(op, (uint32_t)row, c);
    keep = add_rn(keep, c[0]);
  }
  if (keep == 12345.678) sink[0] = keep;
}

extern "C" int pk_debug_bench(pk_ctx* c, const pk_mat* a, int kind, int reps, double* us_out) {
  PK_CHECK_CTX(c);
  if (!a || a->row64 || !us_out) return fail(PK_ERR_INVALID, "bad argument");
  const int64_t n = a->n_rows;
  double* buf = nullptr;
  PK_CUDA(cudaMalloc(&buf, (size_t)n * 8 * 6 + 64));
  cudaMemset(buf, 0, (size_t)n * 8 * 6);
  double *p = buf, *q = buf + n, *r = buf + 2 * n, *ap = buf + 3 * n, *r0 = buf + 4 * n, *cc = buf + 5 * n;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8);
  OpBicgB<int32_t, 5> ob{};
  ob.A = csr_of<int32_t>(a);
  ob.r[0] = ob.r[1] = r;
  ob.ap[0] = ob.ap[1] = ap;
  ob.r0 = r0;
  ob.as = q;
  ob.alpha = 0.5;
  ob.rc = r;
  ob.apc = ap;
  Geom geo = make_geom(n, c->ng, c->gs);
  PK_TRY(ensure_scratch(c, n, 4));
  auto run = [&]() {
    if (kind == 0)
      k_dbg_spmv_simple<<<grid, 256, 0, c->stream>>>(n, (const int32_t*)a->rowptr, a->cols, a->vals, p, q);
    else if (kind == 1)
      k_dbg_bicgb_simple<<<grid, 256, 0, c->stream>>>(n, (const int32_t*)a->rowptr, a->cols, a->vals, r, ap, r0, 0.5,
                                                      q, cc);
    else if (kind == 2)
      launch_reduce<4>(c, c->stream, n, ob, ScalarPtrs{}, cc, 4, 0);
    else if (kind == 3)
      k_dbg_order<4, 2><<<(int)std::min<int64_t>(geo.units, (int64_t)c->sm_count * 4), 256, 0, c->stream>>>(geo, ob, cc);
    else if (kind == 4)
      k_dbg_gridstride<4><<<grid, 256, 0, c->stream>>>(n, ob, cc);
    else if (kind == 5)
      k_dbg_order<4, 2><<<(int)geo.units, 256, 0, c->stream>>>(geo, ob, cc);
    else if (kind == 9)
      k_dbg_order<4, 2, OpBicgB<int32_t, 5>, true><<<(int)std::min<int64_t>(geo.units, (int64_t)c->sm_count * 4), 256, 0, c->stream>>>(geo, ob, cc);
    else if (kind >= 6 && kind <= 8) {
      // the engine kernel itself with an explicit grid (kind 6: one CTA per
      // unit; kind 7: 2 units per CTA; kind 8: occupancy-sized grid)
      auto kern = k_reduce<4, 2, 4, OpBicgB<int32_t, 5>>;
      size_t smem = engine_smem_bytes(geo, 4, 2);
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int grid6 = kind == 6 ? (int)geo.units : kind == 7 ? (int)((geo.units + 1) / 2) : engine_grid(c, kern, smem, geo.units);
      if (reps == 0) printf("kind %d grid %d smem %zu\n", kind, grid6, smem);
      kern<<<grid6, kThreads, smem, c->stream>>>(geo, ob, ScalarPtrs{}, cc, 4, 0, 4, scratch_of(c), nullptr, GATE_NONE,
                                                 nullptr, FIN_NONE, 0);
    }
  };
  for (int i = 0; i < 3; ++i) run();
  if (kind >= 6 && kind <= 8) {
    int r0_ = reps;
    reps = 0;
    run();
    reps = r0_;
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_reduce<4, 2, 4, OpBicgB<int32_t, 5>>, kThreads,
                                                  engine_smem_bytes(geo, 4, 2));
    printf("occupancy %d CTAs/SM\n", occ);
  }
  cudaEventRecord(e0, c->stream);
  for (int i = 0; i < reps; ++i) run();
  cudaEventRecord(e1, c->stream);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  *us_out = ms * 1e3 / reps;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  PK_CUDA(cudaGetLastError());
  return PK_OK;
}
