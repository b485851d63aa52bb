// Fused operators and finalizers of the pipelined Krylov path (sm_100a).
//
// Every reduction kernel is "per-row operator + ordered stage 1"
// (pk_reduce.cuh) with an optional finalizer, run by the CTA that completes
// the last group, which performs the serial stage 2 and the host-side scalar
// recurrences of the reference on the device; the next kernel's prologue only
// reads a few scalars (SolveState).
//
// Per-element arithmetic follows the reference exactly:
//   SpMV row        acc = acc + v*x          _spmvkernels.py:12-18
//   CG update       x+a p; r-a Ap; p b + r   fused.py:145-148
//   BiCG s          r - a Ap                 fused.py:177
//   BiCG xrp        x+((a p)+(w s)); s-w As; ((p-w Ap) b)+r   fused.py:212-216
//   GS update       v - sum_j (c_j b_j)      fused.py:268-272
//   GS normalize    v * (1/||v||)            fused.py:300
//
// Recompute-at-gather fusion.  The solver-loop operators OpCgFused, OpBicgA
// and OpBicgB fold a vector update into the SpMV that consumes it: the SpMV
// input at a gathered column is recomputed from the old vectors with the very
// same IEEE operations the update kernel would have used, so the result is
// bit-identical to update-then-SpMV while the updated vector is never
// re-read.  The updated vectors are written to the other half of a
// ping-pong pair selected by SolveState::parity (flipped by the finalizer).
#pragma once

#include <math.h>

#include "pk_reduce.cuh"
#include "pk_state.cuh"

#ifndef PK_S2_SU
#define PK_S2_SU 0  // stage-2 staging: 0 = one load per loop trip; N = N loads per lane in flight
#endif
#ifndef PK_FIN_PREFETCH
#define PK_FIN_PREFETCH 0
#endif

#ifndef PK_BICG_U
#define PK_BICG_U 2  // rows per thread per batch of the BiCGStab SpMV operators (engine batch = 8 U chunks)
#endif
#ifndef PK_BICGB_MINB
#define PK_BICGB_MINB 4
#endif

namespace pk {

// ---------------------------------------------------------------------------
// finalizers (run by one warp: the fold warp of the finalizer CTA, or k_finalize)
// ---------------------------------------------------------------------------

enum Fin : int32_t {
  FIN_NONE = 0,
  FIN_CG_SETUP,    // p_rr, p_two, p_bb -> scale, alpha, beta
  FIN_CG_FUSED,    // p_three [rr, pAp, ApAp] -> history, checks, alpha, beta; parity ^= 1
  FIN_BICG_SETUP,  // p_pair col 0 (<r,r>), p_bb
  FIN_BICG_ALPHA,  // p_pair [rr0, apr] -> alpha; arg: flip parity
  FIN_BICG_TAIL,   // p_quad [ss, ass, asas, asr] -> omega, beta, history, checks
  FIN_BICG_XTAIL,  // after the stand-alone xrp: parity ^= 1, STOPPED
  FIN_GM_RHO,      // cycle setup: rho (and scale on the first cycle)
  FIN_GM_NORM,     // ||w|| -> R diag, 1/||w|| or lucky
  FIN_GM_COEF,     // projections -> coef[], R column
  FIN_GM_XI,       // xi_i, step += 1
  FIN_DOTV,        // dotv = stage2(p_bb)  (true residual; p_bb is free after setup)
};

enum Gate : int32_t {
  GATE_NONE = 0,      // always run
  GATE_RUNNING = 1,   // run while status == RUNNING
  GATE_STOPPING = 2,  // run only when status == STOPPING (BiCGStab tail update)
  GATE_GMRES = 3,     // run while status == RUNNING and not lucky
  GATE_IN_GRAPH = 0x100,  // flag: the launch is a node of the WHILE graph body
                          // (only such kernels may set the graph condition)
};

__device__ __forceinline__ void set_cond(SolveState* st, unsigned v, bool ing) {
  if (ing && st->use_cond) cudaGraphSetConditional(st->cond, v);
}

// Kernel prologues load the gate word(s) and the operator's scalars in ONE
// memory round trip: gate_load() issues the loads, the operator's scalars()
// issues its own, and only then gate_eval() consumes the gate (a branch on
// the gate before the scalar loads would serialise two L2 round trips in
// front of every CTA's first data load).
struct GateVals {
  int32_t status;
  int32_t lucky;
};

__device__ __forceinline__ GateVals gate_load(const SolveState* st, int gate) {
  GateVals g{RUNNING, 0};
  if (gate == GATE_NONE || st == nullptr) return g;
  // L1-cached loads: the state was written by an earlier kernel (L1 is
  // invalidated at every launch), and a per-thread L2 load of one hot line
  // by every warp of the grid serialises in a single L2 slice (~5k requests)
#ifdef PK_OLD_PROLOGUE
  g.status = *(volatile const int32_t*)&st->status;
  if (gate == GATE_GMRES) g.lucky = *(volatile const int32_t*)&st->lucky;
#else
  g.status = __ldg(&st->status);
  if (gate == GATE_GMRES) g.lucky = __ldg(&st->lucky);
#endif
  return g;
}

__device__ __forceinline__ bool gate_eval(SolveState* st, int gate, bool ing, GateVals g) {
  if (gate == GATE_NONE || st == nullptr) return true;
  bool open;
  if (gate == GATE_STOPPING) open = g.status == STOPPING;
  else if (gate == GATE_GMRES) open = (g.status == RUNNING) && !g.lucky;
  else open = (g.status == RUNNING);
  if (!open && gate != GATE_STOPPING && blockIdx.x == 0 && threadIdx.x == 0) set_cond(st, 0, ing);
  return open;
}

__device__ __forceinline__ bool gate_open(SolveState* st, int gate, bool ing) {
  return gate_eval(st, gate, ing, gate_load(st, gate));
}

__device__ __forceinline__ double msqrt(double v) { return __dsqrt_rn(v); }

// CG scalar step (solvers.py:432-465): history, checks, alpha, beta.
__device__ inline void cg_scalars(SolveState* st, double rr, double pap, double apap, bool setup, double bb, bool ing) {
  st->rr = rr; st->pap = pap; st->apap = apap;
  bool stop = false;
  if (setup) {
    double nb = msqrt(bb);
    st->scale = nb > 0.0 ? nb : 1.0;
    double entry = div_rn(msqrt(rr), st->scale);
    if (entry <= st->tol && (!st->fixed || rr == 0.0)) {
      st->term = PK_TERM_CONVERGED; stop = true;
    } else if (fabs(pap) < st->btol_loop || pap == 0.0) {
      st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_PAP; stop = true;
    }
  } else {
    double mon = div_rn(msqrt(rr), st->scale);
    st->hist[st->iter] = mon;
    st->iter += 1;
    if (!isfinite(mon)) {
      st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_DIVERGENCE; stop = true;
    } else if (mon <= st->tol && (!st->fixed || rr == 0.0)) {
      st->term = PK_TERM_CONVERGED; stop = true;
    } else if (fabs(pap) < st->btol_loop || pap == 0.0) {
      st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_PAP; stop = true;
    }
  }
  if (!stop) {
    double a = div_rn(rr, pap);
    st->alpha = a;
    st->beta = sub_rn(div_rn(mul_rn(mul_rn(a, a), apap), rr), 1.0);
    if (!setup && st->iter >= st->limit) { st->term = PK_TERM_MAX_ITER; stop = true; }
  }
  st->status = stop ? STOPPED : RUNNING;
  set_cond(st, stop ? 0u : 1u, ing);
}

// Serial stage 2 (linalg.py:311-320) of NC partial columns, executed by one
// warp: chunks of the partials are staged through shared memory with
// coalesced warp-wide L2 loads, then lane c adds column c in group order
// (the reference's left-to-right chain); every lane receives the totals.
struct S2Col {
  const double* part;
  int ld;
  int col;
};

template <int NC>
__device__ __noinline__ void stage2_warp(const S2Col* cols, int ng, double* out, double* buf, int buf_d) {
  // groups per staged chunk: up to 128 (4 per lane per column), all of a
  // chunk's loads in flight before its shared-memory stores (one L2 round
  // trip per chunk instead of one per element)
  constexpr int UPL = 4;
  int CH = buf_d / NC;
  CH = CH < 32 * UPL ? CH : 32 * UPL;
  const int lane = threadIdx.x & 31;
  const double* cp[NC];
  int cld[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    cp[c] = cols[c].part + cols[c].col;
    cld[c] = cols[c].ld;
  }
  double tot = 0.0;
  for (int g0 = 0; g0 < ng; g0 += CH) {
    const int cnt = (ng - g0) < CH ? (ng - g0) : CH;
    __syncwarp();
    double v[NC][UPL];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int u = 0; u < UPL; ++u) {
        const int g = u * 32 + lane;
        v[c][u] = g < cnt ? __ldcg(cp[c] + (int64_t)(g0 + g) * cld[c]) : 0.0;
      }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int u = 0; u < UPL; ++u) {
        const int g = u * 32 + lane;
        if (g < cnt) buf[c * CH + g] = v[c][u];
      }
    __syncwarp();
    if (lane < NC) {
      const double* b = buf + lane * CH;
      int g = 0;
      for (; g + 8 <= cnt; g += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b[g + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) tot = add_rn(tot, v[u]);
      }
      for (; g < cnt; ++g) tot = add_rn(tot, b[g]);
    }
  }
#pragma unroll
  for (int c = 0; c < NC; ++c) out[c] = __shfl_sync(0xffffffffu, tot, c);
  __syncwarp();
}

// buf / buf_d: shared-memory staging for the stage-2 loads (>= 32 doubles;
// the launching kernel's dynamic shared memory, free by the time it finalizes)
__device__ inline void finalize(SolveState* st, int fin, int arg, bool ing, double* buf, int buf_d) {
  const int th = threadIdx.x & 31;  // executed by one warp
#if PK_FIN_PREFETCH
  if (th < (int)((sizeof(SolveState) + 127) / 128)) asm volatile("prefetch.global.L1 [%0];" ::"l"((const char*)st + th * 128));
#endif
  const int ng = st->n_groups;
  double tot[4];
  switch (fin) {
    case FIN_CG_SETUP: {
      const S2Col cs[4] = {{st->p_rr, 1, 0}, {st->p_two, 2, 0}, {st->p_two, 2, 1}, {st->p_bb, 1, 0}};
      stage2_warp<4>(cs, ng, tot, buf, buf_d);
      if (th == 0) cg_scalars(st, tot[0], tot[1], tot[2], true, tot[3], ing);
      break;
    }
    case FIN_CG_FUSED: {
      const S2Col cs[3] = {{st->p_three, 3, 0}, {st->p_three, 3, 1}, {st->p_three, 3, 2}};
      stage2_warp<3>(cs, ng, tot, buf, buf_d);
      if (th == 0) {
        st->parity ^= 1;
        cg_scalars(st, tot[0], tot[1], tot[2], false, 0.0, ing);
      }
      break;
    }
    case FIN_BICG_SETUP: {
      const S2Col cs[2] = {{st->p_pair, 2, 0}, {st->p_bb, 1, 0}};
      stage2_warp<2>(cs, ng, tot, buf, buf_d);
      if (th != 0) return;
      double rr = tot[0];
      double nb = msqrt(tot[1]);
      st->scale = nb > 0.0 ? nb : 1.0;
      st->rr = rr;
      bool stop = false;
      if (div_rn(msqrt(rr), st->scale) <= st->tol && (!st->fixed || rr == 0.0)) {
        st->term = PK_TERM_CONVERGED; stop = true;
      }
      st->status = stop ? STOPPED : RUNNING;
      set_cond(st, stop ? 0u : 1u, ing);
      break;
    }
    case FIN_BICG_ALPHA: {
      // fused_bicgstab_s_update's in-kernel alpha (fused.py:172-176)
      const S2Col cs[2] = {{st->p_pair, 2, 0}, {st->p_pair, 2, 1}};
      stage2_warp<2>(cs, ng, tot, buf, buf_d);
      if (th != 0) return;
      if (arg) st->parity ^= 1;
      double rho = tot[0], d = tot[1];
      st->rho0 = rho;
      st->apr = d;
      if (fabs(d) < st->btol_loop) {
        st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_APR0STAR;
        st->status = STOPPED;
        set_cond(st, 0u, ing);
      } else {
        st->alpha = div_rn(rho, d);
      }
      break;
    }
    case FIN_BICG_TAIL: {
      // solvers.py:647-684
      const S2Col cs[4] = {{st->p_quad, 4, 0}, {st->p_quad, 4, 1}, {st->p_quad, 4, 2}, {st->p_quad, 4, 3}};
      stage2_warp<4>(cs, ng, tot, buf, buf_d);
      if (th != 0) return;
      double ss = tot[0], ass = tot[1], asas = tot[2], asr = tot[3], apr = st->apr;
      st->ss = ss; st->ass = ass; st->asas = asas; st->asr = asr;
      double mon_s = div_rn(msqrt(ss), st->scale);
      int status = RUNNING;
      if (!st->fixed && mon_s <= st->tol) {
        st->hist[st->iter] = mon_s;
        st->iter += 1;
        st->half_step = 1;
        st->term = PK_TERM_CONVERGED;
        status = STOPPED;
      } else if (asas < st->btol_loop || asas == 0.0) {
        st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_ASAS; status = STOPPED;
      } else if (apr == 0.0) {
        st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_APR0STAR; status = STOPPED;
      } else {
        double om = div_rn(ass, asas);
        st->omega = om;
        st->beta = div_rn(-asr, apr);
        double ident = add_rn(sub_rn(ss, mul_rn(mul_rn(2.0, om), ass)), mul_rn(mul_rn(om, om), asas));
        st->ident = ident;
        int clamped = ident < 0.0;
        double rr = (0.0 > ident) ? 0.0 : ident;  // Python max(ident, 0.0)
        st->clamped = clamped;
        st->rr = rr;
        double mon = div_rn(msqrt(rr), st->scale);
        st->hist[st->iter] = mon;
        st->iter += 1;
        if (!isfinite(mon)) {
          st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_DIVERGENCE; status = STOPPING;
        } else if (!st->fixed && mon <= st->tol) {
          if (clamped) st->need_check = 1;
          else st->term = PK_TERM_CONVERGED;
          status = STOPPING;
        } else if (st->iter >= st->limit) {
          st->term = PK_TERM_MAX_ITER; status = STOPPING;
        }
      }
      st->status = status;
      set_cond(st, status == RUNNING ? 1u : 0u, ing);
      break;
    }
    case FIN_BICG_XTAIL: {
      if (th == 0) {
        st->parity ^= 1;
        st->status = STOPPED;
      }
      break;
    }
    case FIN_GM_RHO: {
      const S2Col cs[2] = {{st->p_rr, 1, 0}, {st->p_bb, 1, 0}};
      stage2_warp<2>(cs, ng, tot, buf, buf_d);
      if (th != 0) return;
      if (arg) {
        double nb = msqrt(tot[1]);
        st->scale = nb > 0.0 ? nb : 1.0;
      }
      st->rho = msqrt(tot[0]);
      break;
    }
    case FIN_GM_NORM: {
      // arg = step index i (1-based)
      const S2Col cs[1] = {{st->p_ww, 1, 0}};
      stage2_warp<1>(cs, ng, tot, buf, buf_d);
      if (th == 0) {
        double nrm = msqrt(tot[0]);
        st->nrm = nrm;
        if (nrm < st->btol_loop || nrm == 0.0) {
          st->lucky = 1;
        } else {
          st->R[(int64_t)(arg - 1) * st->m + (arg - 1)] = nrm;
          st->inv = div_rn(1.0, nrm);
        }
      }
      break;
    }
    case FIN_GM_COEF: {
      // arg = step index i (>= 2): columns 0..i-2 of p_coef, up to 32 at a
      // time (lane c sums column j0 + c over the groups, serially, in group
      // order -- linalg.py:311-320); the [ng][m] partials are staged through
      // shared memory with coalesced loads
      const int nc = arg - 1, m = st->m;
      for (int j0 = 0; j0 < nc; j0 += 32) {
        const int nj = (nc - j0) < 32 ? (nc - j0) : 32;
        const int CH = buf_d / nj;
        double t = 0.0;
        for (int g0 = 0; g0 < ng; g0 += CH) {
          const int cnt = (ng - g0) < CH ? (ng - g0) : CH;
          __syncwarp();
          for (int idx = th; idx < cnt * nj; idx += 32) {
            const int g = idx / nj, c = idx - g * nj;
            buf[c * CH + g] = __ldcg(st->p_coef + (int64_t)(g0 + g) * m + j0 + c);
          }
          __syncwarp();
          if (th < nj) {
            const double* b = buf + th * CH;
            int g = 0;
            for (; g + 8 <= cnt; g += 8) {
              double v[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) v[u] = b[g + u];
#pragma unroll
              for (int u = 0; u < 8; ++u) t = add_rn(t, v[u]);
            }
            for (; g < cnt; ++g) t = add_rn(t, b[g]);
          }
        }
        if (th < nj) {
          st->coef[j0 + th] = t;
          st->R[(int64_t)(j0 + th) * m + (arg - 1)] = t;
        }
        __syncwarp();
      }
      break;
    }
    case FIN_GM_XI: {
      const S2Col cs[1] = {{st->p_xi + (int64_t)(arg - 1) * ng, 1, 0}};
      stage2_warp<1>(cs, ng, tot, buf, buf_d);
      if (th == 0) {
        st->xi[arg - 1] = tot[0];
        st->step = arg;
      }
      break;
    }
    case FIN_DOTV: {
      const S2Col cs[1] = {{st->p_bb, 1, 0}};
      stage2_warp<1>(cs, ng, tot, buf, buf_d);
      if (th == 0) st->dotv = tot[0];
      break;
    }
    default:
      break;
  }
}

// Device scalar sources for an op: the solver points these at SolveState
// fields written by the previous finalizer; kernel-level entries leave them
// null and pass values.  `par` selects the current half of ping-pong pairs.
struct ScalarPtrs {
  const double* a;
  const double* b;
  const double* c;
  const int32_t* par;
};

// scalars and the ping-pong parity come from the previous kernel's finalizer:
// L1-cached loads (see gate_load)
#ifdef PK_OLD_PROLOGUE
__device__ __forceinline__ double ld_scalar(const double* p, double v) { return p ? __ldcg(p) : v; }
#else
__device__ __forceinline__ double ld_scalar(const double* p, double v) { return p ? __ldg(p) : v; }
#endif

// 16-byte vector access (rows i, i + 1; i even, base 16-byte aligned)
__device__ __forceinline__ double2 ld2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double a, double b) {
  *reinterpret_cast<double2*>(p) = make_double2(a, b);
}
__host__ __device__ inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
__device__ __forceinline__ int ld_par(const int32_t* p) { return p ? __ldg(p) : 0; }

// ---------------------------------------------------------------------------
// SpMV operators (Op::kSpmv): the engine walks the row's CSR entries, the
// operator supplies gload/gval (the SpMV input at a gathered column) and the
// per-row epilogue.  kSlots = entries per pass (all loads of a pass in
// flight): 5 for 2-D 5-point rows, 7 for 3-D 7-point rows.
// ---------------------------------------------------------------------------

// q = A p with NQ fused dots (fused.py:86-120); NQ = 0: plain spmv_csr.
template <typename RowT_, int NQ, int S_, bool SELL_ = false>
struct OpSpmvFused {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = 4;
  static constexpr int kRowsPerThread = 2;
  static constexpr int kSlots = S_;
  Csr<RowT, SELL_> A;
  const double* __restrict__ p;  // gather base (column index space)
  double* q;
  int32_t kind[4];
  const double* w[4];
  int64_t own_off;                // own row i of p is p[own_off + i] (row-partitioned halo layout)
  struct Item { double pv; double wv[NQ > 0 ? NQ : 1]; };
  struct Gat { double v; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const {
    it.pv = 0.0;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      it.wv[k] = 0.0;
      if (kind[k] == PK_DOT_INPUT) it.pv = __ldg(p + own_off + row);
      if (kind[k] == PK_DOT_VECTOR) it.wv[k] = __ldg(w[k] + row);
    }
  }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const { g.v = __ldg(p + col); }
  __device__ __forceinline__ double gval(const Gat& g) const { return g.v; }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double acc, double (&c)[M]) const {
    if (q) q[row] = acc;
#pragma unroll
    for (int k = 0; k < NQ && k < M; ++k) {
      c[k] = kind[k] == PK_DOT_INPUT ? mul_rn(acc, it.pv)
           : kind[k] == PK_DOT_RESULT ? mul_rn(acc, acc) : mul_rn(acc, it.wv[k]);
    }
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// r = b + (-1) A x (add_scaled, linalg.py:450-457); optional copies; <r,r>.
template <typename RowT_, int S_, bool SELL_ = false>
struct OpResidual {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = 4;
  static constexpr int kRowsPerThread = 2;
  static constexpr int kSlots = S_;
  Csr<RowT, SELL_> A;
  const double* __restrict__ x;
  const double* __restrict__ b;
  double* r;
  double* copy1;
  double* copy2;
  struct Item { double bv; };
  struct Gat { double v; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const { it.bv = __ldg(b + row); }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const { g.v = __ldg(x + col); }
  __device__ __forceinline__ double gval(const Gat& g) const { return g.v; }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double q, double (&c)[M]) const {
    double rv = add_rn(it.bv, mul_rn(-1.0, q));
    if (r) r[row] = rv;
    if (copy1) copy1[row] = rv;
    if (copy2) copy2[row] = rv;
    c[0] = mul_rn(rv, rv);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// One pipelined-CG iteration in one kernel (fused.py:123-151 + 86-120):
//   r' = r - a Ap;  p' = p b + r';  x += a p;  Ap' = A p';
//   contributions [r'.r', Ap'.p', Ap'.Ap'].
// p' at a gathered column is recomputed from (p, r, Ap) there.
template <typename RowT_, int S_, bool SELL_ = false>
struct OpCgFused {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = 3;
  static constexpr int kRowsPerThread = 2;
  static constexpr int kSlots = S_;
  Csr<RowT, SELL_> A;
  double* x;
  double* r[2];
  double* p[2];
  double* ap[2];
  double alpha, beta;
  int64_t goff;      // gather base = own base - goff (row-partitioned halo layout; 0 otherwise)
  const double* rc;  // current halves (own rows), resolved in scalars()
  const double* pc;
  const double* apc;
  const double* rg;  // the same vectors in column index space
  const double* pg;
  const double* apg;
  double* rn_;
  double* pn_;
  double* apn_;
  struct Item { double x, r, p, ap; };
  struct Gat { double r, ap, p; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const {
    it.x = __ldg(x + row); it.r = __ldg(rc + row); it.p = __ldg(pc + row); it.ap = __ldg(apc + row);
  }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const {
    g.r = __ldg(rg + col); g.ap = __ldg(apg + col); g.p = __ldg(pg + col);
  }
  __device__ __forceinline__ double gval(const Gat& g) const {
    double rn = sub_rn(g.r, mul_rn(alpha, g.ap));
    return add_rn(mul_rn(g.p, beta), rn);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double q, double (&c)[M]) const {
    double xn = add_rn(it.x, mul_rn(alpha, it.p));
    double rn = sub_rn(it.r, mul_rn(alpha, it.ap));
    double pn = add_rn(mul_rn(it.p, beta), rn);
    x[row] = xn; rn_[row] = rn; pn_[row] = pn; apn_[row] = q;
    c[0] = mul_rn(rn, rn);
    c[1] = mul_rn(q, pn);
    c[2] = mul_rn(q, q);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    beta = ld_scalar(sp.b, beta);
    const int cur = ld_par(sp.par);
    rc = cur ? r[1] : r[0]; pc = cur ? p[1] : p[0]; apc = cur ? ap[1] : ap[0];
    rn_ = cur ? r[0] : r[1]; pn_ = cur ? p[0] : p[1]; apn_ = cur ? ap[0] : ap[1];
    rg = rc - goff; pg = pc - goff; apg = apc - goff;
  }
};

// Split form of OpCgFused (PK_CG_SPLIT=1): the CG vector update as an
// elementwise sweep (cur -> next halves) and a one-gather SpMV of p' with the
// same contributions [r'.r', Ap'.p', Ap'.Ap'].
struct OpCgXSweep {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  double* x;
  double* r[2];
  double* p[2];
  double* ap[2];
  double alpha, beta;
  const double* rc;
  const double* pc;
  const double* apc;
  double* rn_;
  double* pn_;
  struct Item { double x, r, p, ap; };
  struct Item2 { double2 x, r, p, ap; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.x = __ldg(x + i); it.r = __ldg(rc + i); it.p = __ldg(pc + i); it.ap = __ldg(apc + i);
  }
  __device__ __forceinline__ void upd(double xv, double r, double p, double ap, double& xn, double& rn,
                                      double& pn) const {
    xn = add_rn(xv, mul_rn(alpha, p));
    rn = sub_rn(r, mul_rn(alpha, ap));
    pn = add_rn(mul_rn(p, beta), rn);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&)[M]) const {
    double xn, rn, pn;
    upd(it.x, it.r, it.p, it.ap, xn, rn, pn);
    x[i] = xn; rn_[i] = rn; pn_[i] = pn;
  }
  __device__ __forceinline__ void load2(uint32_t i, Item2& t) const {
    t.x = ld2(x + i); t.r = ld2(rc + i); t.p = ld2(pc + i); t.ap = ld2(apc + i);
  }
  __device__ __forceinline__ void compute2(uint32_t i, Item2& t) const {
    double x0, r0, p0, x1, r1, p1;
    upd(t.x.x, t.r.x, t.p.x, t.ap.x, x0, r0, p0);
    upd(t.x.y, t.r.y, t.p.y, t.ap.y, x1, r1, p1);
    st2(x + i, x0, x1); st2(rn_ + i, r0, r1); st2(pn_ + i, p0, p1);
  }
  bool aligned16() const {
    return al16(x) && al16(r[0]) && al16(r[1]) && al16(p[0]) && al16(p[1]) && al16(ap[0]) && al16(ap[1]);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    beta = ld_scalar(sp.b, beta);
    const int cur = ld_par(sp.par);
    rc = cur ? r[1] : r[0]; pc = cur ? p[1] : p[0]; apc = cur ? ap[1] : ap[0];
    rn_ = cur ? r[0] : r[1]; pn_ = cur ? p[0] : p[1];
  }
};

template <typename RowT_, int S_, bool SELL_ = false>
struct OpCgApNext {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = 4;
  static constexpr int kRowsPerThread = 2;
  static constexpr int kSlots = S_;
  Csr<RowT, SELL_> A;
  double* r[2];
  double* p[2];
  double* ap[2];
  int64_t goff;      // gather base = own base - goff (row-partitioned halo layout; 0 otherwise)
  const double* rn;
  const double* pn;
  const double* pg;
  double* apn;
  struct Item { double r, p; };
  struct Gat { double p; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const { it.r = __ldg(rn + row); it.p = __ldg(pn + row); }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const { g.p = __ldg(pg + col); }
  __device__ __forceinline__ double gval(const Gat& g) const { return g.p; }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double q, double (&c)[M]) const {
    apn[row] = q;
    c[0] = mul_rn(it.r, it.r);
    c[1] = mul_rn(q, it.p);
    c[2] = mul_rn(q, q);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    const int cur = ld_par(sp.par);
    rn = cur ? r[0] : r[1]; pn = cur ? p[0] : p[1]; apn = cur ? ap[0] : ap[1];
    pg = pn - goff;
  }
};

// BiCGStab second SpMV with the s-update folded in (fused.py:154-182 + 86-120):
//   s = r - a Ap (recomputed at every gathered column, never stored);
//   As = A s;  contributions [s.s, As.s, As.As, As.r0*].
template <typename RowT_, int S_, bool SELL_ = false>
struct OpBicgB {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = PK_BICGB_MINB;
  static constexpr int kRowsPerThread = PK_BICG_U;
  static constexpr int kSlots = S_;
  Csr<RowT, SELL_> A;
  const double* r[2];
  const double* ap[2];
  const double* __restrict__ r0;
  double* as;
  double alpha;
  const double* rc;
  const double* apc;
  struct Item { double s, r0; };
  struct Gat { double r, ap; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const {
    it.s = sub_rn(__ldg(rc + row), mul_rn(alpha, __ldg(apc + row)));
    it.r0 = __ldg(r0 + row);
  }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const { g.r = __ldg(rc + col); g.ap = __ldg(apc + col); }
  __device__ __forceinline__ double gval(const Gat& g) const { return sub_rn(g.r, mul_rn(alpha, g.ap)); }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double q, double (&c)[M]) const {
    as[row] = q;
    c[0] = mul_rn(it.s, it.s);
    c[1] = mul_rn(q, it.s);
    c[2] = mul_rn(q, q);
    c[3] = mul_rn(q, it.r0);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    const int cur = ld_par(sp.par);
    rc = cur ? r[1] : r[0];
    apc = cur ? ap[1] : ap[0];
  }
};

// BiCGStab xrp update of iteration k fused with the first SpMV of k+1
// (fused.py:185-219 + 86-120):
//   s = r - a Ap;  x += (a p) + (w s);  r' = s - w As;  p' = ((p - w Ap) b) + r';
//   Ap' = A p';  contributions [r'.r0*, Ap'.r0*].
template <typename RowT_, int S_, bool SELL_ = false>
struct OpBicgA {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = 2;
  static constexpr int kRowsPerThread = 4;
  static constexpr int kSlots = S_;
  static constexpr int kWarpRows = 2;
  Csr<RowT, SELL_> A;
  double* x;
  double* r[2];
  double* p[2];
  double* ap[2];
  const double* __restrict__ as;
  const double* __restrict__ r0;
  double alpha, omega, beta;
  const double* rc;
  const double* pc;
  const double* apc;
  double* rn_;
  double* pn_;
  double* apn_;
  struct Item { double x, r, p, ap, as, r0; };
  struct Gat { double r, ap, as, p; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const {
    it.x = __ldg(x + row); it.r = __ldg(rc + row); it.p = __ldg(pc + row); it.ap = __ldg(apc + row);
    it.as = __ldg(as + row); it.r0 = __ldg(r0 + row);
  }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const {
    g.r = __ldg(rc + col); g.ap = __ldg(apc + col); g.as = __ldg(as + col); g.p = __ldg(pc + col);
  }
  __device__ __forceinline__ double gval(const Gat& g) const {
    double s = sub_rn(g.r, mul_rn(alpha, g.ap));
    double rn = sub_rn(s, mul_rn(omega, g.as));
    return add_rn(mul_rn(sub_rn(g.p, mul_rn(omega, g.ap)), beta), rn);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double q, double (&c)[M]) const {
    double s = sub_rn(it.r, mul_rn(alpha, it.ap));
    double xn = add_rn(it.x, add_rn(mul_rn(alpha, it.p), mul_rn(omega, s)));
    double rn = sub_rn(s, mul_rn(omega, it.as));
    double pn = add_rn(mul_rn(sub_rn(it.p, mul_rn(omega, it.ap)), beta), rn);
    x[row] = xn; rn_[row] = rn; pn_[row] = pn; apn_[row] = q;
    c[0] = mul_rn(rn, it.r0);
    c[1] = mul_rn(q, it.r0);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    omega = ld_scalar(sp.b, omega);
    beta = ld_scalar(sp.c, beta);
    const int cur = ld_par(sp.par);
    rc = cur ? r[1] : r[0]; pc = cur ? p[1] : p[0]; apc = cur ? ap[1] : ap[0];
    rn_ = cur ? r[0] : r[1]; pn_ = cur ? p[0] : p[1]; apn_ = cur ? ap[0] : ap[1];
  }
};

// Split form of OpBicgA (the default BiCGStab body): the xrp update as a
// lean elementwise sweep (OpBicgXrpSweep, cur -> next half of the ping-pong
// pairs) followed by a one-gather SpMV of p' carrying the same two
// contributions [r'.r0*, Ap'.r0*] (OpBicgApNext).  Same IEEE operations on
// the same inputs as OpBicgA, so the same bits.  Measured (C2): the fused
// OpBicgA's four gathers per nonzero keep it at 2 CTAs/SM and 2.3 TB/s
// (64 us); sweep + light SpMV take 15 + 34 us.
struct OpBicgXrpSweep {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  double* x;
  double* r[2];
  double* p[2];
  double* ap[2];
  const double* __restrict__ as;
  double alpha, omega, beta;
  const double* rc;
  const double* pc;
  const double* apc;
  double* rn_;
  double* pn_;
  struct Item { double x, r, p, ap, as; };
  struct Item2 { double2 x, r, p, ap, as; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.x = __ldg(x + i); it.r = __ldg(rc + i); it.p = __ldg(pc + i); it.ap = __ldg(apc + i); it.as = __ldg(as + i);
  }
  __device__ __forceinline__ void upd(double xv, double r, double p, double ap, double asv, double& xn, double& rn,
                                      double& pn) const {
    double s = sub_rn(r, mul_rn(alpha, ap));
    xn = add_rn(xv, add_rn(mul_rn(alpha, p), mul_rn(omega, s)));
    rn = sub_rn(s, mul_rn(omega, asv));
    pn = add_rn(mul_rn(sub_rn(p, mul_rn(omega, ap)), beta), rn);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&)[M]) const {
    double xn, rn, pn;
    upd(it.x, it.r, it.p, it.ap, it.as, xn, rn, pn);
    x[i] = xn; rn_[i] = rn; pn_[i] = pn;
  }
  __device__ __forceinline__ void load2(uint32_t i, Item2& t) const {
    t.x = ld2(x + i); t.r = ld2(rc + i); t.p = ld2(pc + i); t.ap = ld2(apc + i); t.as = ld2(as + i);
  }
  __device__ __forceinline__ void compute2(uint32_t i, Item2& t) const {
    double x0, r0, p0, x1, r1, p1;
    upd(t.x.x, t.r.x, t.p.x, t.ap.x, t.as.x, x0, r0, p0);
    upd(t.x.y, t.r.y, t.p.y, t.ap.y, t.as.y, x1, r1, p1);
    st2(x + i, x0, x1); st2(rn_ + i, r0, r1); st2(pn_ + i, p0, p1);
  }
  bool aligned16() const {
    return al16(x) && al16(r[0]) && al16(r[1]) && al16(p[0]) && al16(p[1]) && al16(ap[0]) && al16(ap[1]) && al16(as);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    omega = ld_scalar(sp.b, omega);
    beta = ld_scalar(sp.c, beta);
    const int cur = ld_par(sp.par);
    rc = cur ? r[1] : r[0]; pc = cur ? p[1] : p[0]; apc = cur ? ap[1] : ap[0];
    rn_ = cur ? r[0] : r[1]; pn_ = cur ? p[0] : p[1];
  }
};

template <typename RowT_, int S_, bool SELL_ = false>
struct OpBicgApNext {
  using RowT = RowT_;
  static constexpr bool kSpmv = true;
  static constexpr int kMinBlocks = PK_BICGB_MINB;
  static constexpr int kRowsPerThread = PK_BICG_U;
  static constexpr int kSlots = S_;
  Csr<RowT, SELL_> A;
  double* r[2];
  double* p[2];
  double* ap[2];
  const double* __restrict__ r0;
  const double* rn;
  const double* pn;
  double* apn;
  struct Item { double r, r0; };
  struct Gat { double p; };
  __device__ __forceinline__ void load(uint32_t row, Item& it) const { it.r = __ldg(rn + row); it.r0 = __ldg(r0 + row); }
  __device__ __forceinline__ void gload(uint32_t col, Gat& g) const { g.p = __ldg(pn + col); }
  __device__ __forceinline__ double gval(const Gat& g) const { return g.p; }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t row, Item& it, double q, double (&c)[M]) const {
    apn[row] = q;
    c[0] = mul_rn(it.r, it.r0);
    c[1] = mul_rn(q, it.r0);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    const int cur = ld_par(sp.par);
    rn = cur ? r[0] : r[1]; pn = cur ? p[0] : p[1]; apn = cur ? ap[0] : ap[1];
  }
};

// ---------------------------------------------------------------------------
// elementwise operators
// ---------------------------------------------------------------------------

// Stand-alone BiCGStab xrp of the final iteration (s recomputed from r, Ap);
// contribution r'.r0* (the rr0 partials a resumed loop needs).
struct OpBicgXrpTail {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  double* x;
  double* r[2];
  double* p[2];
  const double* ap[2];
  const double* __restrict__ as;
  const double* __restrict__ r0;
  double alpha, omega, beta;
  int cur;
  struct Item { double x, r, p, ap, as, r0; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.x = x[i]; it.r = (cur ? r[1] : r[0])[i]; it.p = (cur ? p[1] : p[0])[i];
    it.ap = __ldg((cur ? ap[1] : ap[0]) + i); it.as = __ldg(as + i); it.r0 = __ldg(r0 + i);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
    double s = sub_rn(it.r, mul_rn(alpha, it.ap));
    double xn = add_rn(it.x, add_rn(mul_rn(alpha, it.p), mul_rn(omega, s)));
    double rn = sub_rn(s, mul_rn(omega, it.as));
    double pn = add_rn(mul_rn(sub_rn(it.p, mul_rn(omega, it.ap)), beta), rn);
    x[i] = xn; (cur ? r[0] : r[1])[i] = rn; (cur ? p[0] : p[1])[i] = pn;
    c[0] = mul_rn(rn, it.r0);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    omega = ld_scalar(sp.b, omega);
    beta = ld_scalar(sp.c, beta);
    cur = ld_par(sp.par);
  }
};

// fused_cg_vector_update (fused.py:123-151)
struct OpCgUpdate {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  double* x;
  double* r;
  double* p;
  const double* __restrict__ ap;
  double alpha, beta;
  struct Item { double x, r, p, ap; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.x = x[i]; it.r = r[i]; it.p = p[i]; it.ap = __ldg(ap + i);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
    double xn = add_rn(it.x, mul_rn(alpha, it.p));
    double rn = sub_rn(it.r, mul_rn(alpha, it.ap));
    double pn = add_rn(mul_rn(it.p, beta), rn);
    x[i] = xn; r[i] = rn; p[i] = pn;
    c[0] = mul_rn(rn, rn);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    beta = ld_scalar(sp.b, beta);
  }
};

// fused_bicgstab_s_update (fused.py:154-182): s = r - alpha Ap, <s,s>
struct OpBicgS {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  const double* __restrict__ r;
  const double* __restrict__ ap;
  double* s;
  double alpha;
  struct Item { double r, ap; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const { it.r = __ldg(r + i); it.ap = __ldg(ap + i); }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
    double v = sub_rn(it.r, mul_rn(alpha, it.ap));
    s[i] = v;
    c[0] = mul_rn(v, v);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) { alpha = ld_scalar(sp.a, alpha); }
};

// fused_bicgstab_xrp_update (fused.py:185-219)
struct OpBicgXrp {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  double* x;
  double* r;
  double* p;
  const double* __restrict__ s;
  const double* __restrict__ ap;
  const double* __restrict__ as;
  const double* __restrict__ r0;
  double alpha, omega, beta;
  struct Item { double x, p, s, ap, as, r0; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.x = x[i]; it.p = p[i]; it.s = __ldg(s + i); it.ap = __ldg(ap + i); it.as = __ldg(as + i); it.r0 = __ldg(r0 + i);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
    double xn = add_rn(it.x, add_rn(mul_rn(alpha, it.p), mul_rn(omega, it.s)));
    double rn = sub_rn(it.s, mul_rn(omega, it.as));
    double pn = add_rn(mul_rn(sub_rn(it.p, mul_rn(omega, it.ap)), beta), rn);
    x[i] = xn; r[i] = rn; p[i] = pn;
    c[0] = mul_rn(rn, it.r0);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    alpha = ld_scalar(sp.a, alpha);
    omega = ld_scalar(sp.b, omega);
    beta = ld_scalar(sp.c, beta);
  }
};

// x * y contributions (dot, reduce_stage1 of a product)
struct OpDot {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  const double* __restrict__ x;
  const double* __restrict__ y;
  struct Item { double x, y; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const { it.x = __ldg(x + i); it.y = __ldg(y + i); }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const { c[0] = mul_rn(it.x, it.y); }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// NQ precomputed contribution columns (reduce_stage1 of stacked streams).
template <int NQ>
struct OpColumns {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  const double* col[NQ];
  struct Item { double v[NQ]; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
#pragma unroll
    for (int k = 0; k < NQ; ++k) it.v[k] = __ldg(col[k] + i);
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
#pragma unroll
    for (int k = 0; k < NQ && k < M; ++k) c[k] = it.v[k];
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// fused_gs_stage1 (fused.py:222-243): <b_j, v> for j < nb (nb <= NB).
template <int NB>
struct OpMultiDot {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  static constexpr int kWarpRows = NB > 8 ? 1 : 2;
  const double* __restrict__ v;
  int32_t nb;
  const double* b[NB];
  struct Item { double v; double b[NB]; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.v = __ldg(v + i);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      it.b[j] = 0.0;
      if (j < nb) it.b[j] = __ldg(b[j] + i);
    }
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
#pragma unroll
    for (int j = 0; j < NB && j < M; ++j) c[j] = j < nb ? mul_rn(it.b[j], it.v) : 0.0;
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// fused_gs_update (fused.py:246-277): v -= sum_j c_j b_j; <v,v>.
// acc = ((0 + c_0 b_0) + c_1 b_1) + ... in basis order (fused.py:268-272); a
// basis longer than NB is accumulated in chunks (OpGsAcc) through an
// n-vector `acc_in` -- the running sum is stored exactly, so the chunked sum
// is the same sequence of roundings.
template <int NB>
struct OpGsUpdate {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = NB > 8 ? 2 : 4;
  static constexpr int kWarpRows = NB > 8 ? 1 : 2;
  double* v;
  int32_t nb;
  const double* b[NB];
  const double* coef;    // device [nb], finalized by the previous kernel
  const double* acc_in;  // running sum of the earlier chunks, or null (start from 0.0)
  double cf[NB];         // the coefficients, loaded once per thread in scalars()
  struct Item { double v, a; double b[NB]; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.v = v[i];
    it.a = acc_in ? __ldg(acc_in + i) : 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      it.b[j] = 0.0;
      if (j < nb) it.b[j] = __ldg(b[j] + i);
    }
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&cc)[M]) const {
    double acc = it.a;
#pragma unroll
    for (int j = 0; j < NB; ++j) if (j < nb) acc = add_rn(acc, mul_rn(cf[j], it.b[j]));
    double vn = (nb > 0 || acc_in) ? sub_rn(it.v, acc) : it.v;
    v[i] = vn;
    cc[0] = mul_rn(vn, vn);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    if (sp.a) coef = sp.a;
#pragma unroll
    for (int j = 0; j < NB; ++j) cf[j] = j < nb ? __ldg(coef + j) : 0.0;
  }
};

// A leading chunk of the Gram-Schmidt accumulation (no reduction):
// acc_out = acc_in (or 0.0) + sum_j c_j b_j over this chunk, in order.
template <int NB>
struct OpGsAcc {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = NB > 8 ? 2 : 4;
  int32_t nb;
  const double* b[NB];
  const double* coef;
  const double* acc_in;
  double* acc_out;
  double cf[NB];
  static constexpr int kPairs = NB > 8 ? 1 : 2;
  struct Item { double a; double b[NB]; };
  struct Item2 { double2 a; double2 b[NB]; };
  __device__ __forceinline__ void load2(uint32_t i, Item2& t) const {
    t.a = acc_in ? ld2(acc_in + i) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < NB; ++j) t.b[j] = j < nb ? ld2(b[j] + i) : make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ void compute2(uint32_t i, Item2& t) const {
    double a0 = t.a.x, a1 = t.a.y;
#pragma unroll
    for (int j = 0; j < NB; ++j)
      if (j < nb) {
        a0 = add_rn(a0, mul_rn(cf[j], t.b[j].x));
        a1 = add_rn(a1, mul_rn(cf[j], t.b[j].y));
      }
    st2(acc_out + i, a0, a1);
  }
  bool aligned16() const {
    bool ok = al16(acc_out) && (!acc_in || al16(acc_in));
    for (int j = 0; j < NB; ++j) ok = ok && (j >= nb || al16(b[j]));
    return ok;
  }
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.a = acc_in ? __ldg(acc_in + i) : 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      it.b[j] = 0.0;
      if (j < nb) it.b[j] = __ldg(b[j] + i);
    }
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&)[M]) const {
    double acc = it.a;
#pragma unroll
    for (int j = 0; j < NB; ++j) if (j < nb) acc = add_rn(acc, mul_rn(cf[j], it.b[j]));
    acc_out[i] = acc;
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {
#pragma unroll
    for (int j = 0; j < NB; ++j) cf[j] = j < nb ? __ldg(coef + j) : 0.0;
  }
};

// Split Gram-Schmidt update, elementwise half (PK_GS_SPLIT): the same
// v_new = v - acc (acc = acc_in + sum_j c_j b_j in basis order) as OpGsUpdate,
// written through 16-byte accesses at full occupancy; the <v_new, v_new>
// partials follow in a separate dot (OpDot on the LANE engine) -- the same
// products in the same order, so the same bits, for one more read of v.
template <int NB>
struct OpGsSweep {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 2;
  static constexpr int kPairs = NB > 8 ? 1 : 2;
  double* v;
  int32_t nb;
  const double* b[NB];
  const double* coef;
  const double* acc_in;
  double cf[NB];
  struct Item { double v, a; double b[NB]; };
  struct Item2 { double2 v, a; double2 b[NB]; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const {
    it.v = v[i];
    it.a = acc_in ? __ldg(acc_in + i) : 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) it.b[j] = j < nb ? __ldg(b[j] + i) : 0.0;
  }
  __device__ __forceinline__ double upd(double vv, double a, const double (&bb)[NB]) const {
#pragma unroll
    for (int j = 0; j < NB; ++j) if (j < nb) a = add_rn(a, mul_rn(cf[j], bb[j]));
    return (nb > 0 || acc_in) ? sub_rn(vv, a) : vv;
  }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&)[M]) const { v[i] = upd(it.v, it.a, it.b); }
  __device__ __forceinline__ void load2(uint32_t i, Item2& t) const {
    t.v = *reinterpret_cast<const double2*>(v + i);
    t.a = acc_in ? ld2(acc_in + i) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < NB; ++j) t.b[j] = j < nb ? ld2(b[j] + i) : make_double2(0.0, 0.0);
  }
  __device__ __forceinline__ void compute2(uint32_t i, Item2& t) const {
    double b0[NB], b1[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) { b0[j] = t.b[j].x; b1[j] = t.b[j].y; }
    st2(v + i, upd(t.v.x, t.a.x, b0), upd(t.v.y, t.a.y, b1));
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    if (sp.a) coef = sp.a;
#pragma unroll
    for (int j = 0; j < NB; ++j) cf[j] = j < nb ? __ldg(coef + j) : 0.0;
  }
  bool aligned16() const {
    bool ok = al16(v) && (!acc_in || al16(acc_in));
    for (int j = 0; j < NB; ++j) ok = ok && (j >= nb || al16(b[j]));
    return ok;
  }
};

// fused_gs_normalize (fused.py:280-305): v *= inv; <r, v>.
struct OpNormalize {
  static constexpr bool kSpmv = false;
  static constexpr int kMinBlocks = 4;
  double* v;
  const double* __restrict__ r;
  double inv;
  struct Item { double v, r; };
  __device__ __forceinline__ void load(uint32_t i, Item& it) const { it.v = v[i]; it.r = __ldg(r + i); }
  template <int M>
  __device__ __forceinline__ void compute(uint32_t i, Item& it, double (&c)[M]) const {
    double vn = mul_rn(it.v, inv);
    v[i] = vn;
    c[0] = mul_rn(it.r, vn);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) { inv = ld_scalar(sp.a, inv); }
};

}  // namespace pk
