// Fused kernels of the pipelined Krylov path (sm_100a).
//
// Every reduction kernel is "elementwise op + ordered stage 1" (pk_reduce.cuh)
// with an optional last-CTA finalizer that performs the serial stage 2 and the
// host-side scalar recurrences of the reference on the device, so the next
// kernel's prologue only reads a few scalars (SolveState).
//
// Per-element arithmetic follows the reference exactly:
//   SpMV row        acc = acc + v*x          _spmvkernels.py:12-18
//   CG update       x+a p; r-a Ap; p b + r   fused.py:145-148
//   BiCG s          r - a Ap                 fused.py:177
//   BiCG xrp        x+((a p)+(w s)); s-w As; ((p-w Ap) b)+r   fused.py:212-216
//   GS update       v - sum_j (c_j b_j)      fused.py:268-272
//   GS normalize    v * (1/||v||)            fused.py:300
#pragma once

#include <math.h>

#include "pk_reduce.cuh"
#include "pk_state.cuh"

namespace pk {

// ---------------------------------------------------------------------------
// finalizers (run by every thread of the last CTA of a launch)
// ---------------------------------------------------------------------------

enum Fin : int32_t {
  FIN_NONE = 0,
  FIN_CG_SETUP,
  FIN_CG_ITER,
  FIN_BICG_SETUP,
  FIN_BICG_ALPHA,
  FIN_BICG_TAIL,
  FIN_GM_RHO,      // cycle setup: rho (and scale on the first cycle)
  FIN_GM_NORM,     // ||w|| -> R diag, 1/||w|| or lucky
  FIN_GM_COEF,     // projections -> coef[], R column
  FIN_GM_XI,       // xi_i, step += 1
  FIN_DOTV,        // dotv = stage2(p_bb)  (true residual; p_bb is free after setup)
};

enum Gate : int32_t {
  GATE_NONE = 0,      // always run
  GATE_RUNNING = 1,   // run while status == RUNNING
  GATE_TAIL = 2,      // run while status <= STOPPING (BiCGStab xrp)
  GATE_GMRES = 3,     // run while status == RUNNING and not lucky
};

__device__ __forceinline__ void set_cond(SolveState* st, unsigned v) {
  if (st->use_cond) cudaGraphSetConditional(st->cond, v);
}

__device__ __forceinline__ bool gate_open(SolveState* st, int gate) {
  if (gate == GATE_NONE || st == nullptr) return true;
  int s = *(volatile int32_t*)&st->status;
  bool open;
  if (gate == GATE_TAIL) open = s <= STOPPING;
  else if (gate == GATE_GMRES) open = (s == RUNNING) && !*(volatile int32_t*)&st->lucky;
  else open = (s == RUNNING);
  if (!open && blockIdx.x == 0 && threadIdx.x == 0) set_cond(st, 0);
  return open;
}

__device__ __forceinline__ double msqrt(double v) { return __dsqrt_rn(v); }

__device__ inline void finalize(SolveState* st, int fin, int arg) {
  const int th = threadIdx.x;
  const int ng = st->n_groups;
  __shared__ double tot[32];
  switch (fin) {
    case FIN_CG_SETUP:
    case FIN_CG_ITER: {
      if (th == 0) tot[0] = stage2_col(st->p_rr, ng, 1, 0);
      if (th == 1) tot[1] = stage2_col(st->p_two, ng, 2, 0);
      if (th == 2) tot[2] = stage2_col(st->p_two, ng, 2, 1);
      if (fin == FIN_CG_SETUP && th == 3) tot[3] = stage2_col(st->p_bb, ng, 1, 0);
      __syncthreads();
      if (th != 0) return;
      double rr = tot[0], pap = tot[1], apap = tot[2];
      st->rr = rr; st->pap = pap; st->apap = apap;
      bool stop = false;
      if (fin == FIN_CG_SETUP) {
        double nb = msqrt(tot[3]);
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
        if (fin == FIN_CG_ITER && st->iter >= st->limit) { st->term = PK_TERM_MAX_ITER; stop = true; }
      }
      st->status = stop ? STOPPED : RUNNING;
      set_cond(st, stop ? 0u : 1u);
      break;
    }
    case FIN_BICG_SETUP: {
      if (th == 0) tot[0] = stage2_col(st->p_rr, ng, 1, 0);
      if (th == 1) tot[1] = stage2_col(st->p_bb, ng, 1, 0);
      __syncthreads();
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
      set_cond(st, stop ? 0u : 1u);
      break;
    }
    case FIN_BICG_ALPHA: {
      if (th == 0) tot[0] = stage2_col(st->p_rr, ng, 1, 0);
      if (th == 1) tot[1] = stage2_col(st->p_apr, ng, 1, 0);
      __syncthreads();
      if (th != 0) return;
      double rho = tot[0], d = tot[1];
      st->rho0 = rho;
      st->apr = d;
      if (fabs(d) < st->btol_loop) {
        st->term = PK_TERM_BREAKDOWN; st->kind = PK_BK_APR0STAR;
        st->status = STOPPED;
        set_cond(st, 0u);
      } else {
        st->alpha = div_rn(rho, d);
      }
      break;
    }
    case FIN_BICG_TAIL: {
      if (th == 0) tot[0] = stage2_col(st->p_ss, ng, 1, 0);
      if (th >= 1 && th <= 3) tot[th] = stage2_col(st->p_tri, ng, 3, th - 1);
      __syncthreads();
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
      set_cond(st, status == RUNNING ? 1u : 0u);
      break;
    }
    case FIN_GM_RHO: {
      if (th == 0) tot[0] = stage2_col(st->p_rr, ng, 1, 0);
      if (th == 1 && arg) tot[1] = stage2_col(st->p_bb, ng, 1, 0);
      __syncthreads();
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
      if (th == 0) {
        double nrm = msqrt(stage2_col(st->p_ww, ng, 1, 0));
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
      // arg = step index i (>= 2): columns 0..i-2 of p_coef
      for (int j = th; j < arg - 1; j += blockDim.x) {
        double c = stage2_col(st->p_coef, ng, st->m, j);
        st->coef[j] = c;
        st->R[(int64_t)j * st->m + (arg - 1)] = c;
      }
      break;
    }
    case FIN_GM_XI: {
      if (th == 0) {
        st->xi[arg - 1] = stage2_col(st->p_xi + (int64_t)(arg - 1) * ng, ng, 1, 0);
        st->step = arg;
      }
      break;
    }
    case FIN_DOTV: {
      if (th == 0) st->dotv = stage2_col(st->p_bb, ng, 1, 0);
      break;
    }
    default:
      break;
  }
}

// Device scalar sources for an op: the solver points these at SolveState
// fields written by the previous finalizer; kernel-level entries leave them
// null and pass values.
struct ScalarPtrs {
  const double* a;
  const double* b;
  const double* c;
};

__device__ __forceinline__ double ld_scalar(const double* p, double v) { return p ? __ldcg(p) : v; }

// ---------------------------------------------------------------------------
// CSR row gather
// ---------------------------------------------------------------------------

template <typename RowT, int W>
struct RowRegs {
  RowT beg, end;
  double v[W];
  double xv[W];
};

template <typename RowT>
struct Csr {
  const RowT* rp;
  const int32_t* ci;
  const double* va;
};

template <typename RowT, int W>
__device__ __forceinline__ void row_load(const Csr<RowT>& A, const double* __restrict__ x, int64_t row,
                                         RowRegs<RowT, W>& it) {
  it.beg = __ldg(A.rp + row);
  it.end = __ldg(A.rp + row + 1);
#pragma unroll
  for (int s = 0; s < W; ++s) {
    RowT e = it.beg + s;
    if (e < it.end) {
      int32_t c = __ldg(A.ci + e);
      it.v[s] = __ldg(A.va + e);
      it.xv[s] = __ldg(x + c);
    }
  }
}

template <typename RowT, int W>
__device__ __forceinline__ double row_finish(const Csr<RowT>& A, const double* __restrict__ x,
                                             const RowRegs<RowT, W>& it) {
  double acc = 0.0;
#pragma unroll
  for (int s = 0; s < W; ++s) {
    if (it.beg + s < it.end) acc = add_rn(acc, mul_rn(it.v[s], it.xv[s]));
  }
  for (RowT e = it.beg + W; e < it.end; ++e) acc = add_rn(acc, mul_rn(__ldg(A.va + e), __ldg(x + __ldg(A.ci + e))));
  return acc;
}

// ---------------------------------------------------------------------------
// elementwise operators
// ---------------------------------------------------------------------------

// q = A p with NQ fused dots (fused.py:86-120).
template <typename RowT, int W, int NQ>
struct OpSpmvFused {
  Csr<RowT> A;
  const double* __restrict__ p;
  double* __restrict__ q;
  int32_t kind[4];
  const double* w[4];
  struct Item {
    RowRegs<RowT, W> r;
    double pv;
    double wv[NQ > 0 ? NQ : 1];
  };
  __device__ __forceinline__ void load(int64_t row, Item& it) const {
    row_load<RowT, W>(A, p, row, it.r);
    bool need_p = false;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      if (kind[k] == PK_DOT_INPUT) need_p = true;
      if (kind[k] == PK_DOT_VECTOR) it.wv[k] = __ldg(w[k] + row);
    }
    if (need_p) it.pv = __ldg(p + row);
  }
  __device__ __forceinline__ void compute(int64_t row, Item& it, double (&c)[NQ > 0 ? NQ : 1]) const {
    double acc = row_finish<RowT, W>(A, p, it.r);
    if (q) q[row] = acc;
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      c[k] = kind[k] == PK_DOT_INPUT ? mul_rn(acc, it.pv)
           : kind[k] == PK_DOT_RESULT ? mul_rn(acc, acc) : mul_rn(acc, it.wv[k]);
    }
  }
  __device__ __forceinline__ void apply(int64_t row, Item& it) const {
    q[row] = row_finish<RowT, W>(A, p, it.r);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// r = b + (-1) A x (add_scaled, linalg.py:450-457); optional copies; <r,r>.
template <typename RowT, int W>
struct OpResidual {
  Csr<RowT> A;
  const double* __restrict__ x;
  const double* __restrict__ b;
  double* r;
  double* copy1;
  double* copy2;
  struct Item {
    RowRegs<RowT, W> r;
    double bv;
  };
  __device__ __forceinline__ void load(int64_t row, Item& it) const {
    row_load<RowT, W>(A, x, row, it.r);
    it.bv = __ldg(b + row);
  }
  __device__ __forceinline__ void compute(int64_t row, Item& it, double (&c)[1]) const {
    double q = row_finish<RowT, W>(A, x, it.r);
    double rv = add_rn(it.bv, mul_rn(-1.0, q));
    if (r) r[row] = rv;
    if (copy1) copy1[row] = rv;
    if (copy2) copy2[row] = rv;
    c[0] = mul_rn(rv, rv);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};


// fused_cg_vector_update (fused.py:123-151)
struct OpCgUpdate {
  double* x;
  double* r;
  double* p;
  const double* __restrict__ ap;
  double alpha, beta;
  struct Item { double x, r, p, ap; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const {
    it.x = x[i]; it.r = r[i]; it.p = p[i]; it.ap = __ldg(ap + i);
  }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[1]) const {
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
  const double* __restrict__ r;
  const double* __restrict__ ap;
  double* s;
  double alpha;
  struct Item { double r, ap; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const { it.r = __ldg(r + i); it.ap = __ldg(ap + i); }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[1]) const {
    double sv = sub_rn(it.r, mul_rn(alpha, it.ap));
    s[i] = sv;
    c[0] = mul_rn(sv, sv);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) { alpha = ld_scalar(sp.a, alpha); }
};

// fused_bicgstab_xrp_update (fused.py:185-219)
struct OpBicgXrp {
  double* x;
  double* r;
  double* p;
  const double* __restrict__ s;
  const double* __restrict__ ap;
  const double* __restrict__ as;
  const double* __restrict__ r0;
  double alpha, omega, beta;
  struct Item { double x, p, s, ap, as, r0; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const {
    it.x = x[i]; it.p = p[i]; it.s = __ldg(s + i); it.ap = __ldg(ap + i); it.as = __ldg(as + i); it.r0 = __ldg(r0 + i);
  }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[1]) const {
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
  const double* __restrict__ x;
  const double* __restrict__ y;
  struct Item { double x, y; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const { it.x = __ldg(x + i); it.y = __ldg(y + i); }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[1]) const { c[0] = mul_rn(it.x, it.y); }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// NQ precomputed contribution columns (reduce_stage1 of stacked streams).
template <int NQ>
struct OpColumns {
  const double* col[NQ];
  struct Item { double v[NQ]; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const {
#pragma unroll
    for (int k = 0; k < NQ; ++k) it.v[k] = __ldg(col[k] + i);
  }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[NQ]) const {
#pragma unroll
    for (int k = 0; k < NQ; ++k) c[k] = it.v[k];
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// fused_gs_stage1 (fused.py:222-243): <b_j, v> for j < nb (nb <= NB).
template <int NB>
struct OpMultiDot {
  const double* __restrict__ v;
  int32_t nb;
  const double* b[NB];
  struct Item { double v; double b[NB]; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const {
    it.v = __ldg(v + i);
#pragma unroll
    for (int j = 0; j < NB; ++j) if (j < nb) it.b[j] = __ldg(b[j] + i);
  }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[NB]) const {
#pragma unroll
    for (int j = 0; j < NB; ++j) c[j] = j < nb ? mul_rn(it.b[j], it.v) : 0.0;
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs&) {}
};

// fused_gs_update (fused.py:246-277): v -= sum_j c_j b_j; <v,v>.
template <int NB>
struct OpGsUpdate {
  double* v;
  int32_t nb;
  const double* b[NB];
  double c[NB];
  struct Item { double v; double b[NB]; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const {
    it.v = v[i];
#pragma unroll
    for (int j = 0; j < NB; ++j) if (j < nb) it.b[j] = __ldg(b[j] + i);
  }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&cc)[1]) const {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < NB; ++j) if (j < nb) acc = add_rn(acc, mul_rn(c[j], it.b[j]));
    double vn = nb > 0 ? sub_rn(it.v, acc) : it.v;
    v[i] = vn;
    cc[0] = mul_rn(vn, vn);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) {
    if (sp.a) {
#pragma unroll
      for (int j = 0; j < NB; ++j) c[j] = j < nb ? __ldcg(sp.a + j) : 0.0;
    }
  }
};

// fused_gs_normalize (fused.py:280-305): v *= inv; <r, v>.
struct OpNormalize {
  double* v;
  const double* __restrict__ r;
  double inv;
  struct Item { double v, r; };
  __device__ __forceinline__ void load(int64_t i, Item& it) const { it.v = v[i]; it.r = __ldg(r + i); }
  __device__ __forceinline__ void compute(int64_t i, Item& it, double (&c)[1]) const {
    double vn = mul_rn(it.v, inv);
    v[i] = vn;
    c[0] = mul_rn(it.r, vn);
  }
  __device__ __forceinline__ void scalars(const ScalarPtrs& sp) { inv = ld_scalar(sp.a, inv); }
};

}  // namespace pk
