// Device-resident solver state: the scalar block read by every kernel's
// prologue and written by the last-CTA finalizers.  One per solve.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "pipekrylov_b200.h"

namespace pk {

enum Status : int32_t { RUNNING = 0, STOPPING = 1, STOPPED = 2 };

struct SolveState {
  // configuration (written by the host before the loop)
  double tol;
  double btol_loop;   // 0 in fixed-iteration mode (solvers.py:141-145)
  double btol_cfg;    // always SolverConfig.breakdown_tolerance
  int64_t limit;      // iteration limit (fixed or max)
  int32_t fixed;
  int32_t n_groups;
  int32_t use_cond;   // 1 when running inside a conditional-while graph
  int32_t pad0;
  cudaGraphConditionalHandle cond;

  // progress
  int64_t iter;       // completed iterations (history length)
  int32_t status;
  int32_t term;       // PK_TERM_*
  int32_t kind;       // PK_BK_*
  int32_t clamped;
  int32_t need_check; // BiCGStab: identity clamped and monitor below tol
  int32_t half_step;  // BiCGStab: converged on the half step
  int32_t lucky;      // GMRES: lucky breakdown inside the cycle
  int32_t step;       // GMRES: completed steps in the current cycle
  int32_t parity;     // current half of the ping-pong vector pairs
  int32_t pad3;

  // scalars
  double scale;       // ||b|| or 1
  double rr, pap, apap, alpha, beta, omega;
  double ss, ass, asas, asr, apr, rho0;
  double nrm, inv;    // GMRES normalisation
  double dotv;        // generic finalized dot / true residual squared
  double ident;       // BiCGStab: residual identity before the clamp (debug diagnostics)
  double rho;         // GMRES cycle residual norm

  unsigned int ticket;
  unsigned int pad1;

  // buffers (device pointers)
  double* hist;       // history, capacity limit + 1
  double* p_bb;       // [ng]       <b,b>
  double* p_rr;       // [ng]       <r,r> / <r,r0*> (CG rr, BiCG rr0)
  double* p_two;      // [ng x 2]   CG {pAp, ApAp}
  double* p_apr;      // [ng]       BiCG <Ap, r0*>
  double* p_ss;       // [ng]       BiCG <s,s>
  double* p_tri;      // [ng x 3]   BiCG {As.s, As.As, As.r0*}
  double* p_ww;       // [ng]       GMRES <w,w>
  double* p_three;    // [ng x 3]   fused CG {rr, pAp, ApAp}
  double* p_pair;     // [ng x 2]   BiCG {<r,r0*>, <Ap,r0*>}
  double* p_quad;     // [ng x 4]   BiCG {ss, As.s, As.As, As.r0*}
  double* p_coef;     // [ng x m]   GMRES projections (older basis + newest)
  double* p_xi;       // [m x ng]   GMRES <r, v_i> per step
  double* coef;       // [m]        finalized projection coefficients
  double* R;          // [m x m]    GMRES triangular factor, row major
  double* xi;         // [m]        finalized xi
  int32_t m;          // GMRES restart length
  int32_t pad2;
};

}  // namespace pk
