// Ordered two-stage reduction engine for sm_100a.
//
// Reproduces the reference's reduction schedule bit-for-bit
// (pipekrylov/linalg.py:289-320):
//   stage 1: lane t = ((0 + c[t]) + c[t+G]) + c[t+2G] + ...   (G = n_groups*gs)
//            then per group of gs lanes a halving tree buf[l] += buf[l+s].
//   stage 2: serial left-to-right sum over groups.
//
// Only the ORDER of the additions is prescribed; the contributions c[i]
// themselves are independent, so every row is computed by its own thread
// with plain, lean, high-occupancy code (thread-per-row SpMV, CSR and vectors
// straight through L1/L2 -- measured at 5.7-6.8 TB/s on B200 for the
// BiCGStab-shaped row), and only the folding is ordered:
//   phase A  the 8 warps of a CTA each compute U rows (32-row tiles) and park
//            their contributions in shared memory;
//   phase B  warp 0 (the "lane threads", one lane each) folds them into its
//            running lane values in the exact reference order.
//
// Two mappings, chosen per launch from (n, n_groups, group_size):
//   CHAIN (K = ceil(n/G) >= 2, or group_size < 32): a CTA owns a block of 32
//            consecutive lane ids of [0, G) and walks the K chunks
//            (rows k*G + lane), 8U chunks per batch.  Lane values go to a
//            small spill buffer (G x nq doubles); the last CTA of a group
//            (per-group ticket) runs the group's halving tree.
//   LEAF  (K = 1, group_size >= 32): a CTA owns a group; lane thread th owns
//            the lanes {th + 32 j}, whose sub-tree is evaluated by visiting
//            j in bit-reversed order through a binary-counter stack (only
//            tree shape matters -- binary64 addition is commutative).
// The last group to finish (global ticket) runs the serial stage 2 and the
// solver's scalar recurrences (pk_kernels.cuh finalize()).
//
// All arithmetic uses explicit __dadd_rn/__dmul_rn (never contracted into
// DFMA); the library is additionally compiled with -fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#ifndef PK_SWEEP_V
#define PK_SWEEP_V 4
#endif

namespace pk {

constexpr int kWarps = 8;  // warps of an engine CTA
constexpr int kThreads = kWarps * 32;
constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ inline int ilog2_u(uint32_t v) {
  int r = 0;
  while ((1u << r) < v) ++r;
  return r;
}

struct Geom {
  int64_t n;       // rows
  int64_t G;       // n_groups * gs
  int64_t K;       // chunks per lane, max(ceil(n / G), 1)
  int64_t units;   // CHAIN: ceil(G / 32) lane blocks; LEAF: n_groups
  int32_t n_groups;
  int32_t gs;
  int32_t leaf;    // 1 = LEAF mapping
  int32_t m;       // LEAF: leaves per lane thread (gs / 32)
  int32_t logm;
  int32_t logf;    // LEAF: a group is split over F = 2^logf CTAs (units = ne F [+ 1])
  int32_t ne;      // LEAF: groups holding at least one row (ceil(n / gs), <= n_groups); the
                   // rest are all-zero and published by one extra zero-fill unit
  int32_t tT;      // CHAIN group tree: threads = min(gs, kThreads)
  int32_t tm;      // CHAIN group tree: leaves per tree thread
  int32_t tlogm;
  int32_t staged;  // CHAIN + SpMV operator: engine_chain_staged (column indices staged by cp.async)
};

// min_units: LEAF groups are split over F = 2^logf CTAs (each a contiguous
// range of bit-reversed visits = a complete sub-tree) until n_groups F >=
// min_units, so that few large groups still fill the GPU.
// chain_only: CHAIN mapping even for K = 1 (the warp engine's single-chunk
// lanes: lane value = 0.0 + c, exactly the reference's zeros + chunk).
inline Geom make_geom(int64_t n, int32_t n_groups, int32_t gs, int64_t min_units = 0, bool chain_only = false) {
  Geom g{};
  g.n = n;
  g.n_groups = n_groups;
  g.gs = gs;
  g.G = (int64_t)n_groups * gs;
  int64_t k = (n + g.G - 1) / g.G;
  g.K = k < 1 ? 1 : k;
  g.leaf = (g.K == 1 && gs >= 32 && !chain_only) ? 1 : 0;
  if (g.leaf) {
    g.m = gs / 32;
    g.logm = ilog2_u((uint32_t)g.m);
    const int64_t ne = (n + gs - 1) / gs;
    g.ne = (int32_t)(ne < n_groups ? ne : n_groups);
    g.logf = 0;
    while ((int64_t)g.ne << g.logf < min_units && (1 << (g.logf + 1)) <= g.m) ++g.logf;
    g.units = ((int64_t)g.ne << g.logf) + (g.ne < n_groups ? 1 : 0);
  } else {
    g.units = (g.G + 31) / 32;
    g.tT = gs < kThreads ? gs : kThreads;
    g.tm = gs / g.tT;
    g.tlogm = ilog2_u((uint32_t)g.tm);
  }
  return g;
}

// Dynamic shared memory of one engine kernel (doubles):
//   C     [2][kWarps U][nq][32]  parked contributions (double-buffered)
//   tail  LEAF: stack (logm+1) x nq x 32;  CHAIN: tree nq x tT + stack
__host__ __device__ inline size_t engine_tail_doubles(const Geom& g, int nq) {
  return g.leaf ? (g.m > 1 ? (size_t)(g.logm + 1) * nq * 32 : 0)
                : (size_t)nq * g.tT + (g.tm > 1 ? (size_t)(g.tlogm + 1) * nq * g.tT : 0);
}
__host__ __device__ inline size_t engine_smem_bytes(const Geom& g, int nq, int U) {
  return ((size_t)2 * kWarps * U * nq * 32 + engine_tail_doubles(g, nq)) * sizeof(double);
}

__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// Scratch shared by the engine kernels of one context (stream-ordered).
struct Scratch {
  double* spill;      // CHAIN lane values, [nq][G]
  unsigned* gtick;    // per-group tickets [n_groups], self-resetting
  unsigned* ticket;   // global ticket (kernel-level entries; solvers use SolveState)
};

// CSR triple on the device, optionally with a SELL-32 copy of the same
// entries (sp != nullptr): rows are cut into slices of 32 consecutive rows,
// slice s holds its rows' entries slot-major -- slot j of row 32 s + l at
// sp[s] + 32 j + l, the slice padded to its longest row with column -1 (and
// value 0) -- so the 32 lanes of a warp walking 32 aligned rows read slot j
// as one 128-byte (columns) / 256-byte (values) segment instead of 32
// stride-5 scattered words, and need one row-bounds load per warp (sp[s],
// sp[s + 1]) instead of one per row.  Entries keep their stored order, so
// the row sums (and every bit of the result) are those of the CSR loop.
template <typename RowT_, bool SELL_ = false>
struct Csr {
  using RowT = RowT_;
  static constexpr bool kSell = SELL_;  // walk the SELL-32 copy (compile-time: the CSR code stays as lean as before)
  const RowT* rp;
  const int32_t* ci;
  const double* va;
  const RowT* sp = nullptr;   // SELL-32 slice offsets (entries), n_slices + 1
  const int32_t* sc = nullptr;
  const double* sv = nullptr;
  int32_t blk = -1;           // host: most entries in an aligned 32-row block (BULK engine slot size), -1 unknown
  int32_t maxr = 0;           // host: longest row
  int32_t vec = 0;            // host: long-row matrix -- SpMV row sums by the warp-cooperative VEC pre-pass
};

// [b, e) walk of a row and the slot stride: CSR (rp[row], rp[row + 1], 1) or
// SELL-32 (sp[s] + lane, sp[s + 1], 32).
template <typename RowT, bool SELL>
__device__ __forceinline__ void row_span(const Csr<RowT, SELL>& A, uint32_t row, RowT& b, RowT& e) {
  if constexpr (SELL) {
    const uint32_t sl = row >> 5;
    b = __ldg(A.sp + sl) + (RowT)(row & 31u);
    e = __ldg(A.sp + sl + 1);
  } else {
    b = __ldg(A.rp + row);
    e = __ldg(A.rp + row + 1);
  }
}

// ---------------------------------------------------------------------------
// phase A: the contributions of one row (lean thread-per-row code)
// ---------------------------------------------------------------------------
//
// Operator concept (pk_kernels.cuh):
//   static constexpr bool kSpmv;  static constexpr int kMinBlocks;  struct Item;
//   void load(uint32_t row, Item&)                 per-row vector loads
//   kSpmv:  using RowT; Csr<RowT> A; static constexpr int kSlots;
//           struct Gat; void gload(uint32_t col, Gat&)   raw words at col
//           double gval(const Gat&)                      SpMV input value (may recompute)
//           void compute(uint32_t row, Item&, double q, double (&c)[NQ])
//   else:   void compute(uint32_t row, Item&, double (&c)[NQ])
//   void scalars(const ScalarPtrs&)                 prologue: device scalars
//
// SpMV rows are summed acc = ((0 + v0 x0) + v1 x1) + ... in stored order
// (_spmvkernels.py:12-18).  kSlots entries per pass: all loads of a pass are
// issued first (slots past the row end re-read its last entry -- always a
// valid address -- and are not added), then the ordered adds.
template <class Op, class = void>
struct RowBounds { using T = int32_t; };
template <class Op>
struct RowBounds<Op, std::void_t<typename Op::RowT>> { using T = typename Op::RowT; };

// rb_pre/re_pre: the row's CSR bounds when already loaded (software
// pipelining across batches), else rb_pre > re_pre (load them here)
template <int NQ, class Op>
__device__ __forceinline__ void row_contrib(const Op& op, uint32_t row, double (&c)[NQ],
                                            typename RowBounds<Op>::T rb_pre = 1,
                                            typename RowBounds<Op>::T re_pre = 0) {
  typename Op::Item it;
  op.load(row, it);
  if constexpr (Op::kSpmv) {
    using RowT = typename Op::RowT;
    constexpr int S = Op::kSlots;
    const bool have = rb_pre <= re_pre;
    RowT b = rb_pre, e = re_pre;
    if (!have) row_span(op.A, row, b, e);
    constexpr bool sell = std::decay_t<decltype(op.A)>::kSell;
    const RowT st = sell ? 32 : 1;
    const int32_t* __restrict__ ci = sell ? op.A.sc : op.A.ci;
    const double* __restrict__ va = sell ? op.A.sv : op.A.va;
    double acc = 0.0;
    for (RowT k0 = b; k0 < e; k0 += S * st) {
      int32_t col[S];
      double val[S];
      typename Op::Gat gv[S];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const RowT k = (k0 + j * st < e) ? k0 + j * st : b;  // past the end: re-read a valid slot
        col[j] = __ldg(ci + k);
        val[j] = __ldg(va + k);
      }
#pragma unroll
      for (int j = 0; j < S; ++j) op.gload((uint32_t)(sell && col[j] < 0 ? 0 : col[j]), gv[j]);
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (k0 + j * st < e && (!sell || col[j] >= 0)) acc = add_rn(acc, mul_rn(val[j], op.gval(gv[j])));
    }
    op.compute(row, it, acc, c);
  } else {
    op.compute(row, it, c);
  }
}

// ---------------------------------------------------------------------------
// tree helpers
// ---------------------------------------------------------------------------

// Cross-thread halving tree (levels s = T/2 .. 1) over threads 0..T-1.
// v[q] in, result valid in thread 0.  sbuf holds NQ*T doubles.  All threads
// of the CTA call it.
template <int NQ>
__device__ __forceinline__ void block_tree(double (&v)[NQ], double* sbuf, int T) {
  const int th = threadIdx.x;
  int s = T >> 1;
  for (; s >= 32; s >>= 1) {
    if (th < 2 * s) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) sbuf[q * T + th] = v[q];
    }
    __syncthreads();
    if (th < s) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = add_rn(v[q], sbuf[q * T + th + s]);
    }
    __syncthreads();
  }
  if (th < 32 && s >= 1) {
    const unsigned mask = (T >= 32) ? kFull : ((1u << T) - 1u);
    for (; s >= 1; s >>= 1) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double o = __shfl_down_sync(mask, v[q], s);
        if (th < s) v[q] = add_rn(v[q], o);
      }
    }
  }
}

// Binary-counter leaf stack in shared memory (stk holds (logm+1)*NQ*T
// doubles).  push() takes the leaf visited i-th; after the last leaf of a
// power-of-two count `out` holds the whole sub-tree.
template <int NQ>
struct LeafStack {
  double* stk;
  int T;
  int th;
  __device__ __forceinline__ void push(uint32_t i, double (&v)[NQ], double (&out)[NQ]) {
    int lvl = 0;
    for (uint32_t c = i; c & 1u; c >>= 1, ++lvl) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = add_rn(stk[(lvl * NQ + q) * T + th], v[q]);
    }
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      stk[(lvl * NQ + q) * T + th] = v[q];
      out[q] = v[q];
    }
  }
};

__device__ __forceinline__ uint32_t brev_bits(uint32_t i, int bits) {
  return bits ? (__brev(i) >> (32 - bits)) : 0u;
}

// Halving tree of group g over its gs spilled lane values (CHAIN mapping).
template <int NQ>
__device__ __forceinline__ void group_tree(const Geom& geo, int g, const double* spill, double* tail, double* part,
                                        int ld, int col0, int nstore) {
  const int th = threadIdx.x;
  const int T = geo.tT;
  double v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = 0.0;
  if (th < T) {
    const int64_t base = (int64_t)g * geo.gs + th;
    if (geo.tm == 1) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = q < nstore ? __ldcg(spill + (int64_t)q * geo.G + base) : 0.0;
    } else {
      LeafStack<NQ> st{tail + NQ * T, T, th};
      // leaves loaded 4 at a time (one L2 round trip per batch), pushed in visit order
      constexpr int BL = 4;
      for (uint32_t i0 = 0; i0 < (uint32_t)geo.tm; i0 += BL) {
        double x[BL][NQ];
#pragma unroll
        for (int b = 0; b < BL; ++b) {
          const uint32_t i = i0 + b;
          const int64_t idx = base + (int64_t)brev_bits(i < (uint32_t)geo.tm ? i : 0u, geo.tlogm) * T;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            x[b][q] = (q < nstore && i < (uint32_t)geo.tm) ? __ldcg(spill + (int64_t)q * geo.G + idx) : 0.0;
        }
#pragma unroll
        for (int b = 0; b < BL; ++b)
          if (i0 + b < (uint32_t)geo.tm) st.push(i0 + b, x[b], v);
      }
    }
  }
  block_tree<NQ>(v, tail, T);
  if (th == 0 && part) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q < nstore) part[(int64_t)g * ld + col0 + q] = v[q];
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// the engine
// ---------------------------------------------------------------------------

// Ticket increment with release semantics at gpu scope (MEMBAR + ATOM): it
// publishes this CTA's spill / partials before the ticket moves.  The CTA
// that draws the LAST ticket then executes acquire_fence() before it reads
// the others' data (with L2 loads, ld.global.cg) -- only there, because the
// acquire half emits an L1 invalidation (CCTL.IVALL) that would otherwise
// throw away the L1-resident CSR lines of every warp on the SM at every
// ticket.  Other threads of that CTA (warp) read after a barrier (shuffle)
// that orders them behind the fencing thread.
__device__ __forceinline__ unsigned ticket_add(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.add.release.gpu.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void acquire_fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Scalar binary-counter leaf push for quantity q (stk laid out as LeafStack).
template <int NQ>
__device__ __forceinline__ double leaf_push(double* stk, int q, int lane, uint32_t i, double v) {
  int lvl = 0;
  for (uint32_t c = i; c & 1u; c >>= 1, ++lvl) v = add_rn(stk[(lvl * NQ + q) * 32 + lane], v);
  stk[(lvl * NQ + q) * 32 + lane] = v;
  return v;
}

// Runs stage 1 of this CTA's units and writes part[g * ld + col0 + q] for
// q < nstore.  Returns true in every thread of the CTA that completed the
// last group (the finalizer CTA).
//
// Per batch (B = kWarps U chunks / leaves): every thread computes U rows and
// parks the contributions in C[batch & 1]; ONE barrier; then warp w folds
// quantities q = w, w + kWarps, ... of the batch in the reference order while
// the other warps already compute the next batch into the other half of C
// (the barrier of the next batch orders the reuse).
template <int NQ, int U, class Op>
__device__ __forceinline__ bool engine_run(const Geom& geo, const Op& op, double* smem, double* part, int ld,
                                           int col0, int nstore, const Scratch& scr, unsigned* ticket) {
  __shared__ int s_flag;
  __shared__ int s_last;
  constexpr int B = kWarps * U;                   // chunks (CHAIN) / leaves (LEAF) per batch
  constexpr int QPW = (NQ + kWarps - 1) / kWarps; // quantities folded per warp
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  double* Cbuf = smem;  // [2][B][NQ][32]
  double* tail = Cbuf + 2 * B * NQ * 32;
  if (tid == 0) s_last = 0;
  uint32_t bpar = 0;  // which half of C the next batch writes

  for (int64_t unit = blockIdx.x; unit < geo.units; unit += gridDim.x) {
    int ncomplete = 0;
    if (!geo.leaf) {
      // ---- CHAIN: 32 lane ids [lid0, lid0 + nl), chunks k = 0..K-1 ----
      const int64_t lid0 = unit * 32;
      const int nl = (int)((geo.G - lid0) < 32 ? (geo.G - lid0) : 32);
      const bool lane_ok = lane < nl;
      double acc[QPW];
#pragma unroll
      for (int i = 0; i < QPW; ++i) acc[i] = 0.0;
      using RB = typename RowBounds<Op>::T;
      RB nb[U], ne[U];  // CSR bounds of this warp's rows in the next batch
#pragma unroll
      for (int u = 0; u < U; ++u) { nb[u] = 1; ne[u] = 0; }
      for (int64_t k0 = 0; k0 < geo.K; k0 += B) {
        double* C = Cbuf + (bpar & 1u) * (B * NQ * 32);
        ++bpar;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = warp + kWarps * u;
          const int64_t row = (k0 + kk) * geo.G + lid0 + lane;
          double c[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) c[q] = 0.0;
          if (k0 + kk < geo.K && lane_ok && row < geo.n) row_contrib<NQ>(op, (uint32_t)row, c, nb[u], ne[u]);
#pragma unroll
          for (int q = 0; q < NQ; ++q) C[(kk * NQ + q) * 32 + lane] = c[q];
        }
        if constexpr (Op::kSpmv) {
          // software pipelining: the next batch's row bounds load during the
          // barrier and the fold (one dependent DRAM round trip less per row)
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t kn = k0 + B + warp + kWarps * u;
            const int64_t rn = kn * geo.G + lid0 + lane;
            nb[u] = 1;
            ne[u] = 0;
            if (kn < geo.K && lane_ok && rn < geo.n) row_span(op.A, (uint32_t)rn, nb[u], ne[u]);
          }
        }
        __syncthreads();
        const int kend = (int)((geo.K - k0) < B ? (geo.K - k0) : B);
#pragma unroll
        for (int i = 0; i < QPW; ++i) {
          const int q = warp + kWarps * i;
          if (q < NQ) {
            double v[B];
#pragma unroll
            for (int kk = 0; kk < B; ++kk) v[kk] = C[(kk * NQ + q) * 32 + lane];
#pragma unroll
            for (int kk = 0; kk < B; ++kk)
              if (kk < kend) acc[i] = add_rn(acc[i], v[kk]);
          }
        }
      }
      if (lane_ok) {
#pragma unroll
        for (int i = 0; i < QPW; ++i) {
          const int q = warp + kWarps * i;
          if (q < NQ && q < nstore) scr.spill[(int64_t)q * geo.G + lid0 + lane] = acc[i];
        }
      }
      __syncthreads();
      if (geo.gs >= 32) {
        const int g = (int)(lid0 / geo.gs);
        if (tid == 0) {
          const unsigned per = (unsigned)(geo.gs / 32);
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
    } else {
      if (unit >= ((int64_t)geo.ne << geo.logf)) {
        // the zero-fill unit: groups [ne, n_groups) lie wholly past n; their
        // tree of +0.0 lanes is +0.0 (linalg.py:299-307 starts from zeros)
        if (part)
          for (int64_t t = tid; t < (int64_t)(geo.n_groups - geo.ne) * nstore; t += kThreads)
            part[(int64_t)(geo.ne + t / nstore) * ld + col0 + t % nstore] = 0.0;
        ncomplete = geo.n_groups - geo.ne;
      } else {
      // ---- LEAF: group g, part cp of F; the folding lane owns lanes {lane + 32 j} ----
      const int g = (int)(unit >> geo.logf);
      const int F = 1 << geo.logf;
      const int cp = (int)(unit & (F - 1));
      const int msub = geo.m >> geo.logf;  // visits of this part: [cp msub, (cp + 1) msub)
      if ((int64_t)g * geo.gs >= geo.n) {
        // empty group (every lane past n): its tree of +0.0 lanes is +0.0
        // (linalg.py:299-307 starts the lanes from zeros); part 0 publishes it
        if (cp == 0 && part && tid < nstore) part[(int64_t)g * ld + col0 + tid] = 0.0;
        ncomplete = cp == 0 ? 1 : 0;
      } else {
      double out[QPW];
#pragma unroll
      for (int i = 0; i < QPW; ++i) out[i] = 0.0;
      for (int i0 = 0; i0 < msub; i0 += B) {
        double* C = Cbuf + (bpar & 1u) * (B * NQ * 32);
        ++bpar;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ii = warp + kWarps * u;
          const int i = cp * msub + i0 + ii;
          const int64_t row = (int64_t)g * geo.gs + (int64_t)brev_bits((uint32_t)i, geo.logm) * 32 + lane;
          double c[NQ];
#pragma unroll
          for (int q = 0; q < NQ; ++q) c[q] = 0.0;
          if (i0 + ii < msub && row < geo.n) row_contrib<NQ>(op, (uint32_t)row, c);
#pragma unroll
          for (int q = 0; q < NQ; ++q) C[(ii * NQ + q) * 32 + lane] = c[q];
        }
        __syncthreads();
        const int iend = (msub - i0) < B ? (msub - i0) : B;
#pragma unroll
        for (int w = 0; w < QPW; ++w) {
          const int q = warp + kWarps * w;
          if (q < NQ) {
            for (int ii = 0; ii < iend; ++ii) {
              const double x = C[(ii * NQ + q) * 32 + lane];
              out[w] = msub > 1 ? leaf_push<NQ>(tail, q, lane, (uint32_t)(i0 + ii), x) : x;
            }
          }
        }
      }
      bool fin_group = true;
      if (F > 1) {
        // publish this part's sub-tree roots; the last part of the group
        // merges the F roots in visit order (binary counter = halving tree)
#pragma unroll
        for (int w = 0; w < QPW; ++w) {
          const int q = warp + kWarps * w;
          if (q < NQ) scr.spill[((unit * NQ) + q) * 32 + lane] = out[w];
        }
        __syncthreads();
        if (tid == 0) {
          unsigned tk = ticket_add(scr.gtick + g, 1u);
          int lastp = (tk == (unsigned)F - 1);
          if (lastp) {
            scr.gtick[g] = 0u;
            acquire_fence();
          }
          s_flag = lastp;
        }
        __syncthreads();
        fin_group = s_flag != 0;
        if (fin_group) {
#pragma unroll
          for (int w = 0; w < QPW; ++w) {
            const int q = warp + kWarps * w;
            if (q < NQ) {
              for (int c2 = 0; c2 < F; ++c2) {
                const int64_t u2 = ((int64_t)g << geo.logf) + c2;
                const double x = __ldcg(scr.spill + ((u2 * NQ) + q) * 32 + lane);
                out[w] = leaf_push<NQ>(tail, q, lane, (uint32_t)c2, x);
              }
            }
          }
        }
      }
      if (fin_group) {
#pragma unroll
        for (int w = 0; w < QPW; ++w) {
          const int q = warp + kWarps * w;
          if (q < NQ) {
            double o = out[w];
#pragma unroll
            for (int sft = 16; sft >= 1; sft >>= 1) {
              double t = __shfl_down_sync(kFull, o, sft);
              if (lane < sft) o = add_rn(o, t);
            }
            if (lane == 0 && part && q < nstore) part[(int64_t)g * ld + col0 + q] = o;
          }
        }
      }
      ncomplete = fin_group ? 1 : 0;
      }
      }
    }
    // ---- global ticket: the CTA completing the last group finalizes ----
    if (ncomplete > 0) {
      __syncthreads();
      if (tid == 0) {
        unsigned tk = ticket_add(ticket, (unsigned)ncomplete);
        if (tk + (unsigned)ncomplete == (unsigned)geo.n_groups) {
          *ticket = 0u;
          acquire_fence();
          s_last = 1;
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
  return s_last != 0;
}

// ---------------------------------------------------------------------------
// CHAIN engine with staged column indices (SpMV operators)
// ---------------------------------------------------------------------------
//
// Same mapping, fold order, spill / ticket / group-tree protocol as the CHAIN
// branch of engine_run(); what changes is how a row's inputs arrive.  The
// column indices of the first pass (kSlots entries) of every row of batch
// t + 1 are copied global -> shared with cp.async (4-byte LDGSTS, zero-fill
// past the row end: no registers held, no read) while batch t folds, and the
// row bounds are loaded two batches ahead; the CTA's batches are one
// flattened stream across its units, so the pipeline does not drain at unit
// boundaries.  A batch's critical path is then shared-memory columns ->
// gathers (values and the row's own vectors load beside the gathers) instead
// of row bounds -> columns -> gathers.  Same contributions, same order: the
// same bits.

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(gsrc), "r"(valid ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__host__ __device__ inline size_t staged_extra_bytes(int U, int S) { return (size_t)U * S * kThreads * 4; }

// Row contribution with the first pass's columns taken from shared memory
// (cs[j * kThreads], this thread's slots); longer rows continue from global.
template <int NQ, class Op>
__device__ __forceinline__ void row_contrib_staged(const Op& op, uint32_t row, double (&c)[NQ],
                                                   typename Op::RowT b, typename Op::RowT e, const int32_t* cs) {
  using RowT = typename Op::RowT;
  constexpr int S = Op::kSlots;
  typename Op::Item it;
  op.load(row, it);
  constexpr bool sell = std::decay_t<decltype(op.A)>::kSell;
  const RowT st = sell ? 32 : 1;
  const int32_t* __restrict__ ci = sell ? op.A.sc : op.A.ci;
  const double* __restrict__ va = sell ? op.A.sv : op.A.va;
  double acc = 0.0;
  for (RowT k0 = b; k0 < e; k0 += S * st) {
    int32_t col[S];
    double val[S];
    typename Op::Gat gv[S];
    const bool first = k0 == b;
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const RowT k = (k0 + j * st < e) ? k0 + j * st : b;
      col[j] = first ? cs[j * kThreads] : __ldg(ci + k);
      val[j] = __ldg(va + k);
    }
#pragma unroll
    for (int j = 0; j < S; ++j) op.gload((uint32_t)(sell && col[j] < 0 ? 0 : col[j]), gv[j]);
#pragma unroll
    for (int j = 0; j < S; ++j)
      if (k0 + j * st < e && (!sell || col[j] >= 0)) acc = add_rn(acc, mul_rn(val[j], op.gval(gv[j])));
  }
  op.compute(row, it, acc, c);
}

// row of batch t (of this CTA's flattened (unit, batch) stream), slot u of this thread, or -1
__device__ __forceinline__ int64_t staged_row(const Geom& geo, int64_t T, int64_t nbpu, int B, int64_t t, int u,
                                             int warp, int lane) {
  if (t >= T) return -1;
  const int64_t unit = (int64_t)blockIdx.x + (t / nbpu) * gridDim.x;
  const int64_t k = (t % nbpu) * B + warp + kWarps * u;
  const int64_t lid0 = unit * 32;
  if (k >= geo.K || lid0 + lane >= geo.G) return -1;
  const int64_t row = k * geo.G + lid0 + lane;
  return row < geo.n ? row : -1;
}

template <int NQ, int U, class Op>
__device__ __forceinline__ bool engine_chain_staged(const Geom& geo, const Op& op, double* smem, double* part, int ld,
                                                    int col0, int nstore, const Scratch& scr, unsigned* ticket) {
  using RowT = typename Op::RowT;
  constexpr int S = Op::kSlots;
  __shared__ int s_flag;
  __shared__ int s_last;
  constexpr int B = kWarps * U;
  constexpr int QPW = (NQ + kWarps - 1) / kWarps;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  double* Cbuf = smem;  // [2][B][NQ][32]
  double* tail = Cbuf + 2 * B * NQ * 32;
  int32_t* cst = reinterpret_cast<int32_t*>(tail + engine_tail_doubles(geo, NQ));  // [U][S][kThreads]
  if (tid == 0) s_last = 0;
  constexpr bool sell = std::decay_t<decltype(op.A)>::kSell;
  const RowT st = sell ? 32 : 1;
  const int32_t* __restrict__ ci = sell ? op.A.sc : op.A.ci;
  const int64_t nbpu = (geo.K + B - 1) / B;  // batches per unit
  const int64_t my_units =
      geo.units > (int64_t)blockIdx.x ? (geo.units - 1 - (int64_t)blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t T = my_units * nbpu;
#define PK_STG_BOUNDS(t_, bb, ee)                                                   \
  _Pragma("unroll") for (int u = 0; u < U; ++u) {                                   \
    bb[u] = 1;                                                                      \
    ee[u] = 0;                                                                      \
    const int64_t r_ = staged_row(geo, T, nbpu, B, (t_), u, warp, lane);            \
    if (r_ >= 0) row_span(op.A, (uint32_t)r_, bb[u], ee[u]);                        \
  }
#define PK_STG_STAGE(bb, ee)                                                        \
  _Pragma("unroll") for (int u = 0; u < U; ++u) {                                   \
    _Pragma("unroll") for (int j = 0; j < S; ++j) {                                 \
      const RowT k_ = bb[u] + j * st;                                               \
      const bool v_ = bb[u] <= ee[u] && k_ < ee[u];                                 \
      cp_async4(cst + (u * S + j) * kThreads + tid, v_ ? ci + k_ : ci, v_);         \
    }                                                                               \
  }                                                                                 \
  cp_async_commit();
  RowT cb[U], ce[U], nb[U], ne[U], fb[U], fe[U];
  PK_STG_BOUNDS(0, cb, ce)
  PK_STG_BOUNDS(1, nb, ne)
  PK_STG_STAGE(cb, ce)
  double acc[QPW];
#pragma unroll
  for (int i = 0; i < QPW; ++i) acc[i] = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    PK_STG_BOUNDS(t + 2, fb, fe)
    cp_async_wait_all();
    double* C = Cbuf + (t & 1) * (B * NQ * 32);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int kk = warp + kWarps * u;
      const int64_t row = staged_row(geo, T, nbpu, B, t, u, warp, lane);
      double c[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) c[q] = 0.0;
      if (row >= 0) row_contrib_staged<NQ>(op, (uint32_t)row, c, cb[u], ce[u], cst + u * S * kThreads + tid);
#pragma unroll
      for (int q = 0; q < NQ; ++q) C[(kk * NQ + q) * 32 + lane] = c[q];
    }
    PK_STG_STAGE(nb, ne)
    __syncthreads();
    const int64_t unit = (int64_t)blockIdx.x + (t / nbpu) * gridDim.x;
    const int64_t k0 = (t % nbpu) * B;
    const int kend = (int)((geo.K - k0) < B ? (geo.K - k0) : B);
#pragma unroll
    for (int i = 0; i < QPW; ++i) {
      const int q = warp + kWarps * i;
      if (q < NQ) {
        double v[B];
#pragma unroll
        for (int kk = 0; kk < B; ++kk) v[kk] = C[(kk * NQ + q) * 32 + lane];
#pragma unroll
        for (int kk = 0; kk < B; ++kk)
          if (kk < kend) acc[i] = add_rn(acc[i], v[kk]);
      }
    }
    if (t % nbpu == nbpu - 1) {
      // ---- unit epilogue: lane values -> spill, group ticket / tree, global ticket ----
      const int64_t lid0 = unit * 32;
      const int nl = (int)((geo.G - lid0) < 32 ? (geo.G - lid0) : 32);
      if (lane < nl) {
#pragma unroll
        for (int i = 0; i < QPW; ++i) {
          const int q = warp + kWarps * i;
          if (q < NQ && q < nstore) scr.spill[(int64_t)q * geo.G + lid0 + lane] = acc[i];
        }
      }
#pragma unroll
      for (int i = 0; i < QPW; ++i) acc[i] = 0.0;
      __syncthreads();
      const int g = (int)(lid0 / geo.gs);
      if (tid == 0) {
        const unsigned per = (unsigned)(geo.gs / 32);
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
        if (tid == 0) {
          unsigned tk = ticket_add(ticket, 1u);
          if (tk + 1u == (unsigned)geo.n_groups) {
            *ticket = 0u;
            acquire_fence();
            s_last = 1;
          }
        }
        __syncthreads();
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      cb[u] = nb[u]; ce[u] = ne[u];
      nb[u] = fb[u]; ne[u] = fe[u];
    }
  }
#undef PK_STG_BOUNDS
#undef PK_STG_STAGE
  cp_async_wait_all();
  __syncthreads();
  return s_last != 0;
}

// Warp-level halving tree of group g over its gs (>= 32) spilled lane values:
// lane l owns the lanes {l + 32 j}, visited in bit-reversed order of j
// through a binary-counter stack (stk: (log2(gs/32)+1) x NQ x 32 doubles),
// then a shuffle tree across the 32 lanes.
template <int NQ>
__device__ __forceinline__ void group_tree_warp(const Geom& geo, int g, const double* spill, double* stk,
                                                double* part, int ld, int col0, int nstore) {
  const int lane = threadIdx.x & 31;
  double v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = 0.0;
  const int64_t base = (int64_t)g * geo.gs;
  const int mm = geo.gs / 32;
  const int lg = ilog2_u((uint32_t)mm);
  LeafStack<NQ> st{stk, 32, lane};
  // the leaves' loads go out in batches of 8 (one L2 round trip per batch,
  // not per leaf), then the pushes in visit order
  constexpr int BL = 8;
  for (int i0 = 0; i0 < mm; i0 += BL) {
    double x[BL][NQ];
#pragma unroll
    for (int b = 0; b < BL; ++b) {
      const int i = i0 + b;
      const int64_t idx = base + (int64_t)brev_bits((uint32_t)(i < mm ? i : 0), lg) * 32 + lane;
#pragma unroll
      for (int q = 0; q < NQ; ++q) x[b][q] = (q < nstore && i < mm) ? __ldcg(spill + (int64_t)q * geo.G + idx) : 0.0;
    }
#pragma unroll
    for (int b = 0; b < BL; ++b) {
      const int i = i0 + b;
      if (i >= mm) break;
      if (mm > 1) {
        st.push((uint32_t)i, x[b], v);
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[q] = x[b][q];
      }
    }
  }
#pragma unroll
  for (int sft = 16; sft >= 1; sft >>= 1) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double o = __shfl_down_sync(kFull, v[q], sft);
      if (lane < sft) v[q] = add_rn(v[q], o);
    }
  }
  if (lane == 0 && part) {
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q < nstore) part[(int64_t)g * ld + col0 + q] = v[q];
  }
  __syncwarp();
}

inline size_t warp_chain_smem_bytes(const Geom& g, int nq) {
  return (size_t)(ilog2_u((uint32_t)(g.gs / 32)) + 1) * nq * 32 * sizeof(double);
}

// ---------------------------------------------------------------------------
// warp-per-unit CHAIN engine (no shared memory, no CTA barrier)
// ---------------------------------------------------------------------------
//
// R rows of one lane chain, computed with interleaved loads (R independent
// row chains in flight per thread): contributions c[r][q] of rows
// (k0 + r) G + lid0 + lane, r < R; rows outside the matrix contribute 0.
template <int NQ, int R, class Op>
__device__ __forceinline__ void rows_contrib(const Op& op, const Geom& geo, int64_t k0, int64_t lid0, bool lane_ok,
                                             double (&c)[R][NQ]) {
  const int lane = threadIdx.x & 31;
  bool ok[R];
  uint32_t row[R];
  typename Op::Item it[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t rw = (k0 + r) * geo.G + lid0 + lane;
    ok[r] = lane_ok && (k0 + r) < geo.K && rw < geo.n;
    row[r] = ok[r] ? (uint32_t)rw : 0u;
#pragma unroll
    for (int q = 0; q < NQ; ++q) c[r][q] = 0.0;
  }
  if constexpr (Op::kSpmv) {
    using RowT = typename Op::RowT;
    constexpr int S = Op::kSlots;
    RowT b[R], e[R];
    constexpr bool sell = std::decay_t<decltype(op.A)>::kSell;
    const RowT st = sell ? 32 : 1;
    const int32_t* __restrict__ ci = sell ? op.A.sc : op.A.ci;
    const double* __restrict__ va = sell ? op.A.sv : op.A.va;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      b[r] = 0;
      e[r] = 0;
      if (ok[r]) {
        row_span(op.A, row[r], b[r], e[r]);
        op.load(row[r], it[r]);
      }
    }
    // first S entries of every row: all loads in flight, then the ordered adds
    int32_t col[R][S];
    double val[R][S];
    typename Op::Gat gv[R][S];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < S; ++j) {
        const RowT k = (b[r] + j * st < e[r]) ? b[r] + j * st : b[r];
        const bool live = e[r] > b[r];
        col[r][j] = live ? __ldg(ci + k) : 0;
        val[r][j] = live ? __ldg(va + k) : 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int j = 0; j < S; ++j) op.gload((uint32_t)(sell && col[r][j] < 0 ? 0 : col[r][j]), gv[r][j]);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < S; ++j)
        if (b[r] + j * st < e[r] && (!sell || col[r][j] >= 0)) acc = add_rn(acc, mul_rn(val[r][j], op.gval(gv[r][j])));
      // rows longer than S: the rest in order, straight from memory
      for (RowT k = b[r] + S * st; k < e[r]; k += st) {
        const int32_t cj = __ldg(ci + k);
        if (sell && cj < 0) continue;
        typename Op::Gat g;
        op.gload((uint32_t)cj, g);
        acc = add_rn(acc, mul_rn(__ldg(va + k), op.gval(g)));
      }
      if (ok[r]) op.compute(row[r], it[r], acc, c[r]);
    }
  } else {
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (ok[r]) op.load(row[r], it[r]);
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (ok[r]) op.compute(row[r], it[r], c[r]);
  }
}

// One warp per unit of 32 lane ids (CHAIN mapping, group_size >= 32): the warp
// walks the unit's K chunks R at a time and folds each lane's chain in
// registers in the reference order; the warp that completes a group runs the
// group's halving tree (warp-level); the warp completing the last group is
// the finalizer.  Returns true in that warp.
template <int NQ, int R, class Op>
__device__ __forceinline__ bool engine_warp_chain(const Geom& geo, const Op& op, double* stk, double* part, int ld,
                                                  int col0, int nstore, const Scratch& scr, unsigned* ticket) {
  const int lane = threadIdx.x & 31;
  const int wpc = blockDim.x >> 5;
  const int64_t w0 = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * wpc;
  bool last = false;
  for (int64_t unit = w0; unit < geo.units; unit += nw) {
    const int64_t lid0 = unit * 32;
    const int nl = (int)((geo.G - lid0) < 32 ? (geo.G - lid0) : 32);
    const bool lane_ok = lane < nl;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    for (int64_t k0 = 0; k0 < geo.K; k0 += R) {
      double c[R][NQ];
      rows_contrib<NQ, R>(op, geo, k0, lid0, lane_ok, c);
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (k0 + r < geo.K) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[q] = add_rn(acc[q], c[r][q]);
        }
    }
    if (lane_ok) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) scr.spill[(int64_t)q * geo.G + lid0 + lane] = acc[q];
    }
    __syncwarp();
    const int g = (int)(lid0 / geo.gs);
    int lastg = 0;
    if (lane == 0) {
      const unsigned per = (unsigned)(geo.gs / 32);
      unsigned tk = ticket_add(scr.gtick + g, 1u);
      lastg = (tk == per - 1);
      if (lastg) {
        scr.gtick[g] = 0u;
        acquire_fence();
      }
    }
    lastg = __shfl_sync(kFull, lastg, 0);
    if (lastg) {
      group_tree_warp<NQ>(geo, g, scr.spill, stk, part, ld, col0, nstore);
      int l = 0;
      if (lane == 0) {
        unsigned tk = ticket_add(ticket, 1u);
        if (tk + 1u == (unsigned)geo.n_groups) {
          *ticket = 0u;
          acquire_fence();
          l = 1;
        }
      }
      if (__shfl_sync(kFull, l, 0)) last = true;
    }
  }
  return last;
}

// ---------------------------------------------------------------------------
// LANE engine: elementwise operators (no SpMV) on CHAIN geometries (K >= 2)
// ---------------------------------------------------------------------------
//
// One thread per reduction lane t of [0, G): the thread walks its own chain
// rows t, t + G, t + 2G, ... (each warp's 32 rows of a chunk are consecutive
// lanes: coalesced) and folds the contributions in registers in chunk order
// -- exactly linalg.py:300-303 -- with the loads of D chunks issued before
// their folds.  Elementwise rows have no dependent loads, so nothing needs
// staging: no shared-memory fold, no per-batch barrier.  A CTA of T = min(gs,
// kLaneThreads) lanes evaluates the group's halving tree itself when it holds
// the whole group (T == gs); otherwise lane values go to the spill buffer and
// the CTA completing the group runs group_tree().  Global ticket + finalizer as
// in engine_run().
#ifndef PK_LANE_THREADS
#define PK_LANE_THREADS 256
#endif
constexpr int kLaneThreads = PK_LANE_THREADS;

__host__ __device__ inline int lane_cta_threads(const Geom& g) { return g.gs < kLaneThreads ? g.gs : kLaneThreads; }

template <int NQ, int D, class Op>
__device__ __forceinline__ bool engine_lane(const Geom& geo, const Op& op, double* smem, double* part, int ld,
                                            int col0, int nstore, const Scratch& scr, unsigned* ticket) {
  __shared__ int s_flag;
  __shared__ int s_last;
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t t = (int64_t)blockIdx.x * T + tid;  // lane id
  const bool lane_ok = t < geo.G;
  if (tid == 0) s_last = 0;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  if (lane_ok) {
    for (int64_t k0 = 0; k0 < geo.K; k0 += D) {
      typename Op::Item it[D];
      int64_t row[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        row[d] = (k0 + d) * geo.G + t;
        const int64_t rc = row[d] < geo.n ? row[d] : t;  // clamped: every load unconditional
        op.load((uint32_t)rc, it[d]);
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        if (k0 + d < geo.K && row[d] < geo.n) {
          double c[NQ];
          op.compute((uint32_t)row[d], it[d], c);
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[q] = add_rn(acc[q], c[q]);
        }
      }
    }
  }
  const int g = (int)((int64_t)blockIdx.x * T / geo.gs);
  if (T == geo.gs) {
    // the CTA holds the whole group: its halving tree (linalg.py:304-307) here
    block_tree<NQ>(acc, smem, T);
    if (tid == 0 && part) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) part[(int64_t)g * ld + col0 + q] = acc[q];
    }
    __syncthreads();
    if (tid == 0) {
      unsigned tk = ticket_add(ticket, 1u);
      if (tk + 1u == (unsigned)geo.n_groups) {
        *ticket = 0u;
        acquire_fence();
        s_last = 1;
      }
    }
  } else {
    if (lane_ok) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) scr.spill[(int64_t)q * geo.G + t] = acc[q];
    }
    __syncthreads();
    if (tid == 0) {
      const unsigned per = (unsigned)(geo.gs / T);
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
      group_tree<NQ>(geo, g, scr.spill, smem, part, ld, col0, nstore);
      if (tid == 0) {
        unsigned tk = ticket_add(ticket, 1u);
        if (tk + 1u == (unsigned)geo.n_groups) {
          *ticket = 0u;
          acquire_fence();
          s_last = 1;
        }
      }
    }
  }
  __syncthreads();
  return s_last != 0;
}

// ---------------------------------------------------------------------------
// LANE engine for SpMV operators: a software-pipelined lane chain
// ---------------------------------------------------------------------------
//
// Thread = reduction lane t, walking its chain rows kG + t (k = 0..K-1; a
// warp's 32 rows of a chunk are consecutive: coalesced) and folding the
// contributions in registers in chunk order.  A row's loads form a dependent
// chain (row bounds -> columns/values -> gathered inputs), so the chain is
// software-pipelined three deep: in every round the thread
//   (1) folds the P chunks whose gathers were issued in the previous round,
//   (2) issues the gathers of the P chunks whose columns arrived,
//   (3) issues the column/value/own-vector loads of the P chunks whose bounds
//       arrived, and
//   (4) issues the row-bound loads of P new chunks,
// so 3P chunks are in flight per thread and a round waits for ONE memory
// latency instead of three, with no shared-memory fold and no barrier.  Rows
// longer than kSlots finish their remaining entries at fold time.  A CTA of
// T = min(gs, 256) lanes runs the group tree itself when it holds the whole
// group; otherwise spill + group ticket as in engine_lane().
template <int NQ, int P, class Op>
__device__ __forceinline__ bool engine_lane_spmv(const Geom& geo, const Op& op, double* smem, double* part, int ld,
                                                 int col0, int nstore, const Scratch& scr, unsigned* ticket) {
  using RowT = typename Op::RowT;
  constexpr int S = Op::kSlots;
  constexpr bool sell = std::decay_t<decltype(op.A)>::kSell;
  const RowT st = sell ? 32 : 1;
  const int32_t* __restrict__ ci = sell ? op.A.sc : op.A.ci;
  const double* __restrict__ va = sell ? op.A.sv : op.A.va;
  __shared__ int s_flag;
  __shared__ int s_last;
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  const int64_t t = (int64_t)blockIdx.x * T + tid;
  const bool lane_ok = t < geo.G;
  if (tid == 0) s_last = 0;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  // stage A: row bounds; B: columns, values, own-row item; C: gathered inputs
  RowT aB[P], aE[P], bB[P], bE[P], cB[P], cE[P];
  int32_t bC[P][S], cC[P][S];
  double bV[P][S], cV[P][S];
  typename Op::Item bI[P], cI[P];
  typename Op::Gat cG[P][S];
  int64_t aR[P], bR[P], cR[P];  // rows (-1: no row)
#pragma unroll
  for (int p = 0; p < P; ++p) { aR[p] = bR[p] = cR[p] = -1; }
  const int64_t R = lane_ok ? (geo.K + P - 1) / P : 0;
  for (int64_t r = 0; r < R + 3; ++r) {
    // (1) fold stage C (chunks of round r - 3), in chunk order
#pragma unroll
    for (int p = 0; p < P; ++p) {
      if (cR[p] >= 0) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < S; ++j)
          if (cB[p] + j * st < cE[p] && (!sell || cC[p][j] >= 0)) a = add_rn(a, mul_rn(cV[p][j], op.gval(cG[p][j])));
        for (RowT k = cB[p] + S * st; k < cE[p]; k += st) {  // rows longer than kSlots
          const int32_t cj = __ldg(ci + k);
          if (sell && cj < 0) continue;
          typename Op::Gat g;
          op.gload((uint32_t)cj, g);
          a = add_rn(a, mul_rn(__ldg(va + k), op.gval(g)));
        }
        double c[NQ];
        op.compute((uint32_t)cR[p], cI[p], a, c);
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = add_rn(acc[q], c[q]);
      }
    }
    // (2) stage B -> C: gathers
#pragma unroll
    for (int p = 0; p < P; ++p) {
      cR[p] = bR[p];
      cB[p] = bB[p];
      cE[p] = bE[p];
      cI[p] = bI[p];
#pragma unroll
      for (int j = 0; j < S; ++j) {
        cC[p][j] = bC[p][j];
        cV[p][j] = bV[p][j];
        if (cR[p] >= 0) op.gload((uint32_t)(sell && cC[p][j] < 0 ? 0 : cC[p][j]), cG[p][j]);
      }
    }
    // (3) stage A -> B: columns, values, own-row loads
#pragma unroll
    for (int p = 0; p < P; ++p) {
      bR[p] = aR[p];
      bB[p] = aB[p];
      bE[p] = aE[p];
      if (bR[p] >= 0) {
        op.load((uint32_t)bR[p], bI[p]);
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const RowT k = (bB[p] + j * st < bE[p]) ? bB[p] + j * st : bB[p];
          const bool live = bE[p] > bB[p];
          bC[p][j] = live ? __ldg(ci + k) : 0;  // an empty row gathers a valid column and adds nothing
          bV[p][j] = live ? __ldg(va + k) : 0.0;
        }
      }
    }
    // (4) new chunks -> stage A: row bounds
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const int64_t k = r * P + p;
      const int64_t row = k * geo.G + t;
      aR[p] = (r < R && k < geo.K && row < geo.n) ? row : -1;
      aB[p] = 1;
      aE[p] = 0;
      if (aR[p] >= 0) row_span(op.A, (uint32_t)row, aB[p], aE[p]);
    }
  }
  const int g = (int)((int64_t)blockIdx.x * T / geo.gs);
  if (T == geo.gs) {
    block_tree<NQ>(acc, smem, T);
    if (tid == 0 && part) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) part[(int64_t)g * ld + col0 + q] = acc[q];
    }
    __syncthreads();
    if (tid == 0) {
      unsigned tk = ticket_add(ticket, 1u);
      if (tk + 1u == (unsigned)geo.n_groups) {
        *ticket = 0u;
        acquire_fence();
        s_last = 1;
      }
    }
  } else {
    if (lane_ok) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) scr.spill[(int64_t)q * geo.G + t] = acc[q];
    }
    __syncthreads();
    if (tid == 0) {
      const unsigned per = (unsigned)(geo.gs / T);
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
      group_tree<NQ>(geo, g, scr.spill, smem, part, ld, col0, nstore);
      if (tid == 0) {
        unsigned tk = ticket_add(ticket, 1u);
        if (tk + 1u == (unsigned)geo.n_groups) {
          *ticket = 0u;
          acquire_fence();
          s_last = 1;
        }
      }
    }
  }
  __syncthreads();
  return s_last != 0;
}

// Grid-stride thread-per-row sweep (no reduction): plain SpMV / updates.
template <class Op>
__device__ __forceinline__ void sweep_rows(int64_t n, const Op& op) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if constexpr (!Op::kSpmv) {
    // SWEEP_V rows per thread in flight (all loads issued before any compute)
    constexpr int V = PK_SWEEP_V;
    for (; row + (V - 1) * stride < n; row += V * stride) {
      typename Op::Item it[V];
#pragma unroll
      for (int v = 0; v < V; ++v) op.load((uint32_t)(row + v * stride), it[v]);
#pragma unroll
      for (int v = 0; v < V; ++v) {
        double c[1];
        op.compute((uint32_t)(row + v * stride), it[v], c);
      }
    }
  }
  for (; row < n; row += stride) {
    double c[1];
    row_contrib<1>(op, (uint32_t)row, c);
  }
}

// Serial stage 2 (linalg.py:311-320) for quantity column col of a partials
// array with leading dimension ld.  Executed by a single thread.
__device__ __forceinline__ double stage2_col(const double* part, int n_groups, int ld, int col) {
  double tot = 0.0;
  int g = 0;
  for (; g + 8 <= n_groups; g += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(part + (int64_t)(g + u) * ld + col);
#pragma unroll
    for (int u = 0; u < 8; ++u) tot = add_rn(tot, v[u]);
  }
  for (; g < n_groups; ++g) tot = add_rn(tot, __ldcg(part + (int64_t)g * ld + col));
  return tot;
}

}  // namespace pk
