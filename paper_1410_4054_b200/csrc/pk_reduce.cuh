// Ordered two-stage reduction engine for sm_100a.
//
// Reproduces the reference's reduction schedule bit-for-bit
// (pipekrylov/linalg.py:289-320):
//   stage 1: lane t = ((0 + c[t]) + c[t+G]) + c[t+2G] + ...  (G = n_groups*gs)
//            then per group of gs lanes a halving tree buf[l] += buf[l+s].
//   stage 2: serial left-to-right sum over groups.
//
// Mapping.  One CTA owns one group at a time (persistent loop over groups).
// The CTA has T = min(gs, Tmax) threads; thread th owns the m = gs/T lanes
// {th, th+T, th+2T, ...} of its group.  The halving tree over gs lanes
// splits into (a) a tree over each thread's m lanes -- the subtree of lanes
// congruent to th mod T -- and (b) a halving tree across the T threads.
// (a) is evaluated by visiting the thread's lanes in bit-reversed order and
// merging with a binary-counter stack (only tree shape matters; binary64
// addition is commutative), so it needs O(log m) storage instead of m.
// Within a lane the k-chunks are visited in increasing k, as the reference
// does.  Every tile touched by a CTA is T consecutive rows, so all global
// traffic is coalesced.
//
// All arithmetic uses explicit __dadd_rn/__dmul_rn (never contracted into
// DFMA); the library is additionally compiled with -fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace pk {

struct Geom {
  int64_t n;         // number of elements (rows)
  int64_t G;         // n_groups * gs
  int32_t n_groups;
  int32_t gs;        // group size (power of two)
  int32_t T;         // threads per CTA (power of two, <= gs)
  int32_t m;         // leaves (lanes) per thread = gs / T
  int32_t logm;
  uint32_t Keff;     // max(ceil(n / G), 1) chunks per lane
};

__host__ __device__ inline int ilog2_u(uint32_t v) {
  int r = 0;
  while ((1u << r) < v) ++r;
  return r;
}

inline Geom make_geom(int64_t n, int32_t n_groups, int32_t gs, int32_t tmax) {
  Geom g;
  g.n = n;
  g.n_groups = n_groups;
  g.gs = gs;
  g.G = (int64_t)n_groups * gs;
  g.T = gs < tmax ? gs : tmax;
  g.m = gs / g.T;
  g.logm = ilog2_u((uint32_t)g.m);
  int64_t k = (n + g.G - 1) / g.G;
  g.Keff = (uint32_t)(k < 1 ? 1 : k);
  return g;
}

__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// Row index of (leaf position i, chunk k) for thread th of group g.
__device__ __forceinline__ int64_t item_row(const Geom& geo, int g, uint32_t i, uint32_t k, int th) {
  uint32_t j = geo.logm ? (__brev(i) >> (32 - geo.logm)) : 0u;
  return (int64_t)k * geo.G + (int64_t)g * geo.gs + (int64_t)j * geo.T + th;
}

// Cross-thread halving tree (levels s = T/2 .. 1).  v[q] in, result valid in
// thread 0.  sbuf must hold NQ*T doubles.  All threads of the CTA call it.
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
    const unsigned mask = (T >= 32) ? 0xffffffffu : ((1u << T) - 1u);
    for (; s >= 1; s >>= 1) {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        double o = __shfl_down_sync(mask, v[q], s);
        if (th < s) v[q] = add_rn(v[q], o);
      }
    }
  }
}

// Leaf accumulator for one thread: binary-counter stack in shared memory
// (stk holds (logm+1)*NQ*T doubles).  push() takes the leaf at position i.
template <int NQ>
struct LeafStack {
  double* stk;
  int T;
  __device__ __forceinline__ void push(uint32_t i, double (&v)[NQ], double (&out)[NQ]) {
    const int th = threadIdx.x;
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

// Shared-memory bytes the engine needs for a given geometry.
inline size_t engine_smem_bytes(const Geom& geo, int nq) {
  size_t tree = (size_t)nq * geo.T * sizeof(double);
  size_t stack = geo.m > 1 ? (size_t)(geo.logm + 1) * nq * geo.T * sizeof(double) : 0;
  return tree + stack;
}

// Run the ordered stage-1 reduction of group g with elementwise operator op.
// Op must provide:
//   struct Item;                                        per-row registers
//   void load(int64_t row, Item&)                       issue loads
//   void compute(int64_t row, Item&, double (&c)[NQ])   compute, store, emit contributions
// Out-of-range rows (row >= n) contribute 0.0, which leaves a lane unchanged
// (a lane starts at +0.0 and can never become -0.0).
template <int NQ, int U, class Op>
__device__ __forceinline__ void run_group(const Geom& geo, int g, Op& op, double* smem,
                                          double (&lane)[NQ]) {
  const int th = threadIdx.x;
  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) { acc[q] = 0.0; lane[q] = 0.0; }
  LeafStack<NQ> st{smem + NQ * geo.T, geo.T};
  const uint32_t total = (uint32_t)geo.m * geo.Keff;
  uint32_t i = 0, k = 0;
  for (uint32_t it0 = 0; it0 < total; it0 += U) {
    typename Op::Item items[U];
    int64_t rows[U];
    {
      uint32_t ii = i, kk = k;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        int64_t row = item_row(geo, g, ii, kk, th);
        rows[u] = (it0 + u < total && row < geo.n) ? row : -1;
        if (rows[u] >= 0) op.load(rows[u], items[u]);
        if (++kk == geo.Keff) { kk = 0; ++ii; }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (it0 + u < total) {
        double c[NQ];
        if (rows[u] >= 0) {
          op.compute(rows[u], items[u], c);
        } else {
#pragma unroll
          for (int q = 0; q < NQ; ++q) c[q] = 0.0;
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = add_rn(acc[q], c[q]);
        if (++k == geo.Keff) {
          k = 0;
          if (geo.m > 1) {
            st.push(i, acc, lane);
          } else {
#pragma unroll
            for (int q = 0; q < NQ; ++q) lane[q] = acc[q];
          }
#pragma unroll
          for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
          ++i;
        }
      }
    }
  }
}

// Full stage-1 over all groups handled by this CTA; writes
// part[g * ld + col0 + q] for q < nstore.  Returns after the CTA's last group.
template <int NQ, int U, class Op>
__device__ __forceinline__ void stage1_all_groups(const Geom& geo, Op& op, double* smem,
                                                  double* part, int ld, int col0, int nstore) {
  for (int g = blockIdx.x; g < geo.n_groups; g += gridDim.x) {
    double lane[NQ];
    run_group<NQ, U>(geo, g, op, smem, lane);
    block_tree<NQ>(lane, smem, geo.T);
    if (threadIdx.x == 0 && part) {
      // only the nstore live quantities: templates padded to NQ (e.g. a
      // multi-dot over nb < NB vectors) must not spill into other columns
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (q < nstore) part[(int64_t)g * ld + col0 + q] = lane[q];
    }
    __syncthreads();  // smem (tree + stack) reused by the next group
  }
}

// Elementwise-only sweep (no reduction) using the same tile order; used by
// kernels that only update vectors.
template <int U, class Op>
__device__ __forceinline__ void sweep_all(int64_t n, Op& op) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; base < n; base += stride * U) {
    typename Op::Item items[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t row = base + (int64_t)u * stride;
      if (row < n) op.load(row, items[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t row = base + (int64_t)u * stride;
      if (row < n) op.apply(row, items[u]);
    }
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

// Last-CTA election for epilogue finalizers.  All threads call; returns true
// in every thread of the last CTA to finish.  Resets the ticket.
__device__ __forceinline__ bool elect_last_block(unsigned int* ticket) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1 : 0;
    if (s_last) {
      *ticket = 0u;
      __threadfence();
    }
  }
  __syncthreads();
  return s_last != 0;
}

}  // namespace pk
