// Ordered two-stage reduction engine for sm_100a (v2: staged, chunk-parallel).
//
// Reproduces the reference's reduction schedule bit-for-bit
// (pipekrylov/linalg.py:289-320):
//   stage 1: lane t = ((0 + c[t]) + c[t+G]) + c[t+2G] + ...   (G = n_groups*gs)
//            then per group of gs lanes a halving tree buf[l] += buf[l+s].
//   stage 2: serial left-to-right sum over groups.
//
// Only the ORDER of the additions is prescribed; the contributions c[i]
// themselves are independent.  The engine therefore splits every kernel in
// two phases per batch:
//   phase A  all 8 warps of the CTA compute contributions of 32-row tiles
//            (coalesced, CSR products staged through shared memory) and park
//            them in shared memory -- this is where the memory-level
//            parallelism comes from;
//   phase B  warp 0 (the "lane threads", one lane each) folds the parked
//            contributions into its running lane values in the exact
//            reference order.
//
// Two mappings, chosen per launch from (n, n_groups, group_size):
//   CHAIN (K = ceil(n/G) >= 2, or group_size < 32): a CTA owns a block of 32
//            consecutive lane ids of [0, G) and walks the K chunks
//            (rows k*G + lane); the 8 warps take 8 chunks per batch.  Lane
//            values go to a small spill buffer (G x nq doubles); the last CTA
//            of a group (per-group ticket) runs the group's halving tree.
//            The default reference geometry 128 x 256 runs here with
//            G/32 = 1024 CTAs instead of 128.
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

namespace pk {

constexpr int kThreads = 256;  // CTA size of every engine kernel
constexpr int kWarps = kThreads / 32;
constexpr int kPCap = 256;     // staged CSR products per warp tile
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
  int32_t tT;      // CHAIN group tree: threads = min(gs, kThreads)
  int32_t tm;      // CHAIN group tree: leaves per tree thread
  int32_t tlogm;
};

inline Geom make_geom(int64_t n, int32_t n_groups, int32_t gs) {
  Geom g{};
  g.n = n;
  g.n_groups = n_groups;
  g.gs = gs;
  g.G = (int64_t)n_groups * gs;
  int64_t k = (n + g.G - 1) / g.G;
  g.K = k < 1 ? 1 : k;
  g.leaf = (g.K == 1 && gs >= 32) ? 1 : 0;
  if (g.leaf) {
    g.m = gs / 32;
    g.logm = ilog2_u((uint32_t)g.m);
    g.units = n_groups;
  } else {
    g.units = (g.G + 31) / 32;
    g.tT = gs < kThreads ? gs : kThreads;
    g.tm = gs / g.tT;
    g.tlogm = ilog2_u((uint32_t)g.tm);
  }
  return g;
}

// Dynamic shared memory (doubles) of one engine kernel.
//   C     [8U][nq][32]  parked contributions
//   P     [8][kPCap]    CSR products (SpMV operators only)
//   tail  LEAF: stack (logm+1) x nq x 32;  CHAIN: tree nq x tT + stack
inline size_t engine_smem_bytes(const Geom& g, int nq, int U, bool spmv) {
  size_t c = (size_t)kWarps * U * nq * 32;
  size_t p = spmv ? (size_t)kWarps * kPCap : 0;
  size_t t;
  if (g.leaf) {
    t = g.m > 1 ? (size_t)(g.logm + 1) * nq * 32 : 0;
  } else {
    t = (size_t)nq * g.tT + (g.tm > 1 ? (size_t)(g.tlogm + 1) * nq * g.tT : 0);
  }
  return (c + p + t) * sizeof(double);
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

// CSR triple on the device.
template <typename RowT_>
struct Csr {
  using RowT = RowT_;
  const RowT* rp;
  const int32_t* ci;
  const double* va;
};

// ---------------------------------------------------------------------------
// phase A: contributions of one 32-row tile [row0, row0 + valid)
// ---------------------------------------------------------------------------
//
// Operator concept (pk_kernels.cuh):
//   static constexpr bool kSpmv;  struct Item;
//   void load(int64_t row, Item&)                 per-row vector loads
//   kSpmv:  Csr<RowT> A;  struct Gat;  void gload(int32_t col, Gat&)  raw words
//           double gval(const Gat&)          SpMV input value at col (may recompute)
//           void compute(int64_t row, Item&, double q, double (&c)[NQ])
//   else:   void compute(int64_t row, Item&, double (&c)[NQ])
//   void scalars(const ScalarPtrs&)               prologue: device scalars
//
// SpMV rows are summed acc = ((0 + v0 x0) + v1 x1) + ... in stored order
// (_spmvkernels.py:12-18).  The warp loads the tile's contiguous nnz range
// coalesced, forms every product once, parks it in shared memory and each
// lane then adds its own row's products in order.
template <int NQ, class Op>
__device__ __forceinline__ void tile_contrib(const Op& op, int64_t row0, int valid, double* pbuf,
                                             double (&c)[NQ]) {
  const int lane = threadIdx.x & 31;
  const bool v = lane < valid;
  const int64_t row = row0 + lane;
#pragma unroll
  for (int q = 0; q < NQ; ++q) c[q] = 0.0;
  if (valid <= 0) return;
  typename Op::Item it;
  if constexpr (Op::kSpmv) {
    using RowT = typename decltype(Op::A)::RowT;
    RowT beg = 0, end = 0;
    if (v) {
      beg = __ldg(op.A.rp + row);
      end = __ldg(op.A.rp + row + 1);
      op.load(row, it);
    }
    const RowT base = __shfl_sync(kFull, beg, 0);
    const RowT top = __shfl_sync(kFull, end, valid - 1);
    const int64_t L = (int64_t)(top - base);
    constexpr int S = Op::kSlots;  // nnz slots per lane per pass
    double acc = 0.0;
    if (L <= kPCap) {
      for (int e0 = 0; e0 < L; e0 += S * 32) {
        // three explicit stages so every load of a stage is in flight at
        // once: column/value words, then the gathered input words, then
        // the products (Op::Gat holds the raw words of one gathered input).
        // every slot is defined on every path (predicated-off slots keep
        // column 0 / zeros), so the arrays stay in registers
        int32_t col[S];
        double val[S];
        typename Op::Gat gv[S];
#pragma unroll
        for (int j = 0; j < S; ++j) {
          col[j] = 0;
          val[j] = 0.0;
          gv[j] = typename Op::Gat{};
        }
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const int e = e0 + j * 32 + lane;
          if (e < L) {
            col[j] = __ldg(op.A.ci + base + e);
            val[j] = __ldg(op.A.va + base + e);
          }
        }
#pragma unroll
        for (int j = 0; j < S; ++j) {
          if (e0 + j * 32 + lane < L) op.gload(col[j], gv[j]);
        }
#pragma unroll
        for (int j = 0; j < S; ++j) {
          const int e = e0 + j * 32 + lane;
          if (e < L) pbuf[e] = mul_rn(val[j], op.gval(gv[j]));
        }
      }
      __syncwarp();
      if (v) {
        const int hi = (int)(end - base);
        for (int e = (int)(beg - base); e < hi; ++e) acc = add_rn(acc, pbuf[e]);
      }
      __syncwarp();
    } else {
      // long rows: direct ordered loop (correct for any row length)
      if (v) {
        for (RowT e = beg; e < end; ++e) {
          typename Op::Gat g;
          op.gload(__ldg(op.A.ci + e), g);
          acc = add_rn(acc, mul_rn(__ldg(op.A.va + e), op.gval(g)));
        }
      }
    }
    if (v) op.compute(row, it, acc, c);
  } else {
    if (v) {
      op.load(row, it);
      op.compute(row, it, c);
    }
  }
}

// Elementwise tile without contributions (plain SpMV / sweeps).
template <class Op>
__device__ __forceinline__ void tile_apply(const Op& op, int64_t row0, int valid, double* pbuf) {
  double c[1];
  tile_contrib<1>(op, row0, valid, pbuf, c);
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
      for (uint32_t i = 0; i < (uint32_t)geo.tm; ++i) {
        const int64_t idx = base + (int64_t)brev_bits(i, geo.tlogm) * T;
        double x[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) x[q] = q < nstore ? __ldcg(spill + (int64_t)q * geo.G + idx) : 0.0;
        st.push(i, x, v);
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

// Runs stage 1 of this CTA's units and writes part[g * ld + col0 + q] for
// q < nstore.  Returns true in every thread of the CTA that completed the
// last group (the finalizer CTA).
template <int NQ, int U, class Op>
__device__ __forceinline__ bool engine_run(const Geom& geo, const Op& op, double* smem, double* part, int ld,
                                           int col0, int nstore, const Scratch& scr, unsigned* ticket) {
  __shared__ int s_flag;
  __shared__ int s_last;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int B = kWarps * U;  // chunks (or leaves) per batch
  double* C = smem;
  double* pbuf = C + (size_t)B * NQ * 32 + (Op::kSpmv ? warp * kPCap : 0);
  double* tail = C + (size_t)B * NQ * 32 + (Op::kSpmv ? kWarps * kPCap : 0);
  if (tid == 0) s_last = 0;

  for (int64_t unit = blockIdx.x; unit < geo.units; unit += gridDim.x) {
    int ncomplete = 0;
    if (!geo.leaf) {
      // ---- CHAIN: 32 lane ids [lid0, lid0 + nl), chunks k = 0..K-1 ----
      const int64_t lid0 = unit * 32;
      const int nl = (int)((geo.G - lid0) < 32 ? (geo.G - lid0) : 32);
      double acc[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
      for (int64_t k0 = 0; k0 < geo.K; k0 += B) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int kk = warp + kWarps * u;
          const int64_t k = k0 + kk;
          if (k < geo.K) {
            const int64_t row0 = k * geo.G + lid0;
            int64_t rem = geo.n - row0;
            const int valid = rem <= 0 ? 0 : (int)(rem < nl ? rem : nl);
            double c[NQ];
            tile_contrib<NQ>(op, row0, valid, pbuf, c);
#pragma unroll
            for (int q = 0; q < NQ; ++q) C[(kk * NQ + q) * 32 + lane] = c[q];
          }
        }
        __syncthreads();
        if (warp == 0) {
          const int kend = (int)((geo.K - k0) < B ? (geo.K - k0) : B);
          for (int kk = 0; kk < kend; ++kk) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = add_rn(acc[q], C[(kk * NQ + q) * 32 + lane]);
          }
        }
        __syncthreads();
      }
      if (warp == 0 && lane < nl) {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
          if (q < nstore) scr.spill[(int64_t)q * geo.G + lid0 + lane] = acc[q];
      }
      __threadfence();
      __syncthreads();
      if (geo.gs >= 32) {
        const int g = (int)(lid0 / geo.gs);
        if (tid == 0) {
          const unsigned per = (unsigned)(geo.gs / 32);
          unsigned t = atomicAdd(scr.gtick + g, 1u);
          int last = (t == per - 1);
          if (last) scr.gtick[g] = 0u;
          s_flag = last;
        }
        __syncthreads();
        if (s_flag) {
          __threadfence();
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
      // ---- LEAF: group g, lane thread `lane` owns lanes {lane + 32 j} ----
      const int g = (int)unit;
      double out[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) out[q] = 0.0;
      LeafStack<NQ> st{tail, 32, lane};
      for (int i0 = 0; i0 < geo.m; i0 += B) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int ii = warp + kWarps * u;
          const int i = i0 + ii;
          if (i < geo.m) {
            const int64_t row0 = (int64_t)g * geo.gs + (int64_t)brev_bits((uint32_t)i, geo.logm) * 32;
            int64_t rem = geo.n - row0;
            const int valid = rem <= 0 ? 0 : (int)(rem < 32 ? rem : 32);
            double c[NQ];
            tile_contrib<NQ>(op, row0, valid, pbuf, c);
#pragma unroll
            for (int q = 0; q < NQ; ++q) C[(ii * NQ + q) * 32 + lane] = c[q];
          }
        }
        __syncthreads();
        if (warp == 0) {
          const int iend = (geo.m - i0) < B ? (geo.m - i0) : B;
          for (int ii = 0; ii < iend; ++ii) {
            double x[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) x[q] = C[(ii * NQ + q) * 32 + lane];
            if (geo.m > 1) {
              st.push((uint32_t)(i0 + ii), x, out);
            } else {
#pragma unroll
              for (int q = 0; q < NQ; ++q) out[q] = x[q];
            }
          }
        }
        __syncthreads();
      }
      if (warp == 0) {
#pragma unroll
        for (int s = 16; s >= 1; s >>= 1) {
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            double o = __shfl_down_sync(kFull, out[q], s);
            if (lane < s) out[q] = add_rn(out[q], o);
          }
        }
        if (lane == 0 && part) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
            if (q < nstore) part[(int64_t)g * ld + col0 + q] = out[q];
        }
      }
      ncomplete = 1;
    }
    // ---- global ticket: the CTA completing the last group finalizes ----
    if (ncomplete > 0) {
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        unsigned t = atomicAdd(ticket, (unsigned)ncomplete);
        if (t + (unsigned)ncomplete == (unsigned)geo.n_groups) {
          *ticket = 0u;
          s_last = 1;
          __threadfence();
        }
      }
      __syncthreads();
    }
  }
  return s_last != 0;
}

// Grid-stride sweep of 32-row warp tiles (no reduction).
template <class Op>
__device__ __forceinline__ void sweep_tiles(int64_t n, const Op& op, double* smem) {
  const int warp = threadIdx.x >> 5;
  double* pbuf = smem + (Op::kSpmv ? warp * kPCap : 0);
  const int64_t tiles = (n + 31) / 32;
  const int64_t wstride = (int64_t)gridDim.x * kWarps;
  for (int64_t t = (int64_t)blockIdx.x * kWarps + warp; t < tiles; t += wstride) {
    const int64_t row0 = t * 32;
    const int64_t rem = n - row0;
    tile_apply(op, row0, (int)(rem < 32 ? rem : 32), pbuf);
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
