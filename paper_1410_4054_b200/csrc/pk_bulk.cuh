// BULK CHAIN engine: TMA-fed, warp-specialised ordered reduction for SpMV
// operators on CHAIN geometries (K = ceil(n / G) >= 2, group_size >= 32).
//
// Same reduction schedule as engine_run() (pk_reduce.cuh; linalg.py:289-320):
// lane t of [0, G) folds the contributions of rows t, t + G, t + 2G, ... in
// chunk order, then per group a halving tree, then the serial stage 2 in the
// finalizer.  What changes is how the rows' CSR data reaches the threads.
//
// One CTA owns one unit: 32 consecutive lane ids [t0, t0 + 32).  Chunk k of
// the unit is the aligned 32-row block [kG + t0, kG + t0 + 32) -- its row
// bounds, columns and values are three CONTIGUOUS ranges of the CSR arrays,
// which arrive in shared memory by cp.async.bulk (TMA) with one mbarrier
// armed with the byte count per chunk (16-byte aligned ranges, rounded out to
// whole 16-byte words; the arrays are padded).  No register holds an
// in-flight CSR byte: the DRAM queue depth is set by shared memory.
//
//   warps 1..W (rows): warp w takes chunks w - 1, w - 1 + W, ... through a
//     private ring of R slots.  It loads its chunks' bounds (rowptr at the
//     block edges, one round trip per 32 chunks) and is its own producer: per
//     chunk it waits for the slot's bytes, reads its 32 rows' columns and
//     values into registers (rows of at most kSlots entries), re-arms the slot
//     with the chunk R ahead, then gathers the SpMV input through L1/L2, sums
//     each row in stored order (exactly row_contrib()), evaluates the
//     operator (vector outputs stored directly) and parks the NQ contributions
//     in its contribution slot.  The next chunk's own-row loads are issued
//     before the gathers.
//   warp 0 (fold): folds the contributions in chunk order -- lane l is lane
//     t0 + l, acc = ((0 + c_0) + c_1) + ... in registers, the reference's
//     serial lane sum -- and releases each contribution slot.
//
// Barrier phases: a slot's barriers complete once per use and waiters use
// parity (use & 1); every slot has a single producer and a single consumer
// that both walk its uses in order, so no waiter can be two phases behind.
//
// After the last fold warp 0 publishes the lane values (spill), takes the
// group ticket, and the CTA completing a group runs the warp-level halving
// tree (group_tree_warp); the CTA completing the last group finalizes.
#pragma once

#include "pk_reduce.cuh"

#ifndef PK_BULK_LATE
#define PK_BULK_LATE 0  // 1: re-arm a slot after the chunk's gathers are consumed, not right after its rows are read
#endif
#ifndef PK_BULK_RPLDG
#define PK_BULK_RPLDG 0  // 1: row bounds by LDG (prefetched a chunk ahead) instead of a third bulk copy
#endif

namespace pk {

#ifdef PK_BULK_TRACE
// debug: per-CTA %globaltimer stamps (pk_debug_bulk_trace)
__device__ unsigned long long* g_bulk_trace = nullptr;
__device__ __forceinline__ void btrace(int slot) {
  if (g_bulk_trace && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_bulk_trace[(size_t)blockIdx.x * 32 + slot] = t;
  }
}
__device__ __forceinline__ void btrace_abs(size_t slot) {
  if (g_bulk_trace && (threadIdx.x & 31) == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_bulk_trace[slot] = t;
  }
}
#define PK_BT(s) btrace(s)
#define PK_BTA(s) btrace_abs(s)
#else
#define PK_BT(s)
#define PK_BTA(s)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on mbarrier `b`
// (addresses and size multiples of 16 bytes)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

// Shared-memory layout of one engine CTA (host-computed, bytes):
//   [0, base)                         mbarriers: full[W][R], cfull[W][CR], cempty[W][CR]
//   base + (w R + j) * slot           data slot j of row warp w: rowptr segment (rpb) | columns (capc) | values (capv)
//   offq + (w CR + j) * NQ * 256      contribution slot j of row warp w (NQ x 32 doubles)
struct BulkCfg {
  int32_t base;  // data slot area offset
  int32_t slot;  // bytes per data slot
  int32_t offc;  // column range offset in a slot
  int32_t offv;  // value range offset
  int32_t offq;  // contribution slots offset
  int32_t capc;  // column bytes per slot (>= the largest aligned range)
  int32_t capv;
  int32_t total; // bytes
  int32_t pdl;   // launched with programmatic stream serialization
};

constexpr int kBulkCR = 1;  // contribution slots per row warp

// rowptr segment bytes: 33 entries rounded up to 16 bytes
template <typename RowT>
__host__ __device__ constexpr int bulk_rpb() {
  return sizeof(RowT) == 4 ? 144 : 272;
}

template <int NQ, int W, int R, class Op>
__host__ inline BulkCfg bulk_cfg(int64_t blk_max) {
  using RowT = typename Op::RowT;
  BulkCfg c{};
  c.base = ((8 * W * (R + 2 * kBulkCR) + 127) / 128) * 128;
  c.capc = (int32_t)((((blk_max + 6) * 4) + 15) / 16 * 16);
  c.capv = (int32_t)((((blk_max + 2) * 8) + 15) / 16 * 16);
  c.offc = bulk_rpb<RowT>();
  c.offv = c.offc + c.capc;
  c.slot = ((c.offv + c.capv) + 127) / 128 * 128;
  c.offq = c.base + W * R * c.slot;
  c.total = c.offq + W * kBulkCR * NQ * 32 * 8;
  return c;
}

// Row warps w = 1..W (index wi = w - 1) own the chunks wi, wi + W, ...; the
// warp's j-th chunk lives in its data slot j % R.  Each row warp is its own
// TMA producer: it issues chunk j + R into slot j % R as soon as it has read
// chunk j's rows out of the slot (rows of at most kSlots entries: a row's
// columns / values fit in registers), i.e. before its gathers -- R - 1 chunks
// of CSR are always in flight per warp.  Warp 0 only folds.
// `sync()` is called by every thread once the CTA's first R chunks per row
// warp are in flight (their CSR bytes depend only on the matrix): it waits
// for the previous kernel (programmatic dependent launch), loads the
// operator's scalars and evaluates the gate; false = skip this launch (the
// in-flight copies are drained first).
template <int NQ, int W, int R, class Op, class Sync>
__device__ __forceinline__ bool engine_bulk(const Geom& geo, Op& op, unsigned char* sm, const BulkCfg& bc,
                                            double* part, int ld, int col0, int nstore, const Scratch& scr,
                                            unsigned* ticket, Sync sync) {
  using RowT = typename Op::RowT;
  constexpr int S = Op::kSlots;
  constexpr int CR = kBulkCR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);  // [W][R]
  uint64_t* cfull = full + W * R;                     // [W][CR]
  uint64_t* cempty = cfull + W * CR;                  // [W][CR]
  const int64_t lid0 = (int64_t)blockIdx.x * 32;
  const int64_t K = geo.K, G = geo.G, n = geo.n;
  if (threadIdx.x == 0) {
    for (int i = 0; i < W * R; ++i) mbar_init(full + i, 1);
    for (int i = 0; i < W * CR; ++i) {
      mbar_init(cfull + i, 32);
      mbar_init(cempty + i, 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) PK_BT(0);

  if (warp == 0) {
    if (!sync()) return false;
    // ---------------- fold warp: the lane chains in chunk order ----------------
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    for (int kk = 0; kk < (int)K; ++kk) {
      const int wi = kk % W;
      const int j = kk / W;
      const int cs = wi * CR + j % CR;
      mbar_wait(cfull + cs, (unsigned)((j / CR) & 1));
      const double* cq = reinterpret_cast<const double*>(sm + bc.offq + (size_t)cs * NQ * 256);
#pragma unroll
      for (int q = 0; q < NQ; ++q) acc[q] = add_rn(acc[q], cq[q * 32 + lane]);
      mbar_arrive(cempty + cs);
    }
    PK_BT(1);
    // ---------------- lane values -> group tree -> finalizer ticket ----------------
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (q < nstore) scr.spill[(int64_t)q * G + lid0 + lane] = acc[q];
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
    bool last = false;
    if (lastg) {
      // every chunk is folded: the row warps are done with the data slots
      group_tree_warp<NQ>(geo, g, scr.spill, reinterpret_cast<double*>(sm + bc.base), part, ld, col0, nstore);
      int l = 0;
      if (lane == 0) {
        unsigned tk = ticket_add(ticket, 1u);
        if (tk + 1u == (unsigned)geo.n_groups) {
          *ticket = 0u;
          acquire_fence();
          l = 1;
        }
      }
      last = __shfl_sync(kFull, l, 0) != 0;
    }
    PK_BT(2);
    if (lane == 0) {
#ifdef PK_BULK_TRACE
      if (g_bulk_trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_bulk_trace[(size_t)blockIdx.x * 32 + 3] = smid;
      }
#endif
    }
    return last;
  }

  // ---------------- row warps ----------------
  const int wi = warp - 1;
  const int nj = K > wi ? (int)((K - wi + W - 1) / W) : 0;  // chunks of this warp
  const RowT* __restrict__ rp = op.A.rp;
  unsigned char* dslot = sm + bc.base + (size_t)wi * R * bc.slot;
  // chunk bounds (rowptr at the block edges) of local chunks 32 b + lane
  RowT lo_c = 0, hi_c = 0;
  int blk = -1;
  auto ld_bounds = [&](int b) {
    const int j = b * 32 + lane;
    lo_c = 0;
    hi_c = 0;
    if (j < nj) {
      const int64_t r0 = (int64_t)(wi + j * W) * G + lid0;
      lo_c = __ldg(rp + (r0 < n ? r0 : n));
      hi_c = __ldg(rp + (r0 + 32 < n ? r0 + 32 : n));
    }
    blk = b;
  };
  auto issue = [&](int j) {  // whole warp (shuffles); lane 0 issues
    if ((j >> 5) != blk) ld_bounds(j >> 5);
    const RowT lo = __shfl_sync(kFull, lo_c, (int)(j & 31));
    const RowT hi = __shfl_sync(kFull, hi_c, (int)(j & 31));
    if (lane == 0) {
      const int s = j % R;
      unsigned char* b = dslot + (size_t)s * bc.slot;
      uint64_t* fb = full + wi * R + s;
      const int64_t r0 = (int64_t)(wi + j * W) * G + lid0;
      const bool rows = r0 < n;
      const bool ents = hi > lo;
      const RowT cs = lo & ~(RowT)3, ce = (hi + 3) & ~(RowT)3;
      const RowT vs = lo & ~(RowT)1, ve = (hi + 1) & ~(RowT)1;
      unsigned tx = 0;
      if (rows && !PK_BULK_RPLDG) tx += bulk_rpb<RowT>();
      if (ents) tx += (unsigned)((ce - cs) * 4 + (ve - vs) * 8);
      // the slot's previous rows were read by this warp (generic proxy)
      // before the __syncwarp that precedes this issue
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive_expect_tx(fb, tx);
      if (rows && !PK_BULK_RPLDG) bulk_g2s(b, rp + r0, bulk_rpb<RowT>(), fb);
      if (ents) {
        bulk_g2s(b + bc.offc, op.A.ci + cs, (unsigned)((ce - cs) * 4), fb);
        bulk_g2s(b + bc.offv, op.A.va + vs, (unsigned)((ve - vs) * 8), fb);
      }
    }
  };
  for (int j = 0; j < nj && j < R; ++j) issue(j);
  if (wi == 0) PK_BT(4);
  if (!sync()) {
    // skipped launch: the issued copies still land in this CTA's shared memory
    for (int j = 0; j < nj && j < R; ++j) mbar_wait(full + wi * R + j, 0u);
    return false;
  }
  typename Op::Item itn;
  uint32_t rown = 0;
  bool okn = false;
  RowT rbn = 0, ren = 0;  // PK_BULK_RPLDG: the next chunk's row bounds
  if (nj > 0) {
    const int64_t r = (int64_t)wi * G + lid0 + lane;
    okn = r < n;
    rown = okn ? (uint32_t)r : 0u;
    if (okn) {
      op.load(rown, itn);
      if (PK_BULK_RPLDG) {
        rbn = __ldg(rp + rown);
        ren = __ldg(rp + rown + 1);
      }
    }
  }
  for (int j = 0; j < nj; ++j) {
    const typename Op::Item it = itn;
    const uint32_t row = rown;
    const bool ok = okn;
    const RowT rb = rbn, re = ren;
    const int s = j % R;
    const unsigned char* sb = dslot + (size_t)s * bc.slot;
    mbar_wait(full + wi * R + s, (unsigned)((j / R) & 1));
    if (wi == 0 && j < 8) PK_BT(5 + 2 * j);
    // the row's columns / values, out of the slot into registers
    int32_t col[S];
    double val[S];
    int b = 0, e = 0;
    if (ok) {
      const int32_t* csm = reinterpret_cast<const int32_t*>(sb + bc.offc);
      const double* vsm = reinterpret_cast<const double*>(sb + bc.offv);
      RowT lo, b0, e0;
      if (PK_BULK_RPLDG) {
        lo = __shfl_sync(__activemask(), rb, 0);  // lane 0's row is valid whenever any row is
        b0 = rb;
        e0 = re;
      } else {
        const RowT* rps = reinterpret_cast<const RowT*>(sb);
        lo = rps[0];
        b0 = rps[lane];
        e0 = rps[lane + 1];
      }
      const RowT cs = lo & ~(RowT)3, vs = lo & ~(RowT)1;
      b = (int)(b0 - cs);
      e = (int)(e0 - cs);
      const int dv = (int)(cs - vs);  // value index = column index + dv
#pragma unroll
      for (int t = 0; t < S; ++t) {
        const int k = (b + t < e) ? b + t : b;  // past the end: re-read a valid slot
        col[t] = csm[k];
        val[t] = vsm[k + dv];
      }
    } else {
#pragma unroll
      for (int t = 0; t < S; ++t) {
        col[t] = 0;
        val[t] = 0.0;
      }
    }
    __syncwarp();
    if (!PK_BULK_LATE && j + R < nj) issue(j + R);
    if (j + 1 < nj) {
      const int64_t r = (int64_t)(wi + (j + 1) * W) * G + lid0 + lane;
      okn = r < n;
      rown = okn ? (uint32_t)r : 0u;
      if (okn) {
        op.load(rown, itn);
        if (PK_BULK_RPLDG) {
          rbn = __ldg(rp + rown);
          ren = __ldg(rp + rown + 1);
        }
      }
    }
    double c[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) c[q] = 0.0;
    if (ok) {
      typename Op::Gat gv[S];
#pragma unroll
#ifdef PK_BULK_NOGATHER
      for (int t = 0; t < S; ++t) op.gload(row, gv[t]);  // debug: latency experiment, wrong results
#else
      for (int t = 0; t < S; ++t) op.gload((uint32_t)col[t], gv[t]);
#endif
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < S; ++t)
        if (b + t < e) acc = add_rn(acc, mul_rn(val[t], op.gval(gv[t])));
      typename Op::Item itc = it;
      op.compute(row, itc, acc, c);
    }
    if (wi == 0 && j < 8) PK_BT(21 + j);
    const int cs = wi * CR + j % CR;
    mbar_wait(cempty + cs, (unsigned)(((j / CR) & 1) ^ 1));
    double* cq = reinterpret_cast<double*>(sm + bc.offq + (size_t)cs * NQ * 256);
#pragma unroll
    for (int q = 0; q < NQ; ++q) cq[q * 32 + lane] = c[q];
    mbar_arrive(cfull + cs);
    if (PK_BULK_LATE && j + R < nj) issue(j + R);
    if (wi == 0 && j < 8) PK_BT(6 + 2 * j);
  }
  return false;
}

}  // namespace pk
