// Microbenchmark (tools/, not product): DRAM throughput of the BULK engine's
// access pattern.  A CSR-shaped stream (rowptr int32, columns int32, values
// fp64; 5 entries per row, n = 2^20 rows) is read by TMA bulk copies into a
// per-warp ring of shared-memory slots, 32-row chunks, in
//   mode 0: the reference geometry's chunk order (CTA = 32 lanes, chunk k =
//           rows k G + t0 .. + 32, G = 32768 -- the BULK engine's order)
//   mode 1: linear order (CTA c = rows 1024 c .. 1024 c + 1023)
// plus (own = 1) three coalesced 8-byte-per-row vector loads per chunk.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_chunk_order.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mexp(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, unsigned par) {
  asm volatile("{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(su(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

constexpr int W = 4, SLOT = 2176, K = 32;
constexpr long G = 32768;
template <int R>

__global__ void __launch_bounds__(160, 7) k_stream(int mode, int own, int ldgsts, const int* rp, const int* ci, const double* va,
                                                   const double* v0, const double* v1, const double* v2, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = (uint64_t*)sm;
  unsigned char* slots = sm + 128;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < W * R; ++i) minit(full + i, ldgsts ? 32 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) return;
  const int wi = warp - 1;
  auto row0 = [&](int j) -> long {  // first row of this warp's j-th chunk
    const int kk = wi + j * W;
    return mode == 0 ? (long)kk * G + (long)blockIdx.x * 32 : (long)blockIdx.x * 1024 + (long)kk * 32;
  };
  const int nj = K / W;
  int lo_l = 0, hi_l = 0;
  if (lane < nj) {
    lo_l = __ldg(rp + row0(lane));
    hi_l = __ldg(rp + row0(lane) + 32);
  }
  auto issue = [&](int j) {
    const long r0 = row0(j);
    const int lo = __shfl_sync(0xffffffffu, lo_l, j), hi = __shfl_sync(0xffffffffu, hi_l, j);
    if (ldgsts) {
      unsigned char* b = slots + (wi * R + j % R) * SLOT;
      const int cs = lo & ~3, ce = (hi + 3) & ~3, vs = lo & ~1, ve = (hi + 1) & ~1;
      uint64_t* f = full + wi * R + j % R;
      auto cp = [&](unsigned char* d, const void* g, int nb) {
        for (int o = lane * 16; o < nb; o += 512)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(d + o)), "l"((const char*)g + o) : "memory");
      };
      cp(b, rp + r0, 144);
      cp(b + 144, ci + cs, (ce - cs) * 4);
      cp(b + 144 + 672, va + vs, (ve - vs) * 8);
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(f)) : "memory");
    } else if (lane == 0) {
      unsigned char* b = slots + (wi * R + j % R) * SLOT;
      const int cs = lo & ~3, ce = (hi + 3) & ~3, vs = lo & ~1, ve = (hi + 1) & ~1;
      uint64_t* f = full + wi * R + j % R;
      mexp(f, 144 + (ce - cs) * 4 + (ve - vs) * 8);
      bulk(b, rp + r0, 144, f);
      bulk(b + 144, ci + cs, (ce - cs) * 4, f);
      bulk(b + 144 + 672, va + vs, (ve - vs) * 8, f);
    }
  };
  for (int j = 0; j < R; ++j) issue(j);
  double acc = 0.0;
  for (int j = 0; j < nj; ++j) {
    mwait(full + wi * R + j % R, (j / R) & 1);
    const unsigned char* b = slots + (wi * R + j % R) * SLOT;
    acc += ((const double*)(b + 144 + 672))[lane];
    if (own) {
      const long r = row0(j) + lane;
      acc += __ldg(v0 + r) + __ldg(v1 + r) + __ldg(v2 + r);
    }
    __syncwarp();
    if (j + R < nj) issue(j + R);
  }
  if (acc == 12345.0) sink[0] = acc;
}

int main() {
  const long n = 1l << 20, nnz = 5 * n;
  int *rp, *ci;
  double *va, *v0, *v1, *v2, *sink, *flush;
  cudaMalloc(&rp, (n + 1) * 4 + 512);
  cudaMalloc(&ci, nnz * 4 + 64);
  cudaMalloc(&va, nnz * 8 + 64);
  cudaMalloc(&v0, n * 8);
  cudaMalloc(&v1, n * 8);
  cudaMalloc(&v2, n * 8);
  cudaMalloc(&sink, 8);
  cudaMalloc(&flush, 256l << 20);
  int* h = new int[n + 1];
  for (long i = 0; i <= n; ++i) h[i] = (int)(5 * i);
  cudaMemcpy(rp, h, (n + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemset(ci, 0, nnz * 4);
  cudaMemset(va, 0, nnz * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](auto kern, int R, int mode, int own, int lg) {
    const int smem = 128 + W * R * SLOT;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaMemset(flush, it, 256l << 20);
      cudaEventRecord(a);
      kern<<<1024, 160, smem>>>(mode, own, lg, rp, ci, va, v0, v1, v2, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const double bytes = (n + 1) * 4.0 + nnz * 12.0 + (own ? 24.0 * n : 0.0);
    printf("{\"R\": %d, \"mode\": %d, \"own\": %d, \"ldgsts\": %d, \"us\": %.2f, \"GBps\": %.0f, \"err\": \"%s\"}\n", R, mode,
           own, lg, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  for (int lg = 0; lg < 2; ++lg)
    for (int own = 0; own < 2; ++own) {
      run(&k_stream<2>, 2, 0, own, lg);
      run(&k_stream<3>, 3, 0, own, lg);
      run(&k_stream<4>, 4, 0, own, lg);
    }
  return 0;
}
