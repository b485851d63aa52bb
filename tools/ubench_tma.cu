// Microbenchmark (tools/, not product): DRAM read throughput of 1-D TMA bulk
// copies (cp.async.bulk global -> shared) as a function of copy size, copies
// in flight per warp (ring depth R) and producer warps per SM, against plain
// 16-byte LDG streaming.  Reads a 512 MB buffer once (larger than L2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma tools/ubench_tma.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void minit(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mexp(uint64_t* b, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mwait(uint64_t* b, unsigned par) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE;\nbra "
      "LAB_WAIT;\nDONE:\n}\n" ::"r"(su(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void mwait_test(uint64_t* b, unsigned par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n.reg .pred P1;\nmbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(ok) : "r"(su(b)), "r"(par) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mwait_hint(uint64_t* b, unsigned par, unsigned ns) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\nselp.u32 %0, 1, 0, P1;\n}\n"
                 : "=r"(ok) : "r"(su(b)), "r"(par), "r"(ns) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)),
               "l"(s), "r"(n), "r"(su(b))
               : "memory");
}

__device__ __forceinline__ void bulk_cta(void* d, const void* s, unsigned n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)),
               "l"(s), "r"(n), "r"(su(b))
               : "memory");
}

// LDGSTS variant: the whole warp copies a chunk with 16-byte cp.async, completion
// tracked by cp.async.mbarrier.arrive.noinc (count 32 per phase)
__global__ void k_ldgsts(const char* src, long total, int bytes, int R, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = (uint64_t*)sm;
  unsigned char* slots = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < warps * R; ++i) minit(full + i, 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long nch = total / bytes;
  const long gw = (long)blockIdx.x * warps + warp, nw = (long)gridDim.x * warps;
  const long mine = gw < nch ? (nch - gw + nw - 1) / nw : 0;
  auto issue = [&](long j) {
    const int s = (int)(j % R);
    uint64_t* f = full + warp * R + s;
    unsigned char* d = slots + ((size_t)warp * R + s) * bytes;
    const char* p = src + (gw + j * nw) * (long)bytes;
    for (int o = lane * 16; o < bytes; o += 512)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(d + o)), "l"(p + o) : "memory");
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su(f)) : "memory");
  };
  for (long j = 0; j < mine && j < R; ++j) issue(j);
  double acc = 0.0;
  for (long j = 0; j < mine; ++j) {
    const int s = (int)(j % R);
    mwait(full + warp * R + s, (unsigned)((j / R) & 1));
    acc += ((const double*)(slots + ((size_t)warp * R + s) * bytes))[lane];
    __syncwarp();
    if (j + R < mine) issue(j + R);
  }
  if (acc == 1234.5) sink[0] = acc;
}

// tensor-TMA variant: 1-D tiled tensor map over the buffer as fp64, box of
// `box` elements; chunk c = box elements at element c * box
__global__ void k_tmap(const __grid_constant__ CUtensorMap tm, long total, int box, int R, double* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = (uint64_t*)sm;
  unsigned char* slots = sm + 1024;
  const int bytes = box * 8;
  if (threadIdx.x == 0) {
    for (int i = 0; i < warps * R; ++i) minit(full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long nch = total / bytes;
  const long gw = (long)blockIdx.x * warps + warp, nw = (long)gridDim.x * warps;
  const long mine = gw < nch ? (nch - gw + nw - 1) / nw : 0;
  auto issue = [&](long j) {
    if (lane == 0) {
      const int s = (int)(j % R);
      uint64_t* f = full + warp * R + s;
      unsigned char* d = slots + ((size_t)warp * R + s) * bytes;
      const int x = (int)((gw + j * nw) * box);
      mexp(f, bytes);
      asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                   ::"r"(su(d)), "l"(&tm), "r"(x), "r"(su(f)) : "memory");
    }
  };
  for (long j = 0; j < mine && j < R; ++j) issue(j);
  double acc = 0.0;
  for (long j = 0; j < mine; ++j) {
    const int s = (int)(j % R);
    mwait(full + warp * R + s, (unsigned)((j / R) & 1));
    acc += ((const double*)(slots + ((size_t)warp * R + s) * bytes))[lane];
    __syncwarp();
    if (j + R < mine) issue(j + R);
  }
  if (acc == 1234.5) sink[0] = acc;
}

// every warp streams chunks c = gwarp, gwarp + nwarps, ... of `bytes` each
// through a private ring of R slots (lane 0 issues, the warp waits)
__global__ void k_tma(const char* src, long total, int bytes, int R, int nsub, double* sink, int wmode, int lanemode) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int warps = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* full = (uint64_t*)sm;
  unsigned char* slots = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < warps * R; ++i) minit(full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long nch = total / bytes;
  const long gw = (long)blockIdx.x * warps + warp, nw = (long)gridDim.x * warps;
  const long mine = gw < nch ? (nch - gw + nw - 1) / nw : 0;
  auto issue = [&](long j) {
    if (lane == (lanemode ? (int)(j % 32) : 0)) {
      const int s = (int)(j % R);
      uint64_t* f = full + warp * R + s;
      unsigned char* d = slots + ((size_t)warp * R + s) * bytes;
      const char* p = src + (gw + j * nw) * (long)bytes;
      mexp(f, bytes);
      const int sub = bytes / nsub;
      for (int k = 0; k < nsub; ++k) { if (wmode == 7) bulk_cta(d + k * sub, p + k * sub, sub, f); else bulk(d + k * sub, p + k * sub, sub, f); }
    }
  };
  for (long j = 0; j < mine && j < R; ++j) issue(j);
  double acc = 0.0;
  for (long j = 0; j < mine; ++j) {
    const int s = (int)(j % R);
    if (wmode == 0 || wmode == 7) mwait(full + warp * R + s, (unsigned)((j / R) & 1));
    else if (wmode == 1) mwait_test(full + warp * R + s, (unsigned)((j / R) & 1));
    else mwait_hint(full + warp * R + s, (unsigned)((j / R) & 1), (unsigned)wmode);
    acc += ((const double*)(slots + ((size_t)warp * R + s) * bytes))[lane];
    __syncwarp();
    if (j + R < mine) issue(j + R);
  }
  if (acc == 1234.5) sink[0] = acc;
}

__global__ void k_ldg(const double2* src, long n2, double* sink) {
  double acc = 0.0;
  const long T = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += 4 * T) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i + u * T < n2 ? __ldcs(src + i + u * T) : make_double2(0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u].x + v[u].y;
  }
  if (acc == 1234.5) sink[0] = acc;
}

int main() {
  const long total = 512l << 20;
  char* src;
  double* sink;
  char* flush;
  cudaMalloc(&src, total);
  cudaMalloc(&sink, 8);
  cudaMalloc(&flush, 256l << 20);
  cudaMemset(src, 0, total);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      cudaMemset(flush, it, 256l << 20);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    return best;
  };
  {
    float ms = timeit([&] { k_ldg<<<148 * 8, 256>>>((const double2*)src, total / 16, sink); });
    printf("{\"kind\": \"ldg\", \"GBps\": %.0f}\n", total / (ms * 1e-3) / 1e9);
  }
  typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fp = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault);
  EncFn enc = (EncFn)fp;
  cudaFuncSetAttribute(k_tmap, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int box : {256, 1024})
    for (int R : {1, 2, 4, 8})
      for (int c : {1, 7}) {
        CUtensorMap tm;
        cuuint64_t dim[1] = {(cuuint64_t)(total / 8)};
        cuuint64_t str[1] = {0};
        cuuint32_t bx[1] = {(cuuint32_t)box};
        cuuint32_t es[1] = {1};
        CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, src, dim, str, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const size_t smem = 1024 + (size_t)R * box * 8;
        if (smem * c > 220 * 1024) continue;
        float ms = timeit([&] { k_tmap<<<148 * c, 32, smem>>>(tm, total, box, R, sink); });
        printf("{\"kind\": \"tmap\", \"box_bytes\": %d, \"R\": %d, \"ctas\": %d, \"GBps\": %.0f, \"enc\": %d, \"err\": \"%s\"}\n",
               box * 8, R, c, total / (ms * 1e-3) / 1e9, (int)r, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
