// Microbenchmark (tools/, not product): does an LDG issued by a warp right
// after it issued a 1-D bulk copy (cp.async.bulk) wait for that copy?  One
// warp per SM; per trial: optionally issue a bulk copy of `bytes` from a
// cold region, then time (clock64) an independent 8-byte LDG from another
// cold region, then wait for the copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_tma_ldg tools/ubench_tma_ldg.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const char* a, const double* b, int bytes, int with_copy, int trials, long long* out) {
  __shared__ __align__(128) unsigned char buf[16384];
  __shared__ uint64_t bar;
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  long long tot = 0;
  double sink = 0.0;
  for (int t = 0; t < trials; ++t) {
    const long off = ((long)blockIdx.x * trials + t) * 65536;
    if (with_copy && lane == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su(buf)),
                   "l"(a + off), "r"(bytes), "r"(su(&bar))
                   : "memory");
    }
    const long long t0 = clock64();
    double v = __ldcg(b + off / 8 + lane);
    sink += v;
    __syncwarp();
    const long long t1 = clock64();
    tot += t1 - t0;
    if (with_copy) {
      asm volatile(
          "{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra DONE;\nbra "
          "LAB_WAIT;\nDONE:\n}\n" ::"r"(su(&bar)),
          "r"(t & 1)
          : "memory");
    }
  }
  if (lane == 0) out[blockIdx.x] = tot / trials;
  if (sink == 1234.5) out[0] = 0;
}

int main() {
  const int trials = 64;
  char* a;
  double* b;
  long long* out;
  const size_t sz = (size_t)148 * trials * 65536 + 65536;
  cudaMalloc(&a, sz);
  cudaMalloc(&b, sz);
  cudaMalloc(&out, 148 * 8);
  long long h[148];
  for (int wc = 0; wc < 2; ++wc)
    for (int bytes : {2048, 16384}) {
      k<<<148, 32>>>(a, b, bytes, wc, trials, out);
      cudaDeviceSynchronize();
      cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
      long long s = 0;
      for (int i = 0; i < 148; ++i) s += h[i];
      printf("{\"with_copy\": %d, \"bytes\": %d, \"ldg_cycles\": %lld, \"err\": \"%s\"}\n", wc, bytes, s / 148,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
