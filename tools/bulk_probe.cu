// Microbenchmark: cost of issuing cp.async.bulk (UBLKCP) from one thread and
// the completion latency, vs copy size and number of copies in flight.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void probe(const unsigned char* src, size_t src_bytes, int bytes, int ncopies, int iters, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sa(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  unsigned par = 0;
  unsigned long long t_issue = 0, t_total = 0;
  size_t pos = (size_t)blockIdx.x * 4096 * 1024;
  for (int it = 0; it < iters; ++it) {
    unsigned long long t0 = gt();
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" :: "r"(sa(&bar)), "r"(bytes * ncopies) : "memory");
    for (int c = 0; c < ncopies; ++c) {
      pos = (pos + bytes) % (src_bytes - bytes);
      pos &= ~(size_t)15;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   :: "r"(sa(sm + (size_t)c * bytes)), "l"(src + pos), "r"(bytes), "r"(sa(&bar)) : "memory");
    }
    unsigned long long t1 = gt();
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(sa(&bar)), "r"(par) : "memory");
    par ^= 1;
    unsigned long long t2 = gt();
    t_issue += t1 - t0; t_total += t2 - t0;
  }
  if (blockIdx.x == 0) { out[0] = t_issue / iters; out[1] = t_total / iters; }
}
int main() {
  size_t sb = (size_t)2 << 30;
  unsigned char* src; cudaMalloc(&src, sb); cudaMemset(src, 1, sb);
  unsigned long long* out; cudaMalloc(&out, 16);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int sizes[] = {4096, 16384, 20480, 32768};
  int ncs[] = {1, 2, 4, 8};
  for (int grid : {1, 148}) for (int b : sizes) for (int nc : ncs) {
    if ((size_t)b * nc > 200 * 1024) continue;
    probe<<<grid, 32, 200 * 1024>>>(src, sb, b, nc, 200, out);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    double bw = (double)b * nc / (double)h[1];  // bytes per ns per SM
    printf("grid %3d bytes %6d ncopies %d  issue %6llu ns  total %6llu ns  per-SM %.1f GB/s  chip %.0f GB/s %s\n", grid, b, nc, h[0], h[1], bw, bw * grid, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
