// TMA bulk-copy ring throughput: 1 producer lane + NC consumer warps per CTA,
// one CTA per SM, chunks of CH bytes, NS stages; consumers wait for a chunk,
// read one word of it, release it.  Measures what a ring of NS x CH in flight
// per SM delivers from HBM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory"); }
__device__ __forceinline__ void mbar_expect(uint64_t* bar, unsigned b) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned par) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar, uint64_t pol, int hint) {
  if (hint) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
  else asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__global__ void k(const unsigned char* src, size_t per_cta, int CH, int NS, int NC, int hint, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) { for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NC); } asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  const unsigned char* base = src + blockIdx.x * per_cta;
  const int nch = (int)(per_cta / CH);
  if (wid == 0) {
    if (lane == 0) {
      uint64_t pol; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int c = 0; c < nch; ++c) {
        const int s = c % NS, use = c / NS;
        if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
        mbar_expect(&full[s], CH);
        bulk(sm + (size_t)s * CH, base + (size_t)c * CH, CH, &full[s], pol, hint);
      }
    }
    return;
  }
  double acc = 0;
  for (int c = 0; c < nch; ++c) {
    const int s = c % NS;
    mbar_wait(&full[s], (c / NS) & 1);
    acc += reinterpret_cast<const double*>(sm + (size_t)s * CH)[lane + 32 * (wid - 1)];
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (acc == 1.2345) out[0] = acc;
}
int main() {
  const size_t total = (size_t)148 * 2 * 1024 * 1024;  // 2 MB per CTA
  unsigned char* src; cudaMalloc(&src, total); cudaMemset(src, 1, total);
  double* out; cudaMalloc(&out, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  int cfg[][4] = {{16384, 5, 8, 1}, {16384, 5, 8, 0}, {16384, 8, 8, 1}, {16384, 12, 8, 1}, {8192, 10, 8, 1}, {32768, 3, 8, 1}, {32768, 6, 8, 1}, {65536, 3, 8, 1}, {16384, 5, 1, 1}};
  for (auto& c : cfg) {
    const int CH = c[0], NS = c[1], NC = c[2], hint = c[3];
    const size_t smem = (size_t)CH * NS;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k<<<148, 32 * (1 + NC), smem>>>(src, total / 148, CH, NS, NC, hint, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) k<<<148, 32 * (1 + NC), smem>>>(src, total / 148, CH, NS, NC, hint, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    if (err) { printf("CH=%d NS=%d: %s\n", CH, NS, cudaGetErrorString(err)); continue; }
    printf("CH=%6d NS=%2d (in flight %4d KB) NC=%d hint=%d: %.0f GB/s\n", CH, NS, CH * NS / 1024, NC, hint, 10.0 * total / (ms * 1e-3) / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
