// Round-2 design probes (B200, sm_100a):
//  A. shared-memory f64 push y[c] += v: CAS-loop atomicAdd vs plain LDS+STS
//     vs LDS only, random addresses in a W-double window, 8 independent pushes
//     per thread in flight (ILP), 1 CTA x 1024 threads per SM
//  B. L2-resident fp64 RED.ADD (random, region R bytes) and random 8-B loads
//  C. streaming read bandwidth (load-only, 16-B vector loads) -> load-only
//     roofline denominator probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int MODE>
__global__ void __launch_bounds__(1024, 1) ksm(double* out, int W, int iters) {
  extern __shared__ double ys[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) ys[i] = 0;
  __syncthreads();
  uint32_t h = hash32(blockIdx.x * 1024 + threadIdx.x + 1);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    int a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { h = hash32(h + u); a[u] = h % W; }
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) atomicAdd(&ys[a[u]], 1.0);
    } else if (MODE == 1) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = ys[a[u]];
#pragma unroll
      for (int u = 0; u < 8; ++u) ys[a[u]] = v[u] + 1.0;
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += ys[a[u]];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = ys[0] + acc;
}
template <int MODE>
__global__ void __launch_bounds__(512) kl2(double* buf, size_t nel, int iters, double* out) {
  uint32_t h = hash32(blockIdx.x * 512 + threadIdx.x + 7);
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    size_t a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { h = hash32(h + u); a[u] = h % nel; }
    if (MODE == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) atomicAdd(buf + a[u], 1.0);
    } else {
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += __ldcg(buf + a[u]);
    }
  }
  if (acc == 1.5) out[0] = acc;
}
__global__ void kread(const double4* __restrict__ p, size_t n4, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p + i));
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1.5) out[0] = s;
}
int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* out; cudaMalloc(&out, 1 << 20);
  int clk_khz; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double clk = clk_khz * 1e3;
  printf("clock %.0f MHz\n", clk / 1e6);
  // A
  void (*ks[3])(double*, int, int) = {ksm<0>, ksm<1>, ksm<2>};
  const char* nm[3] = {"CAS atomicAdd", "LDS+STS", "LDS"};
  for (int m = 0; m < 3; ++m)
    for (int W : {1024, 4096, 16384}) {
      const int iters = 200;
      cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      ks[m]<<<148, 1024, W * 8>>>(out, W, iters);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) ks[m]<<<148, 1024, W * 8>>>(out, W, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 5.0 * 148 * 1024 * iters * 8;
      printf("A smem %-14s W=%5d: %.2f pushes/clk/SM  (%.1f G/s total)\n", nm[m], W, ops / (ms * 1e-3) / clk / 148, ops / (ms * 1e-3) / 1e9);
    }
  // B
  double* buf; const size_t maxb = (size_t)1 << 31;
  cudaMalloc(&buf, maxb); cudaMemset(buf, 0, maxb);
  for (int m = 0; m < 2; ++m)
    for (size_t R : {(size_t)8 << 20, (size_t)32 << 20, (size_t)64 << 20, (size_t)1 << 31}) {
      const int iters = 64, blocks = 148 * 4;
      void (*kk)(double*, size_t, int, double*) = m == 0 ? kl2<0> : kl2<1>;
      kk<<<blocks, 512>>>(buf, R / 8, iters, out);
      cudaEventRecord(e0);
      for (int r = 0; r < 3; ++r) kk<<<blocks, 512>>>(buf, R / 8, iters, out);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 3.0 * blocks * 512 * iters * 8;
      printf("B L2 %-10s region %6zu MB: %.1f G ops/s\n", m == 0 ? "RED.F64" : "LDG.8 rnd", R >> 20, ops / (ms * 1e-3) / 1e9);
    }
  // C
  for (int bl : {148 * 4, 148 * 8, 148 * 16}) {
    const size_t n4 = maxb / 32;
    kread<<<bl, 512>>>((const double4*)buf, n4, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kread<<<bl, 512>>>((const double4*)buf, n4, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("C load-only stream 2 GiB, %d CTAs x 512: %.1f GB/s\n", bl, 5.0 * maxb / (ms * 1e-3) / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
