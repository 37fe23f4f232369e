// Microbenchmarks, round 2: shared-memory random access costs with negligible
// ALU overhead (indices precomputed in registers), and RED coalescing.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
// MODE 0: LDS.64 x[c]; 1: LDS.64 x[c] + RMW y[c] (separate arrays); 2: LDS.128 xy[c] + STS.64 y; 3: RMW only
template <int MODE>
__global__ void k_sm(double* out, int W, int iters) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < 2 * W; i += blockDim.x) s[i] = i;
  __syncthreads();
  int idx[16];
  uint32_t h = hash32(blockIdx.x * blockDim.x + threadIdx.x + 1);
#pragma unroll
  for (int u = 0; u < 16; ++u) { h = hash32(h + u); idx[u] = h % W; }
  double acc = 0, a = 1.0000001;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int c = idx[u] ^ (it & 1);
      if (MODE == 0) acc += s[c];
      if (MODE == 1) { acc += s[c]; s[W + c] = fma(a, acc, s[W + c]); }
      if (MODE == 2) { double2 v = reinterpret_cast<double2*>(s)[c]; acc += v.x; s[2 * c + 1] = fma(a, acc, v.y); }
      if (MODE == 3) { s[W + c] = fma(a, 1.0, s[W + c]); }
    }
  }
  if (acc == 1.2345) out[blockIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] += s[W];
}
__global__ void k_red(double* y, int n, int per, int mode) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  for (int k = 0; k < per; ++k) {
    uint32_t i = t + k * nt;
    uint32_t a = mode == 0 ? (i % n) : (hash32(i) % n);  // 0: coalesced (warp = 256 contiguous bytes)
    atomicAdd(y + a, 1.0);
  }
}
__global__ void k_st(double* y, int n, int per, int mode) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  for (int k = 0; k < per; ++k) {
    uint32_t i = t + k * nt;
    uint32_t a = mode == 0 ? (i % n) : (hash32(i) % n);
    y[a] = (double)k;
  }
}
int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* out; cudaMalloc(&out, 1 << 20);
  const double clk = 1.92e9 * 148;
  for (int mode = 0; mode < 4; ++mode)
    for (int W : {1024, 4096}) {
      const int thr = 512, blocks = 148 * 2, iters = 200;
      const size_t sm = 2 * W * 8;
      void (*k)(double*, int, int) = mode == 0 ? k_sm<0> : mode == 1 ? k_sm<1> : mode == 2 ? k_sm<2> : k_sm<3>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
      k<<<blocks, thr, sm>>>(out, W, iters);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k<<<blocks, thr, sm>>>(out, W, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double ops = 5.0 * blocks * thr * iters * 16;
      printf("smem mode %d (0 LDS64, 1 LDS64+RMW64, 2 LDS128+STS64, 3 RMW64) W=%d: %.2f entries per SM-clk\n", mode, W, ops / (ms * 1e-3) / clk);
    }
  const int n = 1 << 21;
  double* y; cudaMalloc(&y, n * 8); cudaMemset(y, 0, n * 8);
  for (int mode = 0; mode < 2; ++mode) {
    const int blocks = 148 * 8, thr = 256, per = 64;
    k_red<<<blocks, thr>>>(y, n, per, mode);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_red<<<blocks, thr>>>(y, n, per, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("RED.F64 %s: %.1f G/s\n", mode ? "random" : "coalesced", 5.0 * blocks * thr * per / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_st<<<blocks, thr>>>(y, n, per, mode);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("ST.64   %s: %.1f G/s\n", mode ? "random" : "coalesced", 5.0 * blocks * thr * per / (ms * 1e-3) / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
