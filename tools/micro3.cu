// smem: cost of x[c] load + y[c] read-modify-write per lane when the 32 lanes'
// c are random vs bank-pair conflict-free (c mod 16 distinct per half warp).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
template <int PAT>
__global__ void k(double* out, int W, int iters) {
  extern __shared__ double s[];
  double* xs = s; double* ys = s + W;
  for (int i = threadIdx.x; i < 2 * W; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int idx[8];
  uint32_t h = hash32(blockIdx.x * blockDim.x + threadIdx.x + 7);
  // warp-uniform random base per u so that distinct warps touch different lines
  uint32_t hw = hash32((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    h = hash32(h + u); hw = hash32(hw + u);
    if (PAT == 0) idx[u] = h % W;                                             // random
    if (PAT == 1) idx[u] = ((hw + (h % (W / 16)) * 16) + (lane & 15)) % W;    // bank pair = lane%16 (+const)
    if (PAT == 2) idx[u] = ((hw + (h % (W / 16)) * 16) + (lane >> 1)) % W;    // two lanes per bank pair
    if (PAT == 3) idx[u] = ((hw + (h % (W / 16)) * 16) + ((lane & 15) ^ (lane >> 4))) % W;
  }
  double acc = 0, a = 1.0000001;
  for (int it = 0; it < iters; ++it) {
    double yv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { const int c = idx[u]; acc += xs[c]; yv[u] = ys[c]; }
#pragma unroll
    for (int u = 0; u < 8; ++u) { const int c = idx[u]; ys[c] = fma(a, acc, yv[u]); }
    a += 1e-9;
  }
  if (acc == 1.2345) out[blockIdx.x] = acc;
}
int main() {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double* out; cudaMalloc(&out, 1 << 20);
  const double clk = 1.92e9 * 148;
  void (*ks[4])(double*, int, int) = {k<0>, k<1>, k<2>, k<3>};
  const char* nm[4] = {"random", "bankpair=lane%16", "2 lanes/bankpair", "bankpair=lane%16^half"};
  for (int p = 0; p < 4; ++p) for (int W : {1024, 4096}) {
    const int thr = 512, blocks = 148 * 2, iters = 400;
    const size_t sm = 2 * W * 8;
    cudaFuncSetAttribute(ks[p], cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    ks[p]<<<blocks, thr, sm>>>(out, W, iters);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) ks[p]<<<blocks, thr, sm>>>(out, W, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double ops = 5.0 * blocks * thr * iters * 8;
    printf("%-24s W=%d: %.2f entries (LDS x + RMW y) per SM-clk\n", nm[p], W, ops / (ms * 1e-3) / clk);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
