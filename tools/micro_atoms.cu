// Shared-memory f64 add throughput on sm_100a: CAS-loop atomicAdd (ATOMS.CAST.SPIN.64)
// vs plain LDS+STS read-modify-write vs LDS only; conflict-free lane -> address map.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, int stride) {
  __shared__ double ys[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) ys[i] = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int a = ((w * 32 + lane * stride + it * 97) & 4095);
    if (MODE == 0) atomicAdd(&ys[a], 1.0);
    else if (MODE == 1) ys[a] = ys[a] + 1.0;
    else acc += ys[a];
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = ys[0] + acc;
}
int main() {
  double* o; cudaMalloc(&o, 4096 * 8);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int stride : {1, 2}) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k<0><<<148 * 2, 512>>>(o, iters, stride);
        if (mode == 1) k<1><<<148 * 2, 512>>>(o, iters, stride);
        if (mode == 2) k<2><<<148 * 2, 512>>>(o, iters, stride);
        cudaEventRecord(b); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      double ops = 148.0 * 2 * 512 * iters;
      printf("mode %d (%s) stride %d: %.3f ms, %.2f ops/clk/SM at 1.9 GHz\n", mode, mode == 0 ? "atomicAdd CAS" : mode == 1 ? "LDS+STS" : "LDS", stride, ms, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
  return 0;
}
