// LDS.64 wavefront rule probe: lanes of each half warp on distinct bank pairs
// but scattered over different 128-B lines (as K4's placed row segments) vs
// consecutive addresses vs the same pattern with the halves interleaved.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters) {
  __shared__ double ys[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) ys[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int base;
  const int h = lane >> 4, i = lane & 15;
  if (MODE == 0) base = w * 32 + lane;                                   // consecutive
  else if (MODE == 1) base = 16 * ((i * 7 + h * 3 + w) & 127) + ((i * 5 + 3) & 15);  // distinct pair per half, scattered lines
  else if (MODE == 2) base = 16 * ((i * 7 + w) & 127) + ((lane * 5 + 3) & 15);        // pairs distinct over 16 lanes, halves share pairs
  else base = 16 * ((lane * 13 + w) & 127) + ((lane * 3) & 7);           // only 8 distinct pairs per half (2-way)
  double acc = 0;
  for (int it = 0; it < iters; ++it) acc += ys[(base + it * 16) & 4095];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 2 * 512 * 8);
  const int iters = 8192;
  const char* nm[4] = {"consecutive", "distinct pairs/half, scattered lines", "pairs shared across halves", "2-way per half"};
  for (int mode = 0; mode < 4; ++mode) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<296, 512>>>(o, iters);
      if (mode == 1) k<1><<<296, 512>>>(o, iters);
      if (mode == 2) k<2><<<296, 512>>>(o, iters);
      if (mode == 3) k<3><<<296, 512>>>(o, iters);
      cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    double ops = 296.0 * 512 * iters;
    printf("%-40s %.3f ms  %.2f lanes/clk/SM (1.9 GHz)\n", nm[mode], ms, ops / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
