// Microbenchmarks for the SymmSpMV kernel design (B200, sm_100a).
//   1 global RED.F64 throughput (random / windowed addresses in an L2-resident vector)
//   2 shared-memory f64 add via CAS loop (the only fp64 smem atomic on sm_100a)
//   3 shared-memory random LDS.64
//   4 streaming LDG.128 read bandwidth
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro tools/micro.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// 1: each thread issues `per` REDs; address = base window + hash % win
__global__ void k_red(double* y, int n, int win, int per) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  for (int k = 0; k < per; ++k) {
    const uint32_t i = t + k * nt;
    // window slides with i so that consecutive ops hit a local band (like BFS order)
    const uint32_t base = (uint32_t)(((uint64_t)i * (uint64_t)(n - win)) / ((uint64_t)nt * per));
    const uint32_t a = base + hash32(i) % win;
    atomicAdd(y + a, 1.0);
  }
}

// 2: smem CAS add, random addresses in a window of W doubles
__global__ void k_scas(double* out, int W, int per) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
  for (int k = 0; k < per; ++k) {
    h = hash32(h + k);
    atomicAdd(s + (h % W), 1.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
// 3: random LDS.64
__global__ void k_slds(double* out, int W, int per) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) s[i] = i;
  __syncthreads();
  uint32_t h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
  double acc = 0;
  for (int k = 0; k < per; ++k) {
    h = hash32(h + k);
    acc += s[h % W];
  }
  if (acc == 12345.0) out[blockIdx.x] = acc;
}
// 3b: random LDS.64 + plain STS (non-atomic RMW), to compare with CAS
__global__ void k_srmw(double* out, int W, int per) {
  extern __shared__ double s[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) s[i] = i;
  __syncthreads();
  uint32_t h = hash32(blockIdx.x * blockDim.x + threadIdx.x);
  for (int k = 0; k < per; ++k) {
    h = hash32(h + k);
    volatile double* p = s + (h % W);
    *p = *p + 1.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
// 4: streaming read
__global__ void k_stream(const double4* a, size_t n4, double* out) {
  double acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(a + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const int n = 2097152;
  double* y; cudaMalloc(&y, n * 8); cudaMemset(y, 0, n * 8);
  double* out; cudaMalloc(&out, 1 << 20);
  // 1 RED
  for (int win : {4096, 65536, 1 << 20}) {
    for (int blocks : {148 * 4, 148 * 8}) {
      const int per = 64, thr = 256;
      k_red<<<blocks, thr>>>(y, n, win, per);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_red<<<blocks, thr>>>(y, n, win, per);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double ops = 5.0 * blocks * thr * per;
      printf("RED.F64 win=%8d blocks=%d: %.1f G/s\n", win, blocks, ops / (ms * 1e-3) / 1e9);
    }
  }
  // 2/3 smem
  for (int W : {2048, 8192}) {
    for (int thr : {256, 512, 1024}) {
      const int blocks = 148 * (2048 / thr), per = 256;
      const size_t sm = W * 8;
      cudaFuncSetAttribute(k_scas, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      cudaFuncSetAttribute(k_slds, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      cudaFuncSetAttribute(k_srmw, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
      k_scas<<<blocks, thr, sm>>>(out, W, per);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_scas<<<blocks, thr, sm>>>(out, W, per);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      double ops = 5.0 * blocks * thr * per;
      double clk = 1.9e9 * 148;
      printf("smem CAS-add W=%d thr=%d: %.1f G/s = %.2f per SM-clk\n", W, thr, ops / (ms * 1e-3) / 1e9, ops / (ms * 1e-3) / clk);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_slds<<<blocks, thr, sm>>>(out, W, per);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("smem LDS.64   W=%d thr=%d: %.1f G/s = %.2f per SM-clk\n", W, thr, ops / (ms * 1e-3) / 1e9, ops / (ms * 1e-3) / clk);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) k_srmw<<<blocks, thr, sm>>>(out, W, per);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      printf("smem RMW      W=%d thr=%d: %.1f G/s = %.2f per SM-clk\n", W, thr, ops / (ms * 1e-3) / 1e9, ops / (ms * 1e-3) / clk);
    }
  }
  // 4 stream
  size_t bytes = (size_t)1 << 30;
  double4* a; cudaMalloc(&a, bytes); cudaMemset(a, 0, bytes);
  for (int blocks : {148, 148 * 2, 148 * 4, 148 * 8}) {
    k_stream<<<blocks, 512>>>(a, bytes / 32, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k_stream<<<blocks, 512>>>(a, bytes / 32, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("stream LDG.256 blocks=%d x512: %.1f GB/s\n", blocks, 5.0 * bytes / (ms * 1e-3) / 1e9);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
