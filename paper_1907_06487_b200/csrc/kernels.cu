// sm_100a SymmSpMV kernels (Alg. 2).  No tensor cores: the
// operation is an HBM-bound sparse stream (I = 0.16-0.27 flop/B, §3.2 Eq. 3).
//
//  K1 k_atomic     one launch; V lanes per row; row sums reduced by shuffles;
//                  transposed updates y[c] += a x[r] with native fp64 RED.
//  K2 k_colored    one launch per phase (tiles of one colour); inside a tile the
//                  rows of one intra-tile colour are write-disjoint -> plain
//                  read-modify-write of y in L2, __syncthreads between colours.
//  K3 k_tiled      persistent dataflow kernel: each CTA claims tiles in a
//                  topological order, stages x of the tile's window (own rows +
//                  targets) in shared memory, accumulates y in shared memory
//                  colour by colour, then waits for its predecessor tiles
//                  (RACE's local synchronisation) and
//                  flushes the window to y in a fixed order -> deterministic.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace symm {
namespace {

__device__ __forceinline__ int ld_stream_i32(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned short ld_stream_u16(const unsigned short* p) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ double group_sum(double s) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, V);
  return s;
}

// ---------------------------------------------------------------- zero / gather
__global__ void k_zero(double* __restrict__ y, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) y[i] = 0.0;
}

__global__ void k_gather(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                         int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[idx[i]];
}
__global__ void k_scatter(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                          int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[idx[i]] = src[i];
}

// ---------------------------------------------------------------- K1 atomic
template <int V>
__global__ void __launch_bounds__(256) k_atomic(CsrArgs A, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / V;  // rows per warp per step
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * RPW; base < A.n; base += nwarps * RPW) {  // warp-uniform
    const int64_t row = base + lane / V;
    const bool valid = row < A.n;
    double sum = 0.0;
    if (valid) {
      const int b = A.row_ptr[row], e = A.row_ptr[row + 1];
      const double xr = x[row];
      for (int i = b + sub; i < e; i += V) {
        const int c = ld_stream_i32(A.col + i);
        const double a = ld_stream_f64(A.val + i);
        if (c == (int)row) {
          sum += a * xr;  // diagonal contributes once (reading R1)
        } else {
          sum += a * __ldg(x + c);   // tmp += A[idx] * x[col[idx]]
          atomicAdd(y + c, a * xr);  // b[col[idx]] += A[idx] * x[row]  (RED.F64)
        }
      }
    }
    sum = group_sum<V>(sum);
    if (valid && sub == 0) atomicAdd(y + row, sum);  // b[row] += tmp
  }
}

// ---------------------------------------------------------------- K2 colored
template <int V>
__global__ void __launch_bounds__(256) k_colored(CsrArgs A, ColoredArgs C, const double* __restrict__ x,
                                                 double* __restrict__ y) {
  constexpr int RPW = 32 / V;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int t = C.phase_tiles[blockIdx.x];
  const int r0 = C.tile_ptr[t];
  const int* sp = C.sub_ptr + C.tile_sub_ptr[t];
  const int nsub = C.tile_sub_ptr[t + 1] - C.tile_sub_ptr[t] - 1;
  for (int s = 0; s < nsub; ++s) {
    const int qa = r0 + sp[s], qb = r0 + sp[s + 1];
    for (int base = qa + wid * RPW; base < qb; base += nw * RPW) {
      const int q = base + lane / V;
      const bool valid = q < qb;
      double sum = 0.0;
      int row = 0;
      if (valid) {
        row = C.srow[q];
        const int b = A.row_ptr[row], e = A.row_ptr[row + 1];
        const double xr = x[row];
        for (int i = b + sub; i < e; i += V) {
          const int c = ld_stream_i32(A.col + i);
          const double a = ld_stream_f64(A.val + i);
          if (c == row) {
            sum += a * xr;
          } else {
            sum += a * __ldg(x + c);
            __stcg(y + c, __ldcg(y + c) + a * xr);  // write-disjoint inside the colour
          }
        }
      }
      sum = group_sum<V>(sum);
      if (valid && sub == 0) __stcg(y + row, __ldcg(y + row) + sum);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K3 tiled dataflow
constexpr int kTiledThreads = 512;

template <int V>
__global__ void __launch_bounds__(kTiledThreads, 2) k_tiled(TiledArgs A, const double* __restrict__ x,
                                                            double* __restrict__ y) {
  extern __shared__ double smem[];
  double* xs = smem;
  double* ys = smem + A.window_cap;
  __shared__ long long s_claim;
  constexpr int RPW = 32 / V;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int sub = lane % V;
  const int wid = tid >> 5;
  constexpr int NW = kTiledThreads / 32;
  unsigned long long* counter = A.counter;
  for (;;) {
    if (tid == 0) s_claim = (long long)(atomicAdd(counter, 1ull) - A.claim_base);
    __syncthreads();
    const long long ti = s_claim;
    if (ti >= A.ntiles) break;
    const TileDesc D = A.tiles[ti];
    const int T = D.nrows, S = D.nspill;
    const int32_t* spill = A.spill + D.spill_off;
    // stage the window of x; clear the window of y
    for (int i = tid; i < T; i += kTiledThreads) {
      xs[i] = x[D.row0 + i];
      ys[i] = 0.0;
    }
    for (int i = tid; i < S; i += kTiledThreads) {
      xs[T + i] = x[(uint32_t)spill[i] & kIdxMask];
      ys[T + i] = 0.0;
    }
    __syncthreads();
    const int* sp = A.sub_ptr + D.sub_off;
    const int32_t* start = A.srow_start + D.srow_off + ti;  // T+1 entries per tile
    const uint16_t* lrow = A.srow_lrow + D.srow_off;
    const uint16_t* lcol = A.lcol + D.nnz_off;
    const double* val = A.val + D.nnz_off;
    for (int s = 0; s < D.nsub; ++s) {
      const int qa = sp[s], qb = sp[s + 1];
      for (int base = qa + wid * RPW; base < qb; base += NW * RPW) {
        const int q = base + lane / V;
        const bool valid = q < qb;
        double sum = 0.0;
        int lr = 0;
        if (valid) {
          lr = lrow[q];
          const int eb = start[q], ee = start[q + 1];
          const double xr = xs[lr];
          for (int e = eb + sub; e < ee; e += V) {
            const int lc = ld_stream_u16(lcol + e);
            const double a = ld_stream_f64(val + e);
            sum += a * xs[lc];
            if (lc != lr) ys[lc] += a * xr;  // write-disjoint inside the colour
          }
        }
        sum = group_sum<V>(sum);
        if (valid && sub == 0) ys[lr] += sum;
      }
      __syncthreads();
    }
    // local synchronisation: wait until every conflicting earlier-phase tile flushed
    for (int i = tid; i < D.npred; i += kTiledThreads) {
      const unsigned int* f = A.done + A.pred[D.pred_off + i];
      while (ld_acquire_u32(f) != A.epoch) __nanosleep(64);
      __threadfence();
    }
    __syncthreads();
    const uint32_t* ownf = A.own_first + D.flag_off;
    for (int i = tid; i < T; i += kTiledThreads) {
      const bool first = (ownf[i >> 5] >> (i & 31)) & 1u;
      double* p = y + D.row0 + i;
      __stcg(p, first ? ys[i] : __ldcg(p) + ys[i]);
    }
    for (int i = tid; i < S; i += kTiledThreads) {
      const uint32_t e = (uint32_t)spill[i];
      double* p = y + (e & kIdxMask);
      __stcg(p, (e & kFirstBit) ? ys[T + i] : __ldcg(p) + ys[T + i]);
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_u32(A.done + D.id, A.epoch);
  }
}

int grid_for(int64_t work, int threads) {
  int64_t g = (work + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return (int)g;
}

}  // namespace

int launch_zero(double* y, int64_t n, void* stream) {
  if (n <= 0) return 0;
  k_zero<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(y, n);
  return (int)cudaGetLastError();
}
int launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream) {
  if (n <= 0) return 0;
  k_gather<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, idx, dst, n);
  return (int)cudaGetLastError();
}
int launch_scatter(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream) {
  if (n <= 0) return 0;
  k_scatter<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, idx, dst, n);
  return (int)cudaGetLastError();
}

int launch_atomic(const CsrArgs& A, const double* x, double* y, int vec, int sms, void* stream) {
  if (A.n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  int64_t warps_needed = ((int64_t)A.n * vec + 31) / 32;
  int64_t g = (warps_needed * 32 + threads - 1) / threads;
  int64_t gmax = (int64_t)sms * 8;
  int grid = (int)(g < gmax ? (g < 1 ? 1 : g) : gmax);
  switch (vec) {
    case 1: k_atomic<1><<<grid, threads, 0, st>>>(A, x, y); break;
    case 2: k_atomic<2><<<grid, threads, 0, st>>>(A, x, y); break;
    case 4: k_atomic<4><<<grid, threads, 0, st>>>(A, x, y); break;
    case 8: k_atomic<8><<<grid, threads, 0, st>>>(A, x, y); break;
    case 16: k_atomic<16><<<grid, threads, 0, st>>>(A, x, y); break;
    default: k_atomic<32><<<grid, threads, 0, st>>>(A, x, y); break;
  }
  return (int)cudaGetLastError();
}

int launch_colored_phase(const CsrArgs& A, const ColoredArgs& C, const double* x, double* y, int vec,
                         void* stream) {
  if (C.nphase_tiles <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  switch (vec) {
    case 1: k_colored<1><<<C.nphase_tiles, threads, 0, st>>>(A, C, x, y); break;
    case 2: k_colored<2><<<C.nphase_tiles, threads, 0, st>>>(A, C, x, y); break;
    case 4: k_colored<4><<<C.nphase_tiles, threads, 0, st>>>(A, C, x, y); break;
    case 8: k_colored<8><<<C.nphase_tiles, threads, 0, st>>>(A, C, x, y); break;
    case 16: k_colored<16><<<C.nphase_tiles, threads, 0, st>>>(A, C, x, y); break;
    default: k_colored<32><<<C.nphase_tiles, threads, 0, st>>>(A, C, x, y); break;
  }
  return (int)cudaGetLastError();
}

int tiled_smem_bytes(int window_cap) { return 2 * window_cap * (int)sizeof(double); }

template <int V>
static int tiled_setup(int smem) {
  return (int)cudaFuncSetAttribute(k_tiled<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

int tiled_max_ctas_per_sm(int vec, int window_cap, int* out) {
  const int smem = tiled_smem_bytes(window_cap);
  int rc = 0, occ = 0;
  switch (vec) {
#define OCC(VV)                                                                             \
  case VV:                                                                                  \
    rc = tiled_setup<VV>(smem);                                                             \
    if (!rc) rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<VV>,     \
                                                                     kTiledThreads, smem);  \
    break;
    OCC(1) OCC(2) OCC(4) OCC(8) OCC(16) OCC(32)
#undef OCC
    default: rc = (int)cudaErrorInvalidValue;
  }
  *out = occ;
  return rc;
}

int launch_tiled(const TiledArgs& T, const double* x, double* y, int vec, int grid, void* stream) {
  if (T.ntiles <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = tiled_smem_bytes(T.window_cap);
  switch (vec) {
    case 1: k_tiled<1><<<grid, kTiledThreads, smem, st>>>(T, x, y); break;
    case 2: k_tiled<2><<<grid, kTiledThreads, smem, st>>>(T, x, y); break;
    case 4: k_tiled<4><<<grid, kTiledThreads, smem, st>>>(T, x, y); break;
    case 8: k_tiled<8><<<grid, kTiledThreads, smem, st>>>(T, x, y); break;
    case 16: k_tiled<16><<<grid, kTiledThreads, smem, st>>>(T, x, y); break;
    default: k_tiled<32><<<grid, kTiledThreads, smem, st>>>(T, x, y); break;
  }
  return (int)cudaGetLastError();
}

}  // namespace symm
