// sm_100a SymmSpMV kernels (Alg. 2).  No tensor cores: the
// operation is an HBM-bound sparse stream (I = 0.16-0.27 flop/B, §3.2 Eq. 3).
//
//  K1 k_atomic     one launch; V lanes per row; row sums reduced by shuffles;
//                  transposed updates y[c] += a x[r] with native fp64 RED.
//  K2 k_colored    one launch per phase (tiles of one colour); inside a tile the
//                  rows of one intra-tile colour are write-disjoint -> plain
//                  read-modify-write of y in L2, __syncthreads between colours.
//  K3 k_tiled      persistent owner-computes kernel: TMA bulk copies of whole
//                  tile blocks into double-buffered smem, two conflict-free smem
//                  passes, staged cross-tile contributions with depth-1
//                  dependencies -> deterministic, y written once (see below).
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

// ---------------------------------------------------------------- K3 tiled (owner computes)
// Per tile (one CTA at a time, persistent grid, tiles claimed in BFS order):
//   1. the whole tile block (matrix entries + CSC of the tile) arrives by one
//      cp.async.bulk (TMA) into a double-buffered smem slot; the NEXT tile's
//      block is already in flight while this one is computed;
//   2. x of the tile window (own rows + spill targets) is gathered to smem;
//   3. pass 1 (rows):    ys[i] = sum_e a_e x[c_e]          (tmp)
//                        P[e]  = a_e x[i] for off-diagonal e
//      pass 2 (targets): ys[l] += sum_{e: c_e = l} P[e]  (b[col] += ...)
//      both passes are conflict-free and in a fixed order -> deterministic;
//   4. contributions to rows of later tiles (spill) are staged in spill_buf,
//      then the tile publishes `ready`;
//   5. the owner of a row waits only for the tiles that wrote into its rows
//      (all earlier in claim order, none of them waits before publishing:
//      dependency depth 1, RACE's "local synchronisation"),
//      adds their staged contributions in slot order and stores y once.
// y is written exactly once per row: no pre-zeroing, no atomics.
constexpr int kTiledThreads = 512;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void issue_tile(const TiledArgs& A, long long t, unsigned char* buf, uint64_t* bar) {
  const TileDesc& D = A.tiles[t];
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, (unsigned)D.block_bytes);
  bulk_g2s(buf, A.blocks + D.block_off, (unsigned)D.block_bytes, bar);
}

template <int V>
__global__ void __launch_bounds__(kTiledThreads) k_tiled(TiledArgs A, const double* __restrict__ x,
                                                         double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ long long s_next;
  unsigned char* buf0 = sm;
  unsigned char* buf1 = sm + A.block_cap;
  double* xs = reinterpret_cast<double*>(sm + 2 * (size_t)A.block_cap);
  double* ys = xs + A.window_cap;
  double* Pp = ys + A.window_cap;
  constexpr int RPW = 32 / V;
  constexpr int NW = kTiledThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31, sub = lane % V, wid = tid >> 5;
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    long long t = (long long)(atomicAdd(A.counter, 1ull) - A.claim_base);
    s_next = t;
    if (t < A.ntiles) issue_tile(A, t, buf0, &mbar[0]);
  }
  __syncthreads();
  long long cur = s_next;
  int b = 0;
  unsigned par0 = 0, par1 = 0;
  while (cur < A.ntiles) {
    __syncthreads();  // every thread has read s_next
    if (tid == 0) {
      long long t = (long long)(atomicAdd(A.counter, 1ull) - A.claim_base);
      s_next = t;
      if (t < A.ntiles) issue_tile(A, t, b ? buf0 : buf1, b ? &mbar[0] : &mbar[1]);
    }
    const TileDesc D = A.tiles[cur];
    const int T = D.nrows, S = D.nspill, W = T + S;
    const I2* pairs = A.pairs + D.spill_off;
    for (int i = tid; i < T; i += kTiledThreads) xs[i] = x[D.row0 + i];
    for (int i = tid; i < S; i += kTiledThreads) xs[T + i] = __ldg(x + pairs[i].x);
    unsigned char* blk = b ? buf1 : buf0;
    if (b) { mbar_wait(&mbar[1], par1); par1 ^= 1u; }
    else { mbar_wait(&mbar[0], par0); par0 ^= 1u; }
    __syncthreads();
    const uint16_t* start = reinterpret_cast<const uint16_t*>(blk);
    const uint16_t* lcol = reinterpret_cast<const uint16_t*>(blk + D.o_lcol);
    const uint16_t* tidx = reinterpret_cast<const uint16_t*>(blk + D.o_tidx);
    const uint16_t* tptr = reinterpret_cast<const uint16_t*>(blk + D.o_tptr);
    const double* val = reinterpret_cast<const double*>(blk + D.o_val);
    // pass 1: rows (V lanes per row)
    for (int base = wid * RPW; base < T; base += NW * RPW) {
      const int i = base + lane / V;
      double sum = 0.0;
      if (i < T) {
        const int eb = start[i], ee = start[i + 1];
        const double xi = xs[i];
        for (int e = eb + sub; e < ee; e += V) {
          const int c = lcol[e];
          const double a = val[e];
          sum += a * xs[c];
          if (c != i) Pp[e] = a * xi;
        }
      }
      sum = group_sum<V>(sum);
      if (i < T && sub == 0) ys[i] = sum;
    }
    __syncthreads();
    // pass 2: targets (one thread per local target, entries in stored order)
    for (int l = tid; l < W; l += kTiledThreads) {
      double acc = l < T ? ys[l] : 0.0;
      const int jb = tptr[l], je = tptr[l + 1];
      for (int j = jb; j < je; ++j) acc += Pp[tidx[j]];
      ys[l] = acc;
    }
    __syncthreads();
    // stage contributions to later tiles' rows, then publish
    for (int i = tid; i < S; i += kTiledThreads) __stcg(A.spill_buf + pairs[i].y, ys[T + i]);
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release_u32(A.ready + cur, A.epoch);
    // wait for the writers of this tile's rows (all claimed earlier)
    for (int k = tid; k < D.nwr; k += kTiledThreads) {
      const unsigned int* f = A.ready + A.writers[D.wr_off + k];
      while (ld_acquire_u32(f) != A.epoch) __nanosleep(32);
      __threadfence();
    }
    __syncthreads();
    const int32_t* ip = A.in_ptr + D.in_off;
    const double* inb = A.spill_buf + D.in_base;
    for (int i = tid; i < T; i += kTiledThreads) {
      double acc = ys[i];
      const int jb = ip[i], je = ip[i + 1];
      for (int j = jb; j < je; ++j) acc += __ldcg(inb + j);
      y[D.row0 + i] = acc;
    }
    __syncthreads();
    cur = s_next;
    b ^= 1;
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

int tiled_smem_bytes(const TiledArgs& T) {
  return 2 * T.block_cap + 2 * T.window_cap * 8 + T.nnz_cap * 8;
}

template <int V>
static int tiled_setup(int smem) {
  return (int)cudaFuncSetAttribute(k_tiled<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

int tiled_max_ctas_per_sm(int vec, const TiledArgs& T, int* out) {
  const int smem = tiled_smem_bytes(T);
  int rc = 0, occ = 0;
  switch (vec) {
#define OCC(VV)                                                                                                \
  case VV:                                                                                                     \
    rc = tiled_setup<VV>(smem);                                                                                \
    if (!rc) rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<VV>, kTiledThreads, smem); \
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
  const int smem = tiled_smem_bytes(T);
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
