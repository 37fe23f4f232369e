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
// Warp-specialised persistent kernel, tiles claimed in BFS order:
//   producer warp: claims a tile, TMA-bulk-copies its block (matrix entries +
//     CSC of the tile + staging slots) and cp.async-gathers x of the tile
//     window (own rows + spill targets) into a 2-stage smem ring
//     (mbarrier full/empty per stage);
//   16 consumer warps:
//     pass 1 (rows):    ys[i] = sum_e a_e x[c_e]            (tmp)
//                       P[e]  = a_e x[i] for off-diagonal e
//     pass 2 (targets): ys[l] += sum_{e: c_e = l} P[e]    (b[col] += ...)
//     -> conflict-free, fixed order, deterministic; then contributions to
//     rows of later tiles are staged in spill_buf, the tile waits only for the
//     earlier tiles that wrote into its own rows (depth-1 dependencies: RACE's
//     local synchronisation), adds their staged values in
//     slot order and stores y once.  No pre-zeroing, no atomics on y.
constexpr int kStages = 2;
constexpr int kConsumerWarps = 16;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kTiledThreads = kConsumers + 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory"); }

template <int V>
__global__ void __launch_bounds__(kTiledThreads) k_tiled(TiledArgs A, const double* __restrict__ x,
                                                         double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
  __shared__ long long slot_tile[kStages];
  const size_t slot_bytes = (size_t)A.block_cap + 8 * (size_t)A.window_cap;
  double* ys = reinterpret_cast<double*>(sm + kStages * slot_bytes);
  double* Pp = ys + A.window_cap;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 33);  // 32 producer lanes (cp.async noinc) + 1 expect_tx arrive
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (wid == kConsumerWarps) {
    // ------------------------------------------------ producer warp
    for (int k = 0;; ++k) {
      const int s = k % kStages;
      const int use = k / kStages;
      if (use > 0) mbar_wait(&empty[s], (unsigned)((use - 1) & 1));
      long long t = 0;
      if (lane == 0) t = (long long)(atomicAdd(A.counter, 1ull) - A.claim_base);
      t = __shfl_sync(0xffffffffu, t, 0);
      unsigned char* blk = sm + s * slot_bytes;
      double* xsl = reinterpret_cast<double*>(blk + A.block_cap);
      if (t >= A.ntiles) {
        if (lane == 0) {
          slot_tile[s] = t;
          mbar_arrive(&full[s]);
        }
        cp_async_arrive_noinc(&full[s]);
        break;
      }
      const TileDesc& D = A.tiles[t];
      if (lane == 0) {
        slot_tile[s] = t;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&full[s], (unsigned)D.block_bytes);
        bulk_g2s(blk, A.blocks + D.block_off, (unsigned)D.block_bytes, &full[s]);
      }
      const int T = D.nrows, S = D.nspill;
      const double* xo = x + D.row0;
      for (int i = lane; i < T; i += 32) cp_async8(xsl + i, xo + i);
      const int32_t* tg = A.targets + D.spill_off;
      for (int i = lane; i < S; i += 32) cp_async8(xsl + T + i, x + tg[i]);
      cp_async_arrive_noinc(&full[s]);
    }
    return;
  }
  // -------------------------------------------------- consumer warps
  constexpr int RPW = 32 / V;
  const int sub = lane % V;
  for (int k = 0;; ++k) {
    const int s = k % kStages;
    mbar_wait(&full[s], (unsigned)((k / kStages) & 1));
    const long long t = slot_tile[s];
    if (t >= A.ntiles) break;
    const TileDesc D = A.tiles[t];
    const int T = D.nrows, S = D.nspill, W = T + S;
    const unsigned char* blk = sm + s * slot_bytes;
    const double* xs = reinterpret_cast<const double*>(blk + A.block_cap);
    const uint16_t* start = reinterpret_cast<const uint16_t*>(blk);
    const uint16_t* lcol = reinterpret_cast<const uint16_t*>(blk + D.o_lcol);
    const uint16_t* tidx = reinterpret_cast<const uint16_t*>(blk + D.o_tidx);
    const uint16_t* tptr = reinterpret_cast<const uint16_t*>(blk + D.o_tptr);
    const uint16_t* inptr = reinterpret_cast<const uint16_t*>(blk + D.o_inptr);
    const int32_t* slot = reinterpret_cast<const int32_t*>(blk + D.o_slot);
    const double* val = reinterpret_cast<const double*>(blk + D.o_val);
    // pass 1: rows, V lanes per row
    for (int base = wid * RPW; base < T; base += kConsumerWarps * RPW) {
      const int i = base + lane / V;
      double sum = 0.0;
      if (i < T) {
        const int eb = start[i], ee = start[i + 1];
        const double xi = xs[i];
#pragma unroll 4
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
    consumer_sync();
    // pass 2: targets (one thread per local target, entries in stored order)
    for (int l = tid; l < W; l += kConsumers) {
      double acc = l < T ? ys[l] : 0.0;
      const int jb = tptr[l], je = tptr[l + 1];
#pragma unroll 4
      for (int j = jb; j < je; ++j) acc += Pp[tidx[j]];
      ys[l] = acc;
    }
    consumer_sync();
    // stage contributions to later tiles' rows, then publish (before waiting:
    // publication never depends on another tile -> dependency depth 1)
    for (int i = tid; i < S; i += kConsumers) __stcg(A.spill_buf + slot[i], ys[T + i]);
    if (S > 0) __threadfence();
    consumer_sync();
    if (tid == 0) st_release_u32(A.ready + t, A.epoch);
    // wait for the (earlier) tiles that wrote into this tile's rows
    for (int q = tid; q < D.nwr; q += kConsumers) {
      const unsigned int* f = A.ready + A.writers[D.wr_off + q];
      while (ld_acquire_u32(f) != A.epoch) __nanosleep(20);
      __threadfence();
    }
    consumer_sync();
    const double* inb = A.spill_buf + D.in_base;
    for (int i = tid; i < T; i += kConsumers) {
      double acc = ys[i];
      const int jb = inptr[i], je = inptr[i + 1];
      for (int j = jb; j < je; ++j) acc += __ldcg(inb + j);
      y[D.row0 + i] = acc;
    }
    consumer_sync();  // slot s (block + x window) and ys/P are free again
    if (tid == 0) mbar_arrive(&empty[s]);
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
  return kStages * (T.block_cap + 8 * T.window_cap) + 8 * T.window_cap + 8 * T.nnz_cap;
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
