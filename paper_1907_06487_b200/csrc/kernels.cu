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
#include <algorithm>
#include <cstdint>
#include <cstdlib>

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
__device__ __forceinline__ unsigned int ld_relaxed_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// fp64 reduction without a return value (RED.E.ADD.F64).  Spelled out in PTX:
// with an acquire load elsewhere in the kernel, nvcc compiled atomicAdd's
// unused result as ATOMG (a returning atomic), which made K4 ~15% slower.
__device__ __forceinline__ void red_add_f64(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

__device__ __forceinline__ void red_add_u32(unsigned int* p, unsigned int v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ double group_sum(double s) {
#pragma unroll
  for (int o = V / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, V);
  return s;
}

// ---------------------------------------------------------------- zero / gather
__global__ void k_zero(double* __restrict__ y, int64_t n) {
  // the tiled kernel that follows may start streaming its (constant) tile
  // blocks now; it waits (griddepcontrol.wait) before touching x or y
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // 16-B stores for the aligned body, scalar head/tail
  const int64_t head = ((16 - ((uintptr_t)y & 15)) & 15) / 8;  // 0 or 1 element
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (tid == 0 && head && n > 0) y[0] = 0.0;
  const int64_t body = n > head ? (n - head) / 2 : 0;
  double2* y2 = reinterpret_cast<double2*>(y + head);
  for (int64_t i = tid; i < body; i += stride) y2[i] = make_double2(0.0, 0.0);
  if (tid == 0 && head + 2 * body < n) y[n - 1] = 0.0;
}

__global__ void k_gather(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                         int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[idx[i]];
}
__global__ void k_add(double* __restrict__ y, const double* __restrict__ v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) y[i] += v[i];
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
          red_add_f64(y + c, a * xr);  // b[col[idx]] += A[idx] * x[row]  (RED.F64)
        }
      }
    }
    sum = group_sum<V>(sum);
    if (valid && sub == 0) red_add_f64(y + row, sum);  // b[row] += tmp
  }
}

// Sum of v over the lanes of `peers` (a __match_any_sync set containing this
// lane), delivered to the set's lowest lane.  Pairwise tree over the set's
// ranks: in round k every lane adds the value of the next higher lane still in
// the set, then the lanes of odd rank drop out (their values have been taken).
// Every lane runs every round (the shuffles need the whole warp); all sets of
// the warp reduce at once in ceil(log2(largest set)) rounds.
__device__ __forceinline__ double peer_sum(unsigned peers, double v, int lane) {
  unsigned above = peers & ~((2u << lane) - 1u);          // set members above this lane
  unsigned rank = __popc(peers & ((1u << lane) - 1u));    // set members below it
  while (__any_sync(0xffffffffu, above != 0)) {
    const int nxt = __ffs(above);                          // 1-based, 0: none
    const double t = __shfl_sync(0xffffffffu, v, nxt > 0 ? nxt - 1 : lane);
    if (nxt > 0) v += t;
    above &= ~__ballot_sync(0xffffffffu, rank & 1u);     // odd ranks are consumed
    rank >>= 1;
  }
  return v;
}

// K1 with warp-level segmented pre-reduction (north_star: "native fp64
// atomicAdd for the transpose updates, with warp-level segmented
// pre-reduction").  A warp walks the nonzeros of a chunk of rows flat, 32
// consecutive stored entries per step (coalesced col / val loads), lane i on
// entry p = base + i of row r:
//   b[r] += a x[c]: equal r are contiguous lanes,
//   b[c] += a x[r], c != r: neighbouring rows share columns;
// __match_any_sync groups the lanes of equal destination, peer_sum adds them
// and the lowest lane of each group issues one RED.F64.
constexpr int kK1Rows = 128;  // rows per warp chunk
__global__ void __launch_bounds__(256) k_atomic_pr(CsrArgs A, const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r0 = warp * kK1Rows; r0 < A.n; r0 += nwarps * kK1Rows) {  // warp-uniform
    const int r1 = (int)min((int64_t)A.n, r0 + kK1Rows);
    const int e0 = __ldg(A.row_ptr + r0), e1 = __ldg(A.row_ptr + r1);
    int r = (int)r0;
    for (int base = e0; base < e1; base += 32) {
      const int p = base + lane;
      const bool valid = p < e1;
      double vr = 0.0, vc = 0.0;
      int c = -1;
      if (valid) {
        while (__ldg(A.row_ptr + r + 1) <= p) ++r;  // this lane's row (monotone)
        c = ld_stream_i32(A.col + p);
        const double a = ld_stream_f64(A.val + p);
        const double xr = __ldg(x + r);
        if (c == r) {
          vr = a * xr;  // diagonal contributes once (reading R1)
        } else {
          vr = a * __ldg(x + c);
          vc = a * xr;
        }
      }
      // row part: key r (invalid lanes get a key no valid lane has)
      const int kr = valid ? r : -1 - lane;
      const unsigned mr = __match_any_sync(0xffffffffu, kr);
      vr = peer_sum(mr, vr, lane);
      if (valid && (mr & ((1u << lane) - 1u)) == 0) red_add_f64(y + r, vr);
      // transposed part: key c (diagonal and invalid lanes are singletons, no RED)
      const bool hc = valid && c != r;
      const int kc = hc ? c : -1 - lane;
      const unsigned mc = __match_any_sync(0xffffffffu, kc);
      vc = peer_sum(mc, vc, lane);
      if (hc && (mc & ((1u << lane) - 1u)) == 0) red_add_f64(y + c, vc);
    }
  }
}

// ---------------------------------------------------------------- K6 SpMV (yardstick)
// Alg. 1 on the full CRS: V lanes per row stream the row's
// (col, val) pairs with non-allocating loads, gather x through L1/L2, reduce
// by shuffles and store y[row] once (no atomics, deterministic).
template <int V>
__global__ void __launch_bounds__(256) k_spmv(CsrArgs A, const double* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / V;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * RPW; base < A.n; base += nwarps * RPW) {  // warp-uniform
    const int64_t row = base + lane / V;
    double sum = 0.0;
    if (row < A.n) {
      const int b = A.row_ptr[row], e = A.row_ptr[row + 1];
#pragma unroll 4
      for (int i = b + sub; i < e; i += V) sum += ld_stream_f64(A.val + i) * __ldg(x + ld_stream_i32(A.col + i));
    }
    sum = group_sum<V>(sum);
    if (row < A.n && sub == 0) y[row] = sum;
  }
}

// ---------------------------------------------------------------- NEXT-4 sweeps
// One phase of a Gauss-Seidel (KIND 1) or Kaczmarz (KIND 2) sweep: V lanes per
// row of the full matrix; the rows of a phase are distance-1 (GS) /
// distance-2 (KACZ) independent, so their reads and writes of x commute.
template <int KIND, int V>
__global__ void __launch_bounds__(256) k_sweep(CsrArgs A, const int32_t* __restrict__ rows, int32_t nrows,
                                               const double* __restrict__ b, double* __restrict__ x) {
  constexpr int RPW = 32 / V;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = warp * RPW; base < nrows; base += nwarps * RPW) {  // warp-uniform
    const int64_t q = base + lane / V;
    const bool valid = q < nrows;
    const int row = valid ? rows[q] : 0;
    const int bi = valid ? A.row_ptr[row] : 0, ei = valid ? A.row_ptr[row + 1] : 0;
    double s = 0.0, t = 0.0;  // GS: off-diagonal sum, diagonal; KACZ: <A_r, x>, ||A_r||^2
    for (int i = bi + sub; i < ei; i += V) {
      const int c = A.col[i];
      const double a = A.val[i];
      if (KIND == 1) {
        if (c == row) t += a;
        else s += a * __ldcg(x + c);
      } else {
        s += a * __ldcg(x + c);
        t += a * a;
      }
    }
    s = group_sum<V>(s);
    t = group_sum<V>(t);
    if (KIND == 1) {
      if (valid && sub == 0) __stcg(x + row, (b[row] - s) / t);  // x_r := (b_r - sum_{c!=r} a_rc x_c) / a_rr
    } else if (valid && t > 0.0) {
      const double scale = (b[row] - s) / t;  // (b_r - <A_r, x>) / ||A_r||^2
      for (int i = bi + sub; i < ei; i += V) {
        const int c = A.col[i];
        __stcg(x + c, __ldcg(x + c) + scale * A.val[i]);  // x_c += scale a_rc (distance-2: no other row of the phase)
      }
    }
  }
}

// ---------------------------------------------------------------- K2 colored
// One tile by one CTA: the tile's intra-tile colours one after the other
// (__syncthreads between), V lanes per row, plain read-modify-write of y
// through L2 (write-disjoint inside a colour and across the tiles that may
// run at the same time).
template <int V>
__device__ __forceinline__ void colored_tile(const CsrArgs& A, const ColoredArgs& C, int t,
                                             const double* __restrict__ x, double* __restrict__ y) {
  constexpr int RPW = 32 / V;
  const int lane = threadIdx.x & 31;
  const int sub = lane % V;
  const int wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
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

template <int V>
__global__ void __launch_bounds__(256) k_colored(CsrArgs A, ColoredArgs C, const double* __restrict__ x,
                                                 double* __restrict__ y) {
  colored_tile<V>(A, C, C.phase_tiles[blockIdx.x], x, y);
}

// ---------------------------------------------------------------- K7 tree
// The recursive RACE tree in one persistent launch (NEXT-2).  A CTA claims
// the next leaf in execution order (red subtrees before blue, depth first),
// waits until, at every ancestor where the leaf lies in a blue child, all the
// leaves under that ancestor's red children are done (tree-scoped sync of
// PAPER.md:1418-1421), runs the leaf's tiles like K2, then counts itself at
// every ancestor where it lies in a red child.  Every claimed leaf runs on a
// resident CTA and waits only for leaves claimed before it: no deadlock.
template <int V>
__global__ void __launch_bounds__(256) k_tree(CsrArgs A, ColoredArgs C, TreeArgs T, const double* __restrict__ x,
                                              double* __restrict__ y) {
  __shared__ int s_leaf;
  for (;;) {
    if (threadIdx.x == 0) s_leaf = atomicAdd(T.counters + T.nnodes, 1);  // claim the next leaf
    __syncthreads();
    const int i = s_leaf;
    if (i >= T.nleaves) break;
    if (threadIdx.x == 0) {
      for (int q = T.wait_ptr[i]; q < T.wait_ptr[i + 1]; ++q) {
        const int a = T.wait_node[q];
        const unsigned need = (unsigned)T.red_total[a];
        while (ld_acquire_u32(reinterpret_cast<const unsigned*>(T.counters + a)) < need) __nanosleep(64);
      }
      __threadfence();
    }
    __syncthreads();
    for (int t = T.leaf_t0[i]; t < T.leaf_t1[i]; ++t) colored_tile<V>(A, C, t, x, y);
    // colored_tile ends with __syncthreads: every store of the leaf is issued
    if (threadIdx.x == 0) {
      __threadfence();
      for (int q = T.sig_ptr[i]; q < T.sig_ptr[i + 1]; ++q) atomicAdd(T.counters + T.sig_node[q], 1);
    }
  }
}

// ---------------------------------------------------------------- K3/K4 tiled streaming kernel
// Persistent, static tile assignment (tile = blockIdx.x + k * gridDim.x, tiles
// in BFS order), warp roles on a kStages-deep smem ring:
//   loader warp:  one cp.async.bulk (TMA) per tile block + descriptor ->
//                 blk_full[s] (after the stage was released: empty[s]);
//   gather warp:  when a block has landed, cp.async-gathers x of the tile
//                 window (own rows + spill targets) -> x_full[s];
//   kGroups consumer groups x kGroupWarps warps, round-robin over the tiles
//   of the CTA (several tiles in flight per SM); one pass, thread per target l:
//     y_l = sum_{e in row l} a_e x[c_e]                      (tmp)
//         + sum_{e: c_e = l, e off-diagonal} a_e x[r_e]      (b[col] += ...)
//     fixed order -> deterministic; the result is flushed:
//       K3 (deterministic): own rows -> y (store), spill -> spill_buf[slot]
//                           (k_fixup then adds the staged values in slot order);
//       K4 (atomic):        own rows and spill -> RED.F64 into pre-zeroed y.
// No consumer ever waits on global memory or on another CTA.
constexpr int kMaxStages = 8;
// consumer groups x warps per group + gather warps (<= 31 warps + the loader).
// Measured against the default 4 x 7 + 3 (fem / spin / st27 ms): 4 x 6 + 6:
// 0.198 / 0.194 / 0.0946 (within noise of 0.199 / 0.197 / 0.0935); 3 x 9 + 3:
// 0.203 / 0.203 / 0.0966; 2 x 14 + 3: 0.221 / 0.224 / 0.105
#ifndef K4_GROUP_WARPS
#define K4_GROUP_WARPS 7
#endif
#ifndef K4_GROUPS
#define K4_GROUPS 4
#endif
#ifndef K4_GATHER_WARPS
#define K4_GATHER_WARPS 3
#endif
constexpr int kGroupWarps = K4_GROUP_WARPS;
constexpr int kGroupThreads = kGroupWarps * 32;
constexpr int kGroups = K4_GROUPS;
constexpr int kGatherWarps = K4_GATHER_WARPS;
constexpr int kTiledThreads = kGroups * kGroupThreads + 32 * (1 + kGatherWarps);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_relaxed(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
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
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// bulk copy of data that is read exactly once per multiply (the tile blocks):
// evict-first keeps the L2 for the x / y working set
__device__ __forceinline__ void bulk_g2s_stream(void* dst, const void* src, unsigned bytes, uint64_t* bar,
                                                uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// L2 prefetches (no destination, no completion): issued one to several tiles
// ahead so that the copy into the ring, which can start only when a stage is
// free, finds its data in L2 instead of paying a DRAM round trip
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// trace layout (CTA 0 only): 8 slots per local tile k
//   0 loader issue, 1 gather saw block, 2 gather issued, 3 consumer got x,
//   4 pass A done, 5 pass B done, 6 group id
#ifdef K4_TRACE
#define TRACE(k, slot)                                                               \
  do {                                                                               \
    if (A.trace != nullptr && blockIdx.x == 0) A.trace[(size_t)(k) * 8 + (slot)] = gtimer(); \
  } while (0)
#else
#define TRACE(k, slot) \
  do {                 \
  } while (0)
#endif

__device__ __forceinline__ void group_sync(int g) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + g), "n"(kGroupThreads) : "memory");
}

// K4 zeroes y itself, in a prologue run by every warp except the loader (which
// starts filling the ring at once): the CTA stores zeros over its slice of the
// local y range and takes a ticket from a monotonic launch counter (zero_ctr,
// 64 bit: every launch adds exactly gridDim.x, so the tickets of one launch are
// [m G, (m+1) G) and nothing needs resetting).  Before its first flush, every
// consumer warp waits until the counter has reached (m+1) G: the REDs of any
// tile may hit any CTA's slice.  The tile computations before that overlap the
// other CTAs' zeroing.  Launches of one plan are stream-ordered (one run at a
// time).
constexpr int kZeroThreads = kTiledThreads - 32;
__device__ __forceinline__ void k4_zero_y(const K8Args* z, double* y, int G, int ztid,
                                          unsigned long long* s_target) {
  const int64_t zb = z->zero_begin, zn = z->zero_end - zb;
  const int64_t per = ((zn + G - 1) / G + 1) & ~int64_t(1);
  int64_t a = zb + (int64_t)blockIdx.x * per;
  const int64_t e = min(zb + zn, a + per);
  if (!(z->zero_dbg & 1) && a < e) {
    if (((uintptr_t)(y + a) & 15) && ztid == 0) y[a] = 0.0;  // 16-B stores for the aligned body
    a += ((uintptr_t)(y + a) & 15) ? 1 : 0;
    const int64_t nb = (e - a) / 2;
    double2* y2 = reinterpret_cast<double2*>(y + a);
    for (int64_t i = ztid; i < nb; i += kZeroThreads) y2[i] = make_double2(0.0, 0.0);
    if (ztid == 0 && a + 2 * nb < e) y[e - 1] = 0.0;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kZeroThreads) : "memory");
  if (ztid == 0) {
    __threadfence();
    *s_target = (z->zero_dbg & 2) ? 0ull : (atomicAdd(z->zero_ctr, 1ull) / (unsigned)G + 1) * (unsigned)G;
  }
  asm volatile("bar.sync 1, %0;" ::"n"(kZeroThreads) : "memory");
}
// one poller per warp, once per launch
__device__ __forceinline__ void k4_zero_wait(const K8Args* z, unsigned long long t) {
  if ((threadIdx.x & 31) == 0)
    while (ld_acquire_u64(z->zero_ctr) < t) __nanosleep(128);
  __syncwarp();
}

// MODE 0: K3 (own rows stored, spill staged for k_fixup), 1: K4 (fp64 RED
// into zeroed y), 2: K8 (phase-major order, DAG-ordered store / add: no
// atomics, no zeroing, deterministic)
// diagnostics skip bits (env SYMM_DEBUG_SKIP) only in K4_DEBUG_SKIP builds:
// the bit tests cost the consumer loop measurable time otherwise
#ifdef K4_DEBUG_SKIP
#define K4_DBG A.debug_skip
#else
#define K4_DBG 0
#endif
// K8 signalling of the DAG counters: 1 = a dedicated signaller warp (the last
// gather warp); 2 = lanes 1..kGroups of the loader warp (idle otherwise), so
// all kGatherWarps gather warps keep gathering -- measured slower (st27 0.158
// vs 0.146 ms, fem 0.286 vs 0.271, spin 0.452 vs 0.409: the divergent lanes
// delay the loader lane's bulk-copy issue); 0 = the last-arriving consumer
// warp of a group
#ifndef K8_ACQ
#define K8_ACQ 0
#endif
#ifndef K8_SIGNALLER
#define K8_SIGNALLER 1
#endif
// 1: the gather warps read a short-run tile's spill targets from the block's
// global copy before the stage wait (0: from the staged block, after it
// lands); fem_knn_4M K4 0.206 -> 0.199 ms (profiles/r2/i/ab_tgt_global.txt)
#ifndef K4_TGT_GLOBAL
#define K4_TGT_GLOBAL 1
#endif
// (K3 / K4 only: K8, with two gather warps, measured slower with it on
// fem_knn_4M, 0.288 vs 0.267 ms)
#define K4_TGT_G (K4_TGT_GLOBAL && !ORDERED)
// L2 prefetch (measured slower, off): bit 0 = the loader prefetches the block
// of the tile 3-4 issues ahead (fem 0.201 vs 0.199 ms, spin 0.207 vs 0.197,
// st27 0.0975 vs 0.0935); bit 1 = the gather warps prefetch their next tile's
// own x rows and spill runs / targets before the stage wait (fem 0.210, spin
// 0.263, st27 0.105) -- profiles/r2/i/ab_prefetch_shapes.txt
#ifndef K4_PF
#define K4_PF 0
#endif
template <int MODE, int NS>
__global__ void __launch_bounds__(kTiledThreads, 1) k_tiled(TiledArgs A, const double* __restrict__ x,
                                                            double* __restrict__ y) {
  static_assert(kK4Unroll == 2 && kK4SortedUnroll == 2, "the loop pragmas below must match kK4Unroll / kK4SortedUnroll");
  constexpr bool ATOMIC = MODE == 1;
  constexpr bool ORDERED = MODE == 2;
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t blk_full[NS], x_full[NS], empty[NS];
  __shared__ int loader_k;  // tiles the loader has taken a free stage for (gather warps follow it)
  // K8: warps of a group done flushing a tile (mod 7), by group tile index mod
  // 4 (the warps of a group are at most two group tiles apart: the stage ring)
  __shared__ unsigned k8_arrive[kGroups][4];
  // K8 with a signaller warp: tiles flushed by each consumer warp (release,
  // CTA scope); the signaller turns them into the GPU-wide done[] counters
  __shared__ unsigned k8_prog[kGroups * kGroupWarps];
  // the K3 / K8 table pointers, copied once: read through A.k8 every access
  // was a dependent global load (an L2 round trip after each CCTL.IVALL)
  __shared__ K8Args k8s;
  const size_t slot_bytes = (size_t)A.block_cap + 8 * (size_t)A.window_cap;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&blk_full[s], 1);
      mbar_init(&x_full[s], 32);
      mbar_init(&empty[s], kGroupWarps);  // every consumer warp of the group arrives
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    loader_k = 0;
    k8s = *A.k8;
    for (int q = 0; q < kGroups * 4; ++q) k8_arrive[q / 4][q % 4] = 0;
    for (int q = 0; q < kGroups * kGroupWarps; ++q) k8_prog[q] = 0;
  }
  __syncthreads();
  // ------------------------------------------------ K8 signaller
  // Lane q < kGroups of the signalling lanes `mask` follows consumer group q.
  // A group tile j is flushed once all 7 warps of the group have published
  // progress > j (st.release.cta after their REDs / stores).  Whenever tiles
  // became complete, ONE fence.acq_rel.gpu (cumulative: it orders the REDs the
  // acquire loads observed) precedes their done[] signals.  The consumer warps
  // never wait for their REDs to reach L2 (that wait, one fence per tile on the
  // consumers' path, was 26% of K8's time on st27).
  auto k8_signal = [&](const int q, const unsigned mask) {
    const int nk = (A.ntiles - (int)blockIdx.x + G - 1) / G;  // tiles of this CTA
    const int nq = (q >= 0 && q < kGroups && nk > q) ? (nk - q + kGroups - 1) / kGroups : 0;
    int sig = 0;  // group tiles of group q already signalled
    while (__any_sync(mask, sig < nq)) {
      int m = nq;
      if (sig < nq) {
#pragma unroll
        for (int w = 0; w < kGroupWarps; ++w) {
          unsigned v;
          asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];"
                       : "=r"(v) : "r"(smem_u32(&k8_prog[q * kGroupWarps + w])) : "memory");
          m = min(m, (int)v);
        }
      }
      const bool any = __any_sync(mask, m > sig);
      if (!any) {
        __nanosleep(64);
        continue;
      }
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      for (int j = sig; j < m; ++j) {
        const int t = blockIdx.x + (q + j * kGroups) * G;
        red_add_u32(k8s.done + __ldg(k8s.order + t), (unsigned)kGroupWarps);
      }
      sig = max(sig, m);
    }
  };
  __shared__ unsigned long long zero_target;
  const bool self_zero = ATOMIC && k8s.zero_ctr != nullptr;
  if (self_zero && wid != kGroups * kGroupWarps) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel of the stream is done
    k4_zero_y(A.k8, y, G, wid < kGroups * kGroupWarps ? tid : tid - 32, &zero_target);
  }
  if (wid == kGroups * kGroupWarps) {
    // ------------------------------------------------ loader warp (TMA bulk)
    // lane 0 only; (offset, bytes) of the next 4 tiles of this CTA live in a
    // register ring (loop unrolled by 4) so each issue finds its operands ready.
    if constexpr (ORDERED && K8_SIGNALLER == 2) {
      // lanes 1..kGroups: the K8 signaller (independent thread scheduling
      // interleaves them with lane 0's issue loop; both wait by suspending)
      if (lane >= 1 && lane <= kGroups) {
        k8_signal(lane - 1, ((1u << kGroups) - 1u) << 1);
        return;
      }
    }
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      int4 d0 = make_int4(0, 0, 0, 0), d1 = d0, d2 = d0, d3 = d0;  // (off lo, off hi, bytes, row0)
      int T0 = 0, T1 = 0, T2 = 0, T3 = 0;
      auto ld = [&](int kk, int4& d, int& T) {
        const int tt = blockIdx.x + kk * G;
        if (tt < A.ntiles) {
          const TileDesc& D = A.tiles[ORDERED ? __ldg(k8s.order + tt) : tt];
          const int64_t o = D.block_off;
          d = make_int4((int)(o & 0xffffffff), (int)(o >> 32), D.block_bytes, D.row0);
          T = D.nrows;
        } else {
          d.z = 0;
        }
      };
      auto pf = [&](const int4& d) {
        if ((K4_PF & 1) && d.z > 0)
          bulk_prefetch_l2(A.blocks + ((int64_t)(uint32_t)d.x | ((int64_t)d.y << 32)), (unsigned)d.z);
      };
      auto issue = [&](int k, int4 d, int T) {
        const int s = k % NS, use = k / NS;
        const int64_t off = (int64_t)(uint32_t)d.x | ((int64_t)d.y << 32);
        const int row0 = d.w;
        (void)row0;
        (void)T;
        TRACE(k, 6);
        if (use > 0) mbar_wait(&empty[s], (unsigned)((use - 1) & 1));
        TRACE(k, 7);
        // the stage of tile k is free: gather warps may fill its x window
        asm volatile("st.volatile.shared.s32 [%0], %1;" ::"r"(smem_u32(&loader_k)), "r"(k + 1) : "memory");
        // the loader reads only the plan's tile blocks (never x or y), so it
        // may run while the preceding kernel (k_zero) still runs (PDL)
        mbar_arrive_expect_tx(&blk_full[s], (unsigned)d.z);
        bulk_g2s_stream(sm + s * slot_bytes, A.blocks + off, (unsigned)d.z, &blk_full[s], pol);
        TRACE(k, 0);
      };
      ld(0, d0, T0);
      ld(1, d1, T1);
      ld(2, d2, T2);
      ld(3, d3, T3);
      const int nk = (A.ntiles - (int)blockIdx.x + G - 1) / G;  // tiles of this CTA
      for (int kb = 0; kb < nk; kb += 4) {
        // a descriptor loaded in one step is used for the L2 prefetch in the
        // next one, so the loader lane never waits for it
        issue(kb, d0, T0);
        if (kb > 0) pf(d3);
        ld(kb + 4, d0, T0);
        if (kb + 1 >= nk) break;
        issue(kb + 1, d1, T1);
        pf(d0);
        ld(kb + 5, d1, T1);
        if (kb + 2 >= nk) break;
        issue(kb + 2, d2, T2);
        pf(d1);
        ld(kb + 6, d2, T2);
        if (kb + 3 >= nk) break;
        issue(kb + 3, d3, T3);
        pf(d2);
        ld(kb + 7, d3, T3);
      }
    }
    return;
  }
  if (wid >= kGroups * kGroupWarps + 1) {
    // ------------------------------------------------ gather warps (x window)
    // kGatherWarps warps take the tiles of this CTA in turn.  As soon as the
    // stage is free (no need to wait for the tile's block) a warp fills the
    // spill part of the x window: the spill targets come as runs of
    // consecutive rows laid out with matching 16-B parity, so each run is one
    // bulk copy (TMA) plus at most two 8-B cp.async edge elements; the lane also
    // copies the unaligned own-x edge elements (the loader bulk-copies the rest).
    const int gw = wid - (kGroups * kGroupWarps + 1);
    if constexpr (ORDERED) {
      if (K8_SIGNALLER == 1 && gw == kGatherWarps - 1) {
        k8_signal(lane, 0xffffffffu);
        return;
      }
    }
    constexpr int NGW = (ORDERED && K8_SIGNALLER == 1) ? kGatherWarps - 1 : kGatherWarps;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // x is ready (PDL prerequisite done)
    int k = gw;
    for (int t = blockIdx.x + gw * G; t < A.ntiles; t += NGW * G, k += NGW) {
      const int s = k % NS;
      const TileDesc* Dg = A.tiles + (ORDERED ? __ldg(k8s.order + t) : t);
      const int row0 = __ldg(&Dg->row0), T = __ldg(&Dg->nrows);
      const int nr = __ldg(&Dg->nruns), ro = __ldg(&Dg->run_off);
      const int gruns = __ldg(&Dg->gather_runs) && !(K4_DBG & 8);

      // the first batch of run records (8 per lane) is loaded before the stage
      // wait, so its latency overlaps it
      int4 R[8];
      // short-run tiles (kNN): the first 1024 spill targets are read from the
      // block's global copy into the same registers, also before the stage
      // wait, so the x gather no longer waits for the tile block to land (the
      // chain stage free -> block -> targets -> x was two DRAM round trips)
      const int Sg = (gruns || !K4_TGT_G) ? 0 : __ldg(&Dg->nspill);
      const int32_t* tgt_g =
          K4_TGT_G ? reinterpret_cast<const int32_t*>(A.blocks + __ldg(&Dg->block_off) + __ldg(&Dg->o_tgt)) : nullptr;
      if (K4_TGT_G && !gruns) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i0 = u * 128 + lane;
          R[u].x = i0 < Sg ? __ldg(tgt_g + i0) : -1;
          R[u].y = i0 + 32 < Sg ? __ldg(tgt_g + i0 + 32) : -1;
          R[u].z = i0 + 64 < Sg ? __ldg(tgt_g + i0 + 64) : -1;
          R[u].w = i0 + 96 < Sg ? __ldg(tgt_g + i0 + 96) : -1;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int r = u * 32 + lane;
          R[u] = (gruns && r < nr) ? __ldg(reinterpret_cast<const int4*>(A.runs) + ro + r) : make_int4(0, 0, 0, 0);
        }
      }
      if (K4_PF & 2) {
        // x of this tile into L2 while the stage is still in use
        if (lane == 2 && T > 0) {
          const double* xa = x + row0 + (int)(((uintptr_t)(x + row0) >> 3) & 1);
          const int nf = (T - (int)(xa - (x + row0))) & ~1;
          if (nf > 0) bulk_prefetch_l2(xa, (unsigned)nf * 8u);
        }
        if (gruns) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int len = R[u].z;
            if (len <= 0) continue;
            const double* src = x + R[u].x;
            const int i0 = (int)(((uintptr_t)src >> 3) & 1);
            const int nb = len > i0 ? ((len - i0) & ~1) : 0;
            if (nb > 0) bulk_prefetch_l2(src + i0, (unsigned)nb * 8u);
          }
        } else if (K4_TGT_G) {
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (R[u].x >= 0) prefetch_l2(x + R[u].x);
            if (R[u].y >= 0) prefetch_l2(x + R[u].y);
            if (R[u].z >= 0) prefetch_l2(x + R[u].z);
            if (R[u].w >= 0) prefetch_l2(x + R[u].w);
          }
        }
      }
      // stage free: tile k - NS has been consumed.  With NS % kGatherWarps ==
      // 0 an mbarrier wait (hardware suspend) replaces the poll of loader_k,
      // which cost 9% of the kernel's shared-memory wavefronts on fem_knn_4M
      // (ncu source page).  No parity alias: tile k - NS is this warp's own,
      // and waiting for its stage it saw tile k - 2 NS consumed; tile k itself
      // cannot be consumed yet.  Other ring depths poll loader_k (the loader
      // waits for the stages in order, so its parity waits cannot alias).
      if constexpr (NS % NGW == 0) {
        if (k >= NS) mbar_wait(&empty[s], (unsigned)(((k / NS) - 1) & 1));
      } else {
        while (true) {
          int lk;
          asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(lk) : "r"(smem_u32(&loader_k)) : "memory");
          if (lk > k) break;
          __nanosleep(64);
        }
      }
      if (lane == 0) TRACE(k, 1);
      const int p = (int)(((uintptr_t)(x + row0) >> 3) & 1);
      const int nfull = T > p ? ((T - p) & ~1) : 0;
      double* xs = reinterpret_cast<double*>(sm + s * slot_bytes + A.block_cap) + p;
#ifdef K4_CHECK
      if (T + p > A.window_cap || row0 + T > A.check_n) { printf("K4_CHECK own t=%d T=%d\n", t, T); __trap(); }
#endif
      // own rows: the 16-B aligned part of x[row0 .. row0+T) by one bulk copy,
      // the (at most two) unaligned edge elements by cp.async
      if (lane == 2 && nfull > 0) {
        mbar_expect_tx(&x_full[s], (unsigned)nfull * 8u);
        bulk_g2s(xs + p, x + row0 + p, (unsigned)nfull * 8u, &x_full[s]);
      }
      if (lane == 0 && p == 1) cp_async8(xs, x + row0);
      if (lane == 1 && p + nfull < T) cp_async8(xs + p + nfull, x + row0 + p + nfull);
      if (K4_DBG & 8) {
        // diagnostics: no spill gather
      } else if (gruns) {
        // long runs: one bulk copy per run (+ <= 2 8-B edge elements)
        for (int rb = 0; rb < nr; rb += 32 * 8) {
          if (rb > 0) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int r = rb + u * 32 + lane;
              R[u] = r < nr ? __ldg(reinterpret_cast<const int4*>(A.runs) + ro + r) : make_int4(0, 0, 0, 0);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int len = R[u].z;  // (row, wid, len, 0)
            if (len <= 0) continue;
#ifdef K4_CHECK
            if (R[u].y + len + p > A.window_cap || R[u].x < 0 || R[u].x + len > A.check_n || R[u].y < T) {
              printf("K4_CHECK run t=%d r=%d row=%d wid=%d len=%d T=%d wcap=%d n=%d\n", t, u, R[u].x, R[u].y, len, T, A.window_cap, A.check_n);
              __trap();
            }
#endif
            double* dst = xs + R[u].y;
            const double* src = x + R[u].x;
            const int i0 = (int)(((uintptr_t)src >> 3) & 1);  // dst has the same 16-B phase
            const int nb = len > i0 ? ((len - i0) & ~1) : 0;
            if (nb > 0) {
              mbar_expect_tx(&x_full[s], (unsigned)nb * 8u);
              bulk_g2s(dst + i0, src + i0, (unsigned)nb * 8u, &x_full[s]);
            }
            if (i0) cp_async8(dst, src);
            if (i0 + nb < len) cp_async8(dst + len - 1, src + len - 1);
          }
        }
      } else if (K4_TGT_G) {
        // short runs: slot by slot, targets already in registers
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i0 = u * 128 + lane;
          if (R[u].x >= 0) cp_async8(xs + T + i0, x + R[u].x);
          if (R[u].y >= 0) cp_async8(xs + T + i0 + 32, x + R[u].y);
          if (R[u].z >= 0) cp_async8(xs + T + i0 + 64, x + R[u].z);
          if (R[u].w >= 0) cp_async8(xs + T + i0 + 96, x + R[u].w);
        }
        for (int idx = 1024 + lane; idx < Sg; idx += 32) {
          const int g = __ldg(tgt_g + idx);
          if (g >= 0) cp_async8(xs + T + idx, x + g);
        }
      } else {
        // short runs: slot by slot from the block's target list, spread over the lanes
        mbar_wait(&blk_full[s], (unsigned)((k / NS) & 1));
        const unsigned char* blk = sm + s * slot_bytes;
        const TileDesc& D = *reinterpret_cast<const TileDesc*>(blk);
        const int32_t* tgt = reinterpret_cast<const int32_t*>(blk + D.o_tgt);
        const int S = D.nspill;
#pragma unroll 4
        for (int idx = lane; idx < S; idx += 32) {
          const int g = tgt[idx];
#ifdef K4_CHECK
          if (g >= A.check_n || T + idx + p >= A.window_cap) { printf("K4_CHECK loose t=%d g=%d idx=%d\n", t, g, idx); __trap(); }
#endif
          if (g >= 0) cp_async8(xs + T + idx, x + g);
        }
      }
      cp_async_arrive_noinc(&x_full[s]);
      if (lane == 0) TRACE(k, 2);
    }
    return;
  }
  // -------------------------------------------------- consumer groups
  asm volatile("griddepcontrol.wait;" ::: "memory");  // the previous kernel of the stream is done
  const int g = wid / kGroupWarps;
  const int gt = tid - g * kGroupThreads;
  // K4: zero this CTA's slice of y while the loader fills the ring; the first
  // flush of every warp waits until all CTAs have zeroed theirs (zero_ctr)
  bool zero_pending = self_zero;
  int k = g;
  // K8: (tile id, predecessor range) of this warp's current and next tile and
  // the current tile's predecessor counter index per lane, software-pipelined
  // so that the acquire loads of the done counters, issued before the stage
  // waits, are the only global round trip at the top of a tile
  int4 m_cur = make_int4(0, 0, 0, 0), m_nx = m_cur;
  int pr_cur = 0;
  if constexpr (ORDERED) {
    const int t0 = blockIdx.x + g * G;
    if (t0 < A.ntiles) {
      m_cur = __ldg(reinterpret_cast<const int4*>(k8s.pos_meta) + t0);
      if (m_cur.y + lane < m_cur.z) pr_cur = __ldg(k8s.dag_pred + m_cur.y + lane);
    }
  }
  for (int t = blockIdx.x + g * G; t < A.ntiles; t += kGroups * G, k += kGroups) {
    const int s = k % NS;
    unsigned pv = (unsigned)kGroupWarps;
    if constexpr (ORDERED) {
      if (t + kGroups * G < A.ntiles) m_nx = __ldg(reinterpret_cast<const int4*>(k8s.pos_meta) + t + kGroups * G);
      if (m_cur.y + lane < m_cur.z && !(K4_DBG & 16)) {
        // acquire: a satisfied counter stays satisfied, so an early look is
        // valid; unsatisfied ones are polled again before the flush
        if (K8_ACQ == 0) pv = ld_acquire_u32(k8s.done + pr_cur);
        else pv = ld_relaxed_u32(k8s.done + pr_cur);
      }
    }
    // The parity waits below are safe only once the previous use of stage s
    // (tile k - NS) is complete: a group may finish its previous tile before
    // an older tile's block has landed.  So wait first until tile k - NS has
    // been consumed (empty[s], an mbarrier wait instead of a poll of
    // loader_k).  No alias there either when NS >= kGroups: tile k - 2 NS is
    // consumed (the loader issued this group's previous tile k - kGroups only
    // after every tile <= k - kGroups - NS was consumed), and tile k cannot be
    // yet.  Shallower rings poll loader_k.
    if constexpr (NS >= kGroups) {
      if (k >= NS) mbar_wait(&empty[s], (unsigned)(((k / NS) - 1) & 1));
    } else {
      while (true) {
        int lk;
        asm volatile("ld.volatile.shared.s32 %0, [%1];" : "=r"(lk) : "r"(smem_u32(&loader_k)) : "memory");
        if (lk > k) break;
        __nanosleep(32);
      }
    }
    mbar_wait(&blk_full[s], (unsigned)((k / NS) & 1));  // TMA data visible to this thread
    mbar_wait(&x_full[s], (unsigned)((k / NS) & 1));
    if (gt == 0) TRACE(k, 3);
    const unsigned char* blk = sm + s * slot_bytes;
    const TileDesc& D = *reinterpret_cast<const TileDesc*>(blk);
    const int T = D.nrows, S = D.nspill, W = T + S, row0 = D.row0;
    const double* xs = reinterpret_cast<const double*>(blk + A.block_cap) + (((uintptr_t)(x + row0) >> 3) & 1);
    const uint32_t* rseg = reinterpret_cast<const uint32_t*>(blk + sizeof(TileDesc));  // start | len << 16
    const uint16_t* lcol = reinterpret_cast<const uint16_t*>(blk + D.o_lcol);
    const uint32_t* tcsc = reinterpret_cast<const uint32_t*>(blk + D.o_tidx);
    const uint16_t* tptr = reinterpret_cast<const uint16_t*>(blk + D.o_tptr);
    const uint16_t* sid = reinterpret_cast<const uint16_t*>(blk + D.o_sid);
    const int32_t* tgt = reinterpret_cast<const int32_t*>(blk + D.o_tgt);
    // single-run tiles have no tgt[]: slot l >= wpad flushes to row tgt_base + l
    const int srun = D.gather_runs >> 1, tgt_base = D.tgt_base, wpad = T + (srun >> 1);
    auto spill_row = [&](int l) { return srun ? (l < wpad ? -1 : tgt_base + l) : tgt[l - T]; };
    const int32_t* slot = (ATOMIC || ORDERED) ? nullptr : k8s.slots + D.spill_off;
    const double* val = reinterpret_cast<const double*>(blk + D.o_val);
    // flush of window slot l: K4 one RED per (tile, target); K3 own rows
    // stored, spill contributions staged
    const int tile_id = ORDERED ? m_cur.x : t;
    if constexpr (ORDERED) {
      // K8, software-pipelined so that no L2 round trip sits between two
      // tiles of a group:
      //   1. acquire loads of this tile's DAG predecessors' flush counters
      //      (issued now, inspected after the sums);
      //   2. the slot sums in registers (at most kK8Slots per thread: the plan
      //      checks window_cap), flush targets and first-writer flags;
      //   3. the stage is released (nothing below reads it);
      //   5. wait until every predecessor has flushed (normally already true);
      //   6. flush: the first writer of a target (lowest phase) stores, later
      //      writers add with RED in DAG (= phase) order -- one writer at a time
      //      per target, so the sum order is fixed and the result bitwise
      //      reproducible; no old-value loads, nothing to wait for;
      //   7. signal the tile (last arriving warp of the group).
      // K8_ACQ 0: acquire loads of the predecessors' counters (above, before the
      // stage waits); 1: relaxed loads there, and the acquire is a
      // fence.acq_rel.gpu just before the flush (a strong read followed by a
      // fence is an acquire pattern; measured slower: st27 0.175 vs 0.143 ms)
      const int pb = m_cur.y, pe = m_cur.z;
      double acc8[kK8Slots];
      int gr8[kK8Slots];
      unsigned f8[kK8Slots];  // first-writer flags: loaded now, inspected at the flush
#pragma unroll
      for (int u = 0; u < kK8Slots; ++u) {
        const int i = gt + u * kGroupThreads;
        gr8[u] = -1;
        f8[u] = 0;
        if (i < W) {
          const int l = D.sorted ? (int)sid[i] : i;
          if (l < T) {
            gr8[u] = row0 + l;
            asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(f8[u]) : "l"(k8s.own_first + row0 + l));
          } else {
            gr8[u] = spill_row(l);
            if (gr8[u] >= 0)
              asm volatile("ld.global.nc.u8 %0, [%1];" : "=r"(f8[u]) : "l"(k8s.slot_first + D.spill_off + (l - T)));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kK8Slots; ++u) {
        const int i = gt + u * kGroupThreads;
        acc8[u] = 0.0;
        if (i < W) {
          double acc = 0.0;
          if (!D.sorted) {
            if (i < T) {
              const uint32_t sg = rseg[i];
              const int eb = (int)(sg & 0xffffu), ee = eb + (int)(sg >> 16);
#pragma unroll 2
              for (int e = eb; e < ee; ++e) acc += val[e] * xs[lcol[e]];
            }
            const int jb = tptr[i], je = tptr[i + 1];
#pragma unroll 2
            for (int j = jb; j < je; ++j) {
              const uint32_t q = tcsc[j];
              acc += val[q & 0xffffu] * xs[q >> 16];
            }
          } else {
            const uint32_t* pseg = reinterpret_cast<const uint32_t*>(blk + D.o_lcol);
            const uint32_t* rec = reinterpret_cast<const uint32_t*>(blk + D.o_tidx);
            const uint32_t ps = pseg[i];
            const int jb = (int)(ps & 0xffffu), nt = (int)(ps >> 16);
#pragma unroll 2
            for (int v = 0; v < nt; ++v) {
              const uint32_t q = rec[jb + v];
              acc += val[q & 0xffffu] * xs[q >> 16];
            }
          }
          acc8[u] = acc;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&empty[s]);  // 3. the stage is free
      // 4. the next tile's predecessor counter index (its meta has arrived)
      int pr_nx = 0;
      if (m_nx.y + lane < m_nx.z) pr_nx = __ldg(k8s.dag_pred + m_nx.y + lane);
      if (!(K4_DBG & 16)) {  // 5. (bit 4: diagnostics, no DAG wait)
        unsigned okp;  // pv inspected only here: the memory clobber keeps the compare after the sums
        asm volatile("{\n .reg .pred p;\n setp.ge.u32 p, %1, %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(okp) : "r"(pv), "n"(kGroupWarps) : "memory");
        if (!__all_sync(0xffffffffu, okp != 0)) {
          for (int q = pb + lane; q < pe; q += 32) {
            const unsigned* f = k8s.done + __ldg(k8s.dag_pred + q);
            while (ld_acquire_u32(f) < (unsigned)kGroupWarps) __nanosleep(32);
          }
          __syncwarp();
        } else {
          for (int q = pb + 32 + lane; q < pe; q += 32) {  // (tiles with > 32 predecessors)
            const unsigned* f = k8s.done + __ldg(k8s.dag_pred + q);
            while (ld_acquire_u32(f) < (unsigned)kGroupWarps) __nanosleep(32);
          }
          __syncwarp();
        }
        if (K8_ACQ == 1 && pe > pb) asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      if (!(K4_DBG & 4)) {  // 6.
#pragma unroll
        for (int u = 0; u < kK8Slots; ++u)
          if (gr8[u] >= 0) {
            unsigned fv;  // (the memory clobber keeps the flag's first use here, after the sums)
            asm volatile("mov.b32 %0, %1;" : "=r"(fv) : "r"(f8[u]) : "memory");
            if (fv != 0 || (K4_DBG & 32)) __stcg(y + gr8[u], acc8[u]);
            else red_add_f64(y + gr8[u], acc8[u]);
          }
      }
      // 7. signal: each warp arrives (release, CTA scope) on its group's
      // counter for the tile; the last of the 7 makes the group's flush
      // visible GPU-wide (one fence per tile instead of one per warp: the
      // fence waits for the REDs in flight) and signals for all 7
      __syncwarp();
      if (K8_SIGNALLER) {
        // publish this warp's progress (group tiles flushed); the signaller
        // warp fences and signals done[]
        if (lane == 0)
          asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(&k8_prog[wid])), "r"(k / kGroups + 1)
                       : "memory");
      } else if (lane == 0) {
        unsigned old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "r"(smem_u32(&k8_arrive[g][(k / kGroups) & 3])) : "memory");
        if ((old + 1) % (unsigned)kGroupWarps == 0) {
          if (!(K4_DBG & 64)) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // (bit 6: diagnostics, no fence)
          red_add_u32(k8s.done + tile_id, (unsigned)kGroupWarps);
        }
      }
      m_cur = m_nx;
      pr_cur = pr_nx;
    } else {
    auto flush = [&](int l, int sl, double acc) {
      if (K4_DBG & 4) {
        // diagnostics: no flush
      } else if (ATOMIC) {
        const int gr = l < T ? row0 + l : spill_row(l);
#ifdef K4_CHECK
        if (gr >= A.check_n) { printf("K4_CHECK flush t=%d l=%d gr=%d\n", t, l, gr); __trap(); }
#endif
        if (gr >= 0) red_add_f64(y + gr, acc);  // -1: pad slot of the spill window
      } else if (l < T) {
        y[row0 + l] = acc;
      } else if (sl >= 0) {
        __stcg(k8s.spill_buf + sl, acc);
      }
    };
    // one thread per window slot (fixed summation order per slot ->
    // deterministic):
    //   own row l:  sum_{e in row l} a_e x[c_e]                    (tmp)
    //   then:       sum_{e: c_e = l, e off-diagonal} a_e x[r_e]    (b[col] += ...)
    if (zero_pending) {  // first tile of this warp: every CTA has zeroed its slice of y
      k4_zero_wait(A.k8, zero_target);
      zero_pending = false;
    }
    if (!D.sorted) {
      // slot order: a warp walks the row parts of 32 consecutive slots in
      // lock step, then their transposed parts
      for (int l = gt; l < W; l += kGroupThreads) {
        // K3: the staging slot is fetched first so its latency overlaps the sums
        const int sl = (!ATOMIC && l >= T) ? __ldg(slot + (l - T)) : 0;
        double acc = 0.0;
        if (l < T && !(K4_DBG & 1)) {
          const uint32_t sg = rseg[l];
          const int eb = (int)(sg & 0xffffu), ee = eb + (int)(sg >> 16);
#pragma unroll 2  // kK4Unroll (internal.h)
          for (int e = eb; e < ee; ++e) acc += val[e] * xs[lcol[e]];
        }
        const int jb = tptr[l], je = (K4_DBG & 2) ? jb : tptr[l + 1];
#pragma unroll 2  // kK4Unroll (internal.h)
        for (int j = jb; j < je; ++j) {
          const uint32_t q = tcsc[j];
          acc += val[q & 0xffffu] * xs[q >> 16];
        }
        flush(l, sl, acc);
      }
    } else {
      // work-sorted: lane position i takes slot sid[i] and walks one list,
      // its row part then its transposed part (the lanes of a warp have
      // similar total lengths)
      const uint32_t* pseg = reinterpret_cast<const uint32_t*>(blk + D.o_lcol);  // start | len << 16
      const uint32_t* rec = reinterpret_cast<const uint32_t*>(blk + D.o_tidx);   // val index | x index << 16
      for (int i = gt; i < W; i += kGroupThreads) {
        const int l = sid[i];
        const int sl = (!ATOMIC && l >= T) ? __ldg(slot + (l - T)) : 0;
        const uint32_t ps = pseg[i];
        const int jb = (int)(ps & 0xffffu), nt = (K4_DBG & 3) ? 0 : (int)(ps >> 16);
        double acc = 0.0;
#pragma unroll 2  // kK4SortedUnroll (internal.h)
        for (int u = 0; u < nt; ++u) {
          const uint32_t q = rec[jb + u];
          acc += val[q & 0xffffu] * xs[q >> 16];
        }
        flush(l, sl, acc);
      }
    }
    }  // !ORDERED
    if (gt == 0) TRACE(k, 4);
    if (!ORDERED) {
      // release stage s: each warp arrives once its reads of the stage are done
      // (K8 released it before its flush)
      __syncwarp();
      if (lane == 0) mbar_arrive_relaxed(&empty[s]);
    }
    if (gt == 0) TRACE(k, 5);
  }

}

// K3 second kernel: y[r] += staged contributions of row r in slot order.
__global__ void __launch_bounds__(256) k_fixup(FixupArgs F, double* __restrict__ y) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; r < F.n; r += stride) {
    const int jb = F.in_ptr[r], je = F.in_ptr[r + 1];
    if (jb == je) continue;
    double acc = y[r];
    for (int j = jb; j < je; ++j) acc += __ldcs(F.spill_buf + j);
    y[r] = acc;
  }
}

// ---------------------------------------------------------------- K5 colored_smem
// RACE colouring executed inside a shared-memory window (format: cs_build.cpp).
// One persistent CTA per SM takes the tiles blockIdx.x, +gridDim.x, ... in
// BFS order.  Warp roles:
//   head producer (lane 0 of warp 1): one bulk copy (TMA, cp.async.bulk) per
//     tile head into a double-buffered head area, as soon as the tile two
//     back is finished;
//   chunk producer (lane 0 of warp 0): one bulk copy per chunk of the tile's
//     entry pieces into a kStages-deep ring (mbarrier full/empty); chunk
//     offsets and sizes come from the head in shared memory (no global loads
//     on the producer's critical path);
//   2 gather warps (tiles alternate between them): x of the tile window (own
//     rows row0.., then the spill targets) into a double-buffered xs, with
//     cp.async, while the consumers still work on the previous tile;
//   NC consumer warps: ys = 0; colour by colour (colours in
//     sequence, one barrier between them), one lane per row of the colour:
//         acc = d_r x_r + sum_j a_rj xs[c_j]          (Alg. 2 tmp)
//         ys[c_j] += a_rj x_r                          (Alg. 2 b[col] +=)
//         ys[r]  += acc
//     plain shared-memory read-modify-writes: rows of one colour have disjoint
//     write sets; the step order of every row makes the
//     16 lanes of a half warp hit 16 different bank pairs; then the window is
//     flushed, y[global(l)] += ys[l] (fp64 RED: other tiles share rows).
constexpr int kCsMaxStages = 8;
#ifdef CS_PROF
#define CSP_DECL long long csp_acc[10] = {0}; long long csp_t = clock64();
#define CSP(i) do { const long long _n = clock64(); csp_acc[i] += _n - csp_t; csp_t = _n; } while (0)
#define CSP_CNT(i) (csp_acc[i]++)
#else
#define CSP_DECL
#define CSP(i) do {} while (0)
#define CSP_CNT(i) do {} while (0)
#endif

__device__ __forceinline__ void prefetch_l2(const void* p, int64_t bytes) {
  if (bytes <= 0) return;
  const uintptr_t a = (uintptr_t)p & ~uintptr_t(15);
  const uintptr_t e = ((uintptr_t)p + (uintptr_t)bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}
constexpr int kCsGather = 2;
constexpr int kCsRoleWarps = 2 + kCsGather;  // chunk producer, head producer, gather warps

__device__ __forceinline__ void cs_cbar(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// NU (4, 8, 12 or 16) JDS steps of one piece, straight-line: every lane reads
// an entry at every step (start of step u's run + lane); lanes whose row is
// shorter are redirected to the zero dummy slot `dummy` with a = 0.  The
// columns of one row are distinct and rows of one colour are write-disjoint,
// so all loads of y can precede all stores.
template <int NU, bool V1>
__device__ __forceinline__ void cs_steps(const double* __restrict__ val, const uint16_t* __restrict__ lc,
                                         const uint32_t (&ew)[8], int j0, int L, int lgv, int sub, int lane, unsigned lt,
                                         const double* __restrict__ xs, double* ys, double xr, int dummy,
                                         double (&acc)[4]) {
  double a[NU], xv[NU], yv[NU];
  int c[NU];
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    // lane (row, sub) holds entry (j0 + u) * V + sub of its row; the valid
    // lanes of a step are stored in lane order
    const int e0 = u == 0 ? 0 : (int)((ew[(u - 1) >> 1] >> (((u - 1) & 1) * 16)) & 0xffffu);
    const bool v = (((j0 + u) << lgv) + sub) < L;
    // one lane per row: the valid lanes of a step are a prefix (lengths descend)
    const int ix = V1 ? e0 + lane : e0 + __popc(__ballot_sync(0xffffffffu, v) & lt);
    const double a0 = val[ix];
    const int c0 = lc[ix];
    a[u] = v ? a0 : 0.0;
    c[u] = v ? c0 : dummy;
  }
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    xv[u] = xs[c[u]];
    yv[u] = ys[c[u]];
  }
#pragma unroll
  for (int u = 0; u < NU; ++u) {
    acc[u & 3] = fma(a[u], xv[u], acc[u & 3]);
    ys[c[u]] = fma(a[u], xr, yv[u]);
  }
}

template <int NC>
__global__ void __launch_bounds__(32 * (kCsRoleWarps + NC), 1)
    k_cs(


CsArgs A, const double* __restrict__ x, double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t head_full[2], head_empty[2], x_full[2], x_empty[2];
  __shared__ __align__(8) uint64_t ring_full[kCsMaxStages], ring_empty[kCsMaxStages];
  const int NS = A.stages;
  const int Hb = (A.Hcap + 127) & ~127;
  const int Wc = (A.Wcap + 15) & ~15;  // window slots; slot Wc is a zero dummy
  const int Ws = Wc + 16;
  unsigned char* heads = sm;
  double* xs0 = reinterpret_cast<double*>(sm + 2 * Hb);
  double* ys = xs0 + 2 * Ws;
  unsigned char* ring = reinterpret_cast<unsigned char*>(ys + Ws);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int G = gridDim.x;
  const int nk = A.ntiles > (int)blockIdx.x ? (A.ntiles - (int)blockIdx.x + G - 1) / G : 0;
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&head_full[i], 1);
      mbar_init(&head_empty[i], 1);
      mbar_init(&x_full[i], 32);
      mbar_init(&x_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&ring_full[i], 1);
      mbar_init(&ring_empty[i], kCsReleaseUnits);  // piece weights of a chunk sum to this
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    xs0[Wc] = 0.0;
    xs0[Ws + Wc] = 0.0;
  }
  __syncthreads();
  if (wid == 0) {
    // ------------------------------------------------ chunk producer (TMA bulk copies)
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      uint32_t cseq = 0;
      for (int k = 0; k < nk; ++k) {
        const int hb = k & 1;
        mbar_wait(&head_full[hb], (unsigned)((k >> 1) & 1));
        const CsHeadHdr* H = reinterpret_cast<const CsHeadHdr*>(heads + hb * Hb);
        const int nch = H->nchunks;
        const uint32_t* clen = reinterpret_cast<const uint32_t*>(heads + hb * Hb + H->o_clen);
        int64_t off = H->chunk_base;
        for (int c = 0; c < nch; ++c, ++cseq) {
          const int st = (int)(cseq & (uint32_t)(NS - 1));
          const uint32_t use = cseq >> A.lgstages;
          const unsigned len = clen[c];
          if (A.trace && blockIdx.x == 0 && cseq < (uint32_t)A.trace_cap) A.trace[2 * cseq] = gtimer();
          if (use > 0) mbar_wait(&ring_empty[st], (use - 1) & 1);
          if (A.trace && blockIdx.x == 0 && cseq < (uint32_t)A.trace_cap) A.trace[2 * cseq + 1] = gtimer();
          mbar_arrive_expect_tx(&ring_full[st], len);
          bulk_g2s_stream(ring + (size_t)st * A.chunk, A.blocks + off, len, &ring_full[st], pol);
          off += len;
        }
      }
    }
    return;
  }
  if (wid == 1) {
    // ------------------------------------------------ head producer
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int k = 0; k < nk; ++k) {
        const CsDesc* D = A.desc + blockIdx.x + (size_t)k * G;
        const int hb = k & 1;
        const int64_t hoff = __ldg(&D->head_off);
        const int hbytes = __ldg(&D->head_bytes), bbytes = __ldg(&D->block_bytes);
        if (k >= 2) mbar_wait(&head_empty[hb], (unsigned)(((k >> 1) - 1) & 1));
        mbar_arrive_expect_tx(&head_full[hb], (unsigned)hbytes);
        bulk_g2s_stream(heads + hb * Hb, A.blocks + hoff, (unsigned)hbytes, &head_full[hb], pol);
        // the whole tile into L2 now (about one tile ahead of its consumption):
        // the ring's bulk copies then hit L2 and need far fewer bytes in flight
        if (!(A.debug_skip & 16))
          for (int64_t o = hbytes; o < bbytes; o += 32768)
            prefetch_l2(A.blocks + hoff + o, min((int64_t)32768, (int64_t)bbytes - o));
      }
    }
    return;
  }
  if (wid < kCsRoleWarps) {
    // ------------------------------------------------ gather warps (x windows)
    const int gw = wid - 2;
    for (int k = gw; k < nk; k += kCsGather) {
      const int xb = k & 1;
      mbar_wait(&head_full[xb], (unsigned)((k >> 1) & 1));
      if (k >= 2) mbar_wait(&x_empty[xb], (unsigned)(((k >> 1) - 1) & 1));
      const CsHeadHdr* H = reinterpret_cast<const CsHeadHdr*>(heads + xb * Hb);
      const int row0 = H->row0, T = H->T, S = H->S;
      const int32_t* tgt = reinterpret_cast<const int32_t*>(heads + xb * Hb + H->o_tgt);
      double* xsb = xs0 + xb * Ws;
      if (!(A.debug_skip & 32)) {
        for (int i = lane; i < T; i += 32) cp_async8(xsb + i, x + row0 + i);
#pragma unroll 4
        for (int i = lane; i < S; i += 32) cp_async8(xsb + T + i, x + tgt[i]);
      }
      cp_async_arrive_noinc(&x_full[xb]);
    }
    return;
  }
  // -------------------------------------------------- consumers
  constexpr int NCT = NC * 32;
  const int cw = wid - kCsRoleWarps, ct = tid - 32 * kCsRoleWarps;
  const int smask = NS - 1;
  uint32_t cbase = 0;
  CSP_DECL
  for (int k = 0; k < nk; ++k) {
    const int hb = k & 1;
    unsigned long long* tr = (A.trace && blockIdx.x == 0 && ct == 0 && k < 256) ? A.trace + 2 * A.trace_cap + 4 * k : nullptr;
    if (tr) tr[0] = gtimer();
    mbar_wait(&head_full[hb], (unsigned)((k >> 1) & 1));
    const unsigned char* hd = heads + hb * Hb;
    const CsHeadHdr* H = reinterpret_cast<const CsHeadHdr*>(hd);
    const int row0 = H->row0, T = H->T, S = H->S, nc = H->ncolors, nch = H->nchunks;
    const uint16_t* cslc = reinterpret_cast<const uint16_t*>(hd + H->o_cslc);
    const uint4* srec = reinterpret_cast<const uint4*>(hd + H->o_srec);
    const uint32_t* ploc = reinterpret_cast<const uint32_t*>(hd + H->o_ploc);
    const uint16_t* pw = reinterpret_cast<const uint16_t*>(hd + H->o_pw);
    const int32_t* tgt = reinterpret_cast<const int32_t*>(hd + H->o_tgt);
    for (int i = ct; i < T + S; i += NCT) ys[i] = 0.0;
    mbar_wait(&x_full[hb], (unsigned)((k >> 1) & 1));
    const double* xsb = xs0 + hb * Ws;
    cs_cbar(NCT);
    if (tr) tr[1] = gtimer();
    CSP(6);
    for (int kk = 0; kk < nc; ++kk) {
      const int s1 = cslc[kk + 1];
      for (int s = cslc[kk] + cw; s < s1; s += NC) {
        const uint4 rec = srec[s];  // CsSliceRec
        const uint32_t ploc0 = rec.x;
        const int p0 = (int)(rec.y & 0xffffu), nsteps = (int)(rec.y >> 16);
        const int npc = (int)(rec.z & 0xffu), m = (int)((rec.z >> 8) & 0xffu);
        int L = 0, lr = 0;
        double d = 0.0, xr = 0.0;
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const int sub = lane & ((1 << A.lgv) - 1), row_i = lane >> A.lgv;
        const unsigned lt = (1u << lane) - 1u;
        CSP(0);
        for (int kp = 0; kp < npc; ++kp) {
          const uint32_t loc = kp == 0 ? ploc0 : ploc[p0 + kp];
          const uint32_t ch = cbase + (loc >> 20);
          const int st = (int)(ch & (uint32_t)smask);
          mbar_wait(&ring_full[st], (ch >> A.lgstages) & 1);
          CSP(1);
          const unsigned char* b = ring + (size_t)st * A.chunk + (loc & 0xfffffu);
          const uint4 e0 = reinterpret_cast<const uint4*>(b)[0];  // eo[0..7]
          const uint4 e1 = reinterpret_cast<const uint4*>(b)[1];  // eo[8..15]
          const uint32_t ew[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
          const int nnzp = (int)(e1.w >> 16);
          if (kp == 0) {  // the lane's row: window id, length, diagonal (zeros past m)
            lr = reinterpret_cast<const uint16_t*>(b + 32)[lane];
            L = reinterpret_cast<const uint16_t*>(b + 96)[lane];
            d = reinterpret_cast<const double*>(b + 160)[lane];
            if (A.debug_skip & 1) L = 0;
            xr = xsb[lr];
            b += 416;
          } else {
            b += 32;
          }
          const double* val = reinterpret_cast<const double*>(b);
          const uint16_t* lc = reinterpret_cast<const uint16_t*>(b + 8 * nnzp);
          const int j0 = kp * 16, nst = min(16, nsteps - j0);
          if (A.lgv == 0) {
            switch ((nst + 3) >> 2) {
              case 4: cs_steps<16, true>(val, lc, ew, j0, L, 0, 0, lane, lt, xsb, ys, xr, Wc, acc); break;
              case 3: cs_steps<12, true>(val, lc, ew, j0, L, 0, 0, lane, lt, xsb, ys, xr, Wc, acc); break;
              case 2: cs_steps<8, true>(val, lc, ew, j0, L, 0, 0, lane, lt, xsb, ys, xr, Wc, acc); break;
              case 1: cs_steps<4, true>(val, lc, ew, j0, L, 0, 0, lane, lt, xsb, ys, xr, Wc, acc); break;
              default: break;
            }
          } else {
            switch ((nst + 3) >> 2) {
              case 4: cs_steps<16, false>(val, lc, ew, j0, L, A.lgv, sub, lane, lt, xsb, ys, xr, Wc, acc); break;
              case 3: cs_steps<12, false>(val, lc, ew, j0, L, A.lgv, sub, lane, lt, xsb, ys, xr, Wc, acc); break;
              case 2: cs_steps<8, false>(val, lc, ew, j0, L, A.lgv, sub, lane, lt, xsb, ys, xr, Wc, acc); break;
              case 1: cs_steps<4, false>(val, lc, ew, j0, L, A.lgv, sub, lane, lt, xsb, ys, xr, Wc, acc); break;
              default: break;
            }
          }
          CSP(2);
          __syncwarp();  // every lane is done with the piece: release its share of the stage
          if (lane == 0) mbar_arrive_cnt(&ring_empty[st], pw[p0 + kp]);
          CSP(3);
          CSP_CNT(8);
        }
        double sum = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        for (int o = (1 << A.lgv) >> 1; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (sub == 0 && row_i < m) ys[lr] += fma(d, xr, sum);
        CSP(4);
        CSP_CNT(9);
      }
      cs_cbar(NCT);
      CSP(5);
    }
    if (tr) tr[2] = gtimer();
    // flush (the head's tgt list is still valid: head_empty is released below)
    if (!(A.debug_skip & 4)) {
      for (int i = ct; i < T; i += NCT) red_add_f64(y + row0 + i, ys[i]);
      for (int i = ct; i < S; i += NCT) red_add_f64(y + tgt[i], ys[T + i]);
    }
    cs_cbar(NCT);
    if (tr) tr[3] = gtimer();
    CSP(7);
    if (ct == 0) {
      mbar_arrive(&head_empty[hb]);
      mbar_arrive(&x_empty[hb]);
    }
    cbase += (uint32_t)nch;
  }
#ifdef CS_PROF
  if (lane == 0 && A.trace) for (int i = 0; i < 10; ++i) atomicAdd(A.trace + 2 * A.trace_cap + 1024 + 2048 + i, (unsigned long long)csp_acc[i]);
#endif
}

// K5 bandwidth probe (load-only / copy), 16-B streaming accesses, grid-stride
__global__ void __launch_bounds__(512) k_bw_load(const double2* __restrict__ p, int64_t n2, double* sink) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p + i));
    s += v.x + v.y;
  }
  if (s == 1.2345e-300) *sink = s;  // never true for the probe's data: keeps the loads
}
__global__ void __launch_bounds__(512) k_bw_copy(const double2* __restrict__ a, double2* __restrict__ b, int64_t n2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
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
  k_zero<<<grid_for((n + 1) / 2, 256), 256, 0, (cudaStream_t)stream>>>(y, n);
  return (int)cudaGetLastError();
}
int launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream) {
  if (n <= 0) return 0;
  k_gather<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(src, idx, dst, n);
  return (int)cudaGetLastError();
}
int launch_add(double* y, const double* v, int64_t n, void* stream) {
  if (n <= 0) return 0;
  k_add<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(y, v, n);
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
  // SYMM_K1_PREREDUCE=1: the flat kernel with __match_any_sync pre-reduction
  // (k_atomic_pr).  Not the default: measured on B200 (st27_128, ncu,
  // profiles/r2/k1_prereduce.md) it issues 14% fewer RED instructions but
  // takes 0.345 ms against 0.191 ms for the V-lanes-per-row kernel below,
  // whose shuffle reduction of each row's sum is the warp-level segmented
  // pre-reduction that pays (rows are the segments; equal transposed targets
  // inside one warp step are rare in a bandwidth-reduced order).
  static const bool prered = std::getenv("SYMM_K1_PREREDUCE") && std::atoi(std::getenv("SYMM_K1_PREREDUCE")) != 0;
  if (prered) {
    const int64_t chunks = ((int64_t)A.n + kK1Rows - 1) / kK1Rows;
    const int64_t g = (chunks * 32 + threads - 1) / threads, gmax = (int64_t)sms * 8;
    k_atomic_pr<<<(int)std::max<int64_t>(1, std::min(g, gmax)), threads, 0, st>>>(A, x, y);
    return (int)cudaGetLastError();
  }
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

int launch_spmv(const CsrArgs& A, const double* x, double* y, int vec, int sms, void* stream) {
  if (A.n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  int64_t warps_needed = ((int64_t)A.n * vec + 31) / 32;
  int64_t g = (warps_needed * 32 + threads - 1) / threads;
  int64_t gmax = (int64_t)sms * 8;
  int grid = (int)(g < gmax ? (g < 1 ? 1 : g) : gmax);
  switch (vec) {
    case 1: k_spmv<1><<<grid, threads, 0, st>>>(A, x, y); break;
    case 2: k_spmv<2><<<grid, threads, 0, st>>>(A, x, y); break;
    case 4: k_spmv<4><<<grid, threads, 0, st>>>(A, x, y); break;
    case 8: k_spmv<8><<<grid, threads, 0, st>>>(A, x, y); break;
    case 16: k_spmv<16><<<grid, threads, 0, st>>>(A, x, y); break;
    default: k_spmv<32><<<grid, threads, 0, st>>>(A, x, y); break;
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

int launch_sweep_phase(int kind, const CsrArgs& A, const int32_t* rows, int32_t nrows, const double* b, double* x,
                       int vec, void* stream) {
  if (nrows <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256, rpb = (threads / 32) * (32 / vec);
  const int grid = (int)std::min<int64_t>(((int64_t)nrows + rpb - 1) / rpb, 148 * 16);
#define SWEEP_CASE(VV)                                                                     \
  case VV:                                                                                 \
    if (kind == 1) k_sweep<1, VV><<<grid, threads, 0, st>>>(A, rows, nrows, b, x);          \
    else k_sweep<2, VV><<<grid, threads, 0, st>>>(A, rows, nrows, b, x);                    \
    break;
  switch (vec) {
    SWEEP_CASE(1)
    SWEEP_CASE(2)
    SWEEP_CASE(4)
    SWEEP_CASE(8)
    SWEEP_CASE(16)
    default:
      if (kind == 1) k_sweep<1, 32><<<grid, threads, 0, st>>>(A, rows, nrows, b, x);
      else k_sweep<2, 32><<<grid, threads, 0, st>>>(A, rows, nrows, b, x);
  }
#undef SWEEP_CASE
  return (int)cudaGetLastError();
}

int launch_tree(const CsrArgs& A, const ColoredArgs& C, const TreeArgs& T, const double* x, double* y, int vec,
                int grid, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  switch (vec) {
    case 1: k_tree<1><<<grid, threads, 0, st>>>(A, C, T, x, y); break;
    case 2: k_tree<2><<<grid, threads, 0, st>>>(A, C, T, x, y); break;
    case 4: k_tree<4><<<grid, threads, 0, st>>>(A, C, T, x, y); break;
    case 8: k_tree<8><<<grid, threads, 0, st>>>(A, C, T, x, y); break;
    case 16: k_tree<16><<<grid, threads, 0, st>>>(A, C, T, x, y); break;
    default: k_tree<32><<<grid, threads, 0, st>>>(A, C, T, x, y); break;
  }
  return (int)cudaGetLastError();
}

int tiled_smem_bytes(const TiledArgs& T) {
  return T.stages * (T.block_cap + 8 * T.window_cap);
}

// The dynamic shared-memory limit is a property of the kernel, shared by every
// plan: it is raised to the device's opt-in maximum (never lowered to one
// plan's size, which would break launches of an earlier plan with bigger
// blocks); each launch passes its own plan's size.
template <int NS>
static int tiled_attr(int smem) {
  int rc = (int)cudaFuncSetAttribute(k_tiled<0, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (!rc) rc = (int)cudaFuncSetAttribute(k_tiled<1, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (!rc) rc = (int)cudaFuncSetAttribute(k_tiled<2, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  return rc;
}

// Deepest ring (8, 6, 5, 4, 3 or 2 stages) whose shared memory fits one SM.
int tiled_max_ctas_per_sm(int vec, const TiledArgs& T0, int* out) {
  (void)vec;
  TiledArgs T = T0;
  int devsmem = 0;
  cudaDeviceGetAttribute(&devsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  const int cand[] = {8, 6, 5, 4, 3, 2};
  for (int ns : cand) {
    T.stages = ns;
    const int smem = tiled_smem_bytes(T);
    if (smem + 1024 > devsmem) continue;
    const int lim = devsmem - 1024;  // static smem (mbarriers, loader_k) stays below 1 KB
    int rc = 0;
    switch (ns) {
      case 8: rc = tiled_attr<8>(lim); break;
      case 6: rc = tiled_attr<6>(lim); break;
      case 5: rc = tiled_attr<5>(lim); break;
      case 4: rc = tiled_attr<4>(lim); break;
      case 3: rc = tiled_attr<3>(lim); break;
      default: rc = tiled_attr<2>(lim); break;
    }
    if (rc) return rc;
    // every CTA of the persistent grid (<= one per SM) must be resident at once:
    // K4's zero wait and K8's DAG waits span CTAs
    int occ = 0;
    switch (ns) {
      case 8: rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<1, 8>, kTiledThreads, smem); break;
      case 6: rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<1, 6>, kTiledThreads, smem); break;
      case 5: rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<1, 5>, kTiledThreads, smem); break;
      case 4: rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<1, 4>, kTiledThreads, smem); break;
      case 3: rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<1, 3>, kTiledThreads, smem); break;
      default: rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tiled<1, 2>, kTiledThreads, smem); break;
    }
    if (rc) return rc;
    if (occ < 1) continue;
    *out = ns;
    return 0;
  }
  *out = 0;
  return 0;
}

int launch_tiled(const TiledArgs& T, const double* x, double* y, int vec, int grid, int mode, void* stream) {
  (void)vec;
  if (T.ntiles <= 0) return 0;
  // programmatic dependent launch: the kernel's loader streams tile blocks
  // while the previous kernel of the stream finishes; every access to x or y
  // waits for it (griddepcontrol.wait)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kTiledThreads);
  cfg.dynamicSmemBytes = (size_t)tiled_smem_bytes(T);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // K4 (grid-wide zero wait) and K8 (DAG waits on other CTAs) need every CTA
  // resident at once: a cooperative launch guarantees it or fails
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = 1;
  cfg.attrs = attr;
  // K8 launches cooperatively (its DAG waits span CTAs).  K4's one grid-wide wait
  // (zeroed y) relies on the plan's grid <= SMs x occupancy (checked at plan
  // time); a cooperative launch measured ~2.5 us slower per multiply (it gives
  // up the overlap with the previous kernel).  SYMM_COOP=1 forces it for K4.
  static const bool coop4 = std::getenv("SYMM_COOP") && std::atoi(std::getenv("SYMM_COOP")) != 0;
  cfg.numAttrs = (mode == 2 || (mode == 1 && coop4)) ? 2 : 1;
  cudaError_t e = cudaErrorInvalidValue;
#define LT(NSV)                                                                                  \
  case NSV:                                                                                      \
    e = mode == 1 ? cudaLaunchKernelEx(&cfg, k_tiled<1, NSV>, T, x, y)                           \
                  : mode == 2 ? cudaLaunchKernelEx(&cfg, k_tiled<2, NSV>, T, x, y)                \
                              : cudaLaunchKernelEx(&cfg, k_tiled<0, NSV>, T, x, y);               \
    break;
  switch (T.stages) {
    LT(8) LT(6) LT(5) LT(4) LT(3) LT(2)
    default: return (int)cudaErrorInvalidValue;
  }
#undef LT
  if (e != cudaSuccess) return (int)e;
  return (int)cudaGetLastError();
}

int cs_smem_bytes(const CsArgs& A) {
  const int64_t Hb = (A.Hcap + 127) & ~127, Ws = ((A.Wcap + 15) & ~15) + 16;
  return (int)(2 * Hb + 24 * Ws + (int64_t)A.stages * A.chunk + 1024);  // + over-read pad of the ring
}

#define CS_INSTANCES(X) X(8) X(12) X(16)

int cs_configure(CsArgs& A, int* ctas_per_sm, int nc) {
  const int smem = cs_smem_bytes(A);
  int devsmem = 0;
  cudaDeviceGetAttribute(&devsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  *ctas_per_sm = 0;
  if (smem + 1024 > devsmem || A.stages > kCsMaxStages) return 0;
  int rc = (int)cudaErrorInvalidValue;
#define CS_CFG(NN)                                                                                    \
  if (nc == NN) {                                                                                     \
    rc = (int)cudaFuncSetAttribute(k_cs<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, devsmem - 1024); \
    if (!rc) rc = (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas_per_sm, k_cs<NN>, 32 * (kCsRoleWarps + NN), smem); \
  }
  CS_INSTANCES(CS_CFG)
#undef CS_CFG
  return rc;
}

int launch_cs(const CsArgs& A, const double* x, double* y, int grid, int nc, void* stream) {
  if (A.ntiles <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = cs_smem_bytes(A);
#define CS_LAUNCH(NN) \
  if (nc == NN) k_cs<NN><<<grid, 32 * (kCsRoleWarps + NN), smem, st>>>(A, x, y);
  CS_INSTANCES(CS_LAUNCH)
#undef CS_LAUNCH
  return (int)cudaGetLastError();
}

int bw_probe(int mode, int64_t bytes, int reps, void* stream, double* gbps) {
  cudaStream_t st = (cudaStream_t)stream;
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n2 = bytes / 16;
  double2 *a = nullptr, *b = nullptr;
  double* sink = nullptr;
  cudaError_t e = cudaMalloc(&a, (size_t)n2 * 16);
  if (e == cudaSuccess && mode == 1) e = cudaMalloc(&b, (size_t)n2 * 16);
  if (e == cudaSuccess) e = cudaMalloc(&sink, 8);
  if (e == cudaSuccess) e = cudaMemsetAsync(a, 0, (size_t)n2 * 16, st);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (e == cudaSuccess) e = cudaEventCreate(&e0);
  if (e == cudaSuccess) e = cudaEventCreate(&e1);
  float best = 1e30f;
  const int grid = sms * 4;
  for (int r = 0; e == cudaSuccess && r <= reps; ++r) {
    cudaEventRecord(e0, st);
    if (mode == 1) k_bw_copy<<<grid, 512, 0, st>>>(a, b, n2);
    else k_bw_load<<<grid, 512, 0, st>>>(a, n2, sink);
    cudaEventRecord(e1, st);
    e = cudaEventSynchronize(e1);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
    if (r > 0 && ms < best) best = ms;  // pass 0 is the warm-up
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  cudaFree(a);
  if (b) cudaFree(b);
  if (sink) cudaFree(sink);
  if (e != cudaSuccess) return (int)e;
  *gbps = (double)n2 * 16.0 * (mode == 1 ? 2.0 : 1.0) / (best * 1e-3) / 1e9;
  return 0;
}

int launch_fixup(const FixupArgs& F, double* y, void* stream) {
  if (F.n <= 0) return 0;
  k_fixup<<<grid_for(F.n, 256), 256, 0, (cudaStream_t)stream>>>(F, y);
  return (int)cudaGetLastError();
}

}  // namespace symm
