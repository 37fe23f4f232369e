// C ABI of libsymmspmv.so (include/symmspmv.h): schedule objects, plans
// (device upload of the variant formats), runs.  Host code compiled by nvcc.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"

namespace symm {
const char* last_error();
}

struct race_schedule {
  symm::Schedule S;
};

using namespace symm;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

}  // namespace

struct symmspmv_plan {
  int device = 0;
  int variant = SYMM_VARIANT_AUTO;
  int vec = 4;
  int sms = 148;
  int vec_order = SYMM_ORDER_PERMUTED;
  int32_t n = 0;
  int64_t nnz = 0;
  int nranks = 1, rank = 0;
  int32_t row_begin = 0, row_end = 0, local_end = 0;
  std::vector<DevBuf> bufs;
  int64_t device_bytes = 0;
  // K1 / K2: permuted CRS
  bool has_csr = false;
  int32_t *d_rp = nullptr, *d_col = nullptr;
  double* d_val = nullptr;
  // K2
  bool has_colored = false;
  int32_t *d_tile_ptr = nullptr, *d_phase_tiles = nullptr, *d_srow = nullptr, *d_tile_sub_ptr = nullptr,
          *d_sub_ptr = nullptr;
  std::vector<int32_t> phase_off;  // host: offsets of phases in d_phase_tiles
  // K3
  bool has_tiled = false;
  TiledArgs targs{};
  int tiled_grid = 0;
  // multi-rank plans: tiles that read x or write y beyond row_end (halo rows)
  // form a second launch, so the interior tiles can run while the x halo is in
  // flight (symmspmv_run_part); single-rank plans keep every tile in targs
  TiledArgs targs_b{};
  int tiled_grid_b = 0;
  int64_t nnz_interior = 0, nnz_boundary = 0;
  int32_t tiled_nnz_cap = 0;
  int tiled_occ = 0;
  int32_t* d_in_ptr = nullptr;
  FixupArgs fargs{};
  // K8 tiled_colored
  bool has_tiled_colored = false;
  bool k4_self_zero = true;         // k_tiled<1> zeroes y itself (no k_zero launch)
  unsigned int* k8_done = nullptr;  // host copy of the counters' address (memset per run)
  // K7 recursive tree
  bool has_tree = false;
  TreeArgs tree{};
  int tree_grid = 0;
  // K6 full-matrix SpMV (yardstick)
  bool has_spmv = false;
  int32_t *d_frp = nullptr, *d_fcol = nullptr;
  double* d_fval = nullptr;
  int spmv_vec = 8;
  int64_t spmv_nnz = 0;
  // K5 colored_smem
  bool has_cs = false;
  CsArgs cargs{};
  int cs_grid = 0;
  int cs_occ = 0;
  int cs_nc = 12;
  int64_t cs_sum_colors = 0, cs_sum_spill = 0;
  // vector order / host staging
  int32_t *d_perm = nullptr, *d_inv = nullptr;
  double *d_xp = nullptr, *d_yp = nullptr;
  int last_launches = 0;
  int64_t min_bytes = 0;
};

namespace {

int cuda_fail(cudaError_t e, const char* what) {
  return set_error(SYMM_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

template <class T>
int dev_alloc(symmspmv_plan_t* P, T** out, size_t count) {
  void* p = nullptr;
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(SYMM_ERR_OOM, "cudaMalloc(%zu bytes) failed: %s", bytes, cudaGetErrorString(e));
  }
  P->bufs.push_back({p, bytes});
  P->device_bytes += (int64_t)bytes;
  *out = (T*)p;
  return SYMM_OK;
}

template <class T>
int upload(symmspmv_plan_t* P, T** out, const T* host, size_t count) {
  int rc = dev_alloc(P, out, count);
  if (rc) return rc;
  if (count) {
    cudaError_t e = cudaMemcpy(*out, host, count * sizeof(T), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy H2D");
  }
  return SYMM_OK;
}

void free_plan(symmspmv_plan_t* P) {
  if (!P) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(P->device);
  for (auto& b : P->bufs) cudaFree(b.p);
  cudaSetDevice(cur);
  delete P;
}

int pick_vec(int64_t nnz, int32_t n) {
  double avg = n > 0 ? (double)nnz / (double)n : 1.0;  // SymmNNZR (Eq. 4 with the diagonal)
  int v = 1;
  while (v < 32 && v < avg) v *= 2;
  return std::max(v, 2);
}

static inline int64_t align16(int64_t v) { return (v + 15) & ~int64_t(15); }

// Contiguous tile ranges per rank, balanced by stored nonzeros (R23).
void partition_tiles(const Schedule& S, int nranks, std::vector<int32_t>& tile_bounds,
                     std::vector<int32_t>& row_bounds, std::vector<int32_t>& halo_end) {
  const int32_t nt = (int32_t)S.tile_group.size();
  tile_bounds.assign((size_t)nranks + 1, nt);
  tile_bounds[0] = 0;
  const int64_t total = S.nnz;
  int64_t cum = 0;
  int r = 1;
  for (int32_t t = 0; t < nt && r < nranks; ++t) {
    cum += S.prow_ptr[(size_t)S.tile_ptr[(size_t)t + 1]] - S.prow_ptr[(size_t)S.tile_ptr[(size_t)t]];
    while (r < nranks && cum * nranks >= (int64_t)r * total) tile_bounds[(size_t)r++] = t + 1;
  }
  row_bounds.assign((size_t)nranks + 1, S.n);
  halo_end.assign((size_t)nranks, S.n);
  for (int q = 0; q <= nranks; ++q) row_bounds[(size_t)q] = nt ? S.tile_ptr[(size_t)tile_bounds[(size_t)q]] : 0;
  row_bounds[(size_t)nranks] = S.n;
  for (int q = 0; q < nranks; ++q) {
    int32_t h = row_bounds[(size_t)q + 1];
    for (int32_t t = tile_bounds[(size_t)q]; t < tile_bounds[(size_t)q + 1]; ++t)
      if (S.spill_ptr[(size_t)t + 1] > S.spill_ptr[(size_t)t])
        h = std::max(h, (int32_t)((uint32_t)S.spill[(size_t)S.spill_ptr[(size_t)t + 1] - 1] & kIdxMask) + 1);
    halo_end[(size_t)q] = h;
  }
}

// Window id of column c in a tile [r0, r1) with spill runs tr[0..nrt):
// own rows 0..T-1, spill targets through the runs; -1 if c is not in the window.
static int32_t run_local(const SpillRun* tr, int32_t nrt, int32_t r0, int32_t r1, int32_t c) {
  if (c >= r0 && c < r1) return c - r0;
  int32_t lo = 0, hi = nrt;  // last run with first row <= c
  while (lo < hi) {
    const int32_t mid = (lo + hi) / 2;
    if (tr[mid].row <= c) lo = mid + 1;
    else hi = mid;
  }
  if (lo == 0 || c >= tr[lo - 1].row + tr[lo - 1].len) return -1;
  return tr[lo - 1].wid + (c - tr[lo - 1].row);
}

// K3/K4 format (see TileDesc in internal.h).  Tiles in id (= BFS row) order;
// a multi-rank plan keeps only its own tile range [t_begin, t_end).
struct TiledHost {
  std::vector<char> slot_first;  // K8: spill slot's tile is the target's first writer
  std::vector<TileDesc> desc;
  std::vector<unsigned char> blocks;
  std::vector<int32_t> slot_tgt, slots, in_ptr;
  std::vector<SpillRun> runs;
  int64_t nsp = 0;
  int32_t block_cap = 0, window_cap = 0, nnz_cap = 0;
};

int build_tiled_host(const Schedule& S, int32_t t_begin, int32_t t_end, TiledHost& H) {
  const int32_t nt = (int32_t)S.tile_group.size();
  const int32_t n = S.n;
  std::vector<int32_t> tile_of((size_t)n);
  for (int32_t t = 0; t < nt; ++t)
    for (int32_t r = S.tile_ptr[(size_t)t]; r < S.tile_ptr[(size_t)t + 1]; ++r) tile_of[(size_t)r] = t;
  std::vector<TileDesc> desc((size_t)nt);
  std::vector<int64_t> boff((size_t)nt + 1, 0);
  // spill windows laid out run by run: a run of consecutive target rows g..
  // starts on a window id w with w == g - row0 (mod 2), so that with the
  // window shifted like the own rows (slot parity == row parity) a run can
  // be bulk-copied from x; a pad slot (target -1) fixes the parity
  std::vector<int64_t> slot_ptr((size_t)nt + 1, 0), run_ptr((size_t)nt + 1, 0);
  // runs averaging >= 6 targets are bulk-copied by the gather warps (measured:
  // st27, spin, lap3d); shorter runs (kNN) are gathered slot by slot and need
  // no parity pads
  std::vector<char> use_runs((size_t)nt, 0);
  for (int32_t t = 0; t < nt; ++t) {
    int64_t nr = 0;
    int32_t prev = -2;
    for (int64_t q = S.spill_ptr[(size_t)t]; q < S.spill_ptr[(size_t)t + 1]; ++q) {
      const int32_t g = (int32_t)((uint32_t)S.spill[(size_t)q] & kIdxMask);
      nr += (g != prev + 1);
      prev = g;
    }
    use_runs[(size_t)t] = nr > 0 && (S.spill_ptr[(size_t)t + 1] - S.spill_ptr[(size_t)t]) >= 6 * nr;
  }
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t r0 = S.tile_ptr[(size_t)t], T = S.tile_ptr[(size_t)t + 1] - r0;
    int64_t w = 0, nr = 0;
    int32_t prev = -2;
    for (int64_t q = S.spill_ptr[(size_t)t]; q < S.spill_ptr[(size_t)t + 1]; ++q) {
      const int32_t g = (int32_t)((uint32_t)S.spill[(size_t)q] & kIdxMask);
      if (g != prev + 1) {
        ++nr;
        if (use_runs[(size_t)t] && ((T + w - (g - r0)) & 1) != 0) ++w;  // window id T + w == g - row0 (mod 2)
      }
      ++w;
      prev = g;
    }
    slot_ptr[(size_t)t + 1] = slot_ptr[(size_t)t] + w;
    run_ptr[(size_t)t + 1] = run_ptr[(size_t)t] + nr;
  }
  // single-run tiles carry no tgt[] in their block (TileDesc.gather_runs bit 1)
  const bool single_on = !std::getenv("SYMM_SINGLE_RUN") || std::atoi(std::getenv("SYMM_SINGLE_RUN")) != 0;
  std::vector<char> single_run((size_t)nt, 0);
  for (int32_t t = 0; t < nt; ++t)
    single_run[(size_t)t] = single_on && use_runs[(size_t)t] && run_ptr[(size_t)t + 1] - run_ptr[(size_t)t] == 1;
  std::vector<int32_t> slot_tgt((size_t)slot_ptr[(size_t)nt], -1);
  std::vector<char> slot_first((size_t)slot_ptr[(size_t)nt], 0);  // this tile writes the target first (lowest phase)

  std::vector<SpillRun> runs((size_t)run_ptr[(size_t)nt]);
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t r0 = S.tile_ptr[(size_t)t], T = S.tile_ptr[(size_t)t + 1] - r0;
    int64_t w = 0, nr = run_ptr[(size_t)t];
    int32_t prev = -2;
    for (int64_t q = S.spill_ptr[(size_t)t]; q < S.spill_ptr[(size_t)t + 1]; ++q) {
      const int32_t g = (int32_t)((uint32_t)S.spill[(size_t)q] & kIdxMask);
      if (g != prev + 1) {
        if (use_runs[(size_t)t] && ((T + w - (g - r0)) & 1) != 0) ++w;
        runs[(size_t)nr++] = SpillRun{g, T + (int32_t)w, 0, 0};
      }
      runs[(size_t)nr - 1].len++;
      slot_tgt[(size_t)(slot_ptr[(size_t)t] + w)] = g;
      ++w;
      prev = g;
    }
  }
  // K8 (tiled_colored): the first writer of a row (the writer tile of the
  // lowest phase, schedule.cpp) stores, the others add after it in phase order
  for (int32_t t = 0; t < nt; ++t) {
    int64_t w = slot_ptr[(size_t)t];
    for (int64_t q = S.spill_ptr[(size_t)t]; q < S.spill_ptr[(size_t)t + 1]; ++q) {
      const int32_t g = (int32_t)((uint32_t)S.spill[(size_t)q] & kIdxMask);
      while (slot_tgt[(size_t)w] != g) ++w;  // pads (-1) between runs
      slot_first[(size_t)w] = ((uint32_t)S.spill[(size_t)q] & kFirstBit) != 0;
      ++w;
    }
  }
  // Per tile: lane positions in slot order, or sorted by descending work
  // (row entries + transposed entries of the slot).  The kernel walks each
  // lane's list (row part, then transposed part) in lock step with its warp
  // (32 consecutive positions), so a warp costs its longest list; sorting is
  // used when it saves at least `gain` of those lock steps (own-row REDs lose
  // their coalescing, so a small saving is not worth it).
  double gain = 0.25;
  if (const char* v = std::getenv("SYMM_SORT_GAIN")) gain = std::atof(v);
  std::vector<char> sort_tile((size_t)nt, 0);
  const bool place_peel = !std::getenv("SYMM_PLACE_PEEL") || std::atoi(std::getenv("SYMM_PLACE_PEEL")) != 0;
  // sorted tiles' record loop: blocks of 4 first, leftovers last (measured:
  // SYMM_PEEL_SORTED=1, the leftovers-first model, is slower)
  const bool peel_sorted = std::getenv("SYMM_PEEL_SORTED") && std::atoi(std::getenv("SYMM_PEEL_SORTED")) != 0;
  std::vector<int64_t> lane_off((size_t)nt + 1, 0);
  for (int32_t t = 0; t < nt; ++t)
    lane_off[(size_t)t + 1] = lane_off[(size_t)t] + (S.tile_ptr[(size_t)t + 1] - S.tile_ptr[(size_t)t]) +
                              (slot_ptr[(size_t)t + 1] - slot_ptr[(size_t)t]);
  std::vector<int32_t> lane_slot((size_t)lane_off[(size_t)nt]), vstart((size_t)n, 0), tile_pads((size_t)nt, 0);
  // sorted tiles: one list of records (val index | x index) per lane position,
  // at rec[lane_pst[i]], placed so that a warp's lock-step record loads hit
  // distinct banks
  std::vector<int32_t> lane_pst((size_t)lane_off[(size_t)nt], 0), rec_pads((size_t)nt, 0);
  auto plan_tile = [&](int32_t t, bool allow_sort) {
    const int32_t r0 = S.tile_ptr[(size_t)t], r1 = S.tile_ptr[(size_t)t + 1], T = r1 - r0;
    const int32_t W = T + (int32_t)(slot_ptr[(size_t)t + 1] - slot_ptr[(size_t)t]);
    std::vector<int32_t> work((size_t)W, 0);
    for (int32_t r = r0; r < r1; ++r)
      for (int32_t i = S.prow_ptr[(size_t)r]; i < S.prow_ptr[(size_t)r + 1]; ++i) {
        const int32_t c = S.pcol[(size_t)i];
        work[(size_t)(r - r0)] += 1;
        if (c == r) continue;
        const int32_t lc = run_local(runs.data() + run_ptr[(size_t)t], (int32_t)(run_ptr[(size_t)t + 1] - run_ptr[(size_t)t]), r0, r1, c);
        if (lc >= 0 && lc < W) work[(size_t)lc] += 1;
      }
    auto steps = [&](const std::vector<int32_t>& w) {
      int64_t s = 0;
      for (int32_t g = 0; g < W; g += 32) s += *std::max_element(w.begin() + g, w.begin() + std::min(W, g + 32));
      return s;
    };
    std::vector<int32_t> ws(work);
    std::sort(ws.begin(), ws.end(), std::greater<int32_t>());
    sort_tile[(size_t)t] = allow_sort && W > 32 && (double)steps(ws) <= (1.0 - gain) * (double)steps(work);
    // lane position -> window slot
    int32_t* sa = lane_slot.data() + lane_off[(size_t)t];
    for (int32_t i = 0; i < W; ++i) sa[i] = i;
    if (sort_tile[(size_t)t])
      std::stable_sort(sa, sa + W, [&](int32_t a, int32_t b) { return work[(size_t)a] > work[(size_t)b]; });
    // row segments of the 32 lanes of a warp placed so that within each half
    // warp the segment starts are distinct mod 16: the lanes' lock-step val
    // loads then hit distinct bank pairs (pad entries where no row fits)
    int32_t cur = 0, pads = 0;
    // nvcc's unroll-by-4 of the row loop runs a row's len % 4 leftover steps
    // first, so a lane's unrolled steps start at entry start + len % 4
    // (SYMM_PLACE_PEEL=0: plain starts)
    auto peel = [&](int32_t len) { return place_peel ? (len & (kK4Unroll - 1)) : 0; };
    for (int32_t g0 = 0; g0 < W; g0 += 32) {
      std::vector<int32_t> rem;  // lanes of this warp with a row segment
      for (int32_t i = g0; i < std::min(W, g0 + 32); ++i)
        if (sa[i] < T) rem.push_back(i);
      uint32_t used[2] = {0, 0};
      int nrem[2] = {0, 0};
      for (int32_t i : rem) nrem[(i - g0) >> 4]++;
      while (!rem.empty()) {
        int best = -1, bsc = -1, bkey = 0;
        for (size_t q = 0; q < rem.size(); ++q) {
          const int h = (rem[q] - g0) >> 4;
          const int32_t len = S.prow_ptr[(size_t)(r0 + sa[rem[q]]) + 1] - S.prow_ptr[(size_t)(r0 + sa[rem[q]])];
          // sorted tiles unroll one list of row + transposed entries per lane
          const int32_t key = (cur + (sort_tile[(size_t)t] ? (peel_sorted ? peel(work[(size_t)sa[rem[q]]]) : 0) : peel(len))) & 15;
          if ((used[h] >> key) & 1) continue;
          const int32_t er = (cur + len) & 15;
          int sc = 0;  // halves that can still use the residue this row ends on
          for (int h2 = 0; h2 < 2; ++h2)
            if (nrem[h2] - (h2 == h) > 0 && !((used[h2] | (h2 == h ? 1u << key : 0u)) >> er & 1)) ++sc;
          if (sc > bsc) { bsc = sc; best = (int)q; bkey = key; }
        }
        if (best < 0) { ++cur; ++pads; continue; }  // no row can start here: pad entry
        const int32_t i = rem[(size_t)best];
        const int h = (i - g0) >> 4;
        const int32_t row = r0 + sa[i];
        vstart[(size_t)row] = cur;
        cur += S.prow_ptr[(size_t)row + 1] - S.prow_ptr[(size_t)row];
        used[h] |= 1u << bkey;
        nrem[h]--;
        rem.erase(rem.begin() + best);
      }
    }
    tile_pads[(size_t)t] = pads;
    rec_pads[(size_t)t] = 0;
    if (sort_tile[(size_t)t]) {
      // record lists: keys (start + leftover steps) distinct mod 32 in a warp
      int32_t rcur = 0, rp = 0;
      int32_t* pst = lane_pst.data() + lane_off[(size_t)t];
      for (int32_t g0 = 0; g0 < W; g0 += 32) {
        std::vector<int32_t> rem;
        for (int32_t i = g0; i < std::min(W, g0 + 32); ++i) rem.push_back(i);
        uint32_t used = 0;
        while (!rem.empty()) {
          int best = -1;
          for (size_t q = 0; q < rem.size(); ++q) {
            const int32_t nq = work[(size_t)sa[rem[q]]];
            const int32_t key = (rcur + (peel_sorted ? (nq & 3) : 0)) & 31;
            if (nq == 0 || !((used >> key) & 1)) { best = (int)q; break; }
          }
          if (best < 0) { ++rcur; ++rp; continue; }
          const int32_t i = rem[(size_t)best];
          const int32_t nq = work[(size_t)sa[i]];
          if (nq > 0) used |= 1u << ((rcur + (peel_sorted ? (nq & 3) : 0)) & 31);
          pst[i] = rcur;
          rcur += nq;
          rem.erase(rem.begin() + best);
        }
      }
      rec_pads[(size_t)t] = rp;
    }
  };
#pragma omp parallel for schedule(dynamic, 64)
  for (int32_t t = 0; t < nt; ++t) plan_tile(t, true);
  // the ring depth follows the largest block: pad entries must not grow it.
  // A tile whose padded block would exceed the largest unpadded block keeps
  // its segments contiguous (no pads; bank-pair starts not guaranteed).
  // block layout of tile t (capi.cpp / internal.h TileDesc); sorted tiles
  // carry record lists (pseg u32[W] + rec u32) instead of lcol / tcsc / tptr
  struct Layout { int64_t o_lcol, o_tidx, o_tptr, o_sid, o_tgt, o_val, bytes, nnz, nrec; };
  auto layout = [&](int32_t t, bool srt, int64_t pads, int64_t rpads) -> Layout {
    const int32_t r0 = S.tile_ptr[(size_t)t], r1 = S.tile_ptr[(size_t)t + 1], T = r1 - r0;
    const int64_t S_ = slot_ptr[(size_t)t + 1] - slot_ptr[(size_t)t], W = T + S_;
    const int64_t nnz0 = S.prow_ptr[(size_t)r1] - S.prow_ptr[(size_t)r0];
    int64_t nd = 0;
    for (int32_t r = r0; r < r1; ++r) nd += (S.prow_ptr[(size_t)r + 1] > S.prow_ptr[(size_t)r] && S.pcol[(size_t)S.prow_ptr[(size_t)r]] == r);
    Layout L{};
    L.nnz = nnz0 + pads;
    const int64_t o0 = align16((int64_t)sizeof(TileDesc) + 4 * (int64_t)T);  // rseg u32[T]
    if (!srt) {
      L.o_lcol = o0;
      L.o_tidx = align16(L.o_lcol + 2 * L.nnz);
      L.o_tptr = align16(L.o_tidx + 4 * (nnz0 - nd));
      L.o_sid = align16(L.o_tptr + 2 * (W + 1));
      L.o_tgt = L.o_sid;
    } else {
      L.nrec = nnz0 + (nnz0 - nd) + rpads;
      L.o_lcol = o0;                                  // pseg u32[W]: record list of each position
      L.o_tidx = align16(L.o_lcol + 4 * W);           // rec u32[nrec]: val index | x index << 16
      L.o_tptr = 0;
      L.o_sid = align16(L.o_tidx + 4 * L.nrec);
      L.o_tgt = align16(L.o_sid + 2 * W);
    }
    L.o_val = align16(L.o_tgt + (single_run[(size_t)t] ? 0 : 4 * S_));
    L.bytes = align16(L.o_val + 8 * L.nnz);
    return L;
  };
  {
    // pads must not grow the largest block (the ring depth follows it): a
    // sorted tile whose record format would exceed the largest unpadded
    // unsorted block is planned unsorted; a padded tile that would exceed it
    // keeps its row segments contiguous (no pads)
    int64_t cap0 = 0, maxw = 0;
    for (int32_t t = 0; t < nt; ++t) {
      cap0 = std::max(cap0, layout(t, false, 0, 0).bytes);
      maxw = std::max<int64_t>(maxw, (S.tile_ptr[(size_t)t + 1] - S.tile_ptr[(size_t)t]) + (slot_ptr[(size_t)t + 1] - slot_ptr[(size_t)t]));
    }
    // room left under the 6-stage ring (schedule.cpp kRingBytes / kRingStages)
    const int64_t ring_cap = (232448 - 1024 - 512) / 6 - 8 * (((maxw + 2 + 15) / 16) * 16) - 128;
    if (!std::getenv("SYMM_NO_RING_CAP")) cap0 = std::max(cap0, (ring_cap / 128) * 128);
    for (int32_t t = 0; t < nt; ++t)
      if (sort_tile[(size_t)t] && layout(t, true, tile_pads[(size_t)t], rec_pads[(size_t)t]).bytes > cap0) plan_tile(t, false);
    for (int32_t t = 0; t < nt; ++t)
      if (tile_pads[(size_t)t] > 0 &&
          (layout(t, sort_tile[(size_t)t], tile_pads[(size_t)t], rec_pads[(size_t)t]).bytes > cap0 || std::getenv("SYMM_NO_PLACE"))) {
        const int32_t r0 = S.tile_ptr[(size_t)t], r1 = S.tile_ptr[(size_t)t + 1];
        for (int32_t r = r0; r < r1; ++r) vstart[(size_t)r] = S.prow_ptr[(size_t)r] - S.prow_ptr[(size_t)r0];
        tile_pads[(size_t)t] = 0;
      }
  }
  int32_t block_cap = 16, window_cap = 2, nnz_cap = 2;
  int bad = 0;
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t r0 = S.tile_ptr[(size_t)t], r1 = S.tile_ptr[(size_t)t + 1], T = r1 - r0;
    const int32_t S_ = (int32_t)(slot_ptr[(size_t)t + 1] - slot_ptr[(size_t)t]);
    const int srt = sort_tile[(size_t)t];
    const Layout L = layout(t, srt != 0, tile_pads[(size_t)t], rec_pads[(size_t)t]);
    const int64_t nnz = L.nnz, W = (int64_t)T + S_, bytes = L.bytes;
    const int64_t o_lcol = L.o_lcol, o_tidx = L.o_tidx, o_tptr = L.o_tptr, o_sid = L.o_sid, o_tgt = L.o_tgt,
                  o_val = L.o_val;
    if (nnz >= 65536 || L.nrec >= 65536 || W >= 32767 || bytes >= 65536) { bad = t + 1; break; }
    TileDesc& D = desc[(size_t)t];
    std::memset(&D, 0, sizeof D);
    D.block_bytes = (int32_t)bytes;
    D.nrows = T;
    D.nspill = S_;
    D.nnz = (int32_t)nnz;
    D.row0 = r0;
    D.o_lcol = (uint16_t)o_lcol;
    D.o_tidx = (uint16_t)o_tidx;
    D.o_tptr = (uint16_t)o_tptr;
    D.o_tgt = (uint16_t)o_tgt;
    D.o_sid = (uint16_t)o_sid;
    D.sorted = srt;
    D.o_val = (uint16_t)o_val;
    D.spill_off = (int32_t)slot_ptr[(size_t)t];
    D.run_off = (int32_t)run_ptr[(size_t)t];
    D.nruns = (int32_t)(run_ptr[(size_t)t + 1] - run_ptr[(size_t)t]);
    D.gather_runs = use_runs[(size_t)t];
    if (single_run[(size_t)t]) {
      const SpillRun& R = runs[(size_t)run_ptr[(size_t)t]];
      D.gather_runs |= 2 | (R.wid > T ? 4 : 0);  // (at most one parity pad slot before the run)
      D.tgt_base = R.row - R.wid;
      if (R.wid - T > 1 || R.wid - T + R.len != S_) { bad = t + 1; break; }
    }
    boff[(size_t)t + 1] = boff[(size_t)t] + bytes;
    D.block_off = boff[(size_t)t];
    block_cap = std::max<int32_t>(block_cap, (int32_t)bytes);
    window_cap = std::max<int32_t>(window_cap, (int32_t)W);
    nnz_cap = std::max<int32_t>(nnz_cap, (int32_t)nnz);
  }
  if (bad)
    return set_error(SYMM_ERR_UNSUPPORTED, "tile %d does not fit the 64 KB tile-block format (use smaller tiles)", bad - 1);
  window_cap = (window_cap + 2 + 15) & ~15;  // +2: x window alignment shift; stages stay 128-B aligned
  block_cap = (block_cap + 127) & ~127;
  // staged contributions (K3): one staging slot per (writer tile, target);
  // slot order = (owner row, writer tile) -> contiguous per row
  const int64_t nsl = slot_ptr[(size_t)nt];
  std::vector<int32_t> in_ptr((size_t)n + 1, 0), slots((size_t)nsl, -1);
  for (int64_t q = 0; q < nsl; ++q)
    if (slot_tgt[(size_t)q] >= 0) in_ptr[(size_t)slot_tgt[(size_t)q] + 1]++;
  for (int32_t r = 0; r < n; ++r) in_ptr[(size_t)r + 1] += in_ptr[(size_t)r];
  const int64_t nsp = in_ptr[(size_t)n];
  {
    std::vector<int32_t> pos(in_ptr.begin(), in_ptr.end() - 1);
    for (int64_t q = 0; q < nsl; ++q)  // ascending writer tile, then ascending target
      if (slot_tgt[(size_t)q] >= 0) slots[(size_t)q] = pos[(size_t)slot_tgt[(size_t)q]]++;
  }
  std::vector<unsigned char> blocks((size_t)boff[(size_t)nt], 0);
#pragma omp parallel for schedule(dynamic, 8) reduction(| : bad)
  for (int32_t t = 0; t < nt; ++t) {
    const TileDesc& D = desc[(size_t)t];
    const int32_t r0 = D.row0, T = D.nrows, r1 = r0 + T, ns = D.nspill, W = T + ns;
    unsigned char* blk = blocks.data() + D.block_off;
    std::memcpy(blk, &D, sizeof(TileDesc));  // the descriptor travels with its block
    uint32_t* rseg = reinterpret_cast<uint32_t*>(blk + sizeof(TileDesc));
    // sorted tiles keep the local columns host side (their records carry them)
    std::vector<uint16_t> lcol_host(D.sorted ? (size_t)D.nnz : 0);
    uint16_t* lcol = D.sorted ? lcol_host.data() : reinterpret_cast<uint16_t*>(blk + D.o_lcol);
    uint32_t* tcsc = reinterpret_cast<uint32_t*>(blk + D.o_tidx);  // sorted: the record lists
    uint16_t* tptr = reinterpret_cast<uint16_t*>(blk + D.o_tptr);
    int32_t* tgt = reinterpret_cast<int32_t*>(blk + D.o_tgt);
    double* val = reinterpret_cast<double*>(blk + D.o_val);
    const int32_t* st = slot_tgt.data() + slot_ptr[(size_t)t];
    // flush target of every spill slot (-1 = pad)
    if (!(D.gather_runs & 2))
      for (int32_t j = 0; j < ns; ++j) tgt[j] = st[j];
    const int32_t e0 = S.prow_ptr[(size_t)r0];
    const SpillRun* tr = runs.data() + run_ptr[(size_t)t];
    const int32_t nrt = (int32_t)(run_ptr[(size_t)t + 1] - run_ptr[(size_t)t]);
    const bool bank_aware = !std::getenv("SYMM_NO_BANK_ORDER");
    const int csc_passes = std::getenv("SYMM_CSC_PASSES") ? std::max(1, std::atoi(std::getenv("SYMM_CSC_PASSES"))) : 8;
    // window id of every entry's column; list lengths of every slot
    const int32_t nnz = D.nnz;
    std::vector<int32_t> eloc((size_t)nnz);
    std::vector<int32_t> rl((size_t)W, 0), cl((size_t)W, 0);
    for (int32_t r = r0; r < r1; ++r) {
      rl[(size_t)(r - r0)] = S.prow_ptr[(size_t)r + 1] - S.prow_ptr[(size_t)r];
      for (int32_t i = S.prow_ptr[(size_t)r]; i < S.prow_ptr[(size_t)r + 1]; ++i) {
        const int32_t lc = run_local(tr, nrt, r0, r1, S.pcol[(size_t)i]);
        if (lc < 0) { bad |= 1; continue; }
        eloc[(size_t)(i - e0)] = lc;
        if (S.pcol[(size_t)i] != r) cl[(size_t)lc]++;
      }
    }
    // lane position -> window slot (decided with the segment placement)
    std::vector<int32_t> slot_at(lane_slot.begin() + lane_off[(size_t)t], lane_slot.begin() + lane_off[(size_t)t + 1]);
    // own row l's segment: entries [rst[l], rst[l] + rl[l]) of lcol / val
    std::vector<int32_t> rst((size_t)std::max(T, 1), 0);
    for (int32_t l = 0; l < T; ++l) {
      rst[(size_t)l] = vstart[(size_t)(r0 + l)];
      rseg[l] = (uint32_t)rst[(size_t)l] | ((uint32_t)rl[(size_t)l] << 16);
    }
    if (D.sorted) {
      uint16_t* sid = reinterpret_cast<uint16_t*>(blk + D.o_sid);
      for (int32_t i = 0; i < W; ++i) sid[i] = (uint16_t)slot_at[(size_t)i];
    }
    const bool uni = D.sorted != 0;  // sorted tiles: one list (row part, then transposed part) per lane
    // row part: a warp walks the lists of 32 consecutive lane positions in
    // lock step; order every row's entries so that at each step the x
    // gathers of a half warp hit distinct bank pairs (window id mod 16)
    std::vector<std::vector<std::pair<uint16_t, double>>> ent;
    for (int32_t g0 = 0; g0 < W; g0 += 32) {
      const int32_t g1 = std::min(W, g0 + 32);
      ent.assign((size_t)(g1 - g0), {});
      for (int32_t i = g0; i < g1; ++i) {
        const int32_t l = slot_at[(size_t)i];
        if (l >= T) continue;
        for (int32_t k = S.prow_ptr[(size_t)(r0 + l)]; k < S.prow_ptr[(size_t)(r0 + l) + 1]; ++k)
          ent[(size_t)(i - g0)].push_back({(uint16_t)eloc[(size_t)(k - e0)], S.pval[(size_t)k]});
      }
      if (bank_aware) {
        bank_order_rows(ent, 1);
        // the unrolled loop runs a lane's n % 4 leftover steps first (n = its
        // loop length): the matched order is for the steps after them, so the
        // entries matched last become the leftover (first) entries
        for (int32_t i = g0; i < g1; ++i) {
          const int32_t l = slot_at[(size_t)i];
          if (l >= T || !place_peel) continue;
          auto& e = ent[(size_t)(i - g0)];
          const int32_t off = uni && !peel_sorted ? 0 : std::min<int32_t>((int32_t)e.size(), (uni ? rl[(size_t)l] + cl[(size_t)l] : rl[(size_t)l]) & (uni ? 3 : kK4Unroll - 1));
          std::rotate(e.begin(), e.end() - off, e.end());
        }
      }
      for (int32_t i = g0; i < g1; ++i) {
        const int32_t l = slot_at[(size_t)i];
        if (l >= T) continue;
        const auto& e = ent[(size_t)(i - g0)];
        const int32_t b = rst[(size_t)l];
        for (size_t k = 0; k < e.size(); ++k) {
          lcol[b + (int32_t)k] = e[k].first;
          val[b + (int32_t)k] = e[k].second;
        }
      }
    }
    // transposed part: slot l's list of (entry, local row), walked after the
    // row part in the same lock step; at each step the lanes of a half warp
    // should read val[entry] and xs[row] from bank pairs not used by the
    // other lanes (including those still in their row part)
    std::vector<std::vector<uint32_t>> lists((size_t)W);
    for (int32_t l = 0; l < T; ++l)
      for (int32_t k = rst[(size_t)l]; k < rst[(size_t)l] + rl[(size_t)l]; ++k)
        if (lcol[k] != l) lists[lcol[k]].push_back((uint32_t)k | ((uint32_t)l << 16));
    const int32_t vb = (int32_t)(D.o_val / 8);  // bank-pair phase of val[0]
    // sorted tiles walk one list per lane (row part, then transposed part) in
    // lock step; unsorted tiles walk the two parts as separate lock-step loops
    // Sorted tiles carry explicit (val index | x index) records, so a lane's
    // row records need not come first.  Opt-in (SYMM_REC_FREE=1 or
    // SYMM_VAL_COLOR=1): they join the lane's list and the bank-aware pick
    // below orders all of a lane's records.  Measured on fem_knn_4M (B200,
    // profiles/r2/i/ab_val_color.txt): the model's val / x conflict factors
    // drop from 1.79 / 1.82 to 1.60 / 1.70 with the colouring, the time stays
    // at 0.196-0.201 ms either way, so the default keeps row records first.
    const bool rec_free = uni && ((std::getenv("SYMM_REC_FREE") && std::atoi(std::getenv("SYMM_REC_FREE")) != 0) ||
                                  (std::getenv("SYMM_VAL_COLOR") && std::atoi(std::getenv("SYMM_VAL_COLOR")) != 0));
    if (rec_free)
      for (int32_t l = 0; l < T; ++l) {
        std::vector<uint32_t> all;
        for (int32_t k = rst[(size_t)l]; k < rst[(size_t)l] + rl[(size_t)l]; ++k) all.push_back((uint32_t)k | ((uint32_t)lcol[k] << 16));
        all.insert(all.end(), lists[(size_t)l].begin(), lists[(size_t)l].end());
        lists[(size_t)l].swap(all);
      }
    auto rlen = [&](int32_t l) { return (uni && !rec_free && l < T) ? rl[(size_t)l] : 0; };
    // SYMM_VAL_COLOR=1 (sorted tiles): the record order is chosen for the x
    // gathers alone, and the val array is then permuted so that the entries a
    // half warp reads in one lock step sit in distinct bank pairs (below)
    const bool val_color = rec_free && bank_aware && std::getenv("SYMM_VAL_COLOR") && std::atoi(std::getenv("SYMM_VAL_COLOR")) != 0;
    const int vw = val_color ? 0 : 1;  // weight of the val banks in the pick
    if (bank_aware)
      for (int32_t g0 = 0; g0 < W; g0 += 32) {
        const int32_t g1 = std::min(W, g0 + 32);
        // execution steps of the warp's unrolled loop: first the lanes' n % 4
        // leftover steps (P = the largest), then the blocks of 4 in lock step;
        // lane i is at list index idx(tau) (n = its loop length)
        // (sorted tiles' unified loop: blocks of 4 first, then the leftover
        // steps of every lane together: lane i at 4 (n_i / 4) + t)
        int32_t nn[32], off[32], P = 0, tmax = 0, B4 = 0;
        const bool rem_last = uni && !peel_sorted && place_peel;
        for (int32_t i = g0; i < g1; ++i) {
          const int32_t l = slot_at[(size_t)i];
          nn[i - g0] = rlen(l) + (int32_t)lists[(size_t)l].size();
          off[i - g0] = place_peel && (!uni || peel_sorted) ? (nn[i - g0] & (uni ? 3 : kK4Unroll - 1)) : 0;
          P = std::max(P, off[i - g0]);
          B4 = std::max(B4, nn[i - g0] & ~(kK4SortedUnroll - 1));
        }
        for (int32_t i = g0; i < g1; ++i)
          tmax = std::max(tmax, rem_last ? B4 + (nn[i - g0] & (kK4SortedUnroll - 1)) : P + nn[i - g0] - off[i - g0]);
        auto idx_at = [&](int32_t i, int32_t tau) -> int32_t {
          const int32_t n = nn[i - g0];
          if (rem_last) {
            if (tau < B4) return tau < (n & ~(kK4SortedUnroll - 1)) ? tau : -1;
            const int32_t t = tau - B4;
            return t < (n & (kK4SortedUnroll - 1)) ? (n & ~(kK4SortedUnroll - 1)) + t : -1;
          }
          const int32_t v = tau < P ? (tau < off[i - g0] ? tau : -1) : off[i - g0] + (tau - P);
          return v < n ? v : -1;
        };
        for (int32_t tau = 0; tau < tmax; ++tau)
          for (int32_t h = g0; h < g1; h += 16) {
            const int32_t h1 = std::min(g1, h + 16);
            // bank-pair load counts of this (step, half warp): lanes still in
            // their row part are fixed; each lane in its transposed part picks
            // one of its remaining entries.  Several greedy passes (lane orders)
            // minimise max val load + max x load (= wavefronts of the 2 loads).
            int cv0[16] = {0}, cr0[16] = {0};
            int act[16], actj[16], na = 0;
            for (int32_t i = h; i < h1; ++i) {
              const int32_t l = slot_at[(size_t)i];
              const int32_t v = idx_at(i, tau);
              if (v < 0) continue;
              if (v < rlen(l)) {
                const int32_t k = rst[(size_t)l] + v;
                cv0[(k + vb) & 15]++;
                cr0[lcol[k] & 15]++;
              } else {
                act[na] = i;
                actj[na++] = v - rlen(l);
              }
            }
            if (na == 0) continue;
            int best_cost = INT32_MAX;
            size_t best_pick[16], pick[16];
            uint32_t rs = 0x9e3779b9u ^ (uint32_t)(tau * 131 + h);
            for (int pass = 0; pass < csc_passes; ++pass) {
              int ord[16];
              for (int q = 0; q < na; ++q) ord[q] = q;
              if (pass > 0)
                for (int q = na - 1; q > 0; --q) {  // deterministic shuffle
                  rs = rs * 1664525u + 1013904223u;
                  std::swap(ord[q], ord[(int)((rs >> 8) % (uint32_t)(q + 1))]);
                }
              int cv[16], cr[16];
              std::copy(cv0, cv0 + 16, cv);
              std::copy(cr0, cr0 + 16, cr);
              for (int q = 0; q < na; ++q) {
                const int32_t l = slot_at[(size_t)act[ord[q]]];
                const auto& L = lists[(size_t)l];
                const size_t jj = (size_t)actj[ord[q]];
                size_t bq = jj;
                int bsc = INT32_MAX;
                for (size_t e = jj; e < L.size(); ++e) {
                  const int sc = 4 * (vw * cv[((L[e] & 0xffffu) + vb) & 15] + cr[(L[e] >> 16) & 15]) +
                                 vw * (cv[((L[e] & 0xffffu) + vb) & 15] > 0) + (cr[(L[e] >> 16) & 15] > 0);
                  if (sc < bsc) { bsc = sc; bq = e; if (sc == 0) break; }
                }
                pick[ord[q]] = bq;
                cv[((L[bq] & 0xffffu) + vb) & 15]++;
                cr[(L[bq] >> 16) & 15]++;
              }
              const int cost = vw * *std::max_element(cv, cv + 16) + *std::max_element(cr, cr + 16);
              if (cost < best_cost) {
                best_cost = cost;
                std::copy(pick, pick + na, best_pick);
              }
            }
            for (int q = 0; q < na; ++q) {
              auto& L = lists[(size_t)slot_at[(size_t)act[q]]];
              std::swap(L[(size_t)actj[q]], L[best_pick[q]]);
            }
          }
      }
    if (val_color) {
      // Every stored entry is read by two records (its row's lane and its
      // column's lane; the diagonal by one), i.e. in at most two (half warp,
      // lock step) groups.  Entries are given one of the 16 bank pairs
      // greedily -- the pair least used in their two groups, among the pairs
      // that still have free positions -- and val is permuted accordingly.
      const bool rem_last = !peel_sorted && place_peel;
      int32_t TM = 2;
      for (int32_t i = 0; i < W; ++i) TM = std::max<int32_t>(TM, (int32_t)lists[(size_t)slot_at[(size_t)i]].size() + 2);
      const int32_t nhalf = (W + 15) / 16;
      std::vector<uint8_t> cnt((size_t)nhalf * (size_t)TM * 16, 0);
      std::vector<int32_t> grp((size_t)nnz * 2, -1);
      for (int32_t g0 = 0; g0 < W; g0 += 32) {
        const int32_t g1 = std::min(W, g0 + 32);
        int32_t B = 0;
        for (int32_t i = g0; i < g1; ++i)
          B = std::max<int32_t>(B, (int32_t)lists[(size_t)slot_at[(size_t)i]].size() & ~(kK4SortedUnroll - 1));
        for (int32_t i = g0; i < g1; ++i) {
          const auto& L = lists[(size_t)slot_at[(size_t)i]];
          const int32_t n = (int32_t)L.size(), nb = n & ~(kK4SortedUnroll - 1);
          for (int32_t v = 0; v < n; ++v) {
            const int32_t tau = (rem_last && v >= nb) ? B + (v - nb) : v;
            const int32_t e = (int32_t)(L[(size_t)v] & 0xffffu);
            grp[(size_t)e * 2 + (grp[(size_t)e * 2] >= 0 ? 1 : 0)] = (i / 16) * TM + tau;
          }
        }
      }
      int32_t cap[16] = {0}, used[16] = {0};
      for (int32_t p2 = 0; p2 < nnz; ++p2) cap[(p2 + vb) & 15]++;
      std::vector<int32_t> newpos((size_t)nnz, -1);
      for (int32_t e = 0; e < nnz; ++e) {
        const int32_t a = grp[(size_t)e * 2], b2 = grp[(size_t)e * 2 + 1];
        if (a < 0) continue;  // pad entry: read by nobody
        int best = -1, bsc = INT32_MAX;
        for (int c = 0; c < 16; ++c) {
          if (used[c] >= cap[c]) continue;
          const int sc = 64 * ((int)cnt[(size_t)a * 16 + c] + (b2 >= 0 ? (int)cnt[(size_t)b2 * 16 + c] : 0)) - std::min(63, cap[c] - used[c]);
          if (sc < bsc) { bsc = sc; best = c; }
        }
        cnt[(size_t)a * 16 + best]++;
        if (b2 >= 0) cnt[(size_t)b2 * 16 + best]++;
        newpos[(size_t)e] = ((best - vb) & 15) + 16 * used[best]++;
      }
      std::vector<double> nv((size_t)nnz, 0.0);
      for (int32_t e = 0; e < nnz; ++e)
        if (newpos[(size_t)e] >= 0) nv[(size_t)newpos[(size_t)e]] = val[e];
      std::copy(nv.begin(), nv.end(), val);
      for (int32_t l = 0; l < W; ++l)
        for (uint32_t& q : lists[(size_t)l]) q = (q & 0xffff0000u) | (uint32_t)newpos[(size_t)(q & 0xffffu)];
      for (int32_t l = 0; l < T; ++l) rseg[l] = 0;  // (sorted tiles never read rseg; val is no longer in row order)
    }
    if (!D.sorted) {
      int32_t pos = 0;
      for (int32_t i = 0; i < W; ++i) {
        tptr[i] = (uint16_t)pos;
        for (uint32_t q : lists[(size_t)slot_at[(size_t)i]]) tcsc[pos++] = q;
      }
      tptr[W] = (uint16_t)pos;
    } else {
      // one record list per lane position: row part (val index | local
      // column << 16), then transposed part (entry | local row << 16)
      uint32_t* pseg = reinterpret_cast<uint32_t*>(blk + D.o_lcol);
      const int32_t* pst = lane_pst.data() + lane_off[(size_t)t];
      for (int32_t i = 0; i < W; ++i) {
        const int32_t l = slot_at[(size_t)i];
        int32_t q = pst[i];
        const int32_t nrow = (l < T && !rec_free) ? rl[(size_t)l] : 0;
        for (int32_t k = 0; k < nrow; ++k) {
          const int32_t e = rst[(size_t)l] + k;
          tcsc[q++] = (uint32_t)e | ((uint32_t)lcol[e] << 16);
        }
        for (uint32_t r : lists[(size_t)l]) tcsc[q++] = r;
        pseg[i] = (uint32_t)pst[i] | ((uint32_t)(q - pst[i]) << 16);
      }
    }
  }
  if (bad) return set_error(SYMM_ERR_SCHEDULE, "tiled format: a target is missing from its tile's spill list");
  // multi-rank: keep only this rank's tiles (descriptors re-based to the range)
  if (t_begin != 0 || t_end != nt) {
    const int64_t b0 = boff[(size_t)t_begin], b1 = boff[(size_t)t_end];
    std::vector<TileDesc> d2(desc.begin() + t_begin, desc.begin() + t_end);
    for (auto& D : d2) D.block_off -= b0;  // runs / targets / slots stay global arrays
    std::vector<unsigned char> bl2(blocks.begin() + b0, blocks.begin() + b1);
    for (size_t i = 0; i < d2.size(); ++i)
      std::memcpy(bl2.data() + d2[i].block_off, &d2[i], sizeof(TileDesc));
    desc.swap(d2);
    blocks.swap(bl2);
  }
  H.slot_first.swap(slot_first);
  H.desc.swap(desc);
  H.blocks.swap(blocks);
  H.slot_tgt.swap(slot_tgt);
  H.slots.swap(slots);
  H.in_ptr.swap(in_ptr);
  H.runs.swap(runs);
  H.nsp = nsp;
  H.block_cap = block_cap;
  H.window_cap = window_cap;
  H.nnz_cap = nnz_cap;
  return SYMM_OK;
}

int build_tiled(symmspmv_plan_t* P, const Schedule& S, int32_t t_begin, int32_t t_end) {
  TiledHost H;
  if (int rc = build_tiled_host(S, t_begin, t_end, H)) return rc;
  const int32_t n = S.n;
  const int64_t nsp = H.nsp;
  const int32_t ntl = (int32_t)H.desc.size();
  TileDesc* d_desc;
  unsigned char* d_blocks;
  double* d_spill;
  int32_t* d_slots;
  SpillRun* d_runs;
  int rc;
  // interior / boundary split (multi-rank plans only): a tile is a boundary
  // tile if its window reaches a row >= row_end (the halo)
  std::vector<TileDesc> dbnd;
  if (P->nranks > 1) {
    std::vector<TileDesc> dint;
    for (int32_t i = 0; i < ntl; ++i) {
      const int32_t t = t_begin + i;
      const int64_t a = S.spill_ptr[(size_t)t], b = S.spill_ptr[(size_t)t + 1];
      const bool bnd = b > a && (int32_t)((uint32_t)S.spill[(size_t)b - 1] & kIdxMask) >= P->row_end;
      (bnd ? dbnd : dint).push_back(H.desc[(size_t)i]);
      (bnd ? P->nnz_boundary : P->nnz_interior) += H.desc[(size_t)i].nnz;
    }
    H.desc.swap(dint);
  } else {
    for (const TileDesc& d : H.desc) P->nnz_interior += d.nnz;
  }
  const int32_t nint = (int32_t)H.desc.size(), nbnd = (int32_t)dbnd.size();
  TileDesc* d_desc_b = nullptr;
  if (nbnd > 0 && (rc = upload(P, &d_desc_b, dbnd.data(), dbnd.size()))) return rc;
  if ((rc = upload(P, &d_desc, H.desc.data(), H.desc.size())) || (rc = upload(P, &d_blocks, H.blocks.data(), H.blocks.size())) ||
      (rc = upload(P, &d_slots, H.slots.data(), H.slots.size())) || (rc = upload(P, &d_runs, H.runs.data(), H.runs.size())) ||
      (rc = upload(P, &P->d_in_ptr, H.in_ptr.data(), H.in_ptr.size())) || (rc = dev_alloc(P, &d_spill, (size_t)std::max<int64_t>(nsp, 1))))
    return rc;
  K8Args k8h{};
  k8h.slots = d_slots;
  k8h.spill_buf = d_spill;
  // (K8 holds a thread's slot sums in registers: window_cap <= kK8Slots x 224)
  if (t_begin == 0 && t_end == (int32_t)S.tile_group.size() && !std::getenv("SYMM_NO_K8") &&
      H.window_cap <= kK8Slots * 7 * 32) {
    // K8 (single rank): tiles in id order, DAG of smaller-id writers, flush counters
    // phase-major order (phases are the tile colours: the DAG of conflicting
    // earlier-phase tiles is only n_phases deep)
    std::vector<int32_t> order((size_t)ntl);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return S.tile_phase[(size_t)a] < S.tile_phase[(size_t)b]; });
    std::vector<int32_t> dq(S.dag_pred);
    if (dq.empty()) dq.push_back(0);
    // per processing position: the tile and its predecessor range, one 16-B
    // load (the consumers prefetch it a group tile ahead)
    std::vector<int32_t> pm(4 * (size_t)ntl, 0);
    for (int32_t q = 0; q < ntl; ++q) {
      const int32_t id = order[(size_t)q];
      pm[4 * (size_t)q] = id;
      pm[4 * (size_t)q + 1] = S.dag_ptr[(size_t)id];
      pm[4 * (size_t)q + 2] = S.dag_ptr[(size_t)id + 1];
    }
    int32_t* d_pm;
    int32_t *d_order, *d_dp, *d_dq;
    unsigned int* d_done;
    uint8_t *d_of, *d_sf;
    std::vector<uint8_t> of(S.own_first.begin(), S.own_first.end()), sf(H.slot_first.begin(), H.slot_first.end());
    if (sf.empty()) sf.push_back(0);
    if ((rc = upload(P, &d_of, of.data(), of.size())) || (rc = upload(P, &d_sf, sf.data(), sf.size())) ||
        (rc = upload(P, &d_order, order.data(), order.size())) || (rc = upload(P, &d_pm, pm.data(), pm.size())) ||
        (rc = upload(P, &d_dp, S.dag_ptr.data(), S.dag_ptr.size())) ||
        (rc = upload(P, &d_dq, dq.data(), dq.size())) || (rc = dev_alloc(P, &d_done, (size_t)std::max(ntl, 1))))
      return rc;
    k8h.order = d_order;
    k8h.pos_meta = d_pm;
    k8h.dag_ptr = d_dp;
    k8h.dag_pred = d_dq;
    k8h.done = d_done;
    k8h.own_first = d_of;
    k8h.slot_first = d_sf;
    P->k8_done = d_done;
    P->has_tiled_colored = true;
  }
  // K4 zeroes y in the kernel (ticketed launch counter, kernels.cu k4_zero_y)
  // when the local y is small next to the L2: the zeros then stay in L2 and
  // the in-kernel prologue saves the k_zero launch and its tail.  A y much
  // larger than the L2 costs its 8n bytes of DRAM writes either way; a
  // separate full-bandwidth k_zero launch is then cheaper than zeroing inside
  // the kernel (lap3d_512: 2.23 vs 2.33 ms; st27_128 0.0926 vs 0.0893 ms the
  // other way).  SYMM_K4_ZERO=0/1 forces either (A/B diagnostics).
  unsigned long long* d_zc;
  if ((rc = dev_alloc(P, &d_zc, 1))) return rc;
  if (cudaError_t ze = cudaMemset(d_zc, 0, sizeof(unsigned long long))) return cuda_fail(ze, "zero counter");
  {
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, P->device);
    const int64_t ybytes = 8 * ((int64_t)P->local_end - P->row_begin);
    bool self_zero = ybytes <= (int64_t)l2 / 2;
    if (const char* e = std::getenv("SYMM_K4_ZERO")) self_zero = std::atoi(e) != 0;
    k8h.zero_ctr = self_zero ? d_zc : nullptr;
    P->k4_self_zero = self_zero;
  }
  k8h.zero_begin = P->row_begin;
  k8h.zero_end = P->local_end;
  if (const char* zd = std::getenv("SYMM_ZERO_DBG")) k8h.zero_dbg = std::atoi(zd);
  K8Args* d_k8;
  if ((rc = upload(P, &d_k8, &k8h, 1))) return rc;
  K8Args k8b = k8h;
  k8b.zero_ctr = nullptr;  // the boundary launch follows the interior one, which zeroed y
  K8Args* d_k8b;
  if ((rc = upload(P, &d_k8b, &k8b, 1))) return rc;
  P->targs.k8 = d_k8;
  TiledArgs& A = P->targs;
  A.tiles = d_desc;
  A.ntiles = nint;
  A.blocks = d_blocks;
  A.runs = d_runs;
#if defined(K4_CHECK) || defined(K4_TRACE)
  A.check_n = n;
#endif
  A.block_cap = H.block_cap;
  A.window_cap = H.window_cap;
  P->tiled_nnz_cap = H.nnz_cap;
  if (const char* dbg = std::getenv("SYMM_DEBUG_SKIP")) A.debug_skip = std::atoi(dbg);  // diagnostics only
  P->fargs = FixupArgs{n, P->d_in_ptr, d_spill};
  int stages = 0;
  rc = tiled_max_ctas_per_sm(P->vec, A, &stages);
  if (rc) return cuda_fail((cudaError_t)rc, "shared-memory attribute (tiled)");
  if (stages < 2) {
    A.stages = 2;
    return set_error(SYMM_ERR_UNSUPPORTED, "tiled kernel needs %d B of shared memory for 2 stages", tiled_smem_bytes(A));
  }
  A.stages = stages;
  P->tiled_occ = stages;
  P->tiled_grid = std::max(1, std::min(P->sms, nint));
  P->targs_b = A;
  P->targs_b.tiles = d_desc_b;
  P->targs_b.ntiles = nbnd;
  P->targs_b.k8 = d_k8b;
  P->tiled_grid_b = std::max(1, std::min(P->sms, nbnd));
  P->has_tiled = true;
  return SYMM_OK;
}

// K6: the full matrix A' = U' + U'^T - diag(U') of the permuted order in CRS
// (columns ascending per row), for the Alg. 1 yardstick.
int build_spmv(symmspmv_plan_t* P, const Schedule& S) {
  const int32_t n = S.n;
  std::vector<int64_t> cnt((size_t)n + 1, 0);
  for (int32_t r = 0; r < n; ++r)
    for (int32_t i = S.prow_ptr[(size_t)r]; i < S.prow_ptr[(size_t)r + 1]; ++i) {
      cnt[(size_t)r + 1]++;
      if (S.pcol[(size_t)i] != r) cnt[(size_t)S.pcol[(size_t)i] + 1]++;
    }
  for (int32_t r = 0; r < n; ++r) cnt[(size_t)r + 1] += cnt[(size_t)r];
  if (cnt[(size_t)n] >= ((int64_t)1 << 31)) return set_error(SYMM_ERR_OVERFLOW, "full matrix has >= 2^31 entries");
  std::vector<int32_t> rp((size_t)n + 1), col((size_t)cnt[(size_t)n]);
  std::vector<double> val((size_t)cnt[(size_t)n]);
  for (int32_t r = 0; r <= n; ++r) rp[(size_t)r] = (int32_t)cnt[(size_t)r];
  {
    // lower part first (rows r get (r, c) for c < r from U' rows c), then the upper row
    std::vector<int32_t> pos(rp.begin(), rp.end() - 1);
    for (int32_t c = 0; c < n; ++c)
      for (int32_t i = S.prow_ptr[(size_t)c]; i < S.prow_ptr[(size_t)c + 1]; ++i) {
        const int32_t r = S.pcol[(size_t)i];
        if (r == c) continue;
        col[(size_t)pos[(size_t)r]] = c;  // ascending c by construction
        val[(size_t)pos[(size_t)r]++] = S.pval[(size_t)i];
      }
    for (int32_t r = 0; r < n; ++r)
      for (int32_t i = S.prow_ptr[(size_t)r]; i < S.prow_ptr[(size_t)r + 1]; ++i) {
        col[(size_t)pos[(size_t)r]] = S.pcol[(size_t)i];
        val[(size_t)pos[(size_t)r]++] = S.pval[(size_t)i];
      }
  }
  int rc;
  if ((rc = upload(P, &P->d_frp, rp.data(), rp.size())) || (rc = upload(P, &P->d_fcol, col.data(), col.size())) ||
      (rc = upload(P, &P->d_fval, val.data(), val.size())))
    return rc;
  P->spmv_nnz = (int64_t)col.size();
  {  // lanes per row: the largest power of two <= NNZR / 1.5 (measured on B200: st27 16, kNN 8, 7-pt 4)
    const double avg = n > 0 ? (double)P->spmv_nnz / n : 1.0;
    int v = 1;
    while (v < 32 && 2.0 * v <= avg / 1.5) v *= 2;
    P->spmv_vec = v;
  }
  if (const char* v = std::getenv("SYMM_SPMV_VEC")) P->spmv_vec = std::atoi(v);
  P->has_spmv = true;
  return SYMM_OK;
}

// K5 format (cs_build.cpp); single rank.
int build_cs(symmspmv_plan_t* P, const Schedule& S) {
  const int32_t nt = (int32_t)S.tile_group.size();
  int32_t wcap = 4096, nnzcap = 1 << 30, chunk = 24576, nc = 8, stages = 4, V = 1;
  if (const char* v = std::getenv("SYMM_CS_WINDOW")) wcap = std::atoi(v);
  if (const char* v = std::getenv("SYMM_CS_NNZ")) nnzcap = std::atoi(v);
  if (const char* v = std::getenv("SYMM_CS_CHUNK")) chunk = std::atoi(v);
  if (const char* v = std::getenv("SYMM_CS_NC")) nc = std::atoi(v);
  if (const char* v = std::getenv("SYMM_CS_STAGES")) stages = std::atoi(v);
  if (const char* v = std::getenv("SYMM_CS_V")) V = std::atoi(v);
  if (stages != 4 && stages != 8) return set_error(SYMM_ERR_ARG, "colored_smem ring stages %d (4 or 8)", stages);
  int devsmem = 0;
  cudaDeviceGetAttribute(&devsmem, cudaDevAttrMaxSharedMemoryPerBlockOptin, P->device);
  // ring stages: what is left after heads and windows (capped at kCsMaxStages = 8)
  CsHost H;
  int rc = build_cs_format(S, 0, nt, wcap, nnzcap, chunk, stages, V, &H);
  if (rc) return rc;
  CsArgs& A = P->cargs;
  A.Wcap = H.Wcap;
  A.Hcap = H.Hcap;
  A.chunk = chunk;
  A.stages = stages;
  A.lgstages = stages == 8 ? 3 : 2;
  A.lgv = V == 4 ? 2 : V == 2 ? 1 : 0;
  if (H.max_colour_chunks > stages - 1)
    return set_error(SYMM_ERR_SCHEDULE, "colored_smem: a colour spans %d chunks (ring of %d)", H.max_colour_chunks, stages);
  if (cs_smem_bytes(A) + 1024 > devsmem)
    return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem needs %d B of shared memory (window %d, head %d, ring %d x %d)",
                     cs_smem_bytes(A), H.Wcap, H.Hcap, stages, chunk);
  CsDesc* d_desc;
  unsigned char* d_blocks;
  int64_t* d_coff;
  int32_t* d_clen;
  if ((rc = upload(P, &d_desc, H.desc.data(), H.desc.size())) ||
      (rc = upload(P, &d_blocks, H.blocks.data(), H.blocks.size())) ||
      (rc = upload(P, &d_coff, H.chunk_off.data(), H.chunk_off.size())) ||
      (rc = upload(P, &d_clen, H.chunk_len.data(), H.chunk_len.size())))
    return rc;
  A.desc = d_desc;
  A.ntiles = (int32_t)H.desc.size();
  A.blocks = d_blocks;
  A.chunk_off = d_coff;
  A.chunk_len = d_clen;
  if (const char* dbg = std::getenv("SYMM_DEBUG_SKIP")) A.debug_skip = std::atoi(dbg);  // diagnostics only
  int occ = 0;
  rc = cs_configure(A, &occ, nc);
  if (rc) return cuda_fail((cudaError_t)rc, "colored_smem configure");
  if (occ < 1) return set_error(SYMM_ERR_UNSUPPORTED, "colored_smem needs %d B of shared memory per CTA", cs_smem_bytes(A));
  P->cs_occ = occ;
  P->cs_nc = nc;
  P->cs_grid = std::max(1, std::min(P->sms * occ, A.ntiles));
  P->cs_sum_colors = H.sum_colors;
  P->cs_sum_spill = H.sum_spill;
  P->has_cs = true;
  return SYMM_OK;
}

int build_colored(symmspmv_plan_t* P, const Schedule& S) {
  const int32_t nt = (int32_t)S.tile_group.size();
  std::vector<int32_t> ptiles;
  P->phase_off.assign((size_t)S.n_phases + 1, 0);
  for (int32_t t = 0; t < nt; ++t) P->phase_off[(size_t)S.tile_phase[(size_t)t] + 1]++;
  for (int32_t p = 0; p < S.n_phases; ++p) P->phase_off[(size_t)p + 1] += P->phase_off[(size_t)p];
  ptiles.resize((size_t)nt);
  std::vector<int32_t> pos(P->phase_off.begin(), P->phase_off.end() - 1);
  for (int32_t t = 0; t < nt; ++t) ptiles[(size_t)pos[(size_t)S.tile_phase[(size_t)t]]++] = t;
  int rc;
  if ((rc = upload(P, &P->d_tile_ptr, S.tile_ptr.data(), S.tile_ptr.size())) ||
      (rc = upload(P, &P->d_phase_tiles, ptiles.data(), ptiles.size())) ||
      (rc = upload(P, &P->d_srow, S.srow.data(), S.srow.size())) ||
      (rc = upload(P, &P->d_tile_sub_ptr, S.tile_sub_ptr.data(), S.tile_sub_ptr.size())) ||
      (rc = upload(P, &P->d_sub_ptr, S.sub_ptr.data(), S.sub_ptr.size())))
    return rc;
  P->has_colored = true;
  return SYMM_OK;
}

// K7: the recursive tree's leaves in execution order (depth first, red
// children before blue children), per leaf its tiles, the ancestors it waits
// at (it lies in a blue child) and the ancestors it counts at (red child).
int build_tree(symmspmv_plan_t* P, const Schedule& S) {
  const int32_t nn = (int32_t)S.tree_parent.size();
  if (nn == 0) return set_error(SYMM_ERR_ARG, "variant TREE needs a schedule built with scheme = 3 (recursive tree)");
  std::vector<std::vector<int32_t>> kids((size_t)nn);
  for (int32_t v = 1; v < nn; ++v) kids[(size_t)S.tree_parent[(size_t)v]].push_back(v);
  for (auto& k : kids)
    std::sort(k.begin(), k.end(), [&](int32_t a, int32_t b) { return S.tree_cidx[(size_t)a] < S.tree_cidx[(size_t)b]; });
  std::vector<int32_t> group_of_node((size_t)nn, -1);
  for (size_t g = 0; g < S.tree_leaf.size(); ++g) group_of_node[(size_t)S.tree_leaf[g]] = (int32_t)g;
  const int32_t ng = (int32_t)S.tree_leaf.size(), nt = (int32_t)S.tile_group.size();
  std::vector<int32_t> gt0((size_t)ng, nt), gt1((size_t)ng, 0);
  for (int32_t t = 0; t < nt; ++t) {
    const int32_t g = S.tile_group[(size_t)t];
    gt0[(size_t)g] = std::min(gt0[(size_t)g], t);
    gt1[(size_t)g] = std::max(gt1[(size_t)g], t + 1);
  }
  std::vector<int32_t> order;  // execution order of the leaves (node ids)
  std::vector<int32_t> red_total((size_t)nn, 0);
  std::function<int32_t(int32_t)> visit = [&](int32_t v) -> int32_t {  // returns leaves under v
    if (kids[(size_t)v].empty()) {
      if (group_of_node[(size_t)v] < 0) return 0;  // empty node
      order.push_back(v);
      return 1;
    }
    int32_t red = 0, tot = 0;
    for (int par = 0; par < 2; ++par)
      for (int32_t c : kids[(size_t)v])
        if ((S.tree_cidx[(size_t)c] & 1) == par) {
          const int32_t k = visit(c);
          if (par == 0) red += k;
          tot += k;
        }
    red_total[(size_t)v] = red;
    return tot;
  };
  visit(0);
  const int32_t nl = (int32_t)order.size();
  std::vector<int32_t> t0((size_t)nl), t1((size_t)nl), wptr(1, 0), wnode, sptr(1, 0), snode;
  for (int32_t i = 0; i < nl; ++i) {
    const int32_t g = group_of_node[(size_t)order[(size_t)i]];
    t0[(size_t)i] = gt0[(size_t)g];
    t1[(size_t)i] = std::max(gt0[(size_t)g], gt1[(size_t)g]);
    for (int32_t v = order[(size_t)i]; S.tree_parent[(size_t)v] >= 0; v = S.tree_parent[(size_t)v]) {
      const int32_t a = S.tree_parent[(size_t)v];
      if (S.tree_cidx[(size_t)v] & 1) {
        if (red_total[(size_t)a] > 0) wnode.push_back(a);
      } else {
        snode.push_back(a);
      }
    }
    wptr.push_back((int32_t)wnode.size());
    sptr.push_back((int32_t)snode.size());
  }
  if (wnode.empty()) wnode.push_back(0);
  if (snode.empty()) snode.push_back(0);
  int32_t *d_t0, *d_t1, *d_wp, *d_wn, *d_sp, *d_sn, *d_rt, *d_cnt;
  int rc;
  if ((rc = upload(P, &d_t0, t0.data(), t0.size())) || (rc = upload(P, &d_t1, t1.data(), t1.size())) ||
      (rc = upload(P, &d_wp, wptr.data(), wptr.size())) || (rc = upload(P, &d_wn, wnode.data(), wnode.size())) ||
      (rc = upload(P, &d_sp, sptr.data(), sptr.size())) || (rc = upload(P, &d_sn, snode.data(), snode.size())) ||
      (rc = upload(P, &d_rt, red_total.data(), red_total.size())) || (rc = dev_alloc(P, &d_cnt, (size_t)nn + 1)))
    return rc;
  P->tree = TreeArgs{nl, nn, d_t0, d_t1, d_wp, d_wn, d_sp, d_sn, d_rt, d_cnt};
  // one resident CTA per worker of the tree (256 threads: 8 per SM)
  P->tree_grid = std::max(1, std::min(nl, 8 * P->sms));
  P->has_tree = true;
  return SYMM_OK;
}

int run_permuted(symmspmv_plan_t* P, int variant, const double* x, double* y, cudaStream_t st,
                 int part = SYMM_PART_ALL) {
  int rc = 0;
  P->last_launches = 0;
  if (part != SYMM_PART_ALL && variant != SYMM_VARIANT_TILED_ATOMIC &&
      !(variant == SYMM_VARIANT_AUTO && P->nranks > 1))
    return set_error(SYMM_ERR_ARG, "run_part needs the tiled_atomic variant");
  if (P->n == 0) return SYMM_OK;
  if (variant == SYMM_VARIANT_AUTO) variant = P->variant;
  // AUTO: the fastest measured variant (profiles/) that this plan holds
  if (variant == SYMM_VARIANT_AUTO) variant = P->has_tiled ? SYMM_VARIANT_TILED_ATOMIC : SYMM_VARIANT_COLORED;
  if (variant == SYMM_VARIANT_ATOMIC) {
    if (!P->has_csr) return set_error(SYMM_ERR_ARG, "variant ATOMIC was not uploaded by this plan");
    CsrArgs A{P->n, P->d_rp, P->d_col, P->d_val};
    if ((rc = launch_zero(y, P->n, st))) return cuda_fail((cudaError_t)rc, "zero y");
    if ((rc = launch_atomic(A, x, y, P->vec, P->sms, st))) return cuda_fail((cudaError_t)rc, "k_atomic");
    P->last_launches = 2;
  } else if (variant == SYMM_VARIANT_COLORED) {
    if (!P->has_colored) return set_error(SYMM_ERR_ARG, "variant COLORED was not uploaded by this plan");
    CsrArgs A{P->n, P->d_rp, P->d_col, P->d_val};
    if ((rc = launch_zero(y, P->n, st))) return cuda_fail((cudaError_t)rc, "zero y");
    P->last_launches = 1;
    for (size_t p = 0; p + 1 < P->phase_off.size(); ++p) {
      ColoredArgs C{P->d_tile_ptr, P->d_phase_tiles + P->phase_off[p], P->phase_off[p + 1] - P->phase_off[p],
                    P->d_srow, P->d_tile_sub_ptr, P->d_sub_ptr};
      if ((rc = launch_colored_phase(A, C, x, y, P->vec, st))) return cuda_fail((cudaError_t)rc, "k_colored");
      P->last_launches += C.nphase_tiles > 0;
    }
  } else if (variant == SYMM_VARIANT_TILED) {
    if (!P->has_tiled) return set_error(SYMM_ERR_ARG, "variant TILED was not uploaded by this plan");
    if ((rc = launch_tiled(P->targs, x, y, P->vec, P->tiled_grid, 0, st))) return cuda_fail((cudaError_t)rc, "k_tiled");
    if ((rc = launch_fixup(P->fargs, y, st))) return cuda_fail((cudaError_t)rc, "k_fixup");
    P->last_launches = 2;
  } else if (variant == SYMM_VARIANT_TILED_ATOMIC) {
    if (!P->has_tiled) return set_error(SYMM_ERR_ARG, "variant TILED_ATOMIC was not uploaded by this plan");
    // x, y cover rows [row_begin, local_end); kernels index by global row id
    // k_tiled<1> zeroes y itself (K8Args::zero_*); a rank without tiles only zeroes
    // part INTERIOR (or ALL) zeroes y and runs the interior tiles; part
    // BOUNDARY (or ALL) runs the tiles that touch halo rows
    const int64_t nloc = (int64_t)P->local_end - P->row_begin;
    if (part != SYMM_PART_BOUNDARY) {
      if (P->targs.ntiles <= 0 || !P->k4_self_zero) {
        if ((rc = launch_zero(y, nloc, st))) return cuda_fail((cudaError_t)rc, "zero y");
        P->last_launches = 1;
      }
      if (P->targs.ntiles > 0) {
        if ((rc = launch_tiled(P->targs, x - P->row_begin, y - P->row_begin, P->vec, P->tiled_grid, 1, st)))
          return cuda_fail((cudaError_t)rc, "k_tiled<atomic>");
        P->last_launches += 1;
      }
    }
    if (part != SYMM_PART_INTERIOR && P->targs_b.ntiles > 0) {
      if ((rc = launch_tiled(P->targs_b, x - P->row_begin, y - P->row_begin, P->vec, P->tiled_grid_b, 1, st)))
        return cuda_fail((cudaError_t)rc, "k_tiled<atomic> (boundary tiles)");
      P->last_launches += 1;
    }
  } else if (variant == SYMM_VARIANT_TILED_COLORED) {
    if (!P->has_tiled_colored) return set_error(SYMM_ERR_ARG, "variant TILED_COLORED was not uploaded by this plan");
    cudaError_t e = cudaMemsetAsync(P->k8_done, 0, sizeof(unsigned int) * (size_t)P->targs.ntiles, st);
    if (e != cudaSuccess) return cuda_fail(e, "tile counters");
    if ((rc = launch_tiled(P->targs, x, y, P->vec, P->tiled_grid, 2, st))) return cuda_fail((cudaError_t)rc, "k_tiled<ordered>");
    P->last_launches = 1;
  } else if (variant == SYMM_VARIANT_TREE) {
    if (!P->has_tree) return set_error(SYMM_ERR_ARG, "variant TREE was not uploaded by this plan");
    CsrArgs A{P->n, P->d_rp, P->d_col, P->d_val};
    ColoredArgs C{P->d_tile_ptr, P->d_phase_tiles, 0, P->d_srow, P->d_tile_sub_ptr, P->d_sub_ptr};
    cudaError_t e = cudaMemsetAsync(P->tree.counters, 0, sizeof(int32_t) * ((size_t)P->tree.nnodes + 1), st);
    if (e != cudaSuccess) return cuda_fail(e, "tree counters");
    if ((rc = launch_zero(y, P->n, st))) return cuda_fail((cudaError_t)rc, "zero y");
    if ((rc = launch_tree(A, C, P->tree, x, y, P->vec, P->tree_grid, st))) return cuda_fail((cudaError_t)rc, "k_tree");
    P->last_launches = 2;
  } else if (variant == SYMM_VARIANT_SPMV) {
    if (!P->has_spmv) return set_error(SYMM_ERR_ARG, "variant SPMV was not uploaded by this plan");
    CsrArgs A{P->n, P->d_frp, P->d_fcol, P->d_fval};
    if ((rc = launch_spmv(A, x, y, P->spmv_vec, P->sms, st))) return cuda_fail((cudaError_t)rc, "k_spmv");
    P->last_launches = 1;
  } else if (variant == SYMM_VARIANT_COLORED_SMEM) {
    if (!P->has_cs) return set_error(SYMM_ERR_ARG, "variant COLORED_SMEM was not uploaded by this plan");
    if ((rc = launch_zero(y, P->n, st))) return cuda_fail((cudaError_t)rc, "zero y");
    if ((rc = launch_cs(P->cargs, x, y, P->cs_grid, P->cs_nc, st))) return cuda_fail((cudaError_t)rc, "k_cs");
    P->last_launches = 2;
  } else {
    return set_error(SYMM_ERR_ARG, "unknown variant %d", variant);
  }
  return SYMM_OK;
}

}  // namespace

extern "C" {

const char* symm_status_string(int s) {
  switch (s) {
    case SYMM_OK: return "SYMM_OK";
    case SYMM_ERR_ARG: return "SYMM_ERR_ARG";
    case SYMM_ERR_NOT_UPPER: return "SYMM_ERR_NOT_UPPER";
    case SYMM_ERR_UNSORTED: return "SYMM_ERR_UNSORTED";
    case SYMM_ERR_OVERFLOW: return "SYMM_ERR_OVERFLOW";
    case SYMM_ERR_OOM: return "SYMM_ERR_OOM";
    case SYMM_ERR_CUDA: return "SYMM_ERR_CUDA";
    case SYMM_ERR_NCCL: return "SYMM_ERR_NCCL";
    case SYMM_ERR_MISMATCH: return "SYMM_ERR_MISMATCH";
    case SYMM_ERR_ALIAS: return "SYMM_ERR_ALIAS";
    case SYMM_ERR_SCHEDULE: return "SYMM_ERR_SCHEDULE";
    case SYMM_ERR_K: return "SYMM_ERR_K";
    case SYMM_ERR_UNSUPPORTED: return "SYMM_ERR_UNSUPPORTED";
    default: return "SYMM_ERR_UNKNOWN";
  }
}
const char* symm_last_error(void) { return symm::last_error(); }

void race_config_default(race_config* c) {
  if (!c) return;
  std::memset(c, 0, sizeof *c);
  c->k = 2;
  c->n_workers = 0;
  c->tile_work = 3500;  // measured on B200 (profiles/r1_summary.md): bigger tiles, fewer spill REDs
  c->balance_by = 1;
  c->root = -1;
  c->n_eps = 3;
  c->eps[0] = 0.8;  // eps_0 = eps_1 = 0.8, eps_{s>1} = 0.5
  c->eps[1] = 0.8;
  for (int i = 2; i < 8; ++i) c->eps[i] = 0.5;
  c->max_tile_rows = 1024;
  c->max_tile_window = 1200;
  c->max_tile_nnz = 3000;
  c->reorder = 1;
  c->cone_tiles = 0;
  c->min_group_levels = 2;
  c->validate = 1;
  c->flags = 0;
  c->scheme = 0;
  c->abmc_block = 64;
}

int race_build_schedule(const symm_csr_upper* U, const race_config* cfg, race_schedule_t** out) {
  clear_error();
  if (!out) return set_error(SYMM_ERR_ARG, "out is NULL");
  *out = nullptr;
  std::unique_ptr<race_schedule> s;
  try {
    s.reset(new race_schedule());
    int rc = build_schedule(U, cfg, &s->S);
    if (rc) return rc;
  } catch (const std::bad_alloc&) {
    return set_error(SYMM_ERR_OOM, "host allocation failed while building the schedule");
  }
  *out = s.release();
  return SYMM_OK;
}

int race_schedule_get_stats(const race_schedule_t* s, race_schedule_stats* o) {
  if (!s || !o) return set_error(SYMM_ERR_ARG, "NULL argument");
  const Schedule& S = s->S;
  std::memset(o, 0, sizeof *o);
  o->n = S.n;
  o->total_levels = (int32_t)S.level_ptr.size() - 1;
  o->n_components = (int32_t)S.roots.size();
  o->n_groups = (int32_t)S.group_workers.size();
  o->n_tiles = (int32_t)S.tile_group.size();
  o->n_phases = S.n_phases;
  o->max_subcolors = S.max_subcolors;
  o->max_tile_window = S.max_window;
  o->max_tile_rows = S.max_rows;
  o->n_dag_edges = (int32_t)S.dag_pred.size();
  o->nnz = S.nnz;
  o->bandwidth_before = S.bw_before;
  o->bandwidth_after = S.bw_after;
  o->eta = S.eta;
  o->build_seconds = S.build_seconds;
  o->mean_subcolors = S.mean_subcolors;
  o->spill_entries = (int64_t)S.spill.size();
  return SYMM_OK;
}

int race_schedule_permutation(const race_schedule_t* s, int32_t* perm, int32_t* inv) {
  if (!s) return set_error(SYMM_ERR_ARG, "NULL schedule");
  if (perm) std::copy(s->S.perm.begin(), s->S.perm.end(), perm);
  if (inv) std::copy(s->S.inv.begin(), s->S.inv.end(), inv);
  return SYMM_OK;
}

int race_schedule_table(const race_schedule_t* s, const char* which, int64_t* len, int32_t* out) {
  if (!s || !which || !len) return set_error(SYMM_ERR_ARG, "NULL argument");
  const Schedule& S = s->S;
  const std::vector<int32_t>* v = nullptr;
  std::string w(which);
  if (w == "level_ptr") v = &S.level_ptr;
  else if (w == "dist") v = &S.dist;
  else if (w == "roots") v = &S.roots;
  else if (w == "group_lvl") v = &S.group_lvl;
  else if (w == "group_workers") v = &S.group_workers;
  else if (w == "tile_ptr") v = &S.tile_ptr;
  else if (w == "tile_group") v = &S.tile_group;
  else if (w == "tile_phase") v = &S.tile_phase;
  else if (w == "tile_order") v = &S.tile_order;
  else if (w == "dag_ptr") v = &S.dag_ptr;
  else if (w == "dag_pred") v = &S.dag_pred;
  else if (w == "row_subcolor") v = &S.row_subcolor;
  else if (w == "window_levels") v = &S.windows;
  else if (w == "srow") v = &S.srow;
  else if (w == "tile_sub_ptr") v = &S.tile_sub_ptr;
  else if (w == "sub_ptr") v = &S.sub_ptr;
  else if (w == "spill") v = &S.spill;
  else if (w == "tree_parent") v = &S.tree_parent;
  else if (w == "tree_cidx") v = &S.tree_cidx;
  else if (w == "tree_r0") v = &S.tree_r0;
  else if (w == "tree_r1") v = &S.tree_r1;
  else if (w == "tree_stage") v = &S.tree_stage;
  else if (w == "tree_workers") v = &S.tree_workers;
  else if (w == "tree_leaf") v = &S.tree_leaf;
  else if (w == "own_first") {
    *len = (int64_t)S.own_first.size();
    if (out) for (size_t i = 0; i < S.own_first.size(); ++i) out[i] = S.own_first[i];
    return SYMM_OK;
  } else if (w == "spill_ptr") {
    *len = (int64_t)S.spill_ptr.size();
    if (out) for (size_t i = 0; i < S.spill_ptr.size(); ++i) out[i] = (int32_t)S.spill_ptr[i];
    return SYMM_OK;
  }
  if (!v) return set_error(SYMM_ERR_ARG, "unknown table '%s'", which);
  *len = (int64_t)v->size();
  if (out) std::copy(v->begin(), v->end(), out);
  return SYMM_OK;
}

int race_schedule_permuted_matrix(const race_schedule_t* s, int32_t* row_ptr, int32_t* col, double* val) {
  if (!s) return set_error(SYMM_ERR_ARG, "NULL schedule");
  const Schedule& S = s->S;
  if (row_ptr) std::copy(S.prow_ptr.begin(), S.prow_ptr.end(), row_ptr);
  if (col) std::copy(S.pcol.begin(), S.pcol.end(), col);
  if (val) std::copy(S.pval.begin(), S.pval.end(), val);
  return SYMM_OK;
}

void race_schedule_destroy(race_schedule_t* s) { delete s; }

void symmspmv_options_default(symmspmv_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof *o);
  o->variant = SYMM_VARIANT_AUTO;
  o->device = 0;
  o->vec_order = SYMM_ORDER_PERMUTED;
  o->nranks = 1;
  o->rank = 0;
  o->vec_width = 0;
  o->ctas_per_sm = 0;
  o->build_all = 0;
}

int symmspmv_plan(const race_schedule_t* s, const symm_csr_upper* U, const symmspmv_options* o,
                  symmspmv_plan_t** out) {
  clear_error();
  if (!s || !out) return set_error(SYMM_ERR_ARG, "NULL argument");
  *out = nullptr;
  symmspmv_options opt;
  if (o) opt = *o;
  else symmspmv_options_default(&opt);
  const Schedule& S = s->S;
  if (U && (U->n != S.n || U->nnz != S.nnz))
    return set_error(SYMM_ERR_MISMATCH, "matrix (n=%d, nnz=%lld) does not match the schedule (n=%d, nnz=%lld)", U->n,
                     (long long)U->nnz, S.n, (long long)S.nnz);
  if (opt.variant < 0 || opt.variant > 8) return set_error(SYMM_ERR_ARG, "variant %d", opt.variant);
  if (opt.nranks < 1 || opt.rank < 0 || opt.rank >= opt.nranks)
    return set_error(SYMM_ERR_ARG, "rank %d of %d", opt.rank, opt.nranks);
  if (opt.nranks > 1 && opt.variant != SYMM_VARIANT_TILED_ATOMIC && opt.variant != SYMM_VARIANT_AUTO)
    return set_error(SYMM_ERR_UNSUPPORTED, "multi-rank plans support the tiled_atomic variant only");
  if (opt.vec_width && (opt.vec_width < 1 || opt.vec_width > 32 || (opt.vec_width & (opt.vec_width - 1))))
    return set_error(SYMM_ERR_ARG, "vec_width %d must be a power of two <= 32", opt.vec_width);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return set_error(SYMM_ERR_CUDA, "no CUDA device available (%s)", cudaGetErrorString(e));
  }
  if (opt.device < 0 || opt.device >= ndev) return set_error(SYMM_ERR_ARG, "device %d of %d", opt.device, ndev);
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(opt.device);
  symmspmv_plan_t* P = new symmspmv_plan_t();
  P->device = opt.device;
  P->variant = opt.variant;
  P->vec_order = opt.vec_order;
  P->n = S.n;
  P->nnz = S.nnz;
  std::vector<int32_t> tb, rb, he;
  partition_tiles(S, opt.nranks, tb, rb, he);
  P->nranks = opt.nranks;
  P->rank = opt.rank;
  P->row_begin = rb[(size_t)opt.rank];
  P->row_end = rb[(size_t)opt.rank + 1];
  P->local_end = he[(size_t)opt.rank];
  P->min_bytes = 12 * S.nnz + 4 * ((int64_t)S.n + 1) + 24 * (int64_t)S.n;
  cudaDeviceGetAttribute(&P->sms, cudaDevAttrMultiProcessorCount, opt.device);
  P->vec = opt.vec_width ? opt.vec_width : pick_vec(S.nnz, S.n);
  int rc = SYMM_OK;
  const bool all = opt.build_all != 0;
  const int v = opt.variant;
  bool want_tiled = all || v == SYMM_VARIANT_TILED || v == SYMM_VARIANT_TILED_ATOMIC || v == SYMM_VARIANT_AUTO ||
                    v == SYMM_VARIANT_TILED_COLORED;
  bool want_col = all || v == SYMM_VARIANT_COLORED;
  bool want_csr = all || v == SYMM_VARIANT_ATOMIC || v == SYMM_VARIANT_COLORED;
  bool want_cs = all || v == SYMM_VARIANT_COLORED_SMEM;
  bool want_spmv = all || v == SYMM_VARIANT_SPMV;
  bool want_tree = (all && !S.tree_parent.empty()) || v == SYMM_VARIANT_TREE;
  if (want_tree) want_col = want_csr = true;
  if (opt.nranks > 1) {
    want_col = want_csr = want_cs = want_spmv = want_tree = false;
    P->variant = SYMM_VARIANT_TILED_ATOMIC;
  }
  if (want_tiled) {
    rc = build_tiled(P, S, tb[(size_t)opt.rank], tb[(size_t)opt.rank + 1]);
    if (rc == SYMM_ERR_UNSUPPORTED && opt.nranks > 1) {
      free_plan(P);
      cudaSetDevice(cur);
      return rc;
    }
    if (rc == SYMM_ERR_UNSUPPORTED && (v == SYMM_VARIANT_AUTO || all)) {
      rc = SYMM_OK;  // AUTO falls back to the colored variant
      want_col = want_csr = true;
      if (P->variant == SYMM_VARIANT_AUTO) P->variant = SYMM_VARIANT_COLORED;
    }
  }
  if (!rc && want_csr) {
    if (!(rc = upload(P, &P->d_rp, S.prow_ptr.data(), S.prow_ptr.size())) &&
        !(rc = upload(P, &P->d_col, S.pcol.data(), S.pcol.size())) &&
        !(rc = upload(P, &P->d_val, S.pval.data(), S.pval.size())))
      P->has_csr = true;
  }
  if (!rc && want_col) rc = build_colored(P, S);
  if (!rc && want_cs) rc = build_cs(P, S);
  if (!rc && want_spmv) rc = build_spmv(P, S);
  if (!rc && want_tree) rc = build_tree(P, S);
  if (!rc) {
    if (!(rc = upload(P, &P->d_perm, S.perm.data(), S.perm.size())) &&
        !(rc = upload(P, &P->d_inv, S.inv.data(), S.inv.size())) && !(rc = dev_alloc(P, &P->d_xp, (size_t)S.n)))
      rc = dev_alloc(P, &P->d_yp, (size_t)S.n);
  }
  if (!rc) {
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = cuda_fail(e, "plan upload");
  }
  cudaSetDevice(cur);
  if (rc) {
    free_plan(P);
    return rc;
  }
  *out = P;
  return SYMM_OK;
}

int symmspmv_plan_rows(const symmspmv_plan_t* p, int32_t* b, int32_t* e) {
  if (!p || !b || !e) return set_error(SYMM_ERR_ARG, "NULL argument");
  *b = p->row_begin;
  *e = p->row_end;
  return SYMM_OK;
}

static int run_variant_part(symmspmv_plan_t* P, int32_t variant, const double* x, double* y, void* stream,
                            int32_t part);

int symmspmv_run_variant(symmspmv_plan_t* P, int32_t variant, const double* x, double* y, void* stream) {
  return run_variant_part(P, variant, x, y, stream, SYMM_PART_ALL);
}

int symmspmv_run_part(symmspmv_plan_t* P, int32_t part, const double* x, double* y, void* stream) {
  if (part < SYMM_PART_ALL || part > SYMM_PART_BOUNDARY) return set_error(SYMM_ERR_ARG, "part %d", part);
  if (P && P->vec_order != SYMM_ORDER_PERMUTED && part != SYMM_PART_ALL)
    return set_error(SYMM_ERR_UNSUPPORTED, "run_part takes x/y in the permuted order");
  if (P && P->nranks == 1) {  // every tile is interior
    if (part == SYMM_PART_BOUNDARY) {
      P->last_launches = 0;
      return SYMM_OK;
    }
    return run_variant_part(P, -1, x, y, stream, SYMM_PART_ALL);
  }
  return run_variant_part(P, SYMM_VARIANT_TILED_ATOMIC, x, y, stream, part);
}

int symmspmv_plan_parts(const symmspmv_plan_t* P, int32_t* n_interior_tiles, int32_t* n_boundary_tiles,
                        int64_t* nnz_interior, int64_t* nnz_boundary) {
  if (!P) return set_error(SYMM_ERR_ARG, "NULL plan");
  if (n_interior_tiles) *n_interior_tiles = P->targs.ntiles;
  if (n_boundary_tiles) *n_boundary_tiles = P->targs_b.ntiles;
  if (nnz_interior) *nnz_interior = P->nnz_interior;
  if (nnz_boundary) *nnz_boundary = P->nnz_boundary;
  return SYMM_OK;
}

static int run_variant_part(symmspmv_plan_t* P, int32_t variant, const double* x, double* y, void* stream,
                            int32_t part) {
  if (!P) return set_error(SYMM_ERR_ARG, "NULL plan");
  if (P->n > 0 && (!x || !y)) return set_error(SYMM_ERR_ARG, "NULL vector");
  if (P->nranks > 1 && variant >= 0 && variant != SYMM_VARIANT_TILED_ATOMIC && variant != SYMM_VARIANT_AUTO)
    return set_error(SYMM_ERR_UNSUPPORTED, "multi-rank plans run the tiled_atomic variant only");
  if (P->nranks > 1 && P->vec_order != SYMM_ORDER_PERMUTED)
    return set_error(SYMM_ERR_UNSUPPORTED, "multi-rank plans take x/y in the permuted order");
  const uintptr_t xa = (uintptr_t)x, ya = (uintptr_t)y,
                  nb = (uintptr_t)((int64_t)P->local_end - P->row_begin) * sizeof(double);
  if (P->n > 0 && xa < ya + nb && ya < xa + nb) return set_error(SYMM_ERR_ALIAS, "x and y overlap");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != P->device) cudaSetDevice(P->device);
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  if (P->vec_order == SYMM_ORDER_ORIGINAL) {
    // x_perm[new] = x[inv[new]];  y[old] = y_perm[perm[old]]
    int e1 = launch_gather(x, P->d_inv, P->d_xp, P->n, st);
    if (e1) rc = cuda_fail((cudaError_t)e1, "gather x");
    else {
      rc = run_permuted(P, variant < 0 ? SYMM_VARIANT_AUTO : variant, P->d_xp, P->d_yp, st, part);
      if (!rc) {
        int e2 = launch_gather(P->d_yp, P->d_perm, y, P->n, st);
        if (e2) rc = cuda_fail((cudaError_t)e2, "gather y");
        P->last_launches += 2;
      }
    }
  } else {
    rc = run_permuted(P, variant < 0 ? SYMM_VARIANT_AUTO : variant, x, y, st, part);
  }
  if (cur != P->device) cudaSetDevice(cur);
  return rc;
}

int symmspmv_run(symmspmv_plan_t* P, const double* x, double* y, void* stream) {
  return symmspmv_run_variant(P, -1, x, y, stream);
}

int symmspmv_powers(symmspmv_plan_t* P, int32_t variant, const double* x, double* Y, int32_t npow, int64_t ldy,
                    void* stream) {
  if (!P) return set_error(SYMM_ERR_ARG, "NULL plan");
  if (P->nranks > 1) return set_error(SYMM_ERR_UNSUPPORTED, "matrix powers are single-rank");
  if (npow < 0 || ldy < P->n) return set_error(SYMM_ERR_ARG, "npow %d, ldy %lld (n %d)", npow, (long long)ldy, P->n);
  if (npow == 0 || P->n == 0) {
    P->last_launches = 0;
    return SYMM_OK;
  }
  if (!x || !Y) return set_error(SYMM_ERR_ARG, "NULL vector");
  const uintptr_t xa = (uintptr_t)x, ya = (uintptr_t)Y, xb = (uintptr_t)P->n * sizeof(double),
                  yb = (uintptr_t)(((int64_t)npow - 1) * ldy + P->n) * sizeof(double);
  if (xa < ya + yb && ya < xa + xb) return set_error(SYMM_ERR_ALIAS, "x overlaps Y");
  int launches = 0;
  for (int32_t k = 0; k < npow; ++k) {
    // y_k = A y_{k-1}, y_0 = x (the definition; oracle.matrix_powers)
    const double* src = k == 0 ? x : Y + (int64_t)(k - 1) * ldy;
    if (int rc = run_variant_part(P, variant, src, Y + (int64_t)k * ldy, stream, SYMM_PART_ALL)) return rc;
    launches += P->last_launches;
  }
  P->last_launches = launches;
  return SYMM_OK;
}

int symmspmv_run_host(symmspmv_plan_t* P, const double* x_host, double* y_host, void* stream) {
  if (!P) return set_error(SYMM_ERR_ARG, "NULL plan");
  if (P->nranks > 1) return set_error(SYMM_ERR_UNSUPPORTED, "run_host is single-rank");
  if (P->n == 0) return SYMM_OK;
  if (!x_host || !y_host) return set_error(SYMM_ERR_ARG, "NULL host vector");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != P->device) cudaSetDevice(P->device);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nb = (size_t)P->n * sizeof(double);
  int rc = SYMM_OK;
  // d_yp holds x (original order) on the way in; d_xp = permuted x; d_yp = permuted y
  cudaError_t e = cudaMemcpyAsync(P->d_yp, x_host, nb, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = cuda_fail(e, "H2D x");
  if (!rc) {
    int e1 = launch_gather(P->d_yp, P->d_inv, P->d_xp, P->n, st);
    if (e1) rc = cuda_fail((cudaError_t)e1, "gather x");
  }
  double* yperm = P->d_yp;
  if (!rc) rc = run_permuted(P, SYMM_VARIANT_AUTO, P->d_xp, yperm, st);
  if (!rc) {
    // y_orig[old] = y_perm[perm[old]] -> written into d_xp (x no longer needed)
    int e2 = launch_gather(yperm, P->d_perm, P->d_xp, P->n, st);
    if (e2) rc = cuda_fail((cudaError_t)e2, "gather y");
    P->last_launches += 2;
  }
  if (!rc) {
    e = cudaMemcpyAsync(y_host, P->d_xp, nb, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "D2H y");
  }
  if (!rc) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = cuda_fail(e, "stream sync");
  }
  if (cur != P->device) cudaSetDevice(cur);
  return rc;
}

int symmspmv_last_launches(const symmspmv_plan_t* p) { return p ? p->last_launches : 0; }

int symmspmv_plan_local(const symmspmv_plan_t* p, int32_t* b, int32_t* e) {
  if (!p || !b || !e) return set_error(SYMM_ERR_ARG, "NULL argument");
  *b = p->row_begin;
  *e = p->local_end;
  return SYMM_OK;
}

int symm_bw_probe(int32_t mode, int32_t device, int64_t bytes, int32_t reps, void* stream, double* gbps) {
  clear_error();
  if (!gbps || (mode != 0 && mode != 1) || bytes < 16 || reps < 1) return set_error(SYMM_ERR_ARG, "bad argument");
  int cur = 0;
  cudaGetDevice(&cur);
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return set_error(SYMM_ERR_ARG, "device %d", device);
  }
  const int rc = bw_probe(mode, bytes, reps, stream, gbps);
  cudaSetDevice(cur);
  if (rc == (int)cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return set_error(SYMM_ERR_OOM, "bandwidth probe: cannot allocate %lld bytes", (long long)bytes);
  }
  return rc ? cuda_fail((cudaError_t)rc, "bandwidth probe") : SYMM_OK;
}

int symmspmv_halo_add(double* y, const double* v, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!y || !v))) return set_error(SYMM_ERR_ARG, "bad argument");
  int rc = launch_add(y, v, n, stream);
  return rc ? cuda_fail((cudaError_t)rc, "k_add") : SYMM_OK;
}

int race_schedule_partition(const race_schedule_t* s, int32_t nranks, int32_t* row_bounds, int32_t* halo_end) {
  if (!s || nranks < 1) return set_error(SYMM_ERR_ARG, "bad argument");
  std::vector<int32_t> tb, rb, he;
  partition_tiles(s->S, nranks, tb, rb, he);
  if (row_bounds) std::copy(rb.begin(), rb.end(), row_bounds);
  if (halo_end) std::copy(he.begin(), he.end(), halo_end);
  return SYMM_OK;
}

int symmspmv_plan_bytes(const symmspmv_plan_t* p, int64_t* device_bytes, int64_t* min_bytes) {
  if (!p) return set_error(SYMM_ERR_ARG, "NULL plan");
  if (device_bytes) *device_bytes = p->device_bytes;
  if (min_bytes) *min_bytes = p->min_bytes;
  return SYMM_OK;
}

// Diagnostics (not in the public header): run the tiled kernel once with the
// event trace of CTA 0 enabled; copies up to `cap` tiles x 8 timestamps to host.
extern "C" int symmspmv_debug_trace(symmspmv_plan_t* P, const double* x, double* y, void* stream,
                                    unsigned long long* host_trace, int32_t cap) {
  if (!P || !P->has_tiled) return set_error(SYMM_ERR_ARG, "no tiled plan");
  unsigned long long* d = nullptr;
  size_t bytes = (size_t)cap * 8 * sizeof(unsigned long long);
  if (cudaMalloc(&d, bytes) != cudaSuccess) return set_error(SYMM_ERR_OOM, "trace buffer");
  cudaMemset(d, 0, bytes);
  TiledArgs A = P->targs;
#ifdef K4_TRACE
  A.trace = d;
#else
  (void)A;
  cudaFree(d);
  return set_error(SYMM_ERR_UNSUPPORTED, "build with -DK4_TRACE for the tiled kernel trace");
#endif
  int rc = launch_tiled(A, x, y, P->vec, P->tiled_grid, 0, stream);
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaMemcpy(host_trace, d, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return rc ? cuda_fail((cudaError_t)rc, "trace launch") : SYMM_OK;
}

// Diagnostics (not in the public header): one colored_smem run with the event
// trace of CTA 0: host_trace[2*cap] chunk (wait start, issue) times, then
// 256 x 4 tile times (start, window ready, colours done, flush done).
extern "C" int symm_cs_debug_trace(symmspmv_plan_t* P, const double* x, double* y, void* stream,
                                   unsigned long long* host_trace, int32_t cap) {
  if (!P || !P->has_cs) return set_error(SYMM_ERR_ARG, "no colored_smem plan");
  unsigned long long* d = nullptr;
  size_t bytes = ((size_t)cap * 2 + 256 * 4 + 512 * 4 + 64) * sizeof(unsigned long long);
  if (cudaMalloc(&d, bytes) != cudaSuccess) return set_error(SYMM_ERR_OOM, "trace buffer");
  cudaMemset(d, 0, bytes);
  CsArgs A = P->cargs;
  A.trace = d;
  A.trace_cap = cap;
  int rc = launch_zero(y, P->n, stream);
  if (!rc) rc = launch_cs(A, x, y, P->cs_grid, P->cs_nc, stream);
  cudaStreamSynchronize((cudaStream_t)stream);
  cudaMemcpy(host_trace, d, bytes, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return rc ? cuda_fail((cudaError_t)rc, "trace launch") : SYMM_OK;
}

// Diagnostics (not in the public header): statistics of the K5 format built
// from schedule s with window cap wcap and nnz cap nnzcap (no GPU needed).
// out[0..10] = tiles, Wcap, sum colours, sum slices, sum lane-steps
// (32 x longest row per slice), off-diagonal entries, sum spill targets,
// block bytes, max colours, sum rows, Scap.
extern "C" int symm_cs_format_stats(const race_schedule_t* s, int32_t wcap, int32_t chunk, int32_t stages, int32_t V,
                                    int64_t* out) {
  if (!s || !out) return set_error(SYMM_ERR_ARG, "NULL argument");
  const Schedule& S = s->S;
  CsHost H;
  int rc = build_cs_format(S, 0, (int32_t)S.tile_group.size(), wcap, 1 << 30, chunk, stages, V, &H);
  if (rc) return rc;
  int64_t rows = 0, heads = 0;
  for (const CsDesc& D : H.desc) { rows += D.T; heads += D.head_bytes; }
  int64_t v[13] = {(int64_t)H.desc.size(), H.Wcap, H.sum_colors, H.sum_slices, H.steps, H.nnz_offdiag, H.sum_spill,
                   (int64_t)H.blocks.size(), H.max_colour_chunks, rows, H.conflicts, heads, H.Hcap};
  for (int i = 0; i < 13; ++i) out[i] = v[i];
  return SYMM_OK;
}

// Diagnostics (not in the public header): the K5 format itself, for the CPU
// decoder test (tests/test_cs_format.py).  Call with NULL arrays to get
// sizes[0..2] = tiles, chunks, block bytes; then with arrays of those sizes.
extern "C" int symm_cs_format_dump(const race_schedule_t* s, int32_t wcap, int32_t chunk, int32_t stages, int32_t V,
                                   int64_t* sizes, void* desc, int64_t* chunk_off, int32_t* chunk_len,
                                   unsigned char* blocks) {
  if (!s || !sizes) return set_error(SYMM_ERR_ARG, "NULL argument");
  const Schedule& S = s->S;
  CsHost H;
  int rc = build_cs_format(S, 0, (int32_t)S.tile_group.size(), wcap, 1 << 30, chunk, stages, V, &H);
  if (rc) return rc;
  sizes[0] = (int64_t)H.desc.size();
  sizes[1] = (int64_t)H.chunk_off.size();
  sizes[2] = (int64_t)H.blocks.size();
  if (desc) std::memcpy(desc, H.desc.data(), H.desc.size() * sizeof(CsDesc));
  if (chunk_off) std::memcpy(chunk_off, H.chunk_off.data(), H.chunk_off.size() * sizeof(int64_t));
  if (chunk_len) std::memcpy(chunk_len, H.chunk_len.data(), H.chunk_len.size() * sizeof(int32_t));
  if (blocks) std::memcpy(blocks, H.blocks.data(), H.blocks.size());
  return SYMM_OK;
}

// Diagnostics / CPU tests: the K3/K4 tile blocks exactly as the plan would
// upload them (whole schedule, one rank).  sizes = {tiles, block bytes,
// runs, spill slots}; any output pointer may be NULL (sizes only).
extern "C" int symm_tiled_format_dump(const race_schedule_t* s, int64_t* sizes, void* desc, unsigned char* blocks,
                                      void* runs, int32_t* targets) {
  if (!s || !sizes) return set_error(SYMM_ERR_ARG, "NULL argument");
  TiledHost H;
  if (int rc = build_tiled_host(s->S, 0, (int32_t)s->S.tile_group.size(), H)) return rc;
  sizes[0] = (int64_t)H.desc.size();
  sizes[1] = (int64_t)H.blocks.size();
  sizes[2] = (int64_t)H.runs.size();
  sizes[3] = (int64_t)H.slot_tgt.size();
  if (desc) std::memcpy(desc, H.desc.data(), H.desc.size() * sizeof(TileDesc));
  if (blocks) std::memcpy(blocks, H.blocks.data(), H.blocks.size());
  if (runs) std::memcpy(runs, H.runs.data(), H.runs.size() * sizeof(SpillRun));
  if (targets) std::memcpy(targets, H.slot_tgt.data(), H.slot_tgt.size() * sizeof(int32_t));
  return SYMM_OK;
}

// ---- NEXT-4 sweeps (GS distance-1, KACZ distance-2) on the schedule --------
}  // extern "C"

struct symm_sweep {
  symmspmv_plan_t* P = nullptr;   // device buffers + device id
  int kind = 0;
  int32_t n = 0;
  int vec = 4;
  int32_t *d_rp = nullptr, *d_col = nullptr, *d_rows = nullptr;
  double* d_val = nullptr;
  std::vector<int32_t> rows, phase_ptr;
};

extern "C" {

int symm_sweep_plan(const race_schedule_t* s, int32_t kind, int32_t device, symm_sweep_t** out) {
  clear_error();
  if (!s || !out) return set_error(SYMM_ERR_ARG, "NULL argument");
  *out = nullptr;
  if (kind != SYMM_SWEEP_GS && kind != SYMM_SWEEP_KACZ) return set_error(SYMM_ERR_ARG, "sweep kind %d", kind);
  const Schedule& S = s->S;
  const int32_t n = S.n;
  // full matrix A' of the permuted order (CRS, columns ascending, diagonal included)
  std::vector<int64_t> cnt((size_t)n + 1, 0);
  for (int32_t r = 0; r < n; ++r)
    for (int32_t i = S.prow_ptr[(size_t)r]; i < S.prow_ptr[(size_t)r + 1]; ++i) {
      cnt[(size_t)r + 1]++;
      if (S.pcol[(size_t)i] != r) cnt[(size_t)S.pcol[(size_t)i] + 1]++;
    }
  for (int32_t r = 0; r < n; ++r) cnt[(size_t)r + 1] += cnt[(size_t)r];
  if (cnt[(size_t)n] >= ((int64_t)1 << 31)) return set_error(SYMM_ERR_OVERFLOW, "full matrix has >= 2^31 entries");
  std::vector<int32_t> rp((size_t)n + 1), col((size_t)cnt[(size_t)n]);
  std::vector<double> val((size_t)cnt[(size_t)n]);
  for (int32_t r = 0; r <= n; ++r) rp[(size_t)r] = (int32_t)cnt[(size_t)r];
  {
    std::vector<int32_t> pos(rp.begin(), rp.end() - 1);
    for (int32_t c = 0; c < n; ++c)
      for (int32_t i = S.prow_ptr[(size_t)c]; i < S.prow_ptr[(size_t)c + 1]; ++i) {
        const int32_t r = S.pcol[(size_t)i];
        if (r == c) continue;
        col[(size_t)pos[(size_t)r]] = c;
        val[(size_t)pos[(size_t)r]++] = S.pval[(size_t)i];
      }
    for (int32_t r = 0; r < n; ++r)
      for (int32_t i = S.prow_ptr[(size_t)r]; i < S.prow_ptr[(size_t)r + 1]; ++i) {
        col[(size_t)pos[(size_t)r]] = S.pcol[(size_t)i];
        val[(size_t)pos[(size_t)r]++] = S.pval[(size_t)i];
      }
  }
  if (kind == SYMM_SWEEP_GS)
    for (int32_t r = 0; r < n; ++r) {
      bool diag = false;
      for (int32_t i = rp[(size_t)r]; i < rp[(size_t)r + 1]; ++i) diag |= (col[(size_t)i] == r && val[(size_t)i] != 0.0);
      if (!diag) return set_error(SYMM_ERR_ARG, "Gauss-Seidel needs a nonzero diagonal (row %d of the permuted matrix)", r);
    }
  // colours inside every level group: greedy in row order; a row conflicts
  // with the earlier rows of its group at distance 1 (GS) or <= 2 (KACZ)
  const int32_t ng = (int32_t)S.group_workers.size();
  std::vector<int32_t> colour((size_t)n, 0), gof((size_t)n, 0), ncol((size_t)std::max(ng, 1), 0);
  for (int32_t g = 0; g < ng; ++g)
    for (int32_t r = S.level_ptr[(size_t)S.group_lvl[(size_t)g]]; r < S.level_ptr[(size_t)S.group_lvl[(size_t)g + 1]]; ++r)
      gof[(size_t)r] = g;
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t g = 0; g < ng; ++g) {
    const int32_t a = S.level_ptr[(size_t)S.group_lvl[(size_t)g]], b = S.level_ptr[(size_t)S.group_lvl[(size_t)g + 1]];
    std::vector<char> used;
    for (int32_t r = a; r < b; ++r) {
      std::fill(used.begin(), used.end(), 0);
      auto forbid = [&](int32_t q) {
        if (q >= a && q < r && gof[(size_t)q] == g) {
          const int32_t c = colour[(size_t)q];
          if ((size_t)c >= used.size()) used.resize((size_t)c + 1, 0);
          used[(size_t)c] = 1;
        }
      };
      for (int32_t i = rp[(size_t)r]; i < rp[(size_t)r + 1]; ++i) {
        const int32_t c = col[(size_t)i];
        forbid(c);
        if (kind == SYMM_SWEEP_KACZ)
          for (int32_t k = rp[(size_t)c]; k < rp[(size_t)c + 1]; ++k) forbid(col[(size_t)k]);
      }
      int32_t c = 0;
      while ((size_t)c < used.size() && used[(size_t)c]) ++c;
      colour[(size_t)r] = c;
      ncol[(size_t)g] = std::max(ncol[(size_t)g], c + 1);
    }
  }
  // Phases.  RACE stage-0 groups (scheme 0): groups of one parity are >= k
  // levels apart, so the colour-c rows of all red groups
  // form one phase, then those of the blue groups.  Any other schedule (MC /
  // ABMC colour classes, whose groups may be adjacent; recursive-tree leaves):
  // every (group, colour) is a phase of its own, groups in order.
  const bool merge = S.cfg.scheme == 0;
  std::vector<int32_t> gbase((size_t)ng + 1, 0);
  int32_t nc[2] = {0, 0};
  for (int32_t g = 0; g < ng; ++g) {
    nc[g & 1] = std::max(nc[g & 1], ncol[(size_t)g]);
    gbase[(size_t)g + 1] = gbase[(size_t)g] + ncol[(size_t)g];
  }
  auto phase_of = [&](int32_t r) {
    const int32_t g = gof[(size_t)r];
    if (!merge) return gbase[(size_t)g] + colour[(size_t)r];
    return (g & 1) ? nc[0] + colour[(size_t)r] : colour[(size_t)r];
  };
  symm_sweep_t* W = new symm_sweep_t();
  W->kind = kind;
  W->n = n;
  const int32_t np = merge ? nc[0] + nc[1] : gbase[(size_t)ng];
  W->phase_ptr.assign((size_t)np + 1, 0);
  for (int32_t r = 0; r < n; ++r) W->phase_ptr[(size_t)phase_of(r) + 1]++;
  for (int32_t p = 0; p < np; ++p) W->phase_ptr[(size_t)p + 1] += W->phase_ptr[(size_t)p];
  W->rows.assign((size_t)n, 0);
  {
    std::vector<int32_t> pos(W->phase_ptr.begin(), W->phase_ptr.end() - 1);
    for (int32_t r = 0; r < n; ++r) W->rows[(size_t)pos[(size_t)phase_of(r)]++] = r;  // ascending rows per phase
  }
  {
    const double avg = n > 0 ? (double)col.size() / n : 1.0;
    int v = 1;
    while (v < 32 && 2.0 * v <= avg / 1.5) v *= 2;
    W->vec = v;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  W->P = new symmspmv_plan_t();
  W->P->device = device;
  int rc;
  if ((rc = upload(W->P, &W->d_rp, rp.data(), rp.size())) || (rc = upload(W->P, &W->d_col, col.data(), col.size())) ||
      (rc = upload(W->P, &W->d_val, val.data(), val.size())) || (rc = upload(W->P, &W->d_rows, W->rows.data(), W->rows.size()))) {
    cudaSetDevice(cur);
    free_plan(W->P);
    delete W;
    return rc;
  }
  cudaSetDevice(cur);
  *out = W;
  return SYMM_OK;
}

int symm_sweep_run(symm_sweep_t* W, double* x, const double* b, int32_t symmetric, void* stream) {
  clear_error();
  if (!W || (W->n > 0 && (!x || !b))) return set_error(SYMM_ERR_ARG, "NULL argument");
  if ((const void*)x == (const void*)b) return set_error(SYMM_ERR_ALIAS, "x and b alias");
  const CsrArgs A{W->n, W->d_rp, W->d_col, W->d_val};
  const int32_t np = (int32_t)W->phase_ptr.size() - 1;
  for (int dir = 0; dir < (symmetric ? 2 : 1); ++dir)
    for (int32_t q = 0; q < np; ++q) {
      const int32_t p = dir == 0 ? q : np - 1 - q;  // backward sweep: phases in reverse
      const int32_t a = W->phase_ptr[(size_t)p], e = W->phase_ptr[(size_t)p + 1];
      int rc = launch_sweep_phase(W->kind, A, W->d_rows + a, e - a, b, x, W->vec, stream);
      if (rc) return cuda_fail((cudaError_t)rc, "k_sweep");
    }
  return SYMM_OK;
}

int symm_sweep_order(const symm_sweep_t* W, int32_t* rows, int32_t* phase_ptr, int32_t* nphases) {
  if (!W) return set_error(SYMM_ERR_ARG, "NULL sweep plan");
  if (nphases) *nphases = (int32_t)W->phase_ptr.size() - 1;
  if (rows) std::copy(W->rows.begin(), W->rows.end(), rows);
  if (phase_ptr) std::copy(W->phase_ptr.begin(), W->phase_ptr.end(), phase_ptr);
  return SYMM_OK;
}

int symm_sweep_destroy(symm_sweep_t* W) {
  if (!W) return SYMM_OK;
  free_plan(W->P);
  delete W;
  return SYMM_OK;
}

int symmspmv_plan_info(const symmspmv_plan_t* p, int32_t* out, int32_t n) {
  if (!p || !out) return set_error(SYMM_ERR_ARG, "NULL argument");
  int32_t v[8] = {p->variant, p->vec, p->tiled_grid, p->targs.stages, p->targs.block_cap, p->targs.window_cap,
                  p->tiled_nnz_cap, p->has_tiled ? tiled_smem_bytes(p->targs) : 0};
  int32_t m = n < 8 ? n : 8;
  for (int32_t i = 0; i < m; ++i) out[i] = v[i];
  return m;
}

int symmspmv_destroy(symmspmv_plan_t* p) {
  free_plan(p);
  return SYMM_OK;
}

}  // extern "C"
