// Internal declarations of libsymmspmv.so (product side; never includes or
// links anything under oracle/).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "symmspmv.h"

namespace symm {

// thread-local error message (symm_last_error)
int set_error(int code, const char* fmt, ...);
void clear_error();

// Host-side schedule (race_schedule_t).  Row ids are PERMUTED ids unless a
// field says "original".
struct Schedule {
  int32_t n = 0;
  int64_t nnz = 0;
  race_config cfg{};
  // §4.1 levels and permutation
  std::vector<int32_t> perm, inv;   // perm[old] = new, inv[new] = old
  std::vector<int32_t> dist;        // BFS level of every ORIGINAL vertex
  std::vector<int32_t> roots;       // original id of each island's start
  std::vector<int32_t> level_ptr;   // [totalLvl+1]
  // permuted upper CRS U' = upper(P A P^T), rows sorted
  std::vector<int32_t> prow_ptr, pcol;
  std::vector<double> pval;
  // §4.2-4.4.3 level groups
  std::vector<int32_t> windows;     // (first, end, b) per eps window
  std::vector<int32_t> group_lvl;   // T_ptr [n_groups+1]
  std::vector<int32_t> group_workers;
  // GPU tiles (contiguous row ranges inside level groups)
  std::vector<int32_t> tile_ptr;    // [n_tiles+1]
  std::vector<int32_t> tile_group, tile_phase, tile_order;
  std::vector<int32_t> dag_ptr, dag_pred;  // predecessors of every tile
  int32_t n_phases = 0;
  // intra-tile distance-2 row coloring; stored-row order per tile
  std::vector<int32_t> row_subcolor;  // [n]
  std::vector<int32_t> srow;          // [n] permuted row ids, per tile sorted by (color,row)
  std::vector<int32_t> tile_sub_ptr;  // [n_tiles+1] offsets into sub_ptr
  std::vector<int32_t> sub_ptr;       // per tile (nsub+1) stored-row offsets relative to tile start
  // per tile sorted unique targets outside its own rows; bit 31 = first writer
  std::vector<int64_t> spill_ptr;     // [n_tiles+1]
  std::vector<int32_t> spill;
  std::vector<uint8_t> own_first;     // [n] tile writes row first (stores, not adds)
  int32_t max_subcolors = 0, max_window = 0, max_rows = 0;
  double mean_subcolors = 0.0;
  int64_t bw_before = 0, bw_after = 0;
  double eta = 1.0;
  double build_seconds = 0.0;
  // NEXT-2 recursive RACE tree (race_config.scheme == 3; §4.4.1-4.4.2):
  // node 0 = T_{-1}(0) (all rows), its children the stage-0 level groups,
  // deeper nodes the level groups T_{s+1} found inside a T_s with > 1 worker.
  // Rows of every node are contiguous [tree_r0, tree_r1); the children of a
  // node alternate red (even tree_cidx) / blue (odd).  Leaves = the level
  // groups of the final schedule (group g <-> node tree_leaf[g]).
  std::vector<int32_t> tree_parent, tree_cidx, tree_r0, tree_r1, tree_stage, tree_workers;
  std::vector<int32_t> tree_leaf;   // [n_groups] leaf node of every group (position order)
  double tree_eta = 0.0;            // §5 eta of the tree (rows as the workload)
};

// Paper-algorithm building blocks (exposed for white-box tests through
// race_schedule_table; kept identical in decision order to the cited text).
std::vector<int32_t> eps_aggregate(const std::vector<int64_t>& level_work, int64_t nthreads, int k,
                                   double eps);
int32_t split_window(const std::vector<int64_t>& level_work, int32_t first, int32_t end, int k);
void alg4_balance(std::vector<int32_t>& T_ptr, const std::vector<int32_t>& worker,
                  const std::vector<int64_t>& level_work, int kmin);

int build_schedule(const symm_csr_upper* U, const race_config* cfg, Schedule* S);

// ---- device side -----------------------------------------------------------
constexpr uint32_t kFirstBit = 0x80000000u;
constexpr uint32_t kIdxMask = 0x7fffffffu;

// One tile of the streaming tiled kernels (K3 deterministic / K4 atomic).
// The tile's block (one cp.async.bulk into shared memory) holds, 16-B aligned:
//   TileDesc (64 B) | rseg u32[T] | lcol u16[nnz] | tcsc u32[noff] |
//   tptr u16[W+1] | [sid u16[W]] | tgt i32[S] | val f64[nnz]
// rseg: own row l's entries are [start, start + len) of lcol / val, packed
// start | len << 16; the segments of a warp's rows are placed (with unused pad
// entries counted in nnz) so that the rows of each half warp start on distinct
// bank pairs; lcol: local column of each entry (own rows 0..T-1, then spill
// targets T..W-1);
// tcsc/tptr: the off-diagonal entries grouped by local target (CSC of the
// tile), each as (entry index | local row << 16), one list per lane
// position i (tptr[i] .. tptr[i+1]); sid (sorted tiles only): the window
// slot of lane position i, positions sorted by descending work (row entries
// + transposed entries) so the lanes of a warp have similar list lengths;
// unsorted tiles: position i is slot i.  tgt: global row of each spill
// target.  K3's staging slots live outside the block (`slots`).
struct TileDesc {
  int64_t block_off;    // byte offset of the block
  int32_t block_bytes;  // multiple of 16, < 65536
  int32_t nrows;        // T
  int32_t nspill;       // S = spill window slots (window W = T + S): the spill targets
                        // laid out run by run, a run of consecutive rows starting on a slot
                        // of the same 16-B parity as its first row (bulk-copyable); pad slots
                        // have target -1
  int32_t nnz;          // stored entries of the tile
  int32_t row0;         // first own row (permuted id)
  uint16_t o_lcol, o_tidx, o_tptr, o_tgt, o_sid, o_val;  // byte offsets in the block
  int32_t spill_off;    // first spill slot of this tile (targets / slots arrays)
  int32_t run_off;      // first run of this tile (runs array)
  int32_t nruns;        // runs of consecutive spill targets
  int32_t gather_runs;  // bit 0: the gather warps bulk-copy the runs (long runs); else they
                        // cp.async slot by slot from the block's tgt list (short runs).
                        // bit 1: single-run tile -- the spill window is ONE run of consecutive
                        // rows (every tile of a stencil in BFS order), so the block carries no
                        // tgt[]: window slot l >= T + (bit 2) flushes to row tgt_base + l, the
                        // slot before it (bit 2: one parity pad) to nothing
  int32_t sorted;       // 1: lanes take the window slots in the order sid[] (work-sorted)
  int32_t tgt_base;     // single-run tiles: first row of the run - its window id
};
static_assert(sizeof(TileDesc) == 64, "TileDesc must be 64 B");

struct SpillRun {                 // consecutive spill targets row .. row+len-1 at window ids wid..
  int32_t row, wid, len, pad;
};

// Unroll factor of K3/K4's per-lane row and transposed loops over unsorted
// tiles.  nvcc runs a lane's (n % unroll) leftover steps first, and the
// builder keys its bank placement on that (capi.cpp).  Measured (same box,
// ms, st27 / spin / lap3d_256 / fem): unroll 4: 0.0941 / 0.2027 / 0.2590 /
// 0.2016; unroll 2: 0.0926 / 0.2027 / 0.2584 / 0.2014; unroll 1: 0.0927 /
// 0.2022 / 0.2554 / 0.2080; unroll 8: 0.0943 / 0.2030 / 0.2586 / 0.2081.
// Keep the pragmas in kernels.cu in step.
constexpr int kK4Unroll = 2;
// Unroll factor of the sorted tiles' record loop (blocks first, leftovers
// last; the builder's transposed-list order follows it).  fem: unroll 4
// 0.2004, 2 0.1991, 8 0.2002 ms.
constexpr int kK4SortedUnroll = 2;
// K8 (tiled_colored) keeps a thread's slot sums in registers until the tile's
// DAG predecessors have flushed: at most kK8Slots slots per thread, i.e.
// window_cap <= kK8Slots * 224 (checked at plan time).
constexpr int kK8Slots = 8;

struct K8Args {                   // (K3 / K8 tables, device memory)
  const int32_t* slots;           // K3: staging slot of every spill slot (tile order, -1 = pad)
  double* spill_buf;              // K3: staged contributions to other tiles' rows
  // K8 (tiled_colored, MODE 2): tiles processed in phase-major order; a tile
  // flushes after its DAG predecessors (conflicting tiles of earlier phases)
  const int32_t* order;           // [ntiles] processing order -> tile id
  const int32_t* dag_ptr;         // [ntiles+1] predecessors of every tile id
  const int32_t* dag_pred;
  const int32_t* pos_meta;        // [4 ntiles] by position: (tile id, dag_ptr[id], dag_ptr[id+1], 0), 16-B aligned
  unsigned int* done;             // [ntiles] warps of the owning group that flushed (zeroed per run)
  const uint8_t* own_first;       // [n] K8: the row's own tile writes it first (stores)
  const uint8_t* slot_first;      // [spill slots] K8: this spill slot's tile writes its target first
  // K4 (MODE 1) zeroes y itself (kernels.cu k4_zero_y): monotonic launch
  // counter, +gridDim.x per launch, never reset
  unsigned long long* zero_ctr;   // nullptr: y is zeroed by k_zero before the launch
  int64_t zero_begin, zero_end;   // global row ids of the local y range
  int32_t zero_dbg;               // diagnostics (env SYMM_ZERO_DBG): bit0 no stores, bit1 no wait
};


struct TiledArgs {
  const TileDesc* tiles;          // tile id order (= BFS order)
  int32_t ntiles;
  const unsigned char* blocks;
  const struct K8Args* k8;        // K3 / K8 tables, device memory.  Kept out of the kernel
                                  // parameters: 48 more bytes of TiledArgs made K3/K4 1.5-2.7%
                                  // slower, 24 fewer made st27 0.6% faster (measured, same blocks)
  const struct SpillRun* runs;    // every spill run of every tile (tile order)
  int32_t block_cap, window_cap;
  int32_t stages;                 // smem ring depth (chosen at plan time)
  int32_t debug_skip;             // diagnostics only (env SYMM_DEBUG_SKIP): skip bit0 row part,
                                  // bit1 CSC part, bit2 flush, bit3 spill-x gather (wrong results)
#if defined(K4_CHECK) || defined(K4_TRACE)
  int32_t check_n;                // K4_CHECK builds: length of the x / y vectors
  unsigned long long* trace;      // K4_TRACE builds: per-tile event times of CTA 0 (nullptr = off)
#endif
  // (kept small on purpose: every byte of kernel parameters counts, see k8)
};

struct FixupArgs {                // K3 second kernel: y[r] += sum of staged contributions
  int32_t n;
  const int32_t* in_ptr;          // [n+1] slots of row r: in_ptr[r] .. in_ptr[r+1]
  const double* spill_buf;
};

struct CsrArgs {
  int32_t n;
  const int32_t* row_ptr;
  const int32_t* col;
  const double* val;
};

struct ColoredArgs {
  const int32_t* tile_ptr;     // [n_tiles+1] row ranges (permuted ids)
  const int32_t* phase_tiles;  // tiles of the phase being launched
  int32_t nphase_tiles;
  const int32_t* srow;         // stored rows (global ids), per tile colour-sorted
  const int32_t* tile_sub_ptr; // offsets into sub_ptr per tile
  const int32_t* sub_ptr;      // per tile colour pointers, relative to tile row start
};

// ---- K7 tree (scheme 3): leaves in execution order (red subtrees before blue)
struct TreeArgs {
  int32_t nleaves, nnodes;
  const int32_t* leaf_t0;      // [nleaves] tiles [leaf_t0[i], leaf_t1[i]) of leaf i (execution order)
  const int32_t* leaf_t1;
  const int32_t* wait_ptr;     // [nleaves+1] into wait_node
  const int32_t* wait_node;    // nodes whose red-subtree leaves leaf i waits for
  const int32_t* sig_ptr;      // [nleaves+1] into sig_node
  const int32_t* sig_node;     // nodes whose red-leaf counter leaf i increments
  const int32_t* red_total;    // [nnodes] leaves under the red children of every node
  int32_t* counters;           // [nnodes + 1]; the last one is the claim counter (zeroed per run)
};
int launch_tree(const CsrArgs& A, const ColoredArgs& C, const TreeArgs& T, const double* x, double* y, int vec,
                int grid, void* stream);

// ---- NEXT-4 sweeps: one launch per phase, V lanes per row of the full matrix
int launch_sweep_phase(int kind, const CsrArgs& A, const int32_t* rows, int32_t nrows, const double* b, double* x,
                       int vec, void* stream);

// ---- K5 colored_smem (cs_build.cpp / kernels.cu) ------------------------------
// One tile = consecutive schedule tiles of one level group; rows coloured by
// write sets (RACE distance-2) and executed colour by colour
// inside a shared-memory window of x and y (see cs_build.cpp for the block).
constexpr int kCsReleaseUnits = 4096;  // ring_empty arrivals per chunk (piece weights sum to it)
struct CsDesc {      // global descriptor of one tile (read by the head producer)
  int64_t head_off;  // byte offset of the tile's head in `blocks`
  int32_t head_bytes, row0, T, S, ncolors, nslices, npieces, nchunks;
  int32_t block_bytes;  // head + chunks (the tile's block is contiguous)
  uint16_t o_cslc, o_srec, o_ploc, o_pw, o_tgt, o_clen, pad[4];
};
static_assert(sizeof(CsDesc) == 64, "CsDesc must be 64 B");
struct CsHeadHdr {   // first bytes of every head (read from shared memory)
  int64_t chunk_base;  // byte offset of the tile's first chunk in `blocks` (chunks are contiguous)
  int32_t row0, T, S, ncolors, nslices, npieces, nchunks;
  uint16_t o_cslc, o_srec, o_ploc, o_pw, o_tgt, o_clen;
  int32_t pad[4];
};
static_assert(sizeof(CsHeadHdr) == 64, "CsHeadHdr must be 64 B");
struct CsSliceRec {  // one slice (<= 32 rows of one colour), 16 B
  uint32_t ploc0;    // location of its first piece ((chunk in tile << 20) | offset)
  uint16_t p0;       // index of its first piece
  uint16_t nsteps;   // longest row (off-diagonal entries) = JDS steps
  uint8_t npieces, m, pad[6];
};
static_assert(sizeof(CsSliceRec) == 16, "CsSliceRec must be 16 B");

struct CsHost {
  std::vector<CsDesc> desc;
  std::vector<int64_t> chunk_off;   // byte offset of every chunk (tiles in order)
  std::vector<int32_t> chunk_len;   // bytes of every chunk (multiple of 16)
  std::vector<int32_t> tile_chunk0; // first chunk of every tile
  std::vector<unsigned char> blocks;
  int32_t Wcap = 16, Hcap = 16, max_colour_chunks = 1;
  int64_t nnz_offdiag = 0, sum_colors = 0, sum_slices = 0, sum_spill = 0, conflicts = 0, steps = 0;
};
// Bank-aware step order of the rows of one warp (cs_build.cpp): entry lists
// (window id, value) reordered so that at each step the lanes of a half warp
// address distinct shared-memory bank pairs (window id mod 16).
int64_t bank_order_rows(std::vector<std::vector<std::pair<uint16_t, double>>>& ent, int V);
int32_t color_rows_writeset(const int32_t* rp, const int32_t* pc, int32_t r0, int32_t r1,
                            const std::vector<int32_t>& tgt, std::vector<int32_t>& color);
int build_cs_format(const Schedule& S, int32_t t_begin, int32_t t_end, int32_t wcap, int32_t nnzcap,
                    int32_t chunk_bytes, int32_t stages, int32_t V, CsHost* out);

struct CsArgs {
  const CsDesc* desc;
  int32_t ntiles;
  const unsigned char* blocks;
  const int64_t* chunk_off;
  const int32_t* chunk_len;
  int32_t Wcap, Hcap;             // window entries, head bytes (capacities of the smem buffers)
  int32_t chunk;                  // bytes of one ring stage
  int32_t stages;                 // ring depth (power of two)
  int32_t lgstages;               // log2(stages)
  int32_t lgv;                    // log2 of the lanes per row (1, 2 or 4 lanes)
  int32_t debug_skip;             // diagnostics (env SYMM_DEBUG_SKIP): bit0 entries, bit2 flush, bit3 stream only
  unsigned long long* trace;      // diagnostics: CTA 0 event times (nullptr = off), see k_cs
  int32_t trace_cap;              // chunk events [0, cap) x 2, then tile events x 4
};
int cs_smem_bytes(const CsArgs& A);
int cs_configure(CsArgs& A, int* ctas_per_sm, int nc);   // sets the smem attribute, returns occupancy
int launch_cs(const CsArgs& A, const double* x, double* y, int grid, int nc, void* stream);

// full-matrix SpMV (Alg. 1) on the mirrored permuted CRS
int launch_spmv(const CsrArgs& A, const double* x, double* y, int vec, int sms, void* stream);

// kernel launchers (kernels.cu); return cudaError_t as int
int launch_zero(double* y, int64_t n, void* stream);
int launch_atomic(const CsrArgs& A, const double* x, double* y, int vec, int sms, void* stream);
int launch_colored_phase(const CsrArgs& A, const ColoredArgs& C, const double* x, double* y, int vec,
                         void* stream);
int launch_tiled(const TiledArgs& T, const double* x, double* y, int vec, int grid, int mode, void* stream);
int launch_fixup(const FixupArgs& F, double* y, void* stream);
int tiled_smem_bytes(const TiledArgs& T);
int tiled_max_ctas_per_sm(int vec, const TiledArgs& T, int* out);  // returns the ring depth in *out
int launch_gather(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream);
int launch_scatter(const double* src, const int32_t* idx, double* dst, int64_t n, void* stream);
int launch_add(double* y, const double* v, int64_t n, void* stream);
int bw_probe(int mode, int64_t bytes, int reps, void* stream, double* gbps);  // K5 (returns cudaError_t)

}  // namespace symm
