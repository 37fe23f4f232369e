/* symmspmv.h — C ABI of the B200 SymmSpMV library (libsymmspmv.so).
 *
 * Operation (the hot path this library exists for): SymmSpMV
 * (§3.2, Alg. 2 alg:SymmSpMV): given the upper triangle U (diagonal included)
 * of a symmetric sparse matrix A = U + U^T - diag(U) in CRS with 8-byte values
 * and 4-byte indices, compute
 *
 *        y := A x        (every stored a_ij, i < j, updates y_i += a_ij x_j
 *                         and y_j += a_ij x_i; the diagonal contributes once)
 *
 * Alg. 2 accumulates into b with `+=`; this ABI overwrites
 * y (reading R2).  Rows without a stored diagonal are accepted and
 * contribute no diagonal term (reading R1).
 *
 * The RACE preprocessing (§4) that makes SymmSpMV parallel
 * without write conflicts lives in race_build_schedule(): BFS levels (§4.1,
 * Alg. 3), level permutation, distance-k level groups (§4.2), epsilon level
 * aggregation (§4.4.3) and Alg. 4 load balancing (§4.3), then the GPU
 * adaptation: contiguous tiles per level group, exact tile write-conflict
 * coloring and intra-tile distance-2 row coloring.
 *
 * Conventions for every call:
 *   - 0-based indices, half-open ranges.
 *   - Return value: SYMM_OK (0) or a negative symm_status.  On error nothing
 *     is allocated / nothing is launched; symm_last_error() returns a
 *     thread-local message naming the first offending row/column.
 *   - "HOST" pointers are read during the call only; the library copies what
 *     it keeps.  "DEVICE" pointers must be device memory of the plan's device.
 *   - No call takes or returns a torch type.
 */
#ifndef SYMMSPMV_H
#define SYMMSPMV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SYMM_OK = 0,
  SYMM_ERR_ARG = -1,        /* NULL / negative size / bad option value            */
  SYMM_ERR_NOT_UPPER = -2,  /* a stored col < row, or col >= n                    */
  SYMM_ERR_UNSORTED = -3,   /* columns of a row not strictly ascending (dups)     */
  SYMM_ERR_OVERFLOW = -4,   /* nnz >= 2^31 or n >= 2^31 (int32 CRS) */
  SYMM_ERR_OOM = -5,        /* host or device allocation failed                   */
  SYMM_ERR_CUDA = -6,       /* a CUDA runtime call failed (message has the error) */
  SYMM_ERR_NCCL = -7,       /* multi-GPU communicator failure                     */
  SYMM_ERR_MISMATCH = -8,   /* matrix does not match the schedule it is used with */
  SYMM_ERR_ALIAS = -9,      /* x and y overlap                                    */
  SYMM_ERR_SCHEDULE = -10,  /* internal schedule validator failed (a bug)         */
  SYMM_ERR_K = -11,         /* distance k < 2 requested for SymmSpMV*/
  SYMM_ERR_UNSUPPORTED = -12/* variant cannot run this matrix (e.g. tile > smem)  */
} symm_status;

/* Upper-triangular CRS (double A[nnz]; int col[nnz],
 * rowPtr[nrows+1]).  HOST pointers, caller-owned.  row_ptr[0] = 0,
 * row_ptr[n] = nnz, col[row_ptr[r]..row_ptr[r+1]) strictly ascending, all >= r. */
typedef struct {
  int32_t n;
  int64_t nnz;
  const int32_t* row_ptr;
  const int32_t* col;
  const double* val;
} symm_csr_upper;

/* Schedule-builder options (defaults from race_config_default). */
typedef struct {
  int32_t k;                /* distance of the coloring; SymmSpMV needs 2 */
  int32_t n_workers;        /* workers (GPU tiles) for eps aggregation; 0 = derive from work  */
  int32_t tile_work;        /* target work per tile when n_workers == 0 (nnz + 2 rows units) */
  int32_t balance_by;       /* 0 = rows, 1 = nnz + 2 rows                */
  int32_t root;             /* BFS root of the first island; -1 = pseudo-peripheral           */
  int32_t n_eps;            /* number of valid eps[] entries                                 */
  double eps[8];            /* eps_s per stage (0.8, 0.8, 0.5 ...)             */
  int32_t max_tile_rows;    /* hard cap on rows per tile (<= 65535)                          */
  int32_t max_tile_window;  /* cap on |own rows ∪ targets| per tile (smem entries)           */
  int32_t max_tile_nnz;     /* cap on stored entries per tile (smem staging of the tile)     */
  int32_t reorder;          /* 1 = BFS level permutation; 2 = RCM levels
                               (Cuthill-McKee within-level order, whole order reversed,
                               PAPER.md:1052-1053, 2026, 2047; needs cone_tiles = 0);
                               0 = keep order */
  int32_t cone_tiles;       /* 0 = contiguous tiles (default); 1/2 = tiles are cones across the
                               levels of their level group (1: proportional cuts, 2: cuts
                               follow BFS discovery), rows re-permuted inside the group */
  int32_t min_group_levels; /* >= k: minimum levels per level group ("at least k") */
  int32_t validate;         /* 1 = run the write-set stamping validator (always cheap)       */
  uint32_t flags;           /* bit 0: within-level order = original index (experimental);
                               bit 1: tile phases follow the stage-0 colours (red groups' tiles,
                               then blue, greedy; default for scheme 0 is DSatur over all tiles);
                               bit 2: keep the DSatur colour sizes (default: rebalanced towards
                               equal phase sizes, a proper colouring still) */
  int32_t scheme;           /* 0 = RACE (levels, groups, tiles: the default);
                               3 = RACE with the recursive tree (§4.4.1-4.4.2):
                                   level groups with > 1 worker refined stage by stage on their
                                   distance-1-extended subgraphs; leaves become the level groups;
                                   workers = n_workers (0: 8 x 148); needs reorder >= 1,
                                   cone_tiles = 0; run by the `tree` variant (or any other);
                               1 = MC: greedy distance-2 (write-set) colouring of single rows,
                                   rows ordered colour by colour;
                               2 = ABMC: blocks of `abmc_block` consecutive BFS-ordered rows,
                                   blocks coloured by their write sets and ordered colour by colour
                                   (contiguous blocks stand in for METIS parts).
                               MC / ABMC colour classes become the level groups and phases; they
                               exist to reproduce the paper's comparison. */
  int32_t abmc_block;       /* rows per ABMC block (default 64)                               */
} race_config;

typedef struct race_schedule race_schedule_t;

typedef struct {
  int32_t n, total_levels, n_components, n_groups, n_tiles, n_phases;
  int32_t max_subcolors, max_tile_window, max_tile_rows, n_dag_edges;
  int64_t nnz, bandwidth_before, bandwidth_after;
  double eta;               /* §5 parallel efficiency of the tile tree (work = balance unit) */
  double build_seconds;
  double mean_subcolors;
  int64_t spill_entries;    /* sum over tiles of |targets outside own rows|                 */
} race_schedule_stats;

void race_config_default(race_config* cfg);

/* Builds the RACE schedule for U (HOST).  *out is owned by the caller until
 * race_schedule_destroy.  Deterministic: same U + cfg => same schedule. */
int race_build_schedule(const symm_csr_upper* U, const race_config* cfg, race_schedule_t** out);
int race_schedule_get_stats(const race_schedule_t* s, race_schedule_stats* out);

/* perm_old2new[old] = new, inv_new2old[new] = old (HOST int32[n] each, caller-allocated). */
int race_schedule_permutation(const race_schedule_t* s, int32_t* perm_old2new, int32_t* inv_new2old);

/* Generic table access for tests/tools.  `which` names one int32 table; the
 * call returns its length in *len and copies it to out when out != NULL.
 *   "level_ptr"   [total_levels+1] row ranges of L(i) in the permuted order
 *   "dist"        [n] BFS level of every ORIGINAL vertex (Eq. 5)
 *   "roots"       [n_components] start vertex (original id) of every island
 *   "group_lvl"   [n_groups+1] level-group pointers T_ptr
 *   "group_workers" [n_groups] tiles per group (eps aggregation b)
 *   "tile_ptr"    [n_tiles+1] row ranges of tiles (permuted order)
 *   "tile_group"  [n_tiles] level group of each tile
 *   "tile_phase"  [n_tiles] phase = stage-0 color * C + tile color
 *   "tile_order"  [n_tiles] claim order of the dataflow kernel (topological)
 *   "dag_ptr"/"dag_pred" predecessor tiles (CSR over tiles)
 *   "row_subcolor" [n] intra-tile color of every permuted row
 *   "window_levels" [3*n_windows] (first, end, b) of the eps windows           */
int race_schedule_table(const race_schedule_t* s, const char* which, int64_t* len, int32_t* out);

/* Permuted upper CRS U' = upper(P A P^T) the plan uses (HOST, caller-allocated:
 * row_ptr[n+1], col[nnz], val[nnz]); any pointer may be NULL to skip it. */
int race_schedule_permuted_matrix(const race_schedule_t* s, int32_t* row_ptr, int32_t* col, double* val);
void race_schedule_destroy(race_schedule_t* s);

/* Multi-GPU row-block split of the permuted order (R23):
 * whole tiles are assigned to ranks contiguously, balanced by stored
 * nonzeros.  row_bounds[nranks+1] (HOST, caller-allocated): rank r owns rows
 * [row_bounds[r], row_bounds[r+1]).  halo_end[nranks]: rank r's tiles read x
 * and write y only inside [row_bounds[r], halo_end[r]) (halo_end[r] >=
 * row_bounds[r+1]; every stored entry points forward, c >= r, so the halo
 * lies in later ranks).  Either output may be NULL. */
int race_schedule_partition(const race_schedule_t* s, int32_t nranks, int32_t* row_bounds, int32_t* halo_end);

/* ---- execution ---------------------------------------------------------- */
typedef enum {
  SYMM_VARIANT_AUTO = 0,    /* tiled_atomic if every tile fits, else colored          */
  SYMM_VARIANT_COLORED = 1, /* K2: one launch per phase, global read-modify-write     */
  SYMM_VARIANT_ATOMIC = 2,  /* K1: one launch, native fp64 RED for transposed updates */
  SYMM_VARIANT_TILED = 3,   /* K3: TMA-staged tiles, smem two-pass, staged fixup; deterministic */
  SYMM_VARIANT_TILED_ATOMIC = 4,/* K4: same tiles, window flushed with fp64 RED into zeroed y */
  SYMM_VARIANT_COLORED_SMEM = 5,/* K5: RACE write-set colours run inside a shared-memory x/y window
                                   (plain smem read-modify-write, one barrier per colour); window
                                   flushed with fp64 RED into zeroed y                        */
  SYMM_VARIANT_SPMV = 6,        /* the paper's yardstick (Alg. 1): the same y := A x
                                   from the FULL matrix A = U + U^T - diag(U) in CRS, the plan
                                   mirrors U; deterministic, no atomics   */
  SYMM_VARIANT_TILED_COLORED = 8,/* K8: the K4 tiles in one launch, processed phase by phase
                                   (phase-major order); a tile flushes its window after its
                                   DAG predecessors (conflicting tiles of earlier phases) have:
                                   the first writer of a row stores, later writers add in phase
                                   order.  No atomics, no zeroing of y, deterministic; the
                                   colored scheme at streaming speed        */
  SYMM_VARIANT_TREE = 7         /* K7: the recursive RACE tree (schedule scheme 3 only, else
                                   SYMM_ERR_ARG) in one persistent launch: one CTA per leaf at a
                                   time, leaves claimed in red-before-blue depth-first order,
                                   tree-scoped sync through per-node counters (a blue child waits
                                   for the leaves of its red siblings),
                                   plain read-modify-write of y as in COLORED; deterministic    */
} symm_variant;

typedef enum { SYMM_ORDER_PERMUTED = 0, SYMM_ORDER_ORIGINAL = 1 } symm_vec_order;

typedef struct {
  int32_t variant;          /* symm_variant                                             */
  int32_t device;           /* CUDA device ordinal                                      */
  int32_t vec_order;        /* symm_vec_order of x/y passed to symmspmv_run              */
  int32_t nranks, rank;     /* multi-GPU row-block split (1, 0 = single GPU)            */
  int32_t vec_width;        /* lanes per row (1,2,4,8,16,32); 0 = from SymmNNZR          */
  int32_t ctas_per_sm;      /* persistent grid of the tiled kernel; 0 = default         */
  int32_t build_all;        /* 1 = upload tables of every variant (tests)               */
} symmspmv_options;

typedef struct symmspmv_plan symmspmv_plan_t;

void symmspmv_options_default(symmspmv_options* o);

/* Uploads the schedule's permuted matrix and tables to o->device.  The plan
 * owns all device memory it allocates; s may be destroyed afterwards.  U must
 * be the matrix s was built from (checked: n, nnz; else SYMM_ERR_MISMATCH). */
int symmspmv_plan(const race_schedule_t* s, const symm_csr_upper* U, const symmspmv_options* o,
                  symmspmv_plan_t** out);

/* This rank's row slice [row_begin, row_end) of the permuted order. */
int symmspmv_plan_rows(const symmspmv_plan_t* p, int32_t* row_begin, int32_t* row_end);

/* Rows covered by the x / y vectors symmspmv_run expects on this rank:
 * [row_begin, local_end) with local_end = halo_end of the partition (n for a
 * single rank).  For nranks > 1 (variant TILED_ATOMIC only), symmspmv_run
 * reads x over that range and writes y over it: own rows [row_begin,
 * row_end) hold this rank's contributions, [row_end, local_end) the
 * contributions to later ranks' rows, which the caller sends to their owners
 * and adds (paper_1907_06487_b200/dist.py). */
int symmspmv_plan_local(const symmspmv_plan_t* p, int32_t* row_begin, int32_t* local_end);

/* y[i] += v[i], i < n (DEVICE pointers, `stream`): the owner-side add of halo
 * contributions received from earlier ranks (SURVEY §2.5 K4 halo_add_y). */
int symmspmv_halo_add(double* y_dev, const double* v_dev, int64_t n, void* stream);

/* y := A x on `stream` (a cudaStream_t; NULL = default stream), asynchronous.
 * x_dev, y_dev: DEVICE fp64[n] in the plan's vec_order; must not overlap
 * (SYMM_ERR_ALIAS).  `variant` overrides the plan's variant when >= 0 (it
 * must have been uploaded).  Not re-entrant per plan (one run at a time). */
int symmspmv_run(symmspmv_plan_t* p, const double* x_dev, double* y_dev, void* stream);
int symmspmv_run_variant(symmspmv_plan_t* p, int32_t variant, const double* x_dev, double* y_dev,
                         void* stream);

/* Matrix powers ("in-place matrix powers and polynomials",
 * PAPER.md:2344-2348): Y_dev row k (k = 0 .. npow-1, row stride ldy >= n
 * doubles) := A^(k+1) x.  x_dev, Y_dev: DEVICE fp64 in the plan's vec_order,
 * caller-owned, x must not overlap Y (SYMM_ERR_ALIAS).  Each power is one
 * SymmSpMV of the previous one with `variant` (< 0: the plan's), all on
 * `stream`, asynchronous.  Single-rank plans only (SYMM_ERR_UNSUPPORTED);
 * npow < 0 or ldy < n: SYMM_ERR_ARG; npow = 0 does nothing. */
int symmspmv_powers(symmspmv_plan_t* p, int32_t variant, const double* x_dev, double* Y_dev, int32_t npow,
                    int64_t ldy, void* stream);

/* Halo overlap for multi-rank plans.  A rank's
 * tiles split into INTERIOR tiles (every row they read or write is an own row,
 * < row_end) and BOUNDARY tiles (their window reaches halo rows >= row_end).
 *   part = SYMM_PART_INTERIOR: zero y over [row_begin, local_end) and run the
 *          interior tiles (needs only the rank's own x);
 *   part = SYMM_PART_BOUNDARY: run the boundary tiles (needs the x halo);
 *          must follow the INTERIOR part on the same y (stream-ordered);
 *   part = SYMM_PART_ALL: both (= symmspmv_run).
 * The caller receives the x halo while the interior part runs.  Single-rank
 * plans hold every tile as interior (BOUNDARY is a no-op).  x / y as for
 * symmspmv_run, permuted order only; variant tiled_atomic (multi-rank plans)
 * or the plan's variant (single rank, part ALL / INTERIOR). */
typedef enum { SYMM_PART_ALL = 0, SYMM_PART_INTERIOR = 1, SYMM_PART_BOUNDARY = 2 } symm_part;
int symmspmv_run_part(symmspmv_plan_t* p, int32_t part, const double* x_dev, double* y_dev, void* stream);
/* Tile and stored-nonzero counts of the two parts (any pointer may be NULL). */
int symmspmv_plan_parts(const symmspmv_plan_t* p, int32_t* n_interior_tiles, int32_t* n_boundary_tiles,
                        int64_t* nnz_interior, int64_t* nnz_boundary);

/* K5 bandwidth probe: the measured roofline denominators (PAPER.md:440-456:
 * the paper measures load-only and copy bandwidth and uses both, Eq. 1).
 * mode 0 = load-only (16-B streaming loads, result folded into a never-true
 * store), mode 1 = copy (dst := src, bytes counted read + write).  Allocates
 * `bytes` (mode 0) or 2 x bytes (mode 1) on `device`, runs one warm-up and
 * `reps` timed passes on `stream` (CUDA events), frees the memory and returns
 * the best pass in *gbps (GB/s, 1e9).  SYMM_ERR_OOM if the allocation fails. */
int symm_bw_probe(int32_t mode, int32_t device, int64_t bytes, int32_t reps, void* stream, double* gbps);

/* End-to-end convenience: x_host, y_host are HOST fp64[n] in ORIGINAL order
 * (pinned memory recommended).  H2D copy, permute, run, unpermute, D2H copy,
 * all on `stream`; returns after the stream has been synchronised. */
int symmspmv_run_host(symmspmv_plan_t* p, const double* x_host, double* y_host, void* stream);

/* Number of kernel launches the last symmspmv_run issued (evidence for bench). */
int symmspmv_last_launches(const symmspmv_plan_t* p);

/* Device bytes the plan holds, and the algorithmic bytes of one multiply for
 * the chosen variant (12 nnz + 4 (n+1) + 24 n). */
int symmspmv_plan_bytes(const symmspmv_plan_t* p, int64_t* device_bytes, int64_t* min_bytes);

/* Launch configuration of the plan (diagnostics): out[0..7] = default variant,
 * lanes per row, tiled grid, tiled smem ring depth, tile block cap (B),
 * tile window cap, tile nnz cap, tiled dynamic smem (B).  Returns the count. */
int symmspmv_plan_info(const symmspmv_plan_t* p, int32_t* out, int32_t n);

int symmspmv_destroy(symmspmv_plan_t* p);

/* ---- NEXT-4: distance-k iterative sweeps on the same schedule --------------
 * SURVEY §8f NEXT-4; the kernels appear in PAPER.md's draft text only
 * (Gauss-Seidel, distance-1; Kaczmarz, distance-2, "For its
 * parallelization one typically uses a distance-2 coloring").  The schedule's
 * level groups already separate same-colour groups by distance >= 3
 * (PAPER.md:1227-1229); inside every level group the plan colours the rows
 * greedily, in row order, so that rows of one colour are distance-1 (GS) or
 * distance-2 (KACZ) independent in the FULL graph of A.  A sweep runs phase by
 * phase: the red groups' colour 0, 1, ..., then the blue groups' colours; a
 * backward sweep runs the phases in reverse.  Rows of one phase commute, so
 * the result equals a serial sweep in the plan's row order
 * (symm_sweep_order), bit for bit up to the summation order inside a row.
 *   GS   (kind 1): x_r := (b_r - sum_{c != r} a_rc x_c) / a_rr (textbook
 *        Gauss-Seidel; every row needs a nonzero stored diagonal, else
 *        SYMM_ERR_ARG at plan time);
 *   KACZ (kind 2): x := x + (b_r - <A_r, x>) / ||A_r||^2 * A_r (PAPER.md:
 *        826-851, eq:KACZ); rows with ||A_r|| = 0 are skipped.
 * x_dev, b_dev: DEVICE fp64[n] in the schedule's PERMUTED order; x is read and
 * overwritten; symmetric != 0 appends the backward sweep (SymmGS / SymmKACZ).
 * The plan owns its device memory (full matrix of the permuted order, row
 * order, phase table). */
typedef enum { SYMM_SWEEP_GS = 1, SYMM_SWEEP_KACZ = 2 } symm_sweep_kind;
typedef struct symm_sweep symm_sweep_t;
int symm_sweep_plan(const race_schedule_t* s, int32_t kind, int32_t device, symm_sweep_t** out);
int symm_sweep_run(symm_sweep_t* p, double* x_dev, const double* b_dev, int32_t symmetric, void* stream);
/* Host copy of the execution order: rows[n] (permuted ids, phase by phase) and
 * phase_ptr[nphases+1]; *nphases is set; either array may be NULL. */
int symm_sweep_order(const symm_sweep_t* p, int32_t* rows, int32_t* phase_ptr, int32_t* nphases);
int symm_sweep_destroy(symm_sweep_t* p);

const char* symm_status_string(int status);
const char* symm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SYMMSPMV_H */
