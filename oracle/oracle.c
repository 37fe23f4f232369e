/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the SymmSpMV hot path of
 * Alappat et al., "A Recursive Algebraic Coloring Technique for
 * Hardware-Efficient Symmetric Sparse Matrix-Vector Multiplication"
 * (arXiv 1907.06487).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no
 * code, header, table or helper with the product (paper_1907_06487_b200/).
 *
 * Every routine except oracle_symmspmv_omp (the OpenMP host baseline) is
 * single-threaded, fp64 (or long double where stated), with
 * no blocking, fusion or reordering beyond the algorithm it cites.
 * Citations are PAPER.md line ranges with the section / algorithm label.
 *
 * Pins (tests/test_oracle_pins.py): dense brute force, the 2-D Laplacian
 * eigenpair, SymmSpMV(U) == SpMV(mirror(U)), SPEC hand cases, BFS level-size
 * closed forms, island rule, brute-force distance-k on tiny graphs.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

/* ---------------------------------------------------------------------------
 * Alg. 2 "SymmSpMV b = A x, where A is an upper triangular matrix"
 * PAPER.md:730-745 (§3.2, alg:SymmSpMV).  0-based, half-open loops (reading
 * R3).  b := 0 first, then Alg. 2's `+=` (reading R2: y := A x).  A row's
 * diagonal is the entry with col == row; Alg. 2 assumes it is stored first
 * (PAPER.md:735); rows without a stored diagonal contribute none (reading R1).
 * ------------------------------------------------------------------------- */
void oracle_symmspmv(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A,
                     const double* x, double* b) {
  for (int32_t i = 0; i < n; ++i) b[i] = 0.0;
  for (int32_t row = 0; row < n; ++row) {
    int32_t start = rowPtr[row];
    if (start < rowPtr[row + 1] && col[start] == row) {
      /* diag_idx = rowPtr[row]; b[row] += A[diag_idx]*x[row] */
      b[row] += A[start] * x[row];
      start += 1;
    }
    double tmp = 0.0;
    for (int32_t idx = start; idx < rowPtr[row + 1]; ++idx) {
      tmp += A[idx] * x[col[idx]];          /* tmp += A[idx]*x[col[idx]]       */
      b[col[idx]] += A[idx] * x[row];       /* b[col[idx]] += A[idx]*x[row]    */
    }
    b[row] += tmp;                          /* b[row] += tmp                   */
  }
}

/* ---------------------------------------------------------------------------
 * OpenMP version of Alg. 2 (the host-core baseline the north star asks for),
 * parallelised the way PAPER.md:189-191 names as the general solution:
 * "thread private target arrays".  Rows are split into `nthreads` contiguous
 * blocks of equal row count (OpenMP static schedule); thread t runs Alg. 2
 * unchanged on its block into a private array b_t covering the rows its block
 * can write, [first row of the block, 1 + largest column in the block); then
 * b[i] = sum over t (ascending) of b_t[i].  nthreads <= 0 uses the OpenMP
 * default.  Returns the number of threads used (-1 on allocation failure).
 * With one thread it is oracle_symmspmv bit for bit.
 * ------------------------------------------------------------------------- */
int32_t oracle_symmspmv_omp(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A,
                            const double* x, double* b, int32_t nthreads) {
  int32_t nt = nthreads > 0 ? nthreads : omp_get_max_threads();
  if (nt > n) nt = n > 0 ? n : 1;
  int32_t* lo = (int32_t*)malloc(sizeof(int32_t) * (size_t)nt);
  int32_t* hi = (int32_t*)malloc(sizeof(int32_t) * (size_t)nt);
  double** bt = (double**)calloc((size_t)nt, sizeof(double*));
  int failed = (lo == NULL || hi == NULL || bt == NULL);
  if (!failed) {
#pragma omp parallel num_threads(nt)
    {
      int32_t t = omp_get_thread_num();
      int32_t r0 = (int32_t)((int64_t)n * t / nt), r1 = (int32_t)((int64_t)n * (t + 1) / nt);
      int32_t h = r0;
      for (int32_t row = r0; row < r1; ++row)
        for (int32_t idx = rowPtr[row]; idx < rowPtr[row + 1]; ++idx)
          if (col[idx] + 1 > h) h = col[idx] + 1;
      if (r1 > h) h = r1;
      lo[t] = r0;
      hi[t] = h;
      double* bl = (double*)malloc(sizeof(double) * (size_t)(h - r0 > 0 ? h - r0 : 1));
      bt[t] = bl;
      if (bl != NULL) {
        for (int32_t i = r0; i < h; ++i) bl[i - r0] = 0.0;
        for (int32_t row = r0; row < r1; ++row) {   /* Alg. 2 on the block, into b_t */
          int32_t start = rowPtr[row];
          if (start < rowPtr[row + 1] && col[start] == row) {
            bl[row - r0] += A[start] * x[row];
            start += 1;
          }
          double tmp = 0.0;
          for (int32_t idx = start; idx < rowPtr[row + 1]; ++idx) {
            tmp += A[idx] * x[col[idx]];
            bl[col[idx] - r0] += A[idx] * x[row];
          }
          bl[row - r0] += tmp;
        }
      }
#pragma omp barrier
#pragma omp for schedule(static)
      for (int32_t i = 0; i < n; ++i) {              /* b[i] = sum_t b_t[i], t ascending */
        double s = 0.0;
        for (int32_t u = 0; u < nt; ++u)
          if (bt[u] != NULL && i >= lo[u] && i < hi[u]) s += bt[u][i - lo[u]];
        b[i] = s;
      }
    }
    for (int32_t u = 0; u < nt; ++u) failed |= (bt[u] == NULL);
  }
  if (bt != NULL)
    for (int32_t u = 0; u < nt; ++u) free(bt[u]);
  free(bt);
  free(lo);
  free(hi);
  return failed ? -1 : nt;
}

/* Same algorithm with long double accumulation everywhere ("reference grade",
 * 80-bit on x86-64); used only to measure the fp64 oracle's own rounding. */
void oracle_symmspmv_ld(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A,
                        const double* x, long double* b) {
  for (int32_t i = 0; i < n; ++i) b[i] = 0.0L;
  for (int32_t row = 0; row < n; ++row) {
    int32_t start = rowPtr[row];
    if (start < rowPtr[row + 1] && col[start] == row) {
      b[row] += (long double)A[start] * (long double)x[row];
      start += 1;
    }
    long double tmp = 0.0L;
    for (int32_t idx = start; idx < rowPtr[row + 1]; ++idx) {
      tmp += (long double)A[idx] * (long double)x[col[idx]];
      b[col[idx]] += (long double)A[idx] * (long double)x[row];
    }
    b[row] += tmp;
  }
}

/* ---------------------------------------------------------------------------
 * Mirror: full symmetric A = U + U^T - diag(U) from the stored upper triangle
 * ("exploits the symmetry of the matrix (A_ij = A_ji) ...
 * operating on the upper (or lower) half").  Two passes: count, then fill in
 * ascending column order per row.  Returns nnz of A (or -1 on bad input).
 * Call with fRowPtr only (fCol == NULL) to get the count.
 * ------------------------------------------------------------------------- */
int64_t oracle_mirror(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A,
                      int32_t* fRowPtr, int32_t* fCol, double* fA) {
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!cnt) return -1;
  for (int32_t r = 0; r < n; ++r)
    for (int32_t idx = rowPtr[r]; idx < rowPtr[r + 1]; ++idx) {
      int32_t c = col[idx];
      cnt[r + 1] += 1;
      if (c != r) cnt[c + 1] += 1;
    }
  for (int32_t r = 0; r < n; ++r) cnt[r + 1] += cnt[r];
  int64_t nnz = cnt[n];
  if (fRowPtr)
    for (int32_t r = 0; r <= n; ++r) fRowPtr[r] = (int32_t)cnt[r];
  if (fCol && fA) {
    /* lower part (entries (c, r) for stored (r, c), c > r) arrive in ascending
     * r order; then the row's own upper entries in ascending c order: the row
     * is therefore sorted (all transposed cols < row <= own cols). */
    int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
    if (!pos) { free(cnt); return -1; }
    memcpy(pos, cnt, sizeof(int64_t) * ((size_t)n + 1));
    for (int32_t r = 0; r < n; ++r)
      for (int32_t idx = rowPtr[r]; idx < rowPtr[r + 1]; ++idx) {
        int32_t c = col[idx];
        if (c != r) { fCol[pos[c]] = r; fA[pos[c]] = A[idx]; pos[c] += 1; }
      }
    for (int32_t r = 0; r < n; ++r)
      for (int32_t idx = rowPtr[r]; idx < rowPtr[r + 1]; ++idx) {
        fCol[pos[r]] = col[idx]; fA[pos[r]] = A[idx]; pos[r] += 1;
      }
    free(pos);
  }
  free(cnt);
  return nnz;
}

/* ---------------------------------------------------------------------------
 * Alg. 1 "SpMV using the CRS format: b = A x", PAPER.md:570-584 (§3.1).
 * ------------------------------------------------------------------------- */
void oracle_spmv(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A,
                 const double* x, double* b) {
  for (int32_t row = 0; row < n; ++row) {
    double tmp = 0.0;
    for (int32_t idx = rowPtr[row]; idx < rowPtr[row + 1]; ++idx) tmp += A[idx] * x[col[idx]];
    b[row] = tmp;
  }
}

/* ---------------------------------------------------------------------------
 * NEXT-4 distance-k kernels (draft text of the paper), one
 * serial sweep over the rows in the given order on the FULL matrix (CRS,
 * e.g. from oracle_mirror).
 * Gauss-Seidel, textbook form (reading R32: the draft Alg. GS, PAPER.md:
 * 793-806, adds b to the old x[row]; we use x_r := (b_r - sum_{c != r} a_rc
 * x_c) / a_rr, the fixed point of which is A x = b):
 * ------------------------------------------------------------------------- */
void oracle_gs_sweep(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A, const double* b,
                     double* x, const int32_t* order, int64_t m) {
  (void)n;
  for (int64_t q = 0; q < m; ++q) {
    const int32_t row = order[q];
    double s = 0.0, diag = 0.0;
    for (int32_t idx = rowPtr[row]; idx < rowPtr[row + 1]; ++idx) {
      if (col[idx] == row) diag += A[idx];
      else s += A[idx] * x[col[idx]];
    }
    x[row] = (b[row] - s) / diag;
  }
}

/* Kaczmarz row projections, Alg. KACZ / eq:KACZ (PAPER.md:
 * 828-831): scale = (b_r - <A_r, x>) / ||A_r||^2, then x_c += scale * a_rc for
 * every c in row r; rows with ||A_r|| = 0 are skipped. */
void oracle_kacz_sweep(int32_t n, const int32_t* rowPtr, const int32_t* col, const double* A, const double* b,
                       double* x, const int32_t* order, int64_t m) {
  (void)n;
  for (int64_t q = 0; q < m; ++q) {
    const int32_t row = order[q];
    double scale = b[row], rownorm = 0.0;
    for (int32_t idx = rowPtr[row]; idx < rowPtr[row + 1]; ++idx) {
      scale -= A[idx] * x[col[idx]];
      rownorm += A[idx] * A[idx];
    }
    if (rownorm == 0.0) continue;
    scale = scale / rownorm;
    for (int32_t idx = rowPtr[row]; idx < rowPtr[row + 1]; ++idx) x[col[idx]] += scale * A[idx];
  }
}

/* Dense y = A x for tiny matrices given as a dense row-major array (the
 * textbook definition y_i = sum_j A_ij x_j, "b = Ax"). */
void oracle_dense_matvec(int32_t n, const double* Ad, const double* x, double* y) {
  for (int32_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int32_t j = 0; j < n; ++j) s += Ad[(int64_t)i * n + j] * x[j];
    y[i] = s;
  }
}

/* ---------------------------------------------------------------------------
 * Alg. 3 "Construction of levels", PAPER.md:2391-2420 (Appendix A, alg:BFS),
 * with Eq. 5's text reading "the ith level consists of all vertices that have
 * a minimum distance i from the root" (reading R7).
 * Termination (reading R8): loop until the frontier is empty; already-labelled
 * vertices are skipped when popped, exactly as line 12 of Alg. 3 does.
 * Islands (§4.4.1): "the starting node in the next island
 * is assigned a level number with an increment of two".  `roots` gives the
 * start vertex of each island in order; when they are exhausted the lowest
 * unlabelled vertex index starts the next island.  Self loops are ignored.
 * g_ptr/g_adj: full symmetric adjacency (any order).  Returns totalLvl
 * (= max level + 1, including empty separator levels), dist[v] >= 0.
 * ------------------------------------------------------------------------- */
int32_t oracle_bfs_levels(int32_t n, const int32_t* g_ptr, const int32_t* g_adj, int32_t nroots,
                          const int32_t* roots, int32_t* distFromRoot) {
  for (int32_t v = 0; v < n; ++v) distFromRoot[v] = -1;
  int32_t* curr = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int64_t cap = (int64_t)g_ptr[n] + n + 1;
  int32_t* nxt = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  int32_t maxLvl = -1, nextUnl = 0, rootIdx = 0, labelled = 0;
  while (labelled < n) {
    int32_t root = -1;
    while (rootIdx < nroots && root < 0) {
      int32_t r = roots[rootIdx++];
      if (r >= 0 && r < n && distFromRoot[r] == -1) root = r;
    }
    if (root < 0) {
      while (distFromRoot[nextUnl] != -1) ++nextUnl;
      root = nextUnl;
    }
    int32_t currLvl = (maxLvl < 0) ? 0 : maxLvl + 2;
    int64_t ncurr = 0;
    curr[ncurr++] = root;
    while (ncurr > 0) {
      int64_t nnxt = 0;
      for (int64_t i = 0; i < ncurr; ++i) {
        int32_t u = curr[i];
        if (distFromRoot[u] == -1) {
          distFromRoot[u] = currLvl;
          ++labelled;
          if (currLvl > maxLvl) maxLvl = currLvl;
          for (int32_t e = g_ptr[u]; e < g_ptr[u + 1]; ++e) {
            int32_t j = g_adj[e];
            if (distFromRoot[j] == -1) nxt[nnxt++] = j;
          }
        }
      }
      /* curr_children = nxt_children (duplicates are skipped when popped) */
      if (nnxt > n) {
        /* compact duplicates so curr never overflows its n+1 capacity */
        int64_t m = 0;
        for (int64_t i = 0; i < nnxt; ++i) {
          int32_t j = nxt[i];
          if (distFromRoot[j] == -1) { distFromRoot[j] = -2; nxt[m++] = j; }
        }
        for (int64_t i = 0; i < m; ++i) distFromRoot[nxt[i]] = -1;
        nnxt = m;
      }
      memcpy(curr, nxt, sizeof(int32_t) * (size_t)nnxt);
      ncurr = nnxt;
      currLvl += 1;
    }
  }
  free(curr);
  free(nxt);
  return maxLvl + 1;
}

/* ---------------------------------------------------------------------------
 * Brute-force distance-k relation, Eq. 6 (eq:dk):
 * u ->k v  iff  v in {u ∪ N(u) ∪ ... ∪ N^k(u)}.  For every vertex u a plain
 * BFS to depth k; counts ordered pairs (u, v), u != v, with cls[u] == cls[v]
 * >= 0 and u ->k v.  A correct distance-k coloring gives 0.
 * ------------------------------------------------------------------------- */
int64_t oracle_distk_violations(int32_t n, const int32_t* g_ptr, const int32_t* g_adj, int32_t k,
                                const int32_t* cls) {
  int32_t* d = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* q = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int64_t bad = 0;
  for (int32_t u = 0; u < n; ++u) {
    if (cls[u] < 0) continue;
    for (int32_t v = 0; v < n; ++v) d[v] = -1;
    int32_t h = 0, t = 0;
    d[u] = 0;
    q[t++] = u;
    while (h < t) {
      int32_t a = q[h++];
      if (d[a] == k) continue;
      for (int32_t e = g_ptr[a]; e < g_ptr[a + 1]; ++e) {
        int32_t b = g_adj[e];
        if (d[b] == -1) { d[b] = d[a] + 1; q[t++] = b; }
      }
    }
    for (int32_t v = 0; v < n; ++v)
      if (v != u && d[v] >= 0 && cls[v] == cls[u]) ++bad;
  }
  free(d);
  free(q);
  return bad;
}

/* ---------------------------------------------------------------------------
 * Write conflicts of Alg. 2 rows (PAPER.md:738-745 + 787-789: "two rows which
 * have a nonzero in the same column cannot be computed in parallel").  Row r
 * writes b[r] and b[col] for every stored col > r.  Counts unordered pairs of
 * distinct rows with equal cls >= 0 whose write sets intersect (pairwise
 * brute force; tiny n only).
 * ------------------------------------------------------------------------- */
int64_t oracle_write_conflicts(int32_t n, const int32_t* rowPtr, const int32_t* col, const int32_t* cls) {
  int64_t bad = 0;
  for (int32_t r = 0; r < n; ++r) {
    if (cls[r] < 0) continue;
    for (int32_t s = r + 1; s < n; ++s) {
      if (cls[s] != cls[r]) continue;
      int hit = 0;
      /* W(r) = {r} ∪ cols(r);  W(s) = {s} ∪ cols(s) */
      for (int32_t a = rowPtr[r] - 1; a < rowPtr[r + 1] && !hit; ++a) {
        int32_t wa = (a < rowPtr[r]) ? r : col[a];
        for (int32_t b = rowPtr[s] - 1; b < rowPtr[s + 1]; ++b) {
          int32_t wb = (b < rowPtr[s]) ? s : col[b];
          if (wa == wb) { hit = 1; break; }
        }
      }
      bad += hit;
    }
  }
  return bad;
}
