// RACE schedule builder (host, C++17/OpenMP) — race_build_schedule.
//
// Steps:
//  a1 validate the upper CRS
//  a2 mirror the pattern to the full graph
//  a3 pseudo-peripheral root per island             PAPER.md:1058 ("choose a root"), reading R9
//  a4 BFS levels, island +2 rule                    PAPER.md:1047-1081 (eq:level), 2391-2420 (Alg. 3), 1406-1411
//  a5 level permutation, U' = upper(P A P^T)
//  a6 eps level aggregation + Alg. 4 balancing      PAPER.md:1546-1648 (§4.4.3), 1234-1275 + 2422-2494 (Alg. 4)
//  a7 GPU tiles inside level groups, exact tile write-conflict coloring, DAG,
//     intra-tile distance-2 row coloring, first-writer flags, validator
//                                                   PAPER.md:1191-1217, 1650-1660, 787-789
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <queue>
#include <tuple>
#include <omp.h>

#include "internal.h"

namespace symm {

static thread_local std::string g_err;

int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}
void clear_error() { g_err.clear(); }
const char* last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// §4.4.3 steps 1-3.  Identical decision order to the
// oracle's eps_aggregate (reading R12): aggregate >= 2k levels until
// eps_ = 1 - |a - b| > eps with b = max(1, [a]) ([a] rounds half up); with b
// fixed, add levels while the combined weight stays <= b; leftovers join the
// last window.  Returns triples (first, end, b).
// ---------------------------------------------------------------------------
static int64_t round_half_up(double a) { return (int64_t)std::floor(a + 0.5); }

std::vector<int32_t> eps_aggregate(const std::vector<int64_t>& lw, int64_t nthreads, int k, double eps) {
  std::vector<int32_t> W;
  const int32_t L = (int32_t)lw.size();
  int64_t total = 0;
  for (int64_t v : lw) total += v;
  if (L == 0) return W;
  if (total == 0) return {0, L, 1};
  auto push = [&](int32_t f, int32_t e, int64_t b) {
    W.push_back(f); W.push_back(e); W.push_back((int32_t)b);
  };
  int32_t s = 0;
  while (s < L) {
    if (L - s < 2 * k) {
      if (!W.empty()) W[W.size() - 2] = L;
      else push(s, L, 1);
      break;
    }
    int64_t cum = 0;
    int32_t e = s;
    bool accepted = false;
    int64_t b = 1;
    while (e < L) {
      cum += lw[(size_t)e];
      e += 1;
      if (e - s < 2 * k) continue;
      double a = (double)cum * (double)nthreads / (double)total;
      b = std::max<int64_t>(1, round_half_up(a));
      double ep = 1.0 - std::fabs(a - (double)b);
      if (ep > eps) { accepted = true; break; }
    }
    if (!accepted) {
      double a = (double)cum * (double)nthreads / (double)total;
      b = std::max<int64_t>(1, round_half_up(a));
      push(s, L, b);
      break;
    }
    while (e < L) {
      int64_t nxt = cum + lw[(size_t)e];
      double a2 = (double)nxt * (double)nthreads / (double)total;
      if (a2 <= (double)b) { cum = nxt; e += 1; }
      else break;
    }
    push(s, e, b);
    s = e;
  }
  if (W.size() >= 6) {
    size_t m = W.size();
    if (W[m - 2] - W[m - 3] < 2 * k) {  // tail shorter than 2k joins the previous window
      W[m - 5] = W[m - 2];
      W.resize(m - 3);
    }
  }
  return W;
}

// Initial red/blue split of a window (reading R13): first boundary where the
// red part holds >= half of the window's work, clamped to keep >= k levels.
int32_t split_window(const std::vector<int64_t>& lw, int32_t first, int32_t end, int k) {
  int32_t nl = end - first;
  if (nl < 2 * k) return first + (nl + 1) / 2;
  int64_t tot = 0;
  for (int32_t i = first; i < end; ++i) tot += lw[(size_t)i];
  int64_t cum = 0;
  int32_t m = first;
  while (m < end) {
    cum += lw[(size_t)m];
    m += 1;
    if (2 * cum >= tot) break;
  }
  return std::min(std::max(m, first + k), end - k);
}

// Alg. 4 variance (lines 17-23) with reading R14.
static double alg4_variance(const std::vector<int32_t>& T, const std::vector<int32_t>& worker,
                            const std::vector<int64_t>& cum, std::vector<double>* diff_out) {
  const size_t ng = T.size() - 1;
  std::vector<double> size(ng), tsw(ng);
  for (size_t g = 0; g < ng; ++g) {
    size[g] = (double)(cum[(size_t)T[g + 1]] - cum[(size_t)T[g]]);
    tsw[g] = size[g] / (double)worker[g];
  }
  double sr = 0.0, sb = 0.0;
  int64_t wr = 0, wb = 0;
  for (size_t g = 0; g < ng; ++g) {
    if (g % 2 == 0) { sr += size[g]; wr += worker[g]; }
    else { sb += size[g]; wb += worker[g]; }
  }
  double mean_r = wr ? sr / (double)wr : 0.0;
  double mean_b = wb ? sb / (double)wb : 0.0;
  std::vector<double> diff(ng);
  for (size_t g = 0; g < ng; ++g) diff[g] = tsw[g] - (g % 2 == 0 ? mean_r : mean_b);
  double var = 0.0;
  for (size_t g = 0; g < ng; ++g) var += diff[g] * diff[g];
  var /= (double)ng;
  if (diff_out) *diff_out = std::move(diff);
  return var;
}

static void alg4_shift(std::vector<int32_t>& T, int32_t donor, int32_t receiver) {
  if (donor < receiver)
    for (int32_t j = donor + 1; j <= receiver; ++j) T[(size_t)j] -= 1;
  else if (donor > receiver)
    for (int32_t j = receiver + 1; j <= donor; ++j) T[(size_t)j] += 1;
}

// Alg. 4 "Load Balancing for two sweep, distance-2, two colors"
// (PAPER.md:2422-2494), same loop structure as the oracle's alg4_balance.
void alg4_balance(std::vector<int32_t>& T_ptr, const std::vector<int32_t>& worker,
                  const std::vector<int64_t>& lw, int kmin) {
  const int32_t ng = (int32_t)T_ptr.size() - 1;
  if (ng < 2) return;
  std::vector<int64_t> cum(lw.size() + 1, 0);
  for (size_t i = 0; i < lw.size(); ++i) cum[i + 1] = cum[i] + lw[i];
  bool exit_ = false;
  int64_t it = 0;
  std::vector<double> diff;
  std::vector<int32_t> absRank((size_t)ng), rank((size_t)ng);
  while (!exit_ && it < 1000000) {
    ++it;
    double var = alg4_variance(T_ptr, worker, cum, &diff);
    std::iota(absRank.begin(), absRank.end(), 0);
    std::stable_sort(absRank.begin(), absRank.end(),
                     [&](int32_t a, int32_t b) { return -std::fabs(diff[(size_t)a]) < -std::fabs(diff[(size_t)b]); });
    std::iota(rank.begin(), rank.end(), 0);
    std::stable_sort(rank.begin(), rank.end(), [&](int32_t a, int32_t b) { return diff[(size_t)a] < diff[(size_t)b]; });
    int32_t currRank = 0;
    double newVar = var;
    std::vector<int32_t> old = T_ptr;
    while (newVar >= var) {
      T_ptr = old;
      bool fail = true;
      int32_t g = absRank[(size_t)currRank];
      if (diff[(size_t)g] < 0) {
        int32_t acquire = -1;
        for (int32_t q = ng - 1; q >= 0; --q) {
          int32_t el = rank[(size_t)q];
          if (el != g && (T_ptr[(size_t)el + 1] - T_ptr[(size_t)el]) > kmin) {
            acquire = el;
            fail = false;
            break;
          }
        }
        if (!fail) alg4_shift(T_ptr, acquire, g);
      } else if ((T_ptr[(size_t)g + 1] - T_ptr[(size_t)g]) > kmin) {
        int32_t give = rank[0];
        if (give != g) {
          fail = false;
          alg4_shift(T_ptr, g, give);
        }
      }
      if (!fail) newVar = alg4_variance(T_ptr, worker, cum, nullptr);
      if (currRank == ng - 1 && newVar >= var) {
        T_ptr = old;
        exit_ = true;
        break;
      }
      currRank += 1;
    }
  }
}

// ---------------------------------------------------------------------------
namespace {

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int validate_upper(const symm_csr_upper* U) {
  if (!U) return set_error(SYMM_ERR_ARG, "U is NULL");
  if (U->n < 0) return set_error(SYMM_ERR_ARG, "n = %d < 0", U->n);
  if (U->nnz < 0) return set_error(SYMM_ERR_ARG, "nnz < 0");
  if (U->nnz >= (int64_t(1) << 31)) return set_error(SYMM_ERR_OVERFLOW, "nnz = %lld >= 2^31", (long long)U->nnz);
  if (U->n == 0) return SYMM_OK;
  if (!U->row_ptr || (U->nnz > 0 && (!U->col || !U->val))) return set_error(SYMM_ERR_ARG, "NULL CRS array");
  if (U->row_ptr[0] != 0) return set_error(SYMM_ERR_ARG, "row_ptr[0] = %d != 0", U->row_ptr[0]);
  if ((int64_t)U->row_ptr[U->n] != U->nnz)
    return set_error(SYMM_ERR_ARG, "row_ptr[n] = %d != nnz = %lld", U->row_ptr[U->n], (long long)U->nnz);
  const int32_t n = U->n;
  int32_t bad_row = INT32_MAX;
  int bad_code = 0;
#pragma omp parallel for schedule(static) reduction(min : bad_row)
  for (int32_t r = 0; r < n; ++r) {
    int32_t b = U->row_ptr[r], e = U->row_ptr[r + 1];
    if (e < b) { bad_row = std::min(bad_row, r); continue; }
    for (int32_t i = b; i < e; ++i) {
      int32_t c = U->col[i];
      if (c < r || c >= n || (i > b && c <= U->col[i - 1])) { bad_row = std::min(bad_row, r); break; }
    }
  }
  if (bad_row == INT32_MAX) return SYMM_OK;
  int32_t r = bad_row, b = U->row_ptr[r], e = U->row_ptr[r + 1];
  if (e < b) return set_error(SYMM_ERR_ARG, "row_ptr decreases at row %d", r);
  for (int32_t i = b; i < e; ++i) {
    int32_t c = U->col[i];
    if (c < r || c >= n) {
      bad_code = SYMM_ERR_NOT_UPPER;
      return set_error(bad_code, "row %d: column %d is not in [row, n) (upper triangle required)", r, c);
    }
    if (i > b && c <= U->col[i - 1])
      return set_error(SYMM_ERR_UNSORTED, "row %d: columns not strictly ascending at column %d", r, c);
  }
  return set_error(SYMM_ERR_ARG, "row %d invalid", r);
}

// Full symmetric adjacency without self loops, sorted neighbour lists.
void mirror_graph(const symm_csr_upper* U, std::vector<int64_t>& gp, std::vector<int32_t>& ga) {
  const int32_t n = U->n;
  gp.assign((size_t)n + 1, 0);
  std::vector<int64_t> deg((size_t)n, 0);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int32_t r = 0; r < n; ++r) {
    int64_t own = 0;
    for (int32_t i = U->row_ptr[r]; i < U->row_ptr[r + 1]; ++i) {
      int32_t c = U->col[i];
      if (c == r) continue;
      ++own;
      __atomic_fetch_add(&deg[(size_t)c], 1, __ATOMIC_RELAXED);
    }
    __atomic_fetch_add(&deg[(size_t)r], own, __ATOMIC_RELAXED);
  }
  for (int32_t r = 0; r < n; ++r) gp[(size_t)r + 1] = gp[(size_t)r] + deg[(size_t)r];
  ga.resize((size_t)gp[(size_t)n]);
  std::vector<int64_t> pos(gp.begin(), gp.end() - 1);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int32_t r = 0; r < n; ++r) {
    for (int32_t i = U->row_ptr[r]; i < U->row_ptr[r + 1]; ++i) {
      int32_t c = U->col[i];
      if (c == r) continue;
      int64_t p = __atomic_fetch_add(&pos[(size_t)c], 1, __ATOMIC_RELAXED);
      ga[(size_t)p] = r;
      int64_t q = __atomic_fetch_add(&pos[(size_t)r], 1, __ATOMIC_RELAXED);
      ga[(size_t)q] = c;
    }
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int32_t r = 0; r < n; ++r) std::sort(ga.begin() + gp[(size_t)r], ga.begin() + gp[(size_t)r + 1]);
}

// Plain BFS from src over unlabelled (dist == -1) vertices; returns the
// eccentricity and the last level (for the pseudo-peripheral search).
struct BfsScratch {
  std::vector<int32_t> mark;
  int32_t stamp = 0;
  std::vector<int32_t> frontier, next;
};

int32_t bfs_ecc(int32_t src, const std::vector<int64_t>& gp, const std::vector<int32_t>& ga, BfsScratch& B,
                std::vector<int32_t>& last) {
  B.stamp += 1;
  B.frontier.clear();
  B.frontier.push_back(src);
  B.mark[(size_t)src] = B.stamp;
  int32_t ecc = 0;
  for (;;) {
    B.next.clear();
    for (int32_t u : B.frontier)
      for (int64_t e = gp[(size_t)u]; e < gp[(size_t)u + 1]; ++e) {
        int32_t j = ga[(size_t)e];
        if (B.mark[(size_t)j] != B.stamp) { B.mark[(size_t)j] = B.stamp; B.next.push_back(j); }
      }
    if (B.next.empty()) break;
    std::swap(B.frontier, B.next);
    ++ecc;
  }
  last = B.frontier;
  return ecc;
}

// George-Liu style pseudo-peripheral vertex (reading R9): from `start`, move
// to a minimum-degree vertex of the last BFS level while the eccentricity grows.
int32_t pseudo_peripheral(int32_t start, const std::vector<int64_t>& gp, const std::vector<int32_t>& ga,
                          BfsScratch& B) {
  std::vector<int32_t> last;
  int32_t root = start;
  int32_t ecc = bfs_ecc(root, gp, ga, B, last);
  for (int it = 0; it < 8; ++it) {
    int32_t best = -1;
    int64_t bestdeg = INT64_MAX;
    for (int32_t v : last) {
      int64_t d = gp[(size_t)v + 1] - gp[(size_t)v];
      if (d < bestdeg || (d == bestdeg && v < best)) { bestdeg = d; best = v; }
    }
    if (best < 0 || best == root) break;
    std::vector<int32_t> last2;
    int32_t e2 = bfs_ecc(best, gp, ga, B, last2);
    if (e2 <= ecc) break;
    root = best;
    ecc = e2;
    last.swap(last2);
  }
  return root;
}

}  // namespace

// K3/K4 ring: kRingStages stages of (tile block + x window) should fit the
// dynamic shared memory a B200 CTA gets (227 KB - 1 KB reserved - static)
constexpr int64_t kRingBytes = 232448 - 1024 - 512;
constexpr int64_t kRingStages = 6;

int build_schedule(const symm_csr_upper* U, const race_config* cfgp, Schedule* S) {
  const double t0 = now_s();
  race_config cfg;
  if (cfgp) cfg = *cfgp;
  else race_config_default(&cfg);
  if (cfg.k < 2) return set_error(SYMM_ERR_K, "distance k = %d < 2: SymmSpMV needs distance-2 (PAPER.md:787-789)", cfg.k);
  if (cfg.tile_work <= 0 || cfg.max_tile_rows <= 0 || cfg.max_tile_rows > 65535 || cfg.max_tile_window < 64 ||
      cfg.max_tile_window > 65535 || cfg.max_tile_nnz < 1 || cfg.max_tile_nnz > 65535 || cfg.n_eps < 1 || cfg.n_eps > 8 || cfg.n_workers < 0 ||
      cfg.scheme < 0 || cfg.scheme > 3 || (cfg.scheme == 2 && cfg.abmc_block < 1) || cfg.reorder < 0 ||
      (cfg.scheme == 3 && (cfg.cone_tiles || !cfg.reorder)) ||
      cfg.reorder > 2 || (cfg.reorder == 2 && cfg.cone_tiles))
    return set_error(SYMM_ERR_ARG, "invalid race_config field");
  int rc = validate_upper(U);
  if (rc) return rc;
  S->cfg = cfg;
  const int32_t n = U->n;
  S->n = n;
  S->nnz = U->nnz;
  const int k = cfg.k;
  const int kg = std::max(k, cfg.min_group_levels);  // levels per group: "at least k"

  // ---- a2 mirror, a3 roots, a4 BFS levels (discovery order) -------------------
  std::vector<int64_t> gp;
  std::vector<int32_t> ga;
  mirror_graph(U, gp, ga);
  S->dist.assign((size_t)n, -1);
  std::vector<int32_t> order;
  order.reserve((size_t)n);
  // disc[p]: BFS position of the first vertex discovered by the vertex at BFS
  // position p (= queue length when p is expanded); the children first
  // discovered by positions [a, b) of one level are positions [disc[a], disc[b])
  std::vector<int32_t> disc((size_t)n + 1, n);
  {
    BfsScratch B;
    B.mark.assign((size_t)n, 0);
    int32_t maxLvl = -1, nextUnl = 0;
    bool first = true;
    while ((int32_t)order.size() < n) {
      while (S->dist[(size_t)nextUnl] != -1) ++nextUnl;
      int32_t root;
      if (!cfg.reorder) root = nextUnl;
      else if (first && cfg.root >= 0 && cfg.root < n) root = cfg.root;
      else root = pseudo_peripheral(nextUnl, gp, ga, B);
      first = false;
      S->roots.push_back(root);
      int32_t lvl = maxLvl < 0 ? 0 : maxLvl + 2;  // island rule
      size_t head = order.size();
      order.push_back(root);
      S->dist[(size_t)root] = lvl;
      size_t lvl_begin = head, lvl_end = order.size();
      while (lvl_begin < lvl_end) {
        maxLvl = std::max(maxLvl, lvl);
        for (size_t q = lvl_begin; q < lvl_end; ++q) {
          int32_t u = order[q];
          disc[q] = (int32_t)order.size();
          const size_t c0 = order.size();
          for (int64_t e = gp[(size_t)u]; e < gp[(size_t)u + 1]; ++e) {
            int32_t j = ga[(size_t)e];
            if (S->dist[(size_t)j] == -1) { S->dist[(size_t)j] = lvl + 1; order.push_back(j); }
          }
          if (cfg.reorder == 2)  // Cuthill-McKee: u's new neighbours by ascending degree, then index
            std::sort(order.begin() + (int64_t)c0, order.end(), [&](int32_t a, int32_t b) {
              const int64_t da = gp[(size_t)a + 1] - gp[(size_t)a], db = gp[(size_t)b + 1] - gp[(size_t)b];
              return da != db ? da < db : a < b;
            });
        }
        lvl_begin = lvl_end;
        lvl_end = order.size();
        ++lvl;
      }
    }
    const int32_t totalLvl = maxLvl + 1;
    if (cfg.reorder == 2) {
      // Reverse Cuthill-McKee: the whole CM
      // order reversed; levels stay contiguous, relabelled from the far end
      // (island separators stay empty levels)
      std::reverse(order.begin(), order.end());
      for (int32_t v = 0; v < n; ++v) S->dist[(size_t)v] = maxLvl - S->dist[(size_t)v];
    }
    S->level_ptr.assign((size_t)std::max(totalLvl, 0) + 1, 0);
    if (cfg.reorder) {
      for (int32_t v = 0; v < n; ++v) S->level_ptr[(size_t)S->dist[(size_t)v] + 1] += 1;
      for (int32_t l = 0; l < totalLvl; ++l) S->level_ptr[(size_t)l + 1] += S->level_ptr[(size_t)l];
      if (cfg.flags & 1u) {
        // within-level order = original index (instead of BFS discovery order);
        // levels stay contiguous and in BFS order
#pragma omp parallel for schedule(dynamic, 1)
        for (int32_t l = 0; l < totalLvl; ++l)
          std::sort(order.begin() + S->level_ptr[(size_t)l], order.begin() + S->level_ptr[(size_t)l + 1]);
      }
    } else {
      // no reordering: the whole matrix is one "level" (natural order kept)
      S->level_ptr = {0, n};
      order.resize((size_t)n);
      std::iota(order.begin(), order.end(), 0);
    }
  }

  // ---- a5 permutation and U' = upper(P A P^T) ---------------------------------
  S->inv = order;
  S->perm.assign((size_t)n, 0);
  for (int32_t i = 0; i < n; ++i) S->perm[(size_t)order[(size_t)i]] = i;
  auto build_permuted = [&]() {
    const int32_t* P = S->perm.data();
    std::vector<int32_t> cnt((size_t)n + 1, 0);
    int64_t bwb = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(max : bwb)
    for (int32_t r = 0; r < n; ++r)
      for (int32_t i = U->row_ptr[r]; i < U->row_ptr[r + 1]; ++i) {
        int32_t c = U->col[i];
        bwb = std::max<int64_t>(bwb, (int64_t)c - r);
        int32_t a = std::min(P[r], P[c]);
        __atomic_fetch_add(&cnt[(size_t)a + 1], 1, __ATOMIC_RELAXED);
      }
    S->bw_before = bwb;
    S->prow_ptr.assign((size_t)n + 1, 0);
    for (int32_t r = 0; r < n; ++r) S->prow_ptr[(size_t)r + 1] = S->prow_ptr[(size_t)r] + cnt[(size_t)r + 1];
    S->pcol.resize((size_t)U->nnz);
    S->pval.resize((size_t)U->nnz);
    std::vector<int32_t> pos(S->prow_ptr.begin(), S->prow_ptr.end() - 1);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int32_t r = 0; r < n; ++r)
      for (int32_t i = U->row_ptr[r]; i < U->row_ptr[r + 1]; ++i) {
        int32_t c = U->col[i];
        int32_t a = std::min(P[r], P[c]), b = std::max(P[r], P[c]);
        int32_t p = __atomic_fetch_add(&pos[(size_t)a], 1, __ATOMIC_RELAXED);
        S->pcol[(size_t)p] = b;
        S->pval[(size_t)p] = U->val[i];
      }
    int64_t bwa = 0;
#pragma omp parallel reduction(max : bwa)
    {
    std::vector<std::pair<int32_t, double>> tmp;
#pragma omp for schedule(dynamic, 1024)
    for (int32_t r = 0; r < n; ++r) {
      int32_t b = S->prow_ptr[(size_t)r], e = S->prow_ptr[(size_t)r + 1];
      // sort entries of the row by column (values follow)
      tmp.resize((size_t)(e - b));
      for (int32_t i = b; i < e; ++i) tmp[(size_t)(i - b)] = {S->pcol[(size_t)i], S->pval[(size_t)i]};
      std::sort(tmp.begin(), tmp.end());
      for (int32_t i = b; i < e; ++i) {
        S->pcol[(size_t)i] = tmp[(size_t)(i - b)].first;
        S->pval[(size_t)i] = tmp[(size_t)(i - b)].second;
        bwa = std::max<int64_t>(bwa, (int64_t)S->pcol[(size_t)i] - r);
      }
    }
    }
    S->bw_after = bwa;
  };
  build_permuted();
  if ((cfg.scheme == 1 || cfg.scheme == 2)) {
    // ---- NEXT-3 comparison schemes: MC colours single rows,
    // ABMC colours blocks of consecutive BFS-ordered rows; both greedy in BFS
    // order by closed neighbourhoods N[v] = {v} ∪ adj(v) -- the distance-2
    // relation of PAPER.md:787-789 in its order-independent form (any
    // orientation's write set {r} ∪ {upper columns} lies inside N[r], so the
    // colouring stays valid after the rows are re-ordered colour by colour).
    // Each colour class then becomes one level and one level group, so the
    // tiles, phases and validators below apply unchanged.
    const int32_t B = cfg.scheme == 1 ? 1 : cfg.abmc_block;
    const int32_t nb = (n + B - 1) / B;
    std::vector<int32_t> bcol((size_t)nb, 0), last((size_t)n, -1);  // last[v] = newest colour writing v
    std::vector<std::vector<int32_t>> writers((size_t)n);            // colours writing v so far (original ids)
    int32_t ncol = 0;
    {
      std::vector<uint64_t> used;
      for (int32_t b = 0; b < nb; ++b) {
        used.assign((size_t)(ncol / 64 + 2), 0);
        const int32_t r0b = b * B, r1b = std::min(n, r0b + B);
        for (int32_t r = r0b; r < r1b; ++r) {
          const int32_t v = S->inv[(size_t)r];
          for (int64_t e = gp[(size_t)v] - 1; e < gp[(size_t)v + 1]; ++e) {
            const int32_t c = e < gp[(size_t)v] ? v : ga[(size_t)e];
            for (int32_t q : writers[(size_t)c]) used[(size_t)q / 64] |= uint64_t(1) << (q % 64);
          }
        }
        int32_t col = 0;
        while (used[(size_t)col / 64] >> (col % 64) & 1) ++col;
        bcol[(size_t)b] = col;
        ncol = std::max(ncol, col + 1);
        for (int32_t r = r0b; r < r1b; ++r) {
          const int32_t v = S->inv[(size_t)r];
          for (int64_t e = gp[(size_t)v] - 1; e < gp[(size_t)v + 1]; ++e) {
            const int32_t c = e < gp[(size_t)v] ? v : ga[(size_t)e];
            if (last[(size_t)c] != col) {
              writers[(size_t)c].push_back(col);
              last[(size_t)c] = col;
            }
          }
        }
      }
    }
    std::vector<int32_t> cstart((size_t)ncol + 1, 0);
    for (int32_t b = 0; b < nb; ++b) cstart[(size_t)bcol[(size_t)b] + 1] += std::min(n, b * B + B) - b * B;
    for (int32_t c = 0; c < ncol; ++c) cstart[(size_t)c + 1] += cstart[(size_t)c];
    std::vector<int32_t> pos(cstart.begin(), cstart.end() - 1), inv2((size_t)n);
    for (int32_t b = 0; b < nb; ++b)
      for (int32_t r = b * B; r < std::min(n, b * B + B); ++r) inv2[(size_t)pos[(size_t)bcol[(size_t)b]]++] = S->inv[(size_t)r];
    S->inv.swap(inv2);
    for (int32_t f = 0; f < n; ++f) S->perm[(size_t)S->inv[(size_t)f]] = f;
    build_permuted();
    S->level_ptr = cstart;  // one "level" per colour class
  }
  const int32_t* rp = S->prow_ptr.data();  // re-bound after the cone re-permutation
  const int32_t* pc = S->pcol.data();

  // ---- a6 eps aggregation (§4.4.3) + Alg. 4 (§4.3), work per level ------------
  auto row_work = [&](int32_t r) -> int64_t {
    return cfg.balance_by == 0 ? 1 : (int64_t)(rp[r + 1] - rp[r]) + 2;
  };
  const int32_t totalLvl = (int32_t)S->level_ptr.size() - 1;
  std::vector<int64_t> lw((size_t)std::max(totalLvl, 0), 0);
  int64_t total_work = 0;
  for (int32_t l = 0; l < totalLvl; ++l) {
    int64_t w = 0;
    for (int32_t r = S->level_ptr[(size_t)l]; r < S->level_ptr[(size_t)l + 1]; ++r) w += row_work(r);
    lw[(size_t)l] = w;
    total_work += w;
  }
  int64_t nworkers = cfg.n_workers > 0 ? cfg.n_workers : std::max<int64_t>(1, (total_work + cfg.tile_work - 1) / cfg.tile_work);
  // the recursive tree (scheme 3) targets a thread count like the paper's
  // (one worker = one CTA of the tree kernel): 8 per SM of a B200 by default
  if (cfg.scheme == 3 && cfg.n_workers <= 0) nworkers = 8 * 148;
  if ((cfg.scheme == 1 || cfg.scheme == 2)) {
    // MC / ABMC: every colour class is its own group, split into tiles by work
    S->group_lvl.resize((size_t)totalLvl + 1);
    for (int32_t l = 0; l <= totalLvl; ++l) S->group_lvl[(size_t)l] = l;
    S->group_workers.resize((size_t)totalLvl);
    for (int32_t l = 0; l < totalLvl; ++l)
      S->group_workers[(size_t)l] = (int32_t)std::max<int64_t>(1, (lw[(size_t)l] + cfg.tile_work - 1) / cfg.tile_work);
  } else {
  S->windows = eps_aggregate(lw, nworkers, kg, cfg.eps[0]);
  {
    std::vector<int32_t> T, wk;
    const size_t nw = S->windows.size() / 3;
    if (nw > 0) T.push_back(S->windows[0]);
    for (size_t w = 0; w < nw; ++w) {
      int32_t f = S->windows[3 * w], e = S->windows[3 * w + 1], b = S->windows[3 * w + 2];
      int32_t m = split_window(lw, f, e, kg);
      T.push_back(m);
      T.push_back(e);
      wk.push_back(b);
      wk.push_back(b);
    }
    if (T.size() >= 3) alg4_balance(T, wk, lw, kg);
    S->group_lvl = T;
    S->group_workers = wk;
  }
  }
  if (cfg.scheme == 3) {
    // ---- NEXT-2: the recursive RACE tree (§4.4.1-4.4.2) --
    // A level group T_s(j) with more than one worker is refined: BFS levels
    // on the subgraph of T_s(j) plus its distance-(k-1) = distance-1
    // neighbourhood (no outside vertex can then mediate a
    // distance-2 conflict), island rule +2, only the
    // vertices of T_s(j) kept in the new levels L_{s+1};
    // eps_{s+1} aggregation + Alg. 4 on them give T_{s+1}(:) inside T_s(j),
    // whose rows are re-permuted in the new level order.
    // Readings R29-R31: root = the first vertex of the group in
    // its current order; workload = rows; a group that yields fewer than two
    // level groups stays a leaf.
    auto& TP = S->tree_parent;
    auto& TC = S->tree_cidx;
    auto& T0 = S->tree_r0;
    auto& T1 = S->tree_r1;
    auto& TS = S->tree_stage;
    auto& TW = S->tree_workers;
    auto add_node = [&](int32_t par, int32_t ci, int32_t a, int32_t b, int32_t st, int32_t w) {
      TP.push_back(par); TC.push_back(ci); T0.push_back(a); T1.push_back(b); TS.push_back(st); TW.push_back(w);
      return (int32_t)TP.size() - 1;
    };
    add_node(-1, 0, 0, n, -1, (int32_t)std::min<int64_t>(nworkers, INT32_MAX));
    const int32_t ng0 = (int32_t)S->group_workers.size();
    for (int32_t g = 0; g < ng0; ++g)
      add_node(0, g, S->level_ptr[(size_t)S->group_lvl[(size_t)g]], S->level_ptr[(size_t)S->group_lvl[(size_t)g + 1]], 0,
               S->group_workers[(size_t)g]);
    std::vector<int32_t> ing((size_t)n, -1), inh((size_t)n, -1), vis((size_t)n, -1), hd((size_t)n, 0);
    std::vector<int32_t> ord, keep;
    for (int32_t id = 1; id < (int32_t)TP.size(); ++id) {  // TP grows while we walk it
      const int32_t p0 = T0[(size_t)id], p1 = T1[(size_t)id], w = TW[(size_t)id], st = TS[(size_t)id] + 1;
      if (w <= 1 || p1 - p0 < 2) continue;
      for (int32_t q = p0; q < p1; ++q) {
        const int32_t v = S->inv[(size_t)q];
        ing[(size_t)v] = id;
        inh[(size_t)v] = id;
      }
      for (int32_t q = p0; q < p1; ++q) {
        const int32_t v = S->inv[(size_t)q];
        for (int64_t e = gp[(size_t)v]; e < gp[(size_t)v + 1]; ++e) inh[(size_t)ga[(size_t)e]] = id;
      }
      ord.clear();
      int32_t maxL = -1;
      for (int32_t q = p0; q < p1; ++q) {  // one BFS per island of the subgraph
        const int32_t root = S->inv[(size_t)q];
        if (vis[(size_t)root] == id) continue;
        const int32_t lvl0 = maxL < 0 ? 0 : maxL + 2;
        size_t head = ord.size();
        ord.push_back(root);
        vis[(size_t)root] = id;
        hd[(size_t)root] = lvl0;
        while (head < ord.size()) {
          const int32_t u = ord[head++];
          maxL = std::max(maxL, hd[(size_t)u]);
          for (int64_t e = gp[(size_t)u]; e < gp[(size_t)u + 1]; ++e) {
            const int32_t v = ga[(size_t)e];
            if (inh[(size_t)v] == id && vis[(size_t)v] != id) {
              vis[(size_t)v] = id;
              hd[(size_t)v] = hd[(size_t)u] + 1;
              ord.push_back(v);
            }
          }
        }
      }
      // new levels: only the group's own vertices (BFS order is level-monotone)
      keep.clear();
      for (int32_t v : ord)
        if (ing[(size_t)v] == id) keep.push_back(v);
      std::vector<int64_t> lw2((size_t)maxL + 1, 0);
      for (int32_t v : keep) lw2[(size_t)hd[(size_t)v]] += 1;
      const double eps_s = cfg.eps[(size_t)std::min(st, cfg.n_eps - 1)];
      std::vector<int32_t> win = eps_aggregate(lw2, w, kg, eps_s);
      std::vector<int32_t> Tq, wq;
      const size_t nw = win.size() / 3;
      if (nw > 0) Tq.push_back(win[0]);
      for (size_t q = 0; q < nw; ++q) {
        const int32_t f = win[3 * q], e = win[3 * q + 1], b = win[3 * q + 2];
        Tq.push_back(split_window(lw2, f, e, kg));
        Tq.push_back(e);
        wq.push_back(b);
        wq.push_back(b);
      }
      if (Tq.size() >= 3) alg4_balance(Tq, wq, lw2, kg);
      std::copy(keep.begin(), keep.end(), S->inv.begin() + p0);  // re-permute the group (locality)
      std::vector<std::pair<int32_t, int32_t>> kids;  // (rows, workers)
      for (size_t j = 0; j + 1 < Tq.size(); ++j) {
        int32_t cnt = 0;
        for (int32_t l = Tq[j]; l < Tq[j + 1]; ++l) cnt += (int32_t)lw2[(size_t)l];
        kids.push_back({cnt, wq[j]});
      }
      int32_t nonempty = 0;
      for (auto& kd : kids) nonempty += kd.first > 0;
      if (nonempty < 2) continue;  // no parallelism found: stays a leaf
      int32_t a = p0;
      for (size_t j = 0; j < kids.size(); ++j) {
        // empty groups still count for the red/blue alternation
        add_node(id, (int32_t)j, a, a + kids[j].first, st, kids[j].second);
        a += kids[j].first;
      }
    }
    for (int32_t f = 0; f < n; ++f) S->perm[(size_t)S->inv[(size_t)f]] = f;
    build_permuted();
    rp = S->prow_ptr.data();
    pc = S->pcol.data();
    // leaves (nodes without children) in position order become the groups
    std::vector<int32_t> nkids(TP.size(), 0);
    for (size_t v = 1; v < TP.size(); ++v) nkids[(size_t)TP[v]]++;
    std::vector<int32_t> leaves;
    for (size_t v = 1; v < TP.size(); ++v)
      if (nkids[v] == 0 && T1[v] > T0[v]) leaves.push_back((int32_t)v);
    std::sort(leaves.begin(), leaves.end(), [&](int32_t a, int32_t b) { return T0[(size_t)a] < T0[(size_t)b]; });
    S->tree_leaf = leaves;
    S->level_ptr.assign(1, 0);
    for (int32_t v : leaves) S->level_ptr.push_back(T1[(size_t)v]);
    S->group_lvl.resize(leaves.size() + 1);
    std::iota(S->group_lvl.begin(), S->group_lvl.end(), 0);
    S->group_workers.assign(leaves.size(), 1);
    // §5 nrowsEff / eta of the tree, rows as the workload
    std::vector<int64_t> eff(TP.size(), 0), emax[2];
    emax[0].assign(TP.size(), 0);
    emax[1].assign(TP.size(), 0);
    for (size_t v = TP.size(); v-- > 1;) {  // children have larger ids than parents
      eff[v] = nkids[v] == 0 ? (int64_t)(T1[v] - T0[v]) : emax[0][v] + emax[1][v];
      auto& m = emax[(size_t)(TC[v] & 1)][(size_t)TP[v]];
      m = std::max(m, eff[v]);
    }
    eff[0] = emax[0][0] + emax[1][0];
    S->tree_eta = eff[0] > 0 ? (double)n / ((double)eff[0] * (double)TW[0]) : 1.0;
  }
  const int32_t ngroups = (int32_t)S->group_workers.size();
  int64_t block_budget = 0;  // 0: derived from the ring (below)
  if (const char* v = std::getenv("SYMM_BLOCK_BUDGET")) block_budget = std::atoll(v);  // diagnostics / sweeps

  // ---- a7 tiles --------------------------------------------------------------
  // (a) cone tiles (cfg.cone_tiles, reading R26): inside level group g with b_g
  //     workers, every level of the group is cut into K work-balanced chunks and
  //     tile k = chunk k of every level; the rows of the group are re-permuted
  //     cone by cone (levels stay contiguous per group).  K
  //     starts at b_g and grows until every cone meets the row / nnz / window
  //     caps in the FINAL order.
  // (b) otherwise (or if no K fits): contiguous work-balanced chunks of the
  //     group, halved until they fit.
  std::vector<std::vector<int32_t>> cone_sizes((size_t)ngroups);
  std::vector<char> is_cone((size_t)ngroups, 0);
  if (cfg.cone_tiles && cfg.reorder && ngroups > 0 && n > 0) {
    std::vector<uint8_t> has_diag((size_t)n, 0);
    for (int32_t r = 0; r < n; ++r)
      has_diag[(size_t)r] = (U->row_ptr[r] < U->row_ptr[r + 1] && U->col[U->row_ptr[r]] == r);
    std::vector<int32_t> grp_of_lvl((size_t)totalLvl, 0);
    for (int32_t g = 0; g < ngroups; ++g)
      for (int32_t l = S->group_lvl[(size_t)g]; l < S->group_lvl[(size_t)g + 1]; ++l) grp_of_lvl[(size_t)l] = g;
    std::vector<std::vector<int32_t>> new_order((size_t)ngroups);
    const int32_t* Pb = S->perm.data();  // old -> BFS position
    const int32_t* Ib = S->inv.data();   // BFS position -> old
#pragma omp parallel
    {
      std::vector<int32_t> cone_of, tg;
#pragma omp for schedule(dynamic, 1)
      for (int32_t g = 0; g < ngroups; ++g) {
        const int32_t l0 = S->group_lvl[(size_t)g], l1 = S->group_lvl[(size_t)g + 1];
        const int32_t g0 = S->level_ptr[(size_t)l0], g1 = S->level_ptr[(size_t)l1];
        if (g1 <= g0) continue;
        int64_t stored = 0;
        for (int32_t r = g0; r < g1; ++r) stored += rp[r + 1] - rp[r];
        int64_t K = std::max<int64_t>({(int64_t)S->group_workers[(size_t)g],
                                       (int64_t)std::ceil((double)stored / (0.9 * cfg.max_tile_nnz)),
                                       (int64_t)std::ceil((double)(g1 - g0) / cfg.max_tile_rows), 1});
        cone_of.assign((size_t)(g1 - g0), 0);
        bool ok = false;
        std::vector<std::vector<int32_t>> cuts;
        for (int attempt = 0; attempt < 40 && !ok; ++attempt) {
          cuts.assign((size_t)(l1 - l0), {});
          if (cfg.cone_tiles == 2) {
            // first level: work-balanced cuts; deeper levels: the discovery
            // ranges of the previous level's chunks (children follow parents)
            const int32_t a = S->level_ptr[(size_t)l0], e = S->level_ptr[(size_t)l0 + 1];
            int64_t lwk = 0;
            for (int32_t r = a; r < e; ++r) lwk += row_work(r);
            auto& c0 = cuts[0];
            c0.assign((size_t)K + 1, e);
            c0[0] = a;
            int64_t cum = 0, j = 1;
            for (int32_t r = a; r < e && j < K; ++r) {
              cum += row_work(r);
              while (j < K && cum * K >= j * lwk) c0[(size_t)j++] = r + 1;
            }
            for (int32_t l = l0 + 1; l < l1; ++l) {
              const auto& cp = cuts[(size_t)(l - 1 - l0)];
              auto& c = cuts[(size_t)(l - l0)];
              const int32_t la = S->level_ptr[(size_t)l], le = S->level_ptr[(size_t)l + 1];
              c.assign((size_t)K + 1, le);
              c[0] = la;
              for (int64_t q = 1; q < K; ++q) {
                const int32_t pq = cp[(size_t)q];
                int32_t v = (pq < S->level_ptr[(size_t)l]) ? disc[(size_t)pq] : le;
                c[(size_t)q] = std::min(std::max(v, c[(size_t)q - 1]), le);
              }
            }
            for (int32_t l = l0; l < l1; ++l) {
              const auto& c = cuts[(size_t)(l - l0)];
              for (int64_t q = 0; q < K; ++q)
                for (int32_t r = c[(size_t)q]; r < c[(size_t)q + 1]; ++r) cone_of[(size_t)(r - g0)] = (int32_t)q;
            }
          } else
          for (int32_t l = l0; l < l1; ++l) {
            const int32_t a = S->level_ptr[(size_t)l], e = S->level_ptr[(size_t)l + 1];
            int64_t lwk = 0;
            for (int32_t r = a; r < e; ++r) lwk += row_work(r);
            auto& c = cuts[(size_t)(l - l0)];
            c.assign((size_t)K + 1, e);
            c[0] = a;
            int64_t cum = 0;
            int64_t j = 1;
            for (int32_t r = a; r < e && j < K; ++r) {
              cum += row_work(r);
              while (j < K && cum * K >= j * lwk) c[(size_t)j++] = r + 1;
            }
            for (int64_t q = 0; q < K; ++q)
              for (int32_t r = c[(size_t)q]; r < c[(size_t)q + 1]; ++r) cone_of[(size_t)(r - g0)] = (int32_t)q;
          }
          // exact caps of every cone in the final order: entry (r, v) is stored in
          // row r iff key(v) > key(r), key = (group, cone, BFS position)
          std::vector<int64_t> rows((size_t)K, 0), nnzc((size_t)K, 0);
          std::vector<std::vector<int32_t>> tgts((size_t)K);
          for (int32_t r = g0; r < g1; ++r) {
            const int32_t kr = cone_of[(size_t)(r - g0)];
            rows[(size_t)kr]++;
            const int32_t o = Ib[r];
            nnzc[(size_t)kr] += has_diag[(size_t)o];
            for (int64_t e = gp[(size_t)o]; e < gp[(size_t)o + 1]; ++e) {
              const int32_t v = Pb[ga[(size_t)e]];
              bool later, same_cone = false;
              if (v >= g1) later = true;
              else if (v < g0) later = false;
              else {
                const int32_t kv = cone_of[(size_t)(v - g0)];
                same_cone = (kv == kr);
                later = kv > kr || (same_cone && v > r);
              }
              if (!later) continue;
              nnzc[(size_t)kr]++;
              if (!same_cone) tgts[(size_t)kr].push_back(v);
            }
          }
          ok = true;
          for (int64_t q = 0; q < K && ok; ++q) {
            auto& t = tgts[(size_t)q];
            std::sort(t.begin(), t.end());
            const int64_t w = rows[(size_t)q] + (int64_t)(std::unique(t.begin(), t.end()) - t.begin());
            if (rows[(size_t)q] > cfg.max_tile_rows || nnzc[(size_t)q] > cfg.max_tile_nnz || w > cfg.max_tile_window)
              ok = false;
          }
          if (!ok) {
            int64_t maxlvl = 0;
            for (int32_t l = l0; l < l1; ++l) maxlvl = std::max<int64_t>(maxlvl, S->level_ptr[(size_t)l + 1] - S->level_ptr[(size_t)l]);
            if (K >= maxlvl) break;  // cannot cut finer: fall back to contiguous chunks
            K = std::min<int64_t>(maxlvl, K + std::max<int64_t>(1, K / 5));
          }
        }
        if (!ok) continue;
        is_cone[(size_t)g] = 1;
        auto& ord = new_order[(size_t)g];
        ord.reserve((size_t)(g1 - g0));
        for (int64_t q = 0; q < K; ++q) {
          const size_t before = ord.size();
          for (int32_t l = l0; l < l1; ++l) {
            const auto& c = cuts[(size_t)(l - l0)];
            for (int32_t r = c[(size_t)q]; r < c[(size_t)q + 1]; ++r) ord.push_back(r);
          }
          if (ord.size() > before) cone_sizes[(size_t)g].push_back((int32_t)(ord.size() - before));
        }
      }
    }
    // final order: cone groups re-permuted, other groups unchanged
    std::vector<int32_t> fin((size_t)n);  // final position -> BFS position
    for (int32_t g = 0; g < ngroups; ++g) {
      const int32_t g0 = S->level_ptr[(size_t)S->group_lvl[(size_t)g]], g1 = S->level_ptr[(size_t)S->group_lvl[(size_t)g + 1]];
      if (is_cone[(size_t)g]) std::copy(new_order[(size_t)g].begin(), new_order[(size_t)g].end(), fin.begin() + g0);
      else for (int32_t r = g0; r < g1; ++r) fin[(size_t)r] = r;
    }
    std::vector<int32_t> inv2((size_t)n);
    for (int32_t f = 0; f < n; ++f) inv2[(size_t)f] = S->inv[(size_t)fin[(size_t)f]];
    S->inv.swap(inv2);
    for (int32_t f = 0; f < n; ++f) S->perm[(size_t)S->inv[(size_t)f]] = f;
    build_permuted();
    rp = S->prow_ptr.data();
    pc = S->pcol.data();
  }
  { std::vector<int64_t>().swap(gp); std::vector<int32_t>().swap(ga); }
  auto window_of = [&](int32_t r0, int32_t r1) -> int64_t {
    std::vector<int32_t> t;
    for (int32_t r = r0; r < r1; ++r)
      for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
        if (pc[i] >= r1) t.push_back(pc[i]);
    std::sort(t.begin(), t.end());
    return (int64_t)(r1 - r0) + (int64_t)(std::unique(t.begin(), t.end()) - t.begin());
  };
  {
    std::vector<std::vector<std::pair<int32_t, int32_t>>> per_group((size_t)ngroups);
    // K3/K4 tile block (capi.cpp build_tiled_host) bytes, upper bound:
    // descriptor + rseg 4 B/row + lcol 2 + val 8 + tcsc 4 B per entry +
    // tptr / sid 2+2 B and tgt 4 B per window slot
    auto est_block = [&](int32_t nr, int64_t tnnz, int64_t tw) { return 64 + 4 * (int64_t)nr + 14 * tnnz + 8 * tw + 96; };
    // split [a, b) in halves until every piece meets the row / nnz / window
    // caps and the block-byte budget
    auto split_fit = [&](int32_t a0, int32_t b0, int64_t budget, std::vector<std::pair<int32_t, int32_t>>& out) {
      std::vector<std::pair<int32_t, int32_t>> st{{a0, b0}};
      while (!st.empty()) {
        auto rg = st.back();
        st.pop_back();
        const int32_t nr = rg.second - rg.first;
        const int64_t tnnz = rp[rg.second] - rp[rg.first];
        const int64_t tw = nr <= cfg.max_tile_rows && tnnz <= cfg.max_tile_nnz ? window_of(rg.first, rg.second) : INT64_MAX;
        const bool fits = tw <= cfg.max_tile_window && est_block(nr, tnnz, tw) <= budget;
        if (fits || nr == 1) { out.push_back(rg); continue; }
        const int32_t mid = rg.first + nr / 2;
        st.push_back({mid, rg.second});
        st.push_back({rg.first, mid});
      }
    };
#pragma omp parallel for schedule(dynamic, 1)
    for (int32_t g = 0; g < ngroups; ++g) {
      int32_t r0 = S->level_ptr[(size_t)S->group_lvl[(size_t)g]];
      int32_t r1 = S->level_ptr[(size_t)S->group_lvl[(size_t)g + 1]];
      if (r1 <= r0) continue;
      if (is_cone[(size_t)g]) {
        int32_t a = r0;
        for (int32_t sz : cone_sizes[(size_t)g]) {
          per_group[(size_t)g].push_back({a, a + sz});
          a += sz;
        }
        continue;
      }
      int64_t gw = 0;
      for (int32_t r = r0; r < r1; ++r) gw += row_work(r);
      int64_t b = std::max<int64_t>(1, S->group_workers[(size_t)g]);
      std::vector<int32_t> cuts{r0};
      int64_t cum = 0;
      int64_t j = 1;
      for (int32_t r = r0; r < r1 && j < b; ++r) {
        cum += row_work(r);
        if (cum * b >= j * gw) {
          if (r + 1 > cuts.back() && r + 1 < r1) cuts.push_back(r + 1);
          ++j;
        }
      }
      cuts.push_back(r1);
      // caps (stack of ranges, split in half until they fit)
      std::vector<std::pair<int32_t, int32_t>> out;
      for (size_t c = 0; c + 1 < cuts.size(); ++c) split_fit(cuts[c], cuts[c + 1], INT64_MAX, out);
      per_group[(size_t)g] = out;
    }
    // block-byte budget: the kernel's ring holds `stages` x (block + x window);
    // aim at kRingStages stages with the largest window found, and split the
    // (few) tiles whose block would force a shallower ring
    {
      int64_t maxw = 0;
      std::vector<std::vector<int64_t>> tws((size_t)ngroups);
#pragma omp parallel for schedule(dynamic, 1) reduction(max : maxw)
      for (int32_t g = 0; g < ngroups; ++g)
        for (auto& rg : per_group[(size_t)g]) maxw = std::max<int64_t>(maxw, window_of(rg.first, rg.second));
      int64_t budget = kRingBytes / kRingStages - 8 * (((maxw + 2 + 15) / 16) * 16) - 128;
      if (block_budget > 0) budget = block_budget;  // SYMM_BLOCK_BUDGET (sweeps)
      budget = std::max<int64_t>(budget, 4096);
#pragma omp parallel for schedule(dynamic, 1)
      for (int32_t g = 0; g < ngroups; ++g) {
        std::vector<std::pair<int32_t, int32_t>> out;
        for (auto& rg : per_group[(size_t)g]) split_fit(rg.first, rg.second, budget, out);
        per_group[(size_t)g].swap(out);
      }
    }
    S->tile_ptr.clear();
    S->tile_group.clear();
    S->tile_ptr.push_back(0);
    for (int32_t g = 0; g < ngroups; ++g)
      for (auto& rg : per_group[(size_t)g]) {
        S->tile_ptr.push_back(rg.second);
        S->tile_group.push_back(g);
      }
    if (n > 0 && S->tile_ptr.back() != n) return set_error(SYMM_ERR_SCHEDULE, "tiles do not cover [0, n)");
  }
  const int32_t ntiles = (int32_t)S->tile_group.size();
  std::vector<int32_t> tile_of((size_t)n);
  for (int32_t t = 0; t < ntiles; ++t)
    for (int32_t r = S->tile_ptr[(size_t)t]; r < S->tile_ptr[(size_t)t + 1]; ++r) tile_of[(size_t)r] = t;

  // spill lists: sorted unique targets >= tile end (all targets are >= row)
  S->spill_ptr.assign((size_t)ntiles + 1, 0);
  std::vector<std::vector<int32_t>> spl((size_t)ntiles);
  int32_t maxwin = 0, maxrows = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(max : maxwin, maxrows)
  for (int32_t t = 0; t < ntiles; ++t) {
    int32_t r0 = S->tile_ptr[(size_t)t], r1 = S->tile_ptr[(size_t)t + 1];
    std::vector<int32_t>& v = spl[(size_t)t];
    for (int32_t r = r0; r < r1; ++r)
      for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
        if (pc[i] >= r1) v.push_back(pc[i]);
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    maxwin = std::max<int32_t>(maxwin, (r1 - r0) + (int32_t)v.size());
    maxrows = std::max<int32_t>(maxrows, r1 - r0);
  }
  S->max_window = maxwin;
  S->max_rows = maxrows;
  for (int32_t t = 0; t < ntiles; ++t) S->spill_ptr[(size_t)t + 1] = S->spill_ptr[(size_t)t] + (int64_t)spl[(size_t)t].size();
  S->spill.resize((size_t)S->spill_ptr[(size_t)ntiles]);
#pragma omp parallel for schedule(static)
  for (int32_t t = 0; t < ntiles; ++t)
    std::copy(spl[(size_t)t].begin(), spl[(size_t)t].end(), S->spill.begin() + S->spill_ptr[(size_t)t]);
  { std::vector<std::vector<int32_t>>().swap(spl); }

  // writers(c) for every target c: own tile + tiles whose spill contains c
  std::vector<int64_t> wptr((size_t)n + 1, 0);
  for (int32_t r = 0; r < n; ++r) wptr[(size_t)r + 1] = 1;
  for (int64_t q = 0; q < (int64_t)S->spill.size(); ++q) wptr[(size_t)S->spill[(size_t)q] + 1] += 1;
  for (int32_t r = 0; r < n; ++r) wptr[(size_t)r + 1] += wptr[(size_t)r];
  std::vector<int32_t> writers((size_t)wptr[(size_t)n]);
  {
    std::vector<int64_t> wpos(wptr.begin(), wptr.end() - 1);
    for (int32_t r = 0; r < n; ++r) writers[(size_t)wpos[(size_t)r]++] = tile_of[(size_t)r];
    for (int32_t t = 0; t < ntiles; ++t)  // ascending t => writer lists sorted
      for (int64_t q = S->spill_ptr[(size_t)t]; q < S->spill_ptr[(size_t)t + 1]; ++q)
        writers[(size_t)wpos[(size_t)S->spill[(size_t)q]]++] = t;
  }
  // tile conflict lists
  std::vector<std::vector<int32_t>> conf((size_t)ntiles);
#pragma omp parallel
  {
    std::vector<int32_t> stamp((size_t)ntiles, -1);
#pragma omp for schedule(dynamic, 16)
    for (int32_t t = 0; t < ntiles; ++t) {
      std::vector<int32_t>& v = conf[(size_t)t];
      auto visit = [&](int32_t c) {
        for (int64_t q = wptr[(size_t)c]; q < wptr[(size_t)c + 1]; ++q) {
          int32_t u = writers[(size_t)q];
          if (u != t && stamp[(size_t)u] != t) { stamp[(size_t)u] = t; v.push_back(u); }
        }
      };
      for (int32_t r = S->tile_ptr[(size_t)t]; r < S->tile_ptr[(size_t)t + 1]; ++r) visit(r);
      for (int64_t q = S->spill_ptr[(size_t)t]; q < S->spill_ptr[(size_t)t + 1]; ++q) visit(S->spill[(size_t)q]);
      std::sort(v.begin(), v.end());
    }
  }
  // tile coloring.  Any proper colouring of the tile conflict graph makes
  // every phase write-disjoint; the phase count is the
  // depth of the colored variants' dependency chain (K2: one launch per
  // phase; K8: the DAG's longest path).
  //  - scheme 0 (default): DSatur over all tiles at once (reading R34):
  //    st27_128 14 phases, fem_knn_4M 18, against 31 / 43 below;
  //  - flags bit 1, and schemes 1-3: the stage-0 structure, every red
  //    group's tiles before every blue group's, greedy in ascending tile id
  //    inside each stage-0 colour.
  std::vector<int32_t> tcol((size_t)ntiles, -1);
  int32_t ncol[2] = {0, 0};
  const bool dsatur = cfg.scheme == 0 && !(cfg.flags & 2u);
  if (dsatur) {
    // Brelaz: colour next the uncoloured tile with the most distinct colours
    // among its neighbours (ties: more neighbours, then the smaller id), with
    // the smallest colour none of them has
    std::vector<std::vector<uint64_t>> sat((size_t)ntiles);
    std::vector<int32_t> nsat((size_t)ntiles, 0);
    using Key = std::tuple<int32_t, int32_t, int32_t>;  // (saturation, degree, -id)
    std::priority_queue<Key> pq;
    for (int32_t t = 0; t < ntiles; ++t) pq.emplace(0, (int32_t)conf[(size_t)t].size(), -t);
    auto has = [&](int32_t u, int32_t c) {
      const auto& w = sat[(size_t)u];
      return (size_t)(c >> 6) < w.size() && ((w[(size_t)(c >> 6)] >> (c & 63)) & 1u);
    };
    int32_t nc = 0;
    while (!pq.empty()) {
      const auto [sv, dv, mt] = pq.top();
      pq.pop();
      const int32_t t = -mt;
      if (tcol[(size_t)t] >= 0 || sv != nsat[(size_t)t]) continue;  // stale entry
      int32_t c = 0;
      while (has(t, c)) ++c;
      tcol[(size_t)t] = c;
      nc = std::max(nc, c + 1);
      for (int32_t u : conf[(size_t)t]) {
        if (tcol[(size_t)u] >= 0 || has(u, c)) continue;
        auto& w = sat[(size_t)u];
        if (w.size() <= (size_t)(c >> 6)) w.resize((size_t)(c >> 6) + 1, 0);
        w[(size_t)(c >> 6)] |= uint64_t(1) << (c & 63);
        pq.emplace(++nsat[(size_t)u], (int32_t)conf[(size_t)u].size(), -u);
      }
    }
    { std::vector<std::vector<uint64_t>>().swap(sat); }
    ncol[0] = nc;
    // Equitable rebalancing (flags bit 2 turns it off).  DSatur fills the
    // first colours greedily, so the last ones are small (st27_128: 2281 ...
    // 39, 1 tiles).  K8 runs the phases in order with every tile waiting for
    // its conflicting tiles of earlier phases: small phases at the end form a
    // chain with less than one wave of tiles per link, and a tile at the start
    // of a phase finds its predecessors less than one wave back.  A tile moves
    // from a colour above the mean size to the smallest colour that none of its
    // conflicting tiles has, if that colour is smaller by two or more; sweeps
    // in id order until nothing moves.  The colouring stays proper.
    if (!(cfg.flags & 4u) && nc > 1) {
      std::vector<int64_t> size((size_t)nc, 0);
      for (int32_t t = 0; t < ntiles; ++t) size[(size_t)tcol[(size_t)t]]++;
      const int64_t target = (ntiles + nc - 1) / nc;
      std::vector<int32_t> seen((size_t)nc, -1);
      for (int sweep = 0; sweep < 16; ++sweep) {
        int64_t moved = 0;
        for (int32_t t = 0; t < ntiles; ++t) {
          const int32_t c = tcol[(size_t)t];
          if (size[(size_t)c] <= target) continue;
          for (int32_t u : conf[(size_t)t]) seen[(size_t)tcol[(size_t)u]] = t;
          int32_t best = -1;
          for (int32_t d = 0; d < nc; ++d)
            if (seen[(size_t)d] != t && d != c && size[(size_t)d] + 2 <= size[(size_t)c] &&
                (best < 0 || size[(size_t)d] < size[(size_t)best]))
              best = d;
          if (best >= 0) {
            tcol[(size_t)t] = best;
            size[(size_t)c]--;
            size[(size_t)best]++;
            ++moved;
          }
        }
        if (moved == 0) break;
      }
    }
  }
  for (int32_t t = 0; t < ntiles && !dsatur; ++t) {
    int32_t s0 = S->tile_group[(size_t)t] % 2;
    std::vector<char> used;
    for (int32_t u : conf[(size_t)t]) {
      if (u >= t || S->tile_group[(size_t)u] % 2 != s0) continue;
      int32_t c = tcol[(size_t)u];
      if (c >= (int32_t)used.size()) used.resize((size_t)c + 1, 0);
      used[(size_t)c] = 1;
    }
    int32_t c = 0;
    while (c < (int32_t)used.size() && used[(size_t)c]) ++c;
    tcol[(size_t)t] = c;
    ncol[s0] = std::max(ncol[s0], c + 1);
  }
  S->tile_phase.assign((size_t)ntiles, 0);
  for (int32_t t = 0; t < ntiles; ++t)
    S->tile_phase[(size_t)t] = (dsatur || S->tile_group[(size_t)t] % 2 == 0) ? tcol[(size_t)t] : ncol[0] + tcol[(size_t)t];
  S->n_phases = ncol[0] + ncol[1];
  // DAG: u waits for every conflicting tile of an earlier phase
  S->dag_ptr.assign((size_t)ntiles + 1, 0);
  S->dag_pred.clear();
  for (int32_t t = 0; t < ntiles; ++t) {
    for (int32_t u : conf[(size_t)t])
      if (S->tile_phase[(size_t)u] < S->tile_phase[(size_t)t]) S->dag_pred.push_back(u);
      else if (S->tile_phase[(size_t)u] == S->tile_phase[(size_t)t])
        return set_error(SYMM_ERR_SCHEDULE, "conflicting tiles %d and %d share phase %d", t, u, S->tile_phase[(size_t)t]);
    S->dag_ptr[(size_t)t + 1] = (int32_t)S->dag_pred.size();
  }
  { std::vector<std::vector<int32_t>>().swap(conf); }
  // claim order: Kahn topological sort, smallest tile id first
  {
    std::vector<int32_t> indeg((size_t)ntiles), succ_ptr((size_t)ntiles + 1, 0), succ(S->dag_pred.size());
    for (int32_t t = 0; t < ntiles; ++t) {
      indeg[(size_t)t] = S->dag_ptr[(size_t)t + 1] - S->dag_ptr[(size_t)t];
      for (int32_t q = S->dag_ptr[(size_t)t]; q < S->dag_ptr[(size_t)t + 1]; ++q) succ_ptr[(size_t)S->dag_pred[(size_t)q] + 1]++;
    }
    for (int32_t t = 0; t < ntiles; ++t) succ_ptr[(size_t)t + 1] += succ_ptr[(size_t)t];
    std::vector<int32_t> sp(succ_ptr.begin(), succ_ptr.end() - 1);
    for (int32_t t = 0; t < ntiles; ++t)
      for (int32_t q = S->dag_ptr[(size_t)t]; q < S->dag_ptr[(size_t)t + 1]; ++q) succ[(size_t)sp[(size_t)S->dag_pred[(size_t)q]]++] = t;
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> pq;
    for (int32_t t = 0; t < ntiles; ++t)
      if (indeg[(size_t)t] == 0) pq.push(t);
    S->tile_order.clear();
    while (!pq.empty()) {
      int32_t t = pq.top();
      pq.pop();
      S->tile_order.push_back(t);
      for (int32_t q = succ_ptr[(size_t)t]; q < succ_ptr[(size_t)t + 1]; ++q)
        if (--indeg[(size_t)succ[(size_t)q]] == 0) pq.push(succ[(size_t)q]);
    }
    if ((int32_t)S->tile_order.size() != ntiles) return set_error(SYMM_ERR_SCHEDULE, "tile DAG has a cycle");
  }
  // first writer of every target = its writer of minimal phase (distinct phases)
  std::vector<int32_t> minphase((size_t)n, INT32_MAX);
#pragma omp parallel for schedule(static)
  for (int32_t c = 0; c < n; ++c) {
    int32_t m = INT32_MAX;
    for (int64_t q = wptr[(size_t)c]; q < wptr[(size_t)c + 1]; ++q) m = std::min(m, S->tile_phase[(size_t)writers[(size_t)q]]);
    minphase[(size_t)c] = m;
  }
  if (cfg.validate) {
    // stamping validator 1: writers of every target have pairwise distinct phases
    int32_t bad = -1;
#pragma omp parallel for schedule(dynamic, 4096) reduction(max : bad)
    for (int32_t c = 0; c < n; ++c) {
      std::vector<int32_t> ph;
      for (int64_t q = wptr[(size_t)c]; q < wptr[(size_t)c + 1]; ++q) ph.push_back(S->tile_phase[(size_t)writers[(size_t)q]]);
      std::sort(ph.begin(), ph.end());
      for (size_t i = 1; i < ph.size(); ++i)
        if (ph[i] == ph[i - 1]) bad = std::max(bad, c);
    }
    if (bad >= 0) return set_error(SYMM_ERR_SCHEDULE, "validator: target %d written twice in one phase", bad);
  }
  S->own_first.assign((size_t)n, 0);
#pragma omp parallel for schedule(static)
  for (int32_t r = 0; r < n; ++r)
    S->own_first[(size_t)r] = (uint8_t)(S->tile_phase[(size_t)tile_of[(size_t)r]] == minphase[(size_t)r]);
#pragma omp parallel for schedule(dynamic, 16)
  for (int32_t t = 0; t < ntiles; ++t)
    for (int64_t q = S->spill_ptr[(size_t)t]; q < S->spill_ptr[(size_t)t + 1]; ++q) {
      int32_t c = S->spill[(size_t)q];
      if (S->tile_phase[(size_t)t] == minphase[(size_t)c]) S->spill[(size_t)q] = (int32_t)((uint32_t)c | kFirstBit);
    }
  { std::vector<int64_t>().swap(wptr); std::vector<int32_t>().swap(writers); std::vector<int32_t>().swap(minphase); }

  // ---- intra-tile distance-2 row coloring (write-set disjoint colors) ----------
  S->row_subcolor.assign((size_t)n, 0);
  S->srow.assign((size_t)n, 0);
  std::vector<std::vector<int32_t>> subp((size_t)ntiles);
  int bad_tile = -1;
#pragma omp parallel for schedule(dynamic, 4) reduction(max : bad_tile)
  for (int32_t t = 0; t < ntiles; ++t) {
    const int32_t r0 = S->tile_ptr[(size_t)t], r1 = S->tile_ptr[(size_t)t + 1], T = r1 - r0;
    const int32_t* sp = S->spill.data() + S->spill_ptr[(size_t)t];
    const int64_t ns = S->spill_ptr[(size_t)t + 1] - S->spill_ptr[(size_t)t];
    auto local = [&](int32_t c) -> int64_t {
      if (c < r1) return c - r0;
      int64_t lo = 0, hi = ns;
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if ((int32_t)((uint32_t)sp[mid] & kIdxMask) < c) lo = mid + 1;
        else hi = mid;
      }
      return T + lo;
    };
    // colour masks, layout m[l * nw + word]; grown when a row needs colour >= 64*nw
    const size_t W = (size_t)T + (size_t)ns;
    size_t nw = 1;
    std::vector<uint64_t> m(W, 0);
    int32_t ncolors = 0;
    std::vector<int64_t> tg;
    for (int32_t r = r0; r < r1; ++r) {
      tg.clear();
      tg.push_back(r - r0);
      for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
        if (pc[i] != r) tg.push_back(local(pc[i]));
      int32_t color = -1;
      for (size_t word = 0; color < 0; ++word) {
        if (word == nw) {
          if (nw >= 16) { bad_tile = std::max(bad_tile, t); color = 0; break; }
          std::vector<uint64_t> m2(W * (nw + 1), 0);
          for (size_t l = 0; l < W; ++l)
            for (size_t w = 0; w < nw; ++w) m2[l * (nw + 1) + w] = m[l * nw + w];
          m.swap(m2);
          ++nw;
        }
        uint64_t forbid = 0;
        for (int64_t l : tg) forbid |= m[(size_t)l * nw + word];
        if (~forbid) {
          int32_t bit = __builtin_ctzll(~forbid);
          color = (int32_t)(word * 64) + bit;
          for (int64_t l : tg) m[(size_t)l * nw + word] |= (uint64_t(1) << bit);
        }
      }
      S->row_subcolor[(size_t)r] = color;
      ncolors = std::max(ncolors, color + 1);
    }
    // stored-row order: by (color, row); colour pointers relative to r0
    std::vector<int32_t> cnt((size_t)ncolors + 1, 0);
    for (int32_t r = r0; r < r1; ++r) cnt[(size_t)S->row_subcolor[(size_t)r] + 1]++;
    for (int32_t c = 0; c < ncolors; ++c) cnt[(size_t)c + 1] += cnt[(size_t)c];
    subp[(size_t)t] = cnt;
    std::vector<int32_t> pos(cnt.begin(), cnt.end() - 1);
    for (int32_t r = r0; r < r1; ++r) S->srow[(size_t)(r0 + pos[(size_t)S->row_subcolor[(size_t)r]]++)] = r;
    if (cfg.validate) {
      // stamping validator 2: inside one colour every local target is written once
      std::vector<int32_t> st(W, -1);
      for (int32_t c = 0; c < ncolors; ++c)
        for (int32_t q = cnt[(size_t)c]; q < cnt[(size_t)c + 1]; ++q) {
          int32_t r = S->srow[(size_t)(r0 + q)];
          auto stamp = [&](int64_t l) {
            if (st[(size_t)l] == c) bad_tile = std::max(bad_tile, t);
            st[(size_t)l] = c;
          };
          stamp(r - r0);
          for (int32_t i = rp[r]; i < rp[r + 1]; ++i)
            if (pc[i] != r) stamp(local(pc[i]));
        }
    }
  }
  if (bad_tile >= 0) return set_error(SYMM_ERR_SCHEDULE, "validator: intra-tile colouring of tile %d invalid", bad_tile);
  S->tile_sub_ptr.assign((size_t)ntiles + 1, 0);
  for (int32_t t = 0; t < ntiles; ++t) S->tile_sub_ptr[(size_t)t + 1] = S->tile_sub_ptr[(size_t)t] + (int32_t)subp[(size_t)t].size();
  S->sub_ptr.resize((size_t)S->tile_sub_ptr[(size_t)ntiles]);
  int64_t sum_sub = 0;
  S->max_subcolors = 0;
  for (int32_t t = 0; t < ntiles; ++t) {
    std::copy(subp[(size_t)t].begin(), subp[(size_t)t].end(), S->sub_ptr.begin() + S->tile_sub_ptr[(size_t)t]);
    int32_t ns = (int32_t)subp[(size_t)t].size() - 1;
    sum_sub += ns;
    S->max_subcolors = std::max(S->max_subcolors, ns);
  }
  S->mean_subcolors = ntiles ? (double)sum_sub / ntiles : 0.0;

  // ---- §5 efficiency of the tile tree (work = balance unit) --------------------
  {
    // nrowsEff(group) = sum over tile colours of the max tile work of that colour;
    // nrowsEff(root) = max over red groups + max over blue groups
    std::vector<std::vector<int64_t>> gmax((size_t)ngroups);
    for (int32_t t = 0; t < ntiles; ++t) {
      int64_t w = 0;
      for (int32_t r = S->tile_ptr[(size_t)t]; r < S->tile_ptr[(size_t)t + 1]; ++r) w += row_work(r);
      auto& v = gmax[(size_t)S->tile_group[(size_t)t]];
      size_t c = (size_t)tcol[(size_t)t];
      if (v.size() <= c) v.resize(c + 1, 0);
      v[c] = std::max(v[c], w);
    }
    int64_t red = 0, blue = 0;
    for (int32_t g = 0; g < ngroups; ++g) {
      int64_t e = 0;
      for (int64_t w : gmax[(size_t)g]) e += w;
      if (g % 2 == 0) red = std::max(red, e);
      else blue = std::max(blue, e);
    }
    int64_t eff = red + blue;
    S->eta = (eff > 0 && ntiles > 0) ? (double)total_work / ((double)eff * (double)ntiles) : 1.0;
  }
  if (cfg.scheme == 3) S->eta = S->tree_eta;  // the recursive tree's own §5 eta
  S->build_seconds = now_s() - t0;
  return SYMM_OK;
}

}  // namespace symm
