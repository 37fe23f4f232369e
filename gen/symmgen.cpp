// Seeded synthetic input generators for the five BASELINE.json configs (and
// small test graphs).  This module is shared by the oracle side (tests) and the
// product side (bench); it holds NO SymmSpMV / RACE arithmetic: it only builds
// upper-triangular CRS matrices (diagonal first, strictly ascending columns)
// and input vectors, deterministically from a seed, independent of the number
// of OpenMP threads.
//
// Random numbers: counter-based SplitMix64 (reading R22):
//   u01(seed, key) = (splitmix64(seed ^ splitmix64(key)) >> 11) * 2^-53
// Edge values are keyed by the ORIGINAL (min(i,j), max(i,j)) pair, so they
// do not depend on storage order or thread count.
//
// Matrix shapes follow BASELINE.json `configs` with the readings in
// SURVEY.md §8(c) c19-c22 (restated in DESIGN.md "input recipe").
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>

namespace {

inline uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
inline double u01(uint64_t seed, uint64_t key) {
  return (double)(splitmix64(seed ^ splitmix64(key)) >> 11) * 0x1.0p-53;
}
// Domain separation between the different random streams of one config.
constexpr uint64_t S_EDGE = 0x0123456789abcdefULL;
constexpr uint64_t S_DIAG = 0x1f2e3d4c5b6a7988ULL;
constexpr uint64_t S_PERM = 0x5555aaaa3333ccccULL;
constexpr uint64_t S_PNT = 0x0f0f0f0ff0f0f0f0ULL;
constexpr uint64_t S_VEC = 0x7a7a7a7a1b1b1b1bULL;

inline uint64_t pair_key(uint64_t a, uint64_t b, uint64_t n) {
  uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
  return lo * n + hi;
}

struct Csr {
  int32_t n = 0;
  int64_t nnz = 0;
  int32_t* row_ptr = nullptr;
  int32_t* col = nullptr;
  double* val = nullptr;
  ~Csr() {
    std::free(row_ptr);
    std::free(col);
    std::free(val);
  }
  bool alloc(int64_t n_, int64_t nnz_) {
    if (n_ < 0 || n_ >= (int64_t(1) << 31) || nnz_ >= (int64_t(1) << 31)) return false;
    n = (int32_t)n_;
    nnz = nnz_;
    row_ptr = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)(n_ + 1));
    col = (int32_t*)std::malloc(sizeof(int32_t) * (size_t)std::max<int64_t>(nnz_, 1));
    val = (double*)std::malloc(sizeof(double) * (size_t)std::max<int64_t>(nnz_, 1));
    return row_ptr && col && val;
  }
};

// Build an upper CRS from per-row counts + a row filler (parallel, deterministic).
template <class CountF, class FillF>
Csr* build_rows(int64_t n, CountF count, FillF fill) {
  std::vector<int64_t> cnt((size_t)n + 1, 0);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) cnt[(size_t)r + 1] = count(r);
  for (int64_t r = 0; r < n; ++r) cnt[(size_t)r + 1] += cnt[(size_t)r];
  Csr* A = new Csr();
  if (!A->alloc(n, cnt[(size_t)n])) {
    delete A;
    return nullptr;
  }
  for (int64_t r = 0; r <= n; ++r) A->row_ptr[r] = (int32_t)cnt[(size_t)r];
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t r = 0; r < n; ++r) fill(r, A->col + cnt[(size_t)r], A->val + cnt[(size_t)r]);
  return A;
}

}  // namespace

extern "C" {

// ---- handle accessors -------------------------------------------------------
int32_t gen_n(void* h) { return ((Csr*)h)->n; }
int64_t gen_nnz(void* h) { return ((Csr*)h)->nnz; }
int32_t* gen_row_ptr(void* h) { return ((Csr*)h)->row_ptr; }
int32_t* gen_col(void* h) { return ((Csr*)h)->col; }
double* gen_val(void* h) { return ((Csr*)h)->val; }
void gen_free(void* h) { delete (Csr*)h; }

// ---- config 1: 2-D 5-point Laplacian, N x N, diag 4, off -1, natural order --
void* gen_lap2d(int32_t N) {
  const int64_t n = (int64_t)N * N;
  auto count = [=](int64_t r) -> int64_t {
    int64_t i = r / N, j = r % N;
    return 1 + (j + 1 < N) + (i + 1 < N);
  };
  auto fill = [=](int64_t r, int32_t* c, double* v) {
    int64_t i = r / N, j = r % N;
    int k = 0;
    c[k] = (int32_t)r; v[k++] = 4.0;
    if (j + 1 < N) { c[k] = (int32_t)(r + 1); v[k++] = -1.0; }
    if (i + 1 < N) { c[k] = (int32_t)(r + N); v[k++] = -1.0; }
  };
  return build_rows(n, count, fill);
}

// ---- config 5: 3-D 7-point Laplacian N^3, diag 6+d, off -1+d, d~U(-.01,.01)
// keyed per stored upper entry (r,c); perturb=0 gives the exact 6/-1 stencil.
void* gen_lap3d(int32_t N, uint64_t seed, int32_t perturb) {
  const int64_t n = (int64_t)N * N * N;
  const int64_t NN = (int64_t)N * N;
  auto delta = [=](int64_t r, int64_t c) -> double {
    return perturb ? 0.02 * u01(seed ^ S_EDGE, pair_key(r, c, n)) - 0.01 : 0.0;
  };
  auto count = [=](int64_t r) -> int64_t {
    int64_t k = r % N, j = (r / N) % N, i = r / NN;
    return 1 + (k + 1 < N) + (j + 1 < N) + (i + 1 < N);
  };
  auto fill = [=](int64_t r, int32_t* c, double* v) {
    int64_t k = r % N, j = (r / N) % N, i = r / NN;
    int q = 0;
    c[q] = (int32_t)r; v[q++] = 6.0 + delta(r, r);
    if (k + 1 < N) { c[q] = (int32_t)(r + 1); v[q++] = -1.0 + delta(r, r + 1); }
    if (j + 1 < N) { c[q] = (int32_t)(r + N); v[q++] = -1.0 + delta(r, r + N); }
    if (i + 1 < N) { c[q] = (int32_t)(r + NN); v[q++] = -1.0 + delta(r, r + NN); }
  };
  return build_rows(n, count, fill);
}

// ---- config 4: spin-chain-like Hamiltonian, n = 2^L ------------------------
// row i couples to i XOR (3 << b), b = 0..L-2, value 0.5; diag ~ U(-2,2) keyed by i.
void* gen_spin(int32_t L, uint64_t seed) {
  if (L < 1 || L > 30) return nullptr;
  const int64_t n = int64_t(1) << L;
  auto count = [=](int64_t r) -> int64_t {
    int64_t c = 1;
    for (int b = 0; b + 1 < L; ++b) c += ((r ^ (int64_t(3) << b)) > r);
    return c;
  };
  auto fill = [=](int64_t r, int32_t* c, double* v) {
    int q = 0;
    c[q] = (int32_t)r; v[q++] = 4.0 * u01(seed ^ S_DIAG, (uint64_t)r) - 2.0;
    int32_t tmp[64];
    int m = 0;
    for (int b = 0; b + 1 < L; ++b) {
      int64_t j = r ^ (int64_t(3) << b);
      if (j > r) tmp[m++] = (int32_t)j;
    }
    std::sort(tmp, tmp + m);
    for (int t = 0; t < m; ++t) { c[q] = tmp[t]; v[q++] = 0.5; }
  };
  return build_rows(n, count, fill);
}

// ---- config 2: 3-D 27-point stencil on N^3, off-diag ~ U(-1,0) keyed per edge,
// diag = sum|a| + 1, then a seeded symmetric random shuffle P A P^T (reading c21).
void* gen_st27(int32_t N, uint64_t seed, int32_t shuffle) {
  const int64_t n = (int64_t)N * N * N;
  const int64_t NN = (int64_t)N * N;
  // arr[new] = old ; newidx[old] = new
  std::vector<int32_t> arr((size_t)n), newidx((size_t)n);
  for (int64_t i = 0; i < n; ++i) arr[(size_t)i] = (int32_t)i;
  if (shuffle) {
    for (int64_t i = n - 1; i >= 1; --i) {
      int64_t j = (int64_t)(u01(seed ^ S_PERM, (uint64_t)i) * (double)(i + 1));
      if (j > i) j = i;
      std::swap(arr[(size_t)i], arr[(size_t)j]);
    }
  }
  for (int64_t i = 0; i < n; ++i) newidx[(size_t)arr[(size_t)i]] = (int32_t)i;
  auto edge_val = [=](int64_t a, int64_t b) -> double {
    return -u01(seed ^ S_EDGE, pair_key(a, b, n));
  };
  auto nbrs = [=](int64_t o, int64_t* out) -> int {
    int64_t k = o % N, j = (o / N) % N, i = o / NN;
    int m = 0;
    for (int di = -1; di <= 1; ++di)
      for (int dj = -1; dj <= 1; ++dj)
        for (int dk = -1; dk <= 1; ++dk) {
          if (!di && !dj && !dk) continue;
          int64_t ii = i + di, jj = j + dj, kk = k + dk;
          if (ii < 0 || jj < 0 || kk < 0 || ii >= N || jj >= N || kk >= N) continue;
          out[m++] = (ii * N + jj) * N + kk;
        }
    return m;
  };
  const int32_t* A_arr = arr.data();
  const int32_t* A_new = newidx.data();
  auto count = [=](int64_t r) -> int64_t {
    int64_t nb[26];
    int m = nbrs(A_arr[r], nb);
    int64_t c = 1;
    for (int t = 0; t < m; ++t) c += (A_new[nb[t]] > r);
    return c;
  };
  auto fill = [=](int64_t r, int32_t* c, double* v) {
    int64_t o = A_arr[r];
    int64_t nb[26];
    int m = nbrs(o, nb);
    double dsum = 1.0;
    std::pair<int32_t, double> tmp[26];
    int q = 0;
    for (int t = 0; t < m; ++t) {
      double a = edge_val(o, nb[t]);
      dsum += std::fabs(a);
      int32_t cn = A_new[nb[t]];
      if (cn > r) tmp[q++] = {cn, a};
    }
    std::sort(tmp, tmp + q);
    c[0] = (int32_t)r; v[0] = dsum;
    for (int t = 0; t < q; ++t) { c[t + 1] = tmp[t].first; v[t + 1] = tmp[t].second; }
  };
  return build_rows(n, count, fill);
}

// ---- config 3: FEM-like kNN graph --------------------------------------------
// npts points ~ U[0,1)^3 (seed), each joined to its k nearest neighbours (ties by
// index), union-symmetrised; off-diag ~ U(-1,1) keyed per edge; diag = sum|a|+1.
// The vertex order is the (random) point index order.
void* gen_knn(int32_t npts, int32_t k, uint64_t seed) {
  const int64_t n = npts;
  if (n <= 0 || k <= 0 || k >= n) return nullptr;
  std::vector<double> P((size_t)n * 3);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) P[(size_t)(3 * i + d)] = u01(seed ^ S_PNT, (uint64_t)(3 * i + d));
  int64_t G = (int64_t)std::ceil(std::cbrt((double)n / 2.0));
  if (G < 1) G = 1;
  const double h = 1.0 / (double)G;
  auto cell_of = [&](double x) -> int64_t {
    int64_t c = (int64_t)(x * (double)G);
    return c < 0 ? 0 : (c >= G ? G - 1 : c);
  };
  const int64_t ncell = G * G * G;
  std::vector<int64_t> cstart((size_t)ncell + 1, 0);
  std::vector<int32_t> cell_pts((size_t)n);
  std::vector<int64_t> pc((size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = (cell_of(P[3 * i]) * G + cell_of(P[3 * i + 1])) * G + cell_of(P[3 * i + 2]);
    pc[(size_t)i] = c;
    cstart[(size_t)c + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) cstart[(size_t)c + 1] += cstart[(size_t)c];
  {
    std::vector<int64_t> fillp(cstart.begin(), cstart.end() - 1);
    for (int64_t i = 0; i < n; ++i) cell_pts[(size_t)fillp[(size_t)pc[(size_t)i]]++] = (int32_t)i;
  }
  std::vector<int32_t> knn((size_t)n * k);
#pragma omp parallel
  {
    std::vector<std::pair<double, int32_t>> heap;
    heap.reserve((size_t)k + 1);
#pragma omp for schedule(dynamic, 1024)
    for (int64_t i = 0; i < n; ++i) {
      heap.clear();
      const double px = P[3 * i], py = P[3 * i + 1], pz = P[3 * i + 2];
      const int64_t cx = cell_of(px), cy = cell_of(py), cz = cell_of(pz);
      for (int64_t R = 0; R < G; ++R) {
        for (int64_t ax = cx - R; ax <= cx + R; ++ax) {
          if (ax < 0 || ax >= G) continue;
          for (int64_t ay = cy - R; ay <= cy + R; ++ay) {
            if (ay < 0 || ay >= G) continue;
            for (int64_t az = cz - R; az <= cz + R; ++az) {
              if (az < 0 || az >= G) continue;
              int64_t ring = std::max(std::max(std::llabs(ax - cx), std::llabs(ay - cy)), std::llabs(az - cz));
              if (ring != R) continue;
              int64_t c = (ax * G + ay) * G + az;
              for (int64_t t = cstart[(size_t)c]; t < cstart[(size_t)c + 1]; ++t) {
                int32_t j = cell_pts[(size_t)t];
                if (j == i) continue;
                double dx = P[3 * (size_t)j] - px, dy = P[3 * (size_t)j + 1] - py, dz = P[3 * (size_t)j + 2] - pz;
                std::pair<double, int32_t> e{dx * dx + dy * dy + dz * dz, j};
                if ((int)heap.size() < k) {
                  heap.push_back(e);
                  std::push_heap(heap.begin(), heap.end());
                } else if (e < heap.front()) {
                  std::pop_heap(heap.begin(), heap.end());
                  heap.back() = e;
                  std::push_heap(heap.begin(), heap.end());
                }
              }
            }
          }
        }
        if ((int)heap.size() == k) {
          // distance from p to the outside of the searched (2R+1)^3 cell block
          double bound = 1e300;
          if (cx - R > 0) bound = std::min(bound, px - (double)(cx - R) * h);
          if (cx + R + 1 < G) bound = std::min(bound, (double)(cx + R + 1) * h - px);
          if (cy - R > 0) bound = std::min(bound, py - (double)(cy - R) * h);
          if (cy + R + 1 < G) bound = std::min(bound, (double)(cy + R + 1) * h - py);
          if (cz - R > 0) bound = std::min(bound, pz - (double)(cz - R) * h);
          if (cz + R + 1 < G) bound = std::min(bound, (double)(cz + R + 1) * h - pz);
          if (bound >= 1e299 || heap.front().first < bound * bound) break;
        }
      }
      std::sort_heap(heap.begin(), heap.end());
      for (int t = 0; t < k; ++t) knn[(size_t)(i * k + t)] = heap[(size_t)t].second;
    }
  }
  // union symmetrisation: full adjacency = knn(i) ∪ {j : i ∈ knn(j)}
  std::vector<int64_t> rptr((size_t)n + 1, 0);
  for (int64_t i = 0; i < n; ++i)
    for (int t = 0; t < k; ++t) rptr[(size_t)knn[(size_t)(i * k + t)] + 1]++;
  for (int64_t i = 0; i < n; ++i) rptr[(size_t)i + 1] += rptr[(size_t)i];
  std::vector<int32_t> rev((size_t)rptr[(size_t)n]);
  {
    std::vector<int64_t> fp(rptr.begin(), rptr.end() - 1);
    for (int64_t i = 0; i < n; ++i)
      for (int t = 0; t < k; ++t) {
        int32_t j = knn[(size_t)(i * k + t)];
        rev[(size_t)fp[(size_t)j]++] = (int32_t)i;
      }
  }
  // per-row sorted unique full neighbour list (two passes: sizes, then fill)
  auto row_union = [&](int64_t i, std::vector<int32_t>& tmp) {
    tmp.clear();
    for (int t = 0; t < k; ++t) tmp.push_back(knn[(size_t)(i * k + t)]);
    for (int64_t t = rptr[(size_t)i]; t < rptr[(size_t)i + 1]; ++t) tmp.push_back(rev[(size_t)t]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
  };
  std::vector<int64_t> fptr((size_t)n + 1, 0);
#pragma omp parallel
  {
    std::vector<int32_t> tmp;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      row_union(i, tmp);
      fptr[(size_t)i + 1] = (int64_t)tmp.size();
    }
  }
  for (int64_t i = 0; i < n; ++i) fptr[(size_t)i + 1] += fptr[(size_t)i];
  std::vector<int32_t> full((size_t)fptr[(size_t)n]);
#pragma omp parallel
  {
    std::vector<int32_t> tmp;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      row_union(i, tmp);
      std::copy(tmp.begin(), tmp.end(), full.begin() + fptr[(size_t)i]);
    }
  }
  const int32_t* F = full.data();
  const int64_t* FP = fptr.data();
  auto edge_val = [=](int64_t a, int64_t b) -> double {
    return 2.0 * u01(seed ^ S_EDGE, pair_key(a, b, n)) - 1.0;
  };
  auto count = [=](int64_t r) -> int64_t {
    int64_t c = 1;
    for (int64_t t = FP[r]; t < FP[r + 1]; ++t) c += (F[t] > r);
    return c;
  };
  auto fill = [=](int64_t r, int32_t* c, double* v) {
    double dsum = 1.0;
    int q = 1;
    for (int64_t t = FP[r]; t < FP[r + 1]; ++t) {
      double a = edge_val(r, F[t]);
      dsum += std::fabs(a);
      if (F[t] > r) { c[q] = F[t]; v[q++] = a; }
    }
    c[0] = (int32_t)r; v[0] = dsum;
  };
  return build_rows(n, count, fill);
}

// ---- general: upper CRS from an explicit symmetric edge list (tests) --------
// edges (u[e], v[e]) with u != v, each undirected edge listed once (either
// orientation); off-diag value w[e]; diagonal d[i] (has_diag[i] != 0 keeps it).
void* gen_from_edges(int32_t n, int64_t m, const int32_t* u, const int32_t* v, const double* w,
                     const double* d, const int8_t* has_diag) {
  std::vector<int64_t> cnt((size_t)n + 1, 0);
  for (int64_t e = 0; e < m; ++e) {
    int32_t a = std::min(u[e], v[e]);
    cnt[(size_t)a + 1]++;
  }
  for (int32_t i = 0; i < n; ++i) cnt[(size_t)i + 1] += (has_diag[i] != 0);
  for (int32_t i = 0; i < n; ++i) cnt[(size_t)i + 1] += cnt[(size_t)i];
  Csr* A = new Csr();
  if (!A->alloc(n, cnt[(size_t)n])) { delete A; return nullptr; }
  std::vector<std::vector<std::pair<int32_t, double>>> rows((size_t)n);
  for (int64_t e = 0; e < m; ++e) {
    int32_t a = std::min(u[e], v[e]), b = std::max(u[e], v[e]);
    rows[(size_t)a].push_back({b, w[e]});
  }
  for (int32_t i = 0; i < n; ++i) {
    int64_t p = cnt[(size_t)i];
    A->row_ptr[i] = (int32_t)p;
    if (has_diag[i]) { A->col[p] = i; A->val[p] = d[i]; ++p; }
    std::sort(rows[(size_t)i].begin(), rows[(size_t)i].end());
    for (auto& e : rows[(size_t)i]) { A->col[p] = e.first; A->val[p] = e.second; ++p; }
  }
  A->row_ptr[n] = (int32_t)cnt[(size_t)n];
  return A;
}

// ---- vectors ------------------------------------------------------------------
// x_i ~ U(lo, hi) keyed by (seed, i)
void gen_vector_uniform(int64_t n, uint64_t seed, double lo, double hi, double* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * u01(seed ^ S_VEC, (uint64_t)i);
}
// x_ij = sin(pi i/(N+1)) sin(pi j/(N+1)), i,j = 1..N, row = (i-1) N + (j-1)
void gen_vector_sinsin(int32_t N, double* out) {
  const double pi = 3.14159265358979323846;
  for (int32_t i = 1; i <= N; ++i)
    for (int32_t j = 1; j <= N; ++j)
      out[(int64_t)(i - 1) * N + (j - 1)] = std::sin(pi * i / (N + 1)) * std::sin(pi * j / (N + 1));
}
int gen_num_threads(void) { return omp_get_max_threads(); }

}  // extern "C"
