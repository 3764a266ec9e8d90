// bmg_oracle.cpp -- CPU ORACLE: a plain-C++ restatement of the reference hot path.
//
// TEST INFRASTRUCTURE ONLY.  This file restates the algorithms of the reference
// C++ library (arXiv 2509.06744, `blockmg` 0.1.0, /root/reference/proj) without
// Eigen, so the CUDA product can be checked against it.  It is loaded only by
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.  The product
// (paper_2509_06744_b200/libbmgcuda.so) never links or calls it.
//
// Parity: pinned to the reference run here.  The reference's own build needs Eigen3
// (absent), so its unmodified sources are compiled in place against
// oracle/eigen_shim into oracle/_ref/libblockmg_ref.so (same C API,
// ref_driver.cpp) and compared with this file BITWISE
// (tests/test_reference_build.py, tools/reference_vs_fixtures.py); it is also
// pinned against the reference's own known-answer/property tests
// (tests/test_oracle_pins.py).
//
// Arithmetic conventions (the reference's Eigen kernels have an unspecified
// inner summation order, so the oracle fixes one and the CUDA kernels mirror it
// where bitwise comparison is claimed):
//   * a dense block times a vector: t[r] = fma-chain over c ascending from 0.0,
//     then y[r] += t[r]  (kernels.cpp:45 `yi += blk * x_j`);
//   * a transposed block times a vector: fma-chain over r ascending;
//   * block products c += a*b: tmp = fma-chain over the inner index ascending,
//     then c += tmp (kernels.cpp:71,82,108);
//   * vector updates are written exactly as the reference's expressions with
//     contraction disabled (-ffp-contract=off).
#include "bmg_oracle.h"

#include <immintrin.h>
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace orc {

// ----------------------------------------------------------------------------
// errors (small_cholesky.hpp:10-13 NotPositiveDefinite; std exceptions elsewhere)
struct NotPositiveDefinite : std::runtime_error {
  int pivot;
  NotPositiveDefinite(int p, const std::string& ctx)
      : std::runtime_error("matrix not positive definite at pivot " + std::to_string(p) +
                           (ctx.empty() ? "" : " (" + ctx + ")")),
        pivot(p) {}
};

static void require(bool ok, const char* msg) {
  if (!ok) throw std::invalid_argument(msg);
}

static inline double fma_(double a, double b, double c) { return __builtin_fma(a, b, c); }

// ----------------------------------------------------------------------------
// BlockLayout (block_layout.hpp:8-28, block_layout.cpp:8-16)
struct Layout {
  std::vector<int> sz, off;
  int dim = 0;
  Layout() = default;
  explicit Layout(std::vector<int> s) : sz(std::move(s)) {
    off.reserve(sz.size());
    dim = 0;
    for (int m : sz) {
      if (m < 1) throw std::invalid_argument("BlockLayout: block sizes must be >= 1");
      off.push_back(dim);
      dim += m;
    }
  }
  int blocks() const { return (int)sz.size(); }
  bool operator==(const Layout& o) const { return sz == o.sz; }
};

// ----------------------------------------------------------------------------
// BlockSparseMatrix (block_matrix.hpp:26-70).  Rows hold ascending column lists
// and the concatenated row-major blocks (the reference's std::map iteration
// order is ascending column, block_matrix.hpp:28).
struct Mat {
  Layout rl, cl;
  bool sym = false;
  std::vector<std::vector<int>> cols;
  std::vector<std::vector<size_t>> boff;  // offset of each block inside vals[i]
  std::vector<std::vector<double>> vals;
  // column index: for column j, (row i, block pointer) ascending i
  mutable std::vector<std::vector<std::pair<int, const double*>>> tidx;
  mutable bool tidx_ok = false;

  Mat() = default;
  Mat(Layout r, Layout c, bool s) : rl(std::move(r)), cl(std::move(c)), sym(s) {
    if (sym && !(rl == cl))
      throw std::invalid_argument("BlockSparseMatrix: symmetric matrix must be square");
    cols.resize(rl.blocks());
    boff.resize(rl.blocks());
    vals.resize(rl.blocks());
  }
  int nbr() const { return rl.blocks(); }
  int nbc() const { return cl.blocks(); }
  bool square() const { return rl == cl; }
  int find(int i, int j) const {
    const auto& c = cols[i];
    auto it = std::lower_bound(c.begin(), c.end(), j);
    return (it != c.end() && *it == j) ? (int)(it - c.begin()) : -1;
  }
  bool has(int i, int j) const { return find(i, j) >= 0; }
  const double* blk(int i, int p) const { return vals[i].data() + boff[i][p]; }
  double* blk(int i, int p) { return vals[i].data() + boff[i][p]; }
  const double* block(int i, int j) const {
    int p = find(i, j);
    if (p < 0) throw std::out_of_range("BlockSparseMatrix: block not stored");
    return blk(i, p);
  }
  // replace row i with an ascending map of blocks
  void set_row(int i, const std::map<int, std::vector<double>>& row) {
    cols[i].clear();
    boff[i].clear();
    vals[i].clear();
    for (const auto& [j, b] : row) {
      cols[i].push_back(j);
      boff[i].push_back(vals[i].size());
      vals[i].insert(vals[i].end(), b.begin(), b.end());
    }
    tidx_ok = false;
  }
  size_t nnzb() const {
    size_t n = 0;
    for (auto& c : cols) n += c.size();
    return n;
  }
  const std::vector<std::vector<std::pair<int, const double*>>>& colindex() const {
    if (!tidx_ok) {
      tidx.assign(nbc(), {});
      for (int i = 0; i < nbr(); ++i)
        for (size_t p = 0; p < cols[i].size(); ++p) tidx[cols[i][p]].push_back({i, blk(i, (int)p)});
      tidx_ok = true;
    }
    return tidx;
  }
};

using RowMap = std::map<int, std::vector<double>>;

// ----------------------------------------------------------------------------
// kernels.cpp
// spmv: kernels.cpp:39-47
static void spmv(const Mat& a, const double* x, double* y) {
  const int n = a.nbr();
#pragma omp parallel for schedule(dynamic, 64)
  for (int i = 0; i < n; ++i) {
    const int mi = a.rl.sz[i];
    double* yi = y + a.rl.off[i];
    for (int r = 0; r < mi; ++r) yi[r] = 0.0;
    for (size_t p = 0; p < a.cols[i].size(); ++p) {
      const int j = a.cols[i][p];
      const int mj = a.cl.sz[j];
      const double* xj = x + a.cl.off[j];
      const double* b = a.blk(i, (int)p);
      for (int r = 0; r < mi; ++r) {
        double t = 0.0;
        for (int c = 0; c < mj; ++c) t = fma_(b[r * mj + c], xj[c], t);
        yi[r] += t;
      }
    }
  }
}

// spmv_transpose: kernels.cpp:56-64 (scatter y_j += blk^T x_i, ascending i).
// Evaluated as a pull over the column index, which performs the same additions
// in the same (ascending i) order per output entry.
static void spmv_t(const Mat& a, const double* x, double* y) {
  const auto& ci = a.colindex();
  const int n = a.nbc();
#pragma omp parallel for schedule(dynamic, 64)
  for (int j = 0; j < n; ++j) {
    const int mj = a.cl.sz[j];
    double* yj = y + a.cl.off[j];
    for (int c = 0; c < mj; ++c) yj[c] = 0.0;
    for (const auto& [i, b] : ci[j]) {
      const int mi = a.rl.sz[i];
      const double* xi = x + a.rl.off[i];
      for (int c = 0; c < mj; ++c) {
        double t = 0.0;
        for (int r = 0; r < mi; ++r) t = fma_(b[r * mj + c], xi[r], t);
        yj[c] += t;
      }
    }
  }
}

// Block products.  Every output element keeps its own chain
//   t = fma(a_rk, b_kc, t) over k ascending from 0.0, then acc_rc += t
// (the convention above); the loops below only evaluate up to 16 such chains
// side by side (4-wide vectors over c), which changes no rounding.
// a_rk = a[r * ars + k * aks], b row k = b + k * C (contiguous over c).
static inline void gemm_rows(int R, int K, int C, const double* a, int ars, int aks, const double* b,
                             double* acc) {
  for (int r = 0; r < R; ++r) {
    const double* ar = a + (size_t)r * ars;
    double* accr = acc + (size_t)r * C;
    int c0 = 0;
    for (; c0 + 16 <= C; c0 += 16) {
      __m256d t0 = _mm256_setzero_pd(), t1 = t0, t2 = t0, t3 = t0;
      for (int k = 0; k < K; ++k) {
        const __m256d av = _mm256_set1_pd(ar[(size_t)k * aks]);
        const double* bk = b + (size_t)k * C + c0;
        t0 = _mm256_fmadd_pd(av, _mm256_loadu_pd(bk), t0);
        t1 = _mm256_fmadd_pd(av, _mm256_loadu_pd(bk + 4), t1);
        t2 = _mm256_fmadd_pd(av, _mm256_loadu_pd(bk + 8), t2);
        t3 = _mm256_fmadd_pd(av, _mm256_loadu_pd(bk + 12), t3);
      }
      _mm256_storeu_pd(accr + c0, _mm256_add_pd(_mm256_loadu_pd(accr + c0), t0));
      _mm256_storeu_pd(accr + c0 + 4, _mm256_add_pd(_mm256_loadu_pd(accr + c0 + 4), t1));
      _mm256_storeu_pd(accr + c0 + 8, _mm256_add_pd(_mm256_loadu_pd(accr + c0 + 8), t2));
      _mm256_storeu_pd(accr + c0 + 12, _mm256_add_pd(_mm256_loadu_pd(accr + c0 + 12), t3));
    }
    for (; c0 + 4 <= C; c0 += 4) {
      __m256d t0 = _mm256_setzero_pd();
      for (int k = 0; k < K; ++k)
        t0 = _mm256_fmadd_pd(_mm256_set1_pd(ar[(size_t)k * aks]), _mm256_loadu_pd(b + (size_t)k * C + c0), t0);
      _mm256_storeu_pd(accr + c0, _mm256_add_pd(_mm256_loadu_pd(accr + c0), t0));
    }
    for (; c0 < C; ++c0) {
      double t = 0.0;
      for (int k = 0; k < K; ++k) t = fma_(ar[(size_t)k * aks], b[(size_t)k * C + c0], t);
      accr[c0] += t;
    }
  }
}
// acc (r x c) += a (r x k) * b (k x c)
static void gemm_acc(int R, int K, int C, const double* a, const double* b, double* acc) {
  gemm_rows(R, K, C, a, K, 1, b, acc);
}
// acc (r x c) += a^T * b with a (k x r), b (k x c)
static void gemm_tn_acc(int R, int K, int C, const double* a, const double* b, double* acc) {
  gemm_rows(R, K, C, a, 1, R, b, acc);
}
// acc (r x c) += a * b^T with a (r x k), b (c x k): b is transposed into a
// (k x c) scratch first, the chains are the same
static void gemm_nt_acc(int R, int K, int C, const double* a, const double* b, double* acc) {
  double bt_small[64 * 64];
  std::vector<double> bt_big;
  double* bt = bt_small;
  if ((size_t)K * C > sizeof(bt_small) / sizeof(double)) {
    bt_big.resize((size_t)K * C);
    bt = bt_big.data();
  }
  for (int c = 0; c < C; ++c)
    for (int k = 0; k < K; ++k) bt[(size_t)k * C + c] = b[(size_t)c * K + k];
  gemm_rows(R, K, C, a, K, 1, bt, acc);
}

// multiply: kernels.cpp:66-75 (per output block, ascending k)
static Mat multiply(const Mat& a, const Mat& b) {
  require(a.cl == b.rl, "multiply: inner layouts do not match");
  Mat c(a.rl, b.cl, false);
#pragma omp parallel for schedule(dynamic, 16)
  for (int i = 0; i < a.nbr(); ++i) {
    RowMap row;
    const int mi = a.rl.sz[i];
    for (size_t p = 0; p < a.cols[i].size(); ++p) {
      const int k = a.cols[i][p];
      const int mk = a.cl.sz[k];
      for (size_t q = 0; q < b.cols[k].size(); ++q) {
        const int j = b.cols[k][q];
        const int mj = b.cl.sz[j];
        auto& acc = row[j];
        if (acc.empty()) acc.assign((size_t)mi * mj, 0.0);
        gemm_acc(mi, mk, mj, a.blk(i, (int)p), b.blk(k, (int)q), acc.data());
      }
    }
    c.set_row(i, row);
  }
  c.tidx_ok = false;
  return c;
}

// transpose_multiply: kernels.cpp:77-86 (C = P^T B; per output block, ascending i)
static Mat transpose_multiply(const Mat& p, const Mat& b) {
  require(p.rl == b.rl, "transpose_multiply: row layouts do not match");
  Mat c(p.cl, b.cl, false);
  const auto& pc = p.colindex();
#pragma omp parallel for schedule(dynamic, 16)
  for (int k = 0; k < p.nbc(); ++k) {
    RowMap row;
    const int mk = p.cl.sz[k];
    for (const auto& [i, pik] : pc[k]) {
      const int mi = p.rl.sz[i];
      for (size_t q = 0; q < b.cols[i].size(); ++q) {
        const int j = b.cols[i][q];
        const int mj = b.cl.sz[j];
        auto& acc = row[j];
        if (acc.empty()) acc.assign((size_t)mk * mj, 0.0);
        gemm_tn_acc(mk, mi, mj, pik, b.blk(i, (int)q), acc.data());
      }
    }
    c.set_row(k, row);
  }
  c.tidx_ok = false;
  return c;
}

static void transpose_block(int r, int c, const double* a, double* out) {
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) out[j * r + i] = a[i * c + j];
}

// insert_symmetric (block_matrix.cpp:51-54) into row maps
static void insert_sym(std::vector<RowMap>& rows, const Layout& l, int i, int j,
                       const std::vector<double>& b) {
  rows[i][j] = b;
  if (i != j) {
    std::vector<double> t(b.size());
    transpose_block(l.sz[i], l.sz[j], b.data(), t.data());
    rows[j][i] = std::move(t);
  }
}

static Mat from_rowmaps(const Layout& rl, const Layout& cl, bool sym,
                        const std::vector<RowMap>& rows) {
  Mat m(rl, cl, sym);
  for (int i = 0; i < m.nbr(); ++i) m.set_row(i, rows[i]);
  return m;
}

// triple_product: kernels.cpp:88-119 (F A F^T, exact-zero blocks dropped).  The
// reference visits every j <= i; pairs with no common column contribute nothing
// (any == false), so only rows sharing a column are visited here.
static Mat triple_product(const Mat& f, const Mat& a) {
  require(f.square() && a.square() && f.rl == a.rl,
          "triple_product: layouts must be square and compatible");
  require(a.sym, "triple_product: A must be symmetric");
  const Mat h = multiply(f, a);
  const auto& fc = f.colindex();
  const int n = f.nbr();
  std::vector<std::vector<std::pair<int, std::vector<double>>>> lower(n);
#pragma omp parallel for schedule(dynamic, 16)
  for (int i = 0; i < n; ++i) {
    std::vector<int> cand;
    for (int k : h.cols[i])
      for (const auto& [j, ptr] : fc[k])
        if (j <= i) cand.push_back(j);
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    const int mi = f.rl.sz[i];
    for (int j : cand) {
      const int mj = f.rl.sz[j];
      std::vector<double> blk((size_t)mi * mj, 0.0);
      bool any = false;
      size_t hp = 0, fp = 0;
      const auto& hr = h.cols[i];
      const auto& fr = f.cols[j];
      while (hp < hr.size() && fp < fr.size()) {
        if (hr[hp] < fr[fp]) {
          ++hp;
        } else if (fr[fp] < hr[hp]) {
          ++fp;
        } else {
          const int mk = f.rl.sz[hr[hp]];
          gemm_nt_acc(mi, mk, mj, h.blk(i, (int)hp), f.blk(j, (int)fp), blk.data());
          any = true;
          ++hp;
          ++fp;
        }
      }
      if (i == j) {
        std::vector<double> s(blk.size());
        for (int r = 0; r < mi; ++r)
          for (int c = 0; c < mi; ++c) s[r * mi + c] = 0.5 * (blk[r * mi + c] + blk[c * mi + r]);
        blk = std::move(s);
      }
      double sq = 0.0;
      for (double v : blk) sq += v * v;
      if (any && sq != 0.0) lower[i].push_back({j, std::move(blk)});
    }
  }
  std::vector<RowMap> rows(n);
  for (int i = 0; i < n; ++i)
    for (auto& [j, b] : lower[i]) insert_sym(rows, f.rl, i, j, b);
  return from_rowmaps(f.rl, f.rl, true, rows);
}

// extract: kernels.cpp:15-37 (dense, row-major)
static std::vector<double> extract(const Mat& a, const std::vector<int>& I,
                                   const std::vector<int>& J, int* R, int* C) {
  int rows = 0, cols = 0;
  for (int i : I) rows += a.rl.sz[i];
  for (int j : J) cols += a.cl.sz[j];
  std::vector<double> out((size_t)rows * cols, 0.0);
  int r = 0;
  for (int i : I) {
    int c = 0;
    const int mi = a.rl.sz[i];
    for (int j : J) {
      const int mj = a.cl.sz[j];
      int p = a.find(i, j);
      if (p >= 0) {
        const double* b = a.blk(i, p);
        for (int x = 0; x < mi; ++x)
          for (int y = 0; y < mj; ++y) out[(size_t)(r + x) * cols + c + y] = b[x * mj + y];
      }
      c += mj;
    }
    r += mi;
  }
  *R = rows;
  *C = cols;
  return out;
}

// ----------------------------------------------------------------------------
// SmallCholesky: small_cholesky.cpp:12-47
struct Chol {
  int n = 0;
  std::vector<double> l;  // row-major lower
  double logdet = 0.0;
  Chol() = default;
  Chol(const double* b, int n_, const std::string& ctx) : n(n_), l((size_t)n_ * n_, 0.0) {
    logdet = 0.0;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < j; ++k) s = fma_(l[(size_t)j * n + k], l[(size_t)j * n + k], s);
      const double d = b[(size_t)j * n + j] - s;
      if (!(d > 0.0)) throw NotPositiveDefinite(j, ctx);
      const double ljj = std::sqrt(d);
      l[(size_t)j * n + j] = ljj;
      logdet += 2.0 * std::log(ljj);
      for (int i = j + 1; i < n; ++i) {
        double t = 0.0;
        for (int k = 0; k < j; ++k) t = fma_(l[(size_t)i * n + k], l[(size_t)j * n + k], t);
        l[(size_t)i * n + j] = (b[(size_t)i * n + j] - t) / ljj;
      }
    }
  }
  void solve_l(double* x) const {  // in place, L x = rhs
    for (int i = 0; i < n; ++i) {
      double t = 0.0;
      for (int k = 0; k < i; ++k) t = fma_(l[(size_t)i * n + k], x[k], t);
      x[i] = (x[i] - t) / l[(size_t)i * n + i];
    }
  }
  void solve_lt(double* x) const {  // in place, L^T x = rhs
    for (int i = n - 1; i >= 0; --i) {
      double t = 0.0;
      for (int k = i + 1; k < n; ++k) t = fma_(l[(size_t)k * n + i], x[k], t);
      x[i] = (x[i] - t) / l[(size_t)i * n + i];
    }
  }
  void solve(double* x) const {
    solve_l(x);
    solve_lt(x);
  }
  // B X = RHS for a row-major n x c right-hand side, column by column
  void solve_mat(double* x, int c) const {
    std::vector<double> col(n);
    for (int j = 0; j < c; ++j) {
      for (int i = 0; i < n; ++i) col[i] = x[(size_t)i * c + j];
      solve(col.data());
      for (int i = 0; i < n; ++i) x[(size_t)i * c + j] = col[i];
    }
  }
};

// ----------------------------------------------------------------------------
// LowerPattern (pattern.hpp:12-38, pattern.cpp:10-47)
struct LowerPattern {
  std::vector<std::vector<int>> rows;  // sorted, diagonal last
  static LowerPattern diagonal(int n) {
    LowerPattern p;
    p.rows.resize(n);
    for (int i = 0; i < n; ++i) p.rows[i] = {i};
    return p;
  }
  static LowerPattern full(int n) {
    LowerPattern p = diagonal(n);
    for (int i = 0; i < n; ++i) {
      p.rows[i].clear();
      for (int j = 0; j <= i; ++j) p.rows[i].push_back(j);
    }
    return p;
  }
  static LowerPattern from_matrix(const Mat& a) {
    if (!a.square()) throw std::invalid_argument("LowerPattern::from_matrix: matrix must be square");
    LowerPattern p = diagonal(a.nbr());
    for (int i = 0; i < a.nbr(); ++i) {
      std::vector<int> r;
      for (int j : a.cols[i])
        if (j < i) r.push_back(j);
      r.push_back(i);
      p.rows[i] = r;
    }
    return p;
  }
  std::vector<int> strict(int i) const { return {rows[i].begin(), rows[i].end() - 1}; }
  bool contains(int i, int j) const { return std::binary_search(rows[i].begin(), rows[i].end(), j); }
  void add(int i, int j) {
    if (j >= i) throw std::invalid_argument("LowerPattern::add: entry must be strictly lower");
    auto& r = rows[i];
    auto it = std::lower_bound(r.begin(), r.end(), j);
    if (it != r.end() && *it == j) return;
    r.insert(it, j);
  }
};

// ----------------------------------------------------------------------------
// FSAI (fsai.hpp, fsai.cpp)
struct Factors {
  Layout layout;
  LowerPattern pattern;
  Mat F;
  std::vector<Chol> S;
};

struct Nested {
  Layout layout;
  std::vector<Factors> chain;
  const std::vector<Chol>& final_diag() const { return chain.back().S; }
};

static void check_spd_inputs(const Mat& a) {
  require(a.square(), "fsai: matrix must be square");
  require(a.sym, "fsai: matrix must be symmetric");
}

// build_row: fsai.cpp:18-43
static void build_row(const Mat& a, const LowerPattern& p, int k, RowMap& frow_out, Chol& s_out,
                      Chol& gram_out) {
  const int mk = a.rl.sz[k];
  const std::vector<int> rk{k};
  const std::vector<int> strict = p.strict(k);
  RowMap frow;
  std::vector<double> eye((size_t)mk * mk, 0.0);
  for (int i = 0; i < mk; ++i) eye[(size_t)i * mk + i] = 1.0;
  frow[k] = eye;
  int R, C;
  std::vector<double> s_kk = extract(a, rk, rk, &R, &C);
  if (!strict.empty()) {
    int gR, gC;
    std::vector<double> g = extract(a, strict, strict, &gR, &gC);
    gram_out = Chol(g.data(), gR, "row " + std::to_string(k) + " principal submatrix");
    int aR, aC;
    std::vector<double> a_ks = extract(a, rk, strict, &aR, &aC);  // mk x ns
    std::vector<double> x((size_t)aC * aR);                        // ns x mk = a_ks^T
    transpose_block(aR, aC, a_ks.data(), x.data());
    gram_out.solve_mat(x.data(), aR);
    // f_row = -x^T (mk x ns), split into blocks
    int col = 0;
    for (int j : strict) {
      const int mj = a.rl.sz[j];
      std::vector<double> b((size_t)mk * mj);
      for (int r = 0; r < mk; ++r)
        for (int c = 0; c < mj; ++c) b[(size_t)r * mj + c] = -x[(size_t)(col + c) * aR + r];
      frow[j] = std::move(b);
      col += mj;
    }
    // s_kk -= a_ks * x
    for (int r = 0; r < mk; ++r)
      for (int c = 0; c < mk; ++c) {
        double t = 0.0;
        for (int q = 0; q < aC; ++q) t = fma_(a_ks[(size_t)r * aC + q], x[(size_t)q * aR + c], t);
        s_kk[(size_t)r * mk + c] -= t;
      }
  } else {
    gram_out = Chol();
  }
  s_out = Chol(s_kk.data(), mk, "S row " + std::to_string(k));
  frow_out = std::move(frow);
}

// build_h_row: fsai.cpp:46-51 (H row k = F row k * A)
static RowMap build_h_row(const Mat& a, const RowMap& frow, int k) {
  RowMap h;
  const int mk = a.rl.sz[k];
  for (const auto& [j, fkj] : frow) {
    const int mj = a.rl.sz[j];
    for (size_t q = 0; q < a.cols[j].size(); ++q) {
      const int c = a.cols[j][q];
      const int mc = a.cl.sz[c];
      auto& acc = h[c];
      if (acc.empty()) acc.assign((size_t)mk * mc, 0.0);
      gemm_acc(mk, mj, mc, fkj.data(), a.blk(j, (int)q), acc.data());
    }
  }
  return h;
}

// build_fsai: fsai.cpp:72-83
static Factors build_fsai(const Mat& a, const LowerPattern& p) {
  check_spd_inputs(a);
  require((int)p.rows.size() == a.nbr(), "build_fsai: pattern size does not match matrix");
  Factors fac;
  fac.layout = a.rl;
  fac.pattern = p;
  const int n = a.nbr();
  fac.S.resize(n);
  std::vector<Chol> gram(n);
  std::vector<RowMap> frows(n);
  std::string err;
  int err_pivot = -1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int k = 0; k < n; ++k) {
    try {
      build_row(a, p, k, frows[k], fac.S[k], gram[k]);
    } catch (const NotPositiveDefinite& e) {
#pragma omp critical
      if (err.empty()) { err = e.what(); err_pivot = e.pivot; }
    }
  }
  if (!err.empty()) throw NotPositiveDefinite(err_pivot, err);
  fac.F = from_rowmaps(fac.layout, fac.layout, false, frows);
  return fac;
}

static double frob(const std::vector<double>& b) {
  double s = 0.0;
  for (double v : b) s += v * v;
  return std::sqrt(s);
}

// delta_ratio: fsai.cpp:106-130.  h_kc is H[k, c]; gram_k / s_k the row's state.
static double delta_ratio(const Mat& a, const LowerPattern& pat, const Chol& gram_k,
                          const Chol& s_k, int k, int c, const std::vector<double>& h_kc) {
  require(c >= 0 && c < k, "delta_ratio: candidate must precede the row");
  require(!pat.contains(k, c), "delta_ratio: candidate already in pattern");
  const std::vector<int> cc{c};
  const std::vector<int> strict = pat.strict(k);
  int R, C;
  std::vector<double> w = extract(a, cc, cc, &R, &C);
  const int mc = R;
  if (!strict.empty()) {
    int aR, aC;
    std::vector<double> a_cs = extract(a, cc, strict, &aR, &aC);  // mc x ns
    std::vector<double> y((size_t)aC * aR);                        // ns x mc
    transpose_block(aR, aC, a_cs.data(), y.data());
    gram_k.solve_mat(y.data(), aR);
    for (int r = 0; r < mc; ++r)
      for (int q = 0; q < mc; ++q) {
        double t = 0.0;
        for (int z = 0; z < aC; ++z) t = fma_(a_cs[(size_t)r * aC + z], y[(size_t)z * aR + q], t);
        w[(size_t)r * mc + q] -= t;
      }
  }
  const Chol w_chol(w.data(), mc,
                    "W_c for row " + std::to_string(k) + ", candidate " + std::to_string(c));
  const int mk = a.rl.sz[k];
  // u = w - h_kc^T * S_k^{-1} h_kc
  std::vector<double> sol = h_kc;  // mk x mc
  s_k.solve_mat(sol.data(), mc);
  std::vector<double> u = w;
  for (int r = 0; r < mc; ++r)
    for (int q = 0; q < mc; ++q) {
      double t = 0.0;
      for (int z = 0; z < mk; ++z) t = fma_(h_kc[(size_t)z * mc + r], sol[(size_t)z * mc + q], t);
      u[(size_t)r * mc + q] -= t;
    }
  double log_ratio;
  try {
    log_ratio = Chol(u.data(), mc, "").logdet - w_chol.logdet;
  } catch (const NotPositiveDefinite&) {
    return 0.0;
  }
  return std::min(std::exp(log_ratio), 1.0);
}

// adaptive_build: fsai.cpp:132-198 (rows are independent; parallel over rows)
static Factors adaptive_build(const Mat& a, int t_max, double tau, const LowerPattern& p0) {
  check_spd_inputs(a);
  require(t_max >= 1, "adaptive_build: t_max must be >= 1");
  require(tau > 0.0 && tau <= 1.0, "adaptive_build: tau must be in (0, 1]");
  require((int)p0.rows.size() == a.nbr(), "adaptive_build: pattern size does not match matrix");
  const int n = a.nbr();
  const double eps_drop = 1e-12;  // fsai.hpp:38
  Factors fac;
  fac.layout = a.rl;
  fac.S.resize(n);
  LowerPattern pat = p0;
  std::vector<RowMap> frows(n);
  std::string err;
  int err_pivot = -1;
#pragma omp parallel for schedule(dynamic, 8)
  for (int k = 0; k < n; ++k) {
    try {
      // per-row state (the reference keeps these in vectors indexed by k)
      Chol s_diag, gram;
      RowMap h;
      bool stale = true, active = true;
      for (int t = 1; t <= t_max; ++t) {
        if (stale) {
          build_row(a, pat, k, frows[k], s_diag, gram);
          h = build_h_row(a, frows[k], k);
          stale = false;
        }
        if (!active) continue;
        const double threshold = eps_drop * frob(h.at(k));
        int best = -1;
        double best_rho = 0.0;
        for (const auto& [c, h_kc] : h) {
          if (c >= k) break;
          if (pat.contains(k, c)) continue;
          if (frob(h_kc) <= threshold) continue;
          const double rho = delta_ratio(a, pat, gram, s_diag, k, c, h_kc);
          if (best < 0 || rho < best_rho) {
            best = c;
            best_rho = rho;
          }
        }
        if (best < 0) {
          active = false;
        } else if (best_rho < tau) {
          pat.add(k, best);
          stale = true;
        } else {
          active = false;
        }
      }
      if (stale) {
        build_row(a, pat, k, frows[k], fac.S[k], gram);
      } else {
        fac.S[k] = std::move(s_diag);
      }
    } catch (const NotPositiveDefinite& e) {
#pragma omp critical
      if (err.empty()) { err = e.what(); err_pivot = e.pivot; }
    }
  }
  if (!err.empty()) throw NotPositiveDefinite(err_pivot, err);
  fac.F = from_rowmaps(fac.layout, fac.layout, false, frows);
  fac.pattern = std::move(pat);
  return fac;
}

// NestedFsai::apply: fsai.cpp:200-217
static void nested_apply(const Nested& f, const double* r, double* out) {
  const int N = f.layout.dim;
  std::vector<double> v(r, r + N), tmp(N);
  for (const Factors& fac : f.chain) {
    spmv(fac.F, v.data(), tmp.data());
    v.swap(tmp);
  }
  const auto& s = f.final_diag();
  const int n = f.layout.blocks();
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) s[i].solve(v.data() + f.layout.off[i]);
  for (auto it = f.chain.rbegin(); it != f.chain.rend(); ++it) {
    spmv_t(it->F, v.data(), tmp.data());
    v.swap(tmp);
  }
  std::copy(v.begin(), v.end(), out);
}

// NestedFsai::apply_transformed: fsai.cpp:219-241
static void nested_apply_transformed(const Nested& f, const Mat& a, const double* x, double* out) {
  const int N = f.layout.dim;
  const auto& s = f.final_diag();
  const int n = f.layout.blocks();
  std::vector<double> v(x, x + N), tmp(N);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) s[i].solve_lt(v.data() + f.layout.off[i]);
  for (auto it = f.chain.rbegin(); it != f.chain.rend(); ++it) {
    spmv_t(it->F, v.data(), tmp.data());
    v.swap(tmp);
  }
  spmv(a, v.data(), tmp.data());
  v.swap(tmp);
  for (const Factors& fac : f.chain) {
    spmv(fac.F, v.data(), tmp.data());
    v.swap(tmp);
  }
#pragma omp parallel for schedule(static)
  for (int i = 0; i < n; ++i) s[i].solve_l(v.data() + f.layout.off[i]);
  std::copy(v.begin(), v.end(), out);
}

// nested_build: fsai.cpp:243-253
static Nested nested_build(const Mat& a, int t_max, double tau, int n_levels) {
  require(n_levels >= 0, "nested_build: n_levels must be >= 0");
  Nested out;
  out.layout = a.rl;
  Mat a_k = a;
  for (int level = 0; level <= n_levels; ++level) {
    out.chain.push_back(adaptive_build(a_k, t_max, tau, LowerPattern::diagonal(a.nbr())));
    if (level < n_levels) a_k = triple_product(out.chain.back().F, a_k);
  }
  return out;
}

// ----------------------------------------------------------------------------
// vector helpers (sequential fma dots; Eigen's dot order is unspecified)
static double dot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = fma_(a[i], b[i], s);
  return s;
}
static double norm2(const double* a, int n) { return std::sqrt(dot(a, a, n)); }

// ----------------------------------------------------------------------------
// RNG: rng.hpp:12-57
static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline double rng_uniform(uint64_t seed, uint64_t i) {
  const uint64_t bits = mix64(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
  return (static_cast<double>(bits >> 11) + 0.5) * 0x1.0p-53;
}
static inline double rng_symmetric(uint64_t seed, uint64_t i) {
  return 2.0 * rng_uniform(seed, i) - 1.0;
}

// ----------------------------------------------------------------------------
// symmetric tridiagonal eigenvalues by Sturm-sequence bisection (replaces
// Eigen::SelfAdjointEigenSolver::computeFromTridiagonal, lanczos.hpp:44-45)
static int sturm_count(const std::vector<double>& d, const std::vector<double>& e, double x) {
  int cnt = 0;
  double q = d[0] - x;
  if (q < 0) ++cnt;
  for (size_t i = 1; i < d.size(); ++i) {
    if (q == 0.0) q = 1e-300;
    q = d[i] - x - e[i - 1] * e[i - 1] / q;
    if (q < 0) ++cnt;
  }
  return cnt;
}
static std::vector<double> tridiag_eigs(const std::vector<double>& d, const std::vector<double>& e) {
  const int n = (int)d.size();
  std::vector<double> out(n);
  if (n == 0) return out;
  double lo = d[0], hi = d[0];
  for (int i = 0; i < n; ++i) {
    double rad = 0.0;
    if (i > 0) rad += std::fabs(e[i - 1]);
    if (i + 1 < n) rad += std::fabs(e[i]);
    lo = std::min(lo, d[i] - rad);
    hi = std::max(hi, d[i] + rad);
  }
  const double span = std::max(hi - lo, std::fabs(hi) + std::fabs(lo)) + 1e-300;
  lo -= 1e-12 * span;
  hi += 1e-12 * span;
  for (int k = 0; k < n; ++k) {  // k-th smallest: count(x) > k
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double mid = 0.5 * (a + b);
      if (mid <= a || mid >= b) break;
      if (sturm_count(d, e, mid) > k)
        b = mid;
      else
        a = mid;
    }
    out[k] = 0.5 * (a + b);
  }
  return out;
}

// lanczos_ritz_values: lanczos.hpp:16-47
template <class Op>
static std::vector<double> lanczos_ritz(const Op& op, int n, int iters, uint64_t seed) {
  if (n < 1) throw std::invalid_argument("lanczos: operator dimension must be >= 1");
  iters = std::min(iters, n);
  std::vector<double> v(n), v_prev(n, 0.0), w(n);
  for (int i = 0; i < n; ++i) v[i] = rng_symmetric(seed, (uint64_t)i);
  const double nv = norm2(v.data(), n);
  for (auto& z : v) z /= nv;
  std::vector<double> diag, off;
  double beta = 0.0;
  for (int j = 0; j < iters; ++j) {
    op(v.data(), w.data());
    const double alpha = dot(v.data(), w.data(), n);
    diag.push_back(alpha);
    for (int i = 0; i < n; ++i) w[i] -= alpha * v[i];
    for (int i = 0; i < n; ++i) w[i] -= beta * v_prev[i];
    beta = norm2(w.data(), n);
    if (j + 1 == iters) break;
    if (beta <= 1e-14 * std::fabs(alpha) || beta == 0.0) break;
    off.push_back(beta);
    v_prev = v;
    for (int i = 0; i < n; ++i) v[i] = w[i] / beta;
  }
  off.resize(diag.empty() ? 0 : diag.size() - 1);
  return tridiag_eigs(diag, off);
}

// ----------------------------------------------------------------------------
// Chebyshev / smoothers: chebyshev.hpp:42-129
static double fourth_kind_mu(int n) { return (2.0 * n + 1.0) / (2.0 * n + 3.0); }

template <class OpA, class OpM>
static void cheb_fourth(const OpA& a, const OpM& m, const double* b, double* x, int n, double beta,
                        int k) {
  if (!(beta > 0.0)) throw std::invalid_argument("cheb_fourth_apply: beta must be positive");
  if (k < 1) throw std::invalid_argument("cheb_fourth_apply: degree must be >= 1");
  const double d = 4.0 / beta;
  std::vector<double> r(n), p(n), t(n);
  a(x, t.data());
  for (int i = 0; i < n; ++i) r[i] = b[i] - t[i];
  m(r.data(), p.data());
  double mu = fourth_kind_mu(0);
  double dmu = d * mu;
  for (int i = 0; i < n; ++i) x[i] += dmu * p[i];
  for (int s = 2; s <= k; ++s) {
    a(x, t.data());
    for (int i = 0; i < n; ++i) r[i] = b[i] - t[i];
    m(r.data(), t.data());
    const double mu2 = mu * mu;
    for (int i = 0; i < n; ++i) p[i] = mu2 * p[i] + t[i];
    mu = fourth_kind_mu(s - 1);
    dmu = d * mu;
    for (int i = 0; i < n; ++i) x[i] += dmu * p[i];
  }
}

template <class OpA, class OpM>
static void cheb_first(const OpA& a, const OpM& m, const double* b, double* x, int n, double alpha,
                       double beta, int k) {
  if (!(alpha > 0.0) || !(alpha < beta))
    throw std::invalid_argument("cheb_first_apply: interval must satisfy 0 < alpha < beta");
  if (k < 1) throw std::invalid_argument("cheb_first_apply: degree must be >= 1");
  const double c = 0.5 * (alpha + beta);
  const double d = 0.5 * (beta - alpha);
  std::vector<double> r(n), p(n), t(n);
  a(x, t.data());
  for (int i = 0; i < n; ++i) r[i] = b[i] - t[i];
  m(r.data(), p.data());
  double omega = 1.0 / c;
  double psi = 0.5 * (d * omega) * (d * omega);
  for (int i = 0; i < n; ++i) x[i] += omega * p[i];
  for (int s = 2; s <= k; ++s) {
    a(x, t.data());
    for (int i = 0; i < n; ++i) r[i] = b[i] - t[i];
    m(r.data(), t.data());
    for (int i = 0; i < n; ++i) p[i] = t[i] + psi * p[i];
    omega = 1.0 / (c - psi / omega);
    psi = 0.25 * (d * omega) * (d * omega);
    for (int i = 0; i < n; ++i) x[i] += omega * p[i];
  }
}

template <class OpA, class OpM>
static void richardson(const OpA& a, const OpM& m, const double* b, double* x, int n, double omega,
                       int k) {
  if (k < 1) throw std::invalid_argument("richardson_apply: step count must be >= 1");
  std::vector<double> r(n), t(n);
  for (int s = 0; s < k; ++s) {
    a(x, t.data());
    for (int i = 0; i < n; ++i) r[i] = b[i] - t[i];
    m(r.data(), t.data());
    for (int i = 0; i < n; ++i) x[i] += omega * t[i];
  }
}

template <class OpA, class OpM>
static void apply_smoother(int kind, double alpha, double beta, double omega, int degree,
                           const OpA& a, const OpM& m, const double* b, double* x, int n) {
  switch (kind) {
    case 0: return richardson(a, m, b, x, n, omega, degree);
    case 1: return cheb_first(a, m, b, x, n, alpha, beta, degree);
    case 2: return cheb_fourth(a, m, b, x, n, beta, degree);
  }
  throw std::logic_error("apply_smoother: unknown kind");
}

// poly_eval: chebyshev.cpp:8-44
static double cheb_recurrence(int n, double t, double p1) {
  if (n == 0) return 1.0;
  double prev = 1.0, cur = p1;
  for (int i = 1; i < n; ++i) {
    const double next = 2.0 * t * cur - prev;
    prev = cur;
    cur = next;
  }
  return cur;
}
static double poly_eval(int kind, int degree, double alpha, double beta, double t) {
  if (degree < 0) throw std::invalid_argument("poly_eval: degree must be >= 0");
  switch (kind) {
    case 0: return cheb_recurrence(degree, t, t);
    case 1: return cheb_recurrence(degree, t, 2.0 * t + 1.0);
    case 2: {
      if (!(alpha > 0.0) || !(alpha < beta))
        throw std::invalid_argument("poly_eval: scaled first kind needs 0 < alpha < beta");
      const double u = (2.0 * t - alpha - beta) / (beta - alpha);
      const double u0 = (alpha + beta) / (alpha - beta);
      return cheb_recurrence(degree, u, u) / cheb_recurrence(degree, u0, u0);
    }
    case 3: {
      if (!(beta > 0.0)) throw std::invalid_argument("poly_eval: scaled fourth kind needs beta > 0");
      const double u = 1.0 - 2.0 * t / beta;
      return cheb_recurrence(degree, u, 2.0 * u + 1.0) / (2.0 * degree + 1.0);
    }
  }
  throw std::logic_error("poly_eval: unknown kind");
}

// ----------------------------------------------------------------------------
// multilevel.cpp
// C = P^T (A P) exactly as transpose_multiply(p, multiply(a, p)), without holding
// the whole A P (C4's 3-D fine level: ~105 GB).  A P is formed for a range of
// fine rows at a time; every coarse block C_kj is created at its first term and
// accumulates its terms P_ik^T (AP)_ij in ascending i across the ranges, the same
// sequence of `acc += tmp` as the one-shot product.
static Mat galerkin_product(const Mat& a, const Mat& p) {
  require(a.cl == p.rl && a.rl == p.rl, "galerkin_coarsen: layouts do not match");
  const int nf = a.nbr(), nc = p.nbc();
  const auto& pc = p.colindex();
  std::vector<RowMap> crow(nc);
  std::vector<size_t> cursor(nc, 0);
  const size_t chunk_bytes = size_t(2) << 30;
  int i0 = 0;
  while (i0 < nf) {
    // fine rows [i0, i1): estimate A P bytes from the row's A-by-P block counts
    int i1 = i0;
    size_t bytes = 0;
    // (block products per row / 8 approximates the distinct blocks of an A P row;
    // at least 4096 rows per range keep every thread busy)
    while (i1 < nf && (i1 - i0 < 4096 || bytes < chunk_bytes)) {
      size_t blocks = 0;
      for (int k : a.cols[i1]) blocks += p.cols[k].size();
      bytes += blocks / 8 * (size_t)a.rl.sz[i1] * 8 * 24;
      ++i1;
    }
    std::vector<std::vector<int>> apc(i1 - i0);
    std::vector<std::vector<size_t>> apo(i1 - i0);
    std::vector<std::vector<double>> apv(i1 - i0);
#pragma omp parallel for schedule(dynamic, 16)
    for (int i = i0; i < i1; ++i) {  // multiply(a, p) row i (kernels.cpp:66-75)
      RowMap row;
      const int mi = a.rl.sz[i];
      for (size_t q = 0; q < a.cols[i].size(); ++q) {
        const int k = a.cols[i][q];
        const int mk = a.cl.sz[k];
        for (size_t s = 0; s < p.cols[k].size(); ++s) {
          const int j = p.cols[k][s];
          auto& acc = row[j];
          if (acc.empty()) acc.assign((size_t)mi * p.cl.sz[j], 0.0);
          gemm_acc(mi, mk, p.cl.sz[j], a.blk(i, (int)q), p.blk(k, (int)s), acc.data());
        }
      }
      auto& cc = apc[i - i0];
      auto& oo = apo[i - i0];
      auto& vv = apv[i - i0];
      for (auto& [j, b] : row) {
        cc.push_back(j);
        oo.push_back(vv.size());
        vv.insert(vv.end(), b.begin(), b.end());
      }
    }
#pragma omp parallel for schedule(dynamic, 16)
    for (int k = 0; k < nc; ++k) {  // transpose_multiply(p, ap) row k (kernels.cpp:77-86)
      const int mk = p.cl.sz[k];
      auto& row = crow[k];
      size_t t = cursor[k];
      for (; t < pc[k].size() && pc[k][t].first < i1; ++t) {
        const int i = pc[k][t].first;
        const double* pik = pc[k][t].second;
        const int mi = p.rl.sz[i];
        const auto& cc = apc[i - i0];
        for (size_t q = 0; q < cc.size(); ++q) {
          const int j = cc[q];
          const int mj = p.cl.sz[j];
          auto& acc = row[j];
          if (acc.empty()) acc.assign((size_t)mk * mj, 0.0);
          gemm_tn_acc(mk, mi, mj, pik, apv[i - i0].data() + apo[i - i0][q], acc.data());
        }
      }
      cursor[k] = t;
    }
    i0 = i1;
  }
  Mat c(p.cl, p.cl, false);
  for (int k = 0; k < nc; ++k) {
    c.set_row(k, crow[k]);
    RowMap().swap(crow[k]);
  }
  c.tidx_ok = false;
  return c;
}

// galerkin_coarsen: multilevel.cpp:11-28
static Mat galerkin(const Mat& a, const Mat& p) {
  if (!(a.square() && a.rl == p.rl))
    throw std::invalid_argument("galerkin_coarsen: layouts do not match");
  const Mat c = galerkin_product(a, p);
  const int n = c.nbr();
  // The reference visits every stored (i, j), j <= i, and inserts
  // S = (C_ij + C_ji^T) / 2 (or C_ij / 2 without a mirror block) at (i, j) and S^T
  // at (j, i) (insert_symmetric).  No two visits write the same block, so row i of
  // the result is assembled independently: its lower blocks from C's row i, its
  // upper blocks (i, j > i) as the transposes of the S made for C's (j, i).
  const auto& ccol = c.colindex();
  Mat out(c.rl, c.cl, true);
  auto sym_block = [&](int i, int q, std::vector<double>& s) {  // S for stored (i, cols[i][q])
    const int j = c.cols[i][q];
    const int mi = c.rl.sz[i], mj = c.cl.sz[j];
    const double* blk = c.blk(i, q);
    s.assign(blk, blk + (size_t)mi * mj);
    const int pj = c.find(j, i);
    if (pj >= 0) {
      const double* bt = c.blk(j, pj);  // mj x mi
      for (int r = 0; r < mi; ++r)
        for (int t = 0; t < mj; ++t) s[(size_t)r * mj + t] = 0.5 * (blk[r * mj + t] + bt[t * mi + r]);
    } else {
      for (auto& v : s) v *= 0.5;
    }
  };
#pragma omp parallel for schedule(dynamic, 16)
  for (int i = 0; i < n; ++i) {
    RowMap row;
    std::vector<double> s;
    for (size_t q = 0; q < c.cols[i].size(); ++q) {
      if (c.cols[i][q] > i) continue;
      sym_block(i, (int)q, s);
      row[c.cols[i][q]] = s;
    }
    for (const auto& [j, ptr] : ccol[i]) {  // stored (j, i) with j > i
      if (j <= i) continue;
      const int q = c.find(j, i);
      sym_block(j, q, s);
      std::vector<double> t(s.size());
      transpose_block(c.rl.sz[j], c.cl.sz[i], s.data(), t.data());
      row[j] = std::move(t);
    }
    out.cols[i].clear();
    out.boff[i].clear();
    out.vals[i].clear();
    for (const auto& [j, b] : row) {
      out.cols[i].push_back(j);
      out.boff[i].push_back(out.vals[i].size());
      out.vals[i].insert(out.vals[i].end(), b.begin(), b.end());
    }
  }
  out.tidx_ok = false;
  return out;
}

struct Level {
  Mat A, P;
  Nested fsai;
  double beta = 1.0;  // SmootherSpec (chebyshev.hpp:12-18)
  int kind = 2;
  double alpha = 0.0, omega = 1.0;
};

struct Hier {
  std::vector<Level> levels;  // 0 = coarsest
  Chol coarse;                // dense LLT of A_0 (multilevel.cpp:71-73)
  int finest() const { return (int)levels.size() - 1; }
};

static std::vector<double> to_dense(const Mat& a) {
  const int R = a.rl.dim, C = a.cl.dim;
  std::vector<double> out((size_t)R * C, 0.0);
  for (int i = 0; i < a.nbr(); ++i)
    for (size_t q = 0; q < a.cols[i].size(); ++q) {
      const int j = a.cols[i][q];
      const int mi = a.rl.sz[i], mj = a.cl.sz[j];
      const double* b = a.blk(i, (int)q);
      for (int r = 0; r < mi; ++r)
        for (int c = 0; c < mj; ++c) out[(size_t)(a.rl.off[i] + r) * C + a.cl.off[j] + c] = b[r * mj + c];
    }
  return out;
}

// dense Cholesky of the coarsest operator (same algorithm as SmallCholesky;
// the per-column row loop is independent, so it runs in parallel)
static bool dense_cholesky(const std::vector<double>& b, int n, Chol* out) {
  out->n = n;
  out->l.assign((size_t)n * n, 0.0);
  auto& l = out->l;
  out->logdet = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int k = 0; k < j; ++k) s = fma_(l[(size_t)j * n + k], l[(size_t)j * n + k], s);
    const double d = b[(size_t)j * n + j] - s;
    if (!(d > 0.0)) return false;
    const double ljj = std::sqrt(d);
    l[(size_t)j * n + j] = ljj;
    out->logdet += 2.0 * std::log(ljj);
#pragma omp parallel for schedule(static)
    for (int i = j + 1; i < n; ++i) {
      double t = 0.0;
      const double* li = &l[(size_t)i * n];
      const double* lj = &l[(size_t)j * n];
      for (int k = 0; k < j; ++k) t = fma_(li[k], lj[k], t);
      l[(size_t)i * n + j] = (b[(size_t)i * n + j] - t) / ljj;
    }
  }
  return true;
}

static Nested static_fsai(const Mat& a) {
  Nested f;
  f.layout = a.rl;
  f.chain.push_back(build_fsai(a, LowerPattern::from_matrix(a)));
  return f;
}

static double lanczos_lambda_max(const Mat& a, const Nested& f, int iters, double safety,
                                 uint64_t seed) {
  const int n = a.rl.dim;
  auto op = [&](const double* x, double* y) { nested_apply_transformed(f, a, x, y); };
  const auto ritz = lanczos_ritz(op, n, iters, seed);
  return safety * ritz.back();
}

// setup: multilevel.cpp:36-75
static Hier setup(Mat a_finest, std::vector<Mat> transfers, int t_max, double tau, int nest,
                  int fsai_kind, int lanczos_iters, double safety, uint64_t seed, int cap,
                  bool probe, int kind, double omega, double fraction) {
  Hier h;
  const int depth = (int)transfers.size();
  h.levels.resize(depth + 1);
  h.levels[depth].A = std::move(a_finest);
  for (int l = depth; l >= 1; --l) {
    h.levels[l].P = std::move(transfers[l - 1]);
    h.levels[l - 1].A = galerkin(h.levels[l].A, h.levels[l].P);
  }
  if (probe) {
    for (int l = 0; l < depth; ++l) {
      const Mat& al = h.levels[l].A;
      auto op = [&](const double* x, double* y) { spmv(al, x, y); };
      const double ritz = lanczos_ritz(op, al.rl.dim, 30, seed).front();
      if (!(ritz > 0.0))
        std::fprintf(stderr,
                     "oracle: warning: level %d Galerkin operator looks indefinite (Ritz %.3e)\n", l,
                     ritz);
    }
  }
  for (int l = 1; l <= depth; ++l) {
    Level& lv = h.levels[l];
    lv.fsai = fsai_kind == 0 ? static_fsai(lv.A) : nested_build(lv.A, t_max, tau, nest);
    lv.beta = lanczos_lambda_max(lv.A, lv.fsai, lanczos_iters, safety, seed);
    lv.kind = kind;  // multilevel.cpp:62-65
    lv.alpha = fraction * lv.beta;
    lv.omega = omega;
  }
  const int n0 = h.levels.front().A.rl.dim;
  if (n0 > cap) throw std::invalid_argument("setup: coarsest level exceeds the dense-solve cap");
  if (!dense_cholesky(to_dense(h.levels.front().A), n0, &h.coarse))
    throw std::runtime_error("setup: coarsest operator is not positive definite");
  return h;
}

// v_cycle: multilevel.cpp:77-103 (fourth-kind smoothing)
static void v_cycle(const Hier& h, int k_pre, int k_post, int level, const double* b, double* x) {
  if (k_pre + k_post < 1) throw std::invalid_argument("v_cycle: cycle needs at least one smoothing step");
  if (level < 0 || level > h.finest()) throw std::out_of_range("v_cycle: level out of range");
  if (level == 0) {
    const int n = h.coarse.n;
    std::copy(b, b + n, x);
    h.coarse.solve(x);
    return;
  }
  const Level& lv = h.levels[level];
  const int n = lv.A.rl.dim;
  auto a_op = [&](const double* in, double* out) { spmv(lv.A, in, out); };
  auto m_op = [&](const double* in, double* out) { nested_apply(lv.fsai, in, out); };
  if (k_pre > 0) apply_smoother(lv.kind, lv.alpha, lv.beta, lv.omega, k_pre, a_op, m_op, b, x, n);
  std::vector<double> r(n);
  spmv(lv.A, x, r.data());
  for (int i = 0; i < n; ++i) r[i] = b[i] - r[i];
  const int nc = lv.P.cl.dim;
  std::vector<double> rc(nc), ec(nc, 0.0);
  spmv_t(lv.P, r.data(), rc.data());
  v_cycle(h, k_pre, k_post, level - 1, rc.data(), ec.data());
  std::vector<double> pe(n);
  spmv(lv.P, ec.data(), pe.data());
  for (int i = 0; i < n; ++i) x[i] += pe[i];
  if (k_post > 0) apply_smoother(lv.kind, lv.alpha, lv.beta, lv.omega, k_post, a_op, m_op, b, x, n);
}

}  // namespace orc

// ============================================================================
// C API
using namespace orc;

struct orc_mat { Mat m; };
struct orc_fsai { Nested f; };
struct orc_hier { Hier h; };

static thread_local std::string g_err;
static thread_local int g_pivot = -1;

template <class F>
static int guard(F&& f) {
  try {
    f();
    return ORC_OK;
  } catch (const NotPositiveDefinite& e) {
    g_err = e.what();
    g_pivot = e.pivot;
    return ORC_ENOTSPD;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ORC_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return ORC_ERANGE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_ERUNTIME;
  }
}

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_pivot(void) { return g_pivot; }
int orc_set_threads(int n) {
  omp_set_num_threads(n > 0 ? n : 1);
  return 0;
}
int orc_get_threads(void) { return omp_get_max_threads(); }

int orc_mat_create(int nbr, const int32_t* row_sizes, int nbc, const int32_t* col_sizes,
                   const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                   int symmetric, orc_mat** out) {
  return guard([&] {
    Layout rl(std::vector<int>(row_sizes, row_sizes + nbr));
    Layout cl(std::vector<int>(col_sizes, col_sizes + nbc));
    auto* h = new orc_mat{Mat(rl, cl, symmetric != 0)};
    std::unique_ptr<orc_mat> own(h);
    int64_t voff = 0;
    for (int i = 0; i < nbr; ++i) {
      const int mi = rl.sz[i];
      auto& c = h->m.cols[i];
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
        const int j = col_idx[p];
        if (j < 0 || j >= nbc) throw std::out_of_range("BlockSparseMatrix: block index out of range");
        if (!c.empty() && j <= c.back())
          throw std::invalid_argument("orc_mat_create: columns must be strictly ascending");
        c.push_back(j);
        h->m.boff[i].push_back(h->m.vals[i].size());
        const int mj = cl.sz[j];
        h->m.vals[i].insert(h->m.vals[i].end(), vals + voff, vals + voff + (int64_t)mi * mj);
        voff += (int64_t)mi * mj;
      }
    }
    *out = own.release();
  });
}

void orc_mat_destroy(orc_mat* a) { delete a; }

int orc_mat_info(const orc_mat* a, int* nbr, int* nbc, int64_t* nnzb, int64_t* nvals, int* dim_r,
                 int* dim_c) {
  return guard([&] {
    *nbr = a->m.nbr();
    *nbc = a->m.nbc();
    *nnzb = (int64_t)a->m.nnzb();
    int64_t nv = 0;
    for (auto& v : a->m.vals) nv += (int64_t)v.size();
    *nvals = nv;
    *dim_r = a->m.rl.dim;
    *dim_c = a->m.cl.dim;
  });
}

int orc_mat_export(const orc_mat* a, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  return guard([&] {
    int64_t p = 0, v = 0;
    row_ptr[0] = 0;
    for (int i = 0; i < a->m.nbr(); ++i) {
      for (int j : a->m.cols[i]) col_idx[p++] = j;
      row_ptr[i + 1] = p;
      std::copy(a->m.vals[i].begin(), a->m.vals[i].end(), vals + v);
      v += (int64_t)a->m.vals[i].size();
    }
  });
}

int orc_spmv(const orc_mat* a, const double* x, double* y) {
  return guard([&] { spmv(a->m, x, y); });
}
int orc_spmv_t(const orc_mat* a, const double* x, double* y) {
  return guard([&] { spmv_t(a->m, x, y); });
}
int orc_multiply(const orc_mat* a, const orc_mat* b, orc_mat** out) {
  return guard([&] { *out = new orc_mat{multiply(a->m, b->m)}; });
}
int orc_transpose_multiply(const orc_mat* p, const orc_mat* b, orc_mat** out) {
  return guard([&] { *out = new orc_mat{transpose_multiply(p->m, b->m)}; });
}
int orc_triple_product(const orc_mat* f, const orc_mat* a, orc_mat** out) {
  return guard([&] { *out = new orc_mat{triple_product(f->m, a->m)}; });
}
int orc_galerkin(const orc_mat* a, const orc_mat* p, orc_mat** out) {
  return guard([&] { *out = new orc_mat{galerkin(a->m, p->m)}; });
}

int orc_cholesky(int n, const double* b, double* l_out, double* logdet) {
  return guard([&] {
    Chol c(b, n, "");
    std::copy(c.l.begin(), c.l.end(), l_out);
    *logdet = c.logdet;
  });
}
int orc_chol_solve(int n, const double* l, const double* rhs, double* x) {
  return guard([&] {
    Chol c;
    c.n = n;
    c.l.assign(l, l + (size_t)n * n);
    std::copy(rhs, rhs + n, x);
    c.solve(x);
  });
}

int orc_fsai_build(const orc_mat* a, int kind, int t_max, double tau, int nest, orc_fsai** out) {
  return guard([&] {
    Nested f;
    f.layout = a->m.rl;
    switch (kind) {
      case 0: f.chain.push_back(build_fsai(a->m, LowerPattern::from_matrix(a->m))); break;
      case 1: f.chain.push_back(build_fsai(a->m, LowerPattern::diagonal(a->m.nbr()))); break;
      case 2: f.chain.push_back(build_fsai(a->m, LowerPattern::full(a->m.nbr()))); break;
      case 3: f = nested_build(a->m, t_max, tau, nest); break;
      default: throw std::invalid_argument("orc_fsai_build: unknown kind");
    }
    *out = new orc_fsai{std::move(f)};
  });
}
static LowerPattern pattern_from_csr(int n, const int64_t* pp, const int32_t* pc) {
  LowerPattern p = LowerPattern::diagonal(n);
  for (int i = 0; i < n; ++i)
    for (int64_t q = pp[i]; q < pp[i + 1]; ++q) p.add(i, pc[q]);
  return p;
}
int orc_fsai_build_pattern(const orc_mat* a, const int64_t* pat_ptr, const int32_t* pat_col,
                           orc_fsai** out) {
  return guard([&] {
    Nested f;
    f.layout = a->m.rl;
    f.chain.push_back(build_fsai(a->m, pattern_from_csr(a->m.nbr(), pat_ptr, pat_col)));
    *out = new orc_fsai{std::move(f)};
  });
}
int orc_delta_ratio(const orc_mat* a, const int64_t* pat_ptr, const int32_t* pat_col, int k, int c,
                    double* out) {
  return guard([&] {
    check_spd_inputs(a->m);
    const LowerPattern p = pattern_from_csr(a->m.nbr(), pat_ptr, pat_col);
    RowMap frow;
    Chol s, gram;
    build_row(a->m, p, k, frow, s, gram);  // make_adaptive_state, fsai.cpp:90-104
    const RowMap h = build_h_row(a->m, frow, k);
    auto it = h.find(c);
    if (it == h.end()) throw std::invalid_argument("delta_ratio: H_kc not stored");
    *out = delta_ratio(a->m, p, gram, s, k, c, it->second);
  });
}
void orc_fsai_destroy(orc_fsai* f) { delete f; }
int orc_fsai_apply(const orc_fsai* f, const double* r, double* out) {
  return guard([&] { nested_apply(f->f, r, out); });
}
int orc_fsai_apply_transformed(const orc_fsai* f, const orc_mat* a, const double* x, double* out) {
  return guard([&] { nested_apply_transformed(f->f, a->m, x, out); });
}
int orc_fsai_chain_len(const orc_fsai* f) { return (int)f->f.chain.size(); }
int orc_fsai_factor(const orc_fsai* f, int k, orc_mat** F_out) {
  return guard([&] {
    if (k < 0 || k >= (int)f->f.chain.size()) throw std::out_of_range("orc_fsai_factor");
    *F_out = new orc_mat{f->f.chain[k].F};
  });
}
int orc_fsai_shat(const orc_fsai* f, double* l_packed) {
  return guard([&] {
    size_t o = 0;
    for (const Chol& c : f->f.final_diag()) {
      std::copy(c.l.begin(), c.l.end(), l_packed + o);
      o += c.l.size();
    }
  });
}
// G = L-hat^{-1} F_last (the last factor of the chain): G_kj = L_k^{-1} F_kj,
// column-wise forward substitution with the Chol::solve_l order.
int orc_fsai_G(const orc_fsai* f, orc_mat** G_out) {
  return guard([&] {
    const Factors& fac = f->f.chain.back();
    const Mat& F = fac.F;
    Mat G = F;
    for (int k = 0; k < F.nbr(); ++k) {
      const Chol& s = fac.S[k];
      const int mk = F.rl.sz[k];
      for (size_t q = 0; q < F.cols[k].size(); ++q) {
        const int mj = F.cl.sz[F.cols[k][q]];
        double* g = G.blk(k, (int)q);
        std::vector<double> col(mk);
        for (int c = 0; c < mj; ++c) {
          for (int r = 0; r < mk; ++r) col[r] = g[r * mj + c];
          s.solve_l(col.data());
          for (int r = 0; r < mk; ++r) g[r * mj + c] = col[r];
        }
      }
    }
    G.sym = false;
    G.tidx_ok = false;
    *G_out = new orc_mat{std::move(G)};
  });
}

int orc_lanczos_lambda_max(const orc_mat* a, const orc_fsai* f, int iters, double safety,
                           uint64_t seed, double* beta) {
  return guard([&] { *beta = lanczos_lambda_max(a->m, f->f, iters, safety, seed); });
}
int orc_lanczos_diag(int n, const double* lam, int iters, double safety, uint64_t seed,
                     int smallest, double* out) {
  return guard([&] {
    auto op = [&](const double* x, double* y) {
      for (int i = 0; i < n; ++i) y[i] = lam[i] * x[i];
    };
    auto ritz = lanczos_ritz(op, n, iters, seed);
    *out = smallest ? ritz.front() : safety * ritz.back();
  });
}
int orc_tridiag_eigs(int n, const double* d, const double* e, double* eig_sorted) {
  return guard([&] {
    std::vector<double> dd(d, d + n), ee(e, e + (n > 0 ? n - 1 : 0));
    auto ev = tridiag_eigs(dd, ee);
    std::copy(ev.begin(), ev.end(), eig_sorted);
  });
}

int orc_smoother_apply(const orc_mat* a, const orc_fsai* f, int kind, double alpha, double beta,
                       double omega, int k, const double* b, double* x) {
  return guard([&] {
    const int n = a->m.rl.dim;
    auto a_op = [&](const double* in, double* out) { spmv(a->m, in, out); };
    if (f) {
      auto m_op = [&](const double* in, double* out) { nested_apply(f->f, in, out); };
      apply_smoother(kind, alpha, beta, omega, k, a_op, m_op, b, x, n);
    } else {
      auto m_op = [&](const double* in, double* out) { std::copy(in, in + n, out); };
      apply_smoother(kind, alpha, beta, omega, k, a_op, m_op, b, x, n);
    }
  });
}
int orc_smoother_apply_diag(int n, const double* lam, int kind, double alpha, double beta,
                            double omega, int k, const double* b, double* x) {
  return guard([&] {
    auto a_op = [&](const double* in, double* out) {
      for (int i = 0; i < n; ++i) out[i] = lam[i] * in[i];
    };
    auto m_op = [&](const double* in, double* out) { std::copy(in, in + n, out); };
    apply_smoother(kind, alpha, beta, omega, k, a_op, m_op, b, x, n);
  });
}
int orc_poly_eval(int kind, int degree, double alpha, double beta, double t, double* out) {
  return guard([&] { *out = poly_eval(kind, degree, alpha, beta, t); });
}
double orc_fourth_kind_mu(int n) { return fourth_kind_mu(n); }

static bool g_consume = false;
int orc_set_consume(int on) {
  g_consume = on != 0;
  return 0;
}
int orc_setup(const orc_mat* a_finest, int ntransfers, const orc_mat* const* transfers, int t_max,
              double tau, int nest, int fsai_kind, int lanczos_iters, double lanczos_safety,
              uint64_t seed, int coarse_dim_cap, int smallest_ritz_probe, int smoother_kind,
              double richardson_omega, double first_kind_fraction, orc_hier** out) {
  return guard([&] {
    // consume mode (orc_set_consume): the inputs are moved into the hierarchy and
    // left empty, so a large config (C4: 20 GB of A, 21 GB of P) is not held twice
    std::vector<Mat> tr;
    for (int i = 0; i < ntransfers; ++i)
      tr.push_back(g_consume ? std::move(const_cast<orc_mat*>(transfers[i])->m) : transfers[i]->m);
    Mat a = g_consume ? std::move(const_cast<orc_mat*>(a_finest)->m) : a_finest->m;
    *out = new orc_hier{setup(std::move(a), std::move(tr), t_max, tau, nest, fsai_kind,
                              lanczos_iters, lanczos_safety, seed, coarse_dim_cap,
                              smallest_ritz_probe != 0, smoother_kind, richardson_omega,
                              first_kind_fraction)};
  });
}
void orc_hier_destroy(orc_hier* h) { delete h; }
int orc_hier_levels(const orc_hier* h) { return (int)h->h.levels.size(); }
int orc_hier_level_A(const orc_hier* h, int l, const orc_mat** a) {
  return guard([&] {
    if (l < 0 || l > h->h.finest()) throw std::out_of_range("level");
    *a = reinterpret_cast<const orc_mat*>(&h->h.levels[l].A);
  });
}
int orc_hier_level_P(const orc_hier* h, int l, const orc_mat** p) {
  return guard([&] {
    if (l < 1 || l > h->h.finest()) throw std::out_of_range("level");
    *p = reinterpret_cast<const orc_mat*>(&h->h.levels[l].P);
  });
}
int orc_hier_level_fsai(const orc_hier* h, int l, const orc_fsai** f) {
  return guard([&] {
    if (l < 1 || l > h->h.finest()) throw std::out_of_range("level");
    *f = reinterpret_cast<const orc_fsai*>(&h->h.levels[l].fsai);
  });
}
int orc_hier_beta(const orc_hier* h, int l, double* beta) {
  return guard([&] {
    if (l < 1 || l > h->h.finest()) throw std::out_of_range("level");
    *beta = h->h.levels[l].beta;
  });
}
int orc_hier_coarse_l(const orc_hier* h, double* l_dense) {
  return guard([&] { std::copy(h->h.coarse.l.begin(), h->h.coarse.l.end(), l_dense); });
}
int orc_vcycle(const orc_hier* h, int k_pre, int k_post, int level, const double* b, double* x) {
  return guard([&] { v_cycle(h->h, k_pre, k_post, level, b, x); });
}
int orc_solve(const orc_hier* h, int k_pre, int k_post, const double* b, double* x, double tol,
              int max_iter, double* hist, int* iters, int* status) {
  return guard([&] {
    const Mat& a = h->h.levels.back().A;
    const int n = a.rl.dim;
    std::vector<double> t(n);
    auto resid = [&]() {
      spmv(a, x, t.data());
      for (int i = 0; i < n; ++i) t[i] = b[i] - t[i];
      return norm2(t.data(), n);
    };
    hist[0] = resid();
    int it = 0;
    int st = 1;
    if (hist[0] == 0.0 || hist[0] / hist[0] < tol) st = 0;
    while (st == 1 && it < max_iter) {
      v_cycle(h->h, k_pre, k_post, h->h.finest(), b, x);
      ++it;
      hist[it] = resid();
      const double growth = hist[it] / std::max(hist[it - 1], 1e-300);
      if (!std::isfinite(hist[it]) || growth > 1e6) {  // experiments.cpp:50-56
        st = 2;
        break;
      }
      if (hist[it] / hist[0] < tol) st = 0;
    }
    *iters = it;
    *status = st;
  });
}

// measure_rates: experiments.cpp:15-67.  Initial error e_i = CounterRng(seed)
// .symmetric(i) normalised to unit M-norm, x = u_ref + e; after every cycle record
// the squared M- and A-norms of x - u_ref and ||b - A((x - u_ref) + u_ref)||;
// converged when the squared M-norm drops below tol^2; rates from the histories.
int orc_measure_rates(const orc_hier* h, const orc_mat* mass, const double* b, const double* u_ref, int k_pre,
                      int k_post, uint64_t seed, double tol, int max_iter, double* l2_sq, double* energy_sq,
                      double* residual, int* iters, int* status, int* blowup, double* rates) {
  return guard([&] {
    const Mat& a = h->h.levels.back().A;
    const Mat& m = mass->m;
    const int n = a.rl.dim;
    require(m.rl.dim == n && m.cl.dim == n, "measure_rates: mass matrix does not match the finest level");
    std::vector<double> e(n), tmp(n), x(n), w(n);
    for (int i = 0; i < n; ++i) e[i] = rng_symmetric(seed, (uint64_t)i);  // CounterRng::symmetric
    spmv(m, e.data(), tmp.data());
    const double s = std::sqrt(dot(e.data(), tmp.data(), n));
    for (int i = 0; i < n; ++i) e[i] /= s;
    for (int i = 0; i < n; ++i) x[i] = u_ref[i] + e[i];
    int rec = 0;
    auto record = [&](const double* err) {
      spmv(m, err, tmp.data());
      l2_sq[rec] = dot(err, tmp.data(), n);
      spmv(a, err, tmp.data());
      energy_sq[rec] = dot(err, tmp.data(), n);
      for (int i = 0; i < n; ++i) w[i] = err[i] + u_ref[i];
      spmv(a, w.data(), tmp.data());
      for (int i = 0; i < n; ++i) tmp[i] = b[i] - tmp[i];
      residual[rec] = norm2(tmp.data(), n);
      ++rec;
    };
    record(e.data());
    const double tol_sq = tol * tol;
    int it = 0, st = 1;
    *blowup = -1;
    if (l2_sq[0] < tol_sq) st = 0;
    while (st == 1 && it < max_iter) {
      v_cycle(h->h, k_pre, k_post, h->h.finest(), b, x.data());
      ++it;
      for (int i = 0; i < n; ++i) e[i] = x[i] - u_ref[i];
      record(e.data());
      const double growth = residual[it] / std::max(residual[it - 1], 1e-300);
      if (!std::isfinite(residual[it]) || growth > 1e6) {
        st = 2;
        *blowup = it;
        break;
      }
      if (l2_sq[it] < tol_sq) st = 0;
    }
    *iters = it;
    *status = st;
    rates[0] = rates[1] = rates[2] = 0.0;
    if (it > 0) {
      const double ex = 1.0 / (2.0 * it);
      rates[0] = std::pow(l2_sq[it] / l2_sq[0], ex);
      rates[1] = std::pow(energy_sq[it] / energy_sq[0], ex);
      rates[2] = std::pow(residual[it] / residual[0], 1.0 / it);
    }
  });
}

uint64_t orc_mix64(uint64_t z) { return mix64(z); }
double orc_rng_uniform(uint64_t seed, uint64_t i) { return rng_uniform(seed, i); }

}  // extern "C"
