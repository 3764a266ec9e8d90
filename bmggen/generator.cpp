// generator.cpp -- synthetic BASELINE problems (BASELINE.json configs).
//
// Built as its own library, bmggen/libbmggen.so (C ABI in include/bmg_gen.h),
// shared by both benchmark arms and the tests: it is input data, not the
// solver, so neither the product (libbmgcuda.so) nor the CPU oracle contains it.
//
// Input data only (the reference's PUM discretiser is out of scope):
//   A_ij = (S_p)_ij C            i != j
//   A_ii = (S_p)_ii C + reg D_i
// with S_p = L_D^p, L_D the unscaled Dirichlet 5-point (2-D) / 7-point (3-D)
// Laplacian on an n^dim patch grid (block index ((z n) + y) n + x, as
// pum/cover.hpp:25), C = Q diag(U[1,10]) Q^T (Q from Gram-Schmidt of an m x m
// N(0,1) matrix), D_i = R_i R_i^T + I with R_i ~ N(0,1); C and D_i symmetrised
// exactly.  Random numbers are the reference's SplitMix64 counter stream
// (rng.hpp:12-36) with one derived stream per object; N(0,1) by Box-Muller on
// two uniforms of the stream.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include <exception>
#include <string>

#include "../include/bmg_gen.h"

namespace bmg {
namespace gen {

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static inline double uniform(uint64_t seed, uint64_t i) {
  const uint64_t bits = mix64(seed + (i + 1) * 0x9e3779b97f4a7c15ULL);
  return (static_cast<double>(bits >> 11) + 0.5) * 0x1.0p-53;
}
// stream seeds: one per object
enum : uint64_t { kTagCEig = 1, kTagQ = 2, kTagD = 3, kTagP = 4, kTagB = 5 };
static inline uint64_t stream_seed(uint64_t seed, uint64_t tag) {
  return mix64(seed ^ (0x5bd1e995ULL * (tag + 1)));
}
static inline double normal(uint64_t s, uint64_t i) {
  const double u1 = uniform(s, 2 * i), u2 = uniform(s, 2 * i + 1);
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

struct Grid {
  int dim, n;
  int64_t count() const { return dim == 2 ? (int64_t)n * n : (int64_t)n * n * n; }
};

// row of S_p = L_D^p at node i, returned as (column, value) ascending
static void stencil_row(const Grid& g, int power, int64_t node, std::vector<int64_t>& cols,
                        std::vector<int64_t>& vals) {
  const int R = power;  // support radius in each coordinate
  const int W = 2 * R + 1;
  const int wz = g.dim == 3 ? W : 1;
  int x = (int)(node % g.n), y = (int)((node / g.n) % g.n), z = g.dim == 3 ? (int)(node / ((int64_t)g.n * g.n)) : 0;
  std::vector<int64_t> v((size_t)W * W * wz, 0), t((size_t)W * W * wz, 0);
  auto idx = [&](int dx, int dy, int dz) { return ((size_t)(dz + (g.dim == 3 ? R : 0)) * W + (dy + R)) * W + (dx + R); };
  auto inside = [&](int dx, int dy, int dz) {
    const int X = x + dx, Y = y + dy, Z = z + dz;
    return X >= 0 && X < g.n && Y >= 0 && Y < g.n && (g.dim == 2 || (Z >= 0 && Z < g.n));
  };
  v[idx(0, 0, 0)] = 1;
  const int zr = g.dim == 3 ? R : 0;
  for (int p = 0; p < power; ++p) {
    std::fill(t.begin(), t.end(), 0);
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -R; dy <= R; ++dy)
        for (int dx = -R; dx <= R; ++dx) {
          if (!inside(dx, dy, dz)) continue;
          int64_t s = 2 * g.dim * v[idx(dx, dy, dz)];
          const int nb[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
          for (int q = 0; q < 2 * g.dim; ++q) {
            const int ex = dx + nb[q][0], ey = dy + nb[q][1], ez = dz + nb[q][2];
            if (ex < -R || ex > R || ey < -R || ey > R || ez < -zr || ez > zr) continue;
            if (!inside(ex, ey, ez)) continue;
            s -= v[idx(ex, ey, ez)];
          }
          t[idx(dx, dy, dz)] = s;
        }
    v.swap(t);
  }
  cols.clear();
  vals.clear();
  for (int dz = -zr; dz <= zr; ++dz)
    for (int dy = -R; dy <= R; ++dy)
      for (int dx = -R; dx <= R; ++dx) {
        const int64_t s = v[idx(dx, dy, dz)];
        if (s == 0 || !inside(dx, dy, dz)) continue;
        const int64_t col = (((int64_t)(z + dz) * g.n) + (y + dy)) * g.n + (x + dx);
        cols.push_back(col);
        vals.push_back(s);
      }
}

// C = Q diag(lambda) Q^T, lambda ~ U[1,10], Q = Gram-Schmidt(N(0,1) m x m)
static std::vector<double> make_c(int m, uint64_t seed) {
  const uint64_t se = stream_seed(seed, kTagCEig), sq = stream_seed(seed, kTagQ);
  std::vector<double> q((size_t)m * m);
  for (int i = 0; i < m * m; ++i) q[i] = normal(sq, (uint64_t)i);
  // modified Gram-Schmidt on columns of q (row-major storage, column j = q[:, j])
  for (int j = 0; j < m; ++j) {
    for (int k = 0; k < j; ++k) {
      double d = 0.0;
      for (int i = 0; i < m; ++i) d += q[(size_t)i * m + k] * q[(size_t)i * m + j];
      for (int i = 0; i < m; ++i) q[(size_t)i * m + j] -= d * q[(size_t)i * m + k];
    }
    double nrm = 0.0;
    for (int i = 0; i < m; ++i) nrm += q[(size_t)i * m + j] * q[(size_t)i * m + j];
    nrm = std::sqrt(nrm);
    for (int i = 0; i < m; ++i) q[(size_t)i * m + j] /= nrm;
  }
  std::vector<double> lam(m);
  for (int i = 0; i < m; ++i) lam[i] = 1.0 + 9.0 * uniform(se, (uint64_t)i);
  std::vector<double> c((size_t)m * m, 0.0);
  for (int r = 0; r < m; ++r)
    for (int s = 0; s < m; ++s) {
      double acc = 0.0;
      for (int k = 0; k < m; ++k) acc += q[(size_t)r * m + k] * lam[k] * q[(size_t)s * m + k];
      c[(size_t)r * m + s] = acc;
    }
  for (int r = 0; r < m; ++r)
    for (int s = r + 1; s < m; ++s) {
      const double a = 0.5 * (c[(size_t)r * m + s] + c[(size_t)s * m + r]);
      c[(size_t)r * m + s] = a;
      c[(size_t)s * m + r] = a;
    }
  return c;
}

}  // namespace gen

int64_t gen_stencil(int dim, int n, int power, int m, uint64_t seed, double reg, int64_t row_lo,
                    int64_t row_hi, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  using namespace gen;
  if (dim != 2 && dim != 3) throw std::invalid_argument("gen_stencil: dim must be 2 or 3");
  if (n < 1 || power < 1 || m < 1) throw std::invalid_argument("gen_stencil: bad sizes");
  Grid g{dim, n};
  const int64_t total = g.count();
  if (total >= (int64_t)1 << 31) throw std::invalid_argument("gen_stencil: grid too large");
  if (row_hi < 0) row_hi = total;
  if (row_lo < 0 || row_lo > row_hi || row_hi > total) throw std::invalid_argument("gen_stencil: bad row range");
  const int64_t nodes = row_hi - row_lo;  // rows [row_lo, row_hi), global column indices
  // pass 1: counts
  std::vector<int64_t> cnt(nodes + 1, 0);
#pragma omp parallel
  {
    std::vector<int64_t> c, v;
#pragma omp for schedule(static)
    for (int64_t li = 0; li < nodes; ++li) {
      stencil_row(g, power, row_lo + li, c, v);
      cnt[li + 1] = (int64_t)c.size();
    }
  }
  for (int64_t i = 0; i < nodes; ++i) cnt[i + 1] += cnt[i];
  const int64_t nnzb = cnt[nodes];
  if (!row_ptr) return nnzb;
  std::memcpy(row_ptr, cnt.data(), sizeof(int64_t) * (nodes + 1));
  const std::vector<double> C = make_c(m, seed);
  const uint64_t sd = stream_seed(seed, kTagD);
  const size_t mm = (size_t)m * m;
#pragma omp parallel
  {
    std::vector<int64_t> c, v;
    std::vector<double> R(mm);
#pragma omp for schedule(static)
    for (int64_t li = 0; li < nodes; ++li) {
      const int64_t i = row_lo + li;
      stencil_row(g, power, i, c, v);
      int64_t p = cnt[li];
      for (size_t q = 0; q < c.size(); ++q, ++p) {
        col_idx[p] = (int32_t)c[q];
        double* blk = vals + (size_t)p * mm;
        const double s = (double)v[q];
        for (size_t e = 0; e < mm; ++e) blk[e] = s * C[e];
        if (c[q] == i && reg != 0.0) {
          for (size_t e = 0; e < mm; ++e) R[e] = normal(sd, (uint64_t)i * mm + e);
          // D = R R^T + I, exactly symmetric
          for (int r = 0; r < m; ++r)
            for (int s2 = r; s2 < m; ++s2) {
              double acc = 0.0;
              for (int k = 0; k < m; ++k) acc += R[(size_t)r * m + k] * R[(size_t)s2 * m + k];
              if (r == s2) acc += 1.0;
              const double add = reg * acc;
              blk[(size_t)r * m + s2] += add;
              if (s2 != r) blk[(size_t)s2 * m + r] += add;
            }
        }
      }
    }
  }
  return nnzb;
}

// P rows: fine patch -> parent (coords >> 1) and the parent's 8 (2-D) / 26 (3-D)
// neighbours clipped to the coarse grid; entries N(0,1)/9; each fine block row
// scaled to Frobenius norm sqrt(m) (BASELINE.md §4 decision 2).
int64_t gen_prolongation(int dim, int n_fine, int m, uint64_t seed, int level, int64_t row_lo, int64_t row_hi,
                         int64_t* row_ptr, int32_t* col_idx, double* vals) {
  using namespace gen;
  if (dim != 2 && dim != 3) throw std::invalid_argument("gen_prolongation: dim must be 2 or 3");
  if (n_fine < 2 || (n_fine & 1)) throw std::invalid_argument("gen_prolongation: n_fine must be even");
  const int nf = n_fine, nc = n_fine / 2;
  const int64_t total = dim == 2 ? (int64_t)nf * nf : (int64_t)nf * nf * nf;
  if (row_hi < 0) row_hi = total;
  if (row_lo < 0 || row_lo > row_hi || row_hi > total) throw std::invalid_argument("gen_prolongation: bad row range");
  const int64_t nodes = row_hi - row_lo;
  const int zr = dim == 3 ? 1 : 0;
  auto row_cols = [&](int64_t i, std::vector<int32_t>& cols) {
    cols.clear();
    const int x = (int)(i % nf), y = (int)((i / nf) % nf), z = dim == 3 ? (int)(i / ((int64_t)nf * nf)) : 0;
    const int px = x >> 1, py = y >> 1, pz = z >> 1;
    for (int dz = -zr; dz <= zr; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int X = px + dx, Y = py + dy, Z = pz + dz;
          if (X < 0 || X >= nc || Y < 0 || Y >= nc) continue;
          if (dim == 3 && (Z < 0 || Z >= nc)) continue;
          cols.push_back((int32_t)((((int64_t)(dim == 3 ? Z : 0) * nc) + Y) * nc + X));
        }
  };
  std::vector<int64_t> cnt(nodes + 1, 0);
#pragma omp parallel
  {
    std::vector<int32_t> c;
#pragma omp for schedule(static)
    for (int64_t li = 0; li < nodes; ++li) {
      row_cols(row_lo + li, c);
      cnt[li + 1] = (int64_t)c.size();
    }
  }
  for (int64_t i = 0; i < nodes; ++i) cnt[i + 1] += cnt[i];
  const int64_t nnzb = cnt[nodes];
  if (!row_ptr) return nnzb;
  std::memcpy(row_ptr, cnt.data(), sizeof(int64_t) * (nodes + 1));
  const uint64_t sp = stream_seed(seed ^ ((uint64_t)level << 32), kTagP);
  const size_t mm = (size_t)m * m;
  const int maxb = dim == 3 ? 27 : 9;
#pragma omp parallel
  {
    std::vector<int32_t> c;
#pragma omp for schedule(static)
    for (int64_t li = 0; li < nodes; ++li) {
      const int64_t i = row_lo + li;
      row_cols(i, c);
      const int64_t p0 = cnt[li];
      double ss = 0.0;
      for (size_t q = 0; q < c.size(); ++q) {
        col_idx[p0 + q] = c[q];
        double* blk = vals + (size_t)(p0 + q) * mm;
        for (size_t e = 0; e < mm; ++e) {
          // counter index: (row, slot, entry), slot = position of the block
          const double v = normal(sp, ((uint64_t)i * maxb + q) * mm + e) / 9.0;
          blk[e] = v;
          ss += v * v;
        }
      }
      const double scale = std::sqrt((double)m) / std::sqrt(ss);
      for (size_t e = 0; e < c.size() * mm; ++e) vals[(size_t)p0 * mm + e] *= scale;
    }
  }
  return nnzb;
}

void gen_normal(uint64_t seed, uint64_t tag, int64_t n, double* out) {
  using namespace gen;
  const uint64_t s = stream_seed(seed, kTagB + tag);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) out[i] = normal(s, (uint64_t)i);
}

}  // namespace bmg

// ---- C ABI (include/bmg_gen.h) ------------------------------------------
namespace {
thread_local std::string g_gen_err;
template <class F>
int gen_guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_gen_err = e.what();
    return 1;  // BMG_EINVAL
  } catch (const std::exception& e) {
    g_gen_err = e.what();
    return 4;  // BMG_ERUNTIME
  }
}
}  // namespace

extern "C" {
const char* bmg_gen_last_error(void) { return g_gen_err.c_str(); }
int bmg_gen_stencil(int dim, int n, int power, int m, uint64_t seed, double reg, int64_t row_lo, int64_t row_hi,
                    int64_t* nnzb, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  return gen_guard([&] {
    *nnzb = bmg::gen_stencil(dim, n, power, m, seed, reg, row_lo, row_hi, row_ptr, col_idx, vals);
  });
}
int bmg_gen_prolongation(int dim, int n_fine, int m, uint64_t seed, int level, int64_t row_lo, int64_t row_hi,
                         int64_t* nnzb, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  return gen_guard([&] {
    *nnzb = bmg::gen_prolongation(dim, n_fine, m, seed, level, row_lo, row_hi, row_ptr, col_idx, vals);
  });
}
int bmg_gen_normal(uint64_t seed, uint64_t tag, int64_t n, double* out) {
  return gen_guard([&] { bmg::gen_normal(seed, tag, n, out); });
}
}  // extern "C"
