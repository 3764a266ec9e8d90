// multilevel.cu -- Galerkin coarsening, device Lanczos, the coarse direct solve,
// the device-resident V-cycle (captured as a CUDA graph) and the solve loop.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <tuple>

#include "bmg_abi.h"
#include "bmg_internal.h"

namespace bmg {
namespace kern {

// out = pairs-accumulated block products (Galerkin numeric phase):
// out[o] = sum over pairs (in order) of a_blk * b_blk   (kernels.cpp:71)
//                                   or a_blk^T * b_blk  (kernels.cpp:82)
__global__ void pair_gemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                                 const int64_t* __restrict__ pair_ptr,
                                 const int2* __restrict__ pairs, double* __restrict__ out,
                                 int64_t nout, int m, int bs_a, int bs_b, int bs_o, int transpose_a) {
  const int r = threadIdx.x / m, c = threadIdx.x - (threadIdx.x / m) * m;
  if (r >= m) return;
  for (int64_t o = blockIdx.x; o < nout; o += gridDim.x) {
    double acc = 0.0;
    for (int64_t q = pair_ptr[o]; q < pair_ptr[o + 1]; ++q) {
      const int2 pr = pairs[q];
      const double* a = A + (int64_t)pr.x * bs_a;
      const double* b = B + (int64_t)pr.y * bs_b;
      double t = 0.0;
      if (transpose_a)
        for (int k = 0; k < m; ++k) t = __fma_rn(a[k * m + r], b[k * m + c], t);
      else
        for (int k = 0; k < m; ++k) t = __fma_rn(a[r * m + k], b[k * m + c], t);
      acc = __dadd_rn(acc, t);
    }
    out[o * bs_o + r * m + c] = acc;
  }
}

// out(I,J)[r][c] = 0.5 * (C_IJ[r][c] + C_JI[c][r])   (multilevel.cpp:16-26)
__global__ void symmetrize_kernel(const double* __restrict__ C, const int64_t* __restrict__ tpos,
                                  double* __restrict__ out, int64_t nblk, int m, int bs) {
  const int r = threadIdx.x / m, c = threadIdx.x - (threadIdx.x / m) * m;
  if (r >= m) return;
  for (int64_t o = blockIdx.x; o < nblk; o += gridDim.x) {
    const int64_t t = tpos[o];
    const double v = C[o * bs + r * m + c];
    out[o * bs + r * m + c] = t >= 0 ? __dmul_rn(0.5, __dadd_rn(v, C[t * bs + c * m + r])) : __dmul_rn(v, 0.5);
  }
}

__global__ void bsr_to_dense_kernel(const double* __restrict__ vals, const int64_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ col, int nbr, int m, int bs,
                                    double* __restrict__ dense, int64_t N) {
  for (int i = blockIdx.x; i < nbr; i += gridDim.x)
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int j = col[p];
      for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int r = e / m, c = e - r * m;
        dense[((int64_t)i * m + r) * N + (int64_t)j * m + c] = vals[p * bs + e];
      }
    }
}

__global__ void symmetrize_dense_kernel(double* a, int64_t N) {
  // cuSOLVER potri (column-major lower) leaves the row-major upper triangle
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * N; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / N, c = e - r * N;
    if (r > c) a[e] = a[c * N + r];
  }
}

// x = Ainv b (dense, row-major): warp per row, double2 loads
__global__ void __launch_bounds__(256) gemv_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                   double* __restrict__ x, int64_t N) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= N) return;
  const double* ar = a + row * N;
  double s = 0.0;
  if ((N & 1) == 0) {
    const double2* a2 = reinterpret_cast<const double2*>(ar);
    const double2* b2 = reinterpret_cast<const double2*>(b);
    for (int64_t q = lane; q < N / 2; q += 32) {
      const double2 av = __ldg(a2 + q), bv = __ldg(b2 + q);
      s = __fma_rn(av.x, bv.x, s);
      s = __fma_rn(av.y, bv.y, s);
    }
  } else {
    for (int64_t q = lane; q < N; q += 32) s = __fma_rn(__ldg(ar + q), __ldg(b + q), s);
  }
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xffffffffu, s, o));
  if (lane == 0) x[row] = s;
}

__global__ void rng_symmetric_kernel(double* v, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ULL;  // rng.hpp:22-24
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    const double u = __dmul_rn(__dadd_rn((double)(z >> 11), 0.5), 0x1.0p-53);
    v[i] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
  }
}
__global__ void scale_div_kernel(double* v, int64_t n, double d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __ddiv_rn(v[i], d);
}
// w -= alpha v; w -= beta vp    (lanczos.hpp:31-32)
__global__ void lanczos_update_kernel(double* w, const double* v, const double* vp, int64_t n, double alpha,
                                      double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double t = __dsub_rn(w[i], __dmul_rn(alpha, v[i]));
    w[i] = __dsub_rn(t, __dmul_rn(beta, vp[i]));
  }
}

}  // namespace kern

static int grid1d(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16));
}

// ============================================================================ Galerkin
// Symbolic phase on the host (integer structure only), numeric phase on the
// device with the reference's accumulation order:  C = P^T (A P) then
// A_c = (C + C^T) / 2 blockwise (multilevel.cpp:11-28, kernels.cpp:66-86).
namespace {

struct Product {
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<int64_t> pair_ptr;
  std::vector<int2> pairs;
};

// C = X * Y symbolic with ordered pairs; X given as (rows of X): for output row i,
// `left(i)` yields (k, xblk) ascending k, Y rows give (j, yblk) ascending j.
template <class LeftRow>
Product symbolic(int nrows, const LeftRow& left, const std::vector<int64_t>& yrp, const std::vector<int32_t>& ycol) {
  Product out;
  std::vector<std::vector<int32_t>> rcol(nrows);
  std::vector<std::vector<int64_t>> rpp(nrows);
  std::vector<std::vector<int2>> rpairs(nrows);
#pragma omp parallel
  {
    std::vector<std::tuple<int32_t, int32_t, int32_t>> trip;  // (j, xblk, yblk)
#pragma omp for schedule(dynamic, 64)
    for (int i = 0; i < nrows; ++i) {
      trip.clear();
      left(i, [&](int k, int64_t xb) {
        for (int64_t q = yrp[k]; q < yrp[k + 1]; ++q) trip.emplace_back(ycol[q], (int32_t)xb, (int32_t)q);
      });
      std::stable_sort(trip.begin(), trip.end(),
                       [](const auto& a, const auto& b) { return std::get<0>(a) < std::get<0>(b); });
      auto& c = rcol[i];
      auto& pp = rpp[i];
      auto& pr = rpairs[i];
      for (size_t t = 0; t < trip.size(); ++t) {
        if (t == 0 || std::get<0>(trip[t]) != std::get<0>(trip[t - 1])) {
          c.push_back(std::get<0>(trip[t]));
          pp.push_back((int64_t)pr.size());
        }
        pr.push_back(make_int2(std::get<1>(trip[t]), std::get<2>(trip[t])));
      }
    }
  }
  out.row_ptr.assign(nrows + 1, 0);
  for (int i = 0; i < nrows; ++i) out.row_ptr[i + 1] = out.row_ptr[i] + (int64_t)rcol[i].size();
  out.col.resize(out.row_ptr[nrows]);
  out.pair_ptr.resize(out.row_ptr[nrows] + 1);
  std::vector<int64_t> pbase(nrows + 1, 0);
  for (int i = 0; i < nrows; ++i) pbase[i + 1] = pbase[i] + (int64_t)rpairs[i].size();
  out.pairs.resize(pbase[nrows]);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < nrows; ++i) {
    std::copy(rcol[i].begin(), rcol[i].end(), out.col.begin() + out.row_ptr[i]);
    for (size_t t = 0; t < rpp[i].size(); ++t) out.pair_ptr[out.row_ptr[i] + t] = pbase[i] + rpp[i][t];
    std::copy(rpairs[i].begin(), rpairs[i].end(), out.pairs.begin() + pbase[i]);
  }
  out.pair_ptr[out.row_ptr[nrows]] = pbase[nrows];
  return out;
}

void pair_gemm(Ctx* ctx, const double* A, int bs_a, const double* B, int bs_b, const Product& pr, double* out,
               int bs_o, int m, bool ta) {
  const int64_t nout = (int64_t)pr.col.size();
  if (nout == 0) return;
  DBuf<int64_t> pp(pr.pair_ptr.size());
  DBuf<int2> pairs(std::max<size_t>(pr.pairs.size(), 1));
  BMG_CUDA(cudaMemcpy(pp.p, pr.pair_ptr.data(), pr.pair_ptr.size() * 8, cudaMemcpyHostToDevice));
  if (!pr.pairs.empty())
    BMG_CUDA(cudaMemcpy(pairs.p, pr.pairs.data(), pr.pairs.size() * sizeof(int2), cudaMemcpyHostToDevice));
  const int threads = ((m * m + 31) / 32) * 32;
  const int grid = (int)std::min<int64_t>(nout, (int64_t)ctx->sms * 32);
  kern::pair_gemm_kernel<<<grid, threads, 0, ctx->stream>>>(A, B, pp.p, pairs.p, out, nout, m, bs_a, bs_b, bs_o,
                                                            ta ? 1 : 0);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace

std::unique_ptr<Bsr> galerkin(const Bsr& a, const Bsr& p) {
  if (!(a.rsz == a.csz) || !(a.rsz == p.rsz)) fail(BMG_EINVAL, "galerkin_coarsen: layouts do not match");
  if (!(a.uniform && p.uniform && a.mr == p.mc))
    fail(BMG_EINVAL, "device galerkin_coarsen: uniform square block sizes required");
  Ctx* ctx = a.ctx;
  const int m = a.mr;
  // AP = A * P: row i pairs (A_ik, P_kJ), ascending k per output block
  Product ap = symbolic(
      a.nbr,
      [&](int i, auto&& emit) {
        for (int64_t q = a.h_row_ptr[i]; q < a.h_row_ptr[i + 1]; ++q) emit(a.h_col[q], q);
      },
      p.h_row_ptr, p.h_col);
  // P^T column index: coarse row I -> (fine row i, P block) ascending i
  std::vector<int64_t> pt_ptr(p.nbc + 1, 0);
  for (int64_t q = 0; q < p.nnzb; ++q) pt_ptr[p.h_col[q] + 1]++;
  for (int j = 0; j < p.nbc; ++j) pt_ptr[j + 1] += pt_ptr[j];
  std::vector<int64_t> pt_blk(p.nnzb), fillp(pt_ptr.begin(), pt_ptr.end() - 1);
  std::vector<int32_t> pt_row(p.nnzb);
  for (int i = 0; i < p.nbr; ++i)
    for (int64_t q = p.h_row_ptr[i]; q < p.h_row_ptr[i + 1]; ++q) {
      const int64_t t = fillp[p.h_col[q]]++;
      pt_row[t] = i;
      pt_blk[t] = q;
    }
  // C = P^T AP: coarse row I pairs (P_iI, AP_iJ), ascending i per output block
  Product c = symbolic(
      p.nbc,
      [&](int I, auto&& emit) {
        for (int64_t t = pt_ptr[I]; t < pt_ptr[I + 1]; ++t) emit(pt_row[t], pt_blk[t]);
      },
      ap.row_ptr, ap.col);
  // numeric
  const int bs = a.bs;
  DBuf<double> apv(std::max<size_t>(ap.col.size() * bs, 2));
  pair_gemm(ctx, a.vals.p, bs, p.vals.p, p.bs, ap, apv.p, bs, m, false);
  DBuf<double> cv(std::max<size_t>(c.col.size() * bs, 2));
  pair_gemm(ctx, p.vals.p, p.bs, apv.p, bs, c, cv.p, bs, m, true);
  apv.release();
  // structural symmetry + transpose positions
  const int nc = p.nbc;
  std::vector<int64_t> tpos(c.col.size(), -1);
  for (int I = 0; I < nc; ++I)
    for (int64_t q = c.row_ptr[I]; q < c.row_ptr[I + 1]; ++q) {
      const int J = c.col[q];
      const auto b = c.col.begin() + c.row_ptr[J], e = c.col.begin() + c.row_ptr[J + 1];
      auto it = std::lower_bound(b, e, I);
      if (it == e || *it != I) fail(BMG_ERUNTIME, "galerkin_coarsen: P^T A P is not structurally symmetric");
      tpos[q] = it - c.col.begin();
    }
  std::vector<int> csz(nc, m);
  auto out = make_bsr_structure(ctx, nc, csz.data(), nc, csz.data(), c.row_ptr, c.col, true);
  DBuf<int64_t> dt(std::max<size_t>(tpos.size(), 1));
  if (!tpos.empty()) BMG_CUDA(cudaMemcpy(dt.p, tpos.data(), tpos.size() * 8, cudaMemcpyHostToDevice));
  const int64_t nblk = (int64_t)c.col.size();
  if (nblk) {
    const int threads = ((m * m + 31) / 32) * 32;
    kern::symmetrize_kernel<<<(int)std::min<int64_t>(nblk, (int64_t)ctx->sms * 32), threads, 0, ctx->stream>>>(
        cv.p, dt.p, out->vals.p, nblk, m, bs);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  return out;
}

// ============================================================================ tridiagonal QL
// Eigenvalues of a symmetric tridiagonal matrix by implicit QL with Wilkinson
// shifts (replaces Eigen::SelfAdjointEigenSolver::computeFromTridiagonal,
// lanczos.hpp:44-45).  Returned ascending.
std::vector<double> tridiag_eigenvalues(std::vector<double> d, std::vector<double> e) {
  const int n = (int)d.size();
  e.resize(n, 0.0);
  if (n > 0) e[n - 1] = 0.0;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = std::fabs(d[m]) + std::fabs(d[m + 1]);
        if (std::fabs(e[m]) <= 2.220446049250313e-16 * dd) break;
      }
      if (m != l) {
        if (++iter > 200) fail(BMG_ERUNTIME, "tridiagonal eigensolver did not converge");
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = std::hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = std::hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            underflow = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
        }
        if (underflow) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  std::sort(d.begin(), d.end());
  return d;
}

// ============================================================================ Lanczos
// lanczos_ritz_values (lanczos.hpp:16-47) on G A G^T (= apply_transformed,
// fsai.cpp:219-241), seeded start vector, no reorthogonalisation.
static void apply_transformed(const Fsai& m, const Bsr& a, const double* x, double* y, double* t1, double* t2) {
  // y = fwd_last ... fwd_0 A bwd_0^T... : bwd holds transposes in forward order
  const double* cur = x;
  double* bufs[2] = {t1, t2};
  int w = 0;
  for (size_t i = m.bwd.size(); i-- > 0;) {
    spmv(*m.bwd[i], cur, bufs[w]);
    cur = bufs[w];
    w ^= 1;
  }
  spmv(a, cur, bufs[w]);
  cur = bufs[w];
  w ^= 1;
  for (size_t i = 0; i < m.fwd.size(); ++i) {
    double* out = (i + 1 == m.fwd.size()) ? y : bufs[w];
    spmv(*m.fwd[i], cur, out);
    cur = out;
    w ^= 1;
  }
}

double lanczos_lambda_max(const Bsr& a, const Fsai& m, int iters, double safety, uint64_t seed) {
  Ctx* ctx = a.ctx;
  const int64_t n = a.dim_r;
  if (n < 1) fail(BMG_EINVAL, "lanczos: operator dimension must be >= 1");
  iters = (int)std::min<int64_t>(iters, n);
  DBuf<double> v(n), vp(n), w(n), t1(n), t2(n);
  kern::rng_symmetric_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(v.p, n, seed);
  ctx->count();
  const double nv = std::sqrt(dot(ctx, v.p, v.p, n));
  kern::scale_div_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(v.p, n, nv);
  ctx->count();
  fill(ctx, vp.p, n, 0.0);
  std::vector<double> diag, off;
  double beta = 0.0;
  for (int j = 0; j < iters; ++j) {
    apply_transformed(m, a, v.p, w.p, t1.p, t2.p);
    const double alpha = dot(ctx, v.p, w.p, n);
    diag.push_back(alpha);
    kern::lanczos_update_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(w.p, v.p, vp.p, n, alpha, beta);
    ctx->count();
    beta = std::sqrt(dot(ctx, w.p, w.p, n));
    if (j + 1 == iters) break;
    if (beta <= 1e-14 * std::fabs(alpha) || beta == 0.0) break;
    off.push_back(beta);
    std::swap(v.p, vp.p);  // v_prev = v
    copy(ctx, v.p, w.p, n);
    kern::scale_div_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(v.p, n, beta);
    ctx->count();
  }
  BMG_CUDA(cudaGetLastError());
  off.resize(diag.empty() ? 0 : diag.size() - 1);
  const auto ev = tridiag_eigenvalues(diag, off);
  return safety * ev.back();
}

// ============================================================================ hierarchy
struct Level {
  const Bsr* A = nullptr;
  const Bsr* P = nullptr;  // prolongation from level-1 (unset at 0)
  const Bsr* R = nullptr;  // P^T
  const Fsai* M = nullptr;
  double beta = 1.0;
  std::unique_ptr<Bsr> A_own, P_own, R_own;
  std::unique_ptr<Fsai> M_own;
  DBuf<double> b, x, r, w, p, t;
  int64_t n = 0;
};

struct GraphKey {
  int kpre, kpost;
  const double* b;
  double* x;
  bool operator<(const GraphKey& o) const { return std::tie(kpre, kpost, b, x) < std::tie(o.kpre, o.kpost, o.b, o.x); }
};

struct Hier {
  Ctx* ctx = nullptr;
  std::vector<Level> lv;  // 0 = coarsest
  DBuf<double> ainv;      // dense A_0^{-1}
  int64_t n0 = 0;
  bool use_graph = true;
  struct Captured {
    cudaGraphExec_t exec;
    int64_t kernels;
  };
  std::map<GraphKey, Captured> graphs;
  DBuf<double> io_b, io_x;  // e2e staging
  ~Hier() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
  }
  int finest() const { return (int)lv.size() - 1; }
};

static void alloc_level_vectors(Level& L, bool finest) {
  L.n = L.A->dim_r;
  if (!finest) {
    L.b.alloc(L.n);
    L.x.alloc(L.n);
  }
  L.r.alloc(L.n);
  L.w.alloc(L.n);
  L.p.alloc(L.n);
  L.t.alloc(L.n);
}

static void coarse_factor(Hier& h) {
  Ctx* ctx = h.ctx;
  const Bsr& a0 = *h.lv[0].A;
  if (!(a0.uniform && a0.mr == a0.mc)) fail(BMG_EINVAL, "coarse solve: uniform block sizes required");
  const int64_t N = a0.dim_r;
  h.n0 = N;
  h.ainv.alloc(std::max<int64_t>(N * N, 1));
  BMG_CUDA(cudaMemsetAsync(h.ainv.p, 0, h.ainv.bytes(), ctx->stream));
  kern::bsr_to_dense_kernel<<<std::max(1, std::min(a0.nbr, ctx->sms * 8)), 128, 0, ctx->stream>>>(
      a0.vals.p, a0.row_ptr.p, a0.col.p, a0.nbr, a0.mr, a0.bs, h.ainv.p, N);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  cusolverDnHandle_t s = ctx->cusolver();
  int lwork = 0, lwork2 = 0;
  if (cusolverDnDpotrf_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)N, h.ainv.p, (int)N, &lwork) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotrf_bufferSize failed");
  if (cusolverDnDpotri_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)N, h.ainv.p, (int)N, &lwork2) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotri_bufferSize failed");
  DBuf<double> work(std::max(std::max(lwork, lwork2), 1));
  DBuf<int> info(1);
  if (cusolverDnDpotrf(s, CUBLAS_FILL_MODE_LOWER, (int)N, h.ainv.p, (int)N, work.p, lwork, info.p) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotrf failed");
  int hinfo = 0;
  BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) fail(BMG_ERUNTIME, "setup: coarsest operator is not positive definite");
  if (cusolverDnDpotri(s, CUBLAS_FILL_MODE_LOWER, (int)N, h.ainv.p, (int)N, work.p, lwork2, info.p) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotri failed");
  BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) fail(BMG_ERUNTIME, "setup: coarse inverse failed");
  kern::symmetrize_dense_kernel<<<grid1d(N * N), 256, 0, ctx->stream>>>(h.ainv.p, N);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
}

static void finish_hier(Hier& h, int cap) {
  const int64_t n0 = h.lv[0].A->dim_r;
  if (n0 > cap) fail(BMG_EINVAL, "setup: coarsest level exceeds the dense-solve cap");
  for (int l = 0; l <= h.finest(); ++l) alloc_level_vectors(h.lv[l], l == h.finest());
  coarse_factor(h);
}

// one fourth-kind smoothing application (chebyshev.hpp:48-69) on level l
static void smooth(Level& L, int k, const double* b, double* x, bool xzero) {
  if (k < 1) return;
  const double d = 4.0 / L.beta;
  const Fsai& M = *L.M;
  for (int s = 1; s <= k; ++s) {
    const double* rsrc;
    if (s == 1 && xzero) {
      rsrc = b;  // A * 0 = 0: r = b exactly
    } else {
      residual(*L.A, b, x, L.r.p);
      rsrc = L.r.p;
    }
    // forward chain: w = F_n ... F_0 r  (nest = 0: w = G r)
    const double* cur = rsrc;
    double* bufs[2] = {L.w.p, L.t.p};
    int wsel = 0;
    for (const auto& f : M.fwd) {
      spmv(*f, cur, bufs[wsel]);
      cur = bufs[wsel];
      wsel ^= 1;
    }
    for (size_t i = M.bwd.size(); i-- > 1;) {
      spmv(*M.bwd[i], cur, bufs[wsel]);
      cur = bufs[wsel];
      wsel ^= 1;
    }
    if (s == 1) {
      const double dmu = d * ((2.0 * 0 + 1.0) / (2.0 * 0 + 3.0));
      gt_cheb(*M.bwd[0], cur, L.p.p, x, 0.0, dmu, true, xzero);
    } else {
      const double mu_prev = (2.0 * (s - 2) + 1.0) / (2.0 * (s - 2) + 3.0);
      const double mu = (2.0 * (s - 1) + 1.0) / (2.0 * (s - 1) + 3.0);
      gt_cheb(*M.bwd[0], cur, L.p.p, x, mu_prev * mu_prev, d * mu, false, false);
    }
  }
}

// v_cycle (multilevel.cpp:77-103), recursion unrolled: down, coarse solve, up
static void enqueue_vcycle(Hier& h, int kpre, int kpost, const double* bf, double* xf) {
  Ctx* ctx = h.ctx;
  const int top = h.finest();
  std::vector<const double*> B(top + 1);
  std::vector<double*> X(top + 1);
  for (int l = 0; l <= top; ++l) {
    B[l] = l == top ? bf : h.lv[l].b.p;
    X[l] = l == top ? xf : h.lv[l].x.p;
  }
  for (int l = top; l >= 1; --l) {
    Level& L = h.lv[l];
    const bool xzero = l < top;
    const double* r;
    if (kpre > 0) {
      smooth(L, kpre, B[l], X[l], xzero);
      residual(*L.A, B[l], X[l], L.r.p);
      r = L.r.p;
    } else if (xzero) {
      fill(ctx, X[l], L.n, 0.0);
      r = B[l];
    } else {
      residual(*L.A, B[l], X[l], L.r.p);
      r = L.r.p;
    }
    spmv(*L.R, r, h.lv[l - 1].b.p);  // rc = P^T r
  }
  {
    const int64_t N = h.n0;
    kern::gemv_kernel<<<(int)((N * 32 + 255) / 256), 256, 0, ctx->stream>>>(h.ainv.p, B[0], X[0], N);
    ctx->count();
    BMG_LAUNCHED(ctx->stream, "gemv_kernel");
  }
  for (int l = 1; l <= top; ++l) {
    Level& L = h.lv[l];
    prolong_add(*L.P, X[l - 1], X[l]);  // x += P ec
    smooth(L, kpost, B[l], X[l], false);
  }
}

static void run_vcycle(Hier& h, int kpre, int kpost, const double* bf, double* xf) {
  if (kpre + kpost < 1) fail(BMG_EINVAL, "v_cycle: cycle needs at least one smoothing step");
  Ctx* ctx = h.ctx;
  if (!h.use_graph || h.finest() == 0) {
    if (h.finest() == 0) {
      const int64_t N = h.n0;
      kern::gemv_kernel<<<(int)((N * 32 + 255) / 256), 256, 0, ctx->stream>>>(h.ainv.p, bf, xf, N);
      ctx->count();
      BMG_CUDA(cudaGetLastError());
      return;
    }
    enqueue_vcycle(h, kpre, kpost, bf, xf);
    return;
  }
  GraphKey key{kpre, kpost, bf, xf};
  auto it = h.graphs.find(key);
  if (it == h.graphs.end()) {
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->own;
    const int64_t before = ctx->launches;
    BMG_CUDA(cudaStreamBeginCapture(ctx->own, cudaStreamCaptureModeThreadLocal));
    try {
      enqueue_vcycle(h, kpre, kpost, bf, xf);
    } catch (...) {
      cudaGraph_t g;
      cudaStreamEndCapture(ctx->own, &g);
      if (g) cudaGraphDestroy(g);
      ctx->stream = user;
      throw;
    }
    cudaGraph_t g;
    BMG_CUDA(cudaStreamEndCapture(ctx->own, &g));
    ctx->stream = user;
    cudaGraphExec_t ex;
    BMG_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    it = h.graphs.emplace(key, Hier::Captured{ex, ctx->launches - before}).first;
    ctx->launches = before;
  }
  BMG_CUDA(cudaGraphLaunch(it->second.exec, ctx->stream));
  ctx->launches += it->second.kernels;
}

}  // namespace bmg

// ============================================================================ C ABI
using namespace bmg;

namespace {
const Bsr* B(const bmg_bsr* a) { return reinterpret_cast<const Bsr*>(a); }
const Vec* V(const bmg_vec* v) { return reinterpret_cast<const Vec*>(v); }
Vec* V(bmg_vec* v) { return reinterpret_cast<Vec*>(v); }
const Fsai* M(const bmg_fsai* m) { return reinterpret_cast<const Fsai*>(m); }
void need_len(const Vec* v, int64_t n, const char* what) {
  if (v->n != n) fail(BMG_EINVAL, std::string(what) + ": vector length does not match layout");
}
}  // namespace

extern "C" {

void bmg_setup_params_default(bmg_setup_params* p) {
  p->t_max = 4;
  p->tau = 1.0;
  p->nest = 0;
  p->fsai_kind = BMG_FSAI_ADAPTIVE;
  p->lanczos_iters = 100;
  p->lanczos_safety = 1.01;
  p->seed = 42;
  p->coarse_dim_cap = 5000;
}

int bmg_galerkin(const bmg_bsr* a, const bmg_bsr* p, bmg_bsr** out) {
  return guard([&] {
    B(a)->ctx->activate();
    *out = reinterpret_cast<bmg_bsr*>(galerkin(*B(a), *B(p)).release());
  });
}

int bmg_fsai_build(const bmg_bsr* a, int kind, int t_max, double tau, int nest, bmg_fsai** out) {
  return guard([&] {
    B(a)->ctx->activate();
    *out = reinterpret_cast<bmg_fsai*>(fsai_build(*B(a), kind, t_max, tau, nest).release());
  });
}
int bmg_fsai_from_factors(bmg_ctx* ctx, const bmg_bsr* F, const double* shat, bmg_fsai** out) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->activate();
    *out = reinterpret_cast<bmg_fsai*>(fsai_from_factors(c, *B(F), shat).release());
  });
}
int bmg_fsai_destroy(bmg_fsai* m) {
  return guard([&] {
    Fsai* f = reinterpret_cast<Fsai*>(m);
    if (f) BMG_CUDA(cudaStreamSynchronize(f->ctx->stream));
    delete f;
  });
}
int bmg_fsai_apply(const bmg_fsai* mh, const bmg_vec* r, bmg_vec* z) {
  return guard([&] {
    const Fsai* m = M(mh);
    need_len(V(r), m->dim, "fsai apply");
    need_len(V(z), m->dim, "fsai apply");
    DBuf<double> t1(std::max(m->dim, 1)), t2(std::max(m->dim, 1));
    fsai_apply(*m, V(r)->d.p, V(z)->d.p, t1.p, t2.p);
    BMG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  });
}
int bmg_fsai_apply_transformed(const bmg_fsai* mh, const bmg_bsr* a, const bmg_vec* x, bmg_vec* y) {
  return guard([&] {
    const Fsai* m = M(mh);
    need_len(V(x), m->dim, "apply_transformed");
    need_len(V(y), m->dim, "apply_transformed");
    DBuf<double> t1(std::max(m->dim, 1)), t2(std::max(m->dim, 1));
    apply_transformed(*m, *B(a), V(x)->d.p, V(y)->d.p, t1.p, t2.p);
    BMG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  });
}
int bmg_fsai_G(const bmg_fsai* m, const bmg_bsr** g) {
  return guard([&] { *g = reinterpret_cast<const bmg_bsr*>(&M(m)->G()); });
}

// cheb_fourth_apply (chebyshev.hpp:48-69) on the device
int bmg_cheb4_apply(const bmg_bsr* ah, const bmg_fsai* mh, const bmg_vec* b, bmg_vec* x, double beta, int k) {
  return guard([&] {
    if (!(beta > 0.0)) fail(BMG_EINVAL, "cheb_fourth_apply: beta must be positive");
    if (k < 1) fail(BMG_EINVAL, "cheb_fourth_apply: degree must be >= 1");
    const Bsr* a = B(ah);
    need_len(V(b), a->dim_r, "cheb_fourth_apply");
    need_len(V(x), a->dim_r, "cheb_fourth_apply");
    Level L;
    L.A = a;
    L.M = M(mh);
    L.beta = beta;
    L.n = a->dim_r;
    L.r.alloc(std::max<int64_t>(L.n, 1));
    L.w.alloc(std::max<int64_t>(L.n, 1));
    L.p.alloc(std::max<int64_t>(L.n, 1));
    L.t.alloc(std::max<int64_t>(L.n, 1));
    smooth(L, k, V(b)->d.p, V(x)->d.p, false);
    BMG_CUDA(cudaStreamSynchronize(a->ctx->stream));
  });
}

int bmg_lanczos_lambda_max(const bmg_bsr* a, const bmg_fsai* m, int iters, double safety, uint64_t seed,
                           double* beta) {
  return guard([&] {
    B(a)->ctx->activate();
    *beta = lanczos_lambda_max(*B(a), *M(m), iters, safety, seed);
  });
}

// setup (multilevel.cpp:36-75) with every step on the device
int bmg_hier_setup(const bmg_bsr* a_finest, int ntransfers, const bmg_bsr* const* transfers,
                   const bmg_setup_params* params, bmg_hier** out) {
  return guard([&] {
    bmg_setup_params prm;
    if (params)
      prm = *params;
    else
      bmg_setup_params_default(&prm);
    const Bsr* af = B(a_finest);
    Ctx* ctx = af->ctx;
    ctx->activate();
    if (ntransfers < 0) fail(BMG_EINVAL, "setup: negative transfer count");
    auto h = std::make_unique<Hier>();
    h->ctx = ctx;
    const int depth = ntransfers;
    h->lv.resize(depth + 1);
    h->lv[depth].A = af;
    for (int l = depth; l >= 1; --l) {
      Level& L = h->lv[l];
      L.P = B(transfers[l - 1]);
      L.R_own = bsr_transpose(*L.P);
      L.R = L.R_own.get();
      h->lv[l - 1].A_own = galerkin(*L.A, *L.P);
      h->lv[l - 1].A = h->lv[l - 1].A_own.get();
    }
    for (int l = 1; l <= depth; ++l) {
      Level& L = h->lv[l];
      L.M_own = fsai_build(*L.A, prm.fsai_kind, prm.t_max, prm.tau, prm.nest);
      L.M = L.M_own.get();
      L.beta = lanczos_lambda_max(*L.A, *L.M, prm.lanczos_iters, prm.lanczos_safety, prm.seed);
    }
    finish_hier(*h, prm.coarse_dim_cap);
    *out = reinterpret_cast<bmg_hier*>(h.release());
  });
}

int bmg_hier_create(bmg_ctx* ctx, int nlevels, const bmg_bsr* const* A, const bmg_bsr* const* P,
                    const bmg_fsai* const* Mh, const double* beta, int coarse_dim_cap, bmg_hier** out) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->activate();
    if (nlevels < 1) fail(BMG_EINVAL, "hierarchy needs at least one level");
    auto h = std::make_unique<Hier>();
    h->ctx = c;
    h->lv.resize(nlevels);
    for (int l = 0; l < nlevels; ++l) {
      Level& L = h->lv[l];
      L.A = B(A[l]);
      if (l >= 1) {
        L.P = B(P[l]);
        if (L.P->dim_r != L.A->dim_r || L.P->dim_c != B(A[l - 1])->dim_r)
          fail(BMG_EINVAL, "hierarchy: prolongation shape does not match the levels");
        L.R_own = bsr_transpose(*L.P);
        L.R = L.R_own.get();
        L.M = M(Mh[l]);
        L.beta = beta[l];
        if (!(L.beta > 0.0)) fail(BMG_EINVAL, "cheb_fourth_apply: beta must be positive");
      }
    }
    finish_hier(*h, coarse_dim_cap);
    *out = reinterpret_cast<bmg_hier*>(h.release());
  });
}

int bmg_hier_destroy(bmg_hier* h) {
  return guard([&] {
    Hier* p = reinterpret_cast<Hier*>(h);
    if (p) BMG_CUDA(cudaStreamSynchronize(p->ctx->stream));
    delete p;
  });
}
int bmg_hier_info(const bmg_hier* hh, int* nlevels, int64_t* device_bytes) {
  return guard([&] {
    const Hier* h = reinterpret_cast<const Hier*>(hh);
    if (nlevels) *nlevels = (int)h->lv.size();
    if (device_bytes) {
      int64_t b = (int64_t)h->ainv.bytes();
      for (const auto& L : h->lv) {
        if (L.A_own) b += L.A_own->device_bytes();
        if (L.R_own) b += L.R_own->device_bytes();
        if (L.M_own)
          for (auto& f : L.M_own->fwd) b += f->device_bytes();
        if (L.M_own)
          for (auto& f : L.M_own->bwd) b += f->device_bytes();
        b += (int64_t)(L.b.bytes() + L.x.bytes() + L.r.bytes() + L.w.bytes() + L.p.bytes() + L.t.bytes());
      }
      *device_bytes = b;
    }
  });
}
int bmg_hier_beta(const bmg_hier* hh, int level, double* beta) {
  return guard([&] {
    const Hier* h = reinterpret_cast<const Hier*>(hh);
    if (level < 1 || level > h->finest()) fail(BMG_ERANGE, "hierarchy: level out of range");
    *beta = h->lv[level].beta;
  });
}
int bmg_hier_level(const bmg_hier* hh, int level, const bmg_bsr** a, const bmg_bsr** p, const bmg_fsai** m) {
  return guard([&] {
    const Hier* h = reinterpret_cast<const Hier*>(hh);
    if (level < 0 || level > h->finest()) fail(BMG_ERANGE, "hierarchy: level out of range");
    const Level& L = h->lv[level];
    if (a) *a = reinterpret_cast<const bmg_bsr*>(L.A);
    if (p) *p = reinterpret_cast<const bmg_bsr*>(L.P);
    if (m) *m = reinterpret_cast<const bmg_fsai*>(L.M);
  });
}

// algorithmic HBM bytes of one V(k_pre, k_post) cycle (BASELINE.md §3 byte
// model, with the exact A*0 skip on coarse levels)
int bmg_hier_cycle_bytes(const bmg_hier* hh, int kpre, int kpost, int64_t* bytes) {
  return guard([&] {
    const Hier* h = reinterpret_cast<const Hier*>(hh);
    int64_t tot = 0;
    const int top = h->finest();
    for (int l = 1; l <= top; ++l) {
      const Level& L = h->lv[l];
      const int64_t n = L.n, nc = h->lv[l - 1].A->dim_r;
      int64_t gb = 0;
      for (auto& f : L.M->fwd) gb += f->pass_bytes();
      for (auto& f : L.M->bwd) gb += f->pass_bytes();
      const int64_t apass = L.A->pass_bytes() + 24 * n;  // x, b read; r write
      const int64_t gvec = 16 * n + 40 * n;              // G: r, w; G^T+cheb: w, p rw, x rw
      const int steps = kpre + kpost;
      int64_t lvl = steps * (apass + gb + gvec);
      if (l < top && kpre > 0) lvl -= apass;  // first coarse pre-step: A*0 skipped
      if (l < top && kpre > 0) lvl -= 8 * n;  // and x not read in that step
      lvl += apass;                                        // residual before restriction
      lvl += L.R->pass_bytes() + 8 * n + 8 * nc;           // restriction
      lvl += L.P->pass_bytes() + 8 * nc + 16 * n;          // prolongation x += P e
      tot += lvl;
    }
    tot += h->n0 * h->n0 * 8 + 16 * h->n0;  // dense coarse solve
    *bytes = tot;
  });
}

int bmg_hier_use_graph(bmg_hier* hh, int on) {
  return guard([&] { reinterpret_cast<Hier*>(hh)->use_graph = on != 0; });
}

int bmg_vcycle(bmg_hier* hh, int kpre, int kpost, const bmg_vec* b, bmg_vec* x) {
  return guard([&] {
    Hier* h = reinterpret_cast<Hier*>(hh);
    const int64_t n = h->lv.back().A->dim_r;
    need_len(V(b), n, "v_cycle");
    need_len(V(x), n, "v_cycle");
    run_vcycle(*h, kpre, kpost, V(b)->d.p, V(x)->d.p);
  });
}

int bmg_vcycle_host(bmg_hier* hh, int kpre, int kpost, const double* b, double* x) {
  return guard([&] {
    Hier* h = reinterpret_cast<Hier*>(hh);
    Ctx* ctx = h->ctx;
    const int64_t n = h->lv.back().A->dim_r;
    if (h->io_b.n < (size_t)n) {
      h->io_b.alloc(std::max<int64_t>(n, 1));
      h->io_x.alloc(std::max<int64_t>(n, 1));
    }
    BMG_CUDA(cudaMemcpyAsync(h->io_b.p, b, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    BMG_CUDA(cudaMemcpyAsync(h->io_x.p, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    run_vcycle(*h, kpre, kpost, h->io_b.p, h->io_x.p);
    BMG_CUDA(cudaMemcpyAsync(x, h->io_x.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// residual-history driver modelled on measure_rates (experiments.cpp:15-67)
int bmg_solve(bmg_hier* hh, int kpre, int kpost, const bmg_vec* bh, bmg_vec* xh, double tol, int max_iter,
              double* hist, int* iters, int* status) {
  return guard([&] {
    Hier* h = reinterpret_cast<Hier*>(hh);
    Ctx* ctx = h->ctx;
    Level& F = h->lv.back();
    const int64_t n = F.A->dim_r;
    need_len(V(bh), n, "solve");
    need_len(V(xh), n, "solve");
    const double* b = V(bh)->d.p;
    double* x = V(xh)->d.p;
    auto resid = [&]() {
      residual(*F.A, b, x, F.r.p);
      return std::sqrt(dot(ctx, F.r.p, F.r.p, n));
    };
    hist[0] = resid();
    int it = 0, st = 1;
    if (hist[0] == 0.0) st = 0;
    while (st == 1 && it < max_iter) {
      run_vcycle(*h, kpre, kpost, b, x);
      ++it;
      hist[it] = resid();
      const double growth = hist[it] / std::max(hist[it - 1], 1e-300);
      if (!std::isfinite(hist[it]) || growth > 1e6) {
        st = 2;
        break;
      }
      if (hist[it] / hist[0] < tol) st = 0;
    }
    *iters = it;
    *status = st;
  });
}

int bmg_tridiag_eigs(int n, const double* d, const double* e, double* out) {
  return guard([&] {
    auto ev = tridiag_eigenvalues(std::vector<double>(d, d + n),
                                  std::vector<double>(e, e + (n > 0 ? n - 1 : 0)));
    std::copy(ev.begin(), ev.end(), out);
  });
}

}  // extern "C"
