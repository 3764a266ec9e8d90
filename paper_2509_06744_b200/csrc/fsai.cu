// fsai.cu -- batched block-FSAI setup on the device and the G / G^T apply.
//
// The reference keeps F (unit-diagonal lower) and per-row Cholesky factors of
// S = diag(F A F^T) and applies M = F^T S^{-1} F (fsai.cpp:60-70, 200-217).  The
// device path folds the per-row solves into G = L^{-1} F at setup
// (M = F^T L^{-T} L^{-1} F = G^T G), so the apply is two streaming
// passes: w = G r and z = G^T w (G^T stored as its own BSR, no atomics).
//
// Setup kernels (one CTA per block row, small dense work in shared memory):
//   fsai_select_kernel   adaptive_build with P0 = diagonal, t_max = 1
//                        (fsai.cpp:132-198, delta_ratio fsai.cpp:106-130):
//                        scores every lower candidate c of H row k = A row k and
//                        picks argmin rho (ties -> smallest c).
//   fsai_row_kernel      build_row (fsai.cpp:18-43) for an explicit lower
//                        pattern, then G row k = L_k^{-1} [F_kS, I].
// Dense arithmetic follows the oracle's fixed order (fma chains ascending), so
// G is bitwise equal to the oracle's L^{-1} F for the same pattern.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

#include "bmg_abi.h"
#include "bmg_internal.h"

namespace bmg {
namespace kern {

constexpr int kFsaiThreads = 64;

struct FsaiErr {
  int row;    // -1 = ok
  int pivot;
  int what;   // 1 principal submatrix, 2 S row, 3 W_c
  int cand;
};

// In-place Cholesky of an n x n row-major matrix in shared memory (lower = L,
// upper zeroed); same operation order as small_cholesky.cpp:12-28 restated in
// the oracle.  Returns the failing pivot or -1; logdet accumulated by thread 0.
__device__ int cta_chol(double* a, int n, double* logdet) {
  __shared__ int s_piv;
  __shared__ double s_ljj;
  if (threadIdx.x == 0) {
    s_piv = -1;
    if (logdet) *logdet = 0.0;
  }
  for (int j = 0; j < n; ++j) {
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (int k = 0; k < j; ++k) s = __fma_rn(a[j * n + k], a[j * n + k], s);
      const double d = __dsub_rn(a[j * n + j], s);
      if (!(d > 0.0)) {
        s_piv = j;
      } else {
        const double l = sqrt(d);
        a[j * n + j] = l;
        s_ljj = l;
        if (logdet) *logdet = __dadd_rn(*logdet, __dmul_rn(2.0, log(l)));
      }
    }
    __syncthreads();
    if (s_piv >= 0) return s_piv;
    const double ljj = s_ljj;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double t = 0.0;
      for (int k = 0; k < j; ++k) t = __fma_rn(a[i * n + k], a[j * n + k], t);
      a[i * n + j] = __ddiv_rn(__dsub_rn(a[i * n + j], t), ljj);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, k = e - i * n;
    if (k > i) a[e] = 0.0;
  }
  __syncthreads();
  return -1;
}

// x (n x c, row-major) <- L^{-1} x, column-parallel (Chol::solve_l order)
__device__ void cta_solve_l(const double* l, int n, double* x, int c) {
  for (int col = threadIdx.x; col < c; col += blockDim.x)
    for (int i = 0; i < n; ++i) {
      double t = 0.0;
      for (int k = 0; k < i; ++k) t = __fma_rn(l[i * n + k], x[k * c + col], t);
      x[i * c + col] = __ddiv_rn(__dsub_rn(x[i * c + col], t), l[i * n + i]);
    }
  __syncthreads();
}
// x <- L^{-T} x (Chol::solve_lt order)
__device__ void cta_solve_lt(const double* l, int n, double* x, int c) {
  for (int col = threadIdx.x; col < c; col += blockDim.x)
    for (int i = n - 1; i >= 0; --i) {
      double t = 0.0;
      for (int k = i + 1; k < n; ++k) t = __fma_rn(l[k * n + i], x[k * c + col], t);
      x[i * c + col] = __ddiv_rn(__dsub_rn(x[i * c + col], t), l[i * n + i]);
    }
  __syncthreads();
}
// x <- S^{-1} x = L^{-T} L^{-1} x, column by column (Chol::solve_mat)
__device__ void cta_solve(const double* l, int n, double* x, int c) {
  for (int col = threadIdx.x; col < c; col += blockDim.x) {
    for (int i = 0; i < n; ++i) {
      double t = 0.0;
      for (int k = 0; k < i; ++k) t = __fma_rn(l[i * n + k], x[k * c + col], t);
      x[i * c + col] = __ddiv_rn(__dsub_rn(x[i * c + col], t), l[i * n + i]);
    }
    for (int i = n - 1; i >= 0; --i) {
      double t = 0.0;
      for (int k = i + 1; k < n; ++k) t = __fma_rn(l[k * n + i], x[k * c + col], t);
      x[i * c + col] = __ddiv_rn(__dsub_rn(x[i * c + col], t), l[i * n + i]);
    }
  }
  __syncthreads();
}

__device__ void cta_load_block(double* dst, const double* src, int n) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
  __syncthreads();
}

__device__ double frob_serial(const double* b, int n) {
  double s = 0.0;
  for (int e = 0; e < n; ++e) s = __dadd_rn(s, __dmul_rn(b[e], b[e]));
  return sqrt(s);
}

__device__ int find_col(const int32_t* col, int64_t lo, int64_t hi, int j) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (int)lo;
}

struct MatView {
  const double* vals;
  const int32_t* col;
  const int64_t* row_ptr;
  const int64_t* voff;
  const int* rsz;
  const int64_t* diag;  // position of block (i, i) in row i
};

// adaptive_build, P0 = diagonal, t_max = 1: candidate scoring per row
__global__ void __launch_bounds__(kFsaiThreads) fsai_select_kernel(MatView A, int n, int mmax,
                                                                   int* best, double* best_rho,
                                                                   FsaiErr* err) {
  extern __shared__ double sm[];
  const int mm = mmax * mmax;
  double* Lk = sm;
  double* W = Lk + mm;
  double* X = W + mm;
  double* U = X + mm;
  double* H = U + mm;
  __shared__ double s_ldw, s_ldu, s_thr, s_best_rho;
  __shared__ int s_best, s_skip, s_fail;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int mk = A.rsz[k];
    const int64_t pk = A.diag[k];
    cta_load_block(Lk, A.vals + A.voff[pk], mk * mk);
    if (threadIdx.x == 0) s_thr = 1e-12 * frob_serial(Lk, mk * mk);
    const int piv = cta_chol(Lk, mk, nullptr);
    if (piv >= 0) {
      if (threadIdx.x == 0) atomicCAS(&err->row, -1, k) == -1 ? (err->pivot = piv, err->what = 2) : 0;
      return;
    }
    if (threadIdx.x == 0) {
      s_best = -1;
      s_best_rho = 0.0;
    }
    __syncthreads();
    for (int64_t p = A.row_ptr[k]; p < A.row_ptr[k + 1]; ++p) {
      const int c = A.col[p];
      if (c >= k) break;
      const int mc = A.rsz[c];
      cta_load_block(H, A.vals + A.voff[p], mk * mc);
      if (threadIdx.x == 0) s_skip = frob_serial(H, mk * mc) <= s_thr;
      __syncthreads();
      if (s_skip) continue;
      // W = A_cc (pattern strict part is empty) and its Cholesky
      const double* acc = A.vals + A.voff[A.diag[c]];
      cta_load_block(W, acc, mc * mc);
      const int pw = cta_chol(W, mc, &s_ldw);
      if (pw >= 0) {
        if (threadIdx.x == 0) atomicCAS(&err->row, -1, k) == -1 ? (err->pivot = pw, err->what = 3, err->cand = c) : 0;
        return;
      }
      // X = S_k^{-1} H_kc ; U = W - H_kc^T X
      cta_load_block(X, H, mk * mc);
      cta_solve(Lk, mk, X, mc);
      for (int e = threadIdx.x; e < mc * mc; e += blockDim.x) {
        const int r = e / mc, q = e - r * mc;
        double t = 0.0;
        for (int z = 0; z < mk; ++z) t = __fma_rn(H[z * mc + r], X[z * mc + q], t);
        U[e] = __dsub_rn(acc[e], t);
      }
      __syncthreads();
      const int pu = cta_chol(U, mc, &s_ldu);
      if (threadIdx.x == 0) {
        if (pu >= 0) {
          s_ldu = 0.0;
          s_fail = 1;
        } else {
          s_fail = 0;
        }
        const double rho = s_fail ? 0.0 : fmin(exp(__dsub_rn(s_ldu, s_ldw)), 1.0);
        if (s_best < 0 || rho < s_best_rho) {
          s_best = c;
          s_best_rho = rho;
        }
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      best[k] = s_best;
      best_rho[k] = s_best_rho;
    }
    __syncthreads();
  }
}

// build_row (fsai.cpp:18-43) for the explicit strict lower pattern of row k,
// followed by G row k = L^{-1} [F_kS, I] written into G's value array.
struct RowArgs {
  MatView A;
  const int64_t* pat_ptr;  // strict pattern CSR
  const int32_t* pat_col;
  double* gvals;           // G values, row k's blocks at gvoff[g_row_ptr[k] + q]
  const int64_t* g_row_ptr;
  const int64_t* gvoff;
  int n;
  int mmax;
  int gmax;  // max strict pattern size in scalars
};

__global__ void __launch_bounds__(kFsaiThreads) fsai_row_kernel(RowArgs s, FsaiErr* err) {
  extern __shared__ double sm[];
  const int mm = s.mmax * s.mmax;
  double* gram = sm;                             // gmax^2
  double* X = gram + (size_t)s.gmax * s.gmax;    // gmax x mmax (A_kS^T, then solution)
  double* AKS = X + (size_t)s.gmax * s.mmax;     // mmax x gmax
  double* S = AKS + (size_t)s.gmax * s.mmax;     // mmax^2
  double* Y = S + mm;                            // mmax x max(gmax, mmax)
  const MatView& A = s.A;
  for (int k = blockIdx.x; k < s.n; k += gridDim.x) {
    const int mk = A.rsz[k];
    const int64_t p0 = s.pat_ptr[k], p1 = s.pat_ptr[k + 1];
    const int ns = (int)(p1 - p0);
    // scalar offsets of the strict pattern blocks
    int ng = 0;
    for (int64_t q = p0; q < p1; ++q) ng += A.rsz[s.pat_col[q]];
    // S_kk = A_kk
    cta_load_block(S, A.vals + A.voff[A.diag[k]], mk * mk);
    if (ns > 0) {
      // gram = A[S, S]
      for (int e = threadIdx.x; e < ng * ng; e += blockDim.x) gram[e] = 0.0;
      __syncthreads();
      int ro = 0;
      for (int64_t qa = p0; qa < p1; ++qa) {
        const int ia = s.pat_col[qa], ma = A.rsz[ia];
        int co = 0;
        for (int64_t qb = p0; qb < p1; ++qb) {
          const int ib = s.pat_col[qb], mb = A.rsz[ib];
          const int64_t lo = A.row_ptr[ia], hi = A.row_ptr[ia + 1];
          const int pos = find_col(A.col, lo, hi, ib);
          if (pos < hi && A.col[pos] == ib) {
            const double* blk = A.vals + A.voff[pos];
            for (int e = threadIdx.x; e < ma * mb; e += blockDim.x) {
              const int r = e / mb, c = e - r * mb;
              gram[(ro + r) * ng + co + c] = blk[e];
            }
          }
          co += mb;
        }
        ro += ma;
      }
      // A_kS (mk x ng) and X = A_kS^T
      int co = 0;
      for (int64_t q = p0; q < p1; ++q) {
        const int j = s.pat_col[q], mj = A.rsz[j];
        const int64_t lo = A.row_ptr[k], hi = A.row_ptr[k + 1];
        const int pos = find_col(A.col, lo, hi, j);
        const bool present = pos < hi && A.col[pos] == j;
        const double* blk = present ? A.vals + A.voff[pos] : nullptr;
        for (int e = threadIdx.x; e < mk * mj; e += blockDim.x) {
          const int r = e / mj, c = e - r * mj;
          const double v = present ? blk[e] : 0.0;
          AKS[r * ng + co + c] = v;
          X[(co + c) * mk + r] = v;
        }
        co += mj;
      }
      __syncthreads();
      const int pg = cta_chol(gram, ng, nullptr);
      if (pg >= 0) {
        if (threadIdx.x == 0) atomicCAS(&err->row, -1, k) == -1 ? (err->pivot = pg, err->what = 1) : 0;
        return;
      }
      cta_solve(gram, ng, X, mk);  // X = gram^{-1} A_kS^T  (ng x mk)
      // S_kk -= A_kS X
      for (int e = threadIdx.x; e < mk * mk; e += blockDim.x) {
        const int r = e / mk, c = e - r * mk;
        double t = 0.0;
        for (int q = 0; q < ng; ++q) t = __fma_rn(AKS[r * ng + q], X[q * mk + c], t);
        S[e] = __dsub_rn(S[e], t);
      }
      __syncthreads();
    }
    const int ps = cta_chol(S, mk, nullptr);
    if (ps >= 0) {
      if (threadIdx.x == 0) atomicCAS(&err->row, -1, k) == -1 ? (err->pivot = ps, err->what = 2) : 0;
      return;
    }
    // Y = [F_kS | I] (mk x (ng + mk)), F_kS = -X^T; then Y <- L^{-1} Y
    const int wy = ng + mk;
    for (int e = threadIdx.x; e < mk * wy; e += blockDim.x) {
      const int r = e / wy, c = e - r * wy;
      Y[e] = c < ng ? -X[c * mk + r] : (c - ng == r ? 1.0 : 0.0);
    }
    __syncthreads();
    cta_solve_l(S, mk, Y, wy);
    // scatter into G row k (blocks ascending: strict pattern, then diagonal)
    const int64_t g0 = s.g_row_ptr[k];
    int co = 0;
    for (int q = 0; q <= ns; ++q) {
      const int j = q < ns ? s.pat_col[p0 + q] : k;
      const int mj = A.rsz[j];
      double* dst = s.gvals + s.gvoff[g0 + q];
      for (int e = threadIdx.x; e < mk * mj; e += blockDim.x) {
        const int r = e / mj, c = e - r * mj;
        dst[e] = Y[r * wy + co + c];
      }
      co += mj;
    }
    __syncthreads();
  }
}

// G = L^{-1} F for injected factors: every block of F row k solved with L_k
__global__ void __launch_bounds__(kFsaiThreads) linv_rows_kernel(MatView F, const double* lpack,
                                                                 const int64_t* loff, double* gvals,
                                                                 int n, int mmax) {
  extern __shared__ double sm[];
  double* L = sm;
  double* Y = L + mmax * mmax;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int mk = F.rsz[k];
    cta_load_block(L, lpack + loff[k], mk * mk);
    for (int64_t p = F.row_ptr[k]; p < F.row_ptr[k + 1]; ++p) {
      const int j = F.col[p], mj = F.rsz[j];
      cta_load_block(Y, F.vals + F.voff[p], mk * mj);
      cta_solve_l(L, mk, Y, mj);
      double* dst = gvals + F.voff[p];
      for (int e = threadIdx.x; e < mk * mj; e += blockDim.x) dst[e] = Y[e];
      __syncthreads();
    }
  }
}

}  // namespace kern

// -------------------------------------------------------------------------- host
namespace {

struct Aux {  // per-block value offsets, sizes and diagonal positions on the device
  DBuf<int64_t> voff, diag;
  DBuf<int> rsz;
};

Aux make_aux(const Bsr& a, bool need_diag) {
  Aux x;
  x.voff.alloc(a.nnzb + 1);
  BMG_CUDA(cudaMemcpy(x.voff.p, a.h_voff.data(), (a.nnzb + 1) * 8, cudaMemcpyHostToDevice));
  x.rsz.alloc(std::max(a.nbr, 1));
  BMG_CUDA(cudaMemcpy(x.rsz.p, a.rsz.data(), a.nbr * 4, cudaMemcpyHostToDevice));
  if (need_diag) {
    std::vector<int64_t> d(a.nbr);
    for (int i = 0; i < a.nbr; ++i) {
      const auto b = a.h_col.begin() + a.h_row_ptr[i], e = a.h_col.begin() + a.h_row_ptr[i + 1];
      auto it = std::lower_bound(b, e, i);
      if (it == e || *it != i) fail(BMG_EINVAL, "fsai: missing diagonal block in row " + std::to_string(i));
      d[i] = it - a.h_col.begin();
    }
    x.diag.alloc(std::max(a.nbr, 1));
    BMG_CUDA(cudaMemcpy(x.diag.p, d.data(), a.nbr * 8, cudaMemcpyHostToDevice));
  }
  return x;
}

kern::MatView view(const Bsr& a, const Aux& x) {
  return kern::MatView{a.vals.p, a.col.p, a.row_ptr.p, x.voff.p, x.rsz.p, x.diag.p};
}

void check_err(Ctx* ctx, kern::FsaiErr* d_err) {
  kern::FsaiErr e;
  BMG_CUDA(cudaMemcpyAsync(&e, d_err, sizeof(e), cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (e.row < 0) return;
  std::string ctxs;
  if (e.what == 1) ctxs = "row " + std::to_string(e.row) + " principal submatrix";
  if (e.what == 2) ctxs = "S row " + std::to_string(e.row);
  if (e.what == 3) ctxs = "W_c for row " + std::to_string(e.row) + ", candidate " + std::to_string(e.cand);
  fail(BMG_ENOTSPD, "matrix not positive definite at pivot " + std::to_string(e.pivot) + " (" + ctxs + ")",
       e.pivot);
}

int max_size(const std::vector<int>& s) {
  int m = 1;
  for (int v : s) m = std::max(m, v);
  return m;
}

// build G for an explicit strict pattern; returns G (device) and G^T
std::unique_ptr<Fsai> build_from_pattern(const Bsr& a, const Aux& aux,
                                         const std::vector<int64_t>& pat_ptr,
                                         const std::vector<int32_t>& pat_col) {
  Ctx* ctx = a.ctx;
  const int n = a.nbr;
  // G structure: row k = strict pattern (ascending) + k
  std::vector<int64_t> grp(n + 1, 0);
  std::vector<int32_t> gcol;
  gcol.reserve(pat_col.size() + n);
  int gmax = 1;
  for (int k = 0; k < n; ++k) {
    int ng = 0;
    for (int64_t q = pat_ptr[k]; q < pat_ptr[k + 1]; ++q) {
      gcol.push_back(pat_col[q]);
      ng += a.rsz[pat_col[q]];
    }
    gcol.push_back(k);
    grp[k + 1] = (int64_t)gcol.size();
    gmax = std::max(gmax, ng);
  }
  auto G = make_bsr_structure(ctx, n, a.rsz.data(), n, a.rsz.data(), grp, gcol, false);
  const int mmax = max_size(a.rsz);
  const size_t smem = sizeof(double) * ((size_t)gmax * gmax + 2 * (size_t)gmax * mmax + (size_t)mmax * mmax +
                                        (size_t)mmax * (gmax + mmax));
  if (smem > 200 * 1024) fail(BMG_EINVAL, "fsai: row pattern too large for the device build");
  DBuf<int64_t> dpp(n + 1), dgv(G->nnzb + 1);
  DBuf<int32_t> dpc(std::max<size_t>(pat_col.size(), 1));
  BMG_CUDA(cudaMemcpy(dpp.p, pat_ptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  if (!pat_col.empty()) BMG_CUDA(cudaMemcpy(dpc.p, pat_col.data(), pat_col.size() * 4, cudaMemcpyHostToDevice));
  BMG_CUDA(cudaMemcpy(dgv.p, G->h_voff.data(), (G->nnzb + 1) * 8, cudaMemcpyHostToDevice));
  DBuf<kern::FsaiErr> derr(1);
  kern::FsaiErr e0{-1, -1, 0, -1};
  BMG_CUDA(cudaMemcpy(derr.p, &e0, sizeof(e0), cudaMemcpyHostToDevice));
  kern::RowArgs ra{view(a, aux), dpp.p, dpc.p, G->vals.p, G->row_ptr.p, dgv.p, n, mmax, gmax};
  BMG_CUDA(cudaFuncSetAttribute(kern::fsai_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::max(1, std::min(n, ctx->sms * 16));
  kern::fsai_row_kernel<<<grid, kern::kFsaiThreads, smem, ctx->stream>>>(ra, derr.p);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  check_err(ctx, derr.p);
  auto m = std::make_unique<Fsai>();
  m->ctx = ctx;
  m->dim = a.dim_r;
  auto GT = bsr_transpose(*G);
  m->fwd.push_back(std::move(G));
  m->bwd.push_back(std::move(GT));
  return m;
}

}  // namespace

std::unique_ptr<Fsai> fsai_build(const Bsr& a, int kind, int t_max, double tau, int nest) {
  if (!(a.rsz == a.csz)) fail(BMG_EINVAL, "fsai: matrix must be square");
  if (!a.sym) fail(BMG_EINVAL, "fsai: matrix must be symmetric");
  Ctx* ctx = a.ctx;
  const int n = a.nbr;
  Aux aux = make_aux(a, true);
  std::vector<int64_t> pp(n + 1, 0);
  std::vector<int32_t> pc;
  if (kind == BMG_FSAI_STATIC_LOWER) {
    for (int k = 0; k < n; ++k) {
      for (int64_t p = a.h_row_ptr[k]; p < a.h_row_ptr[k + 1]; ++p)
        if (a.h_col[p] < k) pc.push_back(a.h_col[p]);
      pp[k + 1] = (int64_t)pc.size();
    }
  } else if (kind == BMG_FSAI_DIAGONAL) {
    // pattern stays diagonal
  } else if (kind == BMG_FSAI_ADAPTIVE) {
    if (t_max < 1) fail(BMG_EINVAL, "adaptive_build: t_max must be >= 1");
    if (!(tau > 0.0 && tau <= 1.0)) fail(BMG_EINVAL, "adaptive_build: tau must be in (0, 1]");
    if (nest < 0) fail(BMG_EINVAL, "nested_build: n_levels must be >= 0");
    if (t_max != 1 || nest != 0)
      fail(BMG_EINVAL, "device FSAI build supports t_max = 1, nest = 0 (the BASELINE configs)");
    const int mmax = max_size(a.rsz);
    DBuf<int> best(std::max(n, 1));
    DBuf<double> rho(std::max(n, 1));
    DBuf<kern::FsaiErr> derr(1);
    kern::FsaiErr e0{-1, -1, 0, -1};
    BMG_CUDA(cudaMemcpy(derr.p, &e0, sizeof(e0), cudaMemcpyHostToDevice));
    const size_t smem = 5 * sizeof(double) * mmax * mmax;
    BMG_CUDA(cudaFuncSetAttribute(kern::fsai_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = std::max(1, std::min(n, ctx->sms * 16));
    kern::fsai_select_kernel<<<grid, kern::kFsaiThreads, smem, ctx->stream>>>(view(a, aux), n, mmax, best.p,
                                                                              rho.p, derr.p);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
    check_err(ctx, derr.p);
    std::vector<int> hb(n);
    std::vector<double> hr(n);
    if (n) {
      BMG_CUDA(cudaMemcpy(hb.data(), best.p, n * 4, cudaMemcpyDeviceToHost));
      BMG_CUDA(cudaMemcpy(hr.data(), rho.p, n * 8, cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < n; ++k) {
      if (hb[k] >= 0 && hr[k] < tau) pc.push_back(hb[k]);
      pp[k + 1] = (int64_t)pc.size();
    }
  } else {
    fail(BMG_EINVAL, "bmg_fsai_build: unknown kind");
  }
  return build_from_pattern(a, aux, pp, pc);
}

std::unique_ptr<Fsai> fsai_from_factors(Ctx* ctx, const Bsr& F, const double* shat) {
  if (!(F.rsz == F.csz)) fail(BMG_EINVAL, "fsai: factor must be square");
  const int n = F.nbr;
  Aux aux = make_aux(F, false);
  std::vector<int64_t> loff(n + 1, 0);
  for (int k = 0; k < n; ++k) loff[k + 1] = loff[k] + (int64_t)F.rsz[k] * F.rsz[k];
  DBuf<double> dl(std::max<int64_t>(loff[n], 1));
  DBuf<int64_t> dlo(n + 1);
  BMG_CUDA(cudaMemcpy(dl.p, shat, loff[n] * 8, cudaMemcpyHostToDevice));
  BMG_CUDA(cudaMemcpy(dlo.p, loff.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  auto G = make_bsr_structure(ctx, n, F.rsz.data(), n, F.csz.data(), F.h_row_ptr, F.h_col, false);
  const int mmax = max_size(F.rsz);
  const size_t smem = 2 * sizeof(double) * mmax * mmax;
  // G has F's structure and value layout; solve each block in place into G
  kern::linv_rows_kernel<<<std::max(1, std::min(n, ctx->sms * 16)), kern::kFsaiThreads, smem, ctx->stream>>>(
      view(F, aux), dl.p, dlo.p, G->vals.p, n, mmax);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  auto m = std::make_unique<Fsai>();
  m->ctx = ctx;
  m->dim = F.dim_r;
  auto GT = bsr_transpose(*G);
  m->fwd.push_back(std::move(G));
  m->bwd.push_back(std::move(GT));
  return m;
}

// M r = G^T (G r) for nest = 0; general chains apply fwd in order, bwd after
void fsai_apply(const Fsai& m, const double* r, double* z, double* t1, double* t2) {
  const double* cur = r;
  double* bufs[2] = {t1, t2};
  int which = 0;
  for (const auto& f : m.fwd) {
    spmv(*f, cur, bufs[which]);
    cur = bufs[which];
    which ^= 1;
  }
  for (size_t i = 0; i < m.bwd.size(); ++i) {
    double* out = (i + 1 == m.bwd.size()) ? z : bufs[which];
    spmv(*m.bwd[m.bwd.size() - 1 - i], cur, out);
    cur = out;
    which ^= 1;
  }
}

}  // namespace bmg
