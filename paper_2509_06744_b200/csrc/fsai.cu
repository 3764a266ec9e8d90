// fsai.cu -- batched block-FSAI setup on the device and the G / G^T apply.
//
// The reference keeps F (unit-diagonal lower) and per-row Cholesky factors of
// S = diag(F A F^T) and applies M = F^T S^{-1} F (fsai.cpp:60-70, 200-217).  The
// device path folds the per-row solves into G = L^{-1} F at setup
// (M = F^T L^{-T} L^{-1} F = G^T G), so the apply is two streaming
// passes: w = G r and z = G^T w (G^T stored as its own BSR, no atomics).
//
// Setup kernels (one CTA per block row, small dense work in shared memory):
//   fsai_adaptive_kernel adaptive_build with P0 = diagonal, any t_max
//                        (fsai.cpp:132-198, delta_ratio fsai.cpp:106-130):
//                        scores every lower candidate c of H row k = F_k A and
//                        admits argmin rho (ties -> smallest c) while rho < tau.
//   fsai_row_kernel      build_row (fsai.cpp:18-43) for an explicit lower
//                        pattern, then G row k = L_k^{-1} [F_kS, I].
// Dense arithmetic follows the oracle's fixed order (fma chains ascending), so
// G is bitwise equal to the oracle's L^{-1} F for the same pattern.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
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

// build_row (fsai.cpp:18-43) for row k with the strict lower pattern S (ns
// blocks, ascending): gram = chol(A[S,S]) (ng x ng), X = gram^{-1} A_kS^T
// (ng x mk), AKS = A_kS (mk x ng), S_kk = A_kk - A_kS X and Lk = chol(S_kk).
// Returns 0, or an error code (1 principal submatrix / 2 S row) with *piv.
__device__ int row_factor(const MatView& A, int k, const int32_t* S, int ns, double* gram, double* X,
                          double* AKS, double* Lk, int* ng_out, int* piv) {
  const int mk = A.rsz[k];
  int ng = 0;
  for (int q = 0; q < ns; ++q) ng += A.rsz[S[q]];
  *ng_out = ng;
  cta_load_block(Lk, A.vals + A.voff[A.diag[k]], mk * mk);
  if (ns > 0) {
    for (int e = threadIdx.x; e < ng * ng; e += blockDim.x) gram[e] = 0.0;
    __syncthreads();
    int ro = 0;
    for (int qa = 0; qa < ns; ++qa) {
      const int ia = S[qa], ma = A.rsz[ia];
      int co = 0;
      for (int qb = 0; qb < ns; ++qb) {
        const int ib = S[qb], mb = A.rsz[ib];
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
    int co = 0;
    for (int q = 0; q < ns; ++q) {
      const int j = S[q], mj = A.rsz[j];
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
      *piv = pg;
      return 1;
    }
    cta_solve(gram, ng, X, mk);  // X = gram^{-1} A_kS^T  (ng x mk)
    for (int e = threadIdx.x; e < mk * mk; e += blockDim.x) {
      const int r = e / mk, c = e - r * mk;
      double t = 0.0;
      for (int q = 0; q < ng; ++q) t = __fma_rn(AKS[r * ng + q], X[q * mk + c], t);
      Lk[e] = __dsub_rn(Lk[e], t);
    }
    __syncthreads();
  }
  const int ps = cta_chol(Lk, mk, nullptr);
  if (ps >= 0) {
    *piv = ps;
    return 2;
  }
  return 0;
}

__device__ inline void report(FsaiErr* err, int row, int what, int piv, int cand) {
  if (threadIdx.x == 0 && atomicCAS(&err->row, -1, row) == -1) {
    err->pivot = piv;
    err->what = what;
    err->cand = cand;
  }
}

// build_row for the explicit strict pattern of every row, then write row k of
// G = L^{-1} [F_kS, I] (write_f = 0) or of F = [F_kS, I] itself (write_f = 1,
// intermediate factors of a nested chain, fsai.cpp:243-253).
struct RowArgs {
  MatView A;
  const int64_t* pat_ptr;  // strict pattern CSR
  const int32_t* pat_col;
  double* gvals;           // output values, row k's blocks at gvoff[g_row_ptr[k] + q]
  const int64_t* g_row_ptr;
  const int64_t* gvoff;
  int n;
  int mmax;
  int gmax;  // max strict pattern size in scalars
  int write_f;
};

__global__ void __launch_bounds__(kFsaiThreads) fsai_row_kernel(RowArgs s, FsaiErr* err) {
  extern __shared__ double sm[];
  const int mm = s.mmax * s.mmax;
  double* gram = sm;                             // gmax^2
  double* X = gram + (size_t)s.gmax * s.gmax;    // gmax x mmax
  double* AKS = X + (size_t)s.gmax * s.mmax;     // mmax x gmax
  double* Lk = AKS + (size_t)s.gmax * s.mmax;    // mmax^2
  double* Y = Lk + mm;                           // mmax x (gmax + mmax)
  const MatView& A = s.A;
  for (int k = blockIdx.x; k < s.n; k += gridDim.x) {
    const int mk = A.rsz[k];
    const int64_t p0 = s.pat_ptr[k], p1 = s.pat_ptr[k + 1];
    const int ns = (int)(p1 - p0);
    int ng = 0, piv = -1;
    const int st = row_factor(A, k, s.pat_col + p0, ns, gram, X, AKS, Lk, &ng, &piv);
    if (st != 0) {
      report(err, k, st, piv, -1);
      return;
    }
    // Y = [F_kS | I] (mk x (ng + mk)), F_kS = -X^T; G: Y <- L^{-1} Y
    const int wy = ng + mk;
    for (int e = threadIdx.x; e < mk * wy; e += blockDim.x) {
      const int r = e / wy, c = e - r * wy;
      Y[e] = c < ng ? -X[c * mk + r] : (c - ng == r ? 1.0 : 0.0);
    }
    __syncthreads();
    if (!s.write_f) cta_solve_l(Lk, mk, Y, wy);
    // scatter into row k (blocks ascending: strict pattern, then diagonal)
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

// adaptive_build (fsai.cpp:132-198) with P0 = diagonal for any t_max: per row,
// t_max rounds of {rebuild row if stale; score every lower candidate c of
// H row k = F_k A with delta_ratio (fsai.cpp:106-130); admit argmin rho if
// rho < tau, else retire}.  Writes each row's final strict pattern.
constexpr int kMaxT = 15;
struct AdaptArgs {
  MatView A;
  int n, t_max, mmax;
  double tau;
  int32_t* pat;  // n x t_max, ascending
  int* cnt;
};

__global__ void __launch_bounds__(kFsaiThreads) fsai_adaptive_kernel(AdaptArgs s, FsaiErr* err) {
  extern __shared__ double sm[];
  const int mm = s.mmax * s.mmax, gm = s.t_max * s.mmax;
  double* gram = sm;                   // gm^2
  double* X = gram + (size_t)gm * gm;  // gm x mm
  double* AKS = X + (size_t)gm * s.mmax;
  double* Lk = AKS + (size_t)gm * s.mmax;
  double* H = Lk + mm;
  double* W = H + mm;
  double* U = W + mm;
  double* T = U + mm;
  double* ACS = T + mm;                   // mm x gm
  double* Y = ACS + (size_t)gm * s.mmax;  // gm x mm
  __shared__ int32_t S[kMaxT + 1];
  __shared__ int ns_s, stale_s, best_s, cand_s, skip_s, ng_s;
  __shared__ int64_t jpos[kMaxT + 1];
  __shared__ double thr_s, best_rho_s, ldw_s, ldu_s;
  const MatView& A = s.A;
  for (int k = blockIdx.x; k < s.n; k += gridDim.x) {
    const int mk = A.rsz[k];
    if (threadIdx.x == 0) {
      ns_s = 0;
      stale_s = 1;
    }
    __syncthreads();
    bool active = true;
    for (int t = 1; t <= s.t_max && active; ++t) {
      if (stale_s) {
        int ng = 0, piv = -1;
        const int st = row_factor(A, k, S, ns_s, gram, X, AKS, Lk, &ng, &piv);
        if (st != 0) {
          report(err, k, st, piv, -1);
          return;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          stale_s = 0;
          ng_s = ng;
        }
        __syncthreads();
      }
      const int ns = ns_s, ng = ng_s;
      // H_kc = sum over j in S u {k} (ascending) of F_kj A_jc   (fsai.cpp:46-51)
      auto h_block = [&](int c, double* out) {
        const int mc = A.rsz[c];
        if (threadIdx.x <= ns) {
          const int j = threadIdx.x < ns ? S[threadIdx.x] : k;
          const int64_t lo = A.row_ptr[j], hi = A.row_ptr[j + 1];
          const int pos = find_col(A.col, lo, hi, c);
          jpos[threadIdx.x] = (pos < hi && A.col[pos] == c) ? pos : -1;
        }
        __syncthreads();
        for (int e = threadIdx.x; e < mk * mc; e += blockDim.x) {
          const int r = e / mc, cc = e - r * mc;
          double acc = 0.0;
          int off = 0;
          for (int q = 0; q <= ns; ++q) {
            const int j = q < ns ? S[q] : k;
            const int mj = A.rsz[j];
            if (jpos[q] >= 0) {
              const double* a = A.vals + A.voff[jpos[q]];
              double tt = 0.0;
              for (int z = 0; z < mj; ++z) {
                const double f = q < ns ? -X[(off + z) * mk + r] : (z == r ? 1.0 : 0.0);
                tt = __fma_rn(f, a[z * mc + cc], tt);
              }
              acc = __dadd_rn(acc, tt);
            }
            off += mj;
          }
          out[e] = acc;
        }
        __syncthreads();
      };
      h_block(k, H);
      if (threadIdx.x == 0) {
        thr_s = 1e-12 * frob_serial(H, mk * mk);
        best_s = -1;
        best_rho_s = 0.0;
        cand_s = -1;
      }
      __syncthreads();
      for (;;) {
        // next candidate: smallest column > cand of rows S u {k}, below k, not in S
        if (threadIdx.x == 0) {
          int nxt = k;
          for (int q = 0; q <= ns; ++q) {
            const int j = q < ns ? S[q] : k;
            const int64_t lo = A.row_ptr[j], hi = A.row_ptr[j + 1];
            int64_t p = find_col(A.col, lo, hi, cand_s + 1);
            while (p < hi && A.col[p] < nxt) {
              bool in_s = false;
              for (int z = 0; z < ns; ++z) in_s |= (S[z] == A.col[p]);
              if (!in_s) {
                nxt = A.col[p];
                break;
              }
              ++p;
            }
          }
          cand_s = nxt < k ? nxt : -2;
        }
        __syncthreads();
        const int c = cand_s;
        if (c < 0) break;
        const int mc = A.rsz[c];
        h_block(c, H);
        if (threadIdx.x == 0) skip_s = frob_serial(H, mk * mc) <= thr_s;
        __syncthreads();
        if (skip_s) continue;
        // W = A_cc - A_cS gram^{-1} A_cS^T
        const double* acc_blk = A.vals + A.voff[A.diag[c]];
        cta_load_block(W, acc_blk, mc * mc);
        if (ns > 0) {
          int co = 0;
          for (int q = 0; q < ns; ++q) {
            const int j = S[q], mj = A.rsz[j];
            const int64_t lo = A.row_ptr[c], hi = A.row_ptr[c + 1];
            const int pos = find_col(A.col, lo, hi, j);
            const bool present = pos < hi && A.col[pos] == j;
            const double* blk = present ? A.vals + A.voff[pos] : nullptr;
            for (int e = threadIdx.x; e < mc * mj; e += blockDim.x) {
              const int r = e / mj, cc = e - r * mj;
              const double v = present ? blk[e] : 0.0;
              ACS[r * ng + co + cc] = v;
              Y[(co + cc) * mc + r] = v;
            }
            co += mj;
          }
          __syncthreads();
          cta_solve(gram, ng, Y, mc);
          for (int e = threadIdx.x; e < mc * mc; e += blockDim.x) {
            const int r = e / mc, q = e - r * mc;
            double tt = 0.0;
            for (int z = 0; z < ng; ++z) tt = __fma_rn(ACS[r * ng + z], Y[z * mc + q], tt);
            W[e] = __dsub_rn(W[e], tt);
          }
          __syncthreads();
        }
        for (int e = threadIdx.x; e < mc * mc; e += blockDim.x) U[e] = W[e];
        __syncthreads();
        const int pw = cta_chol(W, mc, &ldw_s);
        if (pw >= 0) {
          report(err, k, 3, pw, c);
          return;
        }
        // U = W - H_kc^T S_k^{-1} H_kc
        for (int e = threadIdx.x; e < mk * mc; e += blockDim.x) T[e] = H[e];
        __syncthreads();
        cta_solve(Lk, mk, T, mc);
        for (int e = threadIdx.x; e < mc * mc; e += blockDim.x) {
          const int r = e / mc, q = e - r * mc;
          double tt = 0.0;
          for (int z = 0; z < mk; ++z) tt = __fma_rn(H[z * mc + r], T[z * mc + q], tt);
          U[e] = __dsub_rn(U[e], tt);
        }
        __syncthreads();
        const int pu = cta_chol(U, mc, &ldu_s);
        if (threadIdx.x == 0) {
          const double rho = pu >= 0 ? 0.0 : fmin(exp(__dsub_rn(ldu_s, ldw_s)), 1.0);
          if (best_s < 0 || rho < best_rho_s) {  // ties keep the smallest column
            best_s = c;
            best_rho_s = rho;
          }
        }
        __syncthreads();
      }
      if (best_s < 0 || !(best_rho_s < s.tau)) {
        active = false;
      } else if (threadIdx.x == 0) {
        int q = ns_s;
        while (q > 0 && S[q - 1] > best_s) {
          S[q] = S[q - 1];
          --q;
        }
        S[q] = best_s;
        ++ns_s;
        stale_s = 1;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      s.cnt[k] = ns_s;
      for (int q = 0; q < ns_s; ++q) s.pat[(int64_t)k * s.t_max + q] = S[q];
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

// F (write_f) or G = L^{-1} F for an explicit strict pattern (row k: pattern
// ascending, then k)
std::unique_ptr<Bsr> factor_from_pattern(const Bsr& a, const Aux& aux, const std::vector<int64_t>& pat_ptr,
                                         const std::vector<int32_t>& pat_col, bool write_f) {
  Ctx* ctx = a.ctx;
  const int n = a.nbr;
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
  kern::RowArgs ra{view(a, aux), dpp.p, dpc.p, G->vals.p, G->row_ptr.p, dgv.p, n, mmax, gmax, write_f ? 1 : 0};
  BMG_CUDA(cudaFuncSetAttribute(kern::fsai_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::max(1, std::min(n, ctx->sms * 16));
  kern::fsai_row_kernel<<<grid, kern::kFsaiThreads, smem, ctx->stream>>>(ra, derr.p);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  check_err(ctx, derr.p);
  return G;
}

// adaptive_build pattern selection on the device (any t_max, P0 = diagonal)
void adaptive_pattern(const Bsr& a, const Aux& aux, int t_max, double tau, std::vector<int64_t>& pp,
                      std::vector<int32_t>& pc) {
  Ctx* ctx = a.ctx;
  const int n = a.nbr;
  if (t_max > kern::kMaxT) fail(BMG_EINVAL, "adaptive_build: t_max above the device limit (15)");
  const int mmax = max_size(a.rsz);
  const size_t gm = (size_t)t_max * mmax, mm = (size_t)mmax * mmax;
  const size_t smem = sizeof(double) * (gm * gm + 4 * gm * mmax + 5 * mm);
  if (smem > 200 * 1024) fail(BMG_EINVAL, "adaptive_build: t_max x block size too large for the device build");
  DBuf<int32_t> pat(std::max<size_t>((size_t)n * t_max, 1));
  DBuf<int> cnt(std::max(n, 1));
  DBuf<kern::FsaiErr> derr(1);
  kern::FsaiErr e0{-1, -1, 0, -1};
  BMG_CUDA(cudaMemcpy(derr.p, &e0, sizeof(e0), cudaMemcpyHostToDevice));
  BMG_CUDA(cudaFuncSetAttribute(kern::fsai_adaptive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern::AdaptArgs args{view(a, aux), n, t_max, mmax, tau, pat.p, cnt.p};
  const int grid = std::max(1, std::min(n, ctx->sms * 16));
  kern::fsai_adaptive_kernel<<<grid, kern::kFsaiThreads, smem, ctx->stream>>>(args, derr.p);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  check_err(ctx, derr.p);
  std::vector<int32_t> hp((size_t)n * t_max);
  std::vector<int> hc(n);
  if (n) {
    BMG_CUDA(cudaMemcpy(hp.data(), pat.p, hp.size() * 4, cudaMemcpyDeviceToHost));
    BMG_CUDA(cudaMemcpy(hc.data(), cnt.p, n * 4, cudaMemcpyDeviceToHost));
  }
  pp.assign(n + 1, 0);
  pc.clear();
  for (int k = 0; k < n; ++k) {
    for (int q = 0; q < hc[k]; ++q) pc.push_back(hp[(size_t)k * t_max + q]);
    pp[k + 1] = (int64_t)pc.size();
  }
}

std::unique_ptr<Fsai> wrap(Ctx* ctx, int dim, std::vector<std::unique_ptr<Bsr>> fwd) {
  auto m = std::make_unique<Fsai>();
  m->ctx = ctx;
  m->dim = dim;
  for (auto& f : fwd) m->bwd.push_back(bsr_transpose(*f));
  m->fwd = std::move(fwd);
  return m;
}

}  // namespace

std::unique_ptr<Fsai> fsai_build(const Bsr& a, int kind, int t_max, double tau, int nest) {
  if (!(a.rsz == a.csz)) fail(BMG_EINVAL, "fsai: matrix must be square");
  if (!a.sym) fail(BMG_EINVAL, "fsai: matrix must be symmetric");
  Ctx* ctx = a.ctx;
  const int n = a.nbr;
  std::vector<int64_t> pp(n + 1, 0);
  std::vector<int32_t> pc;
  std::vector<std::unique_ptr<Bsr>> fwd;
  if (kind == BMG_FSAI_STATIC_LOWER || kind == BMG_FSAI_DIAGONAL) {
    Aux aux = make_aux(a, true);
    if (kind == BMG_FSAI_STATIC_LOWER)
      for (int k = 0; k < n; ++k) {
        for (int64_t p = a.h_row_ptr[k]; p < a.h_row_ptr[k + 1]; ++p)
          if (a.h_col[p] < k) pc.push_back(a.h_col[p]);
        pp[k + 1] = (int64_t)pc.size();
      }
    fwd.push_back(factor_from_pattern(a, aux, pp, pc, false));
    return wrap(ctx, a.dim_r, std::move(fwd));
  }
  if (kind != BMG_FSAI_ADAPTIVE) fail(BMG_EINVAL, "bmg_fsai_build: unknown kind");
  if (t_max < 1) fail(BMG_EINVAL, "adaptive_build: t_max must be >= 1");
  if (!(tau > 0.0 && tau <= 1.0)) fail(BMG_EINVAL, "adaptive_build: tau must be in (0, 1]");
  if (nest < 0) fail(BMG_EINVAL, "nested_build: n_levels must be >= 0");
  // nested_build (fsai.cpp:243-253): A_0 = A, A_{k+1} = F_k A_k F_k^T; the chain
  // applies F_0 .. F_{n-1} and G_n = L-hat^{-1} F_n
  const Bsr* ak = &a;
  std::unique_ptr<Bsr> ak_own;
  static const bool timing = [] {
    const char* e = std::getenv("BMG_SETUP_TIMING");
    return e && e[0] == '1';
  }();
  auto t = std::chrono::steady_clock::now();
  auto mark = [&](const char* what, int level) {
    if (!timing) return;
    cudaStreamSynchronize(ctx->stream);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bmg setup]   fsai %d: %-22s %8.3f s\n", level, what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  };
  for (int level = 0; level <= nest; ++level) {
    Aux aux = make_aux(*ak, true);
    mark("aux", level);
    adaptive_pattern(*ak, aux, t_max, tau, pp, pc);
    mark("adaptive pattern", level);
    if (level < nest) {
      auto F = factor_from_pattern(*ak, aux, pp, pc, true);
      mark("factor", level);
      auto next = triple_product(*F, *ak);
      mark("triple product", level);
      fwd.push_back(std::move(F));
      ak_own = std::move(next);
      ak = ak_own.get();
    } else {
      fwd.push_back(factor_from_pattern(*ak, aux, pp, pc, false));
      mark("factor", level);
    }
  }
  auto out = wrap(ctx, a.dim_r, std::move(fwd));
  mark("transposes", nest);
  return out;
}

// build_fsai(A, p) (fsai.cpp:72-83) for a caller's lower pattern: per row the
// strictly lower block columns (LowerPattern::add semantics: duplicates and the
// diagonal, which is always present, are ignored; j > i is an error)
std::unique_ptr<Fsai> fsai_build_pattern(const Bsr& a, const int64_t* ptr, const int32_t* col) {
  if (!(a.rsz == a.csz)) fail(BMG_EINVAL, "fsai: matrix must be square");
  if (!a.sym) fail(BMG_EINVAL, "fsai: matrix must be symmetric");
  const int n = a.nbr;
  std::vector<int64_t> pp(n + 1, 0);
  std::vector<int32_t> pc;
  if (ptr[0] != 0) fail(BMG_EINVAL, "LowerPattern: row_ptr[0] must be 0");
  std::vector<int32_t> row;
  for (int k = 0; k < n; ++k) {
    if (ptr[k + 1] < ptr[k]) fail(BMG_EINVAL, "LowerPattern: row_ptr must be non-decreasing");
    row.clear();
    for (int64_t q = ptr[k]; q < ptr[k + 1]; ++q) {
      const int c = col[q];
      if (c == k) continue;
      if (c < 0 || c > k) fail(BMG_EINVAL, "LowerPattern: entries must satisfy 0 <= j <= i");
      row.push_back(c);
    }
    std::sort(row.begin(), row.end());
    row.erase(std::unique(row.begin(), row.end()), row.end());
    pc.insert(pc.end(), row.begin(), row.end());
    pp[k + 1] = (int64_t)pc.size();
  }
  Aux aux = make_aux(a, true);
  std::vector<std::unique_ptr<Bsr>> fwd;
  fwd.push_back(factor_from_pattern(a, aux, pp, pc, false));
  return wrap(a.ctx, a.dim_r, std::move(fwd));
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
