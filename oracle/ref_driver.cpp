// ref_driver.cpp -- C entry points over THE REFERENCE ITSELF (test infrastructure).
//
// oracle/_ref/libblockmg_ref.so = the reference's own, unmodified sources
//   /root/reference/proj/src/{block_layout,block_matrix,kernels,small_cholesky,
//   pattern,fsai,chebyshev,multilevel,matrix_io,experiments}.cpp
//   (+ pum/{cover,space,bspline,legendre,jet}.cpp, which experiments.hpp pulls in)
// compiled where they lie (oracle/Makefile target `ref`; nothing is copied into
// this repository) against oracle/eigen_shim -- a from-scratch stand-in for the
// subset of the Eigen API they use, because Eigen3 is not installed -- plus this
// file, which only converts flat arrays to the reference's classes and calls its
// public functions.  It exports the SAME C API as oracle/bmg_oracle.h, so
// oracle/pyoracle.py drives either library and tests compare the two bitwise
// (tests/test_reference_build.py): everything above the dense primitives is then
// the reference's code, not a restatement.
//
// Only tests/, smoke() and bench.py's CPU legs may load it; /root/reference does
// not exist on the GPU box, so the library is built here and travels prebuilt.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "blockmg/block_matrix.hpp"
#include "blockmg/chebyshev.hpp"
#include "blockmg/experiments.hpp"
#include "blockmg/fsai.hpp"
#include "blockmg/kernels.hpp"
#include "blockmg/lanczos.hpp"
#include "blockmg/matrix_io.hpp"
#include "blockmg/multilevel.hpp"
#include "blockmg/pattern.hpp"
#include "blockmg/rng.hpp"
#include "blockmg/small_cholesky.hpp"
#include "bmg_oracle.h"

// The PUM discretiser is out of scope: experiments.cpp's
// build_pum_chain refers to these three; they are never reached from this driver.
namespace bmg::pum {
AssembledSystem assemble(const PuSpace&, const AssembleOptions&, const ManufacturedSolution&) {
  throw std::logic_error("pum::assemble: the PUM discretiser is not part of this build");
}
BlockSparseMatrix build_prolongation(const PuSpace&, const PuSpace&) {
  throw std::logic_error("pum::build_prolongation: the PUM discretiser is not part of this build");
}
ManufacturedSolution manufactured(Problem, const AnisotropySpec&) {
  throw std::logic_error("pum::manufactured: the PUM discretiser is not part of this build");
}
}  // namespace bmg::pum

using namespace bmg;

struct orc_mat { BlockSparseMatrix m; };
struct orc_fsai { NestedFsai f; };
struct orc_hier { Hierarchy h; };

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

static Vector to_vec(const double* p, int n) {
  Vector v(n);
  std::copy(p, p + n, v.data());
  return v;
}
static void from_vec(const Vector& v, double* p) { std::copy(v.data(), v.data() + v.size(), p); }

static BlockSparseMatrix make_mat(int nbr, const int32_t* row_sizes, int nbc, const int32_t* col_sizes,
                                  const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                                  bool symmetric) {
  BlockLayout rl(std::vector<int>(row_sizes, row_sizes + nbr));
  BlockLayout cl(std::vector<int>(col_sizes, col_sizes + nbc));
  BlockSparseMatrix a(rl, cl, symmetric);
  int64_t voff = 0;
  for (int i = 0; i < nbr; ++i) {
    int prev = -1;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int j = col_idx[p];
      if (j < 0 || j >= nbc) throw std::out_of_range("BlockSparseMatrix: block index out of range");
      if (j <= prev) throw std::invalid_argument("orc_mat_create: columns must be strictly ascending");
      prev = j;
      const int mi = rl.size(i), mj = cl.size(j);
      DenseBlock b(mi, mj);
      std::copy(vals + voff, vals + voff + static_cast<int64_t>(mi) * mj, b.data());
      voff += static_cast<int64_t>(mi) * mj;
      a.insert(i, j, std::move(b));
    }
  }
  return a;
}

static LowerPattern pattern_from_csr(int n, const int64_t* pp, const int32_t* pc) {
  LowerPattern p = LowerPattern::diagonal(n);
  for (int i = 0; i < n; ++i)
    for (int64_t q = pp[i]; q < pp[i + 1]; ++q) p.add(i, pc[q]);
  return p;
}

static SmootherSpec make_spec(int kind, double alpha, double beta, double omega, int degree) {
  SmootherSpec s;
  switch (kind) {
    case 0: s.kind = SmootherKind::Richardson; break;
    case 1: s.kind = SmootherKind::ChebFirst; break;
    case 2: s.kind = SmootherKind::ChebFourth; break;
    default: throw std::invalid_argument("smoother: unknown kind");
  }
  s.degree = degree;
  s.alpha = alpha;
  s.beta = beta;
  s.omega = omega;
  return s;
}

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }
int orc_last_pivot(void) { return g_pivot; }
int orc_set_threads(int) { return 0; }  // the reference is single-threaded
int orc_get_threads(void) { return 1; }

int orc_mat_create(int nbr, const int32_t* row_sizes, int nbc, const int32_t* col_sizes,
                   const int64_t* row_ptr, const int32_t* col_idx, const double* vals, int symmetric,
                   orc_mat** out) {
  return guard([&] {
    *out = new orc_mat{make_mat(nbr, row_sizes, nbc, col_sizes, row_ptr, col_idx, vals, symmetric != 0)};
  });
}
void orc_mat_destroy(orc_mat* a) { delete a; }

int orc_mat_info(const orc_mat* a, int* nbr, int* nbc, int64_t* nnzb, int64_t* nvals, int* dim_r,
                 int* dim_c) {
  return guard([&] {
    *nbr = a->m.block_rows();
    *nbc = a->m.block_cols();
    *nnzb = static_cast<int64_t>(a->m.stored_blocks());
    *nvals = static_cast<int64_t>(a->m.stored_scalars());
    *dim_r = a->m.row_layout().dim();
    *dim_c = a->m.col_layout().dim();
  });
}
int orc_mat_export(const orc_mat* a, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  return guard([&] {
    int64_t p = 0, v = 0;
    row_ptr[0] = 0;
    for (int i = 0; i < a->m.block_rows(); ++i) {
      for (const auto& [j, blk] : a->m.row(i)) {
        col_idx[p++] = j;
        for (Eigen::Index r = 0; r < blk.rows(); ++r)
          for (Eigen::Index c = 0; c < blk.cols(); ++c) vals[v++] = blk(r, c);
      }
      row_ptr[i + 1] = p;
    }
  });
}
/* layouts of a matrix produced by the library (orc_mat_info gives the counts) */
int orc_mat_layouts(const orc_mat* a, int32_t* row_sizes, int32_t* col_sizes) {
  return guard([&] {
    for (int i = 0; i < a->m.block_rows(); ++i) row_sizes[i] = a->m.row_layout().size(i);
    for (int j = 0; j < a->m.block_cols(); ++j) col_sizes[j] = a->m.col_layout().size(j);
  });
}

int orc_spmv(const orc_mat* a, const double* x, double* y) {
  return guard([&] {
    Vector yv;
    spmv(a->m, to_vec(x, a->m.col_layout().dim()), yv);
    from_vec(yv, y);
  });
}
int orc_spmv_t(const orc_mat* a, const double* x, double* y) {
  return guard([&] {
    Vector yv;
    spmv_transpose(a->m, to_vec(x, a->m.row_layout().dim()), yv);
    from_vec(yv, y);
  });
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
  return guard([&] { *out = new orc_mat{galerkin_coarsen(a->m, p->m)}; });
}

int orc_cholesky(int n, const double* b, double* l_out, double* logdet) {
  return guard([&] {
    DenseBlock bm(n, n);
    std::copy(b, b + static_cast<size_t>(n) * n, bm.data());
    const SmallCholesky c(bm);
    const DenseBlock& l = c.matrix_l();
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) l_out[static_cast<size_t>(i) * n + j] = l(i, j);
    *logdet = c.logdet();
  });
}
/* B x = rhs with B given (the reference factors it itself): SmallCholesky(B).solve(rhs) */
int orc_chol_solve_spd(int n, const double* b, const double* rhs, double* x) {
  return guard([&] {
    DenseBlock bm(n, n);
    std::copy(b, b + static_cast<size_t>(n) * n, bm.data());
    from_vec(SmallCholesky(bm).solve(to_vec(rhs, n)), x);
  });
}
int orc_chol_solve(int, const double*, const double*, double*) {
  g_err = "orc_chol_solve: the reference's SmallCholesky cannot be built from a given factor; use orc_chol_solve_spd";
  return ORC_ERUNTIME;
}

int orc_fsai_build(const orc_mat* a, int kind, int t_max, double tau, int nest, orc_fsai** out) {
  return guard([&] {
    NestedFsai f;
    f.layout = a->m.row_layout();
    switch (kind) {
      case 0: f.chain.push_back(build_fsai(a->m, LowerPattern::from_matrix(a->m))); break;
      case 1: f.chain.push_back(build_fsai(a->m, LowerPattern::diagonal(a->m.block_rows()))); break;
      case 2: f.chain.push_back(build_fsai(a->m, LowerPattern::full(a->m.block_rows()))); break;
      case 3: f = nested_build(a->m, t_max, tau, nest); break;
      default: throw std::invalid_argument("orc_fsai_build: unknown kind");
    }
    *out = new orc_fsai{std::move(f)};
  });
}
int orc_fsai_build_pattern(const orc_mat* a, const int64_t* pat_ptr, const int32_t* pat_col, orc_fsai** out) {
  return guard([&] {
    NestedFsai f;
    f.layout = a->m.row_layout();
    f.chain.push_back(build_fsai(a->m, pattern_from_csr(a->m.block_rows(), pat_ptr, pat_col)));
    *out = new orc_fsai{std::move(f)};
  });
}
int orc_delta_ratio(const orc_mat* a, const int64_t* pat_ptr, const int32_t* pat_col, int k, int c,
                    double* out) {
  return guard([&] {
    const AdaptiveState st = make_adaptive_state(a->m, pattern_from_csr(a->m.block_rows(), pat_ptr, pat_col));
    *out = delta_ratio(st, a->m, k, c);
  });
}
void orc_fsai_destroy(orc_fsai* f) { delete f; }
int orc_fsai_apply(const orc_fsai* f, const double* r, double* out) {
  return guard([&] { from_vec(f->f.apply(to_vec(r, f->f.layout.dim())), out); });
}
int orc_fsai_apply_transformed(const orc_fsai* f, const orc_mat* a, const double* x, double* out) {
  return guard([&] { from_vec(f->f.apply_transformed(a->m, to_vec(x, f->f.layout.dim())), out); });
}
int orc_fsai_chain_len(const orc_fsai* f) { return static_cast<int>(f->f.chain.size()); }
int orc_fsai_factor(const orc_fsai* f, int k, orc_mat** F_out) {
  return guard([&] {
    if (k < 0 || k >= static_cast<int>(f->f.chain.size())) throw std::out_of_range("orc_fsai_factor");
    *F_out = new orc_mat{f->f.chain[static_cast<size_t>(k)].F};
  });
}
int orc_fsai_shat(const orc_fsai* f, double* l_packed) {
  return guard([&] {
    size_t o = 0;
    for (const SmallCholesky& c : f->f.final_diag()) {
      const DenseBlock& l = c.matrix_l();
      for (Eigen::Index i = 0; i < l.rows(); ++i)
        for (Eigen::Index j = 0; j < l.cols(); ++j) l_packed[o++] = l(i, j);
    }
  });
}
// G = L-hat^{-1} F_last, column by column with the reference's solve_l
int orc_fsai_G(const orc_fsai* f, orc_mat** G_out) {
  return guard([&] {
    const FsaiFactors& fac = f->f.chain.back();
    BlockSparseMatrix g(fac.layout, fac.layout, false);
    for (int k = 0; k < fac.F.block_rows(); ++k)
      for (const auto& [j, blk] : fac.F.row(k)) {
        DenseBlock out(blk.rows(), blk.cols());
        for (Eigen::Index c = 0; c < blk.cols(); ++c)
          out.col(c) = fac.S[static_cast<size_t>(k)].solve_l(Vector(blk.col(c)));
        g.insert(k, j, std::move(out));
      }
    *G_out = new orc_mat{std::move(g)};
  });
}

int orc_lanczos_lambda_max(const orc_mat* a, const orc_fsai* f, int iters, double safety, uint64_t seed,
                           double* beta) {
  return guard([&] { *beta = lanczos_lambda_max(a->m, f->f, iters, safety, seed); });
}
int orc_lanczos_diag(int n, const double* lam, int iters, double safety, uint64_t seed, int smallest,
                     double* out) {
  return guard([&] {
    auto op = [&](const Vector& x, Vector& y) {
      y = x;
      for (int i = 0; i < n; ++i) y[i] = lam[i] * x[i];
    };
    *out = smallest ? lanczos_smallest_ritz(op, n, iters, seed) : lanczos_lambda_max(op, n, iters, safety, seed);
  });
}
int orc_tridiag_eigs(int n, const double* d, const double* e, double* eig_sorted) {
  return guard([&] {
    Eigen::SelfAdjointEigenSolver<Eigen::MatrixXd> es;
    es.computeFromTridiagonal(Eigen::Map<const Eigen::VectorXd>(d, n),
                              Eigen::Map<const Eigen::VectorXd>(e, n > 0 ? n - 1 : 0), Eigen::EigenvaluesOnly);
    from_vec(es.eigenvalues(), eig_sorted);
  });
}

int orc_smoother_apply(const orc_mat* a, const orc_fsai* f, int kind, double alpha, double beta, double omega,
                       int k, const double* b, double* x) {
  return guard([&] {
    const int n = a->m.row_layout().dim();
    const SmootherSpec spec = make_spec(kind, alpha, beta, omega, k);
    auto a_op = [&](const Vector& in, Vector& out) { spmv(a->m, in, out); };
    Vector xv = to_vec(x, n);
    const Vector bv = to_vec(b, n);
    if (f) {
      auto m_op = [&](const Vector& in, Vector& out) { out = f->f.apply(in); };
      xv = apply_smoother(spec, k, a_op, m_op, bv, std::move(xv));
    } else {
      auto m_op = [&](const Vector& in, Vector& out) { out = in; };
      xv = apply_smoother(spec, k, a_op, m_op, bv, std::move(xv));
    }
    from_vec(xv, x);
  });
}
int orc_smoother_apply_diag(int n, const double* lam, int kind, double alpha, double beta, double omega, int k,
                            const double* b, double* x) {
  return guard([&] {
    const SmootherSpec spec = make_spec(kind, alpha, beta, omega, k);
    auto a_op = [&](const Vector& in, Vector& out) {
      out = in;
      for (int i = 0; i < n; ++i) out[i] = lam[i] * in[i];
    };
    auto m_op = [&](const Vector& in, Vector& out) { out = in; };
    from_vec(apply_smoother(spec, k, a_op, m_op, to_vec(b, n), to_vec(x, n)), x);
  });
}
int orc_poly_eval(int kind, int degree, double alpha, double beta, double t, double* out) {
  return guard([&] {
    PolyEval pe;
    switch (kind) {
      case 0: pe.kind = ChebKind::FirstT; break;
      case 1: pe.kind = ChebKind::FourthW; break;
      case 2: pe.kind = ChebKind::ScaledFirst; break;
      case 3: pe.kind = ChebKind::ScaledFourth; break;
      default: throw std::invalid_argument("orc_poly_eval: unknown kind");
    }
    pe.degree = degree;
    pe.alpha = alpha;
    pe.beta = beta;
    *out = poly_eval(pe, t);
  });
}
double orc_fourth_kind_mu(int n) { return fourth_kind_mu(n); }

int orc_set_consume(int) { return 0; }
// the reference's setup() (multilevel.cpp:36-75): nested_build on every level and
// the indefiniteness probe, always
int orc_setup(const orc_mat* a_finest, int ntransfers, const orc_mat* const* transfers, int t_max, double tau,
              int nest, int fsai_kind, int lanczos_iters, double lanczos_safety, uint64_t seed,
              int coarse_dim_cap, int /*smallest_ritz_probe*/, int smoother_kind, double richardson_omega,
              double first_kind_fraction, orc_hier** out) {
  return guard([&] {
    if (fsai_kind != 3) throw std::invalid_argument("orc_setup: the reference's setup() builds nested FSAI only");
    SetupParams p;
    p.t_max = t_max;
    p.tau = tau;
    p.nest = nest;
    p.kind = make_spec(smoother_kind, 0.0, 1.0, 1.0, 1).kind;
    p.richardson_omega = richardson_omega;
    p.first_kind_fraction = first_kind_fraction;
    p.lanczos_iters = lanczos_iters;
    p.lanczos_safety = lanczos_safety;
    p.seed = seed;
    p.coarse_dim_cap = coarse_dim_cap;
    std::vector<BlockSparseMatrix> tr;
    for (int i = 0; i < ntransfers; ++i) tr.push_back(transfers[i]->m);
    *out = new orc_hier{setup(a_finest->m, std::move(tr), p)};
  });
}
void orc_hier_destroy(orc_hier* h) { delete h; }
int orc_hier_levels(const orc_hier* h) { return static_cast<int>(h->h.levels.size()); }
int orc_hier_level_A(const orc_hier* h, int l, const orc_mat** a) {
  return guard([&] {
    if (l < 0 || l > h->h.finest()) throw std::out_of_range("level");
    *a = reinterpret_cast<const orc_mat*>(&h->h.levels[static_cast<size_t>(l)].A);
  });
}
int orc_hier_level_P(const orc_hier* h, int l, const orc_mat** p) {
  return guard([&] {
    if (l < 1 || l > h->h.finest()) throw std::out_of_range("level");
    *p = reinterpret_cast<const orc_mat*>(&h->h.levels[static_cast<size_t>(l)].P);
  });
}
int orc_hier_level_fsai(const orc_hier* h, int l, const orc_fsai** f) {
  return guard([&] {
    if (l < 1 || l > h->h.finest()) throw std::out_of_range("level");
    *f = reinterpret_cast<const orc_fsai*>(&h->h.levels[static_cast<size_t>(l)].fsai);
  });
}
int orc_hier_beta(const orc_hier* h, int l, double* beta) {
  return guard([&] {
    if (l < 1 || l > h->h.finest()) throw std::out_of_range("level");
    *beta = h->h.levels[static_cast<size_t>(l)].smoother.beta;
  });
}
int orc_hier_coarse_l(const orc_hier* h, double* l_dense) {
  return guard([&] {
    const auto& l = h->h.coarse.matrixLLT();
    for (Eigen::Index i = 0; i < l.rows(); ++i)
      for (Eigen::Index j = 0; j < l.cols(); ++j) l_dense[i * l.cols() + j] = l(i, j);
  });
}
int orc_vcycle(const orc_hier* h, int k_pre, int k_post, int level, const double* b, double* x) {
  return guard([&] {
    if (level < 0 || level > h->h.finest()) throw std::out_of_range("v_cycle: level out of range");
    const int n = h->h.levels[static_cast<size_t>(level)].A.row_layout().dim();
    Vector xv = to_vec(x, n);
    v_cycle(h->h, CycleSpec{k_pre, k_post}, level, to_vec(b, n), xv);
    from_vec(xv, x);
  });
}
// the stop-on-tolerance loop of experiments.cpp:46-58 on the residual norm, around
// the reference's v_cycle (same driver as the oracle's orc_solve)
int orc_solve(const orc_hier* h, int k_pre, int k_post, const double* b, double* x, double tol, int max_iter,
              double* hist, int* iters, int* status) {
  return guard([&] {
    const BlockSparseMatrix& a = h->h.levels.back().A;
    const int n = a.row_layout().dim();
    const Vector bv = to_vec(b, n);
    Vector xv = to_vec(x, n), t(n);
    auto resid = [&]() {
      spmv(a, xv, t);
      return Vector(bv - t).norm();
    };
    hist[0] = resid();
    int it = 0, st = 1;
    if (hist[0] == 0.0 || hist[0] / hist[0] < tol) st = 0;
    const CycleSpec spec{k_pre, k_post};
    while (st == 1 && it < max_iter) {
      v_cycle(h->h, spec, h->h.finest(), bv, xv);
      ++it;
      hist[it] = resid();
      const double growth = hist[it] / std::max(hist[it - 1], 1e-300);
      if (!std::isfinite(hist[it]) || growth > 1e6) {
        st = 2;
        break;
      }
      if (hist[it] / hist[0] < tol) st = 0;
    }
    from_vec(xv, x);
    *iters = it;
    *status = st;
  });
}

// the reference's measure_rates (experiments.cpp:15-67) itself
int orc_measure_rates(const orc_hier* h, const orc_mat* mass, const double* b, const double* u_ref, int k_pre,
                      int k_post, uint64_t seed, double tol, int max_iter, double* l2_sq, double* energy_sq,
                      double* residual, int* iters, int* status, int* blowup, double* rates) {
  return guard([&] {
    const BlockSparseMatrix& a = h->h.levels.back().A;
    const int n = a.row_layout().dim();
    pum::AssembledSystem sys;
    sys.A = a;
    sys.mass = mass->m;
    sys.b = BlockVector(a.row_layout(), to_vec(b, n));
    sys.reference = to_vec(u_ref, n);
    const RateReport rep = measure_rates(h->h, sys, CycleSpec{k_pre, k_post}, seed, tol, max_iter);
    std::copy(rep.l2_sq.begin(), rep.l2_sq.end(), l2_sq);
    std::copy(rep.energy_sq.begin(), rep.energy_sq.end(), energy_sq);
    std::copy(rep.residual.begin(), rep.residual.end(), residual);
    *iters = rep.iterations;
    *status = rep.status == SolveStatus::Converged ? 0 : rep.status == SolveStatus::MaxIter ? 1 : 2;
    *blowup = rep.blowup_iteration;
    rates[0] = rep.rho_l2;
    rates[1] = rep.rho_a;
    rates[2] = rep.rho_r;
  });
}

uint64_t orc_mix64(uint64_t z) { return mix64(z); }
double orc_rng_uniform(uint64_t seed, uint64_t i) { return CounterRng(seed).uniform(i); }

/* ---- entries only this library has ---- */
int orc_is_reference(void) { return 1; }

/* the reference's own test problem, fd_biharmonic (experiments.cpp:104-195):
 * A, mass, levels-1 transfers (coarsest first) as matrices, b and the reference
 * coefficients as (n_grid-1)^2 doubles */
int orc_fd_biharmonic(int n_grid, int levels, orc_mat** a, orc_mat** mass, orc_mat** transfers, double* b,
                      double* u_ref, double* h) {
  return guard([&] {
    FdProblem p = fd_biharmonic(n_grid, levels);
    from_vec(p.system.b.values, b);
    from_vec(*p.system.reference, u_ref);
    *h = p.h;
    for (size_t l = 0; l < p.transfers.size(); ++l) transfers[l] = new orc_mat{std::move(p.transfers[l])};
    *a = new orc_mat{std::move(p.system.A)};
    *mass = new orc_mat{std::move(p.system.mass)};
  });
}

/* matrix_io.cpp: read_matrix / write_matrix / read_vector / write_vector; an
 * IoError's line number is returned through orc_last_pivot() */
int orc_read_matrix(const char* path, orc_mat** out) {
  try {
    *out = new orc_mat{read_matrix(path)};
    return ORC_OK;
  } catch (const IoError& e) {
    g_err = e.what();
    g_pivot = e.line;
    return -5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_ERUNTIME;
  }
}
int orc_write_matrix(const char* path, const orc_mat* a) {
  return guard([&] { write_matrix(path, a->m); });
}
int orc_write_vector(const char* path, int n, const double* v) {
  return guard([&] { write_vector(path, to_vec(v, n)); });
}
int orc_read_vector(const char* path, int cap, double* v, int* n) {
  try {
    const Vector r = read_vector(path);
    *n = static_cast<int>(r.size());
    if (r.size() <= cap) from_vec(r, v);
    return ORC_OK;
  } catch (const IoError& e) {
    g_err = e.what();
    g_pivot = e.line;
    return -5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ORC_ERUNTIME;
  }
}

}  // extern "C"
