// blockmg.hpp -- header-only C++ facade over the C ABI (include/bmg_cuda.h).
//
// Mirrors the reference's hot-path interface (/root/reference/proj/include/blockmg):
// the same function names, argument meaning and exception types, so a caller of
// the reference's spmv / nested_build / cheb_fourth_apply / lanczos_lambda_max /
// setup / v_cycle can switch by replacing the matrix type with a device handle.
//
// Everything lives in namespace bmg::cuda, so this header can be included in
// the same translation unit as the reference's own headers (namespace bmg):
// bmg::BlockLayout / bmg::Hierarchy stay the reference's, bmg::cuda::* are the
// device counterparts (tests/cpp/ref_mock + tests/cpp/adapter_compile_test.cpp
// compile both side by side).  The reference's exception types are thrown
// (std::invalid_argument, std::out_of_range, std::runtime_error); the two the
// reference defines itself (NotPositiveDefinite, IoError) have device
// counterparts here with the same members (pivot, line).
//   BlockLayout              block_layout.hpp:8-28
//   NotPositiveDefinite      small_cholesky.hpp:10-13
//   spmv / spmv_transpose    kernels.hpp:15,19
//   galerkin_coarsen         multilevel.hpp:50
//   nested_build             fsai.hpp:68   (NestedFsai::apply fsai.hpp:62)
//   cheb_fourth_apply        chebyshev.hpp:48
//   lanczos_lambda_max       multilevel.hpp:53
//   SetupParams / CycleSpec  multilevel.hpp:13-19, 35-47
//   setup / v_cycle          multilevel.hpp:59-65
// Values are FP64; every object lives on one B200 (sm_100a).  No CPU fallback.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../bmg_cuda.h"

namespace bmg {
namespace cuda {

struct NotPositiveDefinite : std::runtime_error {
  int pivot;
  NotPositiveDefinite(int p, const std::string& msg) : std::runtime_error(msg), pivot(p) {}
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {  // matrix_io.hpp:10-13
  int line;
  IoError(int l, const std::string& msg) : std::runtime_error(msg), line(l) {}
};

inline void check(int status) {
  if (status == BMG_OK) return;
  const std::string msg = bmg_last_error();
  switch (status) {
    case BMG_EINVAL: throw std::invalid_argument(msg);
    case BMG_ERANGE: throw std::out_of_range(msg);
    case BMG_ENOTSPD: throw NotPositiveDefinite(bmg_last_pivot(), msg);
    case BMG_ECUDA: throw CudaError(msg);
    case BMG_EIO: throw IoError(bmg_last_pivot(), msg);
    default: throw std::runtime_error(msg);
  }
}

enum class SmootherKind { Richardson = 0, ChebFirst = 1, ChebFourth = 2 };  // chebyshev.hpp:10

// Partition of {0..N-1} into blocks of sizes m_i >= 1 (block_layout.hpp:8-28).
class BlockLayout {
 public:
  BlockLayout() = default;
  explicit BlockLayout(std::vector<int> sizes) : sizes_(std::move(sizes)) {
    for (int m : sizes_) {
      if (m < 1) throw std::invalid_argument("BlockLayout: block sizes must be >= 1");
      offsets_.push_back(dim_);
      dim_ += m;
    }
  }
  static BlockLayout scalar(int n) { return uniform(n, 1); }
  static BlockLayout uniform(int n, int m) { return BlockLayout(std::vector<int>((size_t)n, m)); }
  int blocks() const { return (int)sizes_.size(); }
  int dim() const { return dim_; }
  int size(int i) const { return sizes_[(size_t)i]; }
  int offset(int i) const { return offsets_[(size_t)i]; }
  const std::vector<int>& sizes() const { return sizes_; }
  bool operator==(const BlockLayout& o) const { return sizes_ == o.sizes_; }

 private:
  std::vector<int> sizes_, offsets_;
  int dim_ = 0;
};

class Context {
 public:
  explicit Context(int device = 0) { check(bmg_ctx_create(device, &h_)); }
  ~Context() {
    if (h_) bmg_ctx_destroy(h_);
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  bmg_ctx* get() const { return h_; }
  void set_stream(void* s) { check(bmg_ctx_set_stream(h_, s)); }
  void sync() { check(bmg_ctx_sync(h_)); }

 private:
  bmg_ctx* h_ = nullptr;
};

// Block-CSR host arrays: rows ascending, columns strictly ascending per row,
// blocks row-major (the reference's DenseBlock, types.hpp:9).
struct HostBsr {
  BlockLayout rows, cols;
  std::vector<int64_t> row_ptr{0};
  std::vector<int32_t> col_idx;
  std::vector<double> vals;
  bool symmetric = false;
};

class DeviceVector;

class DeviceMatrix {
 public:
  DeviceMatrix(Context& ctx, const HostBsr& h) : rows_(h.rows), cols_(h.cols) {
    check(bmg_bsr_create(ctx.get(), h.rows.blocks(), h.rows.sizes().data(), h.cols.blocks(),
                         h.cols.sizes().data(), h.row_ptr.data(), h.col_idx.data(), h.vals.data(),
                         h.symmetric ? BMG_SYMMETRIC : 0, &h_));
  }
  DeviceMatrix(bmg_bsr* borrowed, BlockLayout r, BlockLayout c)
      : h_(borrowed), rows_(std::move(r)), cols_(std::move(c)), owned_(false) {}
  ~DeviceMatrix() {
    if (h_ && owned_) bmg_bsr_destroy(h_);
  }
  DeviceMatrix(DeviceMatrix&& o) noexcept : h_(o.h_), rows_(o.rows_), cols_(o.cols_), owned_(o.owned_) {
    o.h_ = nullptr;
  }
  DeviceMatrix(const DeviceMatrix&) = delete;
  const bmg_bsr* get() const { return h_; }
  const BlockLayout& row_layout() const { return rows_; }
  const BlockLayout& col_layout() const { return cols_; }
  // the operator callable of the reference's smoothers: a(x, y) is y = A x
  inline void operator()(const DeviceVector& x, DeviceVector& y) const;

 private:
  friend DeviceMatrix galerkin_coarsen(const DeviceMatrix&, const DeviceMatrix&);
  bmg_bsr* h_ = nullptr;
  BlockLayout rows_, cols_;
  bool owned_ = true;
};

// A device FP64 vector with the reference's Vector value semantics
// (types.hpp:10): copies are device copies, moves transfer the buffer.
class DeviceVector {
 public:
  DeviceVector(Context& ctx, int64_t n) { check(bmg_vec_create(ctx.get(), n, &h_)); }
  DeviceVector(Context& ctx, const std::vector<double>& v) : DeviceVector(ctx, (int64_t)v.size()) { upload(v); }
  // a zero vector of o's length on o's context (Vector r(x.size()))
  static DeviceVector zeros_like(const DeviceVector& o) {
    bmg_vec* h = nullptr;
    check(bmg_vec_create_like(o.h_, &h));
    return DeviceVector(h);
  }
  ~DeviceVector() {
    if (h_) bmg_vec_destroy(h_);
  }
  DeviceVector(const DeviceVector& o) : h_(nullptr) {
    check(bmg_vec_create_like(o.h_, &h_));
    check(bmg_vec_copy(o.h_, h_));
  }
  DeviceVector(DeviceVector&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  DeviceVector& operator=(const DeviceVector& o) {
    if (this != &o) {
      if (size() != o.size()) {
        DeviceVector t(o);
        std::swap(h_, t.h_);
      } else {
        check(bmg_vec_copy(o.h_, h_));
      }
    }
    return *this;
  }
  DeviceVector& operator=(DeviceVector&& o) noexcept {
    std::swap(h_, o.h_);
    return *this;
  }
  int64_t size() const { return h_ ? bmg_vec_size(h_) : 0; }
  void upload(const std::vector<double>& v) { check(bmg_vec_upload(h_, v.data())); }
  std::vector<double> download() const {
    std::vector<double> out((size_t)bmg_vec_size(h_));
    check(bmg_vec_download(h_, out.data()));
    return out;
  }
  bmg_vec* get() const { return h_; }

 private:
  explicit DeviceVector(bmg_vec* h) : h_(h) {}
  bmg_vec* h_ = nullptr;
};

// z = alpha x + beta y with separately rounded products (the reference's Eigen
// vector expressions, see bmg_vec_axpby); z may alias x or y
inline void axpby(double alpha, const DeviceVector& x, double beta, const DeviceVector& y, DeviceVector& z) {
  check(bmg_vec_axpby(alpha, x.get(), beta, y.get(), z.get()));
}

// y = A x (kernels.hpp:15); y = A^T x (kernels.hpp:19)
inline void spmv(const DeviceMatrix& a, const DeviceVector& x, DeviceVector& y) {
  check(bmg_spmv(a.get(), x.get(), y.get()));
}
inline void spmv_batch(const DeviceMatrix& a, int nrhs, const DeviceVector& x, DeviceVector& y) {
  check(bmg_spmv_batch(a.get(), nrhs, x.get(), y.get()));
}
inline void spmv_transpose(const DeviceMatrix& a, const DeviceVector& x, DeviceVector& y) {
  check(bmg_spmv_t(a.get(), x.get(), y.get()));
}

inline void DeviceMatrix::operator()(const DeviceVector& x, DeviceVector& y) const { spmv(*this, x, y); }

// P^T A P, symmetrised (multilevel.hpp:50)
inline DeviceMatrix galerkin_coarsen(const DeviceMatrix& a, const DeviceMatrix& p) {
  bmg_bsr* out = nullptr;
  check(bmg_galerkin(a.get(), p.get(), &out));
  DeviceMatrix m(out, p.col_layout(), p.col_layout());
  m.owned_ = true;
  return m;
}

// Block-FSAI, M = G^T G on the device (NestedFsai, fsai.hpp:56-66)
class NestedFsai {
 public:
  explicit NestedFsai(bmg_fsai* h) : h_(h) {}
  ~NestedFsai() {
    if (h_) bmg_fsai_destroy(h_);
  }
  NestedFsai(NestedFsai&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  NestedFsai(const NestedFsai&) = delete;
  // Vector apply(const Vector& r) const -- M r (fsai.hpp:62)
  DeviceVector apply(const DeviceVector& r) const {
    DeviceVector z = DeviceVector::zeros_like(r);
    apply(r, z);
    return z;
  }
  // Vector apply_transformed(a, x) const -- L^-1 F A F^T L^-T x (fsai.hpp:65)
  DeviceVector apply_transformed(const DeviceMatrix& a, const DeviceVector& x) const {
    DeviceVector y = DeviceVector::zeros_like(x);
    check(bmg_fsai_apply_transformed(h_, a.get(), x.get(), y.get()));
    return y;
  }
  void apply(const DeviceVector& r, DeviceVector& z) const { check(bmg_fsai_apply(h_, r.get(), z.get())); }
  // the preconditioner callable of the reference's smoothers: m(r, z) is z = M r
  void operator()(const DeviceVector& r, DeviceVector& z) const { apply(r, z); }
  const bmg_fsai* get() const { return h_; }

 private:
  bmg_fsai* h_ = nullptr;
};

inline NestedFsai nested_build(const DeviceMatrix& a, int t_max, double tau, int n_levels) {
  bmg_fsai* out = nullptr;
  check(bmg_fsai_build(a.get(), BMG_FSAI_ADAPTIVE, t_max, tau, n_levels, &out));
  return NestedFsai(out);
}
inline NestedFsai build_fsai_static(const DeviceMatrix& a) {  // build_fsai(A, LowerPattern::from_matrix(A))
  bmg_fsai* out = nullptr;
  check(bmg_fsai_build(a.get(), BMG_FSAI_STATIC_LOWER, 1, 1.0, 0, &out));
  return NestedFsai(out);
}

inline double fourth_kind_mu(int n) { return (2.0 * n + 1.0) / (2.0 * n + 3.0); }  // chebyshev.hpp:42

// Vector cheb_fourth_apply(a, m, b, Vector x, beta, k) (chebyshev.hpp:48-69)
// for any operator callables a(x, t), m(r, z) on device vectors, step for step
// as the reference (separately rounded vector updates, closed-form mu).
template <class OpA, class OpM>
DeviceVector cheb_fourth_apply(const OpA& a, const OpM& m, const DeviceVector& b, DeviceVector x, double beta,
                               int k) {
  if (!(beta > 0.0)) throw std::invalid_argument("cheb_fourth_apply: beta must be positive");
  if (k < 1) throw std::invalid_argument("cheb_fourth_apply: degree must be >= 1");
  const double d = 4.0 / beta;
  DeviceVector r = DeviceVector::zeros_like(x), p = DeviceVector::zeros_like(x), t = DeviceVector::zeros_like(x);
  a(x, t);
  axpby(1.0, b, -1.0, t, r);  // r = b - t
  m(r, p);
  double mu = fourth_kind_mu(0);
  axpby(1.0, x, d * mu, p, x);  // x += d * mu * p
  for (int i = 2; i <= k; ++i) {
    a(x, t);
    axpby(1.0, b, -1.0, t, r);
    m(r, t);
    axpby(mu * mu, p, 1.0, t, p);  // p = mu * mu * p + t
    mu = fourth_kind_mu(i - 1);
    axpby(1.0, x, d * mu, p, x);
  }
  return x;
}
// The device operators themselves: the same recurrence as fused streaming
// passes (residual, G, G^T + update epilogue; bmg_cheb4_apply), bitwise equal
// to the generic template above on the same operands.
inline DeviceVector cheb_fourth_apply(const DeviceMatrix& a, const NestedFsai& m, const DeviceVector& b,
                                      DeviceVector x, double beta, int k) {
  check(bmg_cheb4_apply(a.get(), m.get(), b.get(), x.get(), beta, k));
  return x;
}
// in-place form (no copy of x)
inline void cheb_fourth_apply_inplace(const DeviceMatrix& a, const NestedFsai& m, const DeviceVector& b,
                                      DeviceVector& x, double beta, int k) {
  check(bmg_cheb4_apply(a.get(), m.get(), b.get(), x.get(), beta, k));
}

// cheb_first_apply (chebyshev.hpp:74-98) and richardson_apply (:101-115) for
// generic callables, step for step as the reference
template <class OpA, class OpM>
DeviceVector cheb_first_apply(const OpA& a, const OpM& m, const DeviceVector& b, DeviceVector x, double alpha,
                              double beta, int k) {
  if (!(alpha > 0.0) || !(alpha < beta))
    throw std::invalid_argument("cheb_first_apply: interval must satisfy 0 < alpha < beta");
  if (k < 1) throw std::invalid_argument("cheb_first_apply: degree must be >= 1");
  const double c = 0.5 * (alpha + beta);
  const double d = 0.5 * (beta - alpha);
  DeviceVector r = DeviceVector::zeros_like(x), p = DeviceVector::zeros_like(x), t = DeviceVector::zeros_like(x);
  a(x, t);
  axpby(1.0, b, -1.0, t, r);
  m(r, p);
  double omega = 1.0 / c;
  double psi = 0.5 * (d * omega) * (d * omega);
  axpby(1.0, x, omega, p, x);
  for (int i = 2; i <= k; ++i) {
    a(x, t);
    axpby(1.0, b, -1.0, t, r);
    m(r, t);
    axpby(1.0, t, psi, p, p);  // p = t + psi * p
    omega = 1.0 / (c - psi / omega);
    psi = 0.25 * (d * omega) * (d * omega);
    axpby(1.0, x, omega, p, x);
  }
  return x;
}
template <class OpA, class OpM>
DeviceVector richardson_apply(const OpA& a, const OpM& m, const DeviceVector& b, DeviceVector x, double omega,
                              int k) {
  if (k < 1) throw std::invalid_argument("richardson_apply: step count must be >= 1");
  DeviceVector r = DeviceVector::zeros_like(x), t = DeviceVector::zeros_like(x);
  for (int i = 0; i < k; ++i) {
    a(x, t);
    axpby(1.0, b, -1.0, t, r);
    m(r, t);
    axpby(1.0, x, omega, t, x);
  }
  return x;
}

struct SmootherSpec {  // chebyshev.hpp:12-18
  SmootherKind kind = SmootherKind::ChebFourth;
  int degree = 1;
  double alpha = 0.0, beta = 1.0, omega = 1.0;
};
// Vector apply_smoother(spec, degree, a, m, b, Vector x) (chebyshev.hpp:117-129)
template <class OpA, class OpM>
DeviceVector apply_smoother(const SmootherSpec& s, int degree, const OpA& a, const OpM& m, const DeviceVector& b,
                            DeviceVector x) {
  switch (s.kind) {
    case SmootherKind::Richardson: return richardson_apply(a, m, b, std::move(x), s.omega, degree);
    case SmootherKind::ChebFirst: return cheb_first_apply(a, m, b, std::move(x), s.alpha, s.beta, degree);
    case SmootherKind::ChebFourth: return cheb_fourth_apply(a, m, b, std::move(x), s.beta, degree);
  }
  throw std::logic_error("apply_smoother: unknown kind");
}
// the device operators: one fused-epilogue pass sequence (bmg_smoother_apply)
inline DeviceVector apply_smoother(const SmootherSpec& s, int degree, const DeviceMatrix& a, const NestedFsai& m,
                                   const DeviceVector& b, DeviceVector x) {
  check(bmg_smoother_apply(a.get(), m.get(), (int)s.kind, s.alpha, s.beta, s.omega, degree, b.get(), x.get()));
  return x;
}
inline void apply_smoother_inplace(const SmootherSpec& s, int degree, const DeviceMatrix& a, const NestedFsai& m,
                                   const DeviceVector& b, DeviceVector& x) {
  check(bmg_smoother_apply(a.get(), m.get(), (int)s.kind, s.alpha, s.beta, s.omega, degree, b.get(), x.get()));
}

inline double lanczos_lambda_max(const DeviceMatrix& a, const NestedFsai& m, int iters = 100,
                                 double safety = 1.01, uint64_t seed = 42) {
  double beta = 0.0;
  check(bmg_lanczos_lambda_max(a.get(), m.get(), iters, safety, seed, &beta));
  return beta;
}

struct CycleSpec {  // multilevel.hpp:13-19
  int k_pre = 1;
  int k_post = 1;
  static CycleSpec vkk(int k) { return {k, k}; }
  static CycleSpec v2k0(int k) { return {2 * k, 0}; }
};

struct SetupParams {  // multilevel.hpp:35-47
  SmootherKind kind = SmootherKind::ChebFourth;
  double richardson_omega = 1.0;
  double first_kind_fraction = 1.0 / 30.0;
  int t_max = 4;
  double tau = 1.0;
  int nest = 0;
  int lanczos_iters = 100;
  double lanczos_safety = 1.01;
  uint64_t seed = 42;
  int coarse_dim_cap = 5000;
  bool static_pattern = false;  // lower(P(A)) instead of the adaptive chain
};

class Hierarchy {
 public:
  explicit Hierarchy(bmg_hier* h) : h_(h) {}
  ~Hierarchy() {
    if (h_) bmg_hier_destroy(h_);
  }
  Hierarchy(Hierarchy&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
  Hierarchy(const Hierarchy&) = delete;
  bmg_hier* get() const { return h_; }
  int levels() const {
    int n = 0;
    check(bmg_hier_info(h_, &n, nullptr));
    return n;
  }
  int finest() const { return levels() - 1; }
  double beta(int level) const {
    double b = 0.0;
    check(bmg_hier_beta(h_, level, &b));
    return b;
  }

 private:
  bmg_hier* h_ = nullptr;
};

// setup (multilevel.hpp:59-60): transfers[l-1] prolongates level l-1 to l
inline Hierarchy setup(const DeviceMatrix& a_finest, const std::vector<const DeviceMatrix*>& transfers,
                       const SetupParams& p) {
  bmg_setup_params c;
  bmg_setup_params_default(&c);
  c.t_max = p.t_max;
  c.tau = p.tau;
  c.nest = p.nest;
  c.fsai_kind = p.static_pattern ? BMG_FSAI_STATIC_LOWER : BMG_FSAI_ADAPTIVE;
  c.lanczos_iters = p.lanczos_iters;
  c.lanczos_safety = p.lanczos_safety;
  c.seed = p.seed;
  c.coarse_dim_cap = p.coarse_dim_cap;
  c.smoother_kind = (int)p.kind;
  c.richardson_omega = p.richardson_omega;
  c.first_kind_fraction = p.first_kind_fraction;
  std::vector<const bmg_bsr*> t;
  for (auto* m : transfers) t.push_back(m->get());
  bmg_hier* h = nullptr;
  check(bmg_hier_setup(a_finest.get(), (int)t.size(), t.data(), &c, &h));
  return Hierarchy(h);
}

inline Hierarchy setup(const DeviceMatrix& a_finest, std::initializer_list<const DeviceMatrix*> transfers,
                       const SetupParams& p) {
  return setup(a_finest, std::vector<const DeviceMatrix*>(transfers), p);
}
// the reference's signature, transfers by value (multilevel.hpp:59-60); the
// hierarchy keeps what it needs alive, so the caller's matrices may go away
inline Hierarchy setup(const DeviceMatrix& a_finest, std::vector<DeviceMatrix> transfers, const SetupParams& p) {
  std::vector<const DeviceMatrix*> t;
  for (auto& m : transfers) t.push_back(&m);
  return setup(a_finest, t, p);
}

// v_cycle on the finest level (multilevel.hpp:65); x is updated in place
inline void v_cycle(const Hierarchy& h, const CycleSpec& spec, const DeviceVector& b, DeviceVector& x) {
  check(bmg_vcycle(h.get(), spec.k_pre, spec.k_post, b.get(), x.get()));
}
// the reference signature: v_cycle(h, spec, level, b, x) (multilevel.hpp:65)
inline void v_cycle(const Hierarchy& h, const CycleSpec& spec, int level, const DeviceVector& b, DeviceVector& x) {
  check(bmg_vcycle_level(h.get(), spec.k_pre, spec.k_post, level, b.get(), x.get()));
}
inline void v_cycle(const Hierarchy& h, const CycleSpec& spec, const std::vector<double>& b,
                    std::vector<double>& x) {
  check(bmg_vcycle_host(h.get(), spec.k_pre, spec.k_post, b.data(), x.data()));
}

// K right-hand sides per cycle (K = 1, 2, 4, 8), interleaved per scalar row
// (b[i*K + v]); each RHS bitwise equal to v_cycle on it alone
inline void v_cycle_batch(const Hierarchy& h, const CycleSpec& spec, int nrhs, const DeviceVector& b,
                          DeviceVector& x) {
  check(bmg_vcycle_batch(h.get(), spec.k_pre, spec.k_post, nrhs, b.get(), x.get()));
}
inline void v_cycle_batch(const Hierarchy& h, const CycleSpec& spec, int nrhs, const std::vector<double>& b,
                          std::vector<double>& x) {
  check(bmg_vcycle_batch_host(h.get(), spec.k_pre, spec.k_post, nrhs, b.data(), x.data()));
}

struct SolveReport {  // residual-history analogue of RateReport (experiments.hpp:17-27)
  std::vector<double> residual;
  int iterations = 0;
  int status = 0;  // 0 converged, 1 max_iter, 2 diverged
};
inline SolveReport solve(const Hierarchy& h, const CycleSpec& spec, const DeviceVector& b, DeviceVector& x,
                         double tol, int max_iter) {
  SolveReport r;
  r.residual.assign((size_t)max_iter + 1, 0.0);
  check(bmg_solve(h.get(), spec.k_pre, spec.k_post, b.get(), x.get(), tol, max_iter, r.residual.data(),
                  &r.iterations, &r.status));
  r.residual.resize((size_t)r.iterations + 1);
  return r;
}

// RateReport / measure_rates (experiments.hpp:15-33, experiments.cpp:15-67); the
// assembled system is passed as its parts (mass matrix, b, reference solution)
enum class SolveStatus { Converged = 0, MaxIter = 1, Diverged = 2 };
struct RateReport {
  double rho_l2 = 0.0, rho_a = 0.0, rho_r = 0.0;
  int iterations = 0;
  SolveStatus status = SolveStatus::Converged;
  int blowup_iteration = -1;
  std::vector<double> l2_sq, energy_sq, residual;
};
inline RateReport measure_rates(const Hierarchy& h, const DeviceMatrix& mass, const DeviceVector& b,
                                const DeviceVector& u_ref, const CycleSpec& spec, std::uint64_t seed, double tol,
                                int max_iter) {
  RateReport r;
  r.l2_sq.assign((size_t)max_iter + 1, 0.0);
  r.energy_sq.assign((size_t)max_iter + 1, 0.0);
  r.residual.assign((size_t)max_iter + 1, 0.0);
  int st = 0;
  double rates[3];
  check(bmg_measure_rates(h.get(), mass.get(), b.get(), u_ref.get(), spec.k_pre, spec.k_post, seed, tol, max_iter,
                          r.l2_sq.data(), r.energy_sq.data(), r.residual.data(), &r.iterations, &st,
                          &r.blowup_iteration, rates));
  r.status = static_cast<SolveStatus>(st);
  r.rho_l2 = rates[0];
  r.rho_a = rates[1];
  r.rho_r = rates[2];
  r.l2_sq.resize((size_t)r.iterations + 1);
  r.energy_sq.resize((size_t)r.iterations + 1);
  r.residual.resize((size_t)r.iterations + 1);
  return r;
}

}  // namespace cuda
}  // namespace bmg
