// reference_api.hpp -- Eigen-free stand-in DECLARATIONS of the reference's
// public types (namespace bmg, /root/reference/proj/include/blockmg/*.hpp) for
// the compile test of the adapter (tests/cpp/adapter_compile_test.cpp).
//
// Only the names and member signatures an adapter touches are declared, so a
// translation unit can include them next to include/bmg/blockmg.hpp exactly as a
// reference build would include the real headers: if the facade redeclared any
// of these names in namespace bmg, this TU would not compile.  Nothing here is
// defined or linked; Eigen's dense types are replaced by minimal row-major
// stand-ins with the members the adapter uses (data(), size()).
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

namespace bmg {

// types.hpp: Eigen row-major dynamic matrix / VectorXd
struct DenseBlock {
  std::vector<double> v;
  long r = 0, c = 0;
  const double* data() const { return v.data(); }
  long size() const { return r * c; }
};
struct Vector {
  std::vector<double> v;
  const double* data() const { return v.data(); }
  double* data() { return v.data(); }
  long size() const { return (long)v.size(); }
};

// block_layout.hpp:8-28
class BlockLayout {
 public:
  BlockLayout() = default;
  explicit BlockLayout(std::vector<int> sizes);
  int blocks() const;
  int dim() const;
  const std::vector<int>& sizes() const;
  bool operator==(const BlockLayout& other) const;
};

// block_matrix.hpp:26-70
class BlockSparseMatrix {
 public:
  using Row = std::map<int, DenseBlock>;
  const BlockLayout& row_layout() const;
  const BlockLayout& col_layout() const;
  bool symmetric() const;
  int block_rows() const;
  const Row& row(int i) const;
};

// small_cholesky.hpp:10-13
struct NotPositiveDefinite : std::runtime_error {
  int pivot;
  explicit NotPositiveDefinite(int pivot_, const std::string& context = {});
};

// chebyshev.hpp:10-18
enum class SmootherKind { Richardson, ChebFirst, ChebFourth };
struct SmootherSpec {
  SmootherKind kind = SmootherKind::ChebFourth;
  int degree = 1;
  double alpha = 0.0, beta = 1.0, omega = 1.0;
};
template <class OpA, class OpM>
Vector cheb_fourth_apply(const OpA& a, const OpM& m, const Vector& b, Vector x, double beta, int k);

// fsai.hpp:56-66
struct NestedFsai {
  BlockLayout layout;
  Vector apply(const Vector& r) const;
};

// multilevel.hpp:13-65
struct CycleSpec {
  int k_pre = 1;
  int k_post = 1;
  static CycleSpec vkk(int k) { return {k, k}; }
};
struct Level {
  BlockSparseMatrix A, P;
  NestedFsai fsai;
  SmootherSpec smoother;
};
struct Hierarchy {
  std::vector<Level> levels;
  int finest() const { return (int)levels.size() - 1; }
};
struct SetupParams {
  int t_max = 4;
  double tau = 1.0;
  int nest = 0;
  SmootherKind kind = SmootherKind::ChebFourth;
  double richardson_omega = 1.0;
  double first_kind_fraction = 1.0 / 30.0;
  int lanczos_iters = 100;
  double lanczos_safety = 1.01;
  std::uint64_t seed = 42;
  int coarse_dim_cap = 5000;
};
Hierarchy setup(const BlockSparseMatrix& a_finest, std::vector<BlockSparseMatrix> transfers,
                const SetupParams& params);
void v_cycle(const Hierarchy& h, const CycleSpec& spec, int level, const Vector& b, Vector& x);

// kernels.hpp:15,19
void spmv(const BlockSparseMatrix& a, const Vector& x, Vector& y);
void spmv_transpose(const BlockSparseMatrix& a, const Vector& x, Vector& y);

}  // namespace bmg
