// adapter_compile_test.cpp -- compile-only check (tests/test_facade_compile.py):
// the reference's public declarations (namespace bmg; Eigen-free stand-ins in
// ref_mock/) and the device facade (namespace bmg::cuda) in ONE translation
// unit, the adapter of INTEGRATION.md on top, and the reference-shaped
// templates instantiated with the reference's operator-callable protocol.
#include "blockmg/reference_api.hpp"  // reference declarations (namespace bmg)
#include "bmg/blockmg.hpp"            // this repo (namespace bmg::cuda)
#include "bmg_device_adapter.hpp"     // the binding INTEGRATION.md quotes

namespace {

// a caller written against the reference: names resolve in namespace bmg
[[maybe_unused]] void reference_caller(const bmg::BlockSparseMatrix& a, const std::vector<bmg::BlockSparseMatrix>& t,
                                       const bmg::Vector& b, bmg::Vector& x) {
  bmg::SetupParams params;
  params.t_max = 1;
  bmg::Hierarchy h = bmg::setup(a, t, params);
  bmg::v_cycle(h, bmg::CycleSpec::vkk(3), h.finest(), b, x);
}

// the same caller moved to the device through the adapter
[[maybe_unused]] void device_caller(const bmg::BlockSparseMatrix& a, const std::vector<bmg::BlockSparseMatrix>& t,
                                    const bmg::Vector& b, bmg::Vector& x) {
  bmg::cuda::Context ctx(0);
  bmg::SetupParams params;
  params.t_max = 1;
  bmg::cuda::Hierarchy h = bmg_adapter::setup(ctx, a, t, params);
  bmg_adapter::v_cycle(h, bmg::CycleSpec::vkk(3), b, x);
}

// cheb_fourth_apply(a, m, b, Vector x, beta, k) -> Vector (chebyshev.hpp:48-50) with
// device handles, with generic callables, and apply_smoother / NestedFsai::apply by value
[[maybe_unused]] void reference_shaped_calls(const bmg::cuda::DeviceMatrix& A, const bmg::cuda::NestedFsai& M,
                                             const bmg::cuda::DeviceVector& b, const bmg::cuda::DeviceVector& x0) {
  bmg::cuda::DeviceVector x1 = bmg::cuda::cheb_fourth_apply(A, M, b, x0, 10.0, 3);
  auto a_op = [&](const bmg::cuda::DeviceVector& in, bmg::cuda::DeviceVector& out) { bmg::cuda::spmv(A, in, out); };
  auto m_op = [&](const bmg::cuda::DeviceVector& in, bmg::cuda::DeviceVector& out) { M.apply(in, out); };
  bmg::cuda::DeviceVector x2 = bmg::cuda::cheb_fourth_apply(a_op, m_op, b, x0, 10.0, 3);
  bmg::cuda::SmootherSpec s;
  s.kind = bmg::cuda::SmootherKind::ChebFirst;
  s.alpha = 1.0 / 3.0;
  s.beta = 10.0;
  bmg::cuda::DeviceVector x3 = bmg::cuda::apply_smoother(s, 2, a_op, m_op, b, std::move(x1));
  s.kind = bmg::cuda::SmootherKind::Richardson;
  bmg::cuda::DeviceVector x4 = bmg::cuda::apply_smoother(s, 2, A, M, b, x2);
  bmg::cuda::DeviceVector z = M.apply(x3);                  // Vector NestedFsai::apply(const Vector&) const
  bmg::cuda::DeviceVector w = M.apply_transformed(A, x4);  // fsai.hpp:65
  (void)z;
  (void)w;
}

}  // namespace
