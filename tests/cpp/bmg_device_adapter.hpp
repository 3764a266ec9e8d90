// bmg_device_adapter.hpp -- the reference-side binding a blockmg maintainer adds
// to run the hot path on a B200 (quoted in INTEGRATION.md; compiled next to the
// reference's own declarations by tests/cpp/adapter_compile_test.cpp).
//
// It converts the reference's BlockSparseMatrix (rows of std::map<int,
// DenseBlock>, row-major blocks, ascending columns: block_matrix.hpp:26-70) to
// the C ABI's block-CSR and maps setup / v_cycle (multilevel.hpp:59-65) onto
// their device counterparts in namespace bmg::cuda.
#pragma once

#include <algorithm>
#include <utility>
#include <vector>

#include "bmg/blockmg.hpp"

namespace bmg_adapter {

inline bmg::cuda::HostBsr to_device_layout(const bmg::BlockSparseMatrix& a) {
  bmg::cuda::HostBsr h;
  h.rows = bmg::cuda::BlockLayout(a.row_layout().sizes());
  h.cols = bmg::cuda::BlockLayout(a.col_layout().sizes());
  h.symmetric = a.symmetric();
  for (int i = 0; i < a.block_rows(); ++i) {
    for (const auto& [j, blk] : a.row(i)) {  // ascending j (std::map)
      h.col_idx.push_back(j);
      h.vals.insert(h.vals.end(), blk.data(), blk.data() + blk.size());  // row-major
    }
    h.row_ptr.push_back((int64_t)h.col_idx.size());
  }
  return h;
}

inline bmg::cuda::SetupParams to_device_params(const bmg::SetupParams& p) {
  bmg::cuda::SetupParams q;
  q.t_max = p.t_max;
  q.tau = p.tau;
  q.nest = p.nest;
  q.kind = static_cast<bmg::cuda::SmootherKind>(static_cast<int>(p.kind));  // same enumerator order
  q.richardson_omega = p.richardson_omega;
  q.first_kind_fraction = p.first_kind_fraction;
  q.lanczos_iters = p.lanczos_iters;
  q.lanczos_safety = p.lanczos_safety;
  q.seed = p.seed;
  q.coarse_dim_cap = p.coarse_dim_cap;
  return q;
}

// bmg::setup(a_finest, transfers, params), built on the device
inline bmg::cuda::Hierarchy setup(bmg::cuda::Context& ctx, const bmg::BlockSparseMatrix& a_finest,
                                  const std::vector<bmg::BlockSparseMatrix>& transfers,
                                  const bmg::SetupParams& params) {
  bmg::cuda::DeviceMatrix a(ctx, to_device_layout(a_finest));
  std::vector<bmg::cuda::DeviceMatrix> p;
  p.reserve(transfers.size());
  for (const auto& t : transfers) p.emplace_back(ctx, to_device_layout(t));
  return bmg::cuda::setup(a, std::move(p), to_device_params(params));  // a, p may go away now
}

// bmg::v_cycle(h, spec, h.finest(), b, x) on host vectors
inline void v_cycle(const bmg::cuda::Hierarchy& h, const bmg::CycleSpec& spec, const bmg::Vector& b,
                    bmg::Vector& x) {
  std::vector<double> bh(b.data(), b.data() + b.size()), xh(x.data(), x.data() + x.size());
  bmg::cuda::v_cycle(h, bmg::cuda::CycleSpec{spec.k_pre, spec.k_post}, bh, xh);
  std::copy(xh.begin(), xh.end(), x.data());
}

}  // namespace bmg_adapter
