// facade_test.cpp -- drives the C++ facade (include/bmg/blockmg.hpp) the way a
// reference caller would: build a problem, setup, v_cycle / solve, and the
// reference's exception types.  Exit code 0 = pass.  Needs a B200.
#include <cmath>
#include <cstdio>
#include <vector>

#include "bmg/blockmg.hpp"

static bmg::HostBsr stencil(int n, int m) {
  int64_t nnzb = 0;
  bmg::check(bmg_gen_stencil(2, n, 2, m, 0, 0.01, 0, -1, &nnzb, nullptr, nullptr, nullptr));
  bmg::HostBsr h;
  h.rows = h.cols = bmg::BlockLayout::uniform(n * n, m);
  h.row_ptr.resize((size_t)n * n + 1);
  h.col_idx.resize((size_t)nnzb);
  h.vals.resize((size_t)nnzb * m * m);
  bmg::check(bmg_gen_stencil(2, n, 2, m, 0, 0.01, 0, -1, &nnzb, h.row_ptr.data(), h.col_idx.data(), h.vals.data()));
  h.symmetric = true;
  return h;
}
static bmg::HostBsr prolong(int nf, int m, int level) {
  int64_t nnzb = 0;
  bmg::check(bmg_gen_prolongation(2, nf, m, 0, level, 0, -1, &nnzb, nullptr, nullptr, nullptr));
  bmg::HostBsr h;
  h.rows = bmg::BlockLayout::uniform(nf * nf, m);
  h.cols = bmg::BlockLayout::uniform(nf * nf / 4, m);
  h.row_ptr.resize((size_t)nf * nf + 1);
  h.col_idx.resize((size_t)nnzb);
  h.vals.resize((size_t)nnzb * m * m);
  bmg::check(bmg_gen_prolongation(2, nf, m, 0, level, 0, -1, &nnzb, h.row_ptr.data(), h.col_idx.data(), h.vals.data()));
  return h;
}

#define EXPECT(c)                                            \
  do {                                                       \
    if (!(c)) {                                              \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                              \
    }                                                        \
  } while (0)

int main() {
  bmg::Context ctx(0);
  const int n = 32, m = 10;
  bmg::HostBsr ah = stencil(n, m);
  bmg::DeviceMatrix A(ctx, ah);
  bmg::DeviceMatrix P2(ctx, prolong(32, m, 2)), P1(ctx, prolong(16, m, 1));
  bmg::SetupParams prm;
  prm.t_max = 1;
  prm.coarse_dim_cap = 1 << 30;
  bmg::Hierarchy h = bmg::setup(A, {&P1, &P2}, prm);
  EXPECT(h.levels() == 3);
  EXPECT(h.beta(2) > 0.0 && h.beta(1) > 0.0);
  std::vector<double> b((size_t)ah.rows.dim());
  bmg::check(bmg_gen_normal(0, 0, (int64_t)b.size(), b.data()));
  bmg::DeviceVector bv(ctx, b), xv(ctx, (int64_t)b.size());
  auto rep = bmg::solve(h, bmg::CycleSpec::vkk(3), bv, xv, 5e-2, 200);
  EXPECT(rep.status == 0);
  EXPECT(rep.residual.back() < 5e-2 * rep.residual.front());
  // host-buffer v_cycle matches the device-vector one bitwise
  std::vector<double> x1(b.size(), 0.0);
  bmg::v_cycle(h, bmg::CycleSpec::vkk(3), b, x1);
  bmg::DeviceVector x2(ctx, (int64_t)b.size());
  bmg::v_cycle(h, bmg::CycleSpec::vkk(3), bv, x2);
  EXPECT(x1 == x2.download());
  // exception mapping (kernels.cpp:9-11, small_cholesky.cpp:19)
  bool threw = false;
  try {
    bmg::DeviceVector bad(ctx, 3);
    bmg::spmv(A, bad, xv);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
  bmg::HostBsr ind;
  ind.rows = ind.cols = bmg::BlockLayout({2});
  ind.row_ptr = {0, 1};
  ind.col_idx = {0};
  ind.vals = {1.0, 2.0, 2.0, 1.0};
  ind.symmetric = true;
  bmg::DeviceMatrix I(ctx, ind);
  threw = false;
  try {
    bmg::build_fsai_static(I);
  } catch (const bmg::NotPositiveDefinite& e) {
    threw = e.pivot == 1;
  }
  EXPECT(threw);
  std::printf("facade ok: %d cycles, rho %.3e\n", rep.iterations, rep.residual.back() / rep.residual.front());
  return 0;
}
