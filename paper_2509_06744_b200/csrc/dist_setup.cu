// dist_setup.cu -- setup (multilevel.cpp:36-75) distributed over row strips for
// systems that do not fit one GPU (BASELINE C3, C5); see the section comment.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <tuple>

#include "bmg_abi.h"
#include "hier.h"

namespace bmg {

// ============================================================================ distributed setup
// setup (multilevel.cpp:36-75) without any rank holding the whole hierarchy
// (C3 / C5 do not fit one GPU).  Each rank builds every partitioned level on an
// extended strip (own rows +- a halo of granules) with the single-device setup
// kernels -- principal submatrix, block-FSAI, chunked Galerkin -- and keeps only
// its own rows, which are exact: every kept row depends on rows inside the strip
// (the halo grows by 2x + stencil radius per level, dist_plan).  The first
// agglomerated level is gathered to rank 0, which builds the coarsest levels as
// usual.  beta of a partitioned level comes from a distributed Lanczos whose dots
// sum per-block-row partials in global row order, exactly like the single-device
// Lanczos, so the distributed hierarchy is bitwise the single-device one.
namespace kern {
__global__ void rng_symmetric_off_kernel(double* v, int64_t n, uint64_t seed, int64_t off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (uint64_t)(off + i + 1) * 0x9e3779b97f4a7c15ULL;  // rng.hpp:22-24
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    const double u = __dmul_rn(__dadd_rn((double)(z >> 11), 0.5), 0x1.0p-53);
    v[i] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
  }
}
__global__ void row_partial_dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t nrows,
                                       int m, double* __restrict__ out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nrows; s += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < m; ++q) t = __fma_rn(a[s * m + q], b[s * m + q], t);
    out[s] = t;
  }
}
__global__ void div_kernel(double* v, int64_t n, double d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __ddiv_rn(v[i], d);
}
__global__ void lupd_kernel(double* w, const double* v, const double* vp, int64_t n, double alpha, double beta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = __dsub_rn(w[i], __dmul_rn(alpha, v[i]));
    w[i] = __dsub_rn(t, __dmul_rn(beta, vp[i]));
  }
}
__global__ void gather_blocks_plain_kernel(const double* __restrict__ src, const int64_t* __restrict__ from,
                                           double* __restrict__ dst, int64_t nblk, int bs) {
  for (int64_t o = blockIdx.x; o < nblk; o += gridDim.x)
    for (int e = threadIdx.x; e < bs; e += blockDim.x) dst[o * bs + e] = src[from[o] * bs + e];
}
}  // namespace kern

struct DistPlan {
  int L = 0, world = 1, agg = 1;
  std::vector<int> nbr, gran, rad, halo;
  std::vector<std::vector<int32_t>> B, elo, ehi;  // per level
};

// Halo (granules) of one level's strip so every kept row is exact.  FSAI row i
// reads A over its pattern plus candidates: pattern radius t R after t adaptive
// steps (P0 = diag; static: the lower pattern of A, t = 1), so F / F^T own rows are
// exact with (t+1) R granules on each side; a nested factor is built on
// F A F^T (radius (2t+1) R) and needs (t+2) of its radii more.  Galerkin: coarse
// granule c reads fine granules [2c-2, 2c+3] (P support |y/2 - c| <= 1) whose A
// rows must be untruncated, so the own coarse rows are exact with h >= R + 3
// (partition rounding included).  The next level's strip is then assembled from
// its owners' exact rows (fetch_rows), so halos do not compound over levels.
static int fsai_keep(int R, const bmg_setup_params& prm) {
  const int t = prm.fsai_kind == BMG_FSAI_STATIC_LOWER ? 1 : std::max(1, prm.t_max);
  int Rq = R, keep = (t + 1) * R;
  for (int q = 0; q < prm.nest; ++q) {
    Rq = (2 * t + 1) * Rq;
    keep += (t + 2) * Rq;
  }
  return keep;
}

static DistPlan dist_plan(int L, const int32_t* nbr, const int32_t* gran, const int32_t* rad, int world, int agg,
                          const bmg_setup_params& prm) {
  if (L < 2) fail(BMG_EINVAL, "dist setup: needs at least two levels");
  if (world < 1) fail(BMG_EINVAL, "dist setup: world must be >= 1");
  DistPlan P;
  P.L = L;
  P.world = world;
  P.agg = std::max(1, std::min(agg, L - 1));
  P.nbr.assign(nbr, nbr + L);
  P.gran.resize(L);
  P.rad.resize(L);
  for (int l = 0; l < L; ++l) {
    P.gran[l] = gran ? std::max(1, gran[l]) : 1;
    P.rad[l] = std::max(1, rad[l]);
  }
  P.halo.assign(L, 0);
  for (int l = P.agg; l < L; ++l) {
    const int keep = fsai_keep(P.rad[l], prm);
    P.halo[l] = std::max(keep, P.rad[l] + 3);
  }
  P.B.assign(L, std::vector<int32_t>(world + 1, 0));
  P.elo.assign(L, std::vector<int32_t>(world, 0));
  P.ehi.assign(L, std::vector<int32_t>(world, 0));
  for (int l = 0; l < L; ++l) {
    auto& b = P.B[l];
    if (l < P.agg) {
      for (int r = 1; r <= world; ++r) b[r] = P.nbr[l];
    } else {  // equal granule counts
      const int64_t ng = (P.nbr[l] + P.gran[l] - 1) / P.gran[l];
      for (int r = 0; r <= world; ++r) b[r] = (int32_t)std::min<int64_t>(P.nbr[l], ng * r / world * P.gran[l]);
      b[world] = P.nbr[l];
    }
    for (int r = 0; r < world; ++r) {
      if (l < P.agg) {
        P.ehi[l][r] = r == 0 ? P.nbr[l] : 0;
      } else {
        const int64_t h = (int64_t)P.halo[l] * P.gran[l];
        P.elo[l][r] = (int32_t)std::max<int64_t>(0, b[r] - h);
        P.ehi[l][r] = (int32_t)std::min<int64_t>(P.nbr[l], b[r + 1] + h);
        if (b[r + 1] <= b[r]) P.elo[l][r] = P.ehi[l][r] = b[r];
      }
    }
  }
  return P;
}

// the plan's assumptions, checked on the data: A couples granules at most R apart,
// P maps fine granule y to coarse granules within 1 of y/2
static void check_support(const Bsr& a, int row0, int gran, int R, const char* what) {
  for (int i = 0; i < a.nbr; ++i) {
    const int64_t gi = (row0 + i) / gran;
    for (int64_t q = a.h_row_ptr[i]; q < a.h_row_ptr[i + 1]; ++q)
      if (std::llabs(a.h_col[q] / gran - gi) > R)
        fail(BMG_EINVAL, std::string("dist setup: ") + what + " couples granules farther apart than the radius");
  }
}
static void check_prolongation(const Bsr& p, int row0, int gran, int cgran) {
  for (int i = 0; i < p.nbr; ++i) {
    const int64_t gi = ((row0 + i) / gran) >> 1;
    for (int64_t q = p.h_row_ptr[i]; q < p.h_row_ptr[i + 1]; ++q)
      if (std::llabs(p.h_col[q] / cgran - gi) > 1)
        fail(BMG_EINVAL, "dist setup: prolongation is not a 2:1 granule coarsening");
  }
}

// rows of `a` (rows [row0, row0 + nbr), global columns) restricted to columns in
// [lo, hi), shifted by -lo: the principal submatrix when row0 = lo, nbr = hi - lo
static std::unique_ptr<Bsr> principal(const Bsr& a, int lo, int hi) {
  std::vector<int64_t> rp(a.nbr + 1, 0), from;
  std::vector<int32_t> col;
  for (int i = 0; i < a.nbr; ++i) {
    for (int64_t p = a.h_row_ptr[i]; p < a.h_row_ptr[i + 1]; ++p)
      if (a.h_col[p] >= lo && a.h_col[p] < hi) {
        col.push_back(a.h_col[p] - lo);
        from.push_back(p);
      }
    rp[i + 1] = (int64_t)col.size();
  }
  std::vector<int> csz(hi - lo, a.mr);
  auto out = make_bsr_structure(a.ctx, a.nbr, a.rsz.data(), hi - lo, csz.data(), std::move(rp), std::move(col), true);
  if (!from.empty()) {
    DBuf<int64_t> df(from.size());
    BMG_CUDA(cudaMemcpy(df.p, from.data(), from.size() * 8, cudaMemcpyHostToDevice));
    kern::gather_blocks_plain_kernel<<<(unsigned)std::min<size_t>(from.size(), (size_t)a.ctx->sms * 32), 128, 0,
                                       a.ctx->stream>>>(a.vals.p, df.p, out->vals.p, (int64_t)from.size(), a.bs);
    a.ctx->count();
    BMG_CUDA(cudaGetLastError());
    BMG_CUDA(cudaStreamSynchronize(a.ctx->stream));
  }
  return out;
}

// A phase that only some ranks run (or that may fail on some ranks) followed by
// collectives: with a transport, every rank learns whether any rank failed and all
// of them throw together instead of leaving the others blocked in a collective.
template <class F>
static void collective_phase(Ctx* ctx, bool with_comm, F&& f) {
  if (!with_comm) {
    f();
    return;
  }
  int st = BMG_OK;
  std::string msg;
  try {
    f();
  } catch (const Error& e) {
    st = e.status;
    msg = e.what();
  } catch (const std::exception& e) {
    st = BMG_ERUNTIME;
    msg = e.what();
  }
  DBuf<int32_t> flag(1);
  int32_t h = st != BMG_OK ? 1 : 0;
  BMG_CUDA(cudaMemcpy(flag.p, &h, 4, cudaMemcpyHostToDevice));
  ctx->comm->allreduce(flag.p, flag.p, 1, DType::I32, ROp::Max, ctx->stream);
  BMG_CUDA(cudaMemcpyAsync(&h, flag.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (st != BMG_OK) fail(st, msg);
  if (h) fail(BMG_ERUNTIME, "dist setup: another rank failed");
}

struct Kept {  // one rank's exact own rows of one level, global column indices
  std::unique_ptr<Bsr> A, P, R;
  std::vector<std::unique_ptr<Bsr>> F, Bt;
  std::unique_ptr<Fsai> M_whole;  // agglomerated levels (rank 0): the whole chain
  double beta = 1.0;
};

// concatenate row blocks (each with global cols) into one matrix
static std::unique_ptr<Bsr> concat_rows(Ctx* ctx, const std::vector<std::unique_ptr<Bsr>>& parts, int ncols, int m,
                                        bool sym) {
  std::vector<int64_t> rp{0};
  std::vector<int32_t> col;
  for (const auto& p : parts) {
    if (!p) continue;
    for (int i = 0; i < p->nbr; ++i) {
      for (int64_t q = p->h_row_ptr[i]; q < p->h_row_ptr[i + 1]; ++q) col.push_back(p->h_col[q]);
      rp.push_back((int64_t)col.size());
    }
  }
  const int nr = (int)rp.size() - 1;
  std::vector<int> rsz(nr, m), csz(ncols, m);
  auto out = make_bsr_structure(ctx, nr, rsz.data(), ncols, csz.data(), std::move(rp), std::move(col), sym);
  int64_t off = 0;
  for (const auto& p : parts) {
    if (!p || p->nnzb == 0) continue;
    BMG_CUDA(cudaMemcpyAsync(out->vals.p + off * out->bs, p->vals.p, (size_t)p->nnzb * p->bs * sizeof(double),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    off += p->nnzb;
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  return out;
}

// Rows [want_lo[r], want_hi[r]) for every rank r of a row-distributed matrix whose
// rank s holds exactly its own rows [B[s], B[s+1]) (global columns).
// Emulation: all ranks' pieces are here.
static std::vector<std::unique_ptr<Bsr>> fetch_rows_emulated(Ctx* ctx, const std::vector<const Bsr*>& own,
                                                             const std::vector<int32_t>& B,
                                                             const std::vector<int32_t>& want_lo,
                                                             const std::vector<int32_t>& want_hi, int ncols, int m,
                                                             bool sym) {
  const int world = (int)own.size();
  std::vector<std::unique_ptr<Bsr>> out(world);
  for (int r = 0; r < world; ++r) {
    if (want_hi[r] <= want_lo[r]) continue;
    std::vector<std::unique_ptr<Bsr>> pieces;
    for (int s = 0; s < world; ++s) {
      const int a = std::max(B[s], want_lo[r]), b = std::min(B[s + 1], want_hi[r]);
      if (b <= a) continue;
      if (!own[s]) fail(BMG_ERUNTIME, "dist setup: rows missing on their owner");
      pieces.push_back(slice_rows(*own[s], a - B[s], b - B[s], 0, ncols));
    }
    out[r] = concat_rows(ctx, pieces, ncols, m, sym);
  }
  return out;
}

// NCCL: the same exchange, this rank's piece only (row counts, then cols + values)
static std::unique_ptr<Bsr> fetch_rows_comm(Ctx* ctx, const Bsr* mine, const std::vector<int32_t>& B,
                                            const std::vector<int32_t>& want_lo, const std::vector<int32_t>& want_hi,
                                            int ncols, int m, bool sym) {
  Comm& comm = *ctx->comm;
  const int world = ctx->world, me = ctx->rank;
  const int bs = (m * m + 1) & ~1;
  const int nown = B[me + 1] - B[me];
  const int wlo = want_lo[me], nwant = std::max(0, want_hi[me] - want_lo[me]);
  if (nown > 0 && (!mine || mine->nbr != nown)) fail(BMG_ERUNTIME, "dist setup: own rows missing");
  DBuf<int64_t> mycnt(std::max(nown, 1)), rcnt(std::max(nwant, 1));
  if (nown) {
    std::vector<int64_t> c(nown);
    for (int i = 0; i < nown; ++i) c[i] = mine->h_row_ptr[i + 1] - mine->h_row_ptr[i];
    BMG_CUDA(cudaMemcpy(mycnt.p, c.data(), c.size() * 8, cudaMemcpyHostToDevice));
  }
  auto send_range = [&](int s, int& a, int& b) {  // my rows rank s wants
    a = std::max(B[me], want_lo[s]);
    b = std::min(B[me + 1], want_hi[s]);
  };
  auto recv_range = [&](int s, int& a, int& b) {  // rank s's rows I want
    a = std::max(B[s], want_lo[me]);
    b = std::min(B[s + 1], want_hi[me]);
  };
  comm.group_start();
  for (int s = 0; s < world; ++s) {
    int a, b;
    recv_range(s, a, b);
    if (b > a) {
      if (s == me)
        BMG_CUDA(cudaMemcpyAsync(rcnt.p + (a - wlo), mycnt.p + (a - B[me]), (size_t)(b - a) * 8,
                                 cudaMemcpyDeviceToDevice, ctx->stream));
      else
        comm.recv(rcnt.p + (a - wlo), b - a, DType::I64, s, ctx->stream);
    }
    send_range(s, a, b);
    if (b > a && s != me) comm.send(mycnt.p + (a - B[me]), b - a, DType::I64, s, ctx->stream);
  }
  comm.group_end();
  std::vector<int64_t> c(nwant), rp(nwant + 1, 0);
  if (nwant) BMG_CUDA(cudaMemcpyAsync(c.data(), rcnt.p, (size_t)nwant * 8, cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < nwant; ++i) rp[i + 1] = rp[i] + c[i];
  const int64_t tot = rp[nwant];
  DBuf<int32_t> dcol(std::max<int64_t>(tot, 1));
  DBuf<double> dval(std::max<int64_t>(tot * bs, 1));
  comm.group_start();
  for (int s = 0; s < world; ++s) {
    int a, b;
    recv_range(s, a, b);
    if (b > a) {
      const int64_t q0 = rp[a - wlo], q1 = rp[b - wlo];
      if (q1 > q0) {
        if (s == me) {
          const int64_t p0 = mine->h_row_ptr[a - B[me]];
          BMG_CUDA(cudaMemcpyAsync(dcol.p + q0, mine->col.p + p0, (size_t)(q1 - q0) * 4, cudaMemcpyDeviceToDevice,
                                   ctx->stream));
          BMG_CUDA(cudaMemcpyAsync(dval.p + q0 * bs, mine->vals.p + p0 * bs, (size_t)(q1 - q0) * bs * 8,
                                   cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
          comm.recv(dcol.p + q0, q1 - q0, DType::I32, s, ctx->stream);
          comm.recv(dval.p + q0 * bs, (q1 - q0) * bs, DType::F64, s, ctx->stream);
        }
      }
    }
    send_range(s, a, b);
    if (b > a && s != me) {
      const int64_t p0 = mine->h_row_ptr[a - B[me]], p1 = mine->h_row_ptr[b - B[me]];
      if (p1 > p0) {
        comm.send(mine->col.p + p0, p1 - p0, DType::I32, s, ctx->stream);
        comm.send(mine->vals.p + p0 * bs, (p1 - p0) * bs, DType::F64, s, ctx->stream);
      }
    }
  }
  comm.group_end();
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (nwant == 0) return nullptr;
  std::vector<int32_t> col(tot);
  if (tot) BMG_CUDA(cudaMemcpy(col.data(), dcol.p, (size_t)tot * 4, cudaMemcpyDeviceToHost));
  std::vector<int> rsz(nwant, m), csz(ncols, m);
  auto out = make_bsr_structure(ctx, nwant, rsz.data(), ncols, csz.data(), std::move(rp), std::move(col), sym);
  if (tot) BMG_CUDA(cudaMemcpy(out->vals.p, dval.p, (size_t)tot * bs * 8, cudaMemcpyDeviceToDevice));
  return out;
}

// One partitioned level l of one rank: extended strip of A_l (rows [elo, ehi),
// global cols) -> exact own rows of A_l, the FSAI chain, P_l, R_l, and (l > agg)
// the exact own rows of A_{l-1}.
static void dist_level(Ctx* ctx, const DistPlan& P, int r, int l, const Bsr& aext, const Bsr& pin,
                       const bmg_setup_params& prm, std::vector<Kept>& K) {
  const int agg = P.agg;
  const int lo = P.B[l][r], hi = P.B[l][r + 1], elo = P.elo[l][r], ehi = P.ehi[l][r];
  if (hi <= lo) return;
  if (aext.nbr != ehi - elo) fail(BMG_EINVAL, "dist setup: A rows do not match the plan's extended range");
  check_support(aext, elo, P.gran[l], P.rad[l], "A");
  const int prow0 = l > agg ? elo : 0;
  if (pin.nbr != (l > agg ? ehi - elo : P.nbr[l]))
    fail(BMG_EINVAL, "dist setup: P rows do not match the plan's extended range");
  check_prolongation(pin, prow0, P.gran[l], P.gran[l - 1]);
  auto aloc = principal(aext, elo, ehi);
  auto M = fsai_build(*aloc, prm.fsai_kind, prm.t_max, prm.tau, prm.nest);
  Kept& k = K[l];
  k.A = slice_rows(aext, lo - elo, hi - elo, 0, P.nbr[l]);
  for (auto& f : M->fwd) k.F.push_back(slice_rows(*f, lo - elo, hi - elo, -elo, P.nbr[l]));
  for (auto& f : M->bwd) k.Bt.push_back(slice_rows(*f, lo - elo, hi - elo, -elo, P.nbr[l]));
  k.P = slice_rows(pin, lo - prow0, hi - prow0, 0, P.nbr[l - 1]);
  if (l == agg) return;  // R_agg and A_{agg-1} are built whole on rank 0
  // P restricted to the strip's rows; coarse columns [clo, chi)
  auto pstrip = prow0 == elo ? nullptr : slice_rows(pin, elo - prow0, ehi - prow0, 0, P.nbr[l - 1]);
  const Bsr& ps = pstrip ? *pstrip : pin;
  int clo = P.nbr[l - 1], chi = 0;
  for (int64_t q = 0; q < ps.nnzb; ++q) {
    clo = std::min(clo, ps.h_col[q]);
    chi = std::max(chi, ps.h_col[q] + 1);
  }
  const int clo1 = P.B[l - 1][r], chi1 = P.B[l - 1][r + 1];
  if (chi1 > clo1 && (clo1 < clo || chi1 > chi)) fail(BMG_ERUNTIME, "dist setup: coarse rows outside the strip");
  auto ploc = slice_rows(ps, 0, ps.nbr, clo, chi - clo);
  auto c = galerkin(*aloc, *ploc);
  if (chi1 > clo1) {
    auto rloc = bsr_transpose(*ploc);
    k.R = slice_rows(*rloc, clo1 - clo, chi1 - clo, -elo, P.nbr[l]);
    K[l - 1].A = slice_rows(*c, clo1 - clo, chi1 - clo, -clo, P.nbr[l - 1]);
  }
}

// every partitioned level of the ranks in this process (emulation: all; NCCL:
// K has one entry, this rank's)
static std::vector<std::vector<Kept>> dist_build(Ctx* ctx, const DistPlan& P, bool emulated,
                                                 const std::vector<const Bsr*>& a_top,
                                                 const std::vector<std::vector<const Bsr*>>& pin,
                                                 const bmg_setup_params& prm) {
  const int L = P.L, top = L - 1, world = P.world;
  const int nh = emulated ? world : 1;
  std::vector<std::vector<Kept>> K(nh);
  for (auto& k : K) k.resize(L);
  std::vector<std::unique_ptr<Bsr>> aext(nh);
  const bool with_comm = !emulated && world > 1;
  for (int l = top; l >= P.agg; --l) {
    collective_phase(ctx, with_comm, [&] {
      for (int i = 0; i < nh; ++i) {
        const int r = emulated ? i : ctx->rank;
        const Bsr* a = l == top ? a_top[i] : aext[i].get();
        if (P.B[l][r + 1] <= P.B[l][r]) continue;
        if (!a) fail(BMG_ERUNTIME, "dist setup: missing extended strip");
        dist_level(ctx, P, r, l, *a, *pin[i][l], prm, K[i]);
      }
    });
    for (auto& a : aext) a.reset();
    if (l == P.agg) break;
    // next level's extended strips from the owners' exact rows
    const int m = pin[0][l]->mc;
    if (emulated) {
      std::vector<const Bsr*> own(world);
      for (int r = 0; r < world; ++r) own[r] = K[r][l - 1].A.get();
      aext = fetch_rows_emulated(ctx, own, P.B[l - 1], P.elo[l - 1], P.ehi[l - 1], P.nbr[l - 1], m, false);
    } else if (world > 1) {
      aext[0] = fetch_rows_comm(ctx, K[0][l - 1].A.get(), P.B[l - 1], P.elo[l - 1], P.ehi[l - 1], P.nbr[l - 1], m,
                                false);
    } else {
      aext[0] = slice_rows(*K[0][l - 1].A, 0, P.nbr[l - 1], 0, P.nbr[l - 1]);
    }
  }
  return K;
}

static void dist_dot_partials(Hier& h, int l, Which a, Which b, DBuf<double>& part) {
  Ctx* ctx = h.ctx;
  const int n = h.nbr[l];
  if (part.n < (size_t)n) part.alloc(std::max(n, 1));
  BMG_CUDA(cudaMemsetAsync(part.p, 0, n * sizeof(double), ctx->stream));
  for (Part& p : h.parts) {
    PLevel& L = p.lv[l];
    if (!L.active()) continue;
    kern::row_partial_dot_kernel<<<grid1d(L.hi - L.lo), 256, 0, ctx->stream>>>(
        vec(h, p, l, a) + L.off(), vec(h, p, l, b) + L.off(), L.hi - L.lo, L.m, part.p + L.lo);
    ctx->count();
  }
  if (!h.emulated && h.world > 1)
    ctx->comm->allreduce(part.p, part.p, n, DType::F64, ROp::Sum, ctx->stream);
}
static double dist_dot(Hier& h, int l, Which a, Which b, DBuf<double>& part, std::vector<double>& hp) {
  dist_dot_partials(h, l, a, b, part);
  const int n = h.nbr[l];
  hp.resize(n);
  BMG_CUDA(cudaMemcpyAsync(hp.data(), part.p, n * sizeof(double), cudaMemcpyDeviceToHost, h.ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(h.ctx->stream));
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += hp[i];
  return s;
}

// lanczos_lambda_max (lanczos.hpp:16-58) on the partitioned level l: the same
// passes as the single-device version (G^T chain, A, G chain) with halos
static double dist_lanczos(Hier& h, int l, int iters, double safety, uint64_t seed) {
  Ctx* ctx = h.ctx;
  const int64_t n = (int64_t)h.nbr[l] * h.msz[l];
  iters = (int)std::min<int64_t>(iters, n);
  DBuf<double> part;
  std::vector<double> hp;
  Which V = VB, VPv = VX, W = VR;
  auto own = [&](auto&& fn) {
    for (Part& p : h.parts)
      if (p.lv[l].active()) fn(p, p.lv[l]);
  };
  own([&](Part& p, PLevel& L) {
    kern::rng_symmetric_off_kernel<<<grid1d(L.n_own()), 256, 0, ctx->stream>>>(vec(h, p, l, V) + L.off(), L.n_own(),
                                                                                seed, (int64_t)L.lo * L.m);
    ctx->count();
  });
  const double nv = std::sqrt(dist_dot(h, l, V, V, part, hp));
  own([&](Part& p, PLevel& L) {
    kern::div_kernel<<<grid1d(L.n_own()), 256, 0, ctx->stream>>>(vec(h, p, l, V) + L.off(), L.n_own(), nv);
    fill(ctx, vec(h, p, l, VPv) + L.off(), L.n_own(), 0.0);
    ctx->count();
  });
  const size_t nf = h.nfactors[l];
  std::vector<double> diag, off;
  double beta = 0.0;
  for (int j = 0; j < iters; ++j) {
    // w = G_n .. F_0 A F_0^T .. G_n^T v   (apply_transformed, fsai.cpp:219-241)
    Which cur = V, nxt = VW;
    auto step = [&](auto get, Which out) {
      const Which in = cur;
      run_pass(h, l, in, l, get, [&](Part& p, PLevel& L, const Slice& sl) {
        spmv(*sl.m, vec(h, p, l, in), vec(h, p, l, out) + L.off() + L.sc(sl.row0), h.nrhs);
      });
      cur = out;
    };
    for (size_t i = nf; i-- > 0;) {
      step([&](Part& p) -> const SplitMat* { return p.lv[l].sB.empty() ? nullptr : &p.lv[l].sB[i]; }, nxt);
      nxt = nxt == VW ? VT : VW;
    }
    step([&](Part& p) { return &p.lv[l].sA; }, nxt);
    nxt = nxt == VW ? VT : VW;
    for (size_t q = 0; q < nf; ++q) {
      const Which out = q + 1 == nf ? W : nxt;
      step([&](Part& p) -> const SplitMat* { return p.lv[l].sF.empty() ? nullptr : &p.lv[l].sF[q]; }, out);
      nxt = nxt == VW ? VT : VW;
    }
    const double alpha = dist_dot(h, l, V, W, part, hp);
    diag.push_back(alpha);
    own([&](Part& p, PLevel& L) {
      kern::lupd_kernel<<<grid1d(L.n_own()), 256, 0, ctx->stream>>>(vec(h, p, l, W) + L.off(), vec(h, p, l, V) + L.off(),
                                                                     vec(h, p, l, VPv) + L.off(), L.n_own(), alpha, beta);
      ctx->count();
    });
    beta = std::sqrt(dist_dot(h, l, W, W, part, hp));
    if (j + 1 == iters) break;
    if (beta <= 1e-14 * std::fabs(alpha) || beta == 0.0) break;
    off.push_back(beta);
    std::swap(V, VPv);  // v_prev = v
    own([&](Part& p, PLevel& L) {
      copy(ctx, vec(h, p, l, V) + L.off(), vec(h, p, l, W) + L.off(), L.n_own());
      kern::div_kernel<<<grid1d(L.n_own()), 256, 0, ctx->stream>>>(vec(h, p, l, V) + L.off(), L.n_own(), beta);
      ctx->count();
    });
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  off.resize(diag.empty() ? 0 : diag.size() - 1);
  const auto ev = tridiag_eigenvalues(diag, off);
  return safety * ev.back();
}

// assemble the partitioned hierarchy from every (virtual) rank's kept rows
static std::unique_ptr<Hier> dist_setup(Ctx* ctx, const DistPlan& P, int rank, std::vector<std::vector<Kept>>& K,
                                        const std::vector<const Bsr*>& p_whole, const bmg_setup_params& prm) {
  const int L = P.L, world = P.world, agg = P.agg;
  auto h = std::make_unique<Hier>();
  h->ctx = ctx;
  h->world = world;
  h->emulated = rank < 0;
  h->nbr = P.nbr;
  h->bounds = P.B;
  h->granule_top = P.gran[L - 1];
  // agglomerated levels on rank 0: gather the first agglomerated level's finer level
  std::unique_ptr<Bsr> a_agg;  // whole A_agg on rank 0
  {
    std::vector<int32_t> wl(world, 0), wh(world, 0);
    wh[0] = P.nbr[agg];
    const int m = p_whole[agg]->mr;
    if (h->emulated) {
      std::vector<const Bsr*> own(world);
      for (int r = 0; r < world; ++r) own[r] = K[r][agg].A.get();
      a_agg = std::move(fetch_rows_emulated(ctx, own, P.B[agg], wl, wh, P.nbr[agg], m, true)[0]);
    } else {
      a_agg = fetch_rows_comm(ctx, K[0][agg].A.get(), P.B[agg], wl, wh, P.nbr[agg], m, true);
    }
  }
  const int root = 0;  // index into K of the part holding rank 0 (emulation: rank 0; NCCL: this rank if 0)
  const bool have_root = h->emulated || ctx->rank == 0;
  std::vector<std::unique_ptr<Bsr>> whole_A(agg);
  std::vector<std::unique_ptr<Bsr>> whole_R(agg + 1);
  const bool with_comm = !h->emulated && world > 1;
  collective_phase(ctx, with_comm, [&] {
  if (have_root) {
    const Bsr* ak = a_agg.get();
    for (int l = agg; l >= 1; --l) {
      whole_A[l - 1] = galerkin(*ak, *p_whole[l]);
      whole_R[l] = bsr_transpose(*p_whole[l]);
      ak = whole_A[l - 1].get();
    }
    Kept* k0 = K[root].data();
    for (int l = agg - 1; l >= 0; --l) {
      Kept& k = k0[l];
      k.A.reset();
      if (l >= 1) {
        k.M_whole = fsai_build(*whole_A[l], prm.fsai_kind, prm.t_max, prm.tau, prm.nest);
        k.beta = lanczos_lambda_max(*whole_A[l], *k.M_whole, prm.lanczos_iters, prm.lanczos_safety, prm.seed);
      }
    }
    k0[agg].R = std::move(whole_R[agg]);
  }
  });
  // the parts
  const int nparts = h->emulated ? world : 1;
  for (int pi = 0; pi < nparts; ++pi) {
    const int r = h->emulated ? pi : rank;
    Part p;
    p.rank = r;
    p.lv.resize(L);
    h->parts.push_back(std::move(p));
  }
  h->msz.assign(L, 0);
  for (int l = 1; l < L; ++l) h->msz[l] = p_whole[l]->mr;
  h->msz[0] = p_whole[1]->mc;
  h->wlo.assign(L, std::vector<int32_t>(world, 0));
  h->whi.assign(L, std::vector<int32_t>(world, 0));
  // windows of this process's parts: hull of everything that reads level-l vectors
  // (A, the chain, R_l at level l; P_{l+1} at level l + 1), as in partition()
  for (Part& p : h->parts) {
    const int r = p.rank;
    std::vector<Kept>& k = K[h->emulated ? r : 0];
    for (int l = 0; l < L; ++l) {
      int a = P.B[l][r], b = P.B[l][r + 1];
      auto join = [&](const Bsr* m) {
        if (!m) return;
        for (int i = 0; i < m->nbr; ++i) {
          const int64_t q0 = m->h_row_ptr[i], q1 = m->h_row_ptr[i + 1];
          if (q1 == q0) continue;
          if (a >= b) {
            a = m->h_col[q0];
            b = m->h_col[q1 - 1] + 1;
          } else {
            a = std::min(a, m->h_col[q0]);
            b = std::max(b, m->h_col[q1 - 1] + 1);
          }
        }
      };
      if (l < agg) {  // whole on rank 0
        if (r == 0) {
          a = 0;
          b = P.nbr[l];
        }
      } else {
        join(k[l].A.get());
        for (auto& f : k[l].F) join(f.get());
        for (auto& f : k[l].Bt) join(f.get());
        join(k[l].R.get());
      }
      if (l + 1 < L && l + 1 >= agg) join(k[l + 1].P.get());
      if (a >= b) a = b = 0;
      h->wlo[l][r] = a;
      h->whi[l][r] = b;
    }
  }
  if (!h->emulated && world > 1) {  // everyone needs every window (exchange plans)
    std::vector<int32_t> buf((size_t)2 * L * world, 0);
    for (int l = 0; l < L; ++l) {
      buf[(size_t)(2 * l) * world + rank] = h->wlo[l][rank];
      buf[(size_t)(2 * l + 1) * world + rank] = h->whi[l][rank];
    }
    DBuf<int32_t> d(buf.size());
    BMG_CUDA(cudaMemcpy(d.p, buf.data(), buf.size() * 4, cudaMemcpyHostToDevice));
    ctx->comm->allreduce(d.p, d.p, buf.size(), DType::I32, ROp::Sum, ctx->stream);
    BMG_CUDA(cudaMemcpyAsync(buf.data(), d.p, buf.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int l = 0; l < L; ++l)
      for (int r = 0; r < world; ++r) {
        h->wlo[l][r] = buf[(size_t)(2 * l) * world + r];
        h->whi[l][r] = buf[(size_t)(2 * l + 1) * world + r];
      }
  }
  // local matrices in window coordinates, split for the halo overlap
  h->nfactors.assign(L, 1);
  for (Part& p : h->parts) {
    const int r = p.rank;
    std::vector<Kept>& k = K[h->emulated ? r : 0];
    for (int l = 0; l < L; ++l) {
      PLevel& d = p.lv[l];
      d.lo = P.B[l][r];
      d.hi = P.B[l][r + 1];
      d.wlo = h->wlo[l][r];
      d.whi = h->whi[l][r];
      d.m = h->msz[l];
      const int nwin = d.whi - d.wlo;
      d.spec.kind = prm.smoother_kind;
      d.spec.beta = 1.0;
      d.spec.alpha = prm.first_kind_fraction;
      d.spec.omega = prm.richardson_omega;
      auto split = [&](const Bsr* m, int own_lo, int own_hi, int wl, int nw) {
        SplitMat sm;
        if (m && m->nbr) sm = split_rows(*m, 0, m->nbr, wl, nw, own_lo, own_hi);
        return sm;
      };
      if (l < agg) {
        if (r != 0) continue;
        d.A_own = std::move(whole_A[l]);
        d.A = d.A_own.get();
        d.sA.whole(d.A);
        if (l >= 1) {
          d.M_own = std::move(k[l].M_whole);
          d.M = d.M_own.get();
          d.sF.clear();
          d.sF.resize(d.M->fwd.size());
          d.sB.clear();
          d.sB.resize(d.M->bwd.size());
          for (size_t q = 0; q < d.M->fwd.size(); ++q) d.sF[q].whole(d.M->fwd[q].get());
          for (size_t q = 0; q < d.M->bwd.size(); ++q) d.sB[q].whole(d.M->bwd[q].get());
          d.R_own = std::move(whole_R[l]);
          d.R = d.R_own.get();
          d.sR.whole(d.R);
          d.P_own = slice_rows(*p_whole[l], 0, P.nbr[l], 0, P.nbr[l - 1]);
          d.P = d.P_own.get();
          d.sP.whole(d.P);
          d.spec.beta = k[l].beta;
          d.spec.alpha = prm.first_kind_fraction * k[l].beta;
          h->nfactors[l] = d.M->fwd.size();
        }
        continue;
      }
      if (!d.active()) continue;
      d.sA = split(k[l].A.get(), d.lo, d.hi, d.wlo, nwin);
      d.A = d.sA.s.empty() ? nullptr : d.sA.s[0].m;
      for (auto& f : k[l].F) d.sF.push_back(split(f.get(), d.lo, d.hi, d.wlo, nwin));
      for (auto& f : k[l].Bt) d.sB.push_back(split(f.get(), d.lo, d.hi, d.wlo, nwin));
      h->nfactors[l] = k[l].F.size();
      const int cl = P.B[l - 1][r], ch = P.B[l - 1][r + 1];
      d.sP = split(k[l].P.get(), cl, ch, h->wlo[l - 1][r], h->whi[l - 1][r] - h->wlo[l - 1][r]);
      d.P = d.sP.s.empty() ? nullptr : d.sP.s[0].m;
      if (k[l].R) {
        d.sR = split(k[l].R.get(), d.lo, d.hi, d.wlo, nwin);
        d.R = d.sR.s.empty() ? nullptr : d.sR.s[0].m;
      }
    }
    for (int l = 0; l < L; ++l) alloc_vectors(*h, p.lv[l], false);
  }
  // NCCL: the chain length of partitioned levels is uniform; agglomerated ones come from rank 0
  if (!h->emulated && world > 1) {
    std::vector<int32_t> nf(L);
    for (int l = 0; l < L; ++l) nf[l] = (int32_t)h->nfactors[l];
    DBuf<int32_t> d(L);
    BMG_CUDA(cudaMemcpy(d.p, nf.data(), L * 4, cudaMemcpyHostToDevice));
    ctx->comm->allreduce(d.p, d.p, L, DType::I32, ROp::Max, ctx->stream);
    BMG_CUDA(cudaMemcpyAsync(nf.data(), d.p, L * 4, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    for (int l = 0; l < L; ++l) h->nfactors[l] = nf[l];
  }
  BMG_CUDA(cudaStreamCreateWithFlags(&h->comm, cudaStreamNonBlocking));
  BMG_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  BMG_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  // spectral bounds of the partitioned levels: distributed Lanczos
  if (h->whole()) {  // finest VB / VX alias the caller's vectors in V-cycles; Lanczos uses its own
    h->user_b = h->parts[0].lv[L - 1].v[VB].p;
    h->user_x = h->parts[0].lv[L - 1].v[VX].p;
  }
  for (int l = std::max(1, agg); l < L; ++l) {
    const double beta = dist_lanczos(*h, l, prm.lanczos_iters, prm.lanczos_safety, prm.seed);
    for (Part& p : h->parts) {
      p.lv[l].spec.beta = beta;
      p.lv[l].spec.alpha = prm.first_kind_fraction * beta;
    }
  }
  h->user_b = nullptr;
  h->user_x = nullptr;
  // coarse direct solve on rank 0
  collective_phase(ctx, with_comm, [&] {
    for (Part& p : h->parts)
      if (p.rank == 0) {
        if (P.nbr[0] * (int64_t)h->msz[0] > prm.coarse_dim_cap)
          fail(BMG_EINVAL, "setup: coarsest level exceeds the dense-solve cap");
        coarse_factor(*h, p);
      }
  });
  if (!h->emulated && world > 1) {
    int64_t n0 = h->n0;
    DBuf<int64_t> d(1);
    BMG_CUDA(cudaMemcpy(d.p, &n0, 8, cudaMemcpyHostToDevice));
    ctx->comm->allreduce(d.p, d.p, 1, DType::I64, ROp::Max, ctx->stream);
    BMG_CUDA(cudaMemcpyAsync(&n0, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    h->n0 = n0;
  }
  // half-storage A on the large partitioned levels (after the distributed Lanczos,
  // the setup's last full-storage A passes)
  build_level_psym(*h);
  // global byte-model inputs: sum of own-row pass bytes over ranks
  {
    std::vector<int64_t> st((size_t)6 * L, 0);
    for (Part& p : h->parts)
      for (int l = 0; l < L; ++l) {
        PLevel& d = p.lv[l];
        auto pb = [&](const SplitMat& sm) {
          int64_t b = 0;
          for (const Slice& sl : sm.s) b += sl.m->pass_bytes();
          return b;
        };
        if (!d.active()) continue;
        st[6 * l + 0] += d.n_own();
        st[6 * l + 1] += d.psym ? d.psym->pass_bytes : pb(d.sA);
        for (auto& f : d.sF) st[6 * l + 2] += pb(f);
        for (auto& f : d.sB) st[6 * l + 2] += pb(f);
        st[6 * l + 3] += pb(d.sR);
        st[6 * l + 4] += pb(d.sP);
        st[6 * l + 5] += pb(d.sA);
      }
    if (!h->emulated && world > 1) {
      DBuf<int64_t> d(st.size());
      BMG_CUDA(cudaMemcpy(d.p, st.data(), st.size() * 8, cudaMemcpyHostToDevice));
      ctx->comm->allreduce(d.p, d.p, st.size(), DType::I64, ROp::Sum, ctx->stream);
      BMG_CUDA(cudaMemcpyAsync(st.data(), d.p, st.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
      BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    h->stats.assign(L, LevelStats());
    for (int l = 0; l < L; ++l) {
      h->stats[l].n = st[6 * l + 0];
      h->stats[l].a_pass = st[6 * l + 1];
      h->stats[l].m_pass = st[6 * l + 2];
      h->stats[l].r_pass = st[6 * l + 3];
      h->stats[l].p_pass = st[6 * l + 4];
      h->stats[l].a_pass_ref = st[6 * l + 5];
    }
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

}  // namespace bmg

using namespace bmg;

extern "C" {

// distributed setup (multilevel.cpp:36-75 on row strips, hierarchy.cu "distributed setup")
int bmg_dist_plan(int nlevels, const int32_t* nbr, const int32_t* granule, const int32_t* radius, int world,
                  int agglomerate, const bmg_setup_params* params, int32_t* bounds, int32_t* ext_lo,
                  int32_t* ext_hi, int32_t* halo) {
  return guard([&] {
    bmg_setup_params prm;
    if (params)
      prm = *params;
    else
      bmg_setup_params_default(&prm);
    if (!nbr || !radius) fail(BMG_EINVAL, "dist_plan: nbr and radius are required");
    const DistPlan P = dist_plan(nlevels, nbr, granule, radius, world, agglomerate, prm);
    for (int l = 0; l < nlevels; ++l) {
      for (int r = 0; r <= world; ++r)
        if (bounds) bounds[(size_t)l * (world + 1) + r] = P.B[l][r];
      for (int r = 0; r < world; ++r) {
        if (ext_lo) ext_lo[(size_t)l * world + r] = P.elo[l][r];
        if (ext_hi) ext_hi[(size_t)l * world + r] = P.ehi[l][r];
      }
      if (halo) halo[l] = P.halo[l];
    }
  });
}

static void dist_inputs(int nlevels, const bmg_bsr* a_ext, const bmg_bsr* const* P, std::vector<int32_t>& nbr) {
  nbr.assign(nlevels, 0);
  nbr[nlevels - 1] = B_(a_ext)->nbc;
  for (int l = nlevels - 1; l >= 1; --l) {
    const Bsr* p = B_(P[l - 1]);
    if (!p->uniform) fail(BMG_EINVAL, "dist setup: uniform blocks required");
    if (p->nbc < 1) fail(BMG_EINVAL, "dist setup: empty prolongation");
    nbr[l - 1] = p->nbc;
  }
}

int bmg_hier_setup_dist(bmg_ctx* ch, int nlevels, const int32_t* granule, const int32_t* radius, int agglomerate,
                        const bmg_bsr* a_ext, const bmg_bsr* const* transfers, const bmg_setup_params* params,
                        bmg_hier** out) {
  return guard([&] {
    Ctx* ctx = reinterpret_cast<Ctx*>(ch);
    ctx->activate();
    bmg_setup_params prm;
    if (params)
      prm = *params;
    else
      bmg_setup_params_default(&prm);
    if (!radius) fail(BMG_EINVAL, "dist setup: radius is required");
    const int world = ctx->comm ? ctx->world : 1, rank = ctx->comm ? ctx->rank : 0;
    std::vector<int32_t> nbr;
    dist_inputs(nlevels, a_ext, transfers, nbr);
    const DistPlan P = dist_plan(nlevels, nbr.data(), granule, radius, world, agglomerate, prm);
    std::vector<const Bsr*> pin(nlevels, nullptr);
    for (int l = 1; l < nlevels; ++l) pin[l] = B_(transfers[l - 1]);
    auto K = dist_build(ctx, P, world == 1, {B_(a_ext)}, {pin}, prm);
    auto h = dist_setup(ctx, P, world == 1 ? -1 : rank, K, pin, prm);
    *out = reinterpret_cast<bmg_hier*>(h.release());
  });
}

int bmg_hier_setup_dist_emulated(bmg_ctx* ch, int world, int nlevels, const int32_t* granule, const int32_t* radius,
                                 int agglomerate, const bmg_bsr* const* a_ext, const bmg_bsr* const* transfers,
                                 const bmg_setup_params* params, bmg_hier** out) {
  return guard([&] {
    Ctx* ctx = reinterpret_cast<Ctx*>(ch);
    ctx->activate();
    bmg_setup_params prm;
    if (params)
      prm = *params;
    else
      bmg_setup_params_default(&prm);
    if (!radius) fail(BMG_EINVAL, "dist setup: radius is required");
    if (world < 1) fail(BMG_EINVAL, "dist setup: world must be >= 1");
    std::vector<int32_t> nbr;
    dist_inputs(nlevels, a_ext[0], transfers, nbr);
    const DistPlan P = dist_plan(nlevels, nbr.data(), granule, radius, world, agglomerate, prm);
    std::vector<const Bsr*> atop(world);
    std::vector<std::vector<const Bsr*>> pin(world, std::vector<const Bsr*>(nlevels, nullptr));
    for (int r = 0; r < world; ++r) {
      atop[r] = B_(a_ext[r]);
      for (int l = 1; l < nlevels; ++l) pin[r][l] = B_(transfers[(size_t)r * (nlevels - 1) + l - 1]);
    }
    auto K = dist_build(ctx, P, true, atop, pin, prm);
    auto h = dist_setup(ctx, P, -1, K, pin[0], prm);
    *out = reinterpret_cast<bmg_hier*>(h.release());
  });
}

}  // extern "C"
