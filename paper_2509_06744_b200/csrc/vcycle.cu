// vcycle.cu -- halo exchange, the device-resident V-cycle (multilevel.cpp:77-103;
// captured as a CUDA graph), batched right-hand sides and the residual norm of the
// measure_rates-style solve loop (experiments.cpp:15-67).
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
#include "bsr_stream.cuh"
#include "hier.h"

namespace bmg {
namespace kern {
// Coarse solve x = A_0^{-1} b from packed lower 64 x 64 tiles; K right-hand sides
// interleaved per scalar row.  mode 0: symmetric tiles (row part tile * x_J, column
// part tile^T * x_I for J < I); mode 1: lower-triangular T x (row parts only);
// mode 2: T^T x (column parts, diagonal tiles included).  Partials go to
// part[(out tile row, other tile, row, rhs)] and are summed by symv_reduce_kernel.
// Persistent: each CTA walks tiles
// blockIdx.x, +gridDim.x, ... and streams them through a two-stage shared-memory
// ring with cp.async.bulk (mbarrier complete_tx), so the next tile lands while the
// current one is used.  Row parts read the unpadded tile in a rotated column order
// (c = (c' + t) mod 64: conflict-free banks); column parts read columns directly.
constexpr int kSymvThreads = 256;
constexpr size_t kSymvSmem = 2 * kTile * kTile * sizeof(double) + 2 * kMaxRhs * kTile * sizeof(double) + 16;
__global__ void __launch_bounds__(kSymvThreads) symv_stream_kernel(const double* __restrict__ tiles,
                                                                   const double* __restrict__ x, int64_t N, int nt,
                                                                   int64_t ntiles, double* __restrict__ part, int K,
                                                                   int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* ring = reinterpret_cast<double*>(smem);                    // 2 x 64 x 64
  double* xi = ring + 2 * kTile * kTile;                             // [kMaxRhs][64]
  double* xj = xi + kMaxRhs * kTile;                                 // [kMaxRhs][64]
  uint64_t* full = reinterpret_cast<uint64_t*>(xj + kMaxRhs * kTile);  // 2 barriers
  const int tid = threadIdx.x;
  constexpr uint32_t kBytes = kTile * kTile * sizeof(double);
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t stride = gridDim.x;
  const uint64_t pol = l2_evict_first_policy();
  if (tid == 0)
    for (int st = 0; st < 2; ++st) {
      const int64_t t = blockIdx.x + st * stride;
      if (t < ntiles) {
        mbar_arrive_expect_tx(&full[st], kBytes);
        bulk_g2s_hint(ring + st * kTile * kTile, tiles + t * kTile * kTile, kBytes, &full[st], pol);
      }
    }
  const int it0 = mode == 2 ? kTile * K : 0, it1 = mode == 1 ? kTile * K : 2 * kTile * K;
  // the x segments of a tile (64 K values each for its row and column ranges) are
  // loaded into registers one tile ahead, so their latency overlaps the current
  // tile's work instead of preceding it (K <= kMaxRhs: at most two per thread)
  constexpr int kXPer = (kMaxRhs * kTile + kSymvThreads - 1) / kSymvThreads;
  static_assert(kXPer * kSymvThreads >= kMaxRhs * kTile, "x prefetch must cover kTile * K values for K <= kMaxRhs");
  double pxi[kXPer], pxj[kXPer];
  auto xload = [&](int64_t tt) {
    if (tt >= ntiles) return;
    int I, J;
    tile_of(tt, &I, &J);
#pragma unroll
    for (int u = 0; u < kXPer; ++u) {
      const int e = tid + u * kSymvThreads;
      if (e < kTile * K) {
        const int r = e / K, v = e - (e / K) * K;
        const int64_t gi = (int64_t)I * kTile + r, gj = (int64_t)J * kTile + r;
        pxi[u] = gi < N ? x[gi * K + v] : 0.0;
        pxj[u] = gj < N ? x[gj * K + v] : 0.0;
      }
    }
  };
  xload(blockIdx.x);
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += stride, ++it) {
    const int st = it & 1;
    int I, J;
    tile_of(t, &I, &J);
#pragma unroll
    for (int u = 0; u < kXPer; ++u) {
      const int e = tid + u * kSymvThreads;
      if (e < kTile * K) {
        const int r = e / K, v = e - (e / K) * K;
        xi[v * kTile + r] = pxi[u];
        xj[v * kTile + r] = pxj[u];
      }
    }
    __syncthreads();
    xload(t + stride);
    mbar_wait(&full[st], (it >> 1) & 1);
    const double* tl = ring + st * kTile * kTile;
    for (int q = it0 + tid; q < it1; q += kSymvThreads) {
      const int half = q / (kTile * K);
      const int rem = q - half * kTile * K;
      const int r = rem / K, v = rem - (rem / K) * K;
      if (half == 0) {  // row part: tile * x_J
        double sum = 0.0;
        const double* row = tl + r * kTile;
        const double* xv = xj + v * kTile;
        for (int c0 = 0; c0 < kTile; ++c0) {
          const int c = (c0 + r) & (kTile - 1);
          sum = __fma_rn(row[c], xv[c], sum);
        }
        part[(((int64_t)I * nt + J) * kTile + r) * K + v] = sum;
      } else if (J < I || mode == 2) {  // column part: tile^T * x_I
        double sum = 0.0;
        const double* xv = xi + v * kTile;
        for (int rr = 0; rr < kTile; ++rr) sum = __fma_rn(tl[rr * kTile + r], xv[rr], sum);
        part[(((int64_t)J * nt + I) * kTile + r) * K + v] = sum;
      }
    }
    __syncthreads();  // tile and x segments consumed
    if (tid == 0 && t + 2 * stride < ntiles) {
      mbar_arrive_expect_tx(&full[st], kBytes);
      bulk_g2s_hint(ring + st * kTile * kTile, tiles + (t + 2 * stride) * kTile * kTile, kBytes, &full[st], pol);
    }
  }
}

// y of tile row R = sum over the second tile index S in ascending order: mode 0 all
// S, mode 1 S <= R (lower row parts), mode 2 S >= R (transposed column parts)
__global__ void symv_reduce_kernel(const double* __restrict__ part, int nt, int64_t N, double* __restrict__ y,
                                   int K, int mode) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= N * K) return;
  const int64_t i = K == 1 ? e : e / K;
  const int v = (int)(e - i * K);
  const int I = (int)(i / kTile), r = (int)(i - (int64_t)I * kTile);
  const double* __restrict__ pp = part + (((int64_t)I * nt) * kTile + r) * K + v;
  const int64_t stride = (int64_t)kTile * K;
  double s = 0.0;
  int J = mode == 2 ? I : 0;
  const int J1 = mode == 1 ? I + 1 : nt;
  for (; J + 16 <= J1; J += 16) {  // sixteen loads in flight, additions in tile order
    double t[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) t[u] = __ldg(pp + (int64_t)(J + u) * stride);
#pragma unroll
    for (int u = 0; u < 16; ++u) s = __dadd_rn(s, t[u]);
  }
  for (; J < J1; ++J) s = __dadd_rn(s, __ldg(pp + (int64_t)J * stride));
  y[e] = s;
}

// Partition-invariant squared norm: one fixed-shape tree per segment of
// `seg_len` scalars (a segment = one granule of block rows, never split
// across ranks); segment sums are then added in order on the host.
__global__ void __launch_bounds__(256) segment_sq_kernel(const double* __restrict__ v, int64_t n, int64_t seg_len,
                                                         double* __restrict__ out) {
  __shared__ double sh[256];
  const int64_t s0 = blockIdx.x * seg_len;
  const int64_t s1 = min(n, s0 + seg_len);
  double acc = 0.0;
  for (int64_t i = s0 + threadIdx.x; i < s1; i += 256) acc = __fma_rn(v[i], v[i], acc);
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}
// out = a + s * b   (s = +1 / -1: the reference's Vector sums and differences)
__global__ void axpby_kernel(double* __restrict__ out, const double* __restrict__ a, const double* __restrict__ b,
                             int64_t n, int sub) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = sub ? __dsub_rn(a[i], b[i]) : __dadd_rn(a[i], b[i]);
}
__global__ void scale_inv_kernel(double* v, int64_t n, double d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[i] = __ddiv_rn(v[i], d);
}
}  // namespace kern

// ============================================================================ halo exchange
void exchange(Hier& h, int l, Which w) {
  if (h.world == 1) return;
  Ctx* ctx = h.ctx;
  const int m = h.msz[l] * h.nrhs;  // scalars per block row
  const auto& B = h.bounds[l];
  if (h.emulated) {
    for (Part& dst : h.parts)
      for (Part& src : h.parts) {
        if (&dst == &src) continue;
        const int r = dst.rank, s = src.rank;
        const int g0 = std::max(B[s], h.wlo[l][r]), g1 = std::min(B[s + 1], h.whi[l][r]);
        if (g1 <= g0) continue;
        double* d = vec(h, dst, l, w) + (int64_t)(g0 - h.wlo[l][r]) * m;
        const double* sp = vec(h, src, l, w) + (int64_t)(g0 - h.wlo[l][s]) * m;
        BMG_CUDA(cudaMemcpyAsync(d, sp, (size_t)(g1 - g0) * m * sizeof(double), cudaMemcpyDeviceToDevice,
                                 ctx->stream));
      }
    return;
  }
  Part& me = h.parts[0];
  const int r = me.rank;
  double* base = vec(h, me, l, w);
  Comm& comm = *ctx->comm;
  comm.group_start();
  for (int s = 0; s < h.world; ++s) {
    if (s == r) continue;
    // send my own rows inside s's window
    const int a0 = std::max(B[r], h.wlo[l][s]), a1 = std::min(B[r + 1], h.whi[l][s]);
    if (a1 > a0)
      comm.send(base + (int64_t)(a0 - h.wlo[l][r]) * m, (size_t)(a1 - a0) * m, DType::F64, s, ctx->stream);
    // receive s's own rows inside my window
    const int b0 = std::max(B[s], h.wlo[l][r]), b1 = std::min(B[s + 1], h.whi[l][r]);
    if (b1 > b0)
      comm.recv(base + (int64_t)(b0 - h.wlo[l][r]) * m, (size_t)(b1 - b0) * m, DType::F64, s, ctx->stream);
  }
  comm.group_end();
}

// r = b - A x on a partitioned level in half storage (hier.h PSym): the exchange of x
// forks onto the comm stream while the rows that do not read the lower halo run
// phase 1; then the boundary rows' phase 1, the merge of the in-rank upper
// contributions (rows before t0 finish there) and the tail over the upper-halo
// blocks.  gb / gr give a part's own-row b and r, gx its window x.
template <class GB, class GX, class GR>
static void sym_residual_pass(Hier& h, int l, Which xin, GB gb, GX gx, GR gr) {
  Ctx* ctx = h.ctx;
  BMG_CUDA(cudaEventRecord(h.ev_fork, ctx->stream));
  BMG_CUDA(cudaStreamWaitEvent(h.comm, h.ev_fork, 0));
  cudaStream_t main = ctx->stream;
  ctx->stream = h.comm;
  try {
    exchange(h, l, xin);
  } catch (...) {
    ctx->stream = main;
    throw;
  }
  ctx->stream = main;
  BMG_CUDA(cudaEventRecord(h.ev_join, h.comm));
  for (int phase = 0; phase < 2; ++phase) {
    if (phase == 1) BMG_CUDA(cudaStreamWaitEvent(ctx->stream, h.ev_join, 0));
    for (Part& p : h.parts) {
      PLevel& L = p.lv[l];
      if (!L.active() || !L.psym) continue;
      PSym& S = *L.psym;
      const double* x = gx(p, L);
      const int m = S.m;
      if (phase == 0) {
        if (S.low_int)
          sym_phase1(*S.low_int, SymArgs{S.brow.p + S.brow_int_off, S.colpart.p + S.nlow_bnd * m, S.oc0}, x,
                     S.sbuf.p + (int64_t)S.k1 * m);
        continue;
      }
      if (S.low_bnd) sym_phase1(*S.low_bnd, SymArgs{S.brow.p, S.colpart.p, S.oc0}, x, S.sbuf.p);
      const double* b = gb(p, L);
      double* r = gr(p, L);
      sym_merge(ctx, m, S.n, S.up_ptr.p, S.up_slot.p, S.colpart.p, S.sbuf.p, b, r, S.tbuf.p, S.t0);
      if (S.tail) residual_from(*S.tail, S.tbuf.p, b + (int64_t)S.t0 * m, x, r + (int64_t)S.t0 * m);
    }
  }
}
static bool level_psym(const Hier& h, int l) {
  return h.nrhs == 1 && !h.whole() && l < (int)h.psym_on.size() && h.psym_on[l];
}

// ============================================================================ V-cycle
// one smoother application (apply_smoother, chebyshev.hpp:117-129) on level l, all parts
static void smooth(Hier& h, int l, int k, bool xzero) {
  if (k < 1) return;
  const SmootherSpec* spec = nullptr;
  const Fsai* M0 = nullptr;
  for (Part& p : h.parts)
    if (p.lv[l].active()) {
      spec = &p.lv[l].spec;
      M0 = p.lv[l].M;
    }
  if (!spec) {  // this rank owns no rows of the level: it only serves halos
    spec = &h.parts[0].lv[l].spec;
  }
  const auto steps = smoother_schedule(*spec, k);
  const size_t nf = M0 ? M0->fwd.size() : h.nfactors[l], nb = nf;
  for (size_t s = 0; s < steps.size(); ++s) {
    const StepScalars& st = steps[s];
    Which src;
    const bool zero_x = (s == 0 && xzero);
    if (zero_x) {
      src = VB;  // A * 0 = 0: r = b exactly
    } else if (s == 0 && h.skip_top_res && l == h.cycle_top()) {
      src = VR;  // computed by the host-buffer slices (run_vcycle_hostio); pre-smoothing only
      h.skip_top_res = false;
    } else if (level_psym(h, l)) {
      sym_residual_pass(
          h, l, VX, [&](Part& p, PLevel& L) { return vec(h, p, l, VB) + L.off(); },
          [&](Part& p, PLevel&) { return vec(h, p, l, VX); },
          [&](Part& p, PLevel& L) { return vec(h, p, l, VR) + L.off(); });
      src = VR;
    } else {
      run_pass(h, l, VX, l, [&](Part& p) { return &p.lv[l].sA; },
               [&](Part& p, PLevel& L, const Slice& sl) {
                 const int64_t o = L.off() + L.sc(sl.row0);
                 residual(*sl.m, vec(h, p, l, VB) + o, vec(h, p, l, VX), vec(h, p, l, VR) + o, h.nrhs);
               });
      src = VR;
    }
    // forward chain w = F_n ... F_0 r (nest = 0: w = G r), then all but the last transpose
    Which cur = src;
    Which nxt = VW;
    for (size_t q = 0; q < nf + nb - 1; ++q) {
      const Which in = cur, out = nxt;
      run_pass(h, l, in, l,
               [&](Part& p) -> const SplitMat* {
                 PLevel& L = p.lv[l];
                 if (L.sF.empty()) return nullptr;
                 return q < nf ? &L.sF[q] : &L.sB[nb - 1 - (q - nf)];
               },
               [&](Part& p, PLevel& L, const Slice& sl) {
                 spmv(*sl.m, vec(h, p, l, in), vec(h, p, l, out) + L.off() + L.sc(sl.row0), h.nrhs);
               });
      cur = nxt;
      nxt = (nxt == VW) ? VT : VW;
    }
    run_pass(h, l, cur, l, [&](Part& p) -> const SplitMat* { return p.lv[l].sB.empty() ? nullptr : &p.lv[l].sB[0]; },
             [&](Part& p, PLevel& L, const Slice& sl) {
               const int64_t o = L.off() + L.sc(sl.row0);
               gt_cheb(*sl.m, vec(h, p, l, cur), vec(h, p, l, VP) + o, vec(h, p, l, VX) + o, st.coef, st.c, st.first,
                       zero_x, h.nrhs);
             });
  }
}

static void coarse_solve(Hier& h) {
  for (Part& p : h.parts) {
    PLevel& L = p.lv[0];
    if (!L.active()) continue;
    const int64_t N = h.n0;
    const int nt = (int)((N + kern::kTile - 1) / kern::kTile);
    const int64_t ntiles = (int64_t)nt * (nt + 1) / 2;
    const int K = h.nrhs;
    const unsigned rgrid = (unsigned)((N * K + 255) / 256);
    static const bool attr = [] {
      BMG_CUDA(cudaFuncSetAttribute(kern::symv_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)kern::kSymvSmem));
      return true;
    }();
    (void)attr;
    const unsigned sgrid = (unsigned)std::min<int64_t>(ntiles, (int64_t)h.ctx->sms * 3);
    auto tiles_pass = [&](const double* in, int mode) {
      kern::symv_stream_kernel<<<sgrid, kern::kSymvThreads, kern::kSymvSmem, h.ctx->stream>>>(
          p.ainv.p, in, N, nt, ntiles, p.cpart.p, K, mode);
    };
    if (!p.tri) {  // x = A_0^{-1} b with the symmetric packed inverse
      tiles_pass(vec(h, p, 0, VB) + L.off(), 0);
      kern::symv_reduce_kernel<<<rgrid, 256, 0, h.ctx->stream>>>(p.cpart.p, nt, N, vec(h, p, 0, VX) + L.off(), K, 0);
      h.ctx->count(2);
    } else {  // x = W^T (W b), W = L^{-1}: y in the level's r buffer
      double* y = vec(h, p, 0, VR) + L.off();
      tiles_pass(vec(h, p, 0, VB) + L.off(), 1);
      kern::symv_reduce_kernel<<<rgrid, 256, 0, h.ctx->stream>>>(p.cpart.p, nt, N, y, K, 1);
      tiles_pass(y, 2);
      kern::symv_reduce_kernel<<<rgrid, 256, 0, h.ctx->stream>>>(p.cpart.p, nt, N, vec(h, p, 0, VX) + L.off(), K, 2);
      h.ctx->count(4);
    }
    BMG_LAUNCHED(h.ctx->stream, "symv_kernels");
  }
}

// v_cycle (multilevel.cpp:77-103), recursion unrolled: down, coarse solve, up
static void enqueue_vcycle(Hier& h, int kpre, int kpost) {
  const int top = h.cycle_top();
  for (int l = top; l >= 1; --l) {
    const bool xzero = l < top;
    Which r = VR;
    if (kpre > 0) {
      smooth(h, l, kpre, xzero);
    } else if (xzero) {
      for (Part& p : h.parts)
        if (p.lv[l].active()) fill(h.ctx, vec(h, p, l, VX) + p.lv[l].off(), p.lv[l].n_own(), 0.0);
      r = VB;
    }
    if (r == VR && level_psym(h, l)) {
      sym_residual_pass(
          h, l, VX, [&](Part& p, PLevel& L) { return vec(h, p, l, VB) + L.off(); },
          [&](Part& p, PLevel&) { return vec(h, p, l, VX); },
          [&](Part& p, PLevel& L) { return vec(h, p, l, VR) + L.off(); });
    } else if (r == VR) {
      run_pass(h, l, VX, l, [&](Part& p) { return &p.lv[l].sA; },
               [&](Part& p, PLevel& L, const Slice& sl) {
                 const int64_t o = L.off() + L.sc(sl.row0);
                 residual(*sl.m, vec(h, p, l, VB) + o, vec(h, p, l, VX), vec(h, p, l, VR) + o, h.nrhs);
               });
    }
    // rc = P^T r  (multilevel.cpp:95): R rows are own rows of level l - 1
    run_pass(h, l, r, l - 1, [&](Part& p) { return &p.lv[l].sR; },
             [&](Part& p, PLevel& C, const Slice& sl) {
               spmv(*sl.m, vec(h, p, l, r), vec(h, p, l - 1, VB) + C.off() + C.sc(sl.row0), h.nrhs);
             });
  }
  coarse_solve(h);
  for (int l = 1; l <= top; ++l) {
    // x += P ec  (multilevel.cpp:98-100)
    run_pass(h, l - 1, VX, l, [&](Part& p) { return &p.lv[l].sP; },
             [&](Part& p, PLevel& L, const Slice& sl) {
               prolong_add(*sl.m, vec(h, p, l - 1, VX), vec(h, p, l, VX) + L.off() + L.sc(sl.row0), h.nrhs);
             });
    smooth(h, l, kpost, false);
  }
}

// copy the caller's finest-level b, x into the partitioned buffers (and back);
// emulated: global vectors; NCCL: this rank's own rows
static void stage_in(Hier& h, const double* b, const double* x) {
  if (h.whole()) return;
  const int top = h.finest();
  for (Part& p : h.parts) {
    PLevel& L = p.lv[top];
    if (!L.active()) continue;
    const int64_t src = h.emulated ? L.sc(L.lo) : 0;
    copy(h.ctx, L.v[VB].p + L.off(), b + src, L.n_own());
    copy(h.ctx, L.v[VX].p + L.off(), x + src, L.n_own());
  }
}
static void stage_out(Hier& h, double* x) {
  if (h.whole()) return;
  const int top = h.finest();
  for (Part& p : h.parts) {
    PLevel& L = p.lv[top];
    if (!L.active()) continue;
    const int64_t dst = h.emulated ? L.sc(L.lo) : 0;
    copy(h.ctx, x + dst, L.v[VX].p + L.off(), L.n_own());
  }
}

// batch size of the following cycles: every level's vectors hold K interleaved
// right-hand sides (grown on demand; setup, Lanczos and solve run at K = 1)
// launch plans (and padded copies of variable layouts) for every matrix the cycle
// streams with K right-hand sides: built here, never inside graph capture
static void prepare_plans(Hier& h, int K) {
  for (Part& p : h.parts)
    for (PLevel& L : p.lv) {
      auto plans = [&](const SplitMat& sm) {
        for (const Slice& sl : sm.s) plan_for(*sl.m, K);
      };
      plans(L.sA);
      plans(L.sR);
      plans(L.sP);
      for (auto& f : L.sF) plans(f);
      for (auto& f : L.sB) plans(f);
    }
}

void set_nrhs(Hier& h, int K) {
  static_assert(kern::kMaxRhs == 8, "nrhs set below and the batch kernels' instantiations");
  if (K != 1 && K != 2 && K != 4 && K != kern::kMaxRhs) fail(BMG_EINVAL, "v_cycle batch: nrhs must be 1, 2, 4 or 8");
  if (K == h.nrhs) return;
  BMG_CUDA(cudaStreamSynchronize(h.ctx->stream));
  h.nrhs = K;
  bool moved = false;  // captured graphs of every batch size point at the old buffers
  for (Part& p : h.parts) {
    for (PLevel& L : p.lv) {
      L.k = K;
      for (int w = 0; w < VNUM; ++w) {
        if (!L.v[w].p || L.v[w].n >= (size_t)std::max<int64_t>(L.n_win(), 1)) continue;
        moved = true;
        L.v[w].alloc(L.n_win());
        BMG_CUDA(cudaMemsetAsync(L.v[w].p, 0, L.v[w].bytes(), h.ctx->stream));
      }
    }
    if (p.cpart.p) {
      const int64_t nt = (h.n0 + kern::kTile - 1) / kern::kTile;
      const size_t need = (size_t)(nt * nt * kern::kTile * K);
      if (p.cpart.n < need) {
        moved = true;
        p.cpart.alloc(need);
      }
    }
  }
  if (moved) h.drop_graphs();
  prepare_plans(h, K);
  BMG_CUDA(cudaStreamSynchronize(h.ctx->stream));
}

void run_vcycle(Hier& h, int kpre, int kpost, const double* bf, double* xf) {
  if (kpre + kpost < 1) fail(BMG_EINVAL, "v_cycle: cycle needs at least one smoothing step");
  Ctx* ctx = h.ctx;
  h.user_b = bf;
  h.user_x = xf;
  if (h.cycle_top() == 0) {  // multilevel.cpp:81-84: the coarsest level solves directly
    stage_in(h, bf, xf);
    coarse_solve(h);
    stage_out(h, xf);
    return;
  }
  if (!h.use_graph || (ctx->comm && !ctx->comm->capturable())) {
    stage_in(h, bf, xf);
    enqueue_vcycle(h, kpre, kpost);
    stage_out(h, xf);
    return;
  }
  GraphKey key{kpre, kpost, h.nrhs, h.cycle_top(), bf, xf};
  auto it = h.graphs.find(key);
  if (it == h.graphs.end() && ctx->comm && !h.emulated && !h.warm.count(key)) {
    // NCCL sets up peer connections on first use, which must not happen inside
    // graph capture: the first cycle of every key runs eagerly
    h.warm[key] = 1;
    stage_in(h, bf, xf);
    enqueue_vcycle(h, kpre, kpost);
    stage_out(h, xf);
    return;
  }
  if (it == h.graphs.end()) {
    prepare_plans(h, h.nrhs);
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->own;
    const int64_t before = ctx->launches;
    BMG_CUDA(cudaStreamBeginCapture(ctx->own, cudaStreamCaptureModeThreadLocal));
    try {
      stage_in(h, bf, xf);
      enqueue_vcycle(h, kpre, kpost);
      stage_out(h, xf);
    } catch (...) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(ctx->own, &g);
      if (g) cudaGraphDestroy(g);
      ctx->stream = user;
      ctx->launches = before;
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

// The host-buffer cycles stage b and x in io_b / io_x, whose device addresses
// are baked into every captured graph that uses them: growing them frees the old
// buffers, so the stream is drained and every captured graph dropped first.
void ensure_host_io(Hier& h, int64_t n) {
  if (h.io_b.n >= (size_t)n && h.io_x.n >= (size_t)n) return;
  BMG_CUDA(cudaStreamSynchronize(h.ctx->stream));
  h.drop_graphs();
  h.io_b.alloc(std::max<int64_t>(n, 1));
  h.io_x.alloc(std::max<int64_t>(n, 1));
}

bool run_vcycle_hostio(Hier& h, int kpre, int kpost, const double* hb, double* hx) {
  static const bool off = [] {
    const char* e = std::getenv("BMG_HOSTIO_PIPELINE");
    return e && e[0] == '0';
  }();
  if (off || !h.whole() || h.nrhs != 1 || kpre < 1 || !h.use_graph || h.cycle_top() != h.finest() ||
      h.finest() == 0)
    return false;
  Ctx* ctx = h.ctx;
  Part& P0 = h.parts[0];
  PLevel& L = P0.lv[h.finest()];
  const Bsr& A = *L.A;
  if (!A.uniform || L.m == 0) return false;
  auto pinned = [](const void* p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  if (!pinned(hb) || !pinned(hx)) return false;
  const int64_t n = L.n_own();
  const int m = L.m;
  if (!h.hio) {  // slices, plans, copy stream and events: built once, outside capture
    auto io = std::make_unique<HostIo>();
    static const int nslice = [] {
      const char* e = std::getenv("BMG_HOSTIO_SLICES");
      return e ? std::max(1, std::min(64, std::atoi(e))) : 4;
    }();
    const int S = (int)std::min<int64_t>(nslice, std::max(1, A.nbr / 64));
    for (int s = 0; s < S; ++s) {
      const int r0 = (int)((int64_t)A.nbr * s / S), r1 = (int)((int64_t)A.nbr * (s + 1) / S);
      auto pl = plan_rows(A, r0, r1);
      if (!pl) return false;
      int maxc = -1;
      for (int i = r0; i < r1; ++i)
        if (A.h_row_ptr[i + 1] > A.h_row_ptr[i]) maxc = std::max(maxc, A.h_col[A.h_row_ptr[i + 1] - 1]);
      io->plans.push_back(std::move(pl));
      io->row0.push_back(r0);
      io->row1.push_back(r1);
      io->need.push_back(maxc);
    }
    for (int s = 0; s < S; ++s) {  // column -> the slice whose copy brings it
      int t = s;
      while (t + 1 < S && io->need[s] >= io->row1[t]) ++t;
      io->need[s] = t;
    }
    if (A.half) {  // half-storage A: the same row ranges over its lower triangle
      for (int s = 0; s < S; ++s) {
        auto pl = plan_rows_sym(*A.half->low, io->row0[s], io->row1[s]);
        if (!pl) {
          io->sym_plans.clear();
          break;
        }
        io->sym_plans.push_back(std::move(pl));
      }
    }
    BMG_CUDA(cudaStreamCreateWithFlags(&io->cs, cudaStreamNonBlocking));
    BMG_CUDA(cudaEventCreateWithFlags(&io->fork, cudaEventDisableTiming));
    BMG_CUDA(cudaEventCreateWithFlags(&io->ev_b, cudaEventDisableTiming));
    io->ev.resize(S, nullptr);
    for (auto& e : io->ev) BMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h.hio = std::move(io);
  }
  HostIo& io = *h.hio;
  ensure_host_io(h, n);
  GraphKey key{kpre, kpost, 1, h.cycle_top(), hb, hx, 1};
  auto it = h.graphs.find(key);
  if (it == h.graphs.end()) {
    prepare_plans(h, 1);
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->own;
    const int64_t before = ctx->launches;
    BMG_CUDA(cudaStreamBeginCapture(ctx->own, cudaStreamCaptureModeThreadLocal));
    try {
      double* r = L.v[VR].p;
      BMG_CUDA(cudaEventRecord(io.fork, ctx->own));
      BMG_CUDA(cudaStreamWaitEvent(io.cs, io.fork, 0));
      const int S = (int)io.plans.size();
      if (A.half && (int)io.sym_plans.size() == S) {
        // half-storage A: a row range of the lower triangle reads x up to its own
        // rows only, so phase 1 follows the x slices as they land; b is needed by the
        // merge alone and arrives under phase 1
        const SymHalf& H = *A.half;
        for (int s = 0; s < S; ++s) {
          const int64_t o = (int64_t)io.row0[s] * m, len = (int64_t)(io.row1[s] - io.row0[s]) * m;
          BMG_CUDA(cudaMemcpyAsync(h.io_x.p + o, hx + o, len * 8, cudaMemcpyHostToDevice, io.cs));
          BMG_CUDA(cudaEventRecord(io.ev[s], io.cs));
        }
        BMG_CUDA(cudaMemcpyAsync(h.io_b.p, hb, n * 8, cudaMemcpyHostToDevice, io.cs));
        BMG_CUDA(cudaEventRecord(io.ev_b, io.cs));
        const SymArgs sa{H.brow.p, H.colpart.p, 0};
        for (int s = 0; s < S; ++s) {
          BMG_CUDA(cudaStreamWaitEvent(ctx->own, io.ev[s], 0));
          sym_phase1_rows(*H.low, *io.sym_plans[s], sa, h.io_x.p, H.sbuf.p);
        }
        BMG_CUDA(cudaStreamWaitEvent(ctx->own, io.ev_b, 0));  // joins the copy stream
        sym_merge(ctx, m, A.nbr, H.up_ptr.p, H.up_slot.p, H.colpart.p, H.sbuf.p, h.io_b.p, r, nullptr, A.nbr);
      } else {
        for (int s = 0; s < S; ++s) {
          const int64_t o = (int64_t)io.row0[s] * m, len = (int64_t)(io.row1[s] - io.row0[s]) * m;
          BMG_CUDA(cudaMemcpyAsync(h.io_b.p + o, hb + o, len * 8, cudaMemcpyHostToDevice, io.cs));
          BMG_CUDA(cudaMemcpyAsync(h.io_x.p + o, hx + o, len * 8, cudaMemcpyHostToDevice, io.cs));
          BMG_CUDA(cudaEventRecord(io.ev[s], io.cs));
        }
        for (int s = 0; s < S; ++s) {
          BMG_CUDA(cudaStreamWaitEvent(ctx->own, io.ev[io.need[s]], 0));
          residual_rows(A, *io.plans[s], h.io_b.p, h.io_x.p, r);
        }
        BMG_CUDA(cudaStreamWaitEvent(ctx->own, io.ev[S - 1], 0));  // join the copy stream
      }
      h.user_b = h.io_b.p;
      h.user_x = h.io_x.p;
      h.skip_top_res = true;
      enqueue_vcycle(h, kpre, kpost);
      h.skip_top_res = false;
      BMG_CUDA(cudaMemcpyAsync(hx, h.io_x.p, n * 8, cudaMemcpyDeviceToHost, ctx->own));
    } catch (...) {
      h.skip_top_res = false;
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(ctx->own, &g);
      if (g) cudaGraphDestroy(g);
      ctx->stream = user;
      ctx->launches = before;
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
  return true;
}

// residual r = b - A x of the whole finest level, then its segment sums (the
// enqueue half of finest_residual + finest_norm, no host read)
static int enqueue_residual_segments(Hier& h, const double* b, const double* x) {
  Ctx* ctx = h.ctx;
  const int top = h.finest();
  PLevel& L = h.parts[0].lv[top];
  residual(*L.A, b, x, L.v[VR].p);
  const int m = h.msz[top];
  const int gran = h.granule_top;
  const int nseg = m ? (h.nbr[top] + gran - 1) / gran : (int)((L.dim + 255) / 256);
  BMG_CUDA(cudaMemsetAsync(h.seg.p, 0, nseg * sizeof(double), ctx->stream));
  kern::segment_sq_kernel<<<nseg, 256, 0, ctx->stream>>>(L.v[VR].p, L.n_own(), m ? (int64_t)gran * m : 256, h.seg.p);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  return nseg;
}

bool solve_device(Hier& h, int kpre, int kpost, const double* b, double* x, double tol, int max_iter, double* hist,
                  int* iters, int* status) {
  static const bool off = [] {
    const char* e = std::getenv("BMG_DEVICE_SOLVE");
    return e && e[0] == '0';
  }();
  if (off || !h.whole() || h.nrhs != 1 || !h.use_graph || h.top >= 0 || h.finest() == 0 || max_iter < 0)
    return false;
  Ctx* ctx = h.ctx;
  const int top = h.finest();
  const int m = h.msz[top];
  const int nseg = m ? (h.nbr[top] + h.granule_top - 1) / h.granule_top
                     : (int)((h.parts[0].lv[top].dim + 255) / 256);
  if (h.seg.n < (size_t)nseg) {
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    h.seg.alloc(std::max(nseg, 1));
    h.drop_graphs();
  }
  if (!h.h_seg || h.h_seg_n < nseg) {
    if (h.h_seg) cudaFreeHost(h.h_seg);
    BMG_CUDA(cudaMallocHost(&h.h_seg, (size_t)nseg * sizeof(double)));
    h.h_seg_n = nseg;
    h.drop_graphs();
  }
  // one graph per step: [cycle,] residual, segment sums, their copy to pinned memory
  auto step_graph = [&](int kind, int kp, int kq) -> Hier::Captured& {
    GraphKey key{kp, kq, 1, top, b, x, kind};
    auto it = h.graphs.find(key);
    if (it != h.graphs.end()) return it->second;
    prepare_plans(h, 1);
    h.user_b = b;
    h.user_x = x;
    cudaStream_t user = ctx->stream;
    ctx->stream = ctx->own;
    const int64_t before = ctx->launches;
    BMG_CUDA(cudaStreamBeginCapture(ctx->own, cudaStreamCaptureModeThreadLocal));
    try {
      if (kind == 3) enqueue_vcycle(h, kp, kq);
      enqueue_residual_segments(h, b, x);
      BMG_CUDA(cudaMemcpyAsync(h.h_seg, h.seg.p, nseg * sizeof(double), cudaMemcpyDeviceToHost, ctx->own));
    } catch (...) {
      cudaGraph_t junk = nullptr;
      cudaStreamEndCapture(ctx->own, &junk);
      if (junk) cudaGraphDestroy(junk);
      ctx->stream = user;
      ctx->launches = before;
      throw;
    }
    cudaGraph_t g;
    BMG_CUDA(cudaStreamEndCapture(ctx->own, &g));
    ctx->stream = user;
    cudaGraphExec_t ex;
    BMG_CUDA(cudaGraphInstantiate(&ex, g, 0));
    cudaGraphDestroy(g);
    auto ins = h.graphs.emplace(key, Hier::Captured{ex, ctx->launches - before});
    ctx->launches = before;
    return ins.first->second;
  };
  auto norm = [&](Hier::Captured& c) {  // the host's sequential sum, as finest_norm
    BMG_CUDA(cudaGraphLaunch(c.exec, ctx->stream));
    ctx->launches += c.kernels;
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    double s = 0.0;
    for (int i = 0; i < nseg; ++i) s += h.h_seg[i];
    return std::sqrt(s);
  };
  Hier::Captured& head = step_graph(2, 0, 0);
  Hier::Captured& step = step_graph(3, kpre, kpost);
  hist[0] = norm(head);
  int it = 0, st = 1;
  if (hist[0] == 0.0 || hist[0] / hist[0] < tol) st = 0;
  while (st == 1 && it < max_iter) {
    ++it;
    hist[it] = norm(step);
    const double growth = hist[it] / std::max(hist[it - 1], 1e-300);
    if (!std::isfinite(hist[it]) || growth > 1e6) {
      st = 2;
      break;
    }
    if (hist[it] / hist[0] < tol) st = 0;
  }
  *iters = it;
  *status = st;
  return true;
}

// partition-invariant ||r||_2 of the finest level (segments = granules)
double finest_norm(Hier& h, const double* r_whole) {
  Ctx* ctx = h.ctx;
  const int top = h.finest();
  const int m = h.msz[top];
  const int gran = h.granule_top;
  // variable layouts (whole levels only): fixed 256-scalar segments
  const int64_t dimv = m ? 0 : h.parts[0].lv[top].dim;
  const int nseg = m ? (h.nbr[top] + gran - 1) / gran : (int)((dimv + 255) / 256);
  if (h.seg.n < (size_t)nseg) h.seg.alloc(std::max(nseg, 1));
  BMG_CUDA(cudaMemsetAsync(h.seg.p, 0, nseg * sizeof(double), ctx->stream));
  for (Part& p : h.parts) {
    PLevel& L = p.lv[top];
    if (!L.active()) continue;
    const double* r = h.whole() ? r_whole : L.v[VR].p + L.off();
    const int s0 = m ? L.lo / gran : 0;
    const int ns = m ? (L.hi - L.lo + gran - 1) / gran : nseg;
    if (ns == 0) continue;
    kern::segment_sq_kernel<<<ns, 256, 0, ctx->stream>>>(r, L.n_own(), m ? (int64_t)gran * m : 256, h.seg.p + s0);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
  }
  if (!h.whole() && !h.emulated) {
    // one rank owns each segment; the others contribute exact zeros
    ctx->comm->allreduce(h.seg.p, h.seg.p, nseg, DType::F64, ROp::Sum, ctx->stream);
  }
  std::vector<double> hs(nseg);
  BMG_CUDA(cudaMemcpyAsync(hs.data(), h.seg.p, nseg * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : hs) s += v;
  return std::sqrt(s);
}

void finest_residual(Hier& h, const double* b, double* x, double* rtmp) {
  const int top = h.finest();
  if (h.whole()) {
    residual(*h.parts[0].lv[top].A, b, x, rtmp);
    return;
  }
  h.user_b = b;
  h.user_x = x;
  stage_in(h, b, x);
  if (level_psym(h, top)) {
    sym_residual_pass(
        h, top, VX, [&](Part&, PLevel& L) { return L.v[VB].p + L.off(); }, [&](Part&, PLevel& L) { return L.v[VX].p; },
        [&](Part&, PLevel& L) { return L.v[VR].p + L.off(); });
    return;
  }
  run_pass(h, top, VX, top, [&](Part& p) { return &p.lv[top].sA; },
           [&](Part& p, PLevel& L, const Slice& sl) {
             const int64_t o = L.off() + L.sc(sl.row0);
             residual(*sl.m, L.v[VB].p + o, L.v[VX].p, L.v[VR].p + o);
           });
}

}  // namespace bmg

namespace bmg {

// measure_rates (experiments.cpp:15-67) on a whole device hierarchy: the initial
// error e_i = CounterRng(seed).symmetric(i) normalised to unit M-norm, x = u_ref + e;
// after every cycle the squared M- and A-norms of x - u_ref and the residual
// ||b - A((x - u_ref) + u_ref)||; converged when the squared M-norm < tol^2.
void measure_rates(Hier& h, const Bsr& mass, const double* b, const double* u, int kpre, int kpost, uint64_t seed,
                   double tol, int max_iter, double* l2_sq, double* energy_sq, double* resid, int* iters,
                   int* status, int* blowup, double* rates) {
  if (!h.whole()) fail(BMG_EINVAL, "measure_rates: whole (unpartitioned) hierarchies only");
  set_nrhs(h, 1);
  Ctx* ctx = h.ctx;
  Part& P = h.parts[0];
  const Bsr& a = *P.lv[h.finest()].A;
  const int64_t n = a.dim_r;
  if (mass.dim_r != n || mass.dim_c != n) fail(BMG_EINVAL, "measure_rates: mass matrix does not match the finest level");
  DBuf<double> e(std::max<int64_t>(n, 1)), t(std::max<int64_t>(n, 1)), x(std::max<int64_t>(n, 1)),
      w(std::max<int64_t>(n, 1));
  rng_symmetric(ctx, e.p, n, seed);
  spmv(mass, e.p, t.p);
  const double s = std::sqrt(dot(ctx, e.p, t.p, n));
  kern::scale_inv_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(e.p, n, s);
  kern::axpby_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(x.p, u, e.p, n, 0);
  ctx->count(2);
  int rec = 0;
  auto record = [&]() {  // e holds the error
    spmv(mass, e.p, t.p);
    l2_sq[rec] = dot(ctx, e.p, t.p, n);
    spmv(a, e.p, t.p);
    energy_sq[rec] = dot(ctx, e.p, t.p, n);
    kern::axpby_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(w.p, e.p, u, n, 0);
    ctx->count();
    residual(a, b, w.p, t.p);
    resid[rec] = std::sqrt(dot(ctx, t.p, t.p, n));
    ++rec;
  };
  record();
  const double tol_sq = tol * tol;
  int it = 0, st = 1;
  *blowup = -1;
  if (l2_sq[0] < tol_sq) st = 0;
  while (st == 1 && it < max_iter) {
    run_vcycle(h, kpre, kpost, b, x.p);
    ++it;
    kern::axpby_kernel<<<grid1d(n), 256, 0, ctx->stream>>>(e.p, x.p, u, n, 1);
    ctx->count();
    record();
    const double growth = resid[it] / std::max(resid[it - 1], 1e-300);
    if (!std::isfinite(resid[it]) || growth > 1e6) {
      st = 2;
      *blowup = it;
      break;
    }
    if (l2_sq[it] < tol_sq) st = 0;
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto g = h.graphs.begin(); g != h.graphs.end();) {  // graphs of the local iterate
    if (g->first.x == x.p) {
      cudaGraphExecDestroy(g->second.exec);
      g = h.graphs.erase(g);
    } else {
      ++g;
    }
  }
  *iters = it;
  *status = st;
  rates[0] = rates[1] = rates[2] = 0.0;
  if (it > 0) {
    const double ex = 1.0 / (2.0 * it);
    rates[0] = std::pow(l2_sq[it] / l2_sq[0], ex);
    rates[1] = std::pow(energy_sq[it] / energy_sq[0], ex);
    rates[2] = std::pow(resid[it] / resid[0], 1.0 / it);
  }
}

}  // namespace bmg
