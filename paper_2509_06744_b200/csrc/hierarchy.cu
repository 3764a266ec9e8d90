// hierarchy.cu -- the device-resident multilevel hierarchy, its row partition over
// ranks (NCCL) or virtual ranks (in-process emulation), the V-cycle (captured as
// a CUDA graph) and the measure_rates-style solve loop.
//
// Reference: setup (multilevel.cpp:36-75), v_cycle (multilevel.cpp:77-103),
// measure_rates (experiments.cpp:15-67).  Partitioning: SURVEY.md §8(e).
//
// Every level of every (virtual) rank keeps its vectors in one contiguous window
// of global block rows [wlo, whi) that contains its own rows [lo, hi) plus the
// halo its matrices read; local matrices index columns as `global - wlo`.  A halo
// exchange therefore moves contiguous slices: rank s sends [max(lo_s, wlo_r),
// min(hi_s, whi_r)) to rank r.  Per-row arithmetic does not depend on the
// partition, so partitioned cycles are bitwise equal to the 1-GPU cycle.
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
#include "bmg_internal.h"

namespace bmg {
namespace kern {

__global__ void bsr_to_dense_kernel(const double* __restrict__ vals, BlkView V, const int64_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ col, int nbr, double* __restrict__ dense, int64_t N) {
  for (int i = blockIdx.x; i < nbr; i += gridDim.x) {
    const int rows = V.r(i);
    const int64_t ro = V.ro(i);
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int j = col[p];
      const int cols = V.c(j);
      const int64_t co = V.co(j), off = V.off(p);
      for (int e = threadIdx.x; e < rows * cols; e += blockDim.x) {
        const int r = e / cols, c = e - r * cols;
        dense[(ro + r) * N + co + c] = vals[off + e];
      }
    }
  }
}

__global__ void symmetrize_dense_kernel(double* a, int64_t N) {
  // cuSOLVER potri (column-major lower) leaves the row-major upper triangle
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * N; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / N, c = e - r * N;
    if (r > c) a[e] = a[c * N + r];
  }
}

// Coarse solve x = A_0^{-1} b with the symmetric inverse stored as packed lower
// 64 x 64 tiles (half the bytes of a dense GEMV).  Each tile (I, J), J <= I,
// contributes tile * x_J to rows of I and (J < I) tile^T * x_I to rows of J;
// partials are summed per row in ascending tile order (deterministic).
constexpr int kTile = 64;

__device__ __forceinline__ void tile_of(int64_t t, int* I, int* J) {
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= t) ++i;
  while ((int64_t)i * (i + 1) / 2 > t) --i;
  *I = i;
  *J = (int)(t - (int64_t)i * (i + 1) / 2);
}

__global__ void pack_lower_tiles_kernel(const double* __restrict__ full, int64_t N, double* __restrict__ tiles) {
  int I, J;
  tile_of(blockIdx.x, &I, &J);
  double* dst = tiles + (int64_t)blockIdx.x * kTile * kTile;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e - r * kTile;
    const int64_t gr = (int64_t)I * kTile + r, gc = (int64_t)J * kTile + c;
    dst[e] = (gr < N && gc < N) ? full[gr * N + gc] : 0.0;
  }
}

// K right-hand sides interleaved per scalar row; K = 1 is the plain symv
__global__ void __launch_bounds__(256) symv_tiles_kernel(const double* __restrict__ tiles,
                                                         const double* __restrict__ x, int64_t N, int nt,
                                                         double* __restrict__ part, int K) {
  __shared__ double tl[kTile][kTile + 1];
  __shared__ double xi[8][kTile], xj[8][kTile];
  int I, J;
  tile_of(blockIdx.x, &I, &J);
  const double2* src = reinterpret_cast<const double2*>(tiles + (int64_t)blockIdx.x * kTile * kTile);
  for (int e = threadIdx.x; e < kTile * kTile / 2; e += blockDim.x) {
    const double2 v = __ldg(src + e);
    const int r = (2 * e) / kTile, c = (2 * e) - r * kTile;
    tl[r][c] = v.x;
    tl[r][c + 1] = v.y;
  }
  for (int e = threadIdx.x; e < kTile * K; e += blockDim.x) {
    const int t = e / K, v = e - (e / K) * K;
    const int64_t gi = (int64_t)I * kTile + t, gj = (int64_t)J * kTile + t;
    xi[v][t] = gi < N ? x[gi * K + v] : 0.0;
    xj[v][t] = gj < N ? x[gj * K + v] : 0.0;
  }
  __syncthreads();
  for (int it = threadIdx.x; it < 2 * kTile * K; it += blockDim.x) {
    const int half = it / (kTile * K);
    const int rem = it - half * kTile * K;
    const int t = rem / K, v = rem - (rem / K) * K;
    if (half == 0) {  // row part: tile * x_J
      double s = 0.0;
      for (int c = 0; c < kTile; ++c) s = __fma_rn(tl[t][c], xj[v][c], s);
      part[(((int64_t)I * nt + J) * kTile + t) * K + v] = s;
    } else if (J < I) {  // column part: tile^T * x_I
      double s = 0.0;
      for (int r = 0; r < kTile; ++r) s = __fma_rn(tl[r][t], xi[v][r], s);
      part[(((int64_t)J * nt + I) * kTile + t) * K + v] = s;
    }
  }
}

__global__ void symv_reduce_kernel(const double* __restrict__ part, int nt, int64_t N, double* __restrict__ y,
                                   int K) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= N * K) return;
  const int64_t i = e / K;
  const int v = (int)(e - i * K);
  const int I = (int)(i / kTile), r = (int)(i - (int64_t)I * kTile);
  double s = 0.0;
  for (int J = 0; J < nt; ++J) s = __dadd_rn(s, part[(((int64_t)I * nt + J) * kTile + r) * K + v]);
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

}  // namespace kern

static int grid1d(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }


// ============================================================================ data model
enum Which { VB = 0, VX, VR, VW, VP, VT, VNUM };

// A local matrix cut into row slices (local rows [row0, row0 + nbr)): the
// interior slice reads only the rank's own columns and runs while the halo
// exchange is in flight; boundary slices run after it lands.
struct Slice {
  int row0 = 0;
  const Bsr* m = nullptr;
  std::unique_ptr<Bsr> own;
  bool interior = true;
};
struct SplitMat {
  std::vector<Slice> s;  // interior slice first
  void whole(const Bsr* a) {
    s.clear();
    if (!a) return;
    Slice x;
    x.m = a;
    s.push_back(std::move(x));
  }
};

struct PLevel {  // one (virtual) rank's share of one level
  int lo = 0, hi = 0;    // own block rows
  int wlo = 0, whi = 0;  // vector window (block rows)
  int m = 0;             // uniform block size on this level
  const Bsr* A = nullptr;
  const Bsr* R = nullptr;  // restriction to level l-1 (rows: own rows of l-1)
  const Bsr* P = nullptr;  // prolongation from level l-1 (rows: own rows of l)
  const Fsai* M = nullptr;
  std::unique_ptr<Bsr> A_own, R_own, P_own;
  std::unique_ptr<Fsai> M_own;
  SplitMat sA, sR, sP;                 // the matrices as launched
  std::vector<SplitMat> sF, sB;        // FSAI chain factors and their transposes
  SmootherSpec spec;  // Level::smoother (multilevel.hpp:25)
  DBuf<double> v[VNUM];
  int64_t dim = 0;        // scalar length (variable layouts: m = 0, whole levels only)
  int k = 1;              // right-hand sides per scalar row (batched cycles)
  int64_t off() const { return m ? (int64_t)(lo - wlo) * m * k : 0; }
  int64_t n_own() const { return (m ? (int64_t)(hi - lo) * m : dim) * k; }
  int64_t n_win() const { return (m ? (int64_t)(whi - wlo) * m : dim) * k; }
  int64_t sc(int rows) const { return (int64_t)rows * m * k; }  // scalar offset of local rows
  bool active() const { return hi > lo; }
};

struct Part {
  int rank = 0;
  std::vector<PLevel> lv;
  DBuf<double> ainv;  // A_0^{-1} as packed lower 64x64 tiles (rank owning level 0)
  DBuf<double> cpart; // per-(tile row, tile) partial sums of the coarse solve
};

struct LevelStats {  // global byte model inputs (bmg_hier_cycle_bytes)
  int64_t n = 0, a_pass = 0, m_pass = 0, r_pass = 0, p_pass = 0;
};

struct GraphKey {
  int kpre, kpost, nrhs;
  const double* b;
  double* x;
  bool operator<(const GraphKey& o) const {
    return std::tie(kpre, kpost, nrhs, b, x) < std::tie(o.kpre, o.kpost, o.nrhs, o.b, o.x);
  }
};

struct Hier {
  Ctx* ctx = nullptr;
  int world = 1;          // ranks the rows are split over
  bool emulated = false;  // all virtual ranks live in this process
  std::vector<Part> parts;
  int nrhs = 1;                               // right-hand sides of the current cycle batch
  std::vector<int> nbr, msz;                  // per level
  std::vector<size_t> nfactors;               // per level: FSAI chain length
  std::vector<std::vector<int32_t>> bounds;   // per level: world + 1
  std::vector<std::vector<int32_t>> wlo, whi; // per level, per rank
  int granule_top = 1;                        // block rows per norm segment (top level)
  int64_t n0 = 0;
  std::vector<LevelStats> stats;
  bool use_graph = true;
  struct Captured {
    cudaGraphExec_t exec;
    int64_t kernels;
  };
  std::map<GraphKey, Captured> graphs;
  DBuf<double> io_b, io_x, seg;
  cudaStream_t comm = nullptr;  // halo exchanges overlap interior slices
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  const double* user_b = nullptr;
  double* user_x = nullptr;
  ~Hier() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (comm) cudaStreamDestroy(comm);
  }
  int finest() const { return (int)nbr.size() - 1; }
  bool whole() const { return world == 1; }
  void drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
};

// vector of level l on part p; the unpartitioned top level uses the caller's b, x
static double* vec(Hier& h, Part& p, int l, Which w) {
  if (h.whole() && l == h.finest()) {
    if (w == VB) return const_cast<double*>(h.user_b);
    if (w == VX) return h.user_x;
  }
  return p.lv[l].v[w].p;
}

// ============================================================================ halo exchange
static void exchange(Hier& h, int l, Which w) {
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

// One streaming pass over a split matrix whose input is vector `in` of level
// `in_level`: the exchange of its halo runs on the comm stream while the
// interior slices compute; boundary slices wait for the exchange.  `get`
// returns the SplitMat of a part (nullptr: nothing to do), `launch` runs one
// slice (row offset in scalars = slice.row0 * m of the output level).
template <class Get, class Launch>
static void run_pass(Hier& h, int in_level, Which in, int out_level, Get get, Launch launch) {
  Ctx* ctx = h.ctx;
  if (h.world == 1) {
    for (Part& p : h.parts) {
      PLevel& L = p.lv[out_level];
      const SplitMat* sm = get(p);
      if (!L.active() || !sm) continue;
      for (const Slice& sl : sm->s) launch(p, L, sl);
    }
    return;
  }
  BMG_CUDA(cudaEventRecord(h.ev_fork, ctx->stream));
  BMG_CUDA(cudaStreamWaitEvent(h.comm, h.ev_fork, 0));
  cudaStream_t main = ctx->stream;
  ctx->stream = h.comm;
  try {
    exchange(h, in_level, in);
  } catch (...) {
    ctx->stream = main;
    throw;
  }
  ctx->stream = main;
  BMG_CUDA(cudaEventRecord(h.ev_join, h.comm));
  for (int phase = 0; phase < 2; ++phase) {
    if (phase == 1) BMG_CUDA(cudaStreamWaitEvent(ctx->stream, h.ev_join, 0));
    for (Part& p : h.parts) {
      PLevel& L = p.lv[out_level];
      const SplitMat* sm = get(p);
      if (!L.active() || !sm) continue;
      for (const Slice& sl : sm->s)
        if (sl.interior == (phase == 0)) launch(p, L, sl);
    }
  }
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
    kern::symv_tiles_kernel<<<(unsigned)ntiles, 256, 0, h.ctx->stream>>>(p.ainv.p, vec(h, p, 0, VB) + L.off(), N, nt,
                                                                        p.cpart.p, K);
    kern::symv_reduce_kernel<<<(unsigned)((N * K + 255) / 256), 256, 0, h.ctx->stream>>>(
        p.cpart.p, nt, N, vec(h, p, 0, VX) + L.off(), K);
    h.ctx->count(2);
    BMG_LAUNCHED(h.ctx->stream, "symv_kernels");
  }
}

// v_cycle (multilevel.cpp:77-103), recursion unrolled: down, coarse solve, up
static void enqueue_vcycle(Hier& h, int kpre, int kpost) {
  const int top = h.finest();
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
    if (r == VR) {
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
static void set_nrhs(Hier& h, int K) {
  if (K != 1 && K != 2 && K != 4 && K != 8) fail(BMG_EINVAL, "v_cycle batch: nrhs must be 1, 2, 4 or 8");
  if (K == h.nrhs) return;
  BMG_CUDA(cudaStreamSynchronize(h.ctx->stream));
  h.nrhs = K;
  for (Part& p : h.parts) {
    for (PLevel& L : p.lv) {
      // launch plans for this batch size (built here, never inside graph capture)
      auto plans = [&](const SplitMat& sm) {
        for (const Slice& sl : sm.s) plan_for(*sl.m, K);
      };
      plans(L.sA);
      plans(L.sR);
      plans(L.sP);
      for (auto& f : L.sF) plans(f);
      for (auto& f : L.sB) plans(f);
      L.k = K;
      for (int w = 0; w < VNUM; ++w) {
        if (!L.v[w].p || L.v[w].n >= (size_t)std::max<int64_t>(L.n_win(), 1)) continue;
        L.v[w].alloc(L.n_win());
        BMG_CUDA(cudaMemsetAsync(L.v[w].p, 0, L.v[w].bytes(), h.ctx->stream));
      }
    }
    if (p.cpart.p) {
      const int64_t nt = (h.n0 + kern::kTile - 1) / kern::kTile;
      const size_t need = (size_t)(nt * nt * kern::kTile * K);
      if (p.cpart.n < need) p.cpart.alloc(need);
    }
  }
  BMG_CUDA(cudaStreamSynchronize(h.ctx->stream));
}

static void run_vcycle(Hier& h, int kpre, int kpost, const double* bf, double* xf) {
  if (kpre + kpost < 1) fail(BMG_EINVAL, "v_cycle: cycle needs at least one smoothing step");
  Ctx* ctx = h.ctx;
  h.user_b = bf;
  h.user_x = xf;
  if (h.finest() == 0) {
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
  GraphKey key{kpre, kpost, h.nrhs, bf, xf};
  auto it = h.graphs.find(key);
  if (it == h.graphs.end()) {
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

// BMG_SETUP_TIMING=1: per-phase wall time of the setup on stderr (device synced)
struct SetupClock {
  Ctx* ctx;
  bool on;
  std::chrono::steady_clock::time_point t;
  explicit SetupClock(Ctx* c) : ctx(c) {
    const char* e = std::getenv("BMG_SETUP_TIMING");
    on = e && e[0] == '1';
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* what, int level) {
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[bmg setup] level %d %-24s %8.3f s\n", level, what,
                 std::chrono::duration<double>(now - t).count());
    t = now;
  }
};

// ============================================================================ construction
static void coarse_factor(Hier& h, Part& p) {
  Ctx* ctx = h.ctx;
  const Bsr& a0 = *p.lv[0].A;
  if (!(a0.rsz == a0.csz)) fail(BMG_EINVAL, "coarse solve: square block layout required");
  const int64_t N = a0.dim_r;
  h.n0 = N;
  p.ainv.alloc(std::max<int64_t>(N * N, 1));
  BMG_CUDA(cudaMemsetAsync(p.ainv.p, 0, p.ainv.bytes(), ctx->stream));
  kern::bsr_to_dense_kernel<<<std::max(1, std::min(a0.nbr, ctx->sms * 8)), 128, 0, ctx->stream>>>(
      a0.vals.p, blk_view(a0), a0.row_ptr.p, a0.col.p, a0.nbr, p.ainv.p, N);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  cusolverDnHandle_t s = ctx->cusolver();
  int lwork = 0, lwork2 = 0;
  if (cusolverDnDpotrf_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, &lwork) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotrf_bufferSize failed");
  if (cusolverDnDpotri_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, &lwork2) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotri_bufferSize failed");
  DBuf<double> work(std::max(std::max(lwork, lwork2), 1));
  DBuf<int> info(1);
  if (cusolverDnDpotrf(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, work.p, lwork, info.p) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotrf failed");
  int hinfo = 0;
  BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) fail(BMG_ERUNTIME, "setup: coarsest operator is not positive definite");
  if (cusolverDnDpotri(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, work.p, lwork2, info.p) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotri failed");
  BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) fail(BMG_ERUNTIME, "setup: coarse inverse failed");
  kern::symmetrize_dense_kernel<<<grid1d(N * N), 256, 0, ctx->stream>>>(p.ainv.p, N);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  // keep only the lower 64x64 tiles (packed); the dense copy is released
  const int nt = (int)((N + kern::kTile - 1) / kern::kTile);
  const int64_t ntiles = (int64_t)nt * (nt + 1) / 2;
  DBuf<double> tiles((size_t)ntiles * kern::kTile * kern::kTile);
  kern::pack_lower_tiles_kernel<<<(unsigned)ntiles, 256, 0, ctx->stream>>>(p.ainv.p, N, tiles.p);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  p.ainv = std::move(tiles);
  p.cpart.alloc((size_t)nt * nt * kern::kTile);
  BMG_CUDA(cudaMemsetAsync(p.cpart.p, 0, p.cpart.bytes(), ctx->stream));
}

static void alloc_vectors(Hier& h, PLevel& L, bool top) {
  for (int w = 0; w < VNUM; ++w) {
    if (h.whole() && top && (w == VB || w == VX)) continue;  // caller's vectors
    L.v[w].alloc(std::max<int64_t>(L.n_win(), 1));
    BMG_CUDA(cudaMemsetAsync(L.v[w].p, 0, L.v[w].bytes(), h.ctx->stream));
  }
}

static void record_stats(Hier& h) {
  Part& p = h.parts[0];
  h.stats.assign(h.finest() + 1, LevelStats());
  for (int l = 0; l <= h.finest(); ++l) {
    LevelStats& s = h.stats[l];
    const PLevel& L = p.lv[l];
    s.n = L.A->dim_r;
    s.a_pass = L.A->pass_bytes();
    if (l >= 1) {
      for (auto& f : L.M->fwd) s.m_pass += f->pass_bytes();
      for (auto& f : L.M->bwd) s.m_pass += f->pass_bytes();
      s.r_pass = L.R->pass_bytes();
      s.p_pass = L.P->pass_bytes();
    }
  }
}

// common tail of setup / create: whole-level layout, vectors, coarse factor
static void finish_whole(Hier& h, int cap) {
  Part& p = h.parts[0];
  const int L = (int)p.lv.size();
  h.nbr.assign(L, 0);
  h.msz.assign(L, 0);
  for (int l = 0; l < L; ++l) {
    PLevel& lv = p.lv[l];
    if (!(lv.A->rsz == lv.A->csz)) fail(BMG_EINVAL, "hierarchy: square block layouts required");
    h.nbr[l] = lv.A->nbr;
    h.msz[l] = lv.A->uniform ? lv.A->mr : 0;  // 0: variable block sizes
    lv.lo = lv.wlo = 0;
    lv.hi = lv.whi = lv.A->nbr;
    lv.m = h.msz[l];
    lv.dim = lv.A->dim_r;
  }
  const int64_t n0 = p.lv[0].A->dim_r;
  if (n0 > cap) fail(BMG_EINVAL, "setup: coarsest level exceeds the dense-solve cap");
  for (int l = 0; l < L; ++l) alloc_vectors(h, p.lv[l], l == L - 1);
  h.bounds.assign(L, std::vector<int32_t>{0, 0});
  h.wlo.assign(L, std::vector<int32_t>{0});
  h.whi.assign(L, std::vector<int32_t>{0});
  for (int l = 0; l < L; ++l) {
    h.bounds[l][1] = h.nbr[l];
    h.whi[l][0] = h.nbr[l];
  }
  h.granule_top = 1;
  h.nfactors.assign(L, 1);
  for (int l = 1; l < L; ++l) h.nfactors[l] = p.lv[l].M->fwd.size();
  for (int l = 0; l < L; ++l) {
    PLevel& lv = p.lv[l];
    lv.sA.whole(lv.A);
    if (l >= 1) {
      lv.sR.whole(lv.R);
      lv.sP.whole(lv.P);
      lv.sF.clear();
      lv.sF.resize(lv.M->fwd.size());
      lv.sB.clear();
      lv.sB.resize(lv.M->bwd.size());
      for (size_t q = 0; q < lv.M->fwd.size(); ++q) lv.sF[q].whole(lv.M->fwd[q].get());
      for (size_t q = 0; q < lv.M->bwd.size(); ++q) lv.sB[q].whole(lv.M->bwd[q].get());
    }
  }
  coarse_factor(h, p);
  record_stats(h);
}

// rows [lo, hi) of g with columns shifted by -col_lo into a window of ncols blocks
static std::unique_ptr<Bsr> slice_rows(const Bsr& g, int lo, int hi, int col_lo, int ncols) {
  if (hi <= lo) return nullptr;
  const int64_t p0 = g.h_row_ptr[lo], p1 = g.h_row_ptr[hi];
  std::vector<int64_t> rp(hi - lo + 1);
  for (int i = lo; i <= hi; ++i) rp[i - lo] = g.h_row_ptr[i] - p0;
  std::vector<int32_t> col(p1 - p0);
  for (int64_t q = p0; q < p1; ++q) {
    const int c = g.h_col[q] - col_lo;
    if (c < 0 || c >= ncols) fail(BMG_ERUNTIME, "partition: column outside the window");
    col[q - p0] = c;
  }
  std::vector<int> csz;  // columns beyond g's own (local -> global renumbering): uniform
  if (col_lo < 0 || col_lo + ncols > g.nbc) {
    if (!g.uniform) fail(BMG_EINVAL, "partition: column renumbering needs uniform blocks");
    csz.assign(ncols, g.mc);
  }
  auto out = make_bsr_structure(g.ctx, hi - lo, g.rsz.data() + lo, ncols,
                                csz.empty() ? g.csz.data() + col_lo : csz.data(), std::move(rp), std::move(col), false);
  const int64_t v0 = g.h_voff[p0], v1 = g.h_voff[p1];
  if (v1 > v0)
    BMG_CUDA(cudaMemcpyAsync(out->vals.p, g.vals.p + v0, (v1 - v0) * sizeof(double), cudaMemcpyDeviceToDevice,
                             g.ctx->stream));
  return out;
}

// Rows [lo, hi) of global g (columns shifted into the window [wlo, wlo + nwin)),
// cut into the longest run of rows reading only own columns [own_lo, own_hi)
// (interior) and the boundary rows before / after it.
static SplitMat split_rows(const Bsr& g, int lo, int hi, int wlo, int nwin, int own_lo, int own_hi) {
  SplitMat sm;
  if (hi <= lo) return sm;
  auto interior = [&](int i) {
    const int64_t p0 = g.h_row_ptr[i], p1 = g.h_row_ptr[i + 1];
    return p1 == p0 || (g.h_col[p0] >= own_lo && g.h_col[p1 - 1] < own_hi);
  };
  int ia = hi, ib = hi, best = 0;
  for (int i = lo; i < hi;) {
    if (!interior(i)) {
      ++i;
      continue;
    }
    int j = i;
    while (j < hi && interior(j)) ++j;
    if (j - i > best) {
      best = j - i;
      ia = i;
      ib = j;
    }
    i = j;
  }
  auto add = [&](int a, int b, bool in) {
    if (b <= a) return;
    Slice x;
    x.row0 = a - lo;
    x.own = slice_rows(g, a, b, wlo, nwin);
    x.m = x.own.get();
    x.interior = in;
    sm.s.push_back(std::move(x));
  };
  add(ia, ib, true);
  add(lo, std::min(ia, hi), false);
  add(ib, hi, false);
  return sm;
}

// Split the (identically built) whole hierarchy into row strips.  rank < 0:
// every virtual rank in this process (emulation); else only this rank's share
// and the context's NCCL communicator moves the halos.
static void partition(Hier& h, int world, int rank, const int32_t* granule, int agglomerate) {
  if (!h.whole()) fail(BMG_EINVAL, "partition: hierarchy is already partitioned");
  if (world < 1) fail(BMG_EINVAL, "partition: world must be >= 1");
  for (int m : h.msz)
    if (m == 0) fail(BMG_EINVAL, "partition: variable block layouts are not supported (uniform levels only)");
  if (world == 1) {  // nothing to split; record the norm segmentation so 1-rank
                     // and N-rank residual norms are summed identically
    h.granule_top = granule ? std::max(1, granule[h.finest()]) : 1;
    return;
  }
  if (rank >= 0 && (!h.ctx->comm || h.ctx->world != world || h.ctx->rank != rank))
    fail(BMG_EINVAL, "partition: context is not an NCCL context of this rank/world");
  Ctx* ctx = h.ctx;
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  const int L = h.finest() + 1;
  agglomerate = std::max(1, agglomerate);  // level 0 (dense solve) always on rank 0
  Part& G = h.parts[0];
  std::vector<std::vector<int32_t>> B(L, std::vector<int32_t>(world + 1));
  for (int l = 0; l < L; ++l)
    partition_rows(h.nbr[l], G.lv[l].A->h_row_ptr.data(), world, granule ? granule[l] : 1, l < agglomerate,
                   B[l].data());
  // windows: hull over everything that reads level-l vectors
  std::vector<std::vector<int32_t>> WL(L, std::vector<int32_t>(world)), WH(L, std::vector<int32_t>(world));
  for (int l = 0; l < L; ++l)
    for (int r = 0; r < world; ++r) {
      int a = B[l][r], b = B[l][r + 1];
      auto join = [&](const Bsr& m, int lo, int hi, int clo, int chi) {
        if (hi <= lo) return;
        int32_t e0, e1;
        row_window(m.h_row_ptr.data(), m.h_col.data(), lo, hi, clo, chi, &e0, &e1);
        if (a >= b) {
          a = e0;
          b = e1;
        } else if (e1 > e0) {
          a = std::min(a, e0);
          b = std::max(b, e1);
        }
      };
      const PLevel& lv = G.lv[l];
      join(*lv.A, B[l][r], B[l][r + 1], B[l][r], B[l][r + 1]);
      if (l >= 1) {
        for (auto& f : lv.M->fwd) join(*f, B[l][r], B[l][r + 1], B[l][r], B[l][r + 1]);
        for (auto& f : lv.M->bwd) join(*f, B[l][r], B[l][r + 1], B[l][r], B[l][r + 1]);
        join(*lv.R, B[l - 1][r], B[l - 1][r + 1], B[l][r], B[l][r + 1]);
      }
      if (l + 1 < L) join(*G.lv[l + 1].P, B[l + 1][r], B[l + 1][r + 1], B[l][r], B[l][r + 1]);
      if (a >= b) a = b = 0;
      WL[l][r] = a;
      WH[l][r] = b;
    }
  // build the parts
  std::vector<Part> parts;
  for (int r = 0; r < world; ++r) {
    if (rank >= 0 && r != rank) continue;
    Part p;
    p.rank = r;
    p.lv.resize(L);
    for (int l = 0; l < L; ++l) {
      PLevel& d = p.lv[l];
      const PLevel& s = G.lv[l];
      d.lo = B[l][r];
      d.hi = B[l][r + 1];
      d.wlo = WL[l][r];
      d.whi = WH[l][r];
      d.m = h.msz[l];
      d.spec = s.spec;
      const int nwin = d.whi - d.wlo;
      d.sA = split_rows(*s.A, d.lo, d.hi, d.wlo, nwin, d.lo, d.hi);
      d.A = d.sA.s.empty() ? nullptr : d.sA.s[0].m;
      if (l >= 1) {
        d.M = nullptr;  // chain length comes from h.nfactors
        for (auto& f : s.M->fwd) d.sF.push_back(split_rows(*f, d.lo, d.hi, d.wlo, nwin, d.lo, d.hi));
        for (auto& f : s.M->bwd) d.sB.push_back(split_rows(*f, d.lo, d.hi, d.wlo, nwin, d.lo, d.hi));
        d.sP = split_rows(*s.P, d.lo, d.hi, WL[l - 1][r], WH[l - 1][r] - WL[l - 1][r], B[l - 1][r], B[l - 1][r + 1]);
        d.sR = split_rows(*s.R, B[l - 1][r], B[l - 1][r + 1], d.wlo, nwin, d.lo, d.hi);
        d.P = d.sP.s.empty() ? nullptr : d.sP.s[0].m;
        d.R = d.sR.s.empty() ? nullptr : d.sR.s[0].m;
      }
      alloc_vectors(h, d, false);
    }
    if (r == 0) {
      p.ainv = std::move(G.ainv);
      p.cpart = std::move(G.cpart);
    }
    parts.push_back(std::move(p));
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  h.drop_graphs();
  h.parts = std::move(parts);  // frees the whole-level objects
  h.world = world;
  h.emulated = rank < 0;
  h.bounds = B;
  h.wlo = WL;
  h.whi = WH;
  h.granule_top = granule ? std::max(1, granule[L - 1]) : 1;
  if (!h.comm) {
    BMG_CUDA(cudaStreamCreateWithFlags(&h.comm, cudaStreamNonBlocking));
    BMG_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
    BMG_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
  }
}

// partition-invariant ||r||_2 of the finest level (segments = granules)
static double finest_norm(Hier& h, const double* r_whole) {
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

static void finest_residual(Hier& h, const double* b, double* x, double* rtmp) {
  const int top = h.finest();
  if (h.whole()) {
    residual(*h.parts[0].lv[top].A, b, x, rtmp);
    return;
  }
  h.user_b = b;
  h.user_x = x;
  stage_in(h, b, x);
  run_pass(h, top, VX, top, [&](Part& p) { return &p.lv[top].sA; },
           [&](Part& p, PLevel& L, const Slice& sl) {
             const int64_t o = L.off() + L.sc(sl.row0);
             residual(*sl.m, L.v[VB].p + o, L.v[VX].p, L.v[VR].p + o);
           });
}

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
  for (int l = top; l >= P.agg; --l) {
    for (int i = 0; i < nh; ++i) {
      const int r = emulated ? i : ctx->rank;
      const Bsr* a = l == top ? a_top[i] : aext[i].get();
      if (P.B[l][r + 1] <= P.B[l][r]) continue;
      if (!a) fail(BMG_ERUNTIME, "dist setup: missing extended strip");
      dist_level(ctx, P, r, l, *a, *pin[i][l], prm, K[i]);
    }
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
  for (Part& p : h->parts)
    if (p.rank == 0) {
      if (P.nbr[0] * (int64_t)h->msz[0] > prm.coarse_dim_cap)
        fail(BMG_EINVAL, "setup: coarsest level exceeds the dense-solve cap");
      coarse_factor(*h, p);
    }
  if (!h->emulated && world > 1) {
    int64_t n0 = h->n0;
    DBuf<int64_t> d(1);
    BMG_CUDA(cudaMemcpy(d.p, &n0, 8, cudaMemcpyHostToDevice));
    ctx->comm->allreduce(d.p, d.p, 1, DType::I64, ROp::Max, ctx->stream);
    BMG_CUDA(cudaMemcpyAsync(&n0, d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    h->n0 = n0;
  }
  // global byte-model inputs: sum of own-row pass bytes over ranks
  {
    std::vector<int64_t> st((size_t)5 * L, 0);
    for (Part& p : h->parts)
      for (int l = 0; l < L; ++l) {
        PLevel& d = p.lv[l];
        auto pb = [&](const SplitMat& sm) {
          int64_t b = 0;
          for (const Slice& sl : sm.s) b += sl.m->pass_bytes();
          return b;
        };
        if (!d.active()) continue;
        st[5 * l + 0] += d.n_own();
        st[5 * l + 1] += pb(d.sA);
        for (auto& f : d.sF) st[5 * l + 2] += pb(f);
        for (auto& f : d.sB) st[5 * l + 2] += pb(f);
        st[5 * l + 3] += pb(d.sR);
        st[5 * l + 4] += pb(d.sP);
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
      h->stats[l].n = st[5 * l + 0];
      h->stats[l].a_pass = st[5 * l + 1];
      h->stats[l].m_pass = st[5 * l + 2];
      h->stats[l].r_pass = st[5 * l + 3];
      h->stats[l].p_pass = st[5 * l + 4];
    }
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  return h;
}

}  // namespace bmg

// ============================================================================ C ABI
using namespace bmg;

namespace {
const Bsr* B_(const bmg_bsr* a) { return reinterpret_cast<const Bsr*>(a); }
const Vec* V_(const bmg_vec* v) { return reinterpret_cast<const Vec*>(v); }
Vec* V_(bmg_vec* v) { return reinterpret_cast<Vec*>(v); }
const Fsai* M_(const bmg_fsai* m) { return reinterpret_cast<const Fsai*>(m); }
Hier* H_(bmg_hier* h) { return reinterpret_cast<Hier*>(h); }
const Hier* H_(const bmg_hier* h) { return reinterpret_cast<const Hier*>(h); }
void need_len(const Vec* v, int64_t n, const char* what) {
  if (v->n != n) fail(BMG_EINVAL, std::string(what) + ": vector length does not match layout");
}
// length of the finest-level vectors the caller passes
int64_t finest_len(const Hier& h) {
  const int top = h.finest();
  if (h.whole()) return h.parts[0].lv[top].n_own();
  if (h.emulated) return (int64_t)h.nbr[top] * h.msz[top] * h.nrhs;
  return h.parts[0].lv[top].n_own();
}
}  // namespace

extern "C" {

// setup (multilevel.cpp:36-75) with every step on the device
int bmg_hier_setup(const bmg_bsr* a_finest, int ntransfers, const bmg_bsr* const* transfers,
                   const bmg_setup_params* params, bmg_hier** out) {
  return guard([&] {
    bmg_setup_params prm;
    if (params)
      prm = *params;
    else
      bmg_setup_params_default(&prm);
    const Bsr* af = B_(a_finest);
    Ctx* ctx = af->ctx;
    ctx->activate();
    if (ntransfers < 0) fail(BMG_EINVAL, "setup: negative transfer count");
    auto h = std::make_unique<Hier>();
    h->ctx = ctx;
    h->parts.resize(1);
    Part& p = h->parts[0];
    const int depth = ntransfers;
    p.lv.resize(depth + 1);
    p.lv[depth].A = af;
    SetupClock clk(ctx);
    for (int l = depth; l >= 1; --l) {
      PLevel& L = p.lv[l];
      L.P = B_(transfers[l - 1]);
      L.R_own = bsr_transpose(*L.P);
      L.R = L.R_own.get();
      clk.mark("transpose P", l);
      p.lv[l - 1].A_own = galerkin(*L.A, *L.P);
      p.lv[l - 1].A = p.lv[l - 1].A_own.get();
      clk.mark("galerkin", l);
    }
    for (int l = 1; l <= depth; ++l) {
      PLevel& L = p.lv[l];
      L.M_own = fsai_build(*L.A, prm.fsai_kind, prm.t_max, prm.tau, prm.nest);
      L.M = L.M_own.get();
      clk.mark("fsai", l);
      const double beta = lanczos_lambda_max(*L.A, *L.M, prm.lanczos_iters, prm.lanczos_safety, prm.seed);
      clk.mark("lanczos", l);
      L.spec.kind = prm.smoother_kind;  // multilevel.cpp:62-65
      L.spec.beta = beta;
      L.spec.alpha = prm.first_kind_fraction * beta;
      L.spec.omega = prm.richardson_omega;
    }
    finish_whole(*h, prm.coarse_dim_cap);
    clk.mark("coarse factor + vectors", 0);
    *out = reinterpret_cast<bmg_hier*>(h.release());
  });
}

int bmg_hier_create(bmg_ctx* ctx, int nlevels, const bmg_bsr* const* A, const bmg_bsr* const* P,
                    const bmg_fsai* const* Mh, const double* beta, int coarse_dim_cap, bmg_hier** out) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->activate();
    if (nlevels < 1) fail(BMG_EINVAL, "hierarchy needs at least one level");
    auto h = std::make_unique<Hier>();
    h->ctx = c;
    h->parts.resize(1);
    Part& p = h->parts[0];
    p.lv.resize(nlevels);
    for (int l = 0; l < nlevels; ++l) {
      PLevel& L = p.lv[l];
      L.A = B_(A[l]);
      if (l >= 1) {
        L.P = B_(P[l]);
        if (L.P->dim_r != L.A->dim_r || L.P->dim_c != B_(A[l - 1])->dim_r)
          fail(BMG_EINVAL, "hierarchy: prolongation shape does not match the levels");
        L.R_own = bsr_transpose(*L.P);
        L.R = L.R_own.get();
        L.M = M_(Mh[l]);
        L.spec.kind = 2;
        L.spec.beta = beta[l];
        L.spec.alpha = beta[l] / 30.0;
        if (!(L.spec.beta > 0.0)) fail(BMG_EINVAL, "cheb_fourth_apply: beta must be positive");
      }
    }
    finish_whole(*h, coarse_dim_cap);
    *out = reinterpret_cast<bmg_hier*>(h.release());
  });
}

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

int bmg_hier_partition(bmg_hier* hh, int world, int rank, const int32_t* granule, int agglomerate) {
  return guard([&] {
    Hier* h = H_(hh);
    h->ctx->activate();
    partition(*h, world, rank, granule, agglomerate);
  });
}

int bmg_hier_part_info(const bmg_hier* hh, int level, int rank, int32_t* lo, int32_t* hi, int32_t* wlo,
                       int32_t* whi) {
  return guard([&] {
    const Hier* h = H_(hh);
    if (level < 0 || level > h->finest()) fail(BMG_ERANGE, "hierarchy: level out of range");
    if (rank < 0 || rank >= h->world) fail(BMG_ERANGE, "hierarchy: rank out of range");
    *lo = h->bounds[level][rank];
    *hi = h->bounds[level][rank + 1];
    *wlo = h->wlo[level][h->world == 1 ? 0 : rank];
    *whi = h->whi[level][h->world == 1 ? 0 : rank];
  });
}

int bmg_hier_destroy(bmg_hier* h) {
  return guard([&] {
    Hier* p = H_(h);
    if (p) BMG_CUDA(cudaStreamSynchronize(p->ctx->stream));
    delete p;
  });
}

int bmg_hier_info(const bmg_hier* hh, int* nlevels, int64_t* device_bytes) {
  return guard([&] {
    const Hier* h = H_(hh);
    if (nlevels) *nlevels = h->finest() + 1;
    if (device_bytes) {
      int64_t b = 0;
      for (const Part& p : h->parts) {
        b += (int64_t)(p.ainv.bytes() + p.cpart.bytes());
        for (const auto& L : p.lv) {
          if (L.A_own) b += L.A_own->device_bytes();
          if (L.R_own) b += L.R_own->device_bytes();
          if (L.P_own) b += L.P_own->device_bytes();
          if (L.M_own) {
            for (auto& f : L.M_own->fwd) b += f->device_bytes();
            for (auto& f : L.M_own->bwd) b += f->device_bytes();
          }
          for (int w = 0; w < VNUM; ++w) b += (int64_t)L.v[w].bytes();
          auto sb = [&](const SplitMat& sm) {
            for (const Slice& sl : sm.s)
              if (sl.own) b += sl.own->device_bytes();
          };
          sb(L.sA);
          sb(L.sR);
          sb(L.sP);
          for (auto& f : L.sF) sb(f);
          for (auto& f : L.sB) sb(f);
        }
      }
      *device_bytes = b;
    }
  });
}

int bmg_hier_beta(const bmg_hier* hh, int level, double* beta) {
  return guard([&] {
    const Hier* h = H_(hh);
    if (level < 1 || level > h->finest()) fail(BMG_ERANGE, "hierarchy: level out of range");
    *beta = h->parts[0].lv[level].spec.beta;
  });
}

int bmg_hier_set_smoother(bmg_hier* hh, int level, int kind, double alpha, double beta, double omega) {
  return guard([&] {
    Hier* h = H_(hh);
    if (level < 1 || level > h->finest()) fail(BMG_ERANGE, "hierarchy: level out of range");
    SmootherSpec s;
    s.kind = kind;
    s.alpha = alpha;
    s.beta = beta;
    s.omega = omega;
    smoother_schedule(s, 1);  // validates the spec
    for (Part& p : h->parts) p.lv[level].spec = s;
    h->drop_graphs();
  });
}

int bmg_hier_level(const bmg_hier* hh, int level, const bmg_bsr** a, const bmg_bsr** p, const bmg_fsai** m) {
  return guard([&] {
    const Hier* h = H_(hh);
    if (level < 0 || level > h->finest()) fail(BMG_ERANGE, "hierarchy: level out of range");
    const PLevel& L = h->parts[0].lv[level];
    if (a) *a = reinterpret_cast<const bmg_bsr*>(L.A);
    if (p) *p = reinterpret_cast<const bmg_bsr*>(L.P);
    if (m) *m = reinterpret_cast<const bmg_fsai*>(L.M);
  });
}

// algorithmic HBM bytes of one V(k_pre, k_post) cycle over all ranks (BASELINE.md
// §3 byte model, with the exact A*0 skip on coarse levels)
int bmg_hier_cycle_bytes(const bmg_hier* hh, int kpre, int kpost, int64_t* bytes) {
  return bmg_hier_cycle_bytes_batch(hh, kpre, kpost, 1, bytes);
}

// algorithmic bytes of one (batched) cycle: every matrix streamed once, vector
// traffic per right-hand side
int bmg_hier_cycle_bytes_batch(const bmg_hier* hh, int kpre, int kpost, int nrhs, int64_t* bytes) {
  return guard([&] {
    const Hier* h = H_(hh);
    const int64_t K = std::max(1, nrhs);
    int64_t tot = 0;
    const int top = h->finest();
    for (int l = 1; l <= top; ++l) {
      const LevelStats& s = h->stats[l];
      const int64_t n = s.n * K, nc = h->stats[l - 1].n * K;
      const int64_t apass = s.a_pass + 24 * n;  // x, b read; r write
      const int64_t gvec = 16 * n + 40 * n;     // G: r, w; G^T+cheb: w, p rw, x rw
      const int steps = kpre + kpost;
      int64_t lvl = steps * (apass + s.m_pass + gvec);
      if (l < top && kpre > 0) lvl -= apass + 8 * n;  // first coarse pre-step: A*0 skipped, x not read
      lvl += apass;                                   // residual before restriction
      lvl += s.r_pass + 8 * n + 8 * nc;               // restriction
      lvl += s.p_pass + 8 * nc + 16 * n;              // prolongation x += P e
      tot += lvl;
    }
    {  // coarse solve: packed lower tiles of A_0^{-1}, x, b, tile partials
      const int64_t nt = (h->n0 + 63) / 64;
      tot += nt * (nt + 1) / 2 * 64 * 64 * 8 + (16 * h->n0 + 2 * nt * nt * 64 * 8) * K;
    }
    *bytes = tot;
  });
}

int bmg_hier_use_graph(bmg_hier* hh, int on) {
  return guard([&] { H_(hh)->use_graph = on != 0; });
}

int bmg_vcycle(bmg_hier* hh, int kpre, int kpost, const bmg_vec* b, bmg_vec* x) {
  return bmg_vcycle_batch(hh, kpre, kpost, 1, b, x);
}

int bmg_vcycle_batch(bmg_hier* hh, int kpre, int kpost, int nrhs, const bmg_vec* b, bmg_vec* x) {
  return guard([&] {
    Hier* h = H_(hh);
    h->ctx->activate();
    set_nrhs(*h, nrhs);
    const int64_t n = finest_len(*h);
    need_len(V_(b), n, "v_cycle");
    need_len(V_(x), n, "v_cycle");
    run_vcycle(*h, kpre, kpost, V_(b)->d.p, V_(x)->d.p);
  });
}

int bmg_vcycle_host(bmg_hier* hh, int kpre, int kpost, const double* b, double* x) {
  return bmg_vcycle_batch_host(hh, kpre, kpost, 1, b, x);
}

int bmg_vcycle_batch_host(bmg_hier* hh, int kpre, int kpost, int nrhs, const double* b, double* x) {
  return guard([&] {
    Hier* h = H_(hh);
    Ctx* ctx = h->ctx;
    ctx->activate();
    set_nrhs(*h, nrhs);
    const int64_t n = finest_len(*h);
    if (h->io_b.n < (size_t)n) {
      h->io_b.alloc(std::max<int64_t>(n, 1));
      h->io_x.alloc(std::max<int64_t>(n, 1));
    }
    BMG_CUDA(cudaMemcpyAsync(h->io_b.p, b, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    BMG_CUDA(cudaMemcpyAsync(h->io_x.p, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
    run_vcycle(*h, kpre, kpost, h->io_b.p, h->io_x.p);
    BMG_CUDA(cudaMemcpyAsync(x, h->io_x.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  });
}

// residual-history driver modelled on measure_rates (experiments.cpp:15-67)
int bmg_solve(bmg_hier* hh, int kpre, int kpost, const bmg_vec* bh, bmg_vec* xh, double tol, int max_iter,
              double* hist, int* iters, int* status) {
  return guard([&] {
    Hier* h = H_(hh);
    set_nrhs(*h, 1);
    const int64_t n = finest_len(*h);
    need_len(V_(bh), n, "solve");
    need_len(V_(xh), n, "solve");
    const double* b = V_(bh)->d.p;
    double* x = V_(xh)->d.p;
    PLevel& F = h->parts[0].lv[h->finest()];
    auto resid = [&]() {
      finest_residual(*h, b, x, F.v[VR].p);
      return finest_norm(*h, F.v[VR].p);
    };
    hist[0] = resid();
    int it = 0, st = 1;
    if (hist[0] == 0.0) st = 0;
    while (st == 1 && it < max_iter) {
      run_vcycle(*h, kpre, kpost, b, x);
      ++it;
      hist[it] = resid();
      const double growth = hist[it] / std::max(hist[it - 1], 1e-300);
      if (!std::isfinite(hist[it]) || growth > 1e6) {
        st = 2;
        break;
      }
      if (hist[it] / hist[0] < tol) st = 0;
    }
    *iters = it;
    *status = st;
  });
}

int bmg_ctx_create_nccl(int device, int rank, int world, const unsigned char* id128, bmg_ctx** out) {
  return guard([&] {
    bmg_ctx* c = nullptr;
    const int st = bmg_ctx_create(device, &c);
    if (st != BMG_OK) fail(st, bmg_last_error());
    Ctx* ctx = reinterpret_cast<Ctx*>(c);
    std::unique_ptr<Ctx> own(ctx);
    ctx->comm = make_nccl_comm(rank, world, id128);
    ctx->rank = rank;
    ctx->world = world;
    *out = reinterpret_cast<bmg_ctx*>(own.release());
  });
}

int bmg_nccl_unique_id(unsigned char* id128) {
  return guard([&] { nccl_unique_id(id128); });
}

}  // extern "C"
