// hier.h -- internal data model of the device multilevel hierarchy, shared by
// hierarchy.cu (construction, partition, C ABI), vcycle.cu (halo exchange, the
// V-cycle and the solve loop) and dist_setup.cu (distributed setup).
//
// Every level of every (virtual) rank keeps its vectors in one contiguous window
// of global block rows [wlo, whi) that contains its own rows [lo, hi) plus the
// halo its matrices read; local matrices index columns as `global - wlo`.  A halo
// exchange therefore moves contiguous slices: rank s sends [max(lo_s, wlo_r),
// min(hi_s, whi_r)) to rank r.  Per-row arithmetic does not depend on the
// partition, so partitioned cycles are bitwise equal to the 1-GPU cycle.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <tuple>
#include <vector>

#include "bmg_internal.h"

namespace bmg {
namespace kern {

// Coarse solve x = A_0^{-1} b with the symmetric inverse stored as packed lower
// 64 x 64 tiles (half the bytes of a dense GEMV).  Each tile (I, J), J <= I,
// contributes tile * x_J to rows of I and (J < I) tile^T * x_I to rows of J;
// partials are summed per row in ascending tile order (deterministic).
constexpr int kTile = 64;
// right-hand sides per batched cycle: 1, 2, 4 or kMaxRhs (set_nrhs enforces it; the
// coarse solve's x staging in symv_stream_kernel is sized by it)
constexpr int kMaxRhs = 8;

__device__ __forceinline__ void tile_of(int64_t t, int* I, int* J) {
  int i = (int)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while ((int64_t)(i + 1) * (i + 2) / 2 <= t) ++i;
  while ((int64_t)i * (i + 1) / 2 > t) --i;
  *I = i;
  *J = (int)(t - (int64_t)i * (i + 1) / 2);
}

}  // namespace kern

inline int grid1d(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

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

// Half-storage A on one rank's share of a partitioned level (vcycle.cu
// sym_residual_pass): the rows' blocks up to the diagonal -- those in the lower halo
// (columns below the own ones: row dots only, their mirrors live on another rank)
// and the in-rank lower triangle (row dots + transposed products) -- streamed as two
// slices (rows that read the lower halo first); the in-rank upper blocks come from
// the transposed products in column order (merge); blocks past the own columns
// (upper halo) finish the last rows in a tail pass.  Every row's sum keeps the
// reference's column order, so the pass is bitwise the full-storage one.
struct PSym {
  std::unique_ptr<Bsr> low_bnd, low_int;  // rows [0, k1), [k1, n) of the lower part
  int k1 = 0, n = 0, m = 0, oc0 = 0;      // oc0: the first own column in the window
  int64_t nlow_bnd = 0;                   // lower blocks of low_bnd (colpart / brow offset of low_int)
  DBuf<int32_t> brow;                     // per lower block: window block index of its row
  int64_t brow_int_off = 0;               // low_int's entries start here (16-byte aligned)
  DBuf<int64_t> up_ptr;                   // [n + 1]
  DBuf<int32_t> up_slot;                  // in-rank upper blocks (ascending columns) -> lower block ids
  DBuf<double> colpart, sbuf, tbuf;
  std::unique_ptr<Bsr> tail;              // rows [t0, n): blocks past the own columns
  int t0 = 0;
  int64_t pass_bytes = 0;                 // algorithmic bytes of one pass (matrix + scratch)
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
  std::unique_ptr<PSym> psym;          // half-storage A (partitioned levels; whole ones use Bsr::half)
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
  ShrinkBuf ainv;  // A_0^{-1} as packed lower 64x64 tiles (rank owning level 0), or
                      // W = L^{-1} (A_0 = L L^T) when the coarse level is triangular
  bool tri = false;   // coarse solve as x = W^T (W b): N0^2 >= 2^31 (no 64-bit potri)
  DBuf<double> cpart; // per-(tile row, tile) partial sums of the coarse solve
};

struct LevelStats {  // global byte model inputs (bmg_hier_cycle_bytes)
  int64_t n = 0, a_pass = 0, m_pass = 0, r_pass = 0, p_pass = 0;
  int64_t a_pass_ref = 0;  // full-storage A pass (the reference's storage; 0: = a_pass)
};

struct GraphKey {
  int kpre, kpost, nrhs, top;
  const double* b;
  double* x;
  int kind = 0;  // 0 cycle on device vectors; 1 cycle on the caller's host buffers
                // (copies inside the graph); bmg_solve steps: 2 residual norm, 3 cycle +
                // residual norm (segment sums copied to pinned memory inside the graph)
  bool operator<(const GraphKey& o) const {
    return std::tie(kpre, kpost, nrhs, top, b, x, kind) < std::tie(o.kpre, o.kpost, o.nrhs, o.top, o.b, o.x, o.kind);
  }
};

// Host-buffer cycles (bmg_vcycle_host): b and x go up in row slices on a copy
// stream and the first residual r = b - A x runs per slice as soon as the rows it
// reads have landed, so the upload overlaps the first pass.
struct HostIo {
  std::vector<std::unique_ptr<Plan>> plans;  // row-range plans of the finest A
  std::vector<std::unique_ptr<Plan>> sym_plans;  // ... of its lower triangle (half-storage A)
  cudaEvent_t ev_b = nullptr;                // b landed (half-storage path)
  std::vector<int> row0, row1, need;         // slice rows; last slice whose x it reads
  cudaStream_t cs = nullptr;
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> ev;               // slice s landed
  ~HostIo() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (fork) cudaEventDestroy(fork);
    if (ev_b) cudaEventDestroy(ev_b);
    if (cs) cudaStreamDestroy(cs);
  }
};

struct Hier {
  CtxRef ctx;
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
  std::vector<char> psym_on;  // per level: partitioned A passes in half storage (build_level_psym)
  bool use_graph = true;
  struct Captured {
    cudaGraphExec_t exec;
    int64_t kernels;
  };
  double* h_seg = nullptr;  // pinned copy of the residual's segment sums (bmg_solve)
  int h_seg_n = 0;
  std::map<GraphKey, Captured> graphs;
  std::map<GraphKey, int> warm;  // transport hierarchies: keys already run once eagerly
  DBuf<double> io_b, io_x, seg;
  cudaStream_t comm = nullptr;  // halo exchanges overlap interior slices
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  const double* user_b = nullptr;
  double* user_x = nullptr;
  std::unique_ptr<HostIo> hio;
  bool skip_top_res = false;  // the top level's first residual is already in its r
  std::vector<const Bsr*> held_bsr;    // caller objects the levels point to
  std::vector<const Fsai*> held_fsai;
  void hold(const Bsr* a) {
    bsr_retain(a);
    held_bsr.push_back(a);
  }
  void hold(const Fsai* m) {
    fsai_retain(m);
    held_fsai.push_back(m);
  }
  ~Hier() {
    if (ctx) cudaStreamSynchronize(ctx->stream);
    parts.clear();  // level objects first, then the caller objects they point to
    for (const Bsr* a : held_bsr) bsr_release(a);
    for (const Fsai* m : held_fsai) fsai_release(m);
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (comm) cudaStreamDestroy(comm);
    if (h_seg) cudaFreeHost(h_seg);
  }
  int finest() const { return (int)nbr.size() - 1; }
  int top = -1;  // level the current cycle starts on (v_cycle's `level`; -1: finest)
  int cycle_top() const { return top >= 0 ? top : finest(); }
  bool whole() const { return world == 1; }
  void drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
    warm.clear();
  }
};

// vector of level l on part p; the unpartitioned top level uses the caller's b, x
inline double* vec(Hier& h, Part& p, int l, Which w) {
  if (h.whole() && l == h.cycle_top()) {
    if (w == VB) return const_cast<double*>(h.user_b);
    if (w == VX) return h.user_x;
  }
  return p.lv[l].v[w].p;
}

// ---- shared operations (vcycle.cu, hierarchy.cu) --------------------------------
void exchange(Hier& h, int l, Which w);
void set_nrhs(Hier& h, int K);
void run_vcycle(Hier& h, int kpre, int kpost, const double* bf, double* xf);
// whole single-RHS hierarchies with pinned host b, x and kpre > 0: the pipelined
// host-buffer cycle; false if it does not apply (the caller copies around run_vcycle)
bool run_vcycle_hostio(Hier& h, int kpre, int kpost, const double* hb, double* hx);
void ensure_host_io(Hier& h, int64_t n);
// bmg_solve on whole single-RHS hierarchies: each iteration (cycle, residual,
// segment sums to pinned memory) is one graph launch; the stopping test stays on
// the host in the oracle's order; false if it does not apply (the caller runs the
// eager loop)
bool solve_device(Hier& h, int kpre, int kpost, const double* b, double* x, double tol, int max_iter, double* hist,
                  int* iters, int* status);
double finest_norm(Hier& h, const double* r_whole);
void finest_residual(Hier& h, const double* b, double* x, double* rtmp);
void coarse_factor(Hier& h, Part& p);
void measure_rates(Hier& h, const Bsr& mass, const double* b, const double* u, int kpre, int kpost, uint64_t seed,
                   double tol, int max_iter, double* l2_sq, double* energy_sq, double* resid, int* iters,
                   int* status, int* blowup, double* rates);
void alloc_vectors(Hier& h, PLevel& L, bool top);
// half-storage A on every eligible partitioned level of h (after the parts are built
// and the setup's own A passes are done); consistent over all ranks
void build_level_psym(Hier& h);
std::unique_ptr<Bsr> slice_rows(const Bsr& g, int lo, int hi, int col_lo, int ncols);
SplitMat split_rows(const Bsr& g, int lo, int hi, int wlo, int nwin, int own_lo, int own_hi);

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

// ---- C ABI handle casts ----------------------------------------------------------
inline const Bsr* B_(const bmg_bsr* a) { return reinterpret_cast<const Bsr*>(a); }
inline const Vec* V_(const bmg_vec* v) { return reinterpret_cast<const Vec*>(v); }
inline Vec* V_(bmg_vec* v) { return reinterpret_cast<Vec*>(v); }
inline const Fsai* M_(const bmg_fsai* m) { return reinterpret_cast<const Fsai*>(m); }
inline Hier* H_(bmg_hier* h) { return reinterpret_cast<Hier*>(h); }
inline const Hier* H_(const bmg_hier* h) { return reinterpret_cast<const Hier*>(h); }
inline void need_len(const Vec* v, int64_t n, const char* what) {
  if (v->n != n) fail(BMG_EINVAL, std::string(what) + ": vector length does not match layout");
}
// length of the finest-level vectors the caller passes
inline int64_t finest_len(const Hier& h) {
  const int top = h.finest();
  if (h.whole()) return h.parts[0].lv[top].n_own();
  if (h.emulated) return (int64_t)h.nbr[top] * h.msz[top] * h.nrhs;
  return h.parts[0].lv[top].n_own();
}

}  // namespace bmg
