// bsr_stream.cuh -- the sm_100a block-sparse streaming kernel and its epilogues.
//
// One kernel shape serves every pass of the V-cycle:
//   y = A x                      spmv            (kernels.cpp:39-47)
//   r = b - A x                  residual        (chebyshev.hpp:55-56, multilevel.cpp:91-93)
//   w = G r                      FSAI first half (fsai.cpp:203-211, with S-hat folded into G)
//   z = G^T w; p, x update       FSAI second half + Chebyshev (fsai.cpp:212-215,
//                                                   chebyshev.hpp:57-59,63-66)
//   rc = R r  (R = P^T)          restriction     (multilevel.cpp:95)
//   x += P e                     prolongation    (multilevel.cpp:98-100)
//
// Design (uniform block sizes, the BASELINE configs):
//   * The host plan (build_plan) gives each CTA a contiguous range of block rows
//     balanced by blocks; the rows' value span is contiguous in HBM and is cut
//     into chunks of cb_max blocks (rows may straddle chunks; a per-CTA carry
//     holds the partial row sum).
//   * One producer thread streams chunks into a 2-stage (BMG_STAGES) shared-
//     memory ring with cp.async.bulk (TMA bulk copy, mbarrier complete_tx):
//     values and the chunk's column indices, with an L2 evict-first policy so
//     the gathered vectors stay in L2.  HBM sees large sequential transfers;
//     nothing is re-read (DRAM bytes = algorithmic bytes under ncu).
//   * m = 20: blocks are copied one by one to a shared-memory pitch of bs + 2
//     doubles and quarter-warps span two blocks (SKEW), which removes the bank
//     conflicts of the 160-byte row pitch.  m = 21: a pitch of bs + 4 doubles and
//     22 lanes per block (PAD21), m = 15: 16 lanes per block (HALF): every
//     half-warp of 8-byte loads covers the 16 bank pairs once.
//   * m >= 15 kernels carry a 3-CTA register budget (stream_min_blocks): their
//     chunks fill shared memory at 3 CTAs per SM anyway, and with 72 registers
//     ptxas issues an item's x gathers before the first fma of its chain.
//   * Consumers (8 warps) compute per-(block, scalar row) dot products from
//     shared memory against x gathered through L1/L2 (phase A), release the
//     stage, then sum each row's partials in ascending block order and run the
//     fused epilogue with coalesced vector traffic (phase B).  Partials and the
//     row carry are double-buffered: one named barrier per chunk.
//   * Programmatic dependent launch: dependents are released at entry, vector
//     accesses wait for the predecessor (griddepcontrol).
//   * K > 1 right-hand sides interleaved per scalar row share each staged block
//     (this kernel's gather form, or bsr_batch_kernel below: staged x segments,
//     row-per-thread items; the host picks per (m, K) from measured sweeps);
//     VAR streams a variable layout through zero-padded MR x MC block copies.
//   * Arithmetic order matches the oracle exactly: t = fma-chain over columns
//     from 0.0, then y += t per block in ascending column order, so results
//     are bitwise identical to oracle/bmg_oracle.cpp spmv.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace bmg {
namespace kern {

constexpr int kMaxStages = 8;
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = kConsumerWarps * 32;
constexpr int kThreads = kConsumers + 32;
constexpr unsigned kCarryIn = 1u << 30;
constexpr unsigned kCarryOut = 1u << 31;
constexpr unsigned kRowMask = kCarryIn - 1;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Streamed-once data (matrix blocks and column indices, the coarse inverse's
// tiles) is copied with an L2 evict-first policy, so the stream does not push the
// gathered vectors (x, a few MB, re-read by every block row's neighbours) out of
// the 126 MB L2 while hundreds of MB pass through it.  BMG_L2_HINT=0 disables.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// stream copy: evict-first when `hint`, else the default policy
__device__ __forceinline__ void bulk_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar, bool hint,
                                            uint64_t pol) {
  if (hint)
    bulk_g2s_hint(dst, src, bytes, bar, pol);
  else
    bulk_g2s(dst, src, bytes, bar);
}
// Programmatic dependent launch (sm_90+): the next pass may start streaming its
// matrix while this one drains; vector reads/writes wait for the predecessor.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kConsumers) : "memory");
}

// ---------------------------------------------------------------- epilogues
// Each epilogue receives the scalar output index and the finished row sum y.
// load() issues the epilogue's own vector reads early (before the chunk's
// matrix data has landed) so their latency hides behind phase A.
struct EpiStore {
  double* y;
  struct Pre {};
  __device__ __forceinline__ double init(int64_t) const { return 0.0; }
  __device__ __forceinline__ Pre load(int64_t) const { return {}; }
  __device__ __forceinline__ void store(int64_t i, double v, const Pre&) const { y[i] = v; }
};
struct EpiResidual {  // r = b - A x
  const double* b;
  double* r;
  struct Pre {
    double b;
  };
  __device__ __forceinline__ double init(int64_t) const { return 0.0; }
  __device__ __forceinline__ Pre load(int64_t i) const { return {__ldg(b + i)}; }
  __device__ __forceinline__ void store(int64_t i, double v, const Pre& p) const { r[i] = __dsub_rn(p.b, v); }
};
struct EpiAdd {  // x += P e
  double* x;
  struct Pre {
    double x;
  };
  __device__ __forceinline__ double init(int64_t) const { return 0.0; }
  __device__ __forceinline__ Pre load(int64_t i) const { return {x[i]}; }
  __device__ __forceinline__ void store(int64_t i, double v, const Pre& p) const { x[i] = __dadd_rn(p.x, v); }
};
// z = G^T w; p = first ? z : (mu*mu) p + z; x += (d*mu) p   (chebyshev.hpp:57-59,63-66)
struct EpiCheb {
  double* p;
  double* x;
  double mu2, dmu;
  int first, xzero;
  struct Pre {
    double p, x;
  };
  __device__ __forceinline__ double init(int64_t) const { return 0.0; }
  __device__ __forceinline__ Pre load(int64_t i) const {
    return {first ? 0.0 : p[i], xzero ? 0.0 : x[i]};
  }
  __device__ __forceinline__ void store(int64_t i, double z, const Pre& q) const {
    const double pn = first ? z : __dadd_rn(__dmul_rn(mu2, q.p), z);
    p[i] = pn;
    const double inc = __dmul_rn(dmu, pn);
    x[i] = xzero ? inc : __dadd_rn(q.x, inc);
  }
};

// r = b - (t + A x): the row sum continues from t (a partial sum of the same row's
// earlier blocks, in column order) -- the last segment of a half-storage pass on a
// partitioned level, whose blocks past the rank's own columns come last in the row
struct EpiResidualFrom {
  const double* t;
  const double* b;
  double* r;
  struct Pre {
    double b;
  };
  __device__ __forceinline__ double init(int64_t i) const { return t[i]; }
  __device__ __forceinline__ Pre load(int64_t i) const { return {__ldg(b + i)}; }
  __device__ __forceinline__ void store(int64_t i, double v, const Pre& p) const { r[i] = __dsub_rn(p.b, v); }
};

struct StreamArgs {
  const double* vals;
  const int32_t* col;
  const int64_t* row_ptr;
  const int4* chunks;
  const int* cta_chunk;
  const double* x;
  int bs;      // padded block stride (doubles)
  int cb_max;  // blocks per chunk
  int rmax;    // rows per chunk
  int stages;  // shared-memory ring depth (<= kMaxStages)
  // variable layouts streamed as MR x MC padded blocks (VAR kernels): block
  // offsets / sizes of the real layout, x length for clamped gathers
  const int* coff = nullptr;
  const int* roff = nullptr;
  const int* rsz = nullptr;
  int64_t xlen = 0;
  int l2hint = 1;  // matrix stream with the L2 evict-first policy
  // SYM kernels (lower triangle of an exactly symmetric A): row index of every
  // streamed block (bulk-copied beside the column indices) and the output of the
  // transposed products A_ij^T x_i, MC doubles per block at the block's index
  const int32_t* brow = nullptr;
  double* colpart = nullptr;
  int colmap = 2;  // SYM column items: 0 block-major, 1 block-fastest tiles, 2 block-fastest full tiles +
                   // block-major remainder (BMG_SYM_COLMAP; 2 measured best)
  int sym_lo = 0;  // SYM: blocks in columns below this one (a partitioned level's lower halo)
                   // have no stored mirror here: row dots only
};

// column-index slots per stage: cb_max + 8, rounded to 16 bytes (bulk-copy
// destinations must be 16-byte aligned)
__host__ __device__ inline int stage_cols_of(int cb_max) { return (cb_max + 8 + 3) & ~3; }

struct SmemLayout {
  uint32_t vals, cols, rows, part, carry, bars, total;
  __host__ __device__ SmemLayout(int bs, int cb_max, int rmax, int mr, int kStages, int nrhs = 1, bool sym = false) {
    uint32_t o = 0;
    auto al = [](uint32_t v, uint32_t a) { return (v + a - 1) / a * a; };
    (void)rmax;
    vals = o;
    o += al((uint32_t)kStages * cb_max * bs * 8, 128);
    cols = o;
    o += al((uint32_t)kStages * stage_cols_of(cb_max) * 4, 128);
    rows = o;  // block row indices (SYM)
    if (sym) o += al((uint32_t)kStages * stage_cols_of(cb_max) * 4, 128);
    part = o;  // double-buffered partial sums
    o += al((uint32_t)2 * cb_max * mr * (nrhs > 1 ? nrhs + 1 : 1) * 8, 16);
    carry = o;  // double-buffered row carry
    o += al((uint32_t)2 * mr * nrhs * 8, 16);
    bars = o;
    o += 2 * kStages * 8;
    total = al(o, 128);
  }
};

// K right-hand sides interleaved per scalar row (x[i * K + v]): one matrix stream
// serves K vectors; each RHS keeps the single-vector arithmetic order.
// VAR: a variable layout whose blocks are stored padded to MR x MC with zeros; the
// zero padding adds exact zeros to every fma chain, so each real entry keeps the
// oracle's arithmetic order; padded rows are computed and never stored.
// SYM: the streamed matrix is the lower triangle (diagonal included) of an exactly
// symmetric A.  Besides the row dots, every off-diagonal block (i, j) computes the
// transposed product A_ij^T x_i -- the contribution of the unstored block (j, i)
// to row j -- as column dots over the staged block (fma chain over the block's
// rows ascending: the same chain as the row dot of the stored transpose) and
// writes it to colpart; the row sums (lower blocks only) go to the epilogue, and
// sym_merge_kernel adds the upper contributions in ascending column order.
#ifndef BMG_PAD21
#define BMG_PAD21 1  // m = 21: 22 lanes per block at a shared-memory pitch of bs + 4 (bmg_core.cu follows it)
#endif
#ifndef BMG_SYM_CPT1_MASK
#define BMG_SYM_CPT1_MASK 0
#endif
// columns per SYM column item (bit m of BMG_SYM_CPT1_MASK: one column per item)
constexpr int sym_cpt(int mc) {
  return ((BMG_SYM_CPT1_MASK >> mc) & 1) ? 1 : (mc % 2 == 0) ? 2 : ((mc % 3 == 0) ? 3 : 1);
}
// Register budget.  Blocks of m >= 15 stream 24-36 KB chunks through a two-stage ring,
// so shared memory holds 3 CTAs per SM whatever the registers; telling ptxas so
// (65536 / (3 x 288) = 75 registers instead of the 47-56 it settles on unasked) lets
// it issue a whole item's x gathers before the first fma of the chain instead of
// trickling them in between the dependent fmas (SASS: 12 + 8 loads hoisted instead
// of 5 + 4 in the m = 15 half-storage kernel).  Measured on whole cycles: C5 shape
// 14.4 -> 16.1 V-cycles/s, C3 shape 16.1 -> 16.5, C4 20.0 -> 20.5.  m <= 10 keeps the
// default: 4 CTAs of its smaller chunks fit and need <= 56 registers (C2 474 -> 462
// with the 3-CTA budget).
// (0 = no hint)  Batched kernels (K > 1) keep the default too.
constexpr int stream_min_blocks(int mr, int k) { return (mr >= 15 && k == 1) ? 3 : 0; }
template <int MR, int MC, int K, class Epi, bool VAR = false, bool SYM = false>
__global__ void __launch_bounds__(kThreads, stream_min_blocks(MR, K)) bsr_stream_kernel(StreamArgs s, Epi epi) {
  static_assert(!SYM || (K == 1 && !VAR && MR == MC), "SYM streams uniform square blocks, one RHS");
  extern __shared__ __align__(128) unsigned char smem[];
  const int kStages = s.stages;
  // SKEW (m = 20): blocks land in shared memory at a pitch of bs + 2 doubles (one
  // bulk copy per block) and a quarter-warp takes rows 4k..4k+3 of two adjacent
  // blocks: the 160-byte row pitch alone maps rows r and r + 4 of a block to the
  // same banks (2-way conflicts on every 16-byte load, 2.5e8 per C4 coarse pass)
  constexpr bool SKEW = (MR == 20 && MC == 20 && K == 1 && !VAR);
  // PAD21 (m = 21): 22 lanes per block (one idle) and a pitch of bs + 4 = 446 doubles
  // (one bulk copy per block).  8-byte loads are served per half-warp; with 21 lanes
  // per block at the packed pitch the half-warps that straddle two blocks hit three
  // bank pairs twice (1.64x the wavefronts of the row items, ~52 M per C3-shape
  // pass).  Lane g of a chunk reads double offset 446 j + 21 r + q with g = 22 j + r:
  // 13 (446 j + 21 r) = 6 j + r = g (mod 16), so any 16 consecutive lanes cover the
  // 16 bank pairs once.
  constexpr bool PAD21 = BMG_PAD21 && (MR == 21 && MC == 21 && K == 1 && !VAR);
  const int pitch = SKEW ? s.bs + 2 : (PAD21 ? s.bs + 4 : s.bs);
  const SmemLayout L(pitch, s.cb_max, s.rmax, MR, kStages, K, SYM);
  // partials of one (block, row) item for K > 1 sit at stride K + 1 (bank spread)
  constexpr int KP = K > 1 ? K + 1 : 1;
  double* vals_s = reinterpret_cast<double*>(smem + L.vals);
  int* cols_s = reinterpret_cast<int*>(smem + L.cols);
  int* rows_s = reinterpret_cast<int*>(smem + L.rows);
  double* part_s = reinterpret_cast<double*>(smem + L.part);
  double* carry_s = reinterpret_cast<double*>(smem + L.carry);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kStages;

  const int c0 = s.cta_chunk[blockIdx.x];
  const int c1 = s.cta_chunk[blockIdx.x + 1];
  const int tid = threadIdx.x;
  // single-wave persistent grid: every CTA is resident, so the dependent pass can
  // be scheduled as soon as SMs free up
  pdl_launch_dependents();
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int stage_vals = s.cb_max * pitch;
  const int stage_cols = stage_cols_of(s.cb_max);

  if (tid >= kConsumers) {
    // ------------------------------------------------------------ producer
    if (tid == kConsumers) {
      const uint64_t pol = l2_evict_first_policy();
      for (int c = c0, it = 0; c < c1; ++c, ++it) {
        const int st = it % kStages;
        if (it >= kStages) mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
        const int4 d = s.chunks[c];
        if (d.y == 0) {
          mbar_arrive_expect_tx(&full[st], 0);
          continue;
        }
        const uint32_t vbytes = (uint32_t)d.y * (uint32_t)s.bs * 8u;
        const int cl = d.x & ~3;
        const int ch = (d.x + d.y + 3) & ~3;
        const uint32_t cbytes = (uint32_t)(ch - cl) * 4u;
        mbar_arrive_expect_tx(&full[st], vbytes + (SYM ? 2 : 1) * cbytes);
        if constexpr (SYM) bulk_stream(rows_s + st * stage_cols, s.brow + cl, cbytes, &full[st], s.l2hint, pol);
        if constexpr (SKEW || PAD21) {
          for (int b = 0; b < d.y; ++b)
            bulk_stream(vals_s + (size_t)st * stage_vals + b * pitch, s.vals + (int64_t)(d.x + b) * s.bs,
                        (uint32_t)s.bs * 8u, &full[st], s.l2hint, pol);
        } else {
          bulk_stream(vals_s + (size_t)st * stage_vals, s.vals + (int64_t)d.x * s.bs, vbytes, &full[st], s.l2hint,
                      pol);
        }
        bulk_stream(cols_s + st * stage_cols, s.col + cl, cbytes, &full[st], s.l2hint, pol);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  pdl_wait();  // vectors (x, b, p, outputs) belong to the predecessor pass
  // One named barrier per chunk: partial sums and the row carry are double
  // buffered, so phase B of chunk c overlaps phase A of chunk c+1.
  for (int c = c0, it = 0; c < c1; ++c, ++it) {
    const int st = it % kStages;
    const int pb = it & 1;
    const int4 d = s.chunks[c];
    const int nrows = (int)((unsigned)d.w & kRowMask);
    const bool cin = ((unsigned)d.w & kCarryIn) != 0;
    const bool cout = ((unsigned)d.w & kCarryOut) != 0;
    double* part = part_s + pb * s.cb_max * MR * KP;

    // early loads for this thread's first phase-B item (row bounds + epilogue inputs)
    const int ritems = nrows * MR * K;
    int64_t rlo0 = 0, rhi0 = 0;
    typename Epi::Pre pre0{};
    if (tid < ritems) {
      const int rr = tid / (MR * K);
      const int rv = tid - rr * MR * K;
      rlo0 = __ldg(s.row_ptr + d.z + rr);
      rhi0 = __ldg(s.row_ptr + d.z + rr + 1);
      if constexpr (VAR) {
        if (rv / K < __ldg(s.rsz + d.z + rr))
          pre0 = epi.load(((int64_t)__ldg(s.roff + d.z + rr) + rv / K) * K + (rv - (rv / K) * K));
      } else {
        pre0 = epi.load((int64_t)(d.z + rr) * MR * K + rv);
      }
    }
    mbar_wait(&full[st], (it / kStages) & 1);

    // phase A: partial dot products per (block, scalar row)
    const double* vs = vals_s + (size_t)st * stage_vals;
    const int* cs = cols_s + st * stage_cols + (d.x & 3);
    if constexpr (K > 1) {
      // items (block, rhs, row group), row group fastest: each thread gathers one
      // RHS column of the block's x segment once and reuses it for the rows
      // g, g + RG, ...; lanes of one RHS read consecutive rows of the staged block
      constexpr int RG = MR / K > 0 ? MR / K : 1;
      constexpr int RPG = (MR + RG - 1) / RG;
      const int kitems = d.y * RG * K;
      for (int item = tid; item < kitems; item += kConsumers) {
        const int b = item / (RG * K);
        const int rem = item - b * RG * K;
        const int v = rem / RG, g = rem - (rem / RG) * RG;
        const double* __restrict__ xj = s.x + (int64_t)cs[b] * MC * K + v;
        double xv[MC];
        if constexpr (VAR) {
          const int64_t x0 = (int64_t)__ldg(s.coff + cs[b]);
#pragma unroll
          for (int q = 0; q < MC; ++q) xv[q] = __ldg(s.x + min(x0 + q, s.xlen - 1) * K + v);
        } else {
#pragma unroll
          for (int q = 0; q < MC; ++q) xv[q] = __ldg(xj + q * K);
        }
        const double* ab = vs + b * s.bs;
#pragma unroll
        for (int rr = 0; rr < RPG; ++rr) {
          const int r = g + RG * rr;
          if (r < MR) {
            const double* a = ab + r * MC;
            double t = 0.0;
            if constexpr (MC % 2 == 0) {
#pragma unroll
              for (int q = 0; q < MC / 2; ++q) {
                const double2 a2 = reinterpret_cast<const double2*>(a)[q];
                t = __fma_rn(a2.x, xv[2 * q], t);
                t = __fma_rn(a2.y, xv[2 * q + 1], t);
              }
            } else {
#pragma unroll
              for (int q = 0; q < MC; ++q) t = __fma_rn(a[q], xv[q], t);
            }
            part[(b * MR + r) * KP + v] = t;
          }
        }
      }
    }
    // HALF (m = 15): 16 lanes per block (one idle), so a half-warp -- one wavefront
    // of 8-byte loads -- reads the 15 rows of one block: the 120-byte row pitch
    // spreads them over distinct bank pairs, while two blocks in one half-warp collide
    constexpr bool HALF = (MR == 15 && MC == 15 && K == 1 && !VAR);
    constexpr int LPB = HALF ? 16 : (PAD21 ? 22 : MR);
    const int items = K > 1 ? 0 : d.y * LPB;
    for (int item = tid; item < items; item += kConsumers) {
      int b = item / LPB;
      int r = item - b * LPB;
      if ((HALF || PAD21) && r >= MR) continue;
      if constexpr (SKEW) {  // pairs of blocks: quarter k of a pair = rows 4k..4k+3 of both
        const int pair = item / (2 * MR);
        if (2 * pair + 1 < d.y) {
          const int w = item - pair * 2 * MR;
          b = 2 * pair + ((w & 7) >> 2);
          r = 4 * (w >> 3) + (w & 3);
        }
      }
      const int j = cs[b];
      const double* __restrict__ xj = s.x + (int64_t)j * MC * K;
      const double* a = vs + b * pitch + r * MC;
      if constexpr (K > 1) {
        // unreachable: K > 1 uses the (block, row group, rhs) items below
        continue;
      }
      double xv[MC];
      if constexpr (VAR) {
        const int64_t x0 = (int64_t)__ldg(s.coff + j);
#pragma unroll
        for (int q = 0; q < MC; ++q) xv[q] = __ldg(s.x + min(x0 + q, s.xlen - 1));
      } else if constexpr (MC % 2 == 0) {
#pragma unroll
        for (int q = 0; q < MC / 2; ++q) {
          const double2 t2 = __ldg(reinterpret_cast<const double2*>(xj) + q);
          xv[2 * q] = t2.x;
          xv[2 * q + 1] = t2.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < MC; ++q) xv[q] = __ldg(xj + q);
      }
      double t = 0.0;
      if constexpr (MC % 2 == 0) {
#pragma unroll
        for (int q = 0; q < MC / 2; ++q) {
          const double2 a2 = reinterpret_cast<const double2*>(a)[q];
          t = __fma_rn(a2.x, xv[2 * q], t);
          t = __fma_rn(a2.y, xv[2 * q + 1], t);
        }
      } else {
#pragma unroll
        for (int q = 0; q < MC; ++q) t = __fma_rn(a[q], xv[q], t);
      }
      part[b * MR + r] = t;
    }
    if constexpr (SYM) {  // transposed products of the off-diagonal blocks
      // an item is CPT adjacent columns of one block: x_i is loaded once for them
      // and even block sizes read two columns per 16-byte shared-memory load
      constexpr int CPT = sym_cpt(MC);
      constexpr int NCG = MC / CPT;
      // items run block-fastest within tiles of BB blocks, so the lanes of one
      // shared-memory wavefront read the same column group of different blocks,
      // whose pitch spreads them over distinct banks (16-byte loads: m = 20 pitch
      // 402 -> 2 doubles apart, 8 blocks; m = 10 / 6: 4 apart, 4 blocks x 2
      // groups; 8-byte loads, m = 15 / 21: 8 blocks x 2 groups, even + odd)
      constexpr int BB = (MC == 10 || MC == 6) ? 4 : 8;
      const int* rs = rows_s + st * stage_cols + (d.x & 3);
      const bool tiled = s.colmap != 0;
      // colmap 2: only the chunk's full tiles run block-fastest, the remaining blocks
      // block-major (a partial tile leaves most lanes of its wavefronts idle)
      const int ntiled = !tiled ? 0 : (s.colmap == 2 ? (d.y / BB) * BB : ((d.y + BB - 1) / BB) * BB) * NCG;
      const int citems = !tiled ? d.y * NCG : (s.colmap == 2 ? d.y * NCG : ntiled);
      for (int item = tid; item < citems; item += kConsumers) {
        int b, c0;
        if (item < ntiled) {
          const int tile = item / (BB * NCG);
          const int k = item - tile * BB * NCG;
          b = tile * BB + (k % BB);
          c0 = (k / BB) * CPT;
          if (b >= d.y) continue;
        } else {
          b = item / NCG;
          c0 = (item - b * NCG) * CPT;
        }
        const int i = rs[b];
        if (cs[b] == i || cs[b] < s.sym_lo) continue;  // diagonal / lower-halo block: row dots only
        const double* __restrict__ xi = s.x + (int64_t)i * MR;
        double xv[MR];
        if constexpr (MR % 2 == 0) {
#pragma unroll
          for (int q = 0; q < MR / 2; ++q) {
            const double2 t2 = __ldg(reinterpret_cast<const double2*>(xi) + q);
            xv[2 * q] = t2.x;
            xv[2 * q + 1] = t2.y;
          }
        } else {
#pragma unroll
          for (int q = 0; q < MR; ++q) xv[q] = __ldg(xi + q);
        }
        const double* a = vs + b * pitch + c0;
        double t[CPT];
#pragma unroll
        for (int q = 0; q < CPT; ++q) t[q] = 0.0;
#pragma unroll
        for (int r = 0; r < MR; ++r) {
          if constexpr (CPT == 2) {
            const double2 a2 = *reinterpret_cast<const double2*>(a + r * MC);
            t[0] = __fma_rn(a2.x, xv[r], t[0]);
            t[1] = __fma_rn(a2.y, xv[r], t[1]);
          } else {
#pragma unroll
            for (int q = 0; q < CPT; ++q) t[q] = __fma_rn(a[r * MC + q], xv[r], t[q]);
          }
        }
        double* out = s.colpart + (int64_t)(d.x + b) * MC + c0;
#pragma unroll
        for (int q = 0; q < CPT; ++q) out[q] = t[q];
      }
    }
    consumer_bar();
    if (tid == 0) mbar_arrive(&empty[st]);

    // phase B: ordered row sums + fused epilogue
    const double* carry_in = carry_s + (pb ^ 1) * MR * K;
    double* carry_out = carry_s + pb * MR * K;
    for (int item = tid; item < ritems; item += kConsumers) {
      const int rr = item / (MR * K);
      const int rv = item - rr * MR * K;  // r * K + v
      int64_t rlo = rlo0, rhi = rhi0;
      typename Epi::Pre pre = pre0;
      int64_t oi = (int64_t)(d.z + rr) * MR * K + rv;  // output index
      bool real = true;
      if constexpr (VAR) {
        real = rv / K < __ldg(s.rsz + d.z + rr);
        oi = ((int64_t)__ldg(s.roff + d.z + rr) + rv / K) * K + (rv - (rv / K) * K);
      }
      if (item != tid) {
        rlo = __ldg(s.row_ptr + d.z + rr);
        rhi = __ldg(s.row_ptr + d.z + rr + 1);
        if (real) pre = epi.load(oi);
      }
      const int lo = (int)(max(rlo, (int64_t)d.x) - d.x);
      const int hi = (int)(min(rhi, (int64_t)(d.x + d.y)) - d.x);
      double acc = (rr == 0 && cin) ? carry_in[rv] : epi.init(oi);
      const int r = rv / K, v = rv - (rv / K) * K;
      for (int b = lo; b < hi; ++b) acc = __dadd_rn(acc, part[(b * MR + r) * KP + v]);
      if (rr == nrows - 1 && cout)
        carry_out[rv] = acc;
      else if (real)
        epi.store(oi, acc, pre);
    }
  }
}

// Second half of a SYM pass: y_i = S_i + sum over the upper blocks (i, j), j > i
// ascending, of the transposed products A_ji^T x_j left in colpart by the
// blocks (j, i) -- the reference's row sum continued in its column order
// (kernels.cpp:39-47: blocks ascending, y += block * x_j), so r = b - A x comes
// out bitwise equal to the full-storage pass.  One thread per scalar row; the
// slots and partials of eight upper blocks are loaded before they are added.
// Scalar rows from tsplit on are written to tbuf instead (partitioned levels: a
// tail pass adds the row's blocks beyond the rank's own columns).
template <int MR, class Epi>
__global__ void __launch_bounds__(256) sym_merge_kernel(const int64_t* __restrict__ up_ptr,
                                                        const int32_t* __restrict__ up_slot,
                                                        const double* __restrict__ colpart,
                                                        const double* __restrict__ S, int64_t n, Epi epi,
                                                        double* __restrict__ tbuf, int64_t tsplit) {
  pdl_launch_dependents();
  pdl_wait();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / MR;
    const int r = (int)(e - i * MR);
    const typename Epi::Pre pre = epi.load(e);
    double y = S[e];
    const int64_t u0 = __ldg(up_ptr + i), u1 = __ldg(up_ptr + i + 1);
    int64_t u = u0;
    constexpr int U = 8;  // partials in flight per thread (coarse 3-D rows hold ~230 upper blocks)
    for (; u + U <= u1; u += U) {
      int sl[U];
      double c[U];
#pragma unroll
      for (int q = 0; q < U; ++q) sl[q] = __ldg(up_slot + u + q);
#pragma unroll
      for (int q = 0; q < U; ++q) c[q] = __ldg(colpart + (int64_t)sl[q] * MR + r);
#pragma unroll
      for (int q = 0; q < U; ++q) y = __dadd_rn(y, c[q]);
    }
    for (; u < u1; ++u) y = __dadd_rn(y, __ldg(colpart + (int64_t)__ldg(up_slot + u) * MR + r));
    if (e >= tsplit)
      tbuf[e - tsplit] = y;  // rows continued by a tail pass (EpiResidualFrom)
    else
      epi.store(e, y, pre);
  }
}

// ------------------------------------------------ batched right-hand sides
// K > 1 right-hand sides on uniform layouts.  The producer warp stages, per
// block, both the block (one bulk copy per chunk) and the block's x segment
// x[j*MC*K, (j+1)*MC*K) -- contiguous because the K right-hand sides are
// interleaved per scalar row -- so phase A reads only shared memory and the x
// gathers' L2 latency sits in the async ring instead of the consumers.  A
// phase-A item is (block, scalar row, RHS group of V = K / U): the block row is
// read from shared memory U times in total (not K times), the staged x segment
// is read by the MR row threads of the block together (broadcast), and every
// (row, RHS) keeps the single-vector fma chain over columns from 0.0.
// Partials are stored unpadded at stride K per (block, row) slot with the
// 16-byte pieces XOR-swizzled by slot, so the phase-A stores and the phase-B
// reads are bank-conflict free.
// staged x segment stride (doubles): +2 shifts consecutive segments by 16 bytes of banks
__host__ __device__ inline int batch_xstride(int mc, int K) { return mc * K + 2; }

struct BatchSmem {
  uint32_t vals, xs, part, carry, bars, total;
  __host__ __device__ BatchSmem(int bs, int cb_max, int mr, int mc, int K, int kStages) {
    uint32_t o = 0;
    auto al = [](uint32_t v, uint32_t a) { return (v + a - 1) / a * a; };
    vals = o;
    o += al((uint32_t)kStages * cb_max * bs * 8, 128);
    xs = o;
    o += al((uint32_t)kStages * cb_max * batch_xstride(mc, K) * 8, 128);
    part = o;
    o += al((uint32_t)2 * cb_max * mr * K * 8, 16);
    carry = o;
    o += al((uint32_t)2 * mr * K * 8, 16);
    bars = o;
    o += 2 * kStages * 8;
    total = al(o, 128);
  }
};

// physical double index of (slot, v) in the swizzled partials
template <int K>
__device__ __forceinline__ int batch_part_idx(int slot, int v) {
  constexpr int P = K / 2;        // 16-byte pieces per slot
  constexpr int RPL = 8 / P;      // slots per 128-byte line
  return slot * K + ((((v >> 1) ^ ((slot / RPL) % P))) << 1) + (v & 1);
}

// XL: the x segments do not go through the TMA engine (which the matrix stream
// already keeps busy) but are gathered by the consumer threads with read-only
// 16-byte loads through L1 -- consecutive chunks of a CTA reuse most segments, so
// L1 serves them -- one chunk ahead into registers, and stored to a
// parity-indexed shared buffer at the end of the previous chunk's phase A (before
// the chunk's one barrier).  Chunks hold at most batch_xl_cb(MR) blocks then.
__host__ __device__ constexpr int batch_xl_cb(int mr) { return mr <= 10 ? 32 : (mr <= 15 ? 16 : 8); }

template <int MR, int MC, int K, int U, class Epi, bool XL = false>
__global__ void __launch_bounds__(kThreads, (MR <= 10 || K / U < 8) ? 3 : 2) bsr_batch_kernel(StreamArgs s, Epi epi) {
  static_assert(K % 2 == 0 && K <= 8 && K % U == 0 && (K / U) % 2 == 0, "batch shape");
  constexpr int V = K / U;  // right-hand sides per thread
  constexpr int XS = MC * K + 2;  // == batch_xstride(MC, K)
  extern __shared__ __align__(128) unsigned char smem[];
  const int kStages = s.stages;
  const BatchSmem L(s.bs, s.cb_max, MR, MC, K, kStages);
  double* vals_s = reinterpret_cast<double*>(smem + L.vals);
  double* xs_s = reinterpret_cast<double*>(smem + L.xs);
  double* part_s = reinterpret_cast<double*>(smem + L.part);
  double* carry_s = reinterpret_cast<double*>(smem + L.carry);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* empty = full + kStages;

  const int c0 = s.cta_chunk[blockIdx.x];
  const int c1 = s.cta_chunk[blockIdx.x + 1];
  const int tid = threadIdx.x;
  pdl_launch_dependents();
  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();

  const int stage_vals = s.cb_max * s.bs;
  const int stage_xs = s.cb_max * XS;

  if (tid >= kConsumers) {
    // ------------------------------------------------------ producer warp
    // chunks hold at most 32 blocks (host plan: cb_max = kConsumers / (MR U) <= 25),
    // so lane b owns block b's x segment; the next chunk's descriptor and column
    // indices are loaded one chunk ahead, off the empty-slot wait
    const int lane = tid - kConsumers;
    const uint64_t pol = l2_evict_first_policy();
    constexpr uint32_t xbytes = (uint32_t)MC * K * 8u;
    bool waited = false;
    int4 dn = c0 < c1 ? s.chunks[c0] : make_int4(0, 0, 0, 0);
    int jn = lane < dn.y ? __ldg(s.col + dn.x + lane) : 0;
    for (int c = c0, it = 0; c < c1; ++c, ++it) {
      const int st = it % kStages;
      const int4 d = dn;
      const int j = jn;
      if (c + 1 < c1) dn = s.chunks[c + 1];
      if (lane == 0 && it >= kStages) mbar_wait(&empty[st], ((it / kStages) - 1) & 1);
      __syncwarp();
      if (d.y == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&full[st], 0);
      } else {
        if (lane == 0) {
          const uint32_t vbytes = (uint32_t)d.y * (uint32_t)s.bs * 8u;
          mbar_arrive_expect_tx(&full[st], vbytes + (XL ? 0u : (uint32_t)d.y * xbytes));
          bulk_stream(vals_s + (size_t)st * stage_vals, s.vals + (int64_t)d.x * s.bs, vbytes, &full[st], s.l2hint,
                      pol);
        }
        if (!waited) {  // x belongs to the predecessor pass (the matrix does not)
          pdl_wait();
          waited = true;
        }
        __syncwarp();
        if (!XL && lane < d.y)
          bulk_g2s(xs_s + (size_t)st * stage_xs + lane * XS, s.x + (int64_t)j * MC * K, xbytes, &full[st]);
      }
      jn = (c + 1 < c1 && lane < dn.y) ? __ldg(s.col + dn.x + lane) : 0;
    }
    return;
  }

  // ------------------------------------------------------------ consumers
  pdl_wait();
  // XL staging: pieces (16 bytes) of the chunk's x segments, thread t takes pieces
  // t, t + kConsumers, ...
  constexpr int PPB = MC * K / 2;
  constexpr int NP = XL ? (batch_xl_cb(MR) * PPB + kConsumers - 1) / kConsumers : 1;
  double2 xr[NP];
  int xo[NP];
  auto xload = [&](int c) {
#pragma unroll
    for (int k = 0; k < NP; ++k) xo[k] = -1;
    if (c >= c1) return;
    const int4 d = s.chunks[c];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const int p = tid + k * kConsumers;
      if (p < d.y * PPB) {
        const int b = p / PPB;
        const int o = p - b * PPB;
        const int j = __ldg(s.col + d.x + b);
        xr[k] = __ldg(reinterpret_cast<const double2*>(s.x + (int64_t)j * MC * K) + o);
        xo[k] = b * XS + 2 * o;
      }
    }
  };
  auto xstore = [&](double* dst) {
#pragma unroll
    for (int k = 0; k < NP; ++k)
      if (xo[k] >= 0) *reinterpret_cast<double2*>(dst + xo[k]) = xr[k];
  };
  if constexpr (XL) {
    xload(c0);
    xstore(xs_s);
    xload(c0 + 1);
    consumer_bar();
  }
  for (int c = c0, it = 0; c < c1; ++c, ++it) {
    const int st = it % kStages;
    const int pb = it & 1;
    const int4 d = s.chunks[c];
    const int nrows = (int)((unsigned)d.w & kRowMask);
    const bool cin = ((unsigned)d.w & kCarryIn) != 0;
    const bool cout = ((unsigned)d.w & kCarryOut) != 0;
    double* part = part_s + pb * s.cb_max * MR * K;

    const int ritems = nrows * MR * K;
    int64_t rlo0 = 0, rhi0 = 0;
    typename Epi::Pre pre0{};
    if (tid < ritems) {
      const int rr = tid / (MR * K);
      const int rv = tid - rr * MR * K;
      rlo0 = __ldg(s.row_ptr + d.z + rr);
      rhi0 = __ldg(s.row_ptr + d.z + rr + 1);
      pre0 = epi.load((int64_t)(d.z + rr) * MR * K + rv);
    }
    mbar_wait(&full[st], (it / kStages) & 1);

    // phase A: item = (block, rhs group, row), row fastest
    const double* vs = vals_s + (size_t)st * stage_vals;
    const double* xs = xs_s + (size_t)(XL ? pb : st) * stage_xs;
    const int items = d.y * MR * U;
    for (int item = tid; item < items; item += kConsumers) {
      const int b = item / (MR * U);
      const int rem = item - b * (MR * U);
      const int u = rem / MR;
      const int r = rem - u * MR;
      const double* a = vs + b * s.bs + r * MC;
      const double* xb = xs + b * XS + u * V;
      double acc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = 0.0;
      if constexpr (MC % 2 == 0) {
#pragma unroll
        for (int q2 = 0; q2 < MC / 2; ++q2) {
          const double2 a2 = reinterpret_cast<const double2*>(a)[q2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double aq = h ? a2.y : a2.x;
            const double2* xq = reinterpret_cast<const double2*>(xb + (2 * q2 + h) * K);
#pragma unroll
            for (int v2 = 0; v2 < V / 2; ++v2) {
              const double2 x2 = xq[v2];
              acc[2 * v2] = __fma_rn(aq, x2.x, acc[2 * v2]);
              acc[2 * v2 + 1] = __fma_rn(aq, x2.y, acc[2 * v2 + 1]);
            }
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < MC; ++q) {
          const double aq = a[q];
          const double2* xq = reinterpret_cast<const double2*>(xb + q * K);
#pragma unroll
          for (int v2 = 0; v2 < V / 2; ++v2) {
            const double2 x2 = xq[v2];
            acc[2 * v2] = __fma_rn(aq, x2.x, acc[2 * v2]);
            acc[2 * v2 + 1] = __fma_rn(aq, x2.y, acc[2 * v2 + 1]);
          }
        }
      }
      const int slot = b * MR + r;
#pragma unroll
      for (int v2 = 0; v2 < V / 2; ++v2) {
        const int v = u * V + 2 * v2;
        *reinterpret_cast<double2*>(part + batch_part_idx<K>(slot, v)) = make_double2(acc[2 * v2], acc[2 * v2 + 1]);
      }
    }
    if constexpr (XL) {  // the next chunk's x into the other buffer, then the one after into registers
      xstore(xs_s + (size_t)(pb ^ 1) * stage_xs);
      xload(c + 2);
    }
    consumer_bar();
    if (tid == 0) mbar_arrive(&empty[st]);

    // phase B: ordered row sums + fused epilogue (same order as the K = 1 kernel)
    const double* carry_in = carry_s + (pb ^ 1) * MR * K;
    double* carry_out = carry_s + pb * MR * K;
    for (int item = tid; item < ritems; item += kConsumers) {
      const int rr = item / (MR * K);
      const int rv = item - rr * MR * K;  // r * K + v
      int64_t rlo = rlo0, rhi = rhi0;
      typename Epi::Pre pre = pre0;
      const int64_t oi = (int64_t)(d.z + rr) * MR * K + rv;
      if (item != tid) {
        rlo = __ldg(s.row_ptr + d.z + rr);
        rhi = __ldg(s.row_ptr + d.z + rr + 1);
        pre = epi.load(oi);
      }
      const int lo = (int)(max(rlo, (int64_t)d.x) - d.x);
      const int hi = (int)(min(rhi, (int64_t)(d.x + d.y)) - d.x);
      double acc = (rr == 0 && cin) ? carry_in[rv] : 0.0;
      const int r = rv / K, v = rv - (rv / K) * K;
      for (int b = lo; b < hi; ++b) acc = __dadd_rn(acc, part[batch_part_idx<K>(b * MR + r, v)]);
      if (rr == nrows - 1 && cout)
        carry_out[rv] = acc;
      else
        epi.store(oi, acc, pre);
    }
  }
}

// ------------------------------------------------------ variable block sizes
// Warp per block row, lane per scalar row (looping for m_i > 32); same
// arithmetic order as the streaming kernel and the oracle.
struct VarArgs {
  const double* vals;
  const int32_t* col;
  const int64_t* row_ptr;
  const int64_t* voff;
  const int* roff;
  const int* rsz;
  const int* coff;
  const int* csz;
  const double* x;
  int nbr;
  int nrhs;  // right-hand sides interleaved per scalar row
};

template <class Epi>
__global__ void __launch_bounds__(256) bsr_var_kernel(VarArgs s, Epi epi) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= s.nbr) return;
  const int mi = s.rsz[warp];
  const int64_t b0 = s.row_ptr[warp], b1 = s.row_ptr[warp + 1];
  const int K = s.nrhs;
  for (int r0 = 0; r0 < mi * K; r0 += 32) {
    const int rv = r0 + lane;  // r * K + v
    const int r = rv / K, v = rv - (rv / K) * K;
    double acc = 0.0;
    for (int64_t b = b0; b < b1; ++b) {
      const int j = s.col[b];
      const int mj = s.csz[j];
      const double* xj = s.x + (int64_t)s.coff[j] * K + v;
      const double* a = s.vals + s.voff[b];
      if (r < mi) {
        double t = 0.0;
        for (int q = 0; q < mj; ++q) t = __fma_rn(a[(int64_t)r * mj + q], __ldg(xj + (int64_t)q * K), t);
        acc = __dadd_rn(acc, t);
      }
    }
    if (r < mi) {
      const int64_t i = ((int64_t)s.roff[warp] + r) * K + v;
      epi.store(i, acc, epi.load(i));
    }
  }
}

}  // namespace kern
}  // namespace bmg
