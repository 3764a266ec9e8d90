// bmg_core.cu -- context, device BSR storage + streaming plans, vectors, the
// streaming-kernel launchers, reductions and the corresponding C ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "bmg_abi.h"
#include "bmg_internal.h"
#include "bsr_stream.cuh"

namespace bmg {

// ============================================================================ errors
[[noreturn]] void fail(int status, const std::string& msg, int pivot) { throw Error(status, msg, pivot); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(BMG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void debug_sync(cudaStream_t s, const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("BMG_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  cuda_check(cudaGetLastError(), what);
  if (!on) return;
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) return;
  cuda_check(cudaStreamSynchronize(s), what);
}

thread_local std::string g_last_error;
thread_local int g_last_pivot = -1;

// ============================================================================ context
uint64_t next_object_uid() {
  static std::atomic<uint64_t> n{1};
  return n++;
}

Ctx::~Ctx() {
  // at process exit the runtime may already be unloading: the driver reclaims
  // everything, and communicators / library handles must not be torn down then
  if (cudaFree(nullptr) == cudaErrorCudartUnloading) {
    (void)comm.release();
    return;
  }
  for (auto& kv : smoother_graphs) cudaGraphExecDestroy(kv.second);
  comm.reset();
  if (solver) cusolverDnDestroy(solver);
  if (blas) cublasDestroy(blas);
  if (h_red) cudaFreeHost(h_red);
  if (own) cudaStreamDestroy(own);
}

void bsr_retain(const Bsr* a) {
  if (a) a->refs.fetch_add(1, std::memory_order_relaxed);
}
void bsr_release(const Bsr* a) {
  if (a && a->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete a;
}
void fsai_retain(const Fsai* m) {
  if (m) m->refs.fetch_add(1, std::memory_order_relaxed);
}
void fsai_release(const Fsai* m) {
  if (m && m->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete m;
}

void ctx_retain(Ctx* c) {
  if (c) c->refs.fetch_add(1, std::memory_order_relaxed);
}
void ctx_release(Ctx* c) {
  if (c && c->refs.fetch_sub(1, std::memory_order_acq_rel) == 1) delete c;
}

cublasHandle_t Ctx::cublas() {
  if (!blas) {
    if (cublasCreate(&blas) != CUBLAS_STATUS_SUCCESS) fail(BMG_ECUDA, "cublasCreate failed");
  }
  cublasSetStream(blas, stream);
  return blas;
}

cusolverDnHandle_t Ctx::cusolver() {
  if (!solver) {
    if (cusolverDnCreate(&solver) != CUSOLVER_STATUS_SUCCESS) fail(BMG_ECUDA, "cusolverDnCreate failed");
  }
  cusolverDnSetStream(solver, stream);
  return solver;
}

// ============================================================================ kernels
namespace kern {

__global__ void fill_kernel(double* p, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void copy_kernel(double* __restrict__ d, const double* __restrict__ s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

// z = alpha x + beta y, each product and the sum rounded separately (no fma):
// the reference's Eigen vector expressions r = b - t, p = mu*mu*p + t and
// x += d*mu*p (chebyshev.hpp:55-66, built with -ffp-contract=off in the oracle)
// are this with (alpha, beta) = (1, -1), (mu*mu, 1), (1, d*mu) -- exact scalings
// by +-1 leave the other operand unchanged.
__global__ void axpby_kernel(double* z, double alpha, const double* x, double beta,
                             const double* y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = __dadd_rn(__dmul_rn(alpha, x[i]), __dmul_rn(beta, y[i]));
}

constexpr int kDotBlocks = 592;
constexpr int kDotThreads = 256;

// deterministic two-stage dot: fixed segments per block, fixed tree order
__global__ void __launch_bounds__(kDotThreads) dot_stage1(const double* __restrict__ a,
                                                          const double* __restrict__ b, int64_t n,
                                                          double* partial) {
  __shared__ double sh[kDotThreads];
  const int64_t seg = (n + kDotBlocks - 1) / kDotBlocks;
  const int64_t lo = blockIdx.x * seg;
  const int64_t hi = min(n, lo + seg);
  double s = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += kDotThreads) s = __fma_rn(a[i], b[i], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = kDotThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}
__global__ void __launch_bounds__(1024) dot_stage2(const double* partial, double* out) {
  __shared__ double sh[1024];
  sh[threadIdx.x] = threadIdx.x < kDotBlocks ? partial[threadIdx.x] : 0.0;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] = __dadd_rn(sh[threadIdx.x], sh[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

// per-block transpose through a permutation of blocks (uniform layouts)
__global__ void transpose_uniform_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                         const int64_t* __restrict__ perm, int64_t nnzb, int mr,
                                         int mc, int bs_src, int bs_dst) {
  const int64_t total = nnzb * (int64_t)(mr * mc);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / (mr * mc);
    const int q = (int)(e - t * (mr * mc));
    const int r = q / mr, c = q - r * mr;  // dst block is mc x mr: (r, c) = src (c, r)
    dst[t * bs_dst + q] = src[perm[t] * bs_src + (int64_t)c * mc + r];
  }
}
__global__ void transpose_var_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                     const int64_t* __restrict__ perm,
                                     const int64_t* __restrict__ voff_src,
                                     const int64_t* __restrict__ voff_dst,
                                     const int* __restrict__ trow_of, const int* __restrict__ tcol,
                                     const int* __restrict__ tsz_r, const int* __restrict__ tsz_c,
                                     int64_t nnzb) {
  for (int64_t t = blockIdx.x; t < nnzb; t += gridDim.x) {
    const int mr = tsz_r[trow_of[t]], mc = tsz_c[tcol[t]];  // dst block mr x mc
    const int64_t s0 = voff_src[perm[t]], d0 = voff_dst[t];
    for (int q = threadIdx.x; q < mr * mc; q += blockDim.x) {
      const int r = q / mc, c = q - r * mc;
      dst[d0 + q] = src[s0 + (int64_t)c * mr + r];
    }
  }
}

}  // namespace kern

static int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 16));
}

void fill(Ctx* ctx, double* p, int64_t n, double v) {
  if (n <= 0) return;
  kern::fill_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(p, n, v);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
}
void copy(Ctx* ctx, double* dst, const double* src, int64_t n) {
  if (n <= 0 || dst == src) return;
  kern::copy_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(dst, src, n);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
}

void axpby(Ctx* ctx, double* z, double alpha, const double* x, double beta, const double* y, int64_t n) {
  if (n <= 0) return;
  kern::axpby_kernel<<<grid_for(n), 256, 0, ctx->stream>>>(z, alpha, x, beta, y, n);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
}

double dot(Ctx* ctx, const double* a, const double* b, int64_t n) {
  if (ctx->red.n < (size_t)kern::kDotBlocks + 8) ctx->red.alloc(kern::kDotBlocks + 8);
  if (!ctx->h_red) BMG_CUDA(cudaMallocHost(&ctx->h_red, 8 * sizeof(double)));
  kern::dot_stage1<<<kern::kDotBlocks, kern::kDotThreads, 0, ctx->stream>>>(a, b, n, ctx->red.p);
  kern::dot_stage2<<<1, 1024, 0, ctx->stream>>>(ctx->red.p, ctx->red.p + kern::kDotBlocks);
  ctx->count(2);
  BMG_CUDA(cudaGetLastError());
  BMG_CUDA(cudaMemcpyAsync(ctx->h_red, ctx->red.p + kern::kDotBlocks, sizeof(double),
                           cudaMemcpyDeviceToHost, ctx->stream));
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  return ctx->h_red[0];
}

// ============================================================================ BSR
int64_t Bsr::pass_bytes() const {
  // algorithmic bytes of one streaming pass: every block's values + its column index
  int64_t v = 0;
  if (uniform)
    v = nnzb * ((int64_t)mr * mc * 8 + 4);
  else
    for (int i = 0; i < nbr; ++i)
      for (int64_t p = h_row_ptr[i]; p < h_row_ptr[i + 1]; ++p) v += (int64_t)rsz[i] * csz[h_col[p]] * 8 + 4;
  return v;
}
int64_t Bsr::device_bytes() const {
  return (int64_t)(row_ptr.bytes() + col.bytes() + vals.bytes() + voff.bytes() + d_roff.bytes() +
                   d_coff.bytes() + d_rsz.bytes() + d_csz.bytes() + plan.chunks.bytes() +
                   plan.cta_chunk.bytes()) +
         (half ? half->bytes() : 0);
}

static bool stream_supported(int mr, int mc) {
  return mr == mc && (mr == 3 || mr == 6 || mr == 10 || mr == 15 || mr == 20 || mr == 21);
}

static int ring_stages() {
  static int v = [] {
    const char* e = std::getenv("BMG_STAGES");
    int st = e ? std::atoi(e) : 2;
    return std::max(2, std::min(st, kern::kMaxStages));
  }();
  return v;
}

// chunk size: about one phase-A item per consumer thread, capped in bytes so
// several CTAs fit per SM.  Caps measured on B200 (tools/kernel_sweep.py, residual
// pass on each config family's fine operator): 24 KB for m = 10 and 20, 32 KB for
// m = 15 and 21.  BMG_CHUNK_KB overrides the cap for every m.
static int chunk_blocks(int mr, int bs, int K = 1, bool sym = false) {
  static int env_cap = [] {
    const char* e = std::getenv("BMG_CHUNK_KB");
    if (!e) return 0;
    int kb = std::atoi(e);
    if (kb < 2) kb = 2;
    if (kb > 48) kb = 48;
    return kb * 1024;
  }();
  // measured sweeps (profiles/r01_kernel_sweep.jsonl, r01_batched_spmv_sweep.jsonl):
  // batched 3-D m = 20 wants more blocks per barrier, batched m = 10 fewer
  // m = 20: 32 KB measured on whole C4 cycles (72.5 ms against 73.8 at 24 KB;
  // the coarse levels' 285 / 462-block rows gain most)
  int kb = (mr == 15 || mr == 21 || mr == 20) ? 32 : 24;
  if (K > 1 && mr == 20) kb = 48;
  // the half-storage pass (twice the consumer work per staged block) on m = 20: 11
  // blocks per chunk, still 3 CTAs per SM (C4 fine residual + G pair 2.50 -> 2.42 ms;
  // 40 KB drops to 2 CTAs: 2.68)
  // m = 21 likewise: 10 blocks per chunk (C3 shape 17.79 -> 17.94 V-cycles/s)
  if (sym && (mr == 20 || mr == 21)) kb = 36;
  if (K == 8 && mr == 10) kb = 16;
  const int cap = env_cap ? env_cap : kb * 1024;
  // small blocks: several phase-A items per consumer thread, so a chunk still
  // carries enough bytes per barrier (BMG_SMALL_ITEMS overrides the factor)
  static const int env_items = [] {
    const char* e = std::getenv("BMG_SMALL_ITEMS");
    return e ? std::max(1, std::atoi(e)) : 0;
  }();
  const int per_thread = mr >= 10 ? 1 : (env_items ? env_items : 3);  // measured: m = 3 3.1 -> 4.2, m = 6 5.9 -> 6.1 TB/s
  // m = 15 takes 16 lanes per block in bsr_stream_kernel (bank-conflict-free rows)
  // ... and m = 21 takes 22 (PAD21)
  const int lanes = (K == 1 && mr == 15) ? 16 : ((BMG_PAD21 && K == 1 && mr == 21) ? 22 : mr);
  const int by_items = std::max(1, per_thread * kern::kConsumers / lanes);
  const int by_bytes = std::max(1, cap / (bs * 8));
  return std::min(by_items, by_bytes);
}

// shared-memory attributes of one instantiation: the largest dynamic size; batched
// (K > 1) kernels also ask for a larger shared-memory carveout (their partials grow
// with K) but not the maximum: the x gathers live in L1; K = 1 keeps the default
template <class F>
static void stream_attrs(F kfn, int K) {
  BMG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  if (K > 1)  // ~196 KB of shared memory (3 CTAs of the batched plans), ~60 KB left to L1 for x
    BMG_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributePreferredSharedMemoryCarveout, 86));
}

template <int MR, int MC, int K>
static int stream_occupancy(size_t smem) {
  auto kfn = kern::bsr_stream_kernel<MR, MC, K, kern::EpiStore>;
  stream_attrs(kfn, K);
  int occ = 0;
  BMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kern::kThreads, smem));
  return std::max(occ, 1);
}

template <int MR>
static int sym_occupancy(size_t smem) {
  auto kfn = kern::bsr_stream_kernel<MR, MR, 1, kern::EpiStore, false, true>;
  stream_attrs(kfn, 1);
  int occ = 0;
  BMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kern::kThreads, smem));
  return std::max(occ, 1);
}
static int sym_occupancy_for(int mr, size_t smem) {
  switch (mr) {
    case 3: return sym_occupancy<3>(smem);
    case 6: return sym_occupancy<6>(smem);
    case 10: return sym_occupancy<10>(smem);
    case 15: return sym_occupancy<15>(smem);
    case 20: return sym_occupancy<20>(smem);
    case 21: return sym_occupancy<21>(smem);
  }
  return 1;
}

template <int MR, int MC>
static int occupancy_k(size_t smem, int K) {
  switch (K) {
    case 2: return stream_occupancy<MR, MC, 2>(smem);
    case 4: return stream_occupancy<MR, MC, 4>(smem);
    case 8: return stream_occupancy<MR, MC, 8>(smem);
  }
  return stream_occupancy<MR, MC, 1>(smem);
}

static int occupancy_for(int mr, int mc, size_t smem, int K = 1) {
  switch (mr) {
    case 3: return occupancy_k<3, 3>(smem, K);
    case 6: return occupancy_k<6, 6>(smem, K);
    case 10: return occupancy_k<10, 10>(smem, K);
    case 15: return occupancy_k<15, 15>(smem, K);
    case 20: return occupancy_k<20, 20>(smem, K);
    case 21: return occupancy_k<21, 21>(smem, K);
  }
  return 1;
}

// ---- batched (K > 1) streaming kernel: RHS groups and occupancy
template <int MR, int K, int U>
static int batch_occupancy(size_t smem) {
  auto kfn = kern::bsr_batch_kernel<MR, MR, K, U, kern::EpiStore>;
  stream_attrs(kfn, K);
  int occ = 0;
  BMG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kfn, kern::kThreads, smem));
  return std::max(occ, 1);
}
template <int MR>
static int batch_occupancy_m(size_t smem, int K, int U) {
  if (K == 2) return batch_occupancy<MR, 2, 1>(smem);
  if (K == 4) return U == 1 ? batch_occupancy<MR, 4, 1>(smem) : batch_occupancy<MR, 4, 2>(smem);
  return U == 1 ? batch_occupancy<MR, 8, 1>(smem) : batch_occupancy<MR, 8, 2>(smem);
}
static int batch_occupancy_for(int mr, size_t smem, int K, int U) {
  switch (mr) {
    case 10: return batch_occupancy_m<10>(smem, K, U);
    case 15: return batch_occupancy_m<15>(smem, K, U);
    case 20: return batch_occupancy_m<20>(smem, K, U);
    case 21: return batch_occupancy_m<21>(smem, K, U);
  }
  return 1;
}
// Which kernel streams K > 1 right-hand sides, with its RHS groups U (V = K / U
// per thread), blocks per chunk and x path (bulk copies or XL consumer gathers),
// from measured sweeps on B200 (profiles/r01_batched_kernel_sweep.txt,
// r01_batched_xl_sweep.txt).  The staged-x kernel wins where blocks
// are large (m = 15 for K <= 4, m = 20, 21: up to 2x) and for m = 10 at K = 8;
// for m = 10 at K <= 4 the chunk count per byte is high and the per-chunk
// staging latency loses to the L1 gathers of bsr_stream_kernel.  BMG_BATCH_KERNEL=old|new, BMG_BATCH_U and
// BMG_BATCH_CB override (sweeps).
struct BatchChoice {
  int u = 0;   // 0: bsr_stream_kernel<K>; else bsr_batch_kernel with U groups
  int cb = 0;  // blocks per chunk (0: kConsumers / (mr U))
  int xl = 0;  // x segments gathered by the consumers through L1 (else bulk-copied)
};
static BatchChoice batch_choice(int mr, int K) {
  static const int env_k = [] {
    const char* e = std::getenv("BMG_BATCH_KERNEL");
    return !e ? -1 : (e[0] == 'n' ? 1 : 0);
  }();
  static const int env_u = [] {
    const char* e = std::getenv("BMG_BATCH_U");
    return e ? std::atoi(e) : 0;
  }();
  static const int env_cb = [] {
    const char* e = std::getenv("BMG_BATCH_CB");
    return e ? std::atoi(e) : 0;
  }();
  BatchChoice c;
  if (mr < 10) return c;  // small blocks (m = 3, 6): the gather kernel only
  switch (mr) {
    case 10: if (K == 8) c = {1, 16}; else if (K == 2) c = {1, 25, 1}; break;
    case 15: if (K == 2) c = {1, 16}; else if (K == 4) c = {2, 20}; break;
    case 20: c = K == 2 ? BatchChoice{1, 8, 1} : BatchChoice{1, 8}; break;
    case 21: c = {1, 8}; break;
    default: break;
  }
  if (env_k == 0) c = {};
  if (env_k == 1 && c.u == 0) c = {1, 0};
  auto valid = [&](int u) { return (u == 1 || u == 2) && (K / u) % 2 == 0; };
  if (c.u && valid(env_u)) c.u = env_u;
  if (c.u && env_cb > 0) c.cb = env_cb;
  static const int env_xl = [] {
    const char* e = std::getenv("BMG_BATCH_XL");
    return e ? std::atoi(e) : -1;
  }();
  if (c.u && env_xl >= 0) c.xl = env_xl ? 1 : 0;
  if (K != 2) c.xl = 0;  // instantiated for K = 2 only
  if (c.xl) {
    const int cap = kern::batch_xl_cb(mr);
    if (c.cb <= 0 || c.cb > cap) c.cb = std::min(cap, std::max(1, kern::kConsumers / (mr * c.u)));
  }
  return c;
}

// Partition block rows into per-CTA ranges balanced by blocks; cut each
// range's contiguous block span into chunks of cb_max blocks (bsr_stream.cuh).
// plan for streaming `a` as uniform mr x mr blocks of stride bs (the real layout,
// or a variable layout's padded copy)
// rows [row0, row1) only when row1 > 0 (a row-range plan over the whole matrix's
// storage: chunk descriptors keep absolute block and row indices)
static void build_plan_into(const Bsr& a, Plan& P, int K, int mr, int bs, bool var = false, int row0 = 0,
                            int row1 = 0, bool sym = false) {
  P = Plan();
  if (row1 <= 0) row1 = a.nbr;
  if (!stream_supported(mr, mr) || a.nbr == 0 || row1 <= row0) return;
  P.stages = ring_stages();
  const BatchChoice bc = (K > 1 && !var) ? batch_choice(mr, K) : BatchChoice{};
  if (bc.u) {
    // bsr_batch_kernel: phase-A items (block, row, RHS group); the producer warp
    // stages one x segment per lane, so a chunk holds at most 32 blocks
    P.u = bc.u;
    P.xl = bc.xl;
    P.cb_max = std::min(32, bc.cb > 0 ? bc.cb : std::max(1, kern::kConsumers / (mr * P.u)));
  } else {
    P.cb_max = chunk_blocks(mr, bs, K, sym);
  }
  const auto& rp = a.h_row_ptr;
  // chunk list per CTA range
  std::vector<int4> chunks;
  std::vector<int> cta;
  int rmax = 1;
  // first pass with a provisional rmax to size smem and query occupancy
  // bsr_stream_kernel's SKEW layout (m = 20, K = 1, uniform): block pitch bs + 2 in shared memory
  const int spitch = (K == 1 && mr == 20 && !var) ? bs + 2 : ((BMG_PAD21 && K == 1 && mr == 21 && !var) ? bs + 4 : bs);
  const size_t smem0 = P.u ? kern::BatchSmem(bs, P.cb_max, mr, mr, K, P.stages).total
                           : kern::SmemLayout(spitch, P.cb_max, P.cb_max + 2, mr, P.stages, K, sym).total;
  const int occ = P.u ? batch_occupancy_for(mr, smem0, K, P.u)
                      : (sym ? sym_occupancy_for(mr, smem0) : occupancy_for(mr, mr, smem0, K));
  const int64_t gmax = (int64_t)a.ctx->sms * occ;
  const int64_t nnzb_range = a.h_row_ptr[row1] - a.h_row_ptr[row0];
  const int64_t per = std::max<int64_t>(1, (nnzb_range + gmax - 1) / gmax);
  int row = row0;
  while (row < row1) {
    const int rlo = row;
    const int64_t b0 = rp[rlo];
    while (row < row1 && rp[row + 1] - b0 < per) ++row;
    if (row < row1) ++row;  // include the row that reaches the target
    // rows that are empty right after the cut stay with this CTA
    while (row < row1 && rp[row + 1] == rp[row]) ++row;
    const int rhi = row;
    const int64_t B0 = rp[rlo], B1 = rp[rhi];
    cta.push_back((int)chunks.size());
    int r = rlo;
    int64_t clo = B0;
    do {
      const int64_t chi = std::min(B1, clo + P.cb_max);
      const int row_lo = r;
      while (r < rhi && rp[r + 1] <= chi) ++r;
      const bool cout = (r < rhi && rp[r] < chi);
      const int row_hi = cout ? r + 1 : r;
      const bool cin = rp[row_lo] < clo;
      const int nrows = row_hi - row_lo;
      if (nrows >= (int)kern::kRowMask) fail(BMG_EINVAL, "plan: too many rows in a chunk");
      unsigned w = (unsigned)nrows | (cin ? kern::kCarryIn : 0u) | (cout ? kern::kCarryOut : 0u);
      chunks.push_back(make_int4((int)clo, (int)(chi - clo), row_lo, (int)w));
      rmax = std::max(rmax, nrows);
      clo = chi;
    } while (clo < B1);
    if (r != rhi) fail(BMG_ERUNTIME, "plan: row bookkeeping mismatch");
  }
  cta.push_back((int)chunks.size());
  P.rmax = rmax;
  P.nctas = (int)cta.size() - 1;
  P.nchunks = (int)chunks.size();
  P.smem = P.u ? kern::BatchSmem(bs, P.cb_max, mr, mr, K, P.stages).total
               : kern::SmemLayout(spitch, P.cb_max, P.rmax, mr, P.stages, K, sym).total;
  if (P.smem > 227 * 1024) fail(BMG_EINVAL, "plan: chunk does not fit in shared memory");
  if (P.u)  // sets the shared-memory attributes
    batch_occupancy_for(mr, P.smem, K, P.u);
  else if (sym)
    sym_occupancy_for(mr, P.smem);
  else
    occupancy_for(mr, mr, P.smem, K);
  P.chunks.alloc(chunks.size());
  P.cta_chunk.alloc(cta.size());
  BMG_CUDA(cudaMemcpy(P.chunks.p, chunks.data(), chunks.size() * sizeof(int4), cudaMemcpyHostToDevice));
  BMG_CUDA(cudaMemcpy(P.cta_chunk.p, cta.data(), cta.size() * sizeof(int), cudaMemcpyHostToDevice));
}

void build_plan(Bsr& a) {
  if (a.uniform && a.mr == a.mc) build_plan_into(a, a.plan, 1, a.mr, a.bs);
}

bool var_streamed(const Bsr& a) {
  static const bool off = [] {
    const char* e = std::getenv("BMG_VAR_STREAM");
    return e && e[0] == '0';
  }();
  return !off && !a.uniform && a.nnzb > 0 && stream_supported(a.mmax, a.mmax);
}

namespace kern {
// block b of a variable layout -> its mmax x mmax zero-padded slot (warp per block row)
__global__ void pad_blocks_kernel(const double* __restrict__ vals, const int64_t* __restrict__ voff,
                                  const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                  const int* __restrict__ rsz, const int* __restrict__ csz, int nbr, int M, int pbs,
                                  double* __restrict__ out) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= nbr) return;
  const int mi = rsz[i];
  for (int64_t b = row_ptr[i]; b < row_ptr[i + 1]; ++b) {
    const int mj = csz[col[b]];
    const double* src = vals + voff[b];
    double* dst = out + b * pbs;
    for (int e = lane; e < pbs; e += 32) {
      const int r = e / M, c = e - (e / M) * M;
      dst[e] = (r < mi && c < mj) ? src[r * mj + c] : 0.0;
    }
  }
}
}  // namespace kern

const Plan& plan_for(const Bsr& a, int nrhs) {
  const int idx = nrhs <= 1 ? 0 : nrhs == 2 ? 1 : nrhs == 4 ? 2 : 3;
  if (var_streamed(a)) {
    if (!a.pvals.p) {
      const int M = a.mmax;
      a.pbs = (M * M + 1) & ~1;
      a.pvals.alloc((size_t)a.nnzb * a.pbs);
      kern::pad_blocks_kernel<<<(unsigned)(((int64_t)a.nbr * 32 + 255) / 256), 256, 0, a.ctx->stream>>>(
          a.vals.p, a.voff.p, a.row_ptr.p, a.col.p, a.d_rsz.p, a.d_csz.p, a.nbr, M, a.pbs, a.pvals.p);
      a.ctx->count();
      BMG_CUDA(cudaGetLastError());
      BMG_CUDA(cudaStreamSynchronize(a.ctx->stream));
    }
    if (!a.pplan[idx]) {
      auto p = std::make_unique<Plan>();
      build_plan_into(a, *p, std::max(nrhs, 1), a.mmax, a.pbs, true);
      a.pplan[idx] = std::move(p);
    }
    return *a.pplan[idx];
  }
  if (nrhs <= 1) return a.plan;
  if (!a.kplan[idx]) {
    auto p = std::make_unique<Plan>();
    build_plan_into(a, *p, nrhs, a.mr, a.bs);
    a.kplan[idx] = std::move(p);
  }
  return *a.kplan[idx];
}

static void finish_layouts(Bsr& a, int nbr, const int* rsz, int nbc, const int* csz) {
  a.nbr = nbr;
  a.nbc = nbc;
  a.rsz.assign(rsz, rsz + nbr);
  a.csz.assign(csz, csz + nbc);
  a.roff.resize(nbr);
  a.coff.resize(nbc);
  int d = 0;
  for (int i = 0; i < nbr; ++i) {
    if (rsz[i] < 1) fail(BMG_EINVAL, "BlockLayout: block sizes must be >= 1");
    a.roff[i] = d;
    d += rsz[i];
  }
  a.dim_r = d;
  d = 0;
  for (int j = 0; j < nbc; ++j) {
    if (csz[j] < 1) fail(BMG_EINVAL, "BlockLayout: block sizes must be >= 1");
    a.coff[j] = d;
    d += csz[j];
  }
  a.dim_c = d;
  a.uniform = nbr > 0 && nbc > 0;
  for (int i = 1; i < nbr && a.uniform; ++i) a.uniform = rsz[i] == rsz[0];
  for (int j = 1; j < nbc && a.uniform; ++j) a.uniform = csz[j] == csz[0];
  a.mmax = 1;
  for (int i = 0; i < nbr; ++i) a.mmax = std::max(a.mmax, rsz[i]);
  for (int j = 0; j < nbc; ++j) a.mmax = std::max(a.mmax, csz[j]);
  a.mr = a.uniform ? rsz[0] : 0;
  a.mc = a.uniform ? csz[0] : 0;
  a.bs = a.uniform ? ((a.mr * a.mc + 1) & ~1) : 0;
}

static void upload_structure(Bsr& a) {
  a.nnzb = a.h_row_ptr.empty() ? 0 : a.h_row_ptr.back();
  if (a.nnzb >= ((int64_t)1 << 31)) fail(BMG_EINVAL, "bsr: more than 2^31 blocks");
  a.row_ptr.alloc(a.nbr + 1);
  BMG_CUDA(cudaMemcpy(a.row_ptr.p, a.h_row_ptr.data(), (a.nbr + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  a.col.alloc(a.nnzb + 8);
  BMG_CUDA(cudaMemset(a.col.p, 0, (a.nnzb + 8) * sizeof(int32_t)));
  if (a.nnzb)
    BMG_CUDA(cudaMemcpy(a.col.p, a.h_col.data(), a.nnzb * sizeof(int32_t), cudaMemcpyHostToDevice));
  // value offsets
  a.h_voff.resize(a.nnzb + 1);
  int64_t v = 0;
  for (int i = 0; i < a.nbr; ++i)
    for (int64_t p = a.h_row_ptr[i]; p < a.h_row_ptr[i + 1]; ++p) {
      a.h_voff[p] = v;
      v += a.uniform ? a.bs : (int64_t)a.rsz[i] * a.csz[a.h_col[p]];
    }
  a.h_voff[a.nnzb] = v;
  const bool streamed = a.uniform && stream_supported(a.mr, a.mc);
  if (!streamed) {
    a.voff.alloc(a.nnzb + 1);
    BMG_CUDA(cudaMemcpy(a.voff.p, a.h_voff.data(), (a.nnzb + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
    a.d_roff.alloc(a.nbr);
    a.d_rsz.alloc(a.nbr);
    a.d_coff.alloc(a.nbc);
    a.d_csz.alloc(a.nbc);
    BMG_CUDA(cudaMemcpy(a.d_roff.p, a.roff.data(), a.nbr * sizeof(int), cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(a.d_rsz.p, a.rsz.data(), a.nbr * sizeof(int), cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(a.d_coff.p, a.coff.data(), a.nbc * sizeof(int), cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(a.d_csz.p, a.csz.data(), a.nbc * sizeof(int), cudaMemcpyHostToDevice));
  }
  a.vals.alloc(std::max<int64_t>(v, 2));
  build_plan(a);
}

static void validate_structure(int nbr, int nbc, const int64_t* row_ptr, const int32_t* col) {
  if (nbr < 0 || nbc < 0) fail(BMG_EINVAL, "bsr: negative dimensions");
  if (row_ptr[0] != 0) fail(BMG_EINVAL, "bsr: row_ptr[0] must be 0");
  for (int i = 0; i < nbr; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) fail(BMG_EINVAL, "bsr: row_ptr must be non-decreasing");
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      if (col[p] < 0 || col[p] >= nbc) fail(BMG_ERANGE, "BlockSparseMatrix: block index out of range");
      if (p > row_ptr[i] && col[p] <= col[p - 1])
        fail(BMG_EINVAL, "bsr: column indices must be strictly ascending within a row");
    }
  }
}

BlkView blk_view(const Bsr& a) {
  BlkView v;
  v.bs = a.bs;
  v.mr = a.mr;
  v.mc = a.mc;
  if (!a.uniform) {
    v.voff = a.voff.p;
    v.rsz = a.d_rsz.p;
    v.csz = a.d_csz.p;
    v.roff = a.d_roff.p;
    v.coff = a.d_coff.p;
  }
  return v;
}

int max_block(const Bsr& a) { return a.mmax; }

std::unique_ptr<Bsr> make_bsr_structure(Ctx* ctx, int nbr, const int* rsz, int nbc, const int* csz,
                                        std::vector<int64_t> row_ptr, std::vector<int32_t> col,
                                        bool sym) {
  auto a = std::make_unique<Bsr>();
  a->ctx = ctx;
  finish_layouts(*a, nbr, rsz, nbc, csz);
  if (sym && !(a->rsz == a->csz)) fail(BMG_EINVAL, "BlockSparseMatrix: symmetric matrix must be square");
  a->sym = sym;
  a->h_row_ptr = std::move(row_ptr);
  a->h_col = std::move(col);
  upload_structure(*a);
  return a;
}

// Host -> device upload of nblk blocks (src stride -> padded dst stride, padding
// zero).  Large uploads go through two pinned 64 MB buffers: the next chunk is
// copied (OpenMP) while the previous one is in flight, several times faster than
// a pageable cudaMemcpy of tens of GB.
static void upload_blocks(Ctx* ctx, double* dst, const double* src, int64_t nblk, int src_stride,
                          int dst_stride) {
  const size_t total = (size_t)nblk * dst_stride * sizeof(double);
  constexpr size_t kStage = (size_t)64 << 20;
  if (total < 2 * kStage) {
    if (src_stride == dst_stride) {
      BMG_CUDA(cudaMemcpy(dst, src, total, cudaMemcpyHostToDevice));
    } else {
      BMG_CUDA(cudaMemset(dst, 0, total));
      BMG_CUDA(cudaMemcpy2D(dst, (size_t)dst_stride * 8, src, (size_t)src_stride * 8, (size_t)src_stride * 8, nblk,
                            cudaMemcpyHostToDevice));
    }
    return;
  }
  const int64_t per = std::max<int64_t>(1, (int64_t)(kStage / ((size_t)dst_stride * 8)));
  double* pin[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  auto cleanup = [&] {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) cudaEventDestroy(ev[i]);
      if (pin[i]) cudaFreeHost(pin[i]);
    }
  };
  try {
    for (int i = 0; i < 2; ++i) {
      BMG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&pin[i]), (size_t)per * dst_stride * 8, cudaHostAllocDefault));
      BMG_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    for (int64_t c = 0, i = 0; c < nblk; c += per, ++i) {
      double* buf = pin[i & 1];
      if (i >= 2) BMG_CUDA(cudaEventSynchronize(ev[i & 1]));
      const int64_t n = std::min(per, nblk - c);
      const double* sp = src + (size_t)c * src_stride;
      if (src_stride == dst_stride) {
        const int64_t nd = n * dst_stride, step = 1 << 20;
#pragma omp parallel for schedule(static)
        for (int64_t o = 0; o < nd; o += step)
          std::memcpy(buf + o, sp + o, (size_t)std::min(step, nd - o) * sizeof(double));
      } else {
#pragma omp parallel for schedule(static)
        for (int64_t b = 0; b < n; ++b) {
          std::memcpy(buf + (size_t)b * dst_stride, sp + (size_t)b * src_stride, (size_t)src_stride * 8);
          for (int e = src_stride; e < dst_stride; ++e) buf[(size_t)b * dst_stride + e] = 0.0;
        }
      }
      BMG_CUDA(cudaMemcpyAsync(dst + (size_t)c * dst_stride, buf, (size_t)n * dst_stride * 8, cudaMemcpyHostToDevice,
                               ctx->stream));
      BMG_CUDA(cudaEventRecord(ev[i & 1], ctx->stream));
    }
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  } catch (...) {
    cudaStreamSynchronize(ctx->stream);
    cleanup();
    throw;
  }
  cleanup();
}

std::unique_ptr<Bsr> make_bsr(Ctx* ctx, int nbr, const int* rsz, int nbc, const int* csz,
                              const int64_t* row_ptr, const int32_t* col, const double* vals,
                              bool sym, bool vals_on_device) {
  validate_structure(nbr, nbc, row_ptr, col);
  const int64_t nnzb = row_ptr[nbr];
  auto a = make_bsr_structure(ctx, nbr, rsz, nbc, csz,
                              std::vector<int64_t>(row_ptr, row_ptr + nbr + 1),
                              std::vector<int32_t>(col, col + nnzb), sym);
  if (nnzb == 0) return a;
  const auto kind = vals_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  if (!vals_on_device && a->uniform) {
    upload_blocks(ctx, a->vals.p, vals, nnzb, a->mr * a->mc, a->bs);
    return a;
  }
  if (!a->uniform || a->bs == a->mr * a->mc) {
    BMG_CUDA(cudaMemcpy(a->vals.p, vals, a->h_voff[nnzb] * sizeof(double), kind));
  } else {
    // pad each block to the even stride (16-byte aligned blocks)
    const size_t src = (size_t)a->mr * a->mc * sizeof(double), dst = (size_t)a->bs * sizeof(double);
    BMG_CUDA(cudaMemset(a->vals.p, 0, a->vals.bytes()));
    BMG_CUDA(cudaMemcpy2D(a->vals.p, dst, vals, src, src, nnzb, kind));
  }
  return a;
}

std::unique_ptr<Bsr> bsr_transpose(const Bsr& a) {
  // structure on the host (integer counting sort: transposed rows ascending),
  // values transposed on the device through the block permutation
  std::vector<int64_t> trp(a.nbc + 1, 0);
  for (int64_t p = 0; p < a.nnzb; ++p) trp[a.h_col[p] + 1]++;
  for (int j = 0; j < a.nbc; ++j) trp[j + 1] += trp[j];
  std::vector<int32_t> tcol(a.nnzb);
  std::vector<int64_t> perm(a.nnzb);
  std::vector<int64_t> fillp(trp.begin(), trp.end() - 1);
  for (int i = 0; i < a.nbr; ++i)
    for (int64_t p = a.h_row_ptr[i]; p < a.h_row_ptr[i + 1]; ++p) {
      const int64_t q = fillp[a.h_col[p]]++;
      tcol[q] = i;
      perm[q] = p;
    }
  auto t = make_bsr_structure(a.ctx, a.nbc, a.csz.data(), a.nbr, a.rsz.data(), std::move(trp),
                              std::move(tcol), a.sym);
  if (a.nnzb == 0) return t;
  DBuf<int64_t> dperm(a.nnzb);
  BMG_CUDA(cudaMemcpy(dperm.p, perm.data(), a.nnzb * sizeof(int64_t), cudaMemcpyHostToDevice));
  Ctx* ctx = a.ctx;
  if (a.uniform) {
    kern::transpose_uniform_kernel<<<grid_for(a.nnzb * a.mr * a.mc), 256, 0, ctx->stream>>>(
        a.vals.p, t->vals.p, dperm.p, a.nnzb, a.mr, a.mc, a.bs, t->bs);
  } else {
    std::vector<int> trow_of(a.nnzb);
    for (int j = 0; j < t->nbr; ++j)
      for (int64_t q = t->h_row_ptr[j]; q < t->h_row_ptr[j + 1]; ++q) trow_of[q] = j;
    DBuf<int64_t> vsrc(a.nnzb + 1), vdst(a.nnzb + 1);
    DBuf<int> drow(a.nnzb), dcol(a.nnzb), dr(t->nbr), dc(t->nbc);
    BMG_CUDA(cudaMemcpy(vsrc.p, a.h_voff.data(), (a.nnzb + 1) * 8, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(vdst.p, t->h_voff.data(), (a.nnzb + 1) * 8, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(drow.p, trow_of.data(), a.nnzb * 4, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(dcol.p, t->h_col.data(), a.nnzb * 4, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(dr.p, t->rsz.data(), t->nbr * 4, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(dc.p, t->csz.data(), t->nbc * 4, cudaMemcpyHostToDevice));
    kern::transpose_var_kernel<<<grid_for(a.nnzb * 32, 256), 256, 0, ctx->stream>>>(
        a.vals.p, t->vals.p, dperm.p, vsrc.p, vdst.p, drow.p, dcol.p, dr.p, dc.p, a.nnzb);
    BMG_CUDA(cudaGetLastError());
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  return t;
}

// ============================================================================ launches
// Evict-first on every streamed matrix (BMG_L2_HINT=0 disables).  Sparing small
// operators (BMG_L2_HINT_MB: hint only above that many MB) was measured: C1 (an
// L2-resident working set) does not move (52 us either way) and the C2 cycle is
// best with every matrix hinted (2.115-2.126 ms; 2.15 ms above 128 MB).
static int l2_hint_for(const Bsr& a) {
  static const int on = [] {
    const char* e = std::getenv("BMG_L2_HINT");
    return (e && e[0] == '0') ? 0 : 1;
  }();
  static const double min_bytes = [] {
    const char* e = std::getenv("BMG_L2_HINT_MB");
    return (e ? std::atof(e) : 0.0) * 1e6;
  }();
  return on && (double)a.nnzb * a.bs * 8.0 >= min_bytes ? 1 : 0;
}

static bool pdl_enabled() {
  static bool on = [] {
    const char* e = std::getenv("BMG_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int MR, int MC, int K, class Epi, bool VAR = false, bool SYM = false>
static void launch_stream_plan(const Bsr& a, const Plan& P, const double* x, Epi epi, const SymArgs* sa = nullptr);
template <int MR, int MC, int K, class Epi, bool VAR = false>
static void launch_stream_t(const Bsr& a, const double* x, Epi epi) {
  launch_stream_plan<MR, MC, K, Epi, VAR>(a, plan_for(a, K), x, epi);
}
template <int MR, int MC, int K, class Epi, bool VAR, bool SYM>
static void launch_stream_plan(const Bsr& a, const Plan& P, const double* x, Epi epi, const SymArgs* sa) {
  kern::StreamArgs s;
  if constexpr (SYM) {
    static const int colmap = [] {
      const char* e = std::getenv("BMG_SYM_COLMAP");
      return e ? std::atoi(e) : 2;  // measured: full tiles block-fastest, the rest block-major
    }();
    s.brow = sa->brow;
    s.colpart = sa->colpart;
    s.sym_lo = sa->sym_lo;
    s.colmap = colmap;
  }
  s.vals = VAR ? a.pvals.p : a.vals.p;
  s.col = a.col.p;
  s.row_ptr = a.row_ptr.p;
  s.chunks = P.chunks.p;
  s.cta_chunk = P.cta_chunk.p;
  s.x = x;
  s.bs = VAR ? a.pbs : a.bs;
  if (VAR) {
    s.coff = a.d_coff.p;
    s.roff = a.d_roff.p;
    s.rsz = a.d_rsz.p;
    s.xlen = a.dim_c;
  }
  s.cb_max = P.cb_max;
  s.rmax = P.rmax;
  s.stages = P.stages;
  s.l2hint = l2_hint_for(a);
  // one attribute per template instantiation (covers the largest plan)
  static const bool attr_set = [] {  // thread-safe one-time init (contexts may live on several threads)
    stream_attrs(kern::bsr_stream_kernel<MR, MC, K, Epi, VAR, SYM>, K);
    return true;
  }();
  (void)attr_set;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.nctas);
  cfg.blockDim = dim3(kern::kThreads);
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = a.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BMG_CUDA(cudaLaunchKernelEx(&cfg, kern::bsr_stream_kernel<MR, MC, K, Epi, VAR, SYM>, s, epi));
  a.ctx->count();
  BMG_LAUNCHED(a.ctx->stream, "bsr_stream_kernel");
}

// A SYM pass: the lower triangle streamed (row sums to sbuf, transposed products
// to colpart), then the merge adds the upper contributions and runs the epilogue.
template <int MR, class Epi>
static void launch_merge(Ctx* ctx, int64_t nrows, const int64_t* up_ptr, const int32_t* up_slot, const double* colpart,
                         const double* S, Epi epi, double* tbuf, int64_t tsplit_rows) {
  const int64_t n = nrows * MR;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)ctx->sms * 16)));
  cfg.blockDim = dim3(256);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BMG_CUDA(cudaLaunchKernelEx(&cfg, kern::sym_merge_kernel<MR, Epi>, up_ptr, up_slot, colpart, S, n, epi, tbuf,
                              tsplit_rows * MR));
  ctx->count();
  BMG_LAUNCHED(ctx->stream, "sym_merge_kernel");
}

template <int MR, class Epi>
static void launch_sym(const Bsr& a, const double* x, Epi epi) {
  const SymHalf& H = *a.half;
  const Bsr& low = *H.low;
  const SymArgs sa{H.brow.p, H.colpart.p, 0};
  launch_stream_plan<MR, MR, 1, kern::EpiStore, false, true>(low, low.plan, x, kern::EpiStore{H.sbuf.p}, &sa);
  launch_merge<MR>(a.ctx, a.nbr, H.up_ptr.p, H.up_slot.p, H.colpart.p, H.sbuf.p, epi, nullptr, a.nbr);
}
template <class Epi>
static bool try_launch_sym(const Bsr& a, const double* x, Epi epi, int nrhs) {
  if (nrhs != 1 || !a.half) return false;
  switch (a.mr) {
    case 3: launch_sym<3>(a, x, epi); return true;
    case 6: launch_sym<6>(a, x, epi); return true;
    case 10: launch_sym<10>(a, x, epi); return true;
    case 15: launch_sym<15>(a, x, epi); return true;
    case 20: launch_sym<20>(a, x, epi); return true;
    case 21: launch_sym<21>(a, x, epi); return true;
  }
  return false;
}

template <int MR, int K, int U, class Epi, bool XL>
static void launch_batch_x(const Bsr& a, const Plan& P, const double* x, Epi epi) {
  if (reinterpret_cast<uintptr_t>(x) & 15)
    fail(BMG_EINVAL, "batched pass: x must be 16-byte aligned");
  kern::StreamArgs s;
  s.vals = a.vals.p;
  s.col = a.col.p;
  s.row_ptr = a.row_ptr.p;
  s.chunks = P.chunks.p;
  s.cta_chunk = P.cta_chunk.p;
  s.x = x;
  s.bs = a.bs;
  s.cb_max = P.cb_max;
  s.rmax = P.rmax;
  s.stages = P.stages;
  s.l2hint = l2_hint_for(a);
  static const bool attr_set = [] {
    stream_attrs(kern::bsr_batch_kernel<MR, MR, K, U, Epi, XL>, K);
    return true;
  }();
  (void)attr_set;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P.nctas);
  cfg.blockDim = dim3(kern::kThreads);
  cfg.dynamicSmemBytes = P.smem;
  cfg.stream = a.ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  BMG_CUDA(cudaLaunchKernelEx(&cfg, kern::bsr_batch_kernel<MR, MR, K, U, Epi, XL>, s, epi));
  a.ctx->count();
  BMG_LAUNCHED(a.ctx->stream, "bsr_batch_kernel");
}

template <int MR, int K, int U, class Epi>
static void launch_batch_t(const Bsr& a, const Plan& P, const double* x, Epi epi) {
  if constexpr (K == 2) {  // the only batch size where XL measured faster (batch_choice)
    if (P.xl) return launch_batch_x<MR, K, U, Epi, true>(a, P, x, epi);
  }
  launch_batch_x<MR, K, U, Epi, false>(a, P, x, epi);
}

template <int MR, class Epi>
static void launch_batch(const Bsr& a, const double* x, Epi epi, int nrhs) {
  const Plan& P = plan_for(a, nrhs);
  if (nrhs == 2) return launch_batch_t<MR, 2, 1>(a, P, x, epi);
  if (nrhs == 4) return P.u == 1 ? launch_batch_t<MR, 4, 1>(a, P, x, epi) : launch_batch_t<MR, 4, 2>(a, P, x, epi);
  if (nrhs == 8) {
    return P.u == 1 ? launch_batch_t<MR, 8, 1>(a, P, x, epi) : launch_batch_t<MR, 8, 2>(a, P, x, epi);
  }
  fail(BMG_EINVAL, "right-hand-side batch must be 1, 2, 4 or 8");
}

template <int MR, int MC, class Epi, bool VAR = false>
static void launch_stream_k(const Bsr& a, const double* x, Epi epi, int nrhs) {
  if constexpr (!VAR && MR >= 10) {  // the staged batch kernel serves m >= 10 (batch_choice)
    if (nrhs > 1 && plan_for(a, nrhs).u) return launch_batch<MR>(a, x, epi, nrhs);
  }
  switch (nrhs) {
    case 1: return launch_stream_t<MR, MC, 1, Epi, VAR>(a, x, epi);
    case 2: return launch_stream_t<MR, MC, 2, Epi, VAR>(a, x, epi);
    case 4: return launch_stream_t<MR, MC, 4, Epi, VAR>(a, x, epi);
    case 8: return launch_stream_t<MR, MC, 8, Epi, VAR>(a, x, epi);
  }
  fail(BMG_EINVAL, "right-hand-side batch must be 1, 2, 4 or 8");
}

template <class Epi>
static void launch(const Bsr& a, const double* x, Epi epi, int nrhs) {
  if (a.nbr == 0) return;
  if (a.uniform && stream_supported(a.mr, a.mc)) {
    switch (a.mr) {
      case 3: return launch_stream_k<3, 3>(a, x, epi, nrhs);
      case 6: return launch_stream_k<6, 6>(a, x, epi, nrhs);
      case 10: return launch_stream_k<10, 10>(a, x, epi, nrhs);
      case 15: return launch_stream_k<15, 15>(a, x, epi, nrhs);
      case 20: return launch_stream_k<20, 20>(a, x, epi, nrhs);
      case 21: return launch_stream_k<21, 21>(a, x, epi, nrhs);
    }
  }
  if (var_streamed(a)) {
    switch (a.mmax) {
      case 3: return launch_stream_k<3, 3, Epi, true>(a, x, epi, nrhs);
      case 6: return launch_stream_k<6, 6, Epi, true>(a, x, epi, nrhs);
      case 10: return launch_stream_k<10, 10, Epi, true>(a, x, epi, nrhs);
      case 15: return launch_stream_k<15, 15, Epi, true>(a, x, epi, nrhs);
      case 20: return launch_stream_k<20, 20, Epi, true>(a, x, epi, nrhs);
      case 21: return launch_stream_k<21, 21, Epi, true>(a, x, epi, nrhs);
    }
  }
  if (nrhs < 1 || nrhs > 8) fail(BMG_EINVAL, "right-hand-side batch must be 1..8");
  kern::VarArgs s;
  s.vals = a.vals.p;
  s.col = a.col.p;
  s.row_ptr = a.row_ptr.p;
  s.voff = a.voff.p;
  s.roff = a.d_roff.p;
  s.rsz = a.d_rsz.p;
  s.coff = a.d_coff.p;
  s.csz = a.d_csz.p;
  s.x = x;
  s.nbr = a.nbr;
  s.nrhs = nrhs;
  const int blocks = (int)(((int64_t)a.nbr * 32 + 255) / 256);
  kern::bsr_var_kernel<Epi><<<blocks, 256, 0, a.ctx->stream>>>(s, epi);
  a.ctx->count();
  BMG_LAUNCHED(a.ctx->stream, "bsr_var_kernel");
}

std::unique_ptr<Plan> plan_rows(const Bsr& a, int row0, int row1) {
  if (!a.uniform || !stream_supported(a.mr, a.mc)) return nullptr;
  auto p = std::make_unique<Plan>();
  build_plan_into(a, *p, 1, a.mr, a.bs, false, row0, row1);
  if (p->nctas == 0) return nullptr;
  return p;
}
// row-range plan over the lower triangle of a half-storage A (rows [row0, row1):
// their blocks reach columns <= the row, so the range reads x rows < row1 only)
std::unique_ptr<Plan> plan_rows_sym(const Bsr& low, int row0, int row1) {
  if (!low.uniform || low.mr != low.mc || !stream_supported(low.mr, low.mc)) return nullptr;
  auto p = std::make_unique<Plan>();
  build_plan_into(low, *p, 1, low.mr, low.bs, false, row0, row1, true);
  if (p->nctas == 0) return nullptr;
  return p;
}
void sym_phase1_rows(const Bsr& low, const Plan& P, const SymArgs& sa, const double* x, double* S) {
  const kern::EpiStore epi{S};
  switch (low.mr) {
    case 3: return launch_stream_plan<3, 3, 1, kern::EpiStore, false, true>(low, P, x, epi, &sa);
    case 6: return launch_stream_plan<6, 6, 1, kern::EpiStore, false, true>(low, P, x, epi, &sa);
    case 10: return launch_stream_plan<10, 10, 1, kern::EpiStore, false, true>(low, P, x, epi, &sa);
    case 15: return launch_stream_plan<15, 15, 1, kern::EpiStore, false, true>(low, P, x, epi, &sa);
    case 20: return launch_stream_plan<20, 20, 1, kern::EpiStore, false, true>(low, P, x, epi, &sa);
    case 21: return launch_stream_plan<21, 21, 1, kern::EpiStore, false, true>(low, P, x, epi, &sa);
  }
  fail(BMG_EINVAL, "sym_phase1_rows: streamed block sizes only");
}
void residual_rows(const Bsr& a, const Plan& P, const double* b, const double* x, double* r) {
  const kern::EpiResidual epi{b, r};
  switch (a.mr) {
    case 3: return launch_stream_plan<3, 3, 1>(a, P, x, epi);
    case 6: return launch_stream_plan<6, 6, 1>(a, P, x, epi);
    case 10: return launch_stream_plan<10, 10, 1>(a, P, x, epi);
    case 15: return launch_stream_plan<15, 15, 1>(a, P, x, epi);
    case 20: return launch_stream_plan<20, 20, 1>(a, P, x, epi);
    case 21: return launch_stream_plan<21, 21, 1>(a, P, x, epi);
  }
  fail(BMG_EINVAL, "residual_rows: streamed block sizes only");
}

void spmv(const Bsr& a, const double* x, double* y, int nrhs) {
  if (try_launch_sym(a, x, kern::EpiStore{y}, nrhs)) return;
  launch(a, x, kern::EpiStore{y}, nrhs);
}
void residual(const Bsr& a, const double* b, const double* x, double* r, int nrhs) {
  if (try_launch_sym(a, x, kern::EpiResidual{b, r}, nrhs)) return;
  launch(a, x, kern::EpiResidual{b, r}, nrhs);
}

void build_sym_plan(Bsr& low) {
  if (!low.uniform || low.mr != low.mc || !stream_supported(low.mr, low.mc)) fail(BMG_EINVAL, "sym plan: streamed uniform blocks only");
  build_plan_into(low, low.plan, 1, low.mr, low.bs, false, 0, 0, true);
}

void sym_phase1(const Bsr& low, const SymArgs& sa, const double* x, double* S) {
  if (low.nbr == 0) return;
  const kern::EpiStore epi{S};
  switch (low.mr) {
    case 3: return launch_stream_plan<3, 3, 1, kern::EpiStore, false, true>(low, low.plan, x, epi, &sa);
    case 6: return launch_stream_plan<6, 6, 1, kern::EpiStore, false, true>(low, low.plan, x, epi, &sa);
    case 10: return launch_stream_plan<10, 10, 1, kern::EpiStore, false, true>(low, low.plan, x, epi, &sa);
    case 15: return launch_stream_plan<15, 15, 1, kern::EpiStore, false, true>(low, low.plan, x, epi, &sa);
    case 20: return launch_stream_plan<20, 20, 1, kern::EpiStore, false, true>(low, low.plan, x, epi, &sa);
    case 21: return launch_stream_plan<21, 21, 1, kern::EpiStore, false, true>(low, low.plan, x, epi, &sa);
  }
  fail(BMG_EINVAL, "sym_phase1: streamed block sizes only");
}

void sym_merge(Ctx* ctx, int m, int64_t nrows, const int64_t* up_ptr, const int32_t* up_slot, const double* colpart,
               const double* S, const double* b, double* r, double* tbuf, int64_t tsplit_rows) {
  if (nrows <= 0) return;
  const kern::EpiResidual epi{b, r};
  switch (m) {
    case 3: return launch_merge<3>(ctx, nrows, up_ptr, up_slot, colpart, S, epi, tbuf, tsplit_rows);
    case 6: return launch_merge<6>(ctx, nrows, up_ptr, up_slot, colpart, S, epi, tbuf, tsplit_rows);
    case 10: return launch_merge<10>(ctx, nrows, up_ptr, up_slot, colpart, S, epi, tbuf, tsplit_rows);
    case 15: return launch_merge<15>(ctx, nrows, up_ptr, up_slot, colpart, S, epi, tbuf, tsplit_rows);
    case 20: return launch_merge<20>(ctx, nrows, up_ptr, up_slot, colpart, S, epi, tbuf, tsplit_rows);
    case 21: return launch_merge<21>(ctx, nrows, up_ptr, up_slot, colpart, S, epi, tbuf, tsplit_rows);
  }
  fail(BMG_EINVAL, "sym_merge: streamed block sizes only");
}

void residual_from(const Bsr& tail, const double* t, const double* b, const double* x, double* r) {
  if (tail.nbr == 0) return;
  const kern::EpiResidualFrom epi{t, b, r};
  switch (tail.mr) {
    case 3: return launch_stream_plan<3, 3, 1>(tail, tail.plan, x, epi);
    case 6: return launch_stream_plan<6, 6, 1>(tail, tail.plan, x, epi);
    case 10: return launch_stream_plan<10, 10, 1>(tail, tail.plan, x, epi);
    case 15: return launch_stream_plan<15, 15, 1>(tail, tail.plan, x, epi);
    case 20: return launch_stream_plan<20, 20, 1>(tail, tail.plan, x, epi);
    case 21: return launch_stream_plan<21, 21, 1>(tail, tail.plan, x, epi);
  }
  fail(BMG_EINVAL, "residual_from: streamed block sizes only");
}

// ---- symmetric-half form ----------------------------------------------------------
namespace kern {
// flag = 1 if some stored off-diagonal block differs bitwise from the transpose of
// its mirror block (warp per block)
__global__ void sym_check_kernel(const double* __restrict__ vals, const int64_t* __restrict__ mirror, int64_t nnzb,
                                 int m, int bs, int* __restrict__ flag) {
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= nnzb) return;
  const int64_t q = mirror[p];
  const unsigned long long* A = reinterpret_cast<const unsigned long long*>(vals + p * bs);
  const unsigned long long* B = reinterpret_cast<const unsigned long long*>(vals + q * bs);
  for (int e = lane; e < m * m; e += 32) {
    const int r = e / m, c = e - r * m;
    if (A[r * m + c] != B[c * m + r]) atomicOr(flag, 1);
  }
}
// low block q <- block src[q] (bs doubles each)
__global__ void gather_blocks_kernel(const double* __restrict__ vals, const int64_t* __restrict__ src, int64_t nq,
                                     int bs, double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nq * bs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / bs;
    out[e] = vals[src[q] * bs + (e - q * bs)];
  }
}
}  // namespace kern

int64_t SymHalf::bytes() const {
  return (int64_t)(low ? low->device_bytes() : 0) + (int64_t)(brow.bytes() + up_ptr.bytes() + up_slot.bytes() +
                                                              colpart.bytes() + sbuf.bytes());
}

int64_t sym_pass_bytes(const Bsr& a) {
  if (!a.half) return a.pass_bytes();
  const Bsr& low = *a.half->low;
  const int64_t nup = a.nnzb - low.nnzb;
  const int64_t n = a.dim_r, m = a.mr;
  // phase 1: lower blocks + column and row indices, transposed products written,
  // row sums written; merge: row sums, partials and slots read
  return low.nnzb * (8 * (int64_t)a.mr * a.mc + 8) + nup * m * 8 + 8 * n + 8 * n + nup * (m * 8 + 4) +
         8 * ((int64_t)a.nbr + 1);
}

// BMG_SYM_HALF: 0 off, 1 always, unset: measured choice per matrix
static int sym_mode() {
  static const int v = [] {
    const char* e = std::getenv("BMG_SYM_HALF");
    return !e ? -1 : (e[0] == '0' ? 0 : 1);
  }();
  return v;
}

// Both forms give bitwise the same result; which one streams faster depends on
// the block size and row length (m = 20: the half form saves ~1/3 of the pass
// time; m = 10: its column dots cost what the halved bytes save).  Each is
// timed on this matrix (3 passes after a warm one) and the faster one kept.
// `next` (the level's G, whose pass follows every residual in the cycle) is
// timed behind each form, so the choice includes how the pass overlaps its
// successor under programmatic dependent launch.
static bool sym_faster(const Bsr& a, const Bsr* next) {
  Ctx* ctx = a.ctx;
  const int64_t n = std::max<int64_t>(a.dim_r, 1);
  DBuf<double> x(n), b(n), r(n), w(n);
  BMG_CUDA(cudaMemsetAsync(x.p, 0, x.bytes(), ctx->stream));
  BMG_CUDA(cudaMemsetAsync(b.p, 0, b.bytes(), ctx->stream));
  cudaEvent_t e[3];
  for (auto& v : e) BMG_CUDA(cudaEventCreate(&v));
  auto tail = [&] {
    if (next && next->dim_c == a.dim_r && next->dim_r <= n) launch(*next, r.p, kern::EpiStore{w.p}, 1);
  };
  auto sym_pass = [&] {
    try_launch_sym(a, x.p, kern::EpiResidual{b.p, r.p}, 1);
    tail();
  };
  auto full_pass = [&] {
    launch(a, x.p, kern::EpiResidual{b.p, r.p}, 1);
    tail();
  };
  float t_sym = 0.f, t_full = 0.f;
  for (int rep = 0; rep < 2; ++rep) {  // warm both, then time both
    BMG_CUDA(cudaEventRecord(e[0], ctx->stream));
    for (int k = 0; k < 3; ++k) sym_pass();
    BMG_CUDA(cudaEventRecord(e[1], ctx->stream));
    for (int k = 0; k < 3; ++k) full_pass();
    BMG_CUDA(cudaEventRecord(e[2], ctx->stream));
    BMG_CUDA(cudaEventSynchronize(e[2]));
    BMG_CUDA(cudaEventElapsedTime(&t_sym, e[0], e[1]));
    BMG_CUDA(cudaEventElapsedTime(&t_full, e[1], e[2]));
  }
  for (auto& v : e) cudaEventDestroy(v);
  a.sym_ms = t_sym / 3.0;
  a.full_ms = t_full / 3.0;
  // small passes (C2's levels, < 0.5 ms) measured slower inside whole cycles with
  // the half form even where the pair above was faster (one more launch per pass,
  // less overlap of consecutive passes): full storage there
  return a.full_ms >= 0.5 && t_sym < 0.95f * t_full;
}

bool ensure_sym_half(const Bsr& a, const Bsr* next) {
  const bool off = sym_mode() == 0;
  if (a.half_state != 0) return a.half_state > 0;
  a.half_state = -1;
  if (off || !a.sym || !a.uniform || a.mr != a.mc || a.nbr != a.nbc || a.nnzb == 0 || !stream_supported(a.mr, a.mc))
    return false;
  Ctx* ctx = a.ctx;
  const int m = a.mr;
  const auto& rp = a.h_row_ptr;
  const auto& cl = a.h_col;
  // structural mirror of every block; structurally unsymmetric -> no half form
  std::vector<int64_t> mirror(a.nnzb);
  for (int i = 0; i < a.nbr; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      const int j = cl[p];
      auto b = cl.begin() + rp[j], e = cl.begin() + rp[j + 1];
      auto it = std::lower_bound(b, e, i);
      if (it == e || *it != i) return false;
      mirror[p] = rp[j] + (it - b);
    }
  {
    DBuf<int64_t> dm(a.nnzb);
    DBuf<int> flag(1);
    BMG_CUDA(cudaMemcpyAsync(dm.p, mirror.data(), a.nnzb * 8, cudaMemcpyHostToDevice, ctx->stream));
    BMG_CUDA(cudaMemsetAsync(flag.p, 0, sizeof(int), ctx->stream));
    kern::sym_check_kernel<<<(unsigned)((a.nnzb * 32 + 255) / 256), 256, 0, ctx->stream>>>(a.vals.p, dm.p, a.nnzb, m,
                                                                                          a.bs, flag.p);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
    int h = 0;
    BMG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h) return false;  // not exactly symmetric: keep full storage
  }
  // lower triangle: structure, block ids, rows
  std::vector<int64_t> lrp(a.nbr + 1, 0), lid(a.nnzb, -1), src;
  std::vector<int32_t> lcol, lrow;
  src.reserve(a.nnzb / 2 + a.nbr);
  for (int i = 0; i < a.nbr; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1] && cl[p] <= i; ++p) {
      lid[p] = (int64_t)src.size();
      src.push_back(p);
      lcol.push_back(cl[p]);
      lrow.push_back(i);
    }
    lrp[i + 1] = (int64_t)src.size();
  }
  const int64_t nlow = (int64_t)src.size();
  if (nlow >= ((int64_t)1 << 31)) return false;
  // upper blocks of row i (ascending j > i): the lower block (j, i) holding them
  std::vector<int64_t> uptr(a.nbr + 1, 0);
  std::vector<int32_t> uslot;
  uslot.reserve(a.nnzb - nlow);
  for (int i = 0; i < a.nbr; ++i) {
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (cl[p] > i) uslot.push_back((int32_t)lid[mirror[p]]);
    uptr[i + 1] = (int64_t)uslot.size();
  }
  auto H = std::make_unique<SymHalf>();
  H->low = make_bsr_structure(ctx, a.nbr, a.rsz.data(), a.nbc, a.csz.data(), std::move(lrp), std::move(lcol), false);
  // the SYM kernel's plan (its shared memory carries the row indices too)
  build_plan_into(*H->low, H->low->plan, 1, m, a.bs, false, 0, 0, true);
  {
    DBuf<int64_t> dsrc(nlow);
    BMG_CUDA(cudaMemcpyAsync(dsrc.p, src.data(), nlow * 8, cudaMemcpyHostToDevice, ctx->stream));
    kern::gather_blocks_kernel<<<grid_for(nlow * a.bs), 256, 0, ctx->stream>>>(a.vals.p, dsrc.p, nlow, a.bs,
                                                                              H->low->vals.p);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  H->brow.alloc(nlow + 8);
  BMG_CUDA(cudaMemset(H->brow.p, 0, (nlow + 8) * 4));
  BMG_CUDA(cudaMemcpy(H->brow.p, lrow.data(), nlow * 4, cudaMemcpyHostToDevice));
  H->up_ptr.alloc(a.nbr + 1);
  BMG_CUDA(cudaMemcpy(H->up_ptr.p, uptr.data(), (a.nbr + 1) * 8, cudaMemcpyHostToDevice));
  H->up_slot.alloc(std::max<size_t>(uslot.size(), 1));
  if (!uslot.empty()) BMG_CUDA(cudaMemcpy(H->up_slot.p, uslot.data(), uslot.size() * 4, cudaMemcpyHostToDevice));
  H->colpart.alloc((size_t)nlow * m);
  H->sbuf.alloc(std::max<int64_t>(a.dim_r, 1));
  a.half = std::move(H);
  a.half_state = 1;
  if (sym_mode() < 0 && !sym_faster(a, next)) {
    a.half.reset();
    a.half_state = -1;
    return false;
  }
  return true;
}
void prolong_add(const Bsr& a, const double* e, double* x, int nrhs) { launch(a, e, kern::EpiAdd{x}, nrhs); }
void gt_cheb(const Bsr& gt, const double* w, double* p, double* x, double mu2, double dmu,
             bool first, bool xzero, int nrhs) {
  launch(gt, w, kern::EpiCheb{p, x, mu2, dmu, first ? 1 : 0, xzero ? 1 : 0}, nrhs);
}

}  // namespace bmg

// ============================================================================ C ABI
using namespace bmg;

extern "C" {

const char* bmg_last_error(void) { return g_last_error.c_str(); }
int bmg_last_pivot(void) { return g_last_pivot; }
const char* bmg_version(void) { return "blockmg-b200 0.1.0 (reference blockmg 0.1.0)"; }

int bmg_ctx_create(int device, bmg_ctx** out) {
  return guard([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) fail(BMG_ECUDA, "no CUDA device available");
    if (device < 0 || device >= n) fail(BMG_ERANGE, "bmg_ctx_create: device out of range");
    auto c = std::make_unique<Ctx>();
    c->device = device;
    BMG_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    BMG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) fail(BMG_ECUDA, "libbmgcuda requires an sm_100 (Blackwell) device");
    c->sms = prop.multiProcessorCount;
    // a blocking stream: setup-time cudaMemcpy/cudaMemset on the legacy stream are
    // ordered with the kernels launched here
    BMG_CUDA(cudaStreamCreate(&c->own));
    c->stream = c->own;
    *out = reinterpret_cast<bmg_ctx*>(c.release());
  });
}
int bmg_ctx_destroy(bmg_ctx* ctx) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    if (c) BMG_CUDA(cudaStreamSynchronize(c->stream));
    ctx_release(c);  // freed now, or when its last device object is destroyed
  });
}
int bmg_ctx_set_stream(bmg_ctx* ctx, void* s) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
  });
}
int bmg_ctx_sync(bmg_ctx* ctx) {
  return guard([&] { BMG_CUDA(cudaStreamSynchronize(reinterpret_cast<Ctx*>(ctx)->stream)); });
}
int64_t bmg_ctx_launch_count(const bmg_ctx* ctx) { return reinterpret_cast<const Ctx*>(ctx)->launches; }

int bmg_bsr_create(bmg_ctx* ctx, int nbr, const int32_t* row_sizes, int nbc, const int32_t* col_sizes,
                   const int64_t* row_ptr, const int32_t* col_idx, const double* vals, int flags,
                   bmg_bsr** out) {
  return guard([&] {
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->activate();
    auto a = make_bsr(c, nbr, row_sizes, nbc, col_sizes, row_ptr, col_idx, vals, (flags & BMG_SYMMETRIC) != 0);
    *out = reinterpret_cast<bmg_bsr*>(a.release());
  });
}
// destroying an object first drains its context stream: queued work may still
// reference it (device objects follow CUDA's asynchronous semantics)
int bmg_bsr_destroy(bmg_bsr* a) {
  return guard([&] {
    Bsr* m = reinterpret_cast<Bsr*>(a);
    if (m) BMG_CUDA(cudaStreamSynchronize(m->ctx->stream));
    bsr_release(m);  // freed now, or when the last hierarchy holding it goes
  });
}
int bmg_bsr_info(const bmg_bsr* ah, int* nbr, int* nbc, int64_t* nnzb, int* dim_r, int* dim_c,
                 int64_t* device_bytes, int64_t* pass_bytes) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    if (nbr) *nbr = a->nbr;
    if (nbc) *nbc = a->nbc;
    if (nnzb) *nnzb = a->nnzb;
    if (dim_r) *dim_r = a->dim_r;
    if (dim_c) *dim_c = a->dim_c;
    if (device_bytes) *device_bytes = a->device_bytes();
    if (pass_bytes) *pass_bytes = a->pass_bytes();
  });
}
int bmg_bsr_sym_info(const bmg_bsr* ah, int* half, int64_t* pass_bytes, double* half_ms, double* full_ms) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    if (half) *half = a->half ? 1 : 0;
    if (pass_bytes) *pass_bytes = a->half ? sym_pass_bytes(*a) : a->pass_bytes();
    if (half_ms) *half_ms = a->sym_ms;
    if (full_ms) *full_ms = a->full_ms;
  });
}
int bmg_bsr_download(const bmg_bsr* ah, int64_t* row_ptr, int32_t* col_idx, double* vals) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    a->ctx->activate();
    BMG_CUDA(cudaStreamSynchronize(a->ctx->stream));
    if (row_ptr) std::memcpy(row_ptr, a->h_row_ptr.data(), (a->nbr + 1) * sizeof(int64_t));
    if (col_idx && a->nnzb) std::memcpy(col_idx, a->h_col.data(), a->nnzb * sizeof(int32_t));
    if (vals && a->nnzb) {
      if (!a->uniform || a->bs == a->mr * a->mc) {
        BMG_CUDA(cudaMemcpy(vals, a->vals.p, a->h_voff[a->nnzb] * sizeof(double), cudaMemcpyDeviceToHost));
      } else {
        const size_t w = (size_t)a->mr * a->mc * sizeof(double);
        BMG_CUDA(cudaMemcpy2D(vals, w, a->vals.p, (size_t)a->bs * sizeof(double), w, a->nnzb,
                              cudaMemcpyDeviceToHost));
      }
    }
  });
}
int bmg_bsr_transpose(const bmg_bsr* ah, bmg_bsr** out) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    a->ctx->activate();
    *out = reinterpret_cast<bmg_bsr*>(bsr_transpose(*a).release());
  });
}

int bmg_vec_create(bmg_ctx* ctx, int64_t n, bmg_vec** out) {
  return guard([&] {
    if (n < 0) fail(BMG_EINVAL, "bmg_vec_create: negative length");
    Ctx* c = reinterpret_cast<Ctx*>(ctx);
    c->activate();
    auto v = std::make_unique<Vec>();
    v->ctx = c;
    v->n = n;
    v->d.alloc(std::max<int64_t>(n, 1));
    BMG_CUDA(cudaMemsetAsync(v->d.p, 0, v->d.bytes(), c->stream));
    *out = reinterpret_cast<bmg_vec*>(v.release());
  });
}
int bmg_vec_destroy(bmg_vec* v) {
  return guard([&] {
    Vec* p = reinterpret_cast<Vec*>(v);
    if (p) BMG_CUDA(cudaStreamSynchronize(p->ctx->stream));
    delete p;
  });
}
int bmg_vec_upload(bmg_vec* vh, const double* host) {
  return guard([&] {
    Vec* v = reinterpret_cast<Vec*>(vh);
    BMG_CUDA(cudaMemcpyAsync(v->d.p, host, v->n * sizeof(double), cudaMemcpyHostToDevice, v->ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(v->ctx->stream));
  });
}
int bmg_vec_download(const bmg_vec* vh, double* host) {
  return guard([&] {
    const Vec* v = reinterpret_cast<const Vec*>(vh);
    BMG_CUDA(cudaMemcpyAsync(host, v->d.p, v->n * sizeof(double), cudaMemcpyDeviceToHost, v->ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(v->ctx->stream));
  });
}
int bmg_vec_fill(bmg_vec* vh, double value) {
  return guard([&] {
    Vec* v = reinterpret_cast<Vec*>(vh);
    fill(v->ctx, v->d.p, v->n, value);
  });
}
int bmg_vec_create_like(const bmg_vec* like, bmg_vec** out) {
  return guard([&] {
    const Vec* v = reinterpret_cast<const Vec*>(like);
    if (!v) fail(BMG_EINVAL, "bmg_vec_create_like: null vector");
    v->ctx->activate();
    auto w = std::make_unique<Vec>();
    w->ctx = v->ctx;
    w->n = v->n;
    w->d.alloc(std::max<int64_t>(v->n, 1));
    BMG_CUDA(cudaMemsetAsync(w->d.p, 0, w->d.bytes(), v->ctx->stream));
    *out = reinterpret_cast<bmg_vec*>(w.release());
  });
}
int bmg_vec_copy(const bmg_vec* srch, bmg_vec* dsth) {
  return guard([&] {
    const Vec* s = reinterpret_cast<const Vec*>(srch);
    Vec* d = reinterpret_cast<Vec*>(dsth);
    if (s->n != d->n) fail(BMG_EINVAL, "bmg_vec_copy: length mismatch");
    if (s->ctx != d->ctx) fail(BMG_EINVAL, "bmg_vec_copy: vectors belong to different contexts");
    copy(d->ctx, d->d.p, s->d.p, s->n);
  });
}
int bmg_vec_axpby(double alpha, const bmg_vec* xh, double beta, const bmg_vec* yh, bmg_vec* zh) {
  return guard([&] {
    const Vec* x = reinterpret_cast<const Vec*>(xh);
    const Vec* y = reinterpret_cast<const Vec*>(yh);
    Vec* z = reinterpret_cast<Vec*>(zh);
    if (x->n != z->n || y->n != z->n) fail(BMG_EINVAL, "bmg_vec_axpby: length mismatch");
    if (x->ctx != z->ctx || y->ctx != z->ctx) fail(BMG_EINVAL, "bmg_vec_axpby: vectors belong to different contexts");
    axpby(z->ctx, z->d.p, alpha, x->d.p, beta, y->d.p, z->n);
  });
}
void* bmg_vec_device_ptr(bmg_vec* v) { return reinterpret_cast<Vec*>(v)->d.p; }
int64_t bmg_vec_size(const bmg_vec* v) { return reinterpret_cast<const Vec*>(v)->n; }

static void check_len(const Vec* v, int64_t n, const char* what) {
  if (v->n != n) fail(BMG_EINVAL, std::string(what) + ": vector length does not match layout");
}

int bmg_spmv(const bmg_bsr* ah, const bmg_vec* xh, bmg_vec* yh) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    const Vec* x = reinterpret_cast<const Vec*>(xh);
    Vec* y = reinterpret_cast<Vec*>(yh);
    check_len(x, a->dim_c, "spmv");
    check_len(y, a->dim_r, "spmv");
    spmv(*a, x->d.p, y->d.p);
  });
}
int bmg_spmv_batch(const bmg_bsr* ah, int nrhs, const bmg_vec* xh, bmg_vec* yh) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    const Vec* x = reinterpret_cast<const Vec*>(xh);
    Vec* y = reinterpret_cast<Vec*>(yh);
    if (nrhs < 1) fail(BMG_EINVAL, "spmv: nrhs must be >= 1");
    check_len(x, (int64_t)a->dim_c * nrhs, "spmv");
    check_len(y, (int64_t)a->dim_r * nrhs, "spmv");
    spmv(*a, x->d.p, y->d.p, nrhs);
  });
}
int bmg_spmv_t(const bmg_bsr* ah, const bmg_vec* xh, bmg_vec* yh) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    const Vec* x = reinterpret_cast<const Vec*>(xh);
    Vec* y = reinterpret_cast<Vec*>(yh);
    check_len(x, a->dim_r, "spmv_transpose");
    check_len(y, a->dim_c, "spmv_transpose");
    Bsr* mut = const_cast<Bsr*>(a);
    if (!mut->tcache) mut->tcache = bsr_transpose(*a);
    spmv(*mut->tcache, x->d.p, y->d.p);
  });
}
int bmg_residual(const bmg_bsr* ah, const bmg_vec* bh, const bmg_vec* xh, bmg_vec* rh) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    const Vec* b = reinterpret_cast<const Vec*>(bh);
    const Vec* x = reinterpret_cast<const Vec*>(xh);
    Vec* r = reinterpret_cast<Vec*>(rh);
    check_len(x, a->dim_c, "residual");
    check_len(b, a->dim_r, "residual");
    check_len(r, a->dim_r, "residual");
    residual(*a, b->d.p, x->d.p, r->d.p);
  });
}
int bmg_dot(const bmg_vec* ah, const bmg_vec* bh, double* out) {
  return guard([&] {
    const Vec* a = reinterpret_cast<const Vec*>(ah);
    const Vec* b = reinterpret_cast<const Vec*>(bh);
    if (a->n != b->n) fail(BMG_EINVAL, "dot: length mismatch");
    *out = dot(a->ctx, a->d.p, b->d.p, a->n);
  });
}

int bmg_time_residual(const bmg_bsr* ah, const bmg_vec* bh, const bmg_vec* xh, bmg_vec* rh, int reps,
                      double* ms) {
  return guard([&] {
    const Bsr* a = reinterpret_cast<const Bsr*>(ah);
    const Vec* b = reinterpret_cast<const Vec*>(bh);
    const Vec* x = reinterpret_cast<const Vec*>(xh);
    Vec* r = reinterpret_cast<Vec*>(rh);
    Ctx* c = a->ctx;
    cudaEvent_t e0, e1;
    BMG_CUDA(cudaEventCreate(&e0));
    BMG_CUDA(cudaEventCreate(&e1));
    residual(*a, b->d.p, x->d.p, r->d.p);  // warm
    BMG_CUDA(cudaEventRecord(e0, c->stream));
    for (int i = 0; i < reps; ++i) residual(*a, b->d.p, x->d.p, r->d.p);
    BMG_CUDA(cudaEventRecord(e1, c->stream));
    BMG_CUDA(cudaEventSynchronize(e1));
    float t = 0.f;
    BMG_CUDA(cudaEventElapsedTime(&t, e0, e1));
    *ms = (double)t / std::max(reps, 1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"
