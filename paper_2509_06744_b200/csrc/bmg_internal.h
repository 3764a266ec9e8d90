// bmg_internal.h -- host-side object model behind the C ABI (include/bmg_cuda.h).
#pragma once
#include <cuda_runtime.h>
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <atomic>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bmg_cuda.h"

namespace bmg {

// ---- errors: C++ exceptions inside, status codes at the ABI -----------------
struct Error : std::runtime_error {
  int status;
  int pivot;
  Error(int s, const std::string& m, int p = -1) : std::runtime_error(m), status(s), pivot(p) {}
};
[[noreturn]] void fail(int status, const std::string& msg, int pivot = -1);
void cuda_check(cudaError_t e, const char* what);
#define BMG_CUDA(x) ::bmg::cuda_check((x), #x)
// BMG_DEBUG_SYNC=1: synchronise and check after every launch (fault localisation)
void debug_sync(cudaStream_t s, const char* what);
#define BMG_LAUNCHED(stream, what) ::bmg::debug_sync((stream), (what))

// ---- device memory ------------------------------------------------------------
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) BMG_CUDA(cudaMalloc(&p, count * sizeof(T)));
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// A device buffer whose physical memory can be returned from the tail while the
// front stays in place (CUDA virtual memory management: one reserved address
// range, physical memory mapped in chunks).  The coarse solve factorises A_0 in
// an N0 x N0 buffer and packs the lower 64x64 tiles of the inverse into the front
// of the same buffer, then unmaps the rest: the dense matrix and the packed tiles
// are never held at the same time (C3's N0 = 86,016: 59 GB dense, 30 GB packed).
struct ShrinkBuf {
  double* p = nullptr;
  size_t n = 0;  // doubles currently backed
  ShrinkBuf() = default;
  ShrinkBuf(const ShrinkBuf&) = delete;
  ShrinkBuf& operator=(const ShrinkBuf&) = delete;
  ShrinkBuf(ShrinkBuf&& o) noexcept { swap(o); }
  ShrinkBuf& operator=(ShrinkBuf&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  ~ShrinkBuf() { release(); }
  void alloc(size_t count, int device);  // reserve + map (ceil to the chunk size)
  void shrink(size_t count);             // unmap and free the chunks beyond `count`
  void release();
  size_t bytes() const { return n * sizeof(double); }

 private:
  void swap(ShrinkBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(reserved, o.reserved);
    std::swap(chunk, o.chunk);
    std::swap(handles, o.handles);
  }
  size_t reserved = 0, chunk = 0;  // bytes
  std::vector<unsigned long long> handles;  // CUmemGenericAllocationHandle per mapped chunk
};

// ---- context ------------------------------------------------------------------
// ---- rank-to-rank transport ---------------------------------------------------
// NCCL over NVLink for real multi-GPU runs (bmg_ctx_create_nccl); a loopback
// transport (bmg_ctx_create_loopback: one host thread per rank, all on one GPU,
// send/recv matched in-process) runs the exact same exchange code where only one
// GPU exists.  Semantics follow NCCL: group_start / group_end bracket sends and
// receives; sends and receives between a pair match in posting order.
enum class DType { F64, I32, I64 };
enum class ROp { Sum, Max };
struct Comm {
  virtual ~Comm() = default;
  virtual void group_start() = 0;
  virtual void group_end() = 0;
  virtual void send(const void* p, size_t count, DType t, int peer, cudaStream_t s) = 0;
  virtual void recv(void* p, size_t count, DType t, int peer, cudaStream_t s) = 0;
  virtual void allreduce(const void* sb, void* rb, size_t count, DType t, ROp op, cudaStream_t s) = 0;
  virtual bool capturable() const = 0;  // may run inside CUDA graph capture
};
struct LoopGroup;
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const unsigned char* id128);
std::unique_ptr<Comm> make_loopback_comm(LoopGroup* g, int rank);
void nccl_unique_id(unsigned char* id128);

struct Ctx;
void ctx_retain(Ctx* c);
void ctx_release(Ctx* c);
// A counted reference to the owning context: device objects keep their context
// alive, so handles may be destroyed in any order (bmg_ctx_destroy drops the
// caller's reference; the context goes when its last object does).
struct CtxRef {
  Ctx* p = nullptr;
  CtxRef() = default;
  CtxRef(Ctx* c) : p(c) { ctx_retain(p); }  // NOLINT(google-explicit-constructor)
  CtxRef(const CtxRef& o) : p(o.p) { ctx_retain(p); }
  CtxRef& operator=(const CtxRef& o) {
    if (this != &o) {
      ctx_retain(o.p);
      ctx_release(p);
      p = o.p;
    }
    return *this;
  }
  CtxRef& operator=(Ctx* c) { return *this = CtxRef(c); }
  ~CtxRef() { ctx_release(p); }
  Ctx* operator->() const { return p; }
  operator Ctx*() const { return p; }  // NOLINT(google-explicit-constructor)
};

struct Ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int64_t launches = 0;
  cusolverDnHandle_t solver = nullptr;
  std::unique_ptr<Comm> comm;  // multi-rank context: NCCL or loopback transport
  int rank = 0, world = 1;
  DBuf<double> red;          // reduction partials
  DBuf<double> work;         // scratch of the standalone smoother
  double* h_red = nullptr;   // pinned result slot(s)
  void activate() const { BMG_CUDA(cudaSetDevice(device)); }
  void count(int n = 1) { launches += n; }
  cusolverDnHandle_t cusolver();
  cublasHandle_t blas = nullptr;
  cublasHandle_t cublas();
  std::atomic<int> refs{1};  // the creator's reference plus one per live object
  // captured standalone smoother applications (bmg_cheb4_apply / bmg_smoother_apply)
  std::map<std::vector<uint64_t>, cudaGraphExec_t> smoother_graphs;
  ~Ctx();
};

// ---- streaming plan (see bsr_stream.cuh) --------------------------------------
struct Plan {
  int cb_max = 0;        // blocks per chunk
  int rmax = 0;          // max rows per chunk
  int stages = 4;        // shared-memory ring depth
  int nctas = 0;
  int nchunks = 0;
  size_t smem = 0;
  int u = 0;             // K > 1 on a uniform layout: bsr_batch_kernel with U RHS groups
  int xl = 0;            // ... with x gathered by the consumers (XL)
  DBuf<int4> chunks;     // {blk_lo, nblk, row_lo, nrows | carry flags}
  DBuf<int> cta_chunk;   // [nctas + 1]
};

// Counted references to matrices / preconditioners: every owner (a unique_ptr, or a
// hierarchy holding the caller's inputs -- the reference's setup has value
// semantics) drops one reference and the object goes with the last one.
struct Bsr;
struct Fsai;
void bsr_retain(const Bsr* a);
void bsr_release(const Bsr* a);
void fsai_retain(const Fsai* m);
void fsai_release(const Fsai* m);
}  // namespace bmg
template <>
struct std::default_delete<bmg::Bsr> {
  void operator()(bmg::Bsr* p) const { bmg::bsr_release(p); }
};
template <>
struct std::default_delete<bmg::Fsai> {
  void operator()(bmg::Fsai* p) const { bmg::fsai_release(p); }
};
namespace bmg {

// ---- block-sparse matrix on the device ----------------------------------------
// Uniform layouts (every block m_r x m_c) store blocks row-major with a padded
// stride bs = m_r*m_c rounded up to even (16-byte aligned blocks), streamed by
// the sm_100a bulk-copy kernel.  Variable layouts use per-block value offsets
// and a warp-per-block-row kernel.
// process-unique object ids (graph cache keys must not alias a freed object's address)
uint64_t next_object_uid();

// Symmetric-half streaming of an exactly symmetric uniform A (bsr_stream.cuh SYM):
// the lower triangle as its own BSR (diagonal included, same padded blocks), the
// row of every lower block, and for every row i the lower blocks (j, i), j > i
// ascending, whose transposed products complete y_i.  colpart / sbuf are the
// pass's scratch (one stream per matrix at a time, like the context's vectors).
// what a SYM streaming pass needs besides the matrix (bsr_stream.cuh StreamArgs)
struct SymArgs {
  const int32_t* brow;  // per streamed block: the x segment of its row (vector-local block index)
  double* colpart;      // transposed products, m doubles per streamed block
  int sym_lo;           // blocks in columns below this have no stored mirror (row dots only)
};

struct SymHalf {
  std::unique_ptr<Bsr> low;
  DBuf<int32_t> brow;     // [nnzb_low + 8]
  DBuf<int64_t> up_ptr;   // [nbr + 1]
  DBuf<int32_t> up_slot;  // [nnzb - nnzb_low]: lower-block ids
  DBuf<double> colpart;   // [nnzb_low * m]
  DBuf<double> sbuf;      // [dim]
  int64_t bytes() const;
};

struct Bsr {
  CtxRef ctx;
  mutable std::atomic<int> refs{1};  // the creator's reference + hierarchies holding it
  const uint64_t uid = next_object_uid();
  int nbr = 0, nbc = 0;
  std::vector<int> rsz, csz, roff, coff;  // host layouts
  int dim_r = 0, dim_c = 0;
  bool uniform = false;
  int mr = 0, mc = 0, bs = 0;  // uniform sizes / padded stride (doubles)
  int mmax = 1;                // largest block dimension
  int64_t nnzb = 0;
  bool sym = false;
  std::vector<int64_t> h_row_ptr;
  std::vector<int32_t> h_col;
  std::vector<int64_t> h_voff;  // value offsets (unpadded for variable; padded for uniform)
  DBuf<int64_t> row_ptr;
  DBuf<int32_t> col;            // nnzb + 4 (bulk-copy padding)
  DBuf<double> vals;
  DBuf<int64_t> voff;           // variable layouts only
  DBuf<int> d_roff, d_coff, d_rsz, d_csz;
  Plan plan;                              // single right-hand side
  mutable std::unique_ptr<Plan> kplan[4];  // batched: index log2(nrhs), built on first use
  // variable layouts with a streamed block size: values padded to mmax x mmax
  // (zeros) for the streaming kernel, and its plans; built on first use
  mutable DBuf<double> pvals;
  mutable int pbs = 0;
  mutable std::unique_ptr<Plan> pplan[4];
  std::unique_ptr<Bsr> tcache;  // device transpose (spmv_t)
  // symmetric-half form (ensure_sym_half); state 0 untried, 1 built, -1 not applicable
  mutable std::unique_ptr<SymHalf> half;
  mutable int half_state = 0;
  mutable double sym_ms = 0.0, full_ms = 0.0;  // the measured choice (ensure_sym_half)
  int64_t pass_bytes() const;
  int64_t device_bytes() const;
};
// Builds a.half when a is square, uniform, streamed, flagged symmetric and its
// stored blocks are exactly (bitwise) symmetric and the half form measured
// faster (BMG_SYM_HALF=1 forces it, 0 disables it); true if a.half is usable.
// Outside graph capture.
// `next`: the pass that follows the residual in the cycle (timed with it), or null
bool ensure_sym_half(const Bsr& a, const Bsr* next = nullptr);
// algorithmic bytes of one SYM residual pass (both kernels)
int64_t sym_pass_bytes(const Bsr& a);
// the pieces of a half-storage pass on a partitioned level (vcycle.cu sym_residual_pass):
// phase 1 over a lower-part slice (row sums to S), the merge of the in-rank upper
// contributions (r = b - y, or the partial sum to tbuf from scalar row
// tsplit_rows * m on), and the tail over the blocks past the rank's own columns
void sym_phase1(const Bsr& low, const SymArgs& sa, const double* x, double* S);
void sym_merge(Ctx* ctx, int m, int64_t nrows, const int64_t* up_ptr, const int32_t* up_slot, const double* colpart,
               const double* S, const double* b, double* r, double* tbuf, int64_t tsplit_rows);
void residual_from(const Bsr& tail, const double* t, const double* b, const double* x, double* r);
// the plan of a lower-part slice for the SYM kernel (shared memory carries the row indices)
void build_sym_plan(Bsr& low);

// Device view of a block layout for the setup kernels: uniform layouts address
// block q at q * bs with m_r x m_c blocks; variable layouts through per-block
// value offsets and per-row / per-column sizes and scalar offsets.
struct BlkView {
  const int64_t* voff = nullptr;  // nullptr: q * bs
  int bs = 0;
  const int* rsz = nullptr;  // nullptr: mr
  const int* csz = nullptr;  // nullptr: mc
  const int* roff = nullptr;
  const int* coff = nullptr;
  int mr = 0, mc = 0;
#ifdef __CUDACC__
  __device__ __forceinline__ int64_t off(int64_t q) const { return voff ? voff[q] : q * bs; }
  __device__ __forceinline__ int r(int i) const { return rsz ? rsz[i] : mr; }
  __device__ __forceinline__ int c(int j) const { return csz ? csz[j] : mc; }
  __device__ __forceinline__ int64_t ro(int i) const { return roff ? (int64_t)roff[i] : (int64_t)i * mr; }
  __device__ __forceinline__ int64_t co(int j) const { return coff ? (int64_t)coff[j] : (int64_t)j * mc; }
#endif
};
BlkView blk_view(const struct Bsr& a);
int max_block(const struct Bsr& a);


struct Vec {
  CtxRef ctx;
  int64_t n = 0;
  DBuf<double> d;
};

// M = G^T G with G = L-hat^{-1} F-hat; `fwd` holds the forward factors applied
// in order (one for nest = 0: G itself), `bwd` their transposes (reverse order).
struct Fsai {
  CtxRef ctx;
  mutable std::atomic<int> refs{1};
  const uint64_t uid = next_object_uid();
  int dim = 0;
  std::vector<std::unique_ptr<Bsr>> fwd, bwd;
  const Bsr& G() const { return *fwd.back(); }
};

// ---- uploads / construction -------------------------------------------------
std::unique_ptr<Bsr> make_bsr(Ctx* ctx, int nbr, const int* rsz, int nbc, const int* csz,
                              const int64_t* row_ptr, const int32_t* col, const double* vals,
                              bool sym, bool vals_on_device = false);
// same structure, values already on the device in padded layout
std::unique_ptr<Bsr> make_bsr_structure(Ctx* ctx, int nbr, const int* rsz, int nbc, const int* csz,
                                        std::vector<int64_t> row_ptr, std::vector<int32_t> col,
                                        bool sym);
std::unique_ptr<Bsr> bsr_transpose(const Bsr& a);
void build_plan(Bsr& a);
// launch plan for nrhs right-hand sides (shared-memory size and CTA count depend
// on it); call outside graph capture before the first batched launch
const Plan& plan_for(const Bsr& a, int nrhs);
// a single-RHS plan over block rows [row0, row1) of a uniform streamed matrix (no
// data copy; outputs land at their absolute rows); nullptr if not streamable
std::unique_ptr<Plan> plan_rows(const Bsr& a, int row0, int row1);
// the same over the lower triangle of a half-storage A, and its phase 1 (row and
// transposed products of the rows' blocks; the merge follows once every range ran)
std::unique_ptr<Plan> plan_rows_sym(const Bsr& low, int row0, int row1);
void sym_phase1_rows(const Bsr& low, const Plan& P, const SymArgs& sa, const double* x, double* S);
// r = b - A x on the rows of a plan_rows plan
void residual_rows(const Bsr& a, const Plan& P, const double* b, const double* x, double* r);
// whether a variable layout runs on the streaming kernel through padded blocks
bool var_streamed(const Bsr& a);

// ---- device operations (all enqueue on ctx->stream) --------------------------
// nrhs > 1: right-hand sides interleaved per scalar row (x[i * nrhs + v]); every
// RHS is computed with the single-vector arithmetic order
void spmv(const Bsr& a, const double* x, double* y, int nrhs = 1);
void residual(const Bsr& a, const double* b, const double* x, double* r, int nrhs = 1);
void prolong_add(const Bsr& a, const double* e, double* x, int nrhs = 1);
// z = G^T w fused with the fourth-kind update: p = first ? z : mu2 p + z;
// x = (xzero ? 0 : x) + dmu p
void gt_cheb(const Bsr& gt, const double* w, double* p, double* x, double mu2, double dmu,
             bool first, bool xzero, int nrhs = 1);
// SmootherSpec (chebyshev.hpp:10-18): 0 Richardson, 1 first kind, 2 fourth kind
struct SmootherSpec {
  int kind = 2;
  double alpha = 0.0, beta = 1.0, omega = 1.0;
};
// per step of a smoother application: p = first ? z : coef*p + z; x += c*p
// (cheb_fourth_apply, cheb_first_apply, richardson_apply: chebyshev.hpp:48-115)
struct StepScalars {
  bool first;
  double coef, c;
};
std::vector<StepScalars> smoother_schedule(const SmootherSpec& s, int k);
double dot(Ctx* ctx, const double* a, const double* b, int64_t n);
void rng_symmetric(Ctx* ctx, double* v, int64_t n, uint64_t seed);
void fill(Ctx* ctx, double* p, int64_t n, double v);
void copy(Ctx* ctx, double* dst, const double* src, int64_t n);
void axpby(Ctx* ctx, double* z, double alpha, const double* x, double beta, const double* y, int64_t n);
void fsai_apply(const Fsai& m, const double* r, double* z, double* tmp1, double* tmp2);
std::unique_ptr<Fsai> fsai_build(const Bsr& a, int kind, int t_max, double tau, int nest);
std::unique_ptr<Fsai> fsai_build_pattern(const Bsr& a, const int64_t* ptr, const int32_t* col);
std::unique_ptr<Fsai> fsai_from_factors(Ctx* ctx, const Bsr& F, const double* shat_l_packed);
double lanczos_lambda_max(const Bsr& a, const Fsai& m, int iters, double safety, uint64_t seed);
std::unique_ptr<Bsr> galerkin(const Bsr& a, const Bsr& p);
// F A F^T, exactly symmetric, exact-zero blocks dropped (kernels.cpp:88-119)
std::unique_ptr<Bsr> triple_product(const Bsr& f, const Bsr& a);

// host planning for the partitioned V-cycle (partition.cpp)
void partition_rows(int nbr, const int64_t* row_ptr, int world, int granule, bool agglomerate,
                    int32_t* bounds);
void row_window(const int64_t* row_ptr, const int32_t* col, int lo, int hi, int clo, int chi,
                int32_t* ext_lo, int32_t* ext_hi);

// host helpers
std::vector<double> tridiag_eigenvalues(std::vector<double> d, std::vector<double> e);


}  // namespace bmg
