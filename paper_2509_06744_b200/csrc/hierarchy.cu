// hierarchy.cu -- construction of the device-resident multilevel hierarchy
// (setup, multilevel.cpp:36-75; injected levels), its row partition over ranks
// (NCCL or loopback transport) or virtual ranks (in-process emulation), and the
// C ABI of the hierarchy.  The V-cycle lives in vcycle.cu, the distributed setup
// in dist_setup.cu, the data model in hier.h.  Partitioning: SURVEY.md §8(e).
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
#include <cuda.h>
#include <cudaTypedefs.h>

#include "hier.h"

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

// lower 64x64 tiles of a row-major N x N matrix; `strict` zeroes entries above the
// diagonal (a triangular matrix whose upper half holds other data)
__global__ void pack_lower_tiles_kernel(const double* __restrict__ full, int64_t N, double* __restrict__ tiles,
                                        int strict) {
  int I, J;
  tile_of(blockIdx.x, &I, &J);
  double* dst = tiles + (int64_t)blockIdx.x * kTile * kTile;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e - r * kTile;
    const int64_t gr = (int64_t)I * kTile + r, gc = (int64_t)J * kTile + c;
    dst[e] = (gr < N && gc < N && (!strict || gc <= gr)) ? full[gr * N + gc] : 0.0;
  }
}

// tile row I of the packed lower tiles: block J (0..I) writes tile (I, J) to
// dst + J * 64 * 64 from `src`, which holds dense rows [row0, row0 + 64) with
// leading dimension ld (entries beyond N are zero; `strict` as above)
__global__ void pack_tile_row_kernel(const double* __restrict__ src, int64_t ld, int64_t row0, int I, int64_t N,
                                     double* __restrict__ dst, int strict) {
  const int J = blockIdx.x;
  double* d = dst + (int64_t)J * kTile * kTile;
  for (int e = threadIdx.x; e < kTile * kTile; e += blockDim.x) {
    const int r = e / kTile, c = e - r * kTile;
    const int64_t gr = (int64_t)I * kTile + r, gc = (int64_t)J * kTile + c;
    d[e] = (gr < N && gc < N && (!strict || gc <= gr)) ? src[(gr - row0) * ld + gc] : 0.0;
  }
}
// rows [0, nrows) x columns [0, ncols) of a row-major matrix with leading dimension ld
__global__ void copy_rows_kernel(const double* __restrict__ a, int64_t ld, int64_t nrows, double* __restrict__ out,
                                 int ncols) {
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x)
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) out[r * ncols + c] = c < ld ? a[r * ld + c] : 0.0;
}

// block q <- the block at src[q] (bs doubles), sources anywhere on the device
__global__ void gather_ptr_kernel(const unsigned long long* __restrict__ src, int64_t nq, int bs,
                                  double* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nq * bs; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = e / bs;
    out[e] = reinterpret_cast<const double*>(src[q])[e - q * bs];
  }
}
// flag = 1 if a block differs bitwise from the transpose of its mirror (pairs a[k], b[k])
__global__ void mirror_check_kernel(const unsigned long long* __restrict__ a, const unsigned long long* __restrict__ b,
                                    int64_t npairs, int m, int* __restrict__ flag) {
  const int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (k >= npairs) return;
  const unsigned long long* A = reinterpret_cast<const unsigned long long*>(a[k]);
  const unsigned long long* B = reinterpret_cast<const unsigned long long*>(b[k]);
  for (int e = lane; e < m * m; e += 32) {
    const int r = e / m, c = e - r * m;
    if (A[r * m + c] != B[c * m + r]) atomicOr(flag, 1);
  }
}

}  // namespace kern

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
// In-place inverse of the lower-triangular column-major n x n block at `a` (leading
// dimension lda).  cuSOLVER's Xtrtri rejects n^2 >= 2^31, so larger blocks recurse on
// their diagonal halves and finish the off-diagonal block with two in-place 64-bit
// TRMMs: W21 = -W22 L21 W11.
// Lower Cholesky (column-major, in place) of an n x n matrix with n^2 beyond what
// cuSOLVER's dense factorisations handle (C3's N0 = 86,016: 7.4e9 elements; the
// 64-bit Xpotrf fails there): right-looking blocked algorithm, the diagonal
// blocks by Dpotrf (nb x nb, 32-bit safe), the panel by a 64-bit TRSM and the
// trailing update by a 64-bit SYRK.
static void blocked_potrf(Ctx* ctx, double* a, int64_t n, int64_t lda) {
  constexpr int64_t nb = 2048;
  cusolverDnHandle_t s = ctx->cusolver();
  cublasHandle_t b = ctx->cublas();
  int lwork = 0;
  if (cusolverDnDpotrf_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)nb, a, (int)lda, &lwork) != CUSOLVER_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cusolverDnDpotrf_bufferSize failed");
  DBuf<double> work(std::max(lwork, 1));
  DBuf<int> info(1);
  const double one = 1.0, minus = -1.0;
  for (int64_t k = 0; k < n; k += nb) {
    const int64_t kb = std::min(nb, n - k);
    double* a11 = a + k + k * lda;
    if (cusolverDnDpotrf(s, CUBLAS_FILL_MODE_LOWER, (int)kb, a11, (int)lda, work.p, lwork, info.p) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnDpotrf (diagonal block) failed");
    int hinfo = 0;
    BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hinfo != 0) fail(BMG_ERUNTIME, "setup: coarsest operator is not positive definite");
    const int64_t rest = n - k - kb;
    if (rest <= 0) break;
    double* a21 = a11 + kb;
    double* a22 = a21 + kb * lda;
    if (cublasDtrsm_v2_64(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, rest, kb,
                          &one, a11, lda, a21, lda) != CUBLAS_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cublasDtrsm (Cholesky panel) failed");
    if (cublasDsyrk_v2_64(b, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, rest, kb, &minus, a21, lda, &one, a22, lda) !=
        CUBLAS_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cublasDsyrk (Cholesky update) failed");
  }
}

static void tri_inverse(Ctx* ctx, double* a, int64_t n, int64_t lda, DBuf<double>& scratch) {
  constexpr int64_t kMax = ((int64_t)1 << 31) - 1;
  if (n * n < kMax) {
    const bool compact = lda != n;
    double* w = a;
    if (compact) {
      if (scratch.n < (size_t)(n * n)) scratch.alloc(n * n);
      w = scratch.p;
      BMG_CUDA(cudaMemcpy2DAsync(w, n * 8, a, lda * 8, n * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    cusolverDnHandle_t s = ctx->cusolver();
    size_t dws = 0, hws = 0;
    if (cusolverDnXtrtri_bufferSize(s, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, w, n, &dws,
                                    &hws) != CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnXtrtri_bufferSize failed");
    DBuf<unsigned char> dwork(std::max<size_t>(dws, 1));
    std::vector<unsigned char> hwork(std::max<size_t>(hws, 1));
    DBuf<int> info(1);
    const auto st = cusolverDnXtrtri(s, CUBLAS_FILL_MODE_LOWER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, w, n, dwork.p,
                                     dws, hwork.data(), hws, info.p);
    if (st != CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnXtrtri failed (status " + std::to_string((int)st) + ", n " + std::to_string(n) + ")");
    int hinfo = 0;
    BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hinfo != 0) fail(BMG_ERUNTIME, "setup: coarse triangular inverse failed");
    if (compact)
      BMG_CUDA(cudaMemcpy2DAsync(a, lda * 8, w, n * 8, n * 8, n, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  const int64_t n1 = (n / 2 + 63) / 64 * 64, n2 = n - n1;
  double* a22 = a + n1 + n1 * lda;
  double* a21 = a + n1;
  tri_inverse(ctx, a, n1, lda, scratch);
  tri_inverse(ctx, a22, n2, lda, scratch);
  cublasHandle_t b = ctx->cublas();
  const double one = 1.0, minus = -1.0;
  if (cublasDtrmm_v2_64(b, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n2, n1, &one,
                        a, lda, a21, lda, a21, lda) != CUBLAS_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cublasDtrmm (L21 W11) failed");
  if (cublasDtrmm_v2_64(b, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n2, n1, &minus,
                        a22, lda, a21, lda, a21, lda) != CUBLAS_STATUS_SUCCESS)
    fail(BMG_ECUDA, "cublasDtrmm (W22 L21 W11) failed");
}

// ---- ShrinkBuf (bmg_internal.h) ------------------------------------------------
// The driver's virtual-memory calls are resolved through the runtime
// (cudaGetDriverEntryPoint), so the library does not link libcuda and still loads
// on a GPU-less host (where every compute entry reports BMG_ECUDA).
struct VmmApi {
  PFN_cuMemGetAllocationGranularity granularity = nullptr;
  PFN_cuMemAddressReserve reserve = nullptr;
  PFN_cuMemAddressFree addr_free = nullptr;
  PFN_cuMemCreate create = nullptr;
  PFN_cuMemRelease release = nullptr;
  PFN_cuMemMap map = nullptr;
  PFN_cuMemUnmap unmap = nullptr;
  PFN_cuMemSetAccess set_access = nullptr;
};
static const VmmApi& vmm() {
  static const VmmApi api = [] {
    VmmApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
          !*fn)
        fail(BMG_ECUDA, std::string("driver entry point unavailable: ") + name);
    };
    get("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&a.granularity));
    get("cuMemAddressReserve", reinterpret_cast<void**>(&a.reserve));
    get("cuMemAddressFree", reinterpret_cast<void**>(&a.addr_free));
    get("cuMemCreate", reinterpret_cast<void**>(&a.create));
    get("cuMemRelease", reinterpret_cast<void**>(&a.release));
    get("cuMemMap", reinterpret_cast<void**>(&a.map));
    get("cuMemUnmap", reinterpret_cast<void**>(&a.unmap));
    get("cuMemSetAccess", reinterpret_cast<void**>(&a.set_access));
    return a;
  }();
  return api;
}
static void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) fail(BMG_ECUDA, std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
}

void ShrinkBuf::alloc(size_t count, int device) {
  release();
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  size_t gran = 0;
  cu_check(vmm().granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
  const size_t want = std::max<size_t>(count, 1) * sizeof(double);
  chunk = ((std::max<size_t>(want / 64, (size_t)256 << 20) + gran - 1) / gran) * gran;  // <= 64 chunks, >= 256 MB
  reserved = (want + chunk - 1) / chunk * chunk;
  CUdeviceptr base = 0;
  cu_check(vmm().reserve(&base, reserved, 0, 0, 0), "cuMemAddressReserve");
  p = reinterpret_cast<double*>(base);
  try {
    for (size_t off = 0; off < reserved; off += chunk) {
      CUmemGenericAllocationHandle hd;
      cu_check(vmm().create(&hd, chunk, &prop, 0), "cuMemCreate");
      handles.push_back(hd);
      cu_check(vmm().map(base + off, chunk, 0, hd, 0), "cuMemMap");
    }
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    cu_check(vmm().set_access(base, reserved, &acc, 1), "cuMemSetAccess");
  } catch (...) {
    release();
    throw;
  }
  n = count;
}

void ShrinkBuf::shrink(size_t count) {
  if (!p || count >= n) return;
  const size_t keep = (std::max<size_t>(count, 1) * sizeof(double) + chunk - 1) / chunk;  // chunks kept
  const CUdeviceptr base = reinterpret_cast<CUdeviceptr>(p);
  while (handles.size() > keep) {
    const size_t i = handles.size() - 1;
    cu_check(vmm().unmap(base + i * chunk, chunk), "cuMemUnmap");
    cu_check(vmm().release(handles[i]), "cuMemRelease");
    handles.pop_back();
  }
  n = count;
}

void ShrinkBuf::release() {
  if (p) {
    const CUdeviceptr base = reinterpret_cast<CUdeviceptr>(p);
    for (size_t i = 0; i < handles.size(); ++i) {
      vmm().unmap(base + i * chunk, chunk);
      vmm().release(handles[i]);
    }
    vmm().addr_free(base, reserved);
  }
  handles.clear();
  p = nullptr;
  n = 0;
  reserved = chunk = 0;
}

void coarse_factor(Hier& h, Part& p) {
  Ctx* ctx = h.ctx;
  const Bsr& a0 = *p.lv[0].A;
  if (!(a0.rsz == a0.csz)) fail(BMG_EINVAL, "coarse solve: square block layout required");
  const int64_t N = a0.dim_r;
  h.n0 = N;
  p.ainv.alloc((size_t)std::max<int64_t>(N * N, 1), ctx->device);
  BMG_CUDA(cudaMemsetAsync(p.ainv.p, 0, p.ainv.bytes(), ctx->stream));
  kern::bsr_to_dense_kernel<<<std::max(1, std::min(a0.nbr, ctx->sms * 8)), 128, 0, ctx->stream>>>(
      a0.vals.p, blk_view(a0), a0.row_ptr.p, a0.col.p, a0.nbr, p.ainv.p, N);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  cusolverDnHandle_t s = ctx->cusolver();
  // 32-bit potrf + potri while N^2 < 2^31; beyond that (C3, C5 coarsest levels) the
  // 64-bit Xpotrf + Xtrtri give W = L^{-1} and the solve is x = W^T (W b)
  static const bool force_tri = [] {
    const char* e = std::getenv("BMG_COARSE_TRIANGULAR");
    return e && e[0] == '1';
  }();
  p.tri = force_tri || N * N >= ((int64_t)1 << 31) - 1;
  DBuf<int> info(1);
  int hinfo = 0;
  auto check_info = [&](const char* what) {
    BMG_CUDA(cudaMemcpyAsync(&hinfo, info.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hinfo != 0) fail(BMG_ERUNTIME, what);
  };
  if (!p.tri) {
    int lwork = 0, lwork2 = 0;
    if (cusolverDnDpotrf_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, &lwork) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnDpotrf_bufferSize failed");
    if (cusolverDnDpotri_bufferSize(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, &lwork2) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnDpotri_bufferSize failed");
    DBuf<double> work(std::max(std::max(lwork, lwork2), 1));
    if (cusolverDnDpotrf(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, work.p, lwork, info.p) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnDpotrf failed");
    check_info("setup: coarsest operator is not positive definite");
    if (cusolverDnDpotri(s, CUBLAS_FILL_MODE_LOWER, (int)N, p.ainv.p, (int)N, work.p, lwork2, info.p) !=
        CUSOLVER_STATUS_SUCCESS)
      fail(BMG_ECUDA, "cusolverDnDpotri failed");
    check_info("setup: coarse inverse failed");
  } else {
    blocked_potrf(ctx, p.ainv.p, N, N);
    DBuf<double> scratch;
    tri_inverse(ctx, p.ainv.p, N, N, scratch);
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  // column-major lower = row-major upper: mirror it into the row-major lower half
  kern::symmetrize_dense_kernel<<<grid1d(N * N), 256, 0, ctx->stream>>>(p.ainv.p, N);
  ctx->count();
  BMG_CUDA(cudaGetLastError());
  // keep only the lower 64x64 tiles, packed into the front of the same buffer, one
  // tile row at a time in ascending order: tile row I's packed range ends before
  // the first dense row it reads (I >= 1, N >= 256), and every later row reads
  // behind it, so no unread entry is overwritten; row 0 overlaps its own source
  // and goes through a 64 x 64 staging copy.  The tail is then unmapped.
  const int nt = (int)((N + kern::kTile - 1) / kern::kTile);
  const int64_t ntiles = (int64_t)nt * (nt + 1) / 2;
  const int64_t T2 = (int64_t)kern::kTile * kern::kTile;
  if (N >= 4 * kern::kTile) {
    DBuf<double> stage((size_t)T2);
    kern::copy_rows_kernel<<<kern::kTile, 128, 0, ctx->stream>>>(p.ainv.p, N, std::min<int64_t>(N, kern::kTile),
                                                                 stage.p, kern::kTile);
    kern::pack_tile_row_kernel<<<1, 256, 0, ctx->stream>>>(stage.p, kern::kTile, 0, 0, N, p.ainv.p, p.tri ? 1 : 0);
    ctx->count(2);
    for (int I = 1; I < nt; ++I) {
      kern::pack_tile_row_kernel<<<I + 1, 256, 0, ctx->stream>>>(p.ainv.p + (int64_t)I * kern::kTile * N, N,
                                                                   (int64_t)I * kern::kTile, I, N,
                                                                   p.ainv.p + ((int64_t)I * (I + 1) / 2) * T2,
                                                                   p.tri ? 1 : 0);
      ctx->count();
    }
    BMG_CUDA(cudaGetLastError());
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    p.ainv.shrink((size_t)(ntiles * T2));
  } else {  // tiny coarse levels: a separate packed copy
    DBuf<double> tiles((size_t)(ntiles * T2));
    kern::pack_lower_tiles_kernel<<<(unsigned)ntiles, 256, 0, ctx->stream>>>(p.ainv.p, N, tiles.p, p.tri ? 1 : 0);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    p.ainv.alloc((size_t)(ntiles * T2), ctx->device);
    BMG_CUDA(cudaMemcpyAsync(p.ainv.p, tiles.p, tiles.bytes(), cudaMemcpyDeviceToDevice, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  p.cpart.alloc((size_t)nt * nt * kern::kTile);
  BMG_CUDA(cudaMemsetAsync(p.cpart.p, 0, p.cpart.bytes(), ctx->stream));
}

void alloc_vectors(Hier& h, PLevel& L, bool top) {
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
    s.a_pass = L.A->half ? sym_pass_bytes(*L.A) : L.A->pass_bytes();
    s.a_pass_ref = L.A->pass_bytes();
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
  // symmetric-half streaming of every smoothed level's A (bitwise the same passes,
  // about half the bytes; kept full when A is not exactly symmetric)
  for (int l = 1; l < L; ++l) ensure_sym_half(*p.lv[l].A, p.lv[l].M->fwd.front().get());
  record_stats(h);
}

// rows [lo, hi) of g with columns shifted by -col_lo into a window of ncols blocks
std::unique_ptr<Bsr> slice_rows(const Bsr& g, int lo, int hi, int col_lo, int ncols) {
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
SplitMat split_rows(const Bsr& g, int lo, int hi, int wlo, int nwin, int own_lo, int own_hi) {
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

// ---- half-storage A on partitioned levels (hier.h PSym) -----------------------------
// One rank's share: the SplitMat's slices hold its own rows [0, n) (level rows
// lo + i) with columns in the vector window; own columns are [oc0, oc1).  nullptr
// when the in-rank blocks are not exactly symmetric.
static std::unique_ptr<PSym> build_psym(Ctx* ctx, const SplitMat& sA, int n, int oc0, int oc1, int m) {
  struct Blk {
    int col;
    const double* v;
  };
  std::vector<std::vector<Blk>> rows(n);
  int nwin = 0;
  for (const Slice& sl : sA.s) {
    const Bsr& a = *sl.m;
    if (!a.uniform || a.mr != m || a.mc != m) return nullptr;
    nwin = a.nbc;
    for (int rr = 0; rr < a.nbr; ++rr)
      for (int64_t q = a.h_row_ptr[rr]; q < a.h_row_ptr[rr + 1]; ++q)
        rows[sl.row0 + rr].push_back({a.h_col[q], a.vals.p + q * a.bs});
  }
  auto P = std::make_unique<PSym>();
  P->n = n;
  P->m = m;
  P->oc0 = oc0;
  // rows that read the lower halo come first (phase 1 waits for the exchange there)
  int k1 = 0;
  for (int i = 0; i < n; ++i)
    if (!rows[i].empty() && rows[i].front().col < oc0) k1 = i + 1;
  P->k1 = k1;
  int t0 = n;
  for (int i = n - 1; i >= 0; --i)
    if (!rows[i].empty() && rows[i].back().col >= oc1) t0 = i;
  P->t0 = t0;
  // the lower part (columns <= the diagonal's), boundary rows first
  std::vector<int64_t> rp_b(1, 0), rp_i(1, 0), rp_t(1, 0);
  std::vector<int32_t> col_b, col_i, col_t, brow;
  std::vector<unsigned long long> src_low, src_tail;
  std::vector<std::vector<std::pair<int, int64_t>>> low_of(n);  // (column, lower block id) per row
  int64_t nlow = 0;
  for (int i = 0; i < n; ++i) {
    const int dc = i + oc0;
    for (const Blk& b : rows[i]) {
      if (b.col > dc) continue;
      (i < k1 ? col_b : col_i).push_back(b.col);
      src_low.push_back((unsigned long long)b.v);
      brow.push_back(dc);
      low_of[i].push_back({b.col, nlow++});
    }
    (i < k1 ? rp_b : rp_i).push_back((int64_t)(i < k1 ? col_b.size() : col_i.size()));
    if (i >= t0) {
      for (const Blk& b : rows[i])
        if (b.col >= oc1) {
          col_t.push_back(b.col);
          src_tail.push_back((unsigned long long)b.v);
        }
      rp_t.push_back((int64_t)col_t.size());
    }
  }
  P->nlow_bnd = (int64_t)col_b.size();
  // in-rank upper blocks of every row: the lower block (j, i) holding their products
  std::vector<int64_t> uptr(n + 1, 0);
  std::vector<int32_t> uslot;
  std::vector<unsigned long long> pa, pb;  // (upper block, its mirror) for the exact-symmetry check
  for (int i = 0; i < n; ++i) {
    const int dc = i + oc0;
    for (const Blk& b : rows[i]) {
      if (b.col <= dc || b.col >= oc1) continue;
      const int j = b.col - oc0;
      const auto& lj = low_of[j];
      auto it = std::lower_bound(lj.begin(), lj.end(), std::make_pair(dc, (int64_t)-1));
      if (it == lj.end() || it->first != dc) return nullptr;  // structurally unsymmetric
      uslot.push_back((int32_t)it->second);
      pa.push_back((unsigned long long)b.v);
      pb.push_back(src_low[it->second]);
    }
    uptr[i + 1] = (int64_t)uslot.size();
  }
  if (nlow >= ((int64_t)1 << 31)) return nullptr;
  {  // the half form is kept beside the full-storage slices (batched cycles use those):
     // only where it fits with 2 GB to spare (C5 on 4 GPUs: rank 0 skips the levels
     // that would not fit; every rank then keeps full storage there)
    const int bs_ = (m * m + 1) & ~1;
    const int64_t need = (nlow + (int64_t)src_tail.size()) * (int64_t)bs_ * 8 + nlow * (int64_t)m * 8 +
                         2 * (int64_t)n * m * 8 + ((int64_t)2 << 30);
    size_t fr = 0, tot = 0;
    BMG_CUDA(cudaMemGetInfo(&fr, &tot));
    if ((int64_t)fr < need) return nullptr;
  }
  if (!pa.empty()) {
    DBuf<unsigned long long> da(pa.size()), db(pb.size());
    DBuf<int> flag(1);
    BMG_CUDA(cudaMemcpy(da.p, pa.data(), pa.size() * 8, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemcpy(db.p, pb.data(), pb.size() * 8, cudaMemcpyHostToDevice));
    BMG_CUDA(cudaMemset(flag.p, 0, sizeof(int)));
    kern::mirror_check_kernel<<<(unsigned)((pa.size() * 32 + 255) / 256), 256, 0, ctx->stream>>>(
        da.p, db.p, (int64_t)pa.size(), m, flag.p);
    ctx->count();
    BMG_CUDA(cudaGetLastError());
    int h = 0;
    BMG_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h) return nullptr;
  }
  const int bs = (m * m + 1) & ~1;
  auto make = [&](int nr, std::vector<int64_t> rp, std::vector<int32_t> cl,
                  const unsigned long long* src, int64_t nb, bool sym) -> std::unique_ptr<Bsr> {
    if (nr == 0) return nullptr;
    std::vector<int> rsz(nr, m), csz(nwin, m);
    auto a = make_bsr_structure(ctx, nr, rsz.data(), nwin, csz.data(), std::move(rp), std::move(cl), false);
    if (nb > 0) {
      DBuf<unsigned long long> d(nb);
      BMG_CUDA(cudaMemcpy(d.p, src, nb * 8, cudaMemcpyHostToDevice));
      kern::gather_ptr_kernel<<<grid1d(nb * bs), 256, 0, ctx->stream>>>(d.p, nb, bs, a->vals.p);
      ctx->count();
      BMG_CUDA(cudaGetLastError());
      BMG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (sym) build_sym_plan(*a);
    return a;
  };
  P->low_bnd = make(k1, std::move(rp_b), std::move(col_b), src_low.data(), P->nlow_bnd, true);
  P->low_int = make(n - k1, std::move(rp_i), std::move(col_i), src_low.data() + P->nlow_bnd, nlow - P->nlow_bnd,
                    true);
  P->tail = make(n - t0, std::move(rp_t), std::move(col_t), src_tail.data(), (int64_t)src_tail.size(), false);
  // the interior slice's rows start 16-byte aligned (its bulk copies read from there)
  P->brow_int_off = (P->nlow_bnd + 3) & ~(int64_t)3;
  const int64_t nint = nlow - P->nlow_bnd;
  P->brow.alloc(P->brow_int_off + nint + 8);
  BMG_CUDA(cudaMemset(P->brow.p, 0, (P->brow_int_off + nint + 8) * 4));
  if (P->nlow_bnd) BMG_CUDA(cudaMemcpy(P->brow.p, brow.data(), P->nlow_bnd * 4, cudaMemcpyHostToDevice));
  if (nint)
    BMG_CUDA(cudaMemcpy(P->brow.p + P->brow_int_off, brow.data() + P->nlow_bnd, nint * 4, cudaMemcpyHostToDevice));
  P->up_ptr.alloc(n + 1);
  BMG_CUDA(cudaMemcpy(P->up_ptr.p, uptr.data(), (n + 1) * 8, cudaMemcpyHostToDevice));
  P->up_slot.alloc(std::max<size_t>(uslot.size(), 1));
  if (!uslot.empty()) BMG_CUDA(cudaMemcpy(P->up_slot.p, uslot.data(), uslot.size() * 4, cudaMemcpyHostToDevice));
  P->colpart.alloc(std::max<int64_t>(nlow, 1) * m);
  P->sbuf.alloc(std::max<int64_t>((int64_t)n * m, 1));
  P->tbuf.alloc(std::max<int64_t>((int64_t)(n - t0) * m, 1));
  const int64_t nup = (int64_t)uslot.size(), ntail = (int64_t)src_tail.size();
  P->pass_bytes = nlow * (8 * (int64_t)m * m + 8) + nup * (16 * (int64_t)m + 4) + 16 * (int64_t)n * m +
                  8 * ((int64_t)n + 1) + ntail * (8 * (int64_t)m * m + 4) + 16 * (int64_t)(n - t0) * m;
  return P;
}

void build_level_psym(Hier& h) {
  static const int mode = [] {
    const char* e = std::getenv("BMG_SYM_HALF");
    return !e ? -1 : (e[0] == '0' ? 0 : 1);
  }();
  if (h.whole() || mode == 0) return;
  Ctx* ctx = h.ctx;
  const bool nccl = !h.emulated && h.world > 1;
  auto reduce = [&](std::vector<int64_t>& v, ROp op) {
    if (!nccl) return;
    DBuf<int64_t> d(v.size());
    BMG_CUDA(cudaMemcpy(d.p, v.data(), v.size() * 8, cudaMemcpyHostToDevice));
    ctx->comm->allreduce(d.p, d.p, v.size(), DType::I64, op, ctx->stream);
    BMG_CUDA(cudaMemcpyAsync(v.data(), d.p, v.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    BMG_CUDA(cudaStreamSynchronize(ctx->stream));
  };
  const int L = h.finest() + 1;
  h.psym_on.assign(L, 0);
  // eligibility from the whole level's full-storage bytes (same on every rank): the
  // half form measured faster on the m >= 15 operators of C3 / C4 / C5 with passes of
  // >= 0.5 ms (hierarchy.cu ensure_sym_half); BMG_SYM_HALF=1 forces every level
  std::vector<int64_t> bytes(L, 0);
  for (Part& p : h.parts)
    for (int l = 1; l < L; ++l)
      if (p.lv[l].active() && !p.lv[l].sA.s.empty() && p.lv[l].lo >= 0)
        for (const Slice& sl : p.lv[l].sA.s) bytes[l] += sl.m->pass_bytes();
  reduce(bytes, ROp::Sum);
  std::vector<int64_t> bad(L, 0);  // any rank unable -> full storage everywhere
  for (int l = 1; l < L; ++l) {
    const bool partitioned = h.bounds[l].size() > 2 && h.bounds[l][1] < h.nbr[l];  // not held whole by rank 0
    const int ml = h.msz[l];
    const bool streamed = ml == 3 || ml == 6 || ml == 10 || ml == 15 || ml == 20 || ml == 21;
    const bool eligible = streamed && (mode == 1 || (ml >= 15 && bytes[l] >= (int64_t)3e9));
    if (!partitioned || !eligible) {
      bad[l] = 1;
      continue;
    }
    for (Part& p : h.parts) {
      PLevel& d = p.lv[l];
      if (!d.active()) continue;
      d.psym = build_psym(ctx, d.sA, d.hi - d.lo, d.lo - d.wlo, d.hi - d.wlo, d.m);
      if (!d.psym) bad[l] = 1;
    }
  }
  reduce(bad, ROp::Max);
  for (int l = 1; l < L; ++l) {
    const bool ok = bad[l] == 0;
    h.psym_on[l] = ok ? 1 : 0;
    if (!ok)
      for (Part& p : h.parts) p.lv[l].psym.reset();
  }
  BMG_CUDA(cudaStreamSynchronize(ctx->stream));
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
  build_level_psym(h);
}

}  // namespace bmg

// ============================================================================ C ABI
using namespace bmg;

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
    h->hold(af);
    SetupClock clk(ctx);
    for (int l = depth; l >= 1; --l) {
      PLevel& L = p.lv[l];
      L.P = B_(transfers[l - 1]);
      h->hold(L.P);
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
      h->hold(L.A);
      if (l >= 1) {
        L.P = B_(P[l]);
        h->hold(L.P);
        if (L.P->dim_r != L.A->dim_r || L.P->dim_c != B_(A[l - 1])->dim_r)
          fail(BMG_EINVAL, "hierarchy: prolongation shape does not match the levels");
        L.R_own = bsr_transpose(*L.P);
        L.R = L.R_own.get();
        L.M = M_(Mh[l]);
        h->hold(L.M);
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
// traffic per right-hand side; `ref`: A passes at full storage (the reference's)
static int64_t cycle_bytes(const Hier* h, int kpre, int kpost, int nrhs, bool ref);
int bmg_hier_cycle_bytes_batch(const bmg_hier* hh, int kpre, int kpost, int nrhs, int64_t* bytes) {
  return guard([&] { *bytes = cycle_bytes(H_(hh), kpre, kpost, nrhs, false); });
}
int bmg_hier_cycle_bytes_ref(const bmg_hier* hh, int kpre, int kpost, int64_t* bytes) {
  return guard([&] { *bytes = cycle_bytes(H_(hh), kpre, kpost, 1, true); });
}
static int64_t cycle_bytes(const Hier* h, int kpre, int kpost, int nrhs, bool ref) {
  {
    const int64_t K = std::max(1, nrhs);
    int64_t tot = 0;
    const int top = h->finest();
    for (int l = 1; l <= top; ++l) {
      const LevelStats& s = h->stats[l];
      const int64_t n = s.n * K, nc = h->stats[l - 1].n * K;
      const int64_t a_bytes = (ref && s.a_pass_ref) ? s.a_pass_ref : (nrhs > 1 && s.a_pass_ref ? s.a_pass_ref : s.a_pass);
      const int64_t apass = a_bytes + 24 * n;  // x, b read; r write
      const int64_t gvec = 16 * n + 40 * n;     // G: r, w; G^T+cheb: w, p rw, x rw
      const int steps = kpre + kpost;
      int64_t lvl = steps * (apass + s.m_pass + gvec);
      if (l < top && kpre > 0) lvl -= apass + 8 * n;  // first coarse pre-step: A*0 skipped, x not read
      lvl += apass;                                   // residual before restriction
      lvl += s.r_pass + 8 * n + 8 * nc;               // restriction
      lvl += s.p_pass + 8 * nc + 16 * n;              // prolongation x += P e
      tot += lvl;
    }
    {  // coarse solve: packed lower tiles of A_0^{-1} (or W = L^{-1}, read twice), x, b, partials
      const int64_t nt = (h->n0 + 63) / 64;
      bool tri = h->n0 * h->n0 >= ((int64_t)1 << 31) - 1;
      for (const Part& p : h->parts)
        if (p.ainv.p) tri = p.tri;
      const int64_t one = nt * (nt + 1) / 2 * 64 * 64 * 8 + (16 * h->n0 + 2 * nt * nt * 64 * 8) * K;
      tot += tri ? 2 * one : one;
    }
    return tot;
  }
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

// v_cycle(h, spec, level, b, x) (multilevel.cpp:77-103) started on any level of a
// whole hierarchy; b and x have that level's length (level 0: the direct solve)
int bmg_vcycle_level(bmg_hier* hh, int kpre, int kpost, int level, const bmg_vec* b, bmg_vec* x) {
  return guard([&] {
    Hier* h = H_(hh);
    h->ctx->activate();
    if (kpre + kpost < 1) fail(BMG_EINVAL, "v_cycle: cycle needs at least one smoothing step");
    if (level < 0 || level > h->finest()) fail(BMG_ERANGE, "v_cycle: level out of range");
    if (level != h->finest() && !h->whole())
      fail(BMG_EINVAL, "v_cycle: levels below the finest need an unpartitioned hierarchy");
    set_nrhs(*h, 1);
    const int64_t n = h->parts[0].lv[level].n_own();
    need_len(V_(b), n, "v_cycle");
    need_len(V_(x), n, "v_cycle");
    h->top = level;
    try {
      run_vcycle(*h, kpre, kpost, V_(b)->d.p, V_(x)->d.p);
    } catch (...) {
      h->top = -1;
      throw;
    }
    h->top = -1;
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
    if (kpre + kpost < 1) fail(BMG_EINVAL, "v_cycle: cycle needs at least one smoothing step");
    ensure_host_io(*h, n);
    if (!run_vcycle_hostio(*h, kpre, kpost, b, x)) {
      BMG_CUDA(cudaMemcpyAsync(h->io_b.p, b, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      BMG_CUDA(cudaMemcpyAsync(h->io_x.p, x, n * 8, cudaMemcpyHostToDevice, ctx->stream));
      run_vcycle(*h, kpre, kpost, h->io_b.p, h->io_x.p);
      BMG_CUDA(cudaMemcpyAsync(x, h->io_x.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
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
    if (solve_device(*h, kpre, kpost, b, x, tol, max_iter, hist, iters, status)) return;
    PLevel& F = h->parts[0].lv[h->finest()];
    auto resid = [&]() {
      finest_residual(*h, b, x, F.v[VR].p);
      return finest_norm(*h, F.v[VR].p);
    };
    hist[0] = resid();
    int it = 0, st = 1;
    if (hist[0] == 0.0 || hist[0] / hist[0] < tol) st = 0;  // as the oracle (orc_solve) and measure_rates
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

// measure_rates (experiments.cpp:15-67)
int bmg_measure_rates(bmg_hier* hh, const bmg_bsr* mass, const bmg_vec* b, const bmg_vec* u_ref, int kpre,
                      int kpost, uint64_t seed, double tol, int max_iter, double* l2_sq, double* energy_sq,
                      double* residual_hist, int* iters, int* status, int* blowup, double* rates) {
  return guard([&] {
    Hier* h = H_(hh);
    h->ctx->activate();
    if (max_iter < 0) fail(BMG_EINVAL, "measure_rates: max_iter must be >= 0");
    const int64_t n = finest_len(*h);
    need_len(V_(b), n, "measure_rates");
    need_len(V_(u_ref), n, "measure_rates");
    measure_rates(*h, *B_(mass), V_(b)->d.p, V_(u_ref)->d.p, kpre, kpost, seed, tol, max_iter, l2_sq, energy_sq,
                  residual_hist, iters, status, blowup, rates);
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

int bmg_ctx_transport_selftest(bmg_ctx* c, int64_t count, int reps, int64_t* mismatches) {
  return guard([&] {
    Ctx* ctx = reinterpret_cast<Ctx*>(c);
    if (!ctx || !ctx->comm) fail(BMG_EINVAL, "transport selftest: the context has no transport");
    if (count < 1 || reps < 1) fail(BMG_EINVAL, "transport selftest: count and reps must be >= 1");
    ctx->activate();
    Comm& comm = *ctx->comm;
    const int self = ctx->rank;
    DBuf<double> src, dst, red;
    src.alloc((size_t)count);
    dst.alloc((size_t)count);
    red.alloc(2);
    std::vector<double> hsrc((size_t)count);
    for (int64_t i = 0; i < count; ++i) hsrc[(size_t)i] = 1.0 + (double)(i % 1021) * 0.5;
    BMG_CUDA(cudaMemcpy(src.p, hsrc.data(), (size_t)count * 8, cudaMemcpyHostToDevice));
    cudaStream_t side;
    cudaEvent_t fork, join;
    BMG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    BMG_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    BMG_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    cudaStream_t main = ctx->stream ? ctx->stream : ctx->own;
    auto exchange_once = [&] {  // the shape of vcycle.cu exchange(): fork, grouped send/recv, join
      BMG_CUDA(cudaEventRecord(fork, main));
      BMG_CUDA(cudaStreamWaitEvent(side, fork, 0));
      comm.group_start();
      comm.send(src.p, (size_t)count, DType::F64, self, side);
      comm.recv(dst.p, (size_t)count, DType::F64, self, side);
      comm.group_end();
      BMG_CUDA(cudaEventRecord(join, side));
      BMG_CUDA(cudaStreamWaitEvent(main, join, 0));
    };
    int64_t bad = 0;
    auto check = [&] {
      std::vector<double> h((size_t)count);
      BMG_CUDA(cudaMemcpyAsync(h.data(), dst.p, (size_t)count * 8, cudaMemcpyDeviceToHost, main));
      BMG_CUDA(cudaStreamSynchronize(main));
      for (int64_t i = 0; i < count; ++i)
        if (h[(size_t)i] != hsrc[(size_t)i]) ++bad;
      BMG_CUDA(cudaMemsetAsync(dst.p, 0, (size_t)count * 8, main));
    };
    if (comm.capturable()) {
      cudaGraph_t g = nullptr;
      cudaGraphExec_t ex = nullptr;
      BMG_CUDA(cudaStreamBeginCapture(main, cudaStreamCaptureModeThreadLocal));
      try {
        exchange_once();
      } catch (...) {
        cudaStreamEndCapture(main, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      BMG_CUDA(cudaStreamEndCapture(main, &g));
      BMG_CUDA(cudaGraphInstantiate(&ex, g, 0));
      cudaGraphDestroy(g);
      for (int r = 0; r < reps; ++r) {
        BMG_CUDA(cudaGraphLaunch(ex, main));
        check();
      }
      cudaGraphExecDestroy(ex);
    } else {
      for (int r = 0; r < reps; ++r) {
        exchange_once();
        check();
      }
    }
    // sum all-reduce of {1, rank}: world and world (world - 1) / 2
    const double in[2] = {1.0, (double)ctx->rank};
    double out[2] = {0.0, 0.0};
    BMG_CUDA(cudaMemcpyAsync(red.p, in, 16, cudaMemcpyHostToDevice, main));
    comm.allreduce(red.p, red.p, 2, DType::F64, ROp::Sum, main);
    BMG_CUDA(cudaMemcpyAsync(out, red.p, 16, cudaMemcpyDeviceToHost, main));
    BMG_CUDA(cudaStreamSynchronize(main));
    if (out[0] != (double)ctx->world || out[1] != 0.5 * ctx->world * (ctx->world - 1)) ++bad;
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    cudaStreamDestroy(side);
    *mismatches = bad;
  });
}

int bmg_nccl_unique_id(unsigned char* id128) {
  return guard([&] { nccl_unique_id(id128); });
}

}  // extern "C"

