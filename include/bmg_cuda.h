/*
 * bmg_cuda.h -- C ABI of libbmgcuda.so, the B200 (sm_100a) implementation of
 * the multilevel V-cycle application path of arXiv 2509.06744 (`blockmg`).
 *
 * Each entry point replaces one piece of the reference's C++ hot-path API
 * (paths relative to /root/reference/proj); INTEGRATION.md shows the C++
 * facade (include/bmg/blockmg.hpp) and the ctypes binding that sit on top.
 *
 *   reference                                         C ABI here
 *   ------------------------------------------------  ---------------------------------
 *   BlockSparseMatrix (block_matrix.hpp:26-70)        bmg_bsr_create / _download
 *   spmv (kernels.hpp:15, kernels.cpp:39-47)          bmg_spmv
 *   spmv_transpose (kernels.hpp:19, kernels.cpp:56-64) bmg_spmv_t
 *   r = b - A x (chebyshev.hpp:55-56,61-62;
 *                multilevel.cpp:91-93)                bmg_residual
 *   galerkin_coarsen (multilevel.hpp:50,
 *                     multilevel.cpp:11-28)           bmg_galerkin
 *   build_fsai / adaptive_build / nested_build
 *     (fsai.hpp:25,50,68; fsai.cpp:72-253)            bmg_fsai_build
 *   NestedFsai::apply (fsai.hpp:62, fsai.cpp:200-217) bmg_fsai_apply   (M = G^T G)
 *   NestedFsai::apply_transformed (fsai.cpp:219-241)  bmg_fsai_apply_transformed
 *   cheb_fourth_apply (chebyshev.hpp:48-69)           bmg_cheb4_apply
 *   lanczos_lambda_max (multilevel.hpp:53-54,
 *                       multilevel.cpp:30-34,
 *                       lanczos.hpp:16-58)            bmg_lanczos_lambda_max
 *   setup (multilevel.hpp:59-60, multilevel.cpp:36-75) bmg_hier_setup
 *   v_cycle (multilevel.hpp:65, multilevel.cpp:77-103) bmg_vcycle / bmg_vcycle_host
 *   measure_rates loop (experiments.cpp:15-67)        bmg_solve (residual history)
 *   read_matrix / write_matrix / read_vector /
 *     write_vector (matrix_io.hpp:22-27)              bmg_io_*
 *
 * Conventions
 *   - Every entry returns BMG_OK (0) or a negative status; the message of the
 *     last failure on the calling thread is bmg_last_error(), and for
 *     BMG_ENOTSPD the failing 0-based pivot is bmg_last_pivot().  Status codes
 *     map 1:1 onto the reference's exception types (see below).
 *   - Host buffers are caller-owned, read or written synchronously before the
 *     call returns.  Device objects are owned by their handle.  A context and
 *     its objects are single-threaded unless externally synchronised (the
 *     reference's objects are immutable after setup).
 *   - Block values cross the ABI row-major, unpadded, in row_ptr/col_idx order
 *     (the reference's DenseBlock is row-major, types.hpp:9).  Column indices
 *     within a row must be strictly ascending (the reference's std::map order).
 *   - FP64 everywhere.  There is no CPU fallback: without a CUDA device every
 *     compute entry returns BMG_ECUDA.
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BMG_OK = 0,
  BMG_EINVAL = -1,   /* std::invalid_argument */
  BMG_ERANGE = -2,   /* std::out_of_range */
  BMG_ENOTSPD = -3,  /* bmg::NotPositiveDefinite{pivot} (small_cholesky.hpp:10-13) */
  BMG_ERUNTIME = -4, /* std::runtime_error (e.g. multilevel.cpp:72-73) */
  BMG_ECUDA = -5,    /* CUDA runtime / cuSOLVER failure or no device */
  BMG_ENCCL = -6,    /* NCCL failure (multi-GPU contexts) */
  BMG_EIO = -7,      /* bmg::IoError{line} (matrix_io.hpp:10-13); pivot slot = line */
};

/* bmg_bsr_create flags */
enum {
  BMG_SYMMETRIC = 1, /* validation contract, as BlockSparseMatrix::symmetric() */
};

/* bmg_fsai_build kinds */
enum {
  BMG_FSAI_STATIC_LOWER = 0, /* build_fsai(A, LowerPattern::from_matrix(A)) */
  BMG_FSAI_DIAGONAL = 1,     /* build_fsai(A, LowerPattern::diagonal(n))   */
  BMG_FSAI_ADAPTIVE = 3,     /* nested_build(A, t_max, tau, nest)          */
};

typedef struct bmg_ctx bmg_ctx;
typedef struct bmg_bsr bmg_bsr;
typedef struct bmg_vec bmg_vec;
typedef struct bmg_fsai bmg_fsai;
typedef struct bmg_hier bmg_hier;

/* SetupParams (multilevel.hpp:35-47) */
typedef struct bmg_setup_params {
  int t_max;          /* 4 in the reference; 1 for the BASELINE configs */
  double tau;         /* 1.0 */
  int nest;           /* 0 */
  int fsai_kind;      /* BMG_FSAI_ADAPTIVE (reference setup) or BMG_FSAI_STATIC_LOWER */
  int lanczos_iters;  /* 100 */
  double lanczos_safety; /* 1.01 */
  uint64_t seed;      /* 42 */
  int coarse_dim_cap; /* 5000 */
  int smoother_kind;  /* 0 Richardson, 1 first kind, 2 fourth kind (default) */
  double richardson_omega;    /* 1.0 */
  double first_kind_fraction; /* 1/30: first kind covers [fraction * beta, beta] */
} bmg_setup_params;

const char* bmg_last_error(void);
int bmg_last_pivot(void);
const char* bmg_version(void);
void bmg_setup_params_default(bmg_setup_params* p);

/* ---- context ---------------------------------------------------------- */
int bmg_ctx_create(int device, bmg_ctx** out);
int bmg_ctx_destroy(bmg_ctx* ctx);
/* launch on an external stream (e.g. torch's current stream); NULL = own */
int bmg_ctx_set_stream(bmg_ctx* ctx, void* cuda_stream);
int bmg_ctx_sync(bmg_ctx* ctx);
/* kernels launched by this context since creation (all are libbmgcuda's own) */
int64_t bmg_ctx_launch_count(const bmg_ctx* ctx);

/* ---- block-sparse matrices --------------------------------------------- */
int bmg_bsr_create(bmg_ctx* ctx, int nbr, const int32_t* row_sizes, int nbc,
                   const int32_t* col_sizes, const int64_t* row_ptr, const int32_t* col_idx,
                   const double* vals, int flags, bmg_bsr** out);
int bmg_bsr_destroy(bmg_bsr* a);
/* device bytes held (values + indices + plan) and algorithmic bytes of one
 * streaming pass (nnzb * (8 m_r m_c + 4)) */
int bmg_bsr_info(const bmg_bsr* a, int* nbr, int* nbc, int64_t* nnzb, int* dim_r, int* dim_c,
                 int64_t* device_bytes, int64_t* pass_bytes);
/* symmetric-half streaming (hierarchy setup builds it for every smoothed level's A
 * that is exactly symmetric and keeps it where it measured faster): whether the
 * residual / spmv passes of `a` run on the lower triangle (bitwise the same
 * results), the algorithmic bytes of one such pass, and the measured pass times
 * (ms) of both forms (0 when not measured) */
int bmg_bsr_sym_info(const bmg_bsr* a, int* half, int64_t* pass_bytes, double* half_ms, double* full_ms);
int bmg_bsr_download(const bmg_bsr* a, int64_t* row_ptr, int32_t* col_idx, double* vals);
/* device-built transpose (values transposed per block) */
int bmg_bsr_transpose(const bmg_bsr* a, bmg_bsr** out);

/* ---- vectors ------------------------------------------------------------ */
int bmg_vec_create(bmg_ctx* ctx, int64_t n, bmg_vec** out);
int bmg_vec_destroy(bmg_vec* v);
int bmg_vec_upload(bmg_vec* v, const double* host);
int bmg_vec_download(const bmg_vec* v, double* host);
int bmg_vec_fill(bmg_vec* v, double value);
/* a zero vector of v's length on v's context */
int bmg_vec_create_like(const bmg_vec* v, bmg_vec** out);
/* dst = src (device to device, same context and length) */
int bmg_vec_copy(const bmg_vec* src, bmg_vec* dst);
/* z = alpha x + beta y, products and sum rounded separately (no fma): the
 * reference's vector expressions r = b - t, p = mu*mu*p + t, x += d*mu*p
 * (chebyshev.hpp:55-66) for the generic-operator cheb_fourth_apply of the C++
 * facade; z may alias x or y */
int bmg_vec_axpby(double alpha, const bmg_vec* x, double beta, const bmg_vec* y, bmg_vec* z);
void* bmg_vec_device_ptr(bmg_vec* v);
int64_t bmg_vec_size(const bmg_vec* v);

/* ---- kernels (kernels.cpp) --------------------------------------------- */
int bmg_spmv(const bmg_bsr* a, const bmg_vec* x, bmg_vec* y);
/* Y = A X for nrhs (1, 2, 4, 8) right-hand sides interleaved per scalar row
 * (x[j*nrhs + v]); each column bitwise equal to bmg_spmv */
int bmg_spmv_batch(const bmg_bsr* a, int nrhs, const bmg_vec* x, bmg_vec* y);
int bmg_spmv_t(const bmg_bsr* a, const bmg_vec* x, bmg_vec* y);
int bmg_residual(const bmg_bsr* a, const bmg_vec* b, const bmg_vec* x, bmg_vec* r);
int bmg_dot(const bmg_vec* a, const bmg_vec* b, double* out);
int bmg_galerkin(const bmg_bsr* a, const bmg_bsr* p, bmg_bsr** out);
/* F A F^T, exactly symmetric, exact-zero blocks dropped (kernels.hpp:29) */
int bmg_triple_product(const bmg_bsr* f, const bmg_bsr* a, bmg_bsr** out);

/* ---- block-FSAI (fsai.cpp) ---------------------------------------------- */
int bmg_fsai_build(const bmg_bsr* a, int kind, int t_max, double tau, int nest, bmg_fsai** out);
/* build_fsai(A, p) (fsai.hpp:25) for a caller's LowerPattern p: pat_ptr[n+1] /
 * pat_col list each row's lower block columns (duplicates and the diagonal, always
 * present, are ignored; j > i is BMG_EINVAL) */
int bmg_fsai_build_pattern(const bmg_bsr* a, const int64_t* pat_ptr, const int32_t* pat_col, bmg_fsai** out);
/* inject reference-built factors of a one-factor chain: F (unit-diagonal
 * lower BSR) and the row-major Cholesky factors of S-hat packed per block row */
int bmg_fsai_from_factors(bmg_ctx* ctx, const bmg_bsr* F, const double* shat_l_packed,
                          bmg_fsai** out);
int bmg_fsai_destroy(bmg_fsai* m);
int bmg_fsai_apply(const bmg_fsai* m, const bmg_vec* r, bmg_vec* z);
int bmg_fsai_apply_transformed(const bmg_fsai* m, const bmg_bsr* a, const bmg_vec* x,
                               bmg_vec* y);
/* borrowed handle of the device factor G (M = G^T G; the last factor of a chain) */
int bmg_fsai_G(const bmg_fsai* m, const bmg_bsr** g);
/* chain length and borrowed factor k: F_k for k < last, G = L-hat^{-1} F_last */
int bmg_fsai_chain_len(const bmg_fsai* m);
int bmg_fsai_factor(const bmg_fsai* m, int k, const bmg_bsr** f);

/* ---- smoother / spectral bound ------------------------------------------ */
int bmg_cheb4_apply(const bmg_bsr* a, const bmg_fsai* m, const bmg_vec* b, bmg_vec* x,
                    double beta, int k);
/* apply_smoother (chebyshev.hpp:117-129): kind 0 Richardson (omega), 1 first kind
 * on [alpha, beta], 2 fourth kind (beta); x updated in place */
int bmg_smoother_apply(const bmg_bsr* a, const bmg_fsai* m, int kind, double alpha, double beta,
                       double omega, int k, const bmg_vec* b, bmg_vec* x);
int bmg_lanczos_lambda_max(const bmg_bsr* a, const bmg_fsai* m, int iters, double safety,
                           uint64_t seed, double* beta);

/* ---- multilevel --------------------------------------------------------- */
/* transfers[l-1] prolongates level l-1 to level l (multilevel.hpp:56-60) */
int bmg_hier_setup(const bmg_bsr* a_finest, int ntransfers, const bmg_bsr* const* transfers,
                   const bmg_setup_params* params, bmg_hier** out);
/* inject a hierarchy built elsewhere (apply-phase parity):
 * A[0..L-1] (level 0 coarsest), P[1..L-1] (P[0] ignored), M[1..L-1], beta[1..L-1] */
int bmg_hier_create(bmg_ctx* ctx, int nlevels, const bmg_bsr* const* A, const bmg_bsr* const* P,
                    const bmg_fsai* const* M, const double* beta, int coarse_dim_cap,
                    bmg_hier** out);
int bmg_hier_destroy(bmg_hier* h);
int bmg_hier_info(const bmg_hier* h, int* nlevels, int64_t* device_bytes);
int bmg_hier_beta(const bmg_hier* h, int level, double* beta);
/* the level's SmootherSpec (Level::smoother, multilevel.hpp:25) */
int bmg_hier_set_smoother(bmg_hier* h, int level, int kind, double alpha, double beta, double omega);
int bmg_hier_level(const bmg_hier* h, int level, const bmg_bsr** a, const bmg_bsr** p,
                   const bmg_fsai** m);
/* algorithmic HBM bytes of one V(k_pre,k_post) cycle on the finest level */
int bmg_hier_cycle_bytes(const bmg_hier* h, int k_pre, int k_post, int64_t* bytes);
int bmg_hier_cycle_bytes_batch(const bmg_hier* h, int k_pre, int k_post, int nrhs, int64_t* bytes);
/* the same cycle with every A pass counted at full storage (both halves, as the
 * reference stores them) -- the byte model of the reference's own algorithm */
int bmg_hier_cycle_bytes_ref(const bmg_hier* h, int k_pre, int k_post, int64_t* bytes);
/* 1 (default) = replay each cycle from a captured CUDA graph */
int bmg_hier_use_graph(bmg_hier* h, int on);
int bmg_vcycle(bmg_hier* h, int k_pre, int k_post, const bmg_vec* b, bmg_vec* x);
/* v_cycle(h, spec, level, b, x) (multilevel.hpp:65) started on `level` (0 = the direct
 * coarse solve); b, x have that level's length; levels below the finest need an
 * unpartitioned hierarchy.  BMG_ERANGE for a level out of range. */
int bmg_vcycle_level(bmg_hier* h, int k_pre, int k_post, int level, const bmg_vec* b, bmg_vec* x);
/* end-to-end: host b, host x (in/out); H2D + cycle + D2H inside the call */
int bmg_vcycle_host(bmg_hier* h, int k_pre, int k_post, const double* b, double* x);
/* K right-hand sides in one cycle (K = 1, 2, 4, 8), interleaved per scalar row:
 * b[i*K + v], x[i*K + v].  The reference allows concurrent v_cycle calls on
 * distinct right-hand sides (SURVEY.md §8(b) Threading); batching them lets one
 * stream of every matrix serve all K.  Each right-hand side is bitwise the
 * single cycle.  Vectors hold n*K values (n = finest length for K = 1). */
int bmg_vcycle_batch(bmg_hier* h, int k_pre, int k_post, int nrhs, const bmg_vec* b, bmg_vec* x);
int bmg_vcycle_batch_host(bmg_hier* h, int k_pre, int k_post, int nrhs, const double* b, double* x);
int bmg_solve(bmg_hier* h, int k_pre, int k_post, const bmg_vec* b, bmg_vec* x, double tol,
              int max_iter, double* hist, int* iters, int* status);
/* measure_rates (experiments.cpp:15-67): initial error e_i =
 * CounterRng(seed).symmetric(i) normalised to unit M-norm, x = u_ref + e, V-cycles
 * on b; after each: squared M- and A-norms of x - u_ref and ||b - A x||.  Stops
 * when the squared M-norm < tol^2 (status 0), at max_iter (1), or on divergence
 * (2, blowup = iteration).  Histories hold max_iter + 1 entries; rates =
 * {rho_l2, rho_a, rho_r} (experiments.hpp:17-27).  Whole hierarchies. */
int bmg_measure_rates(bmg_hier* h, const bmg_bsr* mass, const bmg_vec* b, const bmg_vec* u_ref, int k_pre,
                      int k_post, uint64_t seed, double tol, int max_iter, double* l2_sq, double* energy_sq,
                      double* residual, int* iterations, int* status, int* blowup_iteration, double* rates);

/* ---- multi-GPU (row-partitioned V-cycle) ---------------
 * Every rank builds the same hierarchy (setup is deterministic), then keeps its
 * row strip of every level: contiguous block-row ranges balanced by blocks with
 * boundaries on multiples of granule[l] rows (a grid row in 2-D, a plane in
 * 3-D), the `agglomerate` coarsest levels on rank 0.  Halo exchanges are NCCL
 * send/recv of contiguous slices inside the captured V-cycle graph.  After the
 * partition bmg_vcycle / bmg_solve take this rank's own rows of b and x.
 * rank = -1 on a plain context emulates all `world` ranks in this process
 * (virtual ranks, device copies for the halos; b, x stay global): results are
 * bitwise equal to the unpartitioned cycle. */
int bmg_nccl_unique_id(unsigned char* id128);
int bmg_ctx_create_nccl(int device, int rank, int world, const unsigned char* id128, bmg_ctx** out);
/* Transport self-test (no reference counterpart; diagnostic): the halo-exchange
 * pattern of the partitioned V-cycle -- a grouped send + recv of `count` doubles on a
 * side stream forked from and joined to the context's stream, captured in a CUDA
 * graph where the transport allows it and replayed `reps` times -- with this rank as
 * its own peer, plus a sum all-reduce.  *mismatches = entries that did not arrive.
 * Lets one GPU drive the real NCCL point-to-point path (world = 1). */
int bmg_ctx_transport_selftest(bmg_ctx* ctx, int64_t count, int reps, int64_t* mismatches);
/* Loopback transport: `world` ranks as host threads of ONE process, each with
 * its own context on the same device; sends and receives are matched in-process
 * (host-side waits only).  Runs the exact NCCL code path where one GPU exists. */
typedef struct bmg_loopback bmg_loopback;
int bmg_loopback_create(int world, bmg_loopback** out);
int bmg_loopback_destroy(bmg_loopback* g);
int bmg_ctx_create_loopback(int device, bmg_loopback* g, int rank, bmg_ctx** out);
int bmg_hier_partition(bmg_hier* h, int world, int rank, const int32_t* granule, int agglomerate);
/* own rows [lo, hi) and vector window [wlo, whi) of `rank` on `level` */
int bmg_hier_part_info(const bmg_hier* h, int level, int rank, int32_t* lo, int32_t* hi, int32_t* wlo,
                       int32_t* whi);
/* ---- distributed setup (multilevel.cpp:36-75 on row strips) ------------
 * For systems that do not fit one GPU (BASELINE C3, C5): no rank ever holds a
 * whole partitioned level.  Levels >= agglomerate are split into equal
 * granule-aligned strips; each rank passes the plan's EXTENDED strip (own rows
 * +- halo granules, global column indices) of the finest A and of P_l for
 * l > agglomerate, and the whole P_l for l <= agglomerate.  radius[l] bounds
 * the granule distance A_l couples (checked); P must be a 2:1 granule
 * coarsening (checked).  The result is bitwise the hierarchy bmg_hier_setup +
 * bmg_hier_partition would build on one device (same beta, same cycles).
 * bmg_dist_plan: bounds[l*(world+1)+r], ext_lo/ext_hi[l*world+r], halo[l]
 * (granules); any output may be NULL.  No device needed. */
int bmg_dist_plan(int nlevels, const int32_t* nbr, const int32_t* granule, const int32_t* radius, int world,
                  int agglomerate, const bmg_setup_params* params, int32_t* bounds, int32_t* ext_lo,
                  int32_t* ext_hi, int32_t* halo);
/* this rank's share; world/rank from the NCCL context (plain context: world 1) */
int bmg_hier_setup_dist(bmg_ctx* ctx, int nlevels, const int32_t* granule, const int32_t* radius, int agglomerate,
                        const bmg_bsr* a_ext, const bmg_bsr* const* transfers, const bmg_setup_params* params,
                        bmg_hier** out);
/* every rank in this process: a_ext[r], transfers[r*(nlevels-1) + l-1] */
int bmg_hier_setup_dist_emulated(bmg_ctx* ctx, int world, int nlevels, const int32_t* granule,
                                 const int32_t* radius, int agglomerate, const bmg_bsr* const* a_ext,
                                 const bmg_bsr* const* transfers, const bmg_setup_params* params, bmg_hier** out);
/* host planning (no device needed): balanced contiguous row ranges; column hull */
int bmg_partition_rows(int nbr, const int64_t* row_ptr, int world, int granule, int agglomerate,
                       int32_t* bounds);
int bmg_row_window(const int64_t* row_ptr, const int32_t* col, int lo, int hi, int clo, int chi,
                   int32_t* ext_lo, int32_t* ext_hi);

/* ---- reference exchange format (matrix_io.hpp:15-27) --------------------
 * "%%block-matrix n n nnz" + 1-based scalar triplets, sidecar <path>.blocks
 * with one block size per line; vectors one value per line (17 digits). */
int bmg_io_read_matrix(bmg_ctx* ctx, const char* path, bmg_bsr** out, int* symmetric);
int bmg_io_write_matrix(const bmg_bsr* a, const char* path);
int bmg_io_read_vector(bmg_ctx* ctx, const char* path, bmg_vec** out);
int bmg_io_write_vector(const bmg_vec* v, const char* path);

/* ---- profiling helpers (bench.py) --------------------------------------- */
/* time `reps` back-to-back launches of the residual pass r = b - A x on the
 * context stream with CUDA events; returns the average ms per launch */
int bmg_time_residual(const bmg_bsr* a, const bmg_vec* b, const bmg_vec* x, bmg_vec* r, int reps,
                      double* ms);

/* symmetric tridiagonal eigenvalues (ascending), the host step of Lanczos */
int bmg_tridiag_eigs(int n, const double* d, const double* e, double* out);

/* the synthetic BASELINE input generator is a separate library: include/bmg_gen.h */

#ifdef __cplusplus
}
#endif
