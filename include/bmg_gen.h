/* bmg_gen.h -- C ABI of the synthetic BASELINE problem generator
 * (bmggen/libbmggen.so; BASELINE.json configs).
 *
 * Input data, not the solver: the reference builds its systems with the PUM
 * discretiser (out of scope); these seeded block-stencil systems
 * and prolongations stand in for them.  Both benchmark arms and the tests use
 * the same library, so the oracle and the device see identical bytes.
 * Status codes as in bmg_cuda.h (0 ok, 1 invalid argument, 4 runtime error);
 * message from bmg_gen_last_error(). */
#pragma once
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* bmg_gen_last_error(void);
/* S_p = L_D^p block stencil on an n^dim patch grid (dim 2 or 3), blocks
 * A_ij = S_ij C (+ reg D_i on the diagonal); block rows [row_lo, row_hi)
 * (row_hi < 0: all) with global column indices.  Two calls: arrays NULL to
 * query nnzb, then filled. */
int bmg_gen_stencil(int dim, int n, int power, int m, uint64_t seed, double reg, int64_t row_lo,
                    int64_t row_hi, int64_t* nnzb, int64_t* row_ptr, int32_t* col_idx, double* vals);
/* prolongation from an (n/2)^dim coarse grid to the n^dim fine grid, rows as above */
int bmg_gen_prolongation(int dim, int n_fine, int m, uint64_t seed, int level, int64_t row_lo,
                         int64_t row_hi, int64_t* nnzb, int64_t* row_ptr, int32_t* col_idx,
                         double* vals);
/* N(0,1) vector (Box-Muller on the counter RNG), stream `tag` */
int bmg_gen_normal(uint64_t seed, uint64_t tag, int64_t n, double* out);

#ifdef __cplusplus
}

namespace bmg {
int64_t gen_stencil(int dim, int n, int power, int m, uint64_t seed, double reg, int64_t row_lo,
                    int64_t row_hi, int64_t* row_ptr, int32_t* col_idx, double* vals);
int64_t gen_prolongation(int dim, int n_fine, int m, uint64_t seed, int level, int64_t row_lo, int64_t row_hi,
                         int64_t* row_ptr, int32_t* col_idx, double* vals);
void gen_normal(uint64_t seed, uint64_t tag, int64_t n, double* out);
}  // namespace bmg
#endif
