// partition.cpp -- host planning for the row-partitioned (multi-GPU) V-cycle.
//
// The fine levels are split into contiguous block-row ranges (strips in 2-D,
// slabs in 3-D).  A rank's vectors on a level live in one
// contiguous window of global block rows, own rows plus halo, so a local column
// index is `global - window_lo` and every halo exchange is a contiguous slice.
// Agglomerated (coarsest) levels give every row to rank 0; rank 0's window on the
// level above then covers the whole level (the gather) and the other ranks'
// windows on the agglomerated level cover what their prolongation rows read
// (the scatter).  Pure integer work; exported for the CPU tests.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <vector>

#include "bmg_abi.h"
#include "bmg_internal.h"

namespace bmg {

// Balanced contiguous ranges by blocks (+ rows), boundaries on multiples of
// `granule` rows.  bounds has world + 1 entries.
void partition_rows(int nbr, const int64_t* row_ptr, int world, int granule, bool agglomerate,
                    int32_t* bounds) {
  if (world < 1) fail(BMG_EINVAL, "partition: world must be >= 1");
  if (granule < 1) granule = 1;
  bounds[0] = 0;
  if (agglomerate || world == 1) {
    for (int r = 1; r <= world; ++r) bounds[r] = nbr;
    return;
  }
  const int ngran = (nbr + granule - 1) / granule;
  // work per granule: blocks plus one unit per row (vector traffic)
  std::vector<double> pre(ngran + 1, 0.0);
  for (int g = 0; g < ngran; ++g) {
    const int r0 = g * granule, r1 = std::min(nbr, r0 + granule);
    pre[g + 1] = pre[g] + (double)(row_ptr[r1] - row_ptr[r0]) + 0.05 * (r1 - r0);
  }
  int g = 0;
  for (int r = 1; r < world; ++r) {
    const double target = pre[ngran] * r / world;
    while (g < ngran && pre[g + 1] <= target) ++g;
    // pick the closer boundary
    int cut = g;
    if (g < ngran && (target - pre[g]) > (pre[g + 1] - target)) cut = g + 1;
    cut = std::max(cut, (int)((bounds[r - 1] + granule - 1) / granule));
    bounds[r] = std::min(nbr, cut * granule);
  }
  bounds[world] = nbr;
}

// Hull of the columns referenced by rows [lo, hi), joined with [clo, chi) when
// that range is non-empty (the rank's own rows of the column level).
void row_window(const int64_t* row_ptr, const int32_t* col, int lo, int hi, int clo, int chi,
                int32_t* ext_lo, int32_t* ext_hi) {
  long a = INT32_MAX, b = INT32_MIN;
  if (clo < chi) {
    a = clo;
    b = chi;
  }
  for (int i = lo; i < hi; ++i) {
    const int64_t p0 = row_ptr[i], p1 = row_ptr[i + 1];
    if (p1 > p0) {  // columns ascending within a row
      a = std::min<long>(a, col[p0]);
      b = std::max<long>(b, (long)col[p1 - 1] + 1);
    }
  }
  if (a > b) a = b = 0;
  *ext_lo = (int32_t)a;
  *ext_hi = (int32_t)b;
}

}  // namespace bmg

extern "C" {

int bmg_partition_rows(int nbr, const int64_t* row_ptr, int world, int granule, int agglomerate,
                       int32_t* bounds) {
  return bmg::guard([&] { bmg::partition_rows(nbr, row_ptr, world, granule, agglomerate != 0, bounds); });
}

int bmg_row_window(const int64_t* row_ptr, const int32_t* col, int lo, int hi, int clo, int chi,
                   int32_t* ext_lo, int32_t* ext_hi) {
  return bmg::guard([&] { bmg::row_window(row_ptr, col, lo, hi, clo, chi, ext_lo, ext_hi); });
}

}  // extern "C"
