// Deterministic block-sparse matrix x (multi-)vector product.  One CTA per
// output segment; terms summed in list order, each dot product reduced by a
// fixed warp tree, so results are bitwise reproducible run to run.
#pragma once
#include <cuda_runtime.h>

namespace ifmm {

struct SpmvTerm {
  const double* B;  // row-major rows x cols, ld
  int rows, cols, ld, trans;  // trans: use B^T (cols x rows)
  const double* in;           // input segment (length = op cols) x nrhs
};
struct SpmvRow {
  double* out;  // output segment (length h) x nrhs
  int h;
  int t0, nt;   // terms [t0, t0+nt)
  int accumulate;
};

void launch_spmv(const SpmvRow* rows, int nrows, const SpmvTerm* terms, int nrhs, int ldv,
                 cudaStream_t s);

}  // namespace ifmm
