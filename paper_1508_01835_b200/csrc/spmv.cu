#include "common.cuh"
#include "spmv.cuh"

namespace ifmm {
namespace {

__global__ void __launch_bounds__(256)
spmv_kernel(const SpmvRow* __restrict__ rows, int nrows, const SpmvTerm* __restrict__ terms,
            int nrhs, int ldv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
    const SpmvRow R = rows[r];
    for (int i = warp; i < R.h; i += nw) {
      for (int c = 0; c < nrhs; ++c) {
        double acc = R.accumulate ? R.out[(size_t)i * ldv + c] : 0.0;
        for (int t = R.t0; t < R.t0 + R.nt; ++t) {
          const SpmvTerm T = terms[t];
          double s = 0.0;
          if (!T.trans) {
            const double* b = T.B + (size_t)i * T.ld;
            for (int j = lane; j < T.cols; j += 32) s = fma(b[j], T.in[(size_t)j * ldv + c], s);
          } else {
            for (int j = lane; j < T.rows; j += 32)
              s = fma(T.B[(size_t)j * T.ld + i], T.in[(size_t)j * ldv + c], s);
          }
          acc += warp_sum(s);
        }
        if (lane == 0) R.out[(size_t)i * ldv + c] = acc;
      }
    }
  }
}

}  // namespace

void launch_spmv(const SpmvRow* rows, int nrows, const SpmvTerm* terms, int nrhs, int ldv,
                 cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_spmv"};
  if (nrows <= 0) return;
  spmv_kernel<<<nrows < 65535 ? nrows : 65535, 256, 0, s>>>(rows, nrows, terms, nrhs, ldv);
}

}  // namespace ifmm
