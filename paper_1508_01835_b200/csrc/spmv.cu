#include "common.cuh"
#include "spmv.cuh"

namespace ifmm {
namespace {

// One CTA per output segment (SpmvRow).  Untransposed terms: a warp owns an
// output row i, its lanes sweep the block row (coalesced) with one partial sum
// per right-hand side in registers over ALL terms, then one warp reduction per
// right-hand side.  Transposed terms (out = B^T in): a thread owns output i and
// walks the block's rows, so consecutive threads read consecutive addresses
// and no reduction is needed.  Every block is read once for all nrhs columns.
template <int NR>
__global__ void __launch_bounds__(256)
spmv_kernel(const SpmvRow* __restrict__ rows, int nrows, const SpmvTerm* __restrict__ terms,
            int nrhs, int ldv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
    const SpmvRow R = rows[r];
    bool any_t = false;
    for (int t = R.t0; t < R.t0 + R.nt; ++t) any_t |= terms[t].trans != 0;
    for (int i = warp; i < R.h; i += nw) {
      double s[NR];
#pragma unroll
      for (int c = 0; c < NR; ++c) s[c] = 0.0;
      for (int t = R.t0; t < R.t0 + R.nt; ++t) {
        const SpmvTerm T = terms[t];
        if (T.trans) continue;
        const double* b = T.B + (size_t)i * T.ld;
        for (int j = lane; j < T.cols; j += 32) {
          const double bv = b[j];
          const double* in = T.in + (size_t)j * ldv;
#pragma unroll
          for (int c = 0; c < NR; ++c)
            if (c < nrhs) s[c] = fma(bv, in[c], s[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        if (c < nrhs) {
          const double v = warp_sum(s[c]);
          if (lane == 0) {
            double* o = R.out + (size_t)i * ldv + c;
            *o = R.accumulate ? *o + v : v;
          }
        }
      }
    }
    if (any_t) {
      __syncthreads();
      for (int i = threadIdx.x; i < R.h; i += blockDim.x) {
        double s[NR];
#pragma unroll
        for (int c = 0; c < NR; ++c) s[c] = 0.0;
        for (int t = R.t0; t < R.t0 + R.nt; ++t) {
          const SpmvTerm T = terms[t];
          if (!T.trans) continue;
          for (int j = 0; j < T.rows; ++j) {
            const double bv = T.B[(size_t)j * T.ld + i];
            const double* in = T.in + (size_t)j * ldv;
#pragma unroll
            for (int c = 0; c < NR; ++c)
              if (c < nrhs) s[c] = fma(bv, in[c], s[c]);
          }
        }
#pragma unroll
        for (int c = 0; c < NR; ++c)
          if (c < nrhs) R.out[(size_t)i * ldv + c] += s[c];
      }
    }
  }
}

// nrhs > 16: the same product on the column window [c0, c0 + nrhs)
__global__ void __launch_bounds__(256)
spmv_shift_kernel(const SpmvRow* __restrict__ rows, int nrows, const SpmvTerm* __restrict__ terms,
                  int nrhs, int ldv, int c0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = blockIdx.x; r < nrows; r += gridDim.x) {
    const SpmvRow R = rows[r];
    for (int i = warp; i < R.h; i += nw) {
      for (int c = c0; c < c0 + nrhs; ++c) {
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
  const int grid = nrows < 65535 ? nrows : 65535;
  if (nrhs == 1) {
    spmv_kernel<1><<<grid, 256, 0, s>>>(rows, nrows, terms, nrhs, ldv);
  } else if (nrhs <= 16) {
    spmv_kernel<16><<<grid, 256, 0, s>>>(rows, nrows, terms, nrhs, ldv);
  } else {  // column groups of 16: each group re-reads the blocks
    for (int c0 = 0; c0 < nrhs; c0 += 16)
      spmv_shift_kernel<<<grid, 256, 0, s>>>(rows, nrows, terms, nrhs - c0 < 16 ? nrhs - c0 : 16,
                                             ldv, c0);
  }
}

}  // namespace ifmm
