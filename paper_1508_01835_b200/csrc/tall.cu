// Orthonormalisation and sigma_max of a tall row-major n x w matrix (w <= 12)
// on the whole grid, for estimate_sigma0's range finder (graph.py:232-241,
// lowrank.py:74-76, 95-101: Y = E omega, Q = orth(Y), ... sigma_max(E^T Q)).
//
// n is the extended dimension (834k rows at c3, 3.7M at c4) and w = 11: the
// single-CTA Householder kernel of dense.cu took 0.2 s (c3) / 2.4 s (c4) per
// call, four calls per estimate.  Here: CholeskyQR2 -- Gram matrix by a
// two-stage fixed-order reduction (deterministic), an 11 x 11 Cholesky and
// inverse on one CTA, Q = Y R^-1 row by row -- twice; sigma_max(Y) =
// sqrt(lambda_max(Y^T Y)).  The orthonormal basis spans the same subspace as
// the reference's Householder Q, and the estimate only depends on the
// subspace.  A non-positive Cholesky pivot (columns dependent to working
// precision) raises *flag; the caller then repeats the estimate with the
// Householder kernel.
#include "common.cuh"
#include "dense.h"

namespace ifmm {
namespace {

constexpr int TW = 12;                   // largest supported width
constexpr int TNP = TW * (TW + 1) / 2;   // packed upper triangle
constexpr int TGRID = 592;               // 4 x 148 CTAs
constexpr int TBLK = 256;

IFMM_DEV int tri(int i, int j, int w) { return i * w - i * (i - 1) / 2 + (j - i); }  // i <= j

__global__ void __launch_bounds__(TBLK)
tall_gram_kernel(const double* __restrict__ Y, int n, int w, double* __restrict__ part) {
  __shared__ double red[TBLK / 32][TNP];
  const int np = w * (w + 1) / 2;
  double acc[TNP];
#pragma unroll
  for (int p = 0; p < TNP; ++p) acc[p] = 0.0;
  const long long r0 = (long long)n * blockIdx.x / gridDim.x, r1 = (long long)n * (blockIdx.x + 1) / gridDim.x;
  for (long long i = r0 + threadIdx.x; i < r1; i += TBLK) {
    double y[TW];
#pragma unroll
    for (int c = 0; c < TW; ++c) y[c] = c < w ? Y[(size_t)i * w + c] : 0.0;
    int p = 0;
#pragma unroll
    for (int a = 0; a < TW; ++a)
#pragma unroll
      for (int b = a; b < TW; ++b) {
        if (a < w && b < w) acc[p] = fma(y[a], y[b], acc[p]);
        ++p;
      }
  }
  // packed index of (a, b) in the TW-wide enumeration above -> the w-wide one
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int p = 0;
#pragma unroll
  for (int a = 0; a < TW; ++a)
#pragma unroll
    for (int b = a; b < TW; ++b) {
      if (a < w && b < w) {
        const double v = warp_sum(acc[p]);
        if (lane == 0) red[warp][tri(a, b, w)] = v;
      }
      ++p;
    }
  __syncthreads();
  for (int q = threadIdx.x; q < np; q += TBLK) {
    double s = 0.0;
    for (int wv = 0; wv < TBLK / 32; ++wv) s += red[wv][q];
    part[(size_t)blockIdx.x * TNP + q] = s;
  }
}

// mode 0: G = sum of the partial Grams, R = chol(G) (upper), rinv = R^-1.
// mode 1: out = sqrt(lambda_max(G)) by cyclic Jacobi on the w x w matrix.
__global__ void __launch_bounds__(128)
tall_small_kernel(const double* __restrict__ part, int nparts, int w, double* __restrict__ rinv,
                  int mode, double* __restrict__ out, int* __restrict__ flag) {
  __shared__ double G[TW][TW], R[TW][TW], X[TW][TW];
  const int np = w * (w + 1) / 2;
  for (int q = threadIdx.x; q < np; q += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(size_t)b * TNP + q];  // fixed order
    int i = 0, rem = q;
    while (rem >= w - i) { rem -= w - i; ++i; }
    G[i][i + rem] = s;
    G[i + rem][i] = s;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  if (mode == 0) {
    bool bad = false;
    for (int j = 0; j < w; ++j) {  // G = R^T R
      double d = G[j][j];
      for (int k = 0; k < j; ++k) d -= R[k][j] * R[k][j];
      if (!(d > 0.0)) { bad = true; d = 1.0; }
      const double rjj = sqrt(d);
      R[j][j] = rjj;
      for (int c = j + 1; c < w; ++c) {
        double s = G[j][c];
        for (int k = 0; k < j; ++k) s -= R[k][j] * R[k][c];
        R[j][c] = s / rjj;
      }
      for (int c = 0; c < j; ++c) R[j][c] = 0.0;
    }
    for (int c = 0; c < w; ++c) {  // X = R^-1 (upper), column c
      for (int i = w - 1; i >= 0; --i) {
        double s = i == c ? 1.0 : 0.0;
        for (int k = i + 1; k <= c; ++k) s -= R[i][k] * X[k][c];
        X[i][c] = i <= c ? s / R[i][i] : 0.0;
      }
    }
    for (int i = 0; i < w; ++i)
      for (int c = 0; c < w; ++c) rinv[i * w + c] = X[i][c];
    if (bad) *flag = 1;
    return;
  }
  // eigenvalues of the symmetric G by cyclic two-sided Jacobi
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0, dg = 0.0;
    for (int i = 0; i < w; ++i)
      for (int j = 0; j < w; ++j) (i == j ? dg : off) += G[i][j] * G[i][j];
    if (!(off > 1e-30 * dg)) break;
    for (int p = 0; p < w - 1; ++p)
      for (int q = p + 1; q < w; ++q) {
        const double apq = G[p][q];
        if (apq == 0.0) continue;
        const double th = (G[q][q] - G[p][p]) / (2.0 * apq);
        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < w; ++k) {
          const double gkp = G[k][p], gkq = G[k][q];
          G[k][p] = c * gkp - s * gkq;
          G[k][q] = s * gkp + c * gkq;
        }
        for (int k = 0; k < w; ++k) {
          const double gpk = G[p][k], gqk = G[q][k];
          G[p][k] = c * gpk - s * gqk;
          G[q][k] = s * gpk + c * gqk;
        }
      }
  }
  double lm = 0.0;
  for (int i = 0; i < w; ++i) lm = fmax(lm, G[i][i]);
  *out = sqrt(lm);
}

// Q[i][:] = Y[i][:] R^-1 (upper triangular); in place allowed (row by row)
__global__ void __launch_bounds__(TBLK)
tall_apply_kernel(const double* Y, int n, int w, const double* __restrict__ rinv, double* Q) {
  __shared__ double X[TW * TW];
  for (int e = threadIdx.x; e < w * w; e += TBLK) X[e] = rinv[e];
  __syncthreads();
  for (long long i = (long long)blockIdx.x * TBLK + threadIdx.x; i < n; i += (long long)gridDim.x * TBLK) {
    double y[TW], q[TW];
#pragma unroll
    for (int c = 0; c < TW; ++c) y[c] = c < w ? Y[(size_t)i * w + c] : 0.0;
#pragma unroll
    for (int c = 0; c < TW; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < TW; ++k)
        if (k <= c && c < w) s = fma(y[k], X[k * w + c], s);
      q[c] = s;
    }
#pragma unroll
    for (int c = 0; c < TW; ++c)
      if (c < w) Q[(size_t)i * w + c] = q[c];
  }
}

}  // namespace

bool tall_grid_supported(int w) { return w >= 1 && w <= TW; }

size_t tall_grid_work_doubles(int w) { return (size_t)TGRID * TNP + (size_t)w * w + 16; }

void launch_tall_orth_grid(const double* Y, int n, int w, double* Q, double* work, int* flag,
                           cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_tall_orth_grid"};
  double* part = work;
  double* rinv = work + (size_t)TGRID * TNP;
  const int grid = n < TGRID * TBLK ? (n + TBLK - 1) / TBLK : TGRID;
  const double* src = Y;
  for (int pass = 0; pass < 2; ++pass) {  // CholeskyQR2
    tall_gram_kernel<<<grid, TBLK, 0, s>>>(src, n, w, part);
    tall_small_kernel<<<1, 128, 0, s>>>(part, grid, w, rinv, 0, nullptr, flag);
    tall_apply_kernel<<<grid, TBLK, 0, s>>>(src, n, w, rinv, Q);
    src = Q;
  }
}

void launch_tall_sigmax_grid(const double* Y, int n, int w, double* out, double* work,
                             cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_tall_sigmax_grid"};
  const int grid = n < TGRID * TBLK ? (n + TBLK - 1) / TBLK : TGRID;
  tall_gram_kernel<<<grid, TBLK, 0, s>>>(Y, n, w, work);
  tall_small_kernel<<<1, 128, 0, s>>>(work, grid, w, nullptr, 1, out, nullptr);
}

}  // namespace ifmm
