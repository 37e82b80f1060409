// H2 setup kernels (sm_100a, fp64): Chebyshev interpolation matrices and
// fused kernel-evaluation blocks (P2P near field, grid-grid M2L tiles).
//
// Restates h2.py:29-67 (cheb_nodes / cheb_interp_1d / _grid /
// _interp_matrix) and the plugin Kernel.block contract (kernels.py:22-39)
// for the kernel families of the BASELINE configs.
#include "common.cuh"
#include "h2_kernels.h"

namespace ifmm {

__device__ __forceinline__ double kernel_value(const KernelSpec& k, double r) {
  switch (k.kind) {
    case KERNEL_EXP:
      return exp(-r);
    case KERNEL_IMQ:
      return 1.0 / sqrt(r * r + k.p0 * k.p0);
    case KERNEL_BENCH: {
      const double d = k.p0;
      if (r == 0.0) return 1.0;
      return r < d ? r / d : d / r;
    }
    case KERNEL_ZERO:
      return 0.0;
    default:
      return 0.0;
  }
}

// scipy cdist 'euclidean': sqrt of the ordered sum of squared differences
__device__ __forceinline__ double euclid(double ax, double ay, double az, double bx, double by,
                                         double bz) {
  const double dx = ax - bx, dy = ay - by, dz = az - bz;
  double s = __dmul_rn(dx, dx);
  s = __dadd_rn(s, __dmul_rn(dy, dy));
  s = __dadd_rn(s, __dmul_rn(dz, dz));
  return sqrt(s);
}

// Rotne-Prager-Yamakawa mobility block f(r) I + g(r) rhat rhat^T
// (kernels.py:59-91): far field r > 2a, overlap r <= 2a, self r = 0.
// d = P_i - Q_j; writes the row-major 3 x 3 block into B.
__device__ __forceinline__ void rpy_block(const KernelSpec& k, double dx, double dy, double dz,
                                          double (&B)[9]) {
  const double a = k.p0, c0 = k.p1;
  const double r = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
  const double rs = r == 0.0 ? 1.0 : r;
  double f, g;
  if (r > 2.0 * a) {
    const double a3 = a * a * a, r3 = rs * rs * rs;
    f = c0 * (3.0 * a / (4.0 * rs) + a3 / (2.0 * r3));
    g = c0 * (3.0 * a / (4.0 * rs) - 3.0 * a3 / (2.0 * r3));
  } else {
    f = c0 * (1.0 - 9.0 * r / (32.0 * a));
    g = c0 * (3.0 * r / (32.0 * a));
  }
  if (r == 0.0) g = 0.0;
  const double h[3] = {dx / rs, dy / rs, dz / rs};
#pragma unroll
  for (int p = 0; p < 3; ++p)
#pragma unroll
    for (int q = 0; q < 3; ++q) B[3 * p + q] = (p == q ? f : 0.0) + g * (h[p] * h[q]);
}

namespace {

// One CTA per block: the source points Q are staged once in shared memory
// (structure of arrays, chunks of EV_QC points); a warp owns a target row i
// (P_i in registers) and its lanes sweep the columns, so the row's stores are
// one coalesced 256-byte segment per 32 columns and there is no per-element
// integer division.  HBM-bound: 8 B written per entry.
constexpr int EV_QC = 512;
__global__ void __launch_bounds__(256)
eval_blocks_kernel(const EvalDesc* __restrict__ descs, int n, KernelSpec k) {
  __shared__ double qx[EV_QC], qy[EV_QC], qz[EV_QC];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const EvalDesc d = descs[b];
    for (int j0 = 0; j0 < d.n; j0 += EV_QC) {
      const int nj = d.n - j0 < EV_QC ? d.n - j0 : EV_QC;
      __syncthreads();
      for (int j = threadIdx.x; j < nj; j += blockDim.x) {
        const double* q = d.Q + 3 * (size_t)(j0 + j);
        qx[j] = q[0]; qy[j] = q[1]; qz[j] = q[2];
      }
      __syncthreads();
      for (int i = warp; i < d.m; i += nw) {
        const double* p = d.P + 3 * (size_t)i;
        const double px = p[0], py = p[1], pz = p[2];
        if (k.kind == KERNEL_RPY) {
          double* o = d.out + (size_t)(3 * i) * d.ldo + 3 * j0;
          for (int j = lane; j < nj; j += 32) {
            double B[9];
            rpy_block(k, px - qx[j], py - qy[j], pz - qz[j], B);
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int c = 0; c < 3; ++c) o[(size_t)a * d.ldo + 3 * j + c] = B[3 * a + c];
          }
          continue;
        }
        double* o = d.out + (size_t)i * d.ldo + j0;
        for (int j = lane; j < nj; j += 32)
          o[j] = kernel_value(k, euclid(px, py, pz, qx[j], qy[j], qz[j]));
      }
    }
  }
}

// 1D Chebyshev interpolation weights S_n(t, x_m) (h2.py:34-49)
__device__ void cheb_row(double t, int nc, double* S) {
  const double pi = 3.141592653589793;
  t = fmin(fmax(t, -1.0), 1.0);
  const double tt = acos(t);
  for (int m = 0; m < nc; ++m) {
    const double xm = cos((2.0 * m + 1.0) * pi / (2.0 * nc));
    const double tx = acos(xm);
    double acc = 0.0;
    for (int kk = 1; kk < nc; ++kk) acc += cos(tt * kk) * cos(tx * kk);
    S[m] = 1.0 / nc + (2.0 / nc) * acc;
  }
}

__global__ void interp_kernel(const InterpDesc* __restrict__ descs, int n, int nc) {
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const InterpDesc d = descs[b];
    const int g3 = nc * nc * nc;
    for (int p = threadIdx.x; p < d.count; p += blockDim.x) {
      const double* pt = d.pts + 3 * (size_t)p;
      double Sx[MAX_CHEB], Sy[MAX_CHEB], Sz[MAX_CHEB];
      cheb_row((pt[0] - d.cx) / d.hw, nc, Sx);
      cheb_row((pt[1] - d.cy) / d.hw, nc, Sy);
      cheb_row((pt[2] - d.cz) / d.hw, nc, Sz);
      double* o = d.out + (size_t)p * d.ldo;
      for (int i = 0; i < nc; ++i)
        for (int j = 0; j < nc; ++j) {
          const double sxy = Sx[i] * Sy[j];
          for (int kk = 0; kk < nc; ++kk) o[(i * nc + j) * nc + kk] = sxy * Sz[kk];
        }
      (void)g3;
    }
  }
}

__global__ void grid_kernel(const GridDesc* __restrict__ descs, int n, int nc) {
  const double pi = 3.141592653589793;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const GridDesc d = descs[b];
    const int g3 = nc * nc * nc;
    for (int e = threadIdx.x; e < g3; e += blockDim.x) {
      const int i = e / (nc * nc), j = (e / nc) % nc, kk = e % nc;
      const double xi = cos((2.0 * i + 1.0) * pi / (2.0 * nc));
      const double xj = cos((2.0 * j + 1.0) * pi / (2.0 * nc));
      const double xk = cos((2.0 * kk + 1.0) * pi / (2.0 * nc));
      d.out[3 * e + 0] = d.cx + d.hw * xi;
      d.out[3 * e + 1] = d.cy + d.hw * xj;
      d.out[3 * e + 2] = d.cz + d.hw * xk;
    }
  }
}

}  // namespace

void launch_eval(const EvalDesc* d_descs, int n, const KernelSpec& k, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_eval"};
  if (n <= 0) return;
  eval_blocks_kernel<<<n < 16384 ? n : 16384, 256, 0, s>>>(d_descs, n, k);
}

void launch_interp(const InterpDesc* d_descs, int n, int nc, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_interp"};
  if (n <= 0) return;
  interp_kernel<<<n < 16384 ? n : 16384, 64, 0, s>>>(d_descs, n, nc);
}

void launch_grid(const GridDesc* d_descs, int n, int nc, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_grid"};
  if (n <= 0) return;
  grid_kernel<<<n < 16384 ? n : 16384, 128, 0, s>>>(d_descs, n, nc);
}

}  // namespace ifmm

// ============================================================================
// Exact dense matvec y = A x, A_ij = K(|p_i - p_j|), evaluated on the fly
// (no storage, replaces dense.dense_matrix in
// experiments._matvec_oracle).  One thread per row, columns staged through
// shared memory in tiles; each row sums in a fixed order (deterministic).
// ============================================================================
namespace ifmm {
namespace {
constexpr int EM_TILE = 256;
__global__ void __launch_bounds__(256)
exact_matvec_kernel(const double* __restrict__ pts, const double* __restrict__ x, int n,
                    KernelSpec k, double* __restrict__ y) {
  __shared__ double sp[EM_TILE * 3];
  __shared__ double sx[EM_TILE * 3];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double px = 0, py = 0, pz = 0;
  if (i < n) { px = pts[3 * i]; py = pts[3 * i + 1]; pz = pts[3 * i + 2]; }
  const int bd = k.bd();
  double acc = 0.0, acc1 = 0.0, acc2 = 0.0;
  for (int t0 = 0; t0 < n; t0 += EM_TILE) {
    const int cnt = min(EM_TILE, n - t0);
    for (int e = threadIdx.x; e < cnt; e += blockDim.x) {
      sp[3 * e] = pts[3 * (t0 + e)];
      sp[3 * e + 1] = pts[3 * (t0 + e) + 1];
      sp[3 * e + 2] = pts[3 * (t0 + e) + 2];
      for (int a = 0; a < bd; ++a) sx[bd * e + a] = x[(size_t)bd * (t0 + e) + a];
    }
    __syncthreads();
    if (i < n) {
      if (bd == 3) {
        for (int e = 0; e < cnt; ++e) {
          double B[9];
          rpy_block(k, px - sp[3 * e], py - sp[3 * e + 1], pz - sp[3 * e + 2], B);
          const double x0 = sx[3 * e], x1 = sx[3 * e + 1], x2 = sx[3 * e + 2];
          acc = fma(B[0], x0, fma(B[1], x1, fma(B[2], x2, acc)));
          acc1 = fma(B[3], x0, fma(B[4], x1, fma(B[5], x2, acc1)));
          acc2 = fma(B[6], x0, fma(B[7], x1, fma(B[8], x2, acc2)));
        }
      } else {
        for (int e = 0; e < cnt; ++e) {
          const double r = euclid(px, py, pz, sp[3 * e], sp[3 * e + 1], sp[3 * e + 2]);
          acc = fma(kernel_value(k, r), sx[e], acc);
        }
      }
    }
    __syncthreads();
  }
  if (i < n) {
    if (bd == 3) { y[3 * (size_t)i] = acc; y[3 * (size_t)i + 1] = acc1; y[3 * (size_t)i + 2] = acc2; }
    else y[i] = acc;
  }
}
}  // namespace

void launch_exact_matvec(const double* pts, const double* x, int n, const KernelSpec& k,
                         double* y, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_exact_matvec"};
  exact_matvec_kernel<<<(n + 255) / 256, 256, 0, s>>>(pts, x, n, k, y);
}
}  // namespace ifmm
