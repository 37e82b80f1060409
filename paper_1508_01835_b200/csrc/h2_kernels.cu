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

namespace {

__global__ void eval_blocks_kernel(const EvalDesc* __restrict__ descs, int n, KernelSpec k) {
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const EvalDesc d = descs[b];
    const long long tot = (long long)d.m * d.n;
    for (long long e = threadIdx.x; e < tot; e += blockDim.x) {
      const int i = (int)(e / d.n), j = (int)(e % d.n);
      const double* p = d.P + 3 * (size_t)i;
      const double* q = d.Q + 3 * (size_t)j;
      const double r = euclid(p[0], p[1], p[2], q[0], q[1], q[2]);
      d.out[(size_t)i * d.ldo + j] = kernel_value(k, r);
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
  if (n <= 0) return;
  eval_blocks_kernel<<<n < 16384 ? n : 16384, 256, 0, s>>>(d_descs, n, k);
}

void launch_interp(const InterpDesc* d_descs, int n, int nc, cudaStream_t s) {
  if (n <= 0) return;
  interp_kernel<<<n < 16384 ? n : 16384, 64, 0, s>>>(d_descs, n, nc);
}

void launch_grid(const GridDesc* d_descs, int n, int nc, cudaStream_t s) {
  if (n <= 0) return;
  grid_kernel<<<n < 16384 ? n : 16384, 128, 0, s>>>(d_descs, n, nc);
}

}  // namespace ifmm
