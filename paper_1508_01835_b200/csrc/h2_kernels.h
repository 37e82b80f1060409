#pragma once
#include <cuda_runtime.h>

namespace ifmm {

enum KernelKind { KERNEL_EXP = 1, KERNEL_IMQ = 2, KERNEL_BENCH = 3, KERNEL_ZERO = 4, KERNEL_RPY = 5 };
constexpr int KERNEL_KIND_MAX = 5;
constexpr int MAX_CHEB = 12;

struct KernelSpec {
  int kind;
  double p0;  // IMQ: h, BENCH: d, RPY: particle radius a
  double p1;  // RPY: c = 1 / (6 pi eta a)
  // block_dim of the plugin (kernels.py:33): rows / columns per point
  __host__ __device__ int bd() const { return kind == KERNEL_RPY ? 3 : 1; }
};

// out(i,j) = K(|P_i - Q_j|), P: m x 3, Q: n x 3 (row-major), out ld ldo; a
// block_dim-3 kernel writes the 3 x 3 block of (i, j) at rows 3i.., columns 3j..
// (point-major ordering, kernels.py:28)
struct EvalDesc {
  const double* P;
  const double* Q;
  int m, n;
  double* out;
  int ldo;
};

// out (count x nc^3, ld ldo) = interpolation matrix of pts in cell (c, hw)
struct InterpDesc {
  const double* pts;
  int count;
  double cx, cy, cz, hw;
  double* out;
  int ldo;
};

// out (nc^3 x 3) = Chebyshev grid of cell (c, hw)
struct GridDesc {
  double cx, cy, cz, hw;
  double* out;
};

void launch_eval(const EvalDesc* d_descs, int n, const KernelSpec& k, cudaStream_t s);
void launch_interp(const InterpDesc* d_descs, int n, int nc, cudaStream_t s);
void launch_grid(const GridDesc* d_descs, int n, int nc, cudaStream_t s);
// y = A x with A_ij = K(|p_i - p_j|) on the fly (pts n x 3 row-major; x, y of
// length n * block_dim)
void launch_exact_matvec(const double* pts, const double* x, int n, const KernelSpec& k,
                         double* y, cudaStream_t s);

}  // namespace ifmm
