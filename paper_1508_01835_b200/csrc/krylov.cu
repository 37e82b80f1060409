// Device Arnoldi pieces of the non-restarted GMRES (krylov.py:32-116):
// modified Gram-Schmidt against the resident basis V (one row per Krylov
// vector, fp64, row stride ldv), the normalisation V[k+1] = w / h, and the
// final combination u = sum_i y_i V[i].  The Givens rotations and the
// triangular solve stay on the host, as SURVEY A18 prescribes (O(k) scalars).
//
// HBM-bound: step k of MGS reads V[0..k] and w (k+1) times; each pass of
// the kernel below does "w -= h[i-1] V[i-1]; partial dot(V[i], w)", so
// each projection costs 3 reads + 1 write of n doubles (V[i-1] mostly from
// L2).  Reductions are deterministic (fixed grid, warp shuffles, fixed-order
// sums of the partials), so
// repeated runs are bitwise identical.  The elementwise updates use explicit
// _rn intrinsics (no FMA contraction) to round exactly like the reference's
// numpy expressions w - h*V[i], w / h and u + y_i*V[i].
#include <cooperative_groups.h>

#include "engine.h"

namespace cg = cooperative_groups;

namespace ifmm {
namespace {

constexpr int kThreads = 512;

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int j = 0; j < (int)(blockDim.x >> 5); ++j) s += red[j];
  return s;
}

// All k1+1 passes of one MGS call in one cooperative launch.  Pass i:
// (if i > 0) w -= h[i-1] * V[i-1]; block partial of a*c, (a, c) = (V[i], w),
// or (w, w) for the norm pass; grid barrier; every CTA adds the partials in
// the same fixed order, so all CTAs hold the identical h[i].  32 registers
// (launch bounds) keep 4 x 512-thread CTAs resident per SM.  Measured against
// a launch per pass + a one-CTA finish: n = 8.4M, k1 = 100: 4.47 vs 4.78 ms;
// n = 1M, k1 = 50: 0.36 vs 0.61 ms (profiles/r01e_gmres_mgs.md).  The
// partials are double-buffered: pass i+2 overwrites buffer i%2 only after
// barrier i+1, which every CTA reaches after reading it.
__global__ void __launch_bounds__(kThreads, 4) k_mgs_coop(const double* __restrict__ V, long long ldv,
                                                          int k1, long long n, double* __restrict__ w,
                                                          double* __restrict__ h,
                                                          double* __restrict__ part) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[kThreads / 32];
  __shared__ double hs;
  const int nb = gridDim.x;
  double hp = 0.0;
  for (int i = 0; i <= k1; ++i) {
    const int norm = (i == k1);
    const double* vp = (i > 0) ? V + (long long)(i - 1) * ldv : nullptr;
    const double* vi = norm ? nullptr : V + (long long)i * ldv;
    double acc = 0.0;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (long long)gridDim.x * blockDim.x) {
      double x = w[e];
      if (vp) {
        x = __dsub_rn(x, __dmul_rn(hp, vp[e]));
        w[e] = x;
      }
      acc = __fma_rn(norm ? x : vi[e], x, acc);
    }
    double* pb = part + (i & 1) * nb;
    const double s = block_sum(acc, red);
    if (threadIdx.x == 0) pb[blockIdx.x] = s;
    grid.sync();
    double t = 0.0;
    for (int j = threadIdx.x; j < nb; j += blockDim.x) t += __ldcg(pb + j);
    __syncthreads();  // red[] reuse
    const double tot = block_sum(t, red);
    if (threadIdx.x == 0) {
      hs = norm ? sqrt(tot) : tot;
      if (blockIdx.x == 0) h[i] = hs;
    }
    __syncthreads();
    hp = hs;
  }
}

__global__ void __launch_bounds__(kThreads, 4) k_div(const double* __restrict__ w, long long n, double hs,
                      double* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    out[e] = __ddiv_rn(w[e], hs);
}

// u[e] = (((0 + y0 V0) + y1 V1) + ...) in basis order, per element.
__global__ void k_combine(const double* __restrict__ V, long long ldv, int k,
                          const double* __restrict__ y, long long n, double* __restrict__ u) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < k; ++i) acc = __dadd_rn(acc, __dmul_rn(y[i], V[(long long)i * ldv + e]));
    u[e] = acc;
  }
}

int grid_for(Ctx& C, long long n) {
  const int sms = C.sm_count();
  long long want = (n + kThreads - 1) / kThreads;
  long long cap = 4LL * sms;  // 4 resident 512-thread CTAs per SM
  return (int)std::max(1LL, std::min(want, cap));
}

}  // namespace

void krylov_mgs(Ctx& C, const double* V, long long ldv, int k1, long long n, double* w,
                double* h_host) {
  const int nb = grid_for(C, n);
  Blk part = C.alloc(1, 2 * nb), h = C.alloc(1, k1 + 1);
  if (C.mgs_occ < 0)  // per context (= per device), not a process-wide static
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&C.mgs_occ, k_mgs_coop, kThreads, 0));
  const int g = std::min(nb, std::max(1, C.mgs_occ) * C.sm_count());
  void* args[] = {(void*)&V, (void*)&ldv, (void*)&k1, (void*)&n, (void*)&w, (void*)&h.p,
                  (void*)&part.p};
  CUDA_CHECK(cudaLaunchCooperativeKernel((void*)k_mgs_coop, dim3(g), dim3(kThreads), args, 0, C.st));
  CUDA_CHECK(cudaGetLastError());
  CUDA_CHECK(cudaMemcpyAsync(h_host, h.p, 8 * (size_t)(k1 + 1), cudaMemcpyDeviceToHost, C.st));
  C.sync();
  C.free(part);
  C.free(h);
  C.flush();
}

void krylov_div(Ctx& C, const double* w, long long n, double hs, double* out) {
  k_div<<<grid_for(C, n), kThreads, 0, C.st>>>(w, n, hs, out);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
}

void krylov_combine(Ctx& C, const double* V, long long ldv, int k, const double* y_host,
                    long long n, double* u) {
  Blk y = C.alloc(1, std::max(k, 1));
  CUDA_CHECK(cudaMemcpyAsync(y.p, y_host, 8 * (size_t)k, cudaMemcpyHostToDevice, C.st));
  k_combine<<<grid_for(C, n), kThreads, 0, C.st>>>(V, ldv, k, y.p, n, u);
  CUDA_CHECK(cudaGetLastError());
  C.sync();
  C.free(y);
  C.flush();
}

}  // namespace ifmm
