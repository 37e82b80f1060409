// Batched small dense fp64 linear algebra for the IFMM elimination (sm_100a).
//
//  * grouped GEMM on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA),
//  * LU with partial pivoting (getrf semantics, factor.py:166-173) and
//    multi-RHS LU solves (factor.py:160-163),
//  * one-sided Jacobi SVD (truncated_svd, lowrank.py:54-61),
//  * full-pivot ACA + Householder QR-QR-SVD basis union
//    (aca_svd / weighted_basis_union, lowrank.py:128-199),
//  * strided block copy / accumulate (graph edge updates, merge tiling).
//
// Every routine is a CTA-cooperative device function over generic pointers
// (shared or global memory) wrapped by a batched kernel: one CTA per matrix,
// many matrices per launch.
#include "common.cuh"
#include "dense.h"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#include <cstdio>
#include <cstdlib>

namespace ifmm {

// per-phase cycle counters of the union kernel (diagnostics)
__device__ unsigned long long g_uprof[48];

__device__ __forceinline__ void cta_geqrf(double* A, int rows, int cols, int lda, double* tau, double* red);
__device__ __forceinline__ void cta_orgqr(const double* A, int rows, int cols, int lda, const double* tau,
                          double* Q, int ldq);

// ============================================================================
// Strided copy / accumulate
// ============================================================================

namespace {
__global__ void copy_kernel(const CopyDesc* __restrict__ descs, int n) {
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const CopyDesc d = descs[b];
    const long long tot = (long long)d.rows * d.cols;
    for (long long e = threadIdx.x; e < tot; e += blockDim.x) {
      const int i = (int)(e / d.cols), j = (int)(e % d.cols);
      double* o = d.dst + (size_t)i * d.ds_r + (size_t)j * d.ds_c;
      switch (d.mode) {
        case 0: *o = (d.rscale ? d.alpha * d.rscale[i] : d.alpha) * d.src[(size_t)i * d.ss_r + (size_t)j * d.ss_c]; break;
        case 1: *o += (d.rscale ? d.alpha * d.rscale[i] : d.alpha) * d.src[(size_t)i * d.ss_r + (size_t)j * d.ss_c]; break;
        case 2: *o = (i == j) ? d.alpha : 0.0; break;
        case 4: *o = d.alpha; break;
        default: *o = 0.0; break;
      }
    }
  }
}
}  // namespace

void launch_copy(const CopyDesc* d_descs, int n, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_copy"};
  if (n <= 0) return;
  copy_kernel<<<n < 4096 ? n : 4096, 256, 0, s>>>(d_descs, n);
}

// ============================================================================
// One-sided Jacobi SVD (Hestenes) -- CTA cooperative
// ============================================================================

// W: col-major rows x cols (ld ldw, rows >= cols); V: col-major cols x cols
// (ld cols) initialised here to I.  On exit W's columns are sigma_j u_j
// (unsorted) and V holds the accumulated rotations.
template <int T>
__device__ __forceinline__ double team_sum(double v) {
#pragma unroll
  for (int o = T / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One round-robin sweep pass with teams of T lanes per column pair.
template <int T>
__device__ __forceinline__ void jacobi_round(double* W, int rows, int cols, int ldw, double* V,
                                             int cp, int r, double tol_rot, double tol_conv,
                                             int* sflag) {
  const int tl = threadIdx.x & (T - 1);
  const int team = threadIdx.x / T, nteam = blockDim.x / T;
  const int first_team_of_warp = (threadIdx.x & ~31) / T;
  for (int pi0 = 0; pi0 < cp / 2; pi0 += nteam) {
    if (pi0 + first_team_of_warp >= cp / 2) break;  // whole warp idle this round
    const int pi = pi0 + team;
    int p = 0, q = cols;
    if (pi < cp / 2) {
      if (pi == 0) { p = r; q = cp - 1; }
      else { p = (r + pi) % (cp - 1); q = (r - pi + cp - 1) % (cp - 1); }
      if (p > q) { int t = p; p = q; q = t; }
    }
    const bool act = pi < cp / 2 && q < cols;
    double a = 0.0, b = 0.0, g = 0.0;
    double* x = W + (size_t)p * ldw;
    double* y = W + (size_t)(act ? q : p) * ldw;
    if (act)
      for (int i = tl; i < rows; i += T) {
        const double u = x[i], v = y[i];
        a = fma(u, u, a); b = fma(v, v, b); g = fma(u, v, g);
      }
    // all lanes of the warp take part in the shuffles (teams never straddle)
    a = team_sum<T>(a); b = team_sum<T>(b); g = team_sum<T>(g);
    if (!act) continue;
    const double ab = a * b, g2 = g * g;
    if (g != 0.0 && g2 > tol_rot * tol_rot * ab) {
      // t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)) with zeta = (b - a) / 2g, as
      // t = sign(d gg) |gg| / (|d| + sqrt(d^2 + gg^2)): one sqrt + one division,
      // full FP64 (an inexact t makes convergence linear instead of quadratic)
      const double d = b - a, gg = 2.0 * g;
      const double t = copysign(fabs(gg), d * gg) / (fabs(d) + hypot(d, gg));
      const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
      for (int i = tl; i < rows; i += T) {
        const double u = x[i], v = y[i];
        x[i] = c * u - s * v;
        y[i] = s * u + c * v;
      }
      double* vx = V + (size_t)p * cols;
      double* vy = V + (size_t)q * cols;
      for (int i = tl; i < cols; i += T) {
        const double u = vx[i], v = vy[i];
        vx[i] = c * u - s * v;
        vy[i] = s * u + c * v;
      }
      if (tl == 0 && g2 > tol_conv * tol_conv * ab) *sflag = 1;
    }
  }
}

// One-sided Jacobi (Hestenes), round-robin ordering.  Rotations are applied
// whenever a pair is not orthogonal to working precision; only rotations
// above the dot-product rounding level (rows * eps) keep the sweeps going.
__device__ __forceinline__ int cta_jacobi(double* W, int rows, int cols, int ldw, double* V, int* sflag) {
  for (int e = threadIdx.x; e < cols * cols; e += blockDim.x)
    V[e] = (e % (cols + 1) == 0) ? 1.0 : 0.0;
  const double tol_rot = kEps;
  const double tol_conv = fmax(kEps * (double)(rows > 4 ? rows : 4), 1e-13);
  const int cp = cols + (cols & 1);
  __syncthreads();
  if (cols < 2) return 0;
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    if (threadIdx.x == 0) *sflag = 0;
    __syncthreads();
    for (int r = 0; r < cp - 1; ++r) {
      if (rows <= 64) jacobi_round<8>(W, rows, cols, ldw, V, cp, r, tol_rot, tol_conv, sflag);
      else if (rows <= 192) jacobi_round<16>(W, rows, cols, ldw, V, cp, r, tol_rot, tol_conv, sflag);
      else jacobi_round<32>(W, rows, cols, ldw, V, cp, r, tol_rot, tol_conv, sflag);
      __syncthreads();
    }
    const int again = *sflag;
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&g_uprof[10], 1ull);
    if (!again) break;
  }
  return sweep + 1;
}

// Union-core Jacobi (one-sided, Hestenes, round-robin).  W (s x s, col-major,
// ld s) holds the matrix; V (s x s, ld s) accumulates the rotations (set to
// I here).  W and V may live in different memory spaces (V goes to global
// memory when 2 s^2 does not fit in shared memory).
//
// One sweep: s-1 (or s) rounds with one barrier each.  A team of T lanes
// handles one column pair per pass, holding its NE rows per lane of the W
// columns in registers between the dot products and the rotation; the
// pair schedule of pass 0 advances incrementally, later passes use the
// closed form.  Returns the per-thread "not yet converged" flag.
template <int T, int NE>
__device__ __forceinline__ bool jac_sweep(double* W, double* V, int s, int cp, double tr2, double tc2) {
  const int tl = threadIdx.x & (T - 1), team = threadIdx.x / T, nteam = blockDim.x / T;
  const int half = cp >> 1, m1 = cp - 1;
  const int first_team_of_warp = (threadIdx.x & ~31) / T;
  int p0 = team, q0 = team == 0 ? m1 : m1 - team;  // pass-0 pair, advanced each round
  bool again = false;
  for (int r = 0; r < m1; ++r) {
    for (int pi = team, pass = 0; pi - team + first_team_of_warp < half; pi += nteam, ++pass) {
      int p, q;
      if (pass == 0) { p = p0; q = q0; }
      else { p = (r + pi) % m1; q = (r - pi + m1) % m1; }
      const int lo = p < q ? p : q, hi = p < q ? q : p;
      const bool act = pi < half && hi < s;
      double* x = W + (size_t)(act ? lo : 0) * s;
      double* y = W + (size_t)(act ? hi : 0) * s;
      double xr[NE], yr[NE];
      double a = 0.0, b = 0.0, g = 0.0;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int i = tl + e * T;
        const bool in = act && i < s;
        xr[e] = in ? x[i] : 0.0;
        yr[e] = in ? y[i] : 0.0;
        a = fma(xr[e], xr[e], a); b = fma(yr[e], yr[e], b); g = fma(xr[e], yr[e], g);
      }
      if (act)  // rows beyond the register tile (s > NE T only)
        for (int i = tl + NE * T; i < s; i += T) {
          const double u = x[i], v = y[i];
          a = fma(u, u, a); b = fma(v, v, b); g = fma(u, v, g);
        }
      a = team_sum<T>(a); b = team_sum<T>(b); g = team_sum<T>(g);
      const double ab = a * b, g2 = g * g;
      if (act && g != 0.0 && g2 > tr2 * ab) {
        // t = tan(theta) = sign(d gg) |gg| / (|d| + sqrt(d^2 + gg^2)), d = b - a, gg = 2g
        const double d = b - a, gg = 2.0 * g;
        const double t = copysign(fabs(gg), d * gg) / (fabs(d) + sqrt(fma(d, d, gg * gg)));
        const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const int i = tl + e * T;
          if (i < s) {
            x[i] = fma(c, xr[e], -sn * yr[e]);
            y[i] = fma(sn, xr[e], c * yr[e]);
          }
        }
        for (int i = tl + NE * T; i < s; i += T) {
          const double u = x[i], v = y[i];
          x[i] = fma(c, u, -sn * v);
          y[i] = fma(sn, u, c * v);
        }
        // V columns in batches of 4 rows per lane, all loads before the
        // stores (a load after a possibly aliasing store would wait for it)
        double* vx = V + (size_t)lo * s;
        double* vy = V + (size_t)hi * s;
        for (int i0 = tl; i0 < s; i0 += 4 * T) {
          double u[4], v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = i0 + e * T;
            u[e] = i < s ? vx[i] : 0.0;
            v[e] = i < s ? vy[i] : 0.0;
          }
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = i0 + e * T;
            if (i < s) {
              vx[i] = fma(c, u[e], -sn * v[e]);
              vy[i] = fma(sn, u[e], c * v[e]);
            }
          }
        }
        again |= g2 > tc2 * ab;
      }
    }
    __syncthreads();
    if (team == 0) p0 = r + 1;
    else { p0 = p0 + 1 == m1 ? 0 : p0 + 1; q0 = q0 + 1 == m1 ? 0 : q0 + 1; }
  }
  return again;
}

// Returns the number of sweeps.  Rotations are applied whenever a pair is not
// orthogonal to working precision; only rotations above the dot-product
// rounding level (s * eps) keep the sweeps going.
__device__ __forceinline__ int cta_jacobi_wv(double* W, double* V, int s) {
  for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
    const int j = e / s, i = e - j * s;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  const double tol_rot = kEps;
  const double tol_conv = fmax(kEps * (double)(s > 4 ? s : 4), 1e-13);
  const double tr2 = tol_rot * tol_rot, tc2 = tol_conv * tol_conv;
  const int cp = s + (s & 1);
  __syncthreads();
  if (s < 2) return 0;
  // rows per lane NE <= 16 (xr, yr: 64 registers; union_svd_kernel has the
  // budget); rows beyond NE T (s > 256) are streamed from memory
  const int kind = s <= 32 ? 0 : s <= 64 ? 1 : s <= 128 ? 2 : 3;
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    bool ag;
    if (kind == 0) ag = jac_sweep<32, 1>(W, V, s, cp, tr2, tc2);
    else if (kind == 1) ag = jac_sweep<16, 4>(W, V, s, cp, tr2, tc2);
    else if (kind == 2) ag = jac_sweep<8, 16>(W, V, s, cp, tr2, tc2);
    else ag = jac_sweep<32, 8>(W, V, s, cp, tr2, tc2);  // + memory tail
    if (!__syncthreads_or(ag)) break;
  }
  return sweep + 1;
}

// Column norms -> sigma[j]; order[pos] = j sorted by sigma desc (ties: lower j).
__device__ __forceinline__ void cta_sv_order(const double* W, int rows, int cols, int ldw, double* sig, int* order) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < cols; j += nw) {
    double a = 0.0;
    for (int i = lane; i < rows; i += 32) { const double u = W[(size_t)j * ldw + i]; a = fma(u, u, a); }
    a = warp_sum(a);
    if (lane == 0) sig[j] = sqrt(a);
  }
  __syncthreads();
  // rank by value (NaN sorts last): a permutation even for non-finite input
  for (int j = threadIdx.x; j < cols; j += blockDim.x) {
    const double sj = isnan(sig[j]) ? -1.0 : sig[j];
    int pos = 0;
    for (int l = 0; l < cols; ++l) {
      const double sl = isnan(sig[l]) ? -1.0 : sig[l];
      pos += (sl > sj) || (sl == sj && l < j);
    }
    order[pos] = j;
  }
  __syncthreads();
}

__host__ __device__ size_t svd_work_doubles(int m, int n) {
  const int rows = m > n ? m : n, cols = m > n ? n : m;
  const size_t jac = (size_t)rows * cols + (size_t)cols * cols + 2 * (size_t)cols + 8;
  // QRCP path: A (m n) + Q0 (m k) + W2 (n k) + Vacc (k k) + norms/perm/tau/sig/order
  const size_t k = cols;
  const size_t qr = (size_t)m * n + (size_t)m * k + (size_t)n * k + k * k + 2 * (size_t)n + 4 * k + 16;
  return jac > qr ? jac : qr;
}

namespace {
__global__ void __launch_bounds__(512)
svd_kernel(const SvdDesc* __restrict__ descs, int n, double thr, int smem_doubles, int rel_mode) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ int sflag;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const SvdDesc d = descs[b];
    const bool tr = d.m < d.n;
    const int rows = tr ? d.n : d.m, cols = tr ? d.m : d.n;
    if (cols == 0) { if (threadIdx.x == 0) *d.rank = 0; continue; }
    const size_t need = svd_work_doubles(d.m, d.n);
    double* W = (need <= (size_t)smem_doubles) ? smem : d.work;
    double* V = W + (size_t)rows * cols;
    double* sig = V + (size_t)cols * cols;
    int* order = (int*)(sig + cols);
    // load (col-major rows x cols) and Frobenius norm
    double fro = 0.0;
    for (long long e = threadIdx.x; e < (long long)rows * cols; e += blockDim.x) {
      const int j = (int)(e / rows), i = (int)(e % rows);
      // element (i,j) of the oriented matrix
      const double v = tr ? d.src[(size_t)j * d.s_r + (size_t)i * d.s_c]
                          : d.src[(size_t)i * d.s_r + (size_t)j * d.s_c];
      W[e] = v;
      fro = fma(v, v, fro);
    }
    fro = block_sum(fro, red);
    // exact pre-filter: sigma_1 <= ||F||_F <= thr  =>  rank 0
    if (!rel_mode && sqrt(fro) <= thr * (1.0 - 1e-12)) {
      if (threadIdx.x == 0) *d.rank = 0;
      __syncthreads();
      continue;
    }
    cta_jacobi(W, rows, cols, rows, V, &sflag);
    cta_sv_order(W, rows, cols, rows, sig, order);
    int k = 0;
    if (rel_mode) {  // h2.py:124-127: max(1, #{s > rel * s0})
      const double t = thr * sig[order[0]];
      for (int j = 0; j < cols; ++j) k += sig[order[j]] > t;
      if (k < 1) k = 1;
    } else {
      for (int j = 0; j < cols; ++j) k += sig[order[j]] > thr;
    }
    // write U (m x k) col-major ld m, S, V (n x k) col-major ld n
    for (long long e = threadIdx.x; e < (long long)rows * k; e += blockDim.x) {
      const int pos = (int)(e / rows), i = (int)(e % rows);
      const int j = order[pos];
      const double u = W[(size_t)j * rows + i] / sig[j];
      if (!tr) d.U[(size_t)pos * d.m + i] = u; else d.V[(size_t)pos * d.n + i] = u;
    }
    for (long long e = threadIdx.x; e < (long long)cols * k; e += blockDim.x) {
      const int pos = (int)(e / cols), i = (int)(e % cols);
      const double v = V[(size_t)order[pos] * cols + i];
      if (!tr) d.V[(size_t)pos * d.n + i] = v; else d.U[(size_t)pos * d.m + i] = v;
    }
    for (int pos = threadIdx.x; pos < k; pos += blockDim.x) d.S[pos] = sig[order[pos]];
    if (threadIdx.x == 0) *d.rank = k;
    __syncthreads();
  }
}
}  // namespace

size_t svd_smem_doubles(int max_smem_dim) {
  size_t need = svd_work_doubles(max_smem_dim, max_smem_dim);
  return need * sizeof(double) > 200 * 1024 ? 0 : need;
}


// Householder QR with column pivoting of col-major A (m x n, ld m), in place
// (R upper, scaled reflectors below, taus), stopping once the remaining
// Frobenius mass sum(nrm[j:]) <= stop2.  nrm must hold the squared column
// norms on entry; perm receives the pivot order.  Returns the step count.
__device__ int cta_qrcp(double* A, int m, int nn, int kmax, double* nrm, int* perm, double* tau,
                        double stop2, double* red, long long* redi) {
  __shared__ double s_beta, s_tau, s_scale;
  __shared__ int s_p, s_stop;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int r0 = 0;
  for (int j = 0; j < kmax; ++j) {
    double t = 0.0, bv = -1.0;
    long long bi = (1LL << 62);
    for (int c2 = j + threadIdx.x; c2 < nn; c2 += blockDim.x) {
      const double v = nrm[c2];
      t += v;
      if (v > bv || (v == bv && c2 < bi)) { bv = v; bi = c2; }
    }
    t = block_sum(t, red);
    block_argmax(bv, bi, red, redi);
    // non-finite norms (a failed pivot upstream): stop instead of indexing garbage
    if (threadIdx.x == 0) { s_stop = !(t > stop2) || bi < j || bi >= nn; s_p = (int)bi; }
    __syncthreads();
    if (s_stop) break;
    const int p = s_p;
    if (p != j) {
      for (int i = threadIdx.x; i < m; i += blockDim.x) {
        const double u = A[(size_t)j * m + i];
        A[(size_t)j * m + i] = A[(size_t)p * m + i];
        A[(size_t)p * m + i] = u;
      }
      if (threadIdx.x == 0) {
        const double u = nrm[j]; nrm[j] = nrm[p]; nrm[p] = u;
        const int q = perm[j]; perm[j] = perm[p]; perm[p] = q;
      }
    }
    __syncthreads();
    double* a = A + (size_t)j * m;
    double nx = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) nx = fma(a[i], a[i], nx);
    nx = block_sum(nx, red);
    if (threadIdx.x == 0) {
      const double alpha = a[j];
      if (nx == 0.0) { s_tau = 0.0; s_beta = alpha; s_scale = 0.0; }
      else {
        const double beta = -copysign(sqrt(alpha * alpha + nx), alpha);
        s_tau = (beta - alpha) / beta;
        s_scale = 1.0 / (alpha - beta);
        s_beta = beta;
      }
      tau[j] = s_tau;
    }
    __syncthreads();
    const double sc = s_scale, tj = s_tau;
    if (tj != 0.0)
      for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) a[i] *= sc;
    __syncthreads();
    if (threadIdx.x == 0) a[j] = s_beta;
    for (int c2 = j + 1 + warp; c2 < nn; c2 += nw) {
      double* ac = A + (size_t)c2 * m;
      if (tj != 0.0) {
        double w = (lane == 0) ? ac[j] : 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) w = fma(a[i], ac[i], w);
        w = warp_sum(w) * tj;
        if (lane == 0) ac[j] -= w;
        for (int i = j + 1 + lane; i < m; i += 32) ac[i] -= w * a[i];
      }
      double s = 0.0;
      for (int i = j + 1 + lane; i < m; i += 32) s = fma(ac[i], ac[i], s);
      s = warp_sum(s);
      if (lane == 0) nrm[c2] = s;
    }
    r0 = j + 1;
    __syncthreads();
  }
  return r0;
}

namespace {
// Truncated SVD through a rank-revealing pivoted QR (fill compression).
// F P = Q R; stop at step r0 once ||R22||_F <= delta, delta = max(1e-9 thr,
// rounding level of F).  Then one-sided Jacobi on M^T = (R0 P^T)^T
// (n x r0):  F ~= Q0 M = (Q0 Vacc) S (W2 Vacc / S)^T.  Weyl: every
// singular value moves by <= delta, so `sigma > thr` only differs from an
// exact SVD for sigma within delta of thr.
__global__ void __launch_bounds__(512)
fill_svd_kernel(const SvdDesc* __restrict__ descs, int n, double thr, int smem_doubles,
                double delta_rel) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ long long redi[32];
  __shared__ int sflag;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int bb = blockIdx.x; bb < n; bb += gridDim.x) {
    const SvdDesc d = descs[bb];
    const int m = d.m, nn = d.n;
    const int kmax = m < nn ? m : nn;
    if (kmax == 0) { if (threadIdx.x == 0) *d.rank = 0; continue; }
    const size_t need = svd_work_doubles(m, nn);
    double* A = (need <= (size_t)smem_doubles) ? smem : d.work;
    double* Q0 = A + (size_t)m * nn;
    double* W2 = Q0 + (size_t)m * kmax;
    double* Vc = W2 + (size_t)nn * kmax;
    double* nrm = Vc + (size_t)kmax * kmax;
    double* tau = nrm + nn;
    double* sig = tau + kmax;
    int* perm = (int*)(sig + kmax);
    int* order = perm + nn;
    // load col-major + column norms
    for (long long e = threadIdx.x; e < (long long)m * nn; e += blockDim.x) {
      const int j = (int)(e / m), i = (int)(e % m);
      A[e] = d.src[(size_t)i * d.s_r + (size_t)j * d.s_c];
    }
    for (int j = threadIdx.x; j < nn; j += blockDim.x) perm[j] = j;
    __syncthreads();
    for (int j = warp; j < nn; j += nw) {
      double s = 0.0;
      for (int i = lane; i < m; i += 32) { const double u = A[(size_t)j * m + i]; s = fma(u, u, s); }
      s = warp_sum(s);
      if (lane == 0) nrm[j] = s;
    }
    __syncthreads();
    double fro = 0.0;
    for (int j = threadIdx.x; j < nn; j += blockDim.x) fro += nrm[j];
    fro = block_sum(fro, red);
    if (!(sqrt(fro) > thr * (1.0 - 1e-12))) {  // sigma_1 <= ||F||_F <= thr (or non-finite F)
      if (threadIdx.x == 0) *d.rank = 0;
      __syncthreads();
      continue;
    }
    const double delta = fmax(delta_rel * thr, 2.2e-16 * sqrt(fro) * sqrt((double)kmax));
    const int r0 = cta_qrcp(A, m, nn, kmax, nrm, perm, tau, delta * delta, red, redi);
    if (r0 == 0) { if (threadIdx.x == 0) *d.rank = 0; __syncthreads(); continue; }
    // Q0 (m x r0) and W2 = (R0 P^T)^T (n x r0)
    cta_orgqr(A, m, r0, m, tau, Q0, m);
    for (long long e = threadIdx.x; e < (long long)nn * r0; e += blockDim.x) {
      const int aa = (int)(e / nn), jj = (int)(e % nn);  // row aa of R, column position jj
      W2[(size_t)aa * nn + perm[jj]] = (aa <= jj) ? A[(size_t)jj * m + aa] : 0.0;
    }
    __syncthreads();
    cta_jacobi(W2, nn, r0, nn, Vc, &sflag);
    cta_sv_order(W2, nn, r0, nn, sig, order);
    int k = 0;
    for (int j = 0; j < r0; ++j) k += sig[order[j]] > thr;
    // U = Q0 Vc[:, order] (m x k); V = W2[:, order] / sig (n x k)
    for (long long e = threadIdx.x; e < (long long)m * k; e += blockDim.x) {
      const int pos = (int)(e / m), i = (int)(e % m);
      const double* v = Vc + (size_t)order[pos] * r0;
      double acc = 0.0;
      for (int l = 0; l < r0; ++l) acc = fma(Q0[(size_t)l * m + i], v[l], acc);
      d.U[(size_t)pos * m + i] = acc;
    }
    for (long long e = threadIdx.x; e < (long long)nn * k; e += blockDim.x) {
      const int pos = (int)(e / nn), i = (int)(e % nn);
      const int j = order[pos];
      d.V[(size_t)pos * nn + i] = W2[(size_t)j * nn + i] / sig[j];
    }
    for (int pos = threadIdx.x; pos < k; pos += blockDim.x) d.S[pos] = sig[order[pos]];
    if (threadIdx.x == 0) *d.rank = k;
    __syncthreads();
  }
}
}  // namespace

void launch_svd(const SvdDesc* d_descs, int n, double thr, int max_smem_dim, cudaStream_t s,
                int rel_mode) {
  DbgSync dbg_sync_{s, "launch_svd"};
  if (n > 0 && !rel_mode) {
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(fill_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      attr2 = true;
    }
    const size_t bytes = svd_smem_doubles(max_smem_dim) * sizeof(double);
    static double delta_rel = -1.0;
    if (delta_rel < 0) {  // IFMM_FILL_DELTA: truncation tolerance of the QRCP (x thr)
      const char* e = getenv("IFMM_FILL_DELTA");
      delta_rel = e ? atof(e) : 1e-6;
    }
    fill_svd_kernel<<<n < 4096 ? n : 4096, 512, bytes, s>>>(d_descs, n, thr,
                                                           (int)(bytes / sizeof(double)),
                                                           delta_rel);
    return;
  }
  if (n <= 0) return;
  // shared-memory workspace for blocks up to max_smem_dim^2 (fits 200 KB)
  size_t bytes = svd_smem_doubles(max_smem_dim) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  svd_kernel<<<n < 4096 ? n : 4096, 512, bytes, s>>>(d_descs, n, thr, (int)(bytes / sizeof(double)),
                                                     rel_mode);
}

// ============================================================================
// Householder QR (dgeqrf/dlarfg conventions) -- CTA cooperative
// ============================================================================

// A: col-major rows x cols (ld lda), rows >= cols.  In place: R in the upper
// triangle, Householder vectors (implicit unit head) below; tau[cols].
__device__ __forceinline__ void cta_geqrf(double* A, int rows, int cols, int lda, double* tau, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __shared__ double s_beta, s_tau, s_scale;
  for (int j = 0; j < cols; ++j) {
    double* a = A + (size_t)j * lda;
    double nx = 0.0;
    for (int i = j + 1 + threadIdx.x; i < rows; i += blockDim.x) nx = fma(a[i], a[i], nx);
    nx = block_sum(nx, red);
    if (threadIdx.x == 0) {
      const double alpha = a[j];
      if (nx == 0.0) { s_tau = 0.0; s_beta = alpha; s_scale = 0.0; }
      else {
        const double beta = -copysign(sqrt(alpha * alpha + nx), alpha);
        s_tau = (beta - alpha) / beta;
        s_scale = 1.0 / (alpha - beta);
        s_beta = beta;
      }
      tau[j] = s_tau;
    }
    __syncthreads();
    const double sc = s_scale, tj = s_tau;
    if (tj != 0.0)
      for (int i = j + 1 + threadIdx.x; i < rows; i += blockDim.x) a[i] *= sc;
    __syncthreads();
    if (threadIdx.x == 0) a[j] = s_beta;
    // apply H = I - tau v v^T to trailing columns
    if (tj != 0.0) {
      for (int c = j + 1 + warp; c < cols; c += nw) {
        double* ac = A + (size_t)c * lda;
        double w = (lane == 0) ? ac[j] : 0.0;
        for (int i = j + 1 + lane; i < rows; i += 32) w = fma(a[i], ac[i], w);
        w = warp_sum(w) * tj;
        if (lane == 0) ac[j] -= w;
        for (int i = j + 1 + lane; i < rows; i += 32) ac[i] -= w * a[i];
      }
    }
    __syncthreads();
  }
}

// Form Q (rows x cols, col-major ld ldq) from cta_geqrf output.
__device__ __forceinline__ void cta_orgqr(const double* A, int rows, int cols, int lda, const double* tau,
                          double* Q, int ldq) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long e = threadIdx.x; e < (long long)rows * cols; e += blockDim.x) {
    const int c = (int)(e / rows), i = (int)(e % rows);
    Q[(size_t)c * ldq + i] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = cols - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj != 0.0) {
      const double* v = A + (size_t)j * lda;
      for (int c = j + warp; c < cols; c += nw) {
        double* qc = Q + (size_t)c * ldq;
        double w = (lane == 0) ? qc[j] : 0.0;
        for (int i = j + 1 + lane; i < rows; i += 32) w = fma(v[i], qc[i], w);
        w = warp_sum(w) * tj;
        if (lane == 0) qc[j] -= w;
        for (int i = j + 1 + lane; i < rows; i += 32) qc[i] -= w * v[i];
      }
    }
    __syncthreads();
  }
}

// ============================================================================
// Weighted basis union: ACA (full pivot) + QR + QR + Jacobi SVD
// ============================================================================

__host__ __device__ size_t union_work_doubles(int m, int k_old, int k_f) {
  const size_t C = (size_t)k_old + k_f;
  const size_t s = (size_t)(m < (int)C ? m : (int)C);
  const size_t sp = s + (s & 1);
  // Mreg: ACA residual (m C), then 6 s x sp CholeskyQR matrices, or QA
  //       (m s) on the Householder path
  // | Acol (m s) | Bt (C s) | QB (C s, Householder path) | W, V (2 s^2)
  // | D, tauA, tauB, sig (4 s) | order (s ints) | acts, pos (2 C ints)
  const size_t mreg = (size_t)m * C > 6 * s * sp ? (size_t)m * C : 6 * s * sp;
  return mreg + (size_t)m * s + 2 * C * s + 2 * s * s + 5 * s + C + 16;
}

void union_profile(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_uprof, sizeof(unsigned long long) * 48);
  if (reset) {
    unsigned long long z[48] = {};
    cudaMemcpyToSymbol(g_uprof, z, sizeof z);
  }
}

namespace {
constexpr int UNION_SMEM_DOUBLES = 28500;  // 228 KB
constexpr int UNION_SVD_SMEM_DOUBLES = 28900;  // 231 KB

// Interleaved Householder QR of two column-major matrices A (ra x s) and
// B (rb x s): two barriers per column for both.  On exit: R in the upper
// triangles, scaled reflectors below, taus in tauA / tauB.
__device__ __forceinline__ void cta_geqrf2(double* A, int ra, double* B, int rb, int s, double* tauA, double* tauB,
                           double* pa, double* pb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double scA = 0.0, scB = 0.0, bA = 0.0, bB = 0.0;
  for (int j = 0; j < s; ++j) {
    // finish column j-1: scale its reflector and set the diagonal
    if (j > 0) {
      double* a = A + (size_t)(j - 1) * ra;
      double* b = B + (size_t)(j - 1) * rb;
      for (int i = j + threadIdx.x; i < ra; i += blockDim.x) a[i] *= scA;
      for (int i = j + threadIdx.x; i < rb; i += blockDim.x) b[i] *= scB;
      if (threadIdx.x == 0) { a[j - 1] = bA; b[j - 1] = bB; }
    }
    const double* a = A + (size_t)j * ra;
    const double* b = B + (size_t)j * rb;
    double na = 0.0, nb = 0.0;
    for (int i = j + 1 + threadIdx.x; i < ra; i += blockDim.x) na = fma(a[i], a[i], na);
    for (int i = j + 1 + threadIdx.x; i < rb; i += blockDim.x) nb = fma(b[i], b[i], nb);
    na = warp_sum(na);
    nb = warp_sum(nb);
    if (lane == 0) { pa[warp] = na; pb[warp] = nb; }
    __syncthreads();
    na = 0.0; nb = 0.0;
    for (int w = 0; w < nw; ++w) { na += pa[w]; nb += pb[w]; }
    const double alA = a[j], alB = b[j];
    double tA = 0.0, tB = 0.0;
    if (na == 0.0) { tA = 0.0; bA = alA; scA = 0.0; }
    else { bA = -copysign(sqrt(alA * alA + na), alA); tA = (bA - alA) / bA; scA = 1.0 / (alA - bA); }
    if (nb == 0.0) { tB = 0.0; bB = alB; scB = 0.0; }
    else { bB = -copysign(sqrt(alB * alB + nb), alB); tB = (bB - alB) / bB; scB = 1.0 / (alB - bB); }
    if (threadIdx.x == 0) { tauA[j] = tA; tauB[j] = tB; }
    // trailing updates: columns of A then of B, one warp per column
    const int ntr = s - j - 1;
    for (int t = warp; t < 2 * ntr; t += nw) {
      const bool isA = t < ntr;
      const int cidx = j + 1 + (isA ? t : t - ntr);
      const double tau = isA ? tA : tB;
      if (tau == 0.0) continue;
      const double sc = isA ? scA : scB;
      const double* v = isA ? a : b;
      double* col = (isA ? A + (size_t)cidx * ra : B + (size_t)cidx * rb);
      const int rr = isA ? ra : rb;
      double w = (lane == 0) ? col[j] : 0.0;
      for (int i = j + 1 + lane; i < rr; i += 32) w = fma(v[i] * sc, col[i], w);
      w = warp_sum(w) * tau;
      if (lane == 0) col[j] -= w;
      for (int i = j + 1 + lane; i < rr; i += 32) col[i] -= w * (v[i] * sc);
    }
    __syncthreads();
  }
  if (s > 0) {
    double* a = A + (size_t)(s - 1) * ra;
    double* b = B + (size_t)(s - 1) * rb;
    for (int i = s + threadIdx.x; i < ra; i += blockDim.x) a[i] *= scA;
    for (int i = s + threadIdx.x; i < rb; i += blockDim.x) b[i] *= scB;
    if (threadIdx.x == 0) { a[s - 1] = bA; b[s - 1] = bB; }
  }
  __syncthreads();
}

// Interleaved Q formation for the two factorizations (one barrier / column).
__device__ __forceinline__ void cta_orgqr2(const double* A, int ra, const double* tauA, double* QA,
                           const double* B, int rb, const double* tauB, double* QB, int s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long e = threadIdx.x; e < (long long)ra * s; e += blockDim.x) {
    const int c = (int)(e / ra), i = (int)(e % ra);
    QA[e] = (i == c) ? 1.0 : 0.0;
  }
  for (long long e = threadIdx.x; e < (long long)rb * s; e += blockDim.x) {
    const int c = (int)(e / rb), i = (int)(e % rb);
    QB[e] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = s - 1; j >= 0; --j) {
    const int ntr = s - j;
    for (int t = warp; t < 2 * ntr; t += nw) {
      const bool isA = t < ntr;
      const int cidx = j + (isA ? t : t - ntr);
      const double tau = isA ? tauA[j] : tauB[j];
      if (tau == 0.0) continue;
      const double* v = isA ? A + (size_t)j * ra : B + (size_t)j * rb;
      double* q = isA ? QA + (size_t)cidx * ra : QB + (size_t)cidx * rb;
      const int rr = isA ? ra : rb;
      double w = (lane == 0) ? q[j] : 0.0;
      for (int i = j + 1 + lane; i < rr; i += 32) w = fma(v[i], q[i], w);
      w = warp_sum(w) * tau;
      if (lane == 0) q[j] -= w;
      for (int i = j + 1 + lane; i < rr; i += 32) q[i] -= w * v[i];
    }
    __syncthreads();
  }
}

// ---- CholeskyQR2 pieces for the ACA factors ---------------------------------
// The ACA is an LU with full pivoting: X = P L~ D with L~ unit lower
// trapezoidal, |L~| <= 1, D = diag(pivots), and Y unit lower trapezoidal.
// L~ and Y are well conditioned (cond <= 40 on every large union of the c3
// recipe at N=32768, measured on oracle unions), while the pivots carry the
// grading.  Householder QR of X D^{-1} and of Y is therefore replaced by two
// CholeskyQR passes (Gram, Cholesky, row-wise triangular solve): two
// parallel phases + s barriers instead of ~3s barriers.  R_A = R~ D keeps the
// column-wise backward error of Householder QR.  A Cholesky pivot ratio
// below kCholFloor (cond(L~) > ~1e6) sends the union to the Householder path.
constexpr double kCholFloor = 1e-12;

// Upper triangles of G_A = A^T A and G_B = B^T B (A: ra x s, B: rb x s,
// col-major), row-major with ld sp.  One warp per 4x4 tile, lanes split rows.
// wbase / wstride: this CTA's first warp index and the warp stride over the
// tiles (one CTA: 0 / warps per CTA; several CTAs share the tiles otherwise)
__device__ __forceinline__ void cta_gram2(const double* A, int ra, const double* B, int rb, int s,
                                          int sp, double* GA, double* GB, int wbase = 0,
                                          int wstride = 0) {
  const int lane = threadIdx.x & 31;
  const int warp = wbase + (threadIdx.x >> 5);
  const int nw = wstride > 0 ? wstride : (blockDim.x >> 5);
  const int nb = (s + 3) >> 2, ntile = nb * (nb + 1) / 2;
  for (int t = warp; t < 2 * ntile; t += nw) {
    const bool isA = t < ntile;
    const int tt = isA ? t : t - ntile;
    int bj = 0;
    while ((bj + 1) * (bj + 2) / 2 <= tt) ++bj;
    const int bi = tt - bj * (bj + 1) / 2;
    const double* X = isA ? A : B;
    const int r = isA ? ra : rb;
    double* G = isA ? GA : GB;
    const int i0 = bi * 4, j0 = bj * 4;
    int ci[4], cj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { ci[u] = min(i0 + u, s - 1); cj[u] = min(j0 + u, s - 1); }
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    for (int row = lane; row < r; row += 32) {
      double xi[4], xj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { xi[u] = X[(size_t)ci[u] * r + row]; xj[u] = X[(size_t)cj[u] * r + row]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(xi[u], xj[v], acc[u][v]);
    }
    // transpose-reduce the 16 partial sums: 8+4+2+1+1 shuffles; afterwards
    // lane pair (2 idx, 2 idx + 1) holds the total of value idx = 4u + v
    double v16[16];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) v16[4 * u + v] = acc[u][v];
#pragma unroll
    for (int h = 8, bit = 16; h >= 1; h >>= 1, bit >>= 1) {
      const bool up = lane & bit;
#pragma unroll
      for (int k = 0; k < h; ++k) {
        const double send = up ? v16[k] : v16[k + h];
        const double keep = up ? v16[k + h] : v16[k];
        v16[k] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
      }
    }
    v16[0] += __shfl_xor_sync(0xffffffffu, v16[0], 1);
    if (!(lane & 1)) {
      const int idx = lane >> 1, i = i0 + (idx >> 2), j = j0 + (idx & 3);
      if (i < s && j < s && i <= j) G[(size_t)i * sp + j] = v16[0];
    }
  }
}

// In-place right-looking Cholesky G = R^T R of two SPD matrices at once
// (upper triangles, row-major ld sp), one barrier per step: step k
// eliminates with row k unscaled and scales row k-1 (no longer read) into
// R.  On exit the upper triangles hold R (the strict lower parts are never
// read); rinv[k] = 1 / R[k][k].  Returns the smallest pivot ratio
// R_kk^2 / max_i G_ii over both matrices (uniform across the CTA).
__device__ __forceinline__ double cta_chol2(double* GA, double* ia, double* GB, double* ib, int s, int sp) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  double minr = 1.0, mxA = 0.0, mxB = 0.0;
  for (int k = 0; k < s; ++k) {
    mxA = fmax(mxA, GA[(size_t)k * sp + k]);
    mxB = fmax(mxB, GB[(size_t)k * sp + k]);
  }
  const double imxA = 1.0 / mxA, imxB = 1.0 / mxB;
  __syncthreads();
  for (int k = 0; k <= s; ++k) {
    if (k > 0) {  // finalise row k-1 of both R factors
      const double ra = ia[k - 1], rb = ib[k - 1];
      double* gra = GA + (size_t)(k - 1) * sp;
      double* grb = GB + (size_t)(k - 1) * sp;
      for (int j = k - 1 + threadIdx.x; j < s; j += blockDim.x) {
        gra[j] *= ra;
        grb[j] *= rb;
      }
    }
    if (k < s) {
      // both pivots' reciprocals first (independent long-latency chains)
      const double* ga = GA + (size_t)k * sp;
      const double* gb = GB + (size_t)k * sp;
      const double pa = ga[k], pb = gb[k];
      const double inva = 1.0 / pa, invb = 1.0 / pb;
      const double ra = rsqrt(pa), rb = rsqrt(pb);
      const double qa = pa * imxA, qb = pb * imxB;
      minr = (qa > 0.0 && isfinite(pa)) ? fmin(minr, qa) : 0.0;
      minr = (qb > 0.0 && isfinite(pb)) ? fmin(minr, qb) : 0.0;
      if (threadIdx.x == 0) { ia[k] = ra; ib[k] = rb; }
      // trailing rows i > k of both matrices, one warp per (matrix, row),
      // lanes along the row; all loads of a row before its stores
      const int nr = s - k - 1;
      for (int t = wid; t < 2 * nr; t += nwp) {
        const bool isA = t < nr;
        const int i = k + 1 + (isA ? t : t - nr);
        const double* g = isA ? ga : gb;
        double* Gi = (isA ? GA : GB) + (size_t)i * sp;
        const double fi = g[i] * (isA ? inva : invb);
        for (int j0 = i + lane; j0 < s; j0 += 128) {
          double gv[4], gw[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + 32 * u;
            gv[u] = j < s ? g[j] : 0.0;
            gw[u] = j < s ? Gi[j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + 32 * u;
            if (j < s) Gi[j] = fma(-fi, gv[u], gw[u]);
          }
        }
      }
    }
    __syncthreads();
  }
  return minr;
}

// A <- A R^{-1} row by row (A: r x s col-major; R row-major upper, ld sp,
// rinv = 1 / diag), both matrices at once; 8-column register blocks.
__device__ __forceinline__ void cta_trsm2(double* A, int ra, const double* RA, const double* ia,
                                          double* B, int rb, const double* RB, const double* ib,
                                          int s, int sp, int tbase = 0, int tstride = 0) {
  const int t0 = tbase + threadIdx.x, ts = tstride > 0 ? tstride : blockDim.x;
  for (int row = t0; row < ra + rb; row += ts) {
    const bool isA = row < ra;
    double* X = isA ? A : B;
    const int r = isA ? ra : rb, rr = isA ? row : row - ra;
    const double* R = isA ? RA : RB;
    const double* iv = isA ? ia : ib;
    for (int j0 = 0; j0 < s; j0 += 8) {
      double a[8];
      int cj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) { cj[u] = min(j0 + u, s - 1); a[u] = X[(size_t)cj[u] * r + rr]; }
      // already-solved entries of the row, 8 independent loads per batch
      // (X may sit in global memory: one L2 round trip per batch, not per entry)
      for (int i0 = 0; i0 < j0; i0 += 8) {
        double xv[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) xv[v] = X[(size_t)(i0 + v) * r + rr];  // i0 + 8 <= j0
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const double* Ri = R + (size_t)(i0 + v) * sp;
#pragma unroll
          for (int u = 0; u < 8; ++u) a[u] = fma(-xv[v], Ri[cj[u]], a[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        a[u] *= iv[cj[u]];
        const double* Ru = R + (size_t)cj[u] * sp;
#pragma unroll
        for (int v = u + 1; v < 8; ++v) a[v] = fma(-a[u], Ru[cj[v]], a[v]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j0 + u < s) X[(size_t)(j0 + u) * r + rr] = a[u];
    }
  }
}

// T = R2 R1 (row-major upper, ld sp) for two pairs at once.
__device__ __forceinline__ void cta_trmul2(const double* A2, const double* A1, double* TA, const double* B2,
                                           const double* B1, double* TB, int s, int sp,
                                           int tbase = 0, int tstride = 0) {
  const int t0 = tbase + threadIdx.x, ts = tstride > 0 ? tstride : blockDim.x;
  for (int e = t0; e < 2 * s * s; e += ts) {
    const bool isA = e < s * s;
    const int f = isA ? e : e - s * s;
    const int i = f / s, j = f - i * s;
    const double* R2 = isA ? A2 : B2;
    const double* R1 = isA ? A1 : B1;
    double acc = 0.0;
    for (int l = i; l <= j; ++l) acc = fma(R2[(size_t)i * sp + l], R1[(size_t)l * sp + j], acc);
    (isA ? TA : TB)[(size_t)i * sp + j] = (i <= j) ? acc : 0.0;
  }
}

template <bool SM>
__global__ void __launch_bounds__(512)
union_kernel(const UnionDesc* __restrict__ descs, int n, double thr, int smem_doubles, int force_hh) {
  extern __shared__ double smem[];
  __shared__ double wv[32];
  __shared__ long long wi[32];
  __shared__ double pa[32], pb[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int bb = blockIdx.x; bb < n; bb += gridDim.x) {
    const UnionDesc d = descs[bb];
    if (d.giant == 3) continue;  // union_post_kernel's (uniform per CTA)
    const int m = d.m, ko = d.k_old, C = d.k_old + d.k_f;
    const int smax = m < C ? m : C;
    const int spx = smax + (smax & 1);
    // Mw: the workspace's residual region.  M: where the ACA residual lives --
    // shared memory on the smem variant, and on the global variant too when
    // m x C fits (the rest of the workspace stays in global memory).
    double* Mw = SM ? smem : d.work;  // compile-time space: LDS/STS on the smem path
    // global variant: the ACA's per-step vectors (pivot column, pivot row /
    // piv) and the active-column list live in shared memory after the
    // residual (when that fits) -- they are read for every residual entry
    const size_t scr_d = (size_t)m + C + C + 8;  // cc, rr, acts+pos (ints)
    const bool msm = !SM && (size_t)m * C + scr_d <= (size_t)smem_doubles;
    double* M = msm ? smem : Mw;
    const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
    double* Acol = Mw + mreg;
    double* Bt = Acol + (size_t)m * smax;
    double* QB = Bt + (size_t)C * smax;
    double* core = QB + (size_t)C * smax;
    double* Dp = core + 2 * (size_t)smax * smax;
    double* tauA = Dp + smax;
    double* tauB = tauA + smax;
    double* sig = tauB + smax;
    int* order = (int*)(sig + smax);
    int* acts = order + smax + 1;
    int* pos = acts + C;
    double* ccs = nullptr;  // on-chip copies of the current pivot column / row (global variant)
    double* rrs = nullptr;
    if (!SM) {
      double* scr = smem + (msm ? (size_t)m * C : 0);
      ccs = scr;
      rrs = scr + m;
      acts = (int*)(rrs + C);
      pos = acts + C;
    }

    int steps = 0;
    unsigned long long t0 = clock64();
    bool giant_hh = false;
    if (d.giant == 1) {
      // the ACA (union_aca_coop) and CholeskyQR (union_cholqr_coop) ran on
      // several CTAs; only a Householder fallback (hdr[1]) or s = 0 is left here
      const int* hg = (const int*)(Dp + 4 * (size_t)smax);
      steps = hg[0];
      if (steps > 0 && hg[1] == 0) continue;  // uniform per CTA
      giant_hh = steps > 0;
    } else if (d.giant == 2) {
      // the register-resident ACA (union_aca_reg, union_aca.cu) ran: X, Y and
      // the pivots sit in the global workspace (same offsets as Acol / Bt / Dp
      // of the global variant); the shared-memory variant copies them in
      double* gA = d.work + mreg;
      double* gB = gA + (size_t)m * smax;
      double* gD = gB + 2 * (size_t)C * smax + 2 * (size_t)smax * smax;
      steps = *(const int*)(gD + 4 * (size_t)smax);
      if (SM) {
        for (int e = threadIdx.x; e < m * steps; e += blockDim.x) Acol[e] = gA[e];
        for (int e = threadIdx.x; e < C * steps; e += blockDim.x) Bt[e] = gB[e];
        for (int e = threadIdx.x; e < steps; e += blockDim.x) Dp[e] = gD[e];
      }
    } else {
      // concat [B*diag(w) | F*diag(wf)] (col-major m x C) + first local argmax.
      // Thread layout: R threads cover the rows (coalesced), G = nthreads / R
      // column groups over the list of active (unpivoted) columns; the flat
      // (row-major, numpy) index only breaks exact ties.
      const int R = m < (int)blockDim.x ? m : (int)blockDim.x;
      const int G = blockDim.x / R;
      const int i0 = threadIdx.x % R, g0 = threadIdx.x / R;
      const bool on = g0 < G;
      double bv = -1.0;
      int bi = 0, bj = 0;
      auto better = [&](double av, int i, int j) {
        return av > bv || (av == bv && (long long)i * C + j < (long long)bi * C + bj);
      };
      for (int j = threadIdx.x; j < C; j += blockDim.x) { acts[j] = j; pos[j] = j; }
      int nact = C;  // every thread tracks the active count
      if (on)
        for (int i = i0; i < m; i += R)
          for (int j = g0; j < C; j += G) {
            const double v = j < ko ? d.B[(size_t)i * d.b_r + (size_t)j * d.b_c] * d.w[j]
                                    : d.F[(size_t)i * d.f_r + (size_t)(j - ko) * d.f_c] * d.wf[j - ko];
            M[(size_t)j * m + i] = v;
            const double av = fabs(v);
            if (better(av, i, j)) { bv = av; bi = i; bj = j; }
          }
      // ---- ACA, full pivoting, floor thr/8 (lowrank.py:128-151): 2 barriers/step.
      // A pivoted column becomes exactly zero (its row factor entry is piv/piv
      // = 1), so it leaves the active list; pivoted rows keep their rounding
      // residue and stay, as in the reference.
      t0 = clock64();
      const double floor_ = thr / 8.0;
      for (int it = 0; it < smax; ++it) {
        long long bflat = bv < 0.0 ? (1LL << 62) : (long long)bi * C + bj;
        warp_argmax(bv, bflat);
        if (lane == 0) { wv[warp] = bv; wi[warp] = bflat; }
        __syncthreads();
        double gv = lane < nw ? wv[lane] : -1.0;
        long long gi = lane < nw ? wi[lane] : (1LL << 62);
        warp_argmax(gv, gi);  // every lane of every warp: the block's pivot
        const int p = (int)(gi / C), q = (int)(gi - (long long)p * C);
        if (p < 0 || p >= m || q < 0 || q >= C) {
          if (threadIdx.x == 0)
            printf("[union] bad pivot m=%d C=%d step=%d nact=%d gi=%lld gv=%g\n", m, C, steps, nact, gi, gv);
          __trap();
        }
        const double piv = M[(size_t)q * m + p];
        if (piv == 0.0 || (fabs(piv) <= floor_ && steps >= d.min_rank)) break;  // uniform
        double* cc = Acol + (size_t)steps * m;
        double* rr = Bt + (size_t)steps * C;
        // column q leaves the active list: its residual is exactly zero from
        // here on (q's row factor entry is piv / piv = 1), stored as such
        // (the pivot entry itself is cleared after the barrier: every thread
        // reads it above)
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
          const double v = M[(size_t)q * m + i];
          cc[i] = v;
          if (!SM) ccs[i] = v;
          if (i != p) M[(size_t)q * m + i] = 0.0;
        }
        for (int j = threadIdx.x; j < C; j += blockDim.x) {
          const double v = j == q ? 1.0 : M[(size_t)j * m + p] / piv;
          rr[j] = v;
          if (!SM) rrs[j] = v;
        }
        if (threadIdx.x == 0) {  // swap-remove q from the active list
          const int k = pos[q], last = acts[nact - 1];
          if (k < 0 || k >= nact || acts[k] != q) {
            printf("[union] bad active list m=%d C=%d step=%d nact=%d q=%d k=%d\n", m, C, steps, nact, q, k);
            __trap();
          }
          acts[k] = last;
          pos[last] = k;
          Dp[steps] = piv;
        }
        --nact;
        __syncthreads();
        if (threadIdx.x == 0) M[(size_t)q * m + p] = 0.0;
        const int na = nact;
        bv = -1.0;
        if (SM) {
          if (on)
            for (int i = i0; i < m; i += R) {
              const double ci = cc[i];
              int l = g0;
              for (; l + 7 * G < na; l += 8 * G) {
                int jj[8];
                double v[8];
  #pragma unroll
                for (int u = 0; u < 8; ++u) { jj[u] = acts[l + u * G]; v[u] = M[(size_t)jj[u] * m + i]; }
  #pragma unroll
                for (int u = 0; u < 8; ++u) {
                  v[u] = fma(-ci, rr[jj[u]], v[u]);
                  M[(size_t)jj[u] * m + i] = v[u];
                  const double av = fabs(v[u]);
                  if (better(av, i, jj[u])) { bv = av; bi = i; bj = jj[u]; }
                }
              }
              for (; l < na; l += G) {
                const int j = acts[l];
                double* mp = M + (size_t)j * m + i;
                const double v = fma(-ci, rr[j], *mp);
                *mp = v;
                const double av = fabs(v);
                if (better(av, i, j)) { bv = av; bi = i; bj = j; }
              }
            }
        } else {
          // global workspace: M streams through L2 every step.  The m x na
          // active block is flattened (row fastest, coalesced) and dealt out
          // evenly; every batch issues all UN loads before any store, also in
          // the last partial batch (a load after a possibly aliasing store
          // would serialise on the L2 round trip).
          constexpr int UN = 16;
          const int total = m * na, nthr = blockDim.x;
          const int di = nthr % m, dl = nthr / m;
          int f = threadIdx.x, i = f % m, l = f / m;
          while (f < total) {
            int ii[UN], jj[UN];
            double v[UN];
  #pragma unroll
            for (int u = 0; u < UN; ++u) {
              const bool ok = f + u * nthr < total;
              ii[u] = i;
              jj[u] = ok ? acts[l] : -1;
              v[u] = ok ? M[(size_t)jj[u] * m + i] : 0.0;
              i += di; l += dl;
              if (i >= m) { i -= m; ++l; }
            }
  #pragma unroll
            for (int u = 0; u < UN; ++u) {
              if (jj[u] < 0) break;
              v[u] = fma(-ccs[ii[u]], rrs[jj[u]], v[u]);
              M[(size_t)jj[u] * m + ii[u]] = v[u];
              const double av = fabs(v[u]);
              if (better(av, ii[u], jj[u])) { bv = av; bi = ii[u]; bj = jj[u]; }
            }
            f += UN * nthr;
          }
        }
        ++steps;
      }
    }
    __syncthreads();
    if (steps == 0) {
      if (threadIdx.x == 0) {
        *d.rank = 0;
        double* gW = d.work + mreg + (size_t)m * smax + 2 * (size_t)C * smax;
        *(int*)(gW + 2 * (size_t)smax * smax) = 0;  // header: s = 0
      }
      __syncthreads();
      continue;
    }
    const int s = steps;
    const int sp = s + (s & 1);
    unsigned long long t1 = clock64();
    // ---- scale X columns by 1/pivot: L~ = X D^{-1} ----
    // thread per row, 8 columns per batch with all loads before the stores
    // (giant unions: already scaled by union_cholqr_coop)
    if (d.giant != 1)
    for (int i = threadIdx.x; i < m; i += blockDim.x)
      for (int t0 = 0; t0 < s; t0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = t0 + u < s ? Acol[(size_t)(t0 + u) * m + i] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t0 + u < s) Acol[(size_t)(t0 + u) * m + i] = v[u] / Dp[t0 + u];
      }
    // ---- CholeskyQR2 of L~ (m x s) and Y (C x s); M is free now ----
    // CholeskyQR workspace: G_A, G_B (Cholesky in place -> R) in shared
    // memory for the global variant when 2 s x sp fit; R1 and the products
    // T = R2 R1 live in the (dead) residual region.
    const bool qsm = !SM && 2 * (size_t)s * sp <= (size_t)smem_doubles;
    double* GA = qsm ? smem : Mw;
    double* GB = GA + (size_t)s * sp;
    double* RA1s = Mw + (qsm ? 0 : 2 * (size_t)s * sp);
    double* RB1s = RA1s + (size_t)s * sp;
    double* TA = RB1s + (size_t)s * sp;
    double* TB = TA + (size_t)s * sp;
    double* ia = tauA;  // 1 / diag
    double* ib = tauB;
    __syncthreads();
    double r1 = 0.0;
    if (!force_hh && !giant_hh) {
      cta_gram2(Acol, m, Bt, C, s, sp, GA, GB);
      __syncthreads();
      r1 = cta_chol2(GA, ia, GB, ib, s, sp);
    }
    // cond(L~) or cond(Y) above ~1e6: Householder path instead
    const bool hh = force_hh || giant_hh || !(r1 > kCholFloor);
    const double* QAp;
    const double* QBp;
    // W = core^T (s x s): in shared memory on the global variant when it fits
    double* Wc = (!SM && (size_t)s * s <= (size_t)smem_doubles) ? smem : core;
    if (!hh) {
      unsigned long long c0 = clock64();
      cta_trsm2(Acol, m, GA, ia, Bt, C, GB, ib, s, sp);
      for (int e = threadIdx.x; e < 2 * s * sp; e += blockDim.x) RA1s[e] = GA[e];  // park R1
      __syncthreads();
      unsigned long long c1 = clock64();
      cta_gram2(Acol, m, Bt, C, s, sp, GA, GB);
      __syncthreads();
      unsigned long long c2 = clock64();
      cta_chol2(GA, ia, GB, ib, s, sp);
      unsigned long long c3 = clock64();
      cta_trsm2(Acol, m, GA, ia, Bt, C, GB, ib, s, sp);
      // R_A = R_A2 R_A1, R_B = R_B2 R_B1
      cta_trmul2(GA, RA1s, TA, GB, RB1s, TB, s, sp);
      __syncthreads();
      unsigned long long c4 = clock64();
      if (threadIdx.x == 0 && m > 200) {  // CholeskyQR sub-phases of larger unions
        atomicAdd(&g_uprof[34], c1 - c0);
        atomicAdd(&g_uprof[35], c2 - c1);
        atomicAdd(&g_uprof[36], c3 - c2);
        atomicAdd(&g_uprof[37], c4 - c3);
        atomicAdd(&g_uprof[38], c0 - t1);
        atomicAdd(&g_uprof[39], 1ull);
      }
      // W = core^T = R_B D R_A^T
      for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int j = e / s, i = e - j * s;
        double acc = 0.0;
        for (int l = (i > j ? i : j); l < s; ++l)
          acc = fma(TB[(size_t)i * sp + l] * Dp[l], TA[(size_t)j * sp + l], acc);
        Wc[(size_t)j * s + i] = acc;
      }
      QAp = Acol;
      QBp = Bt;
    } else {
      // Householder fallback (ill-conditioned L~ or Y)
      __syncthreads();
      cta_geqrf2(Acol, m, Bt, C, s, tauA, tauB, pa, pb);
      for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int j = e / s, i = e - j * s;
        double acc = 0.0;
        for (int l = (i > j ? i : j); l < s; ++l)
          acc = fma(Bt[(size_t)l * C + i] * Dp[l], Acol[(size_t)l * m + j], acc);
        Wc[(size_t)j * s + i] = acc;
      }
      cta_orgqr2(Acol, m, tauA, Mw, Bt, C, tauB, QB, s);
      QAp = Mw;
      QBp = QB;
      if (threadIdx.x == 0) atomicAdd(&g_uprof[13], 1ull);
    }
    unsigned long long t2 = clock64();
    // ---- hand-off to union_svd_kernel: QA, QB and W = core^T persist in the
    // global workspace at fixed offsets, plus a header (s, QA / QB offsets)
    {
      double* g = d.work;
      double* gQA = g + mreg;
      double* gQB = gQA + (size_t)m * smax;
      double* gW = gQB + 2 * (size_t)C * smax;
      const double* QAsrc = QAp;
      const double* QBsrc = QBp;
      if (QAsrc != gQA)
        for (long long e = threadIdx.x; e < (long long)m * s; e += blockDim.x) gQA[e] = QAsrc[e];
      if (QBsrc != gQB)
        for (long long e = threadIdx.x; e < (long long)C * s; e += blockDim.x) gQB[e] = QBsrc[e];
      if (Wc != gW)
        for (int e = threadIdx.x; e < s * s; e += blockDim.x) gW[e] = Wc[e];
      __syncthreads();  // W formation read Dp
      if (threadIdx.x == 0) {
        int* hdr = (int*)(gW + 2 * (size_t)smax * smax);  // the (dead) pivot slot
        hdr[0] = s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicAdd(&g_uprof[0], t1 - t0);
      atomicAdd(&g_uprof[1], t2 - t1);
      atomicAdd(&g_uprof[5], (unsigned long long)s);
      atomicAdd(&g_uprof[6], 1ull);
      atomicAdd(&g_uprof[7], (unsigned long long)m);
      atomicAdd(&g_uprof[8], (unsigned long long)C);
      atomicAdd(&g_uprof[9], (unsigned long long)(M == smem));  // residual on chip
      if (m > 128) {  // larger unions separately: 128 < m <= 400 -> [16, 25), m > 400 -> [25, 34)
        unsigned long long* u = g_uprof + (m > 400 ? 25 : 16);
        atomicAdd(&u[0], t1 - t0);
        atomicAdd(&u[1], t2 - t1);
        atomicAdd(&u[5], (unsigned long long)s);
        atomicAdd(&u[6], 1ull);
        atomicAdd(&u[7], (unsigned long long)m);
        atomicAdd(&u[8], (unsigned long long)C);
      }
    }
  }
}

// new basis = QA phi[:, :k] and maps = (QB sigma psi)[col][a] / weight[col]:
// each thread owns one output row and a strip of 4 output columns (every Q
// element is loaded once per strip); threads tbase + threadIdx.x, stride tstride.
__device__ __forceinline__ void union_output(const UnionDesc& d, int s, int k, const double* gQA,
                                             const double* gQB, const double* Wc, const double* Vc,
                                             const int* order, int tbase, int tstride) {
  const int m = d.m, ko = d.k_old, C = d.k_old + d.k_f;
  const int kb = (k + 3) >> 2;
  for (long long e = tbase + threadIdx.x; e < (long long)(m + C) * kb; e += tstride) {
    const int row = (int)(e % (m + C)), a0 = 4 * (int)(e / (m + C));
    const bool isA = row < m;
    const int i = isA ? row : row - m;
    const double* Q = isA ? gQA + i : gQB + i;
    const int ldq = isA ? m : C;
    const double* col[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = order[min(a0 + u, k - 1)];
      col[u] = (isA ? Vc : Wc) + (size_t)j * s;
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l = 0; l < s; ++l) {
      const double q = Q[(size_t)l * ldq];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(q, col[u][l], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int a = a0 + u;
      if (a >= k) break;
      if (isA) d.NB[(size_t)i * d.nb_r + (size_t)a * d.nb_c] = acc[u];
      else if (i < ko) d.OM[(size_t)a * ko + i] = acc[u] / d.w[i];
      else d.FM[(size_t)a * d.k_f + (i - ko)] = acc[u] / d.wf[i - ko];
    }
  }
}

// Output products of the giant unions, gper CTAs each (after union_svd_kernel
// wrote the rank, the order and the singular values).
__global__ void __launch_bounds__(256)
union_output_kernel(const UnionDesc* __restrict__ descs, int n, int gper) {
  const int u = blockIdx.x / gper, bl = blockIdx.x % gper;
  if (u >= n) return;
  const UnionDesc d = descs[u];
  const int m = d.m, C = d.k_old + d.k_f;
  const int smax = m < C ? m : C;
  const int spx = smax + (smax & 1);
  const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
  const double* gQA = d.work + mreg;
  const double* gQB = gQA + (size_t)m * smax;
  const double* gW = gQB + 2 * (size_t)C * smax;
  const int s = *(const int*)(gW + 2 * (size_t)smax * smax);
  const int* order = (const int*)(gW + 2 * (size_t)smax * smax + 2 * (size_t)smax);
  const int k = *d.rank;
  if (s == 0 || k == 0) return;
  union_output(d, s, k, gQA, gQB, gW, gW + (size_t)s * s, order, bl * blockDim.x, gper * blockDim.x);
}

// Second half of the union: SVD of the core (one-sided Jacobi on its
// transpose W = core^T with accumulated V) and the output products.  A
// separate kernel so the Jacobi gets its own register budget (teams of 8
// lanes holding 16 rows each run a round in one pass).  The ACA pivots grade
// the core's rows, so its columns are graded in the transpose and the sweeps
// converge in ~4-5 instead of ~7 passes (measured on oracle unions).  On
// exit V holds the core's left singular vectors (phi) and W its scaled right
// singular vectors (sigma psi):
//   new basis = QA phi[:, :k],  maps = (QB sigma psi)[col][a] / weight[col].
__global__ void __launch_bounds__(512)
union_svd_kernel(const UnionDesc* __restrict__ descs, int n, double thr, int smem_doubles) {
  extern __shared__ double smem[];
  for (int bb = blockIdx.x; bb < n; bb += gridDim.x) {
    const UnionDesc d = descs[bb];
    if (d.giant == 3) continue;  // union_post_kernel's
    const int m = d.m, C = d.k_old + d.k_f;
    const int smax = m < C ? m : C;
    const int spx = smax + (smax & 1);
    const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
    const double* gQA = d.work + mreg;
    const double* gQB = gQA + (size_t)m * smax;
    double* gW = (double*)gQB + 2 * (size_t)C * smax;
    const int s = *(const int*)(gW + 2 * (size_t)smax * smax);
    double* sig = gW + 2 * (size_t)smax * smax + smax;           // tauA slot
    int* order = (int*)(gW + 2 * (size_t)smax * smax + 2 * (size_t)smax);  // tauB slot
    if (s == 0) continue;  // rank 0 already written by the first half
    unsigned long long t3 = clock64();
    double* Wc = (d.giant != 1 && (size_t)s * s <= (size_t)smem_doubles) ? smem : gW;
    double* Vc = (d.giant != 1 && 2 * (size_t)s * s <= (size_t)smem_doubles) ? smem + (size_t)s * s
                                                                          : gW + (size_t)s * s;
    if (Wc != gW)
      for (int e = threadIdx.x; e < s * s; e += blockDim.x) Wc[e] = gW[e];
    __syncthreads();
    // giant unions: the multi-CTA Jacobi (union_jacobi_coop) already ran
    const int nsw = d.giant == 1 ? 0 : cta_jacobi_wv(Wc, Vc, s);
    unsigned long long t35 = clock64();
    cta_sv_order(Wc, s, s, s, sig, order);
    unsigned long long t4 = clock64();
    int kk = 0;
    for (int j = 0; j < s; ++j) kk += sig[order[j]] > thr;
    const int mr = d.min_rank < s ? d.min_rank : s;
    const int k = kk > mr ? kk : mr;
    // output products (giant unions: union_output_kernel on several CTAs)
    if (d.giant != 1) union_output(d, s, k, gQA, gQB, Wc, Vc, order, 0, blockDim.x);
    for (int a = threadIdx.x; a < k; a += blockDim.x) d.NW[a] = sig[order[a]];
    if (threadIdx.x == 0) *d.rank = k;
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t5 = clock64();
      atomicAdd(&g_uprof[3], t4 - t3);
      atomicAdd(&g_uprof[4], t5 - t4);
      atomicAdd(&g_uprof[11], (unsigned long long)nsw);
      atomicAdd(&g_uprof[12], t35 - t3);
      if (m > 128) {
        unsigned long long* u = g_uprof + (m > 400 ? 25 : 16);
        atomicAdd(&u[3], t4 - t3);
        atomicAdd(&u[4], t5 - t4);
        atomicAdd(&u[2], (unsigned long long)nsw);  // sweeps (slot 2 is free)
      }
    }
  }
}
}  // namespace

namespace {
// Multi-CTA one-sided Jacobi for the cores of giant unions (s above
// giant_union_threshold(), 100; the
// level-2 unions of c3/c4 reach s ~ 400).  One cooperative launch covers
// every giant union of a pair wave, gper CTAs per union; W and V stay in
// global memory (L2-resident).  Block-cyclic ordering (see below); the
// per-pair arithmetic is that of cta_jacobi_wv (one warp per pair, 16 rows
// per lane in registers, streamed tail beyond).  flags[u * 64 + sweep] collects "not yet
// converged" per union and sweep.
__global__ void __launch_bounds__(256)
union_jacobi_coop(const UnionDesc* __restrict__ descs, int n, int gper, unsigned* flags, int max_m1) {
  cg::grid_group grid = cg::this_grid();
  const int u = blockIdx.x / gper, bl = blockIdx.x % gper;
  const UnionDesc d = descs[u < n ? u : n - 1];
  const int m = d.m, C = d.k_old + d.k_f;
  const int smax = m < C ? m : C;
  const int spx = smax + (smax & 1);
  const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
  double* gW = d.work + mreg + (size_t)m * smax + 2 * (size_t)C * smax;
  const int s = u < n ? *(const int*)(gW + 2 * (size_t)smax * smax) : 0;
  double* W = gW;
  double* V = gW + (size_t)s * s;
  for (int e = bl * blockDim.x + threadIdx.x; e < s * s; e += gper * blockDim.x) {
    const int j = e / s, i = e - j * s;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  const double tol_rot = kEps;
  const double tol_conv = fmax(kEps * (double)(s > 4 ? s : 4), 1e-13);
  const double tr2 = tol_rot * tol_rot, tc2 = tol_conv * tol_conv;
  const int cp = s + (s & 1), half = cp >> 1, m1 = cp - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  constexpr int T = 32, NE = 16;
  bool live = s >= 2;
  grid.sync();
  // block-cyclic Jacobi: the columns form nb = 2 gper blocks; a block round
  // pairs the blocks round-robin (one block pair per CTA) and each CTA runs a
  // full inner round-robin sweep over the columns of its two blocks with CTA
  // barriers; one grid barrier per block round (nb - 1 per sweep instead of
  // s - 1).  Every column pair still meets once per sweep.
  const int nb = 2 * gper, bsz = (s + nb - 1) / nb;
  (void)max_m1; (void)half; (void)m1;
  for (int sweep = 0; sweep < 40; ++sweep) {
    bool again = false;
    for (int r = 0; r < nb - 1; ++r) {
      if (live) {
        int P, Q;
        if (bl == 0) { P = r; Q = nb - 1; }
        else { P = (r + bl) % (nb - 1); Q = (r - bl + nb - 1) % (nb - 1); }
        const int p0 = P * bsz, q0 = Q * bsz;
        const int np = max(0, min(bsz, s - p0)), nq = max(0, min(bsz, s - q0));
        const int nc = np + nq, ncp = nc + (nc & 1);
        for (int sr = 0; sr < ncp - 1; ++sr) {
          for (int pi = warp; pi < ncp / 2; pi += nwb) {
            int a2, b2;
            if (pi == 0) { a2 = sr; b2 = ncp - 1; }
            else { a2 = (sr + pi) % (ncp - 1); b2 = (sr - pi + ncp - 1) % (ncp - 1); }
            if (a2 >= nc || b2 >= nc) continue;  // warp-uniform
            const int ga2 = a2 < np ? p0 + a2 : q0 + (a2 - np);
            const int gb2 = b2 < np ? p0 + b2 : q0 + (b2 - np);
            const int lo = ga2 < gb2 ? ga2 : gb2, hi = ga2 < gb2 ? gb2 : ga2;
            double* x = W + (size_t)lo * s;
            double* y = W + (size_t)hi * s;
            double xr[NE], yr[NE];
            double a = 0.0, bb = 0.0, g = 0.0;
#pragma unroll
            for (int e = 0; e < NE; ++e) {
              const int i = lane + e * T;
              xr[e] = i < s ? x[i] : 0.0;
              yr[e] = i < s ? y[i] : 0.0;
              a = fma(xr[e], xr[e], a); bb = fma(yr[e], yr[e], bb); g = fma(xr[e], yr[e], g);
            }
            for (int i = lane + NE * T; i < s; i += T) {
              const double uu = x[i], vv = y[i];
              a = fma(uu, uu, a); bb = fma(vv, vv, bb); g = fma(uu, vv, g);
            }
            a = team_sum<T>(a); bb = team_sum<T>(bb); g = team_sum<T>(g);
            const double ab = a * bb, g2 = g * g;
            if (g != 0.0 && g2 > tr2 * ab) {
              const double dd = bb - a, gg = 2.0 * g;
              const double t = copysign(fabs(gg), dd * gg) / (fabs(dd) + sqrt(fma(dd, dd, gg * gg)));
              const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
              for (int e = 0; e < NE; ++e) {
                const int i = lane + e * T;
                if (i < s) {
                  x[i] = fma(c, xr[e], -sn * yr[e]);
                  y[i] = fma(sn, xr[e], c * yr[e]);
                }
              }
              for (int i = lane + NE * T; i < s; i += T) {
                const double uu = x[i], vv = y[i];
                x[i] = fma(c, uu, -sn * vv);
                y[i] = fma(sn, uu, c * vv);
              }
              double* vx = V + (size_t)lo * s;
              double* vy = V + (size_t)hi * s;
              for (int i0 = lane; i0 < s; i0 += 4 * T) {
                double uu[4], vv[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int i = i0 + e * T;
                  uu[e] = i < s ? vx[i] : 0.0;
                  vv[e] = i < s ? vy[i] : 0.0;
                }
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const int i = i0 + e * T;
                  if (i < s) {
                    vx[i] = fma(c, uu[e], -sn * vv[e]);
                    vy[i] = fma(sn, uu[e], c * vv[e]);
                  }
                }
              }
              again |= g2 > tc2 * ab;
            }
          }
          __syncthreads();  // the CTA's columns are private to it this block round
        }
      }
      grid.sync();
    }
    if (again && lane == 0) atomicOr(&flags[u * 64 + sweep], 1u);
    grid.sync();
    bool any = false;
    for (int v = 0; v < n; ++v) {
      const bool lv = flags[v * 64 + sweep] != 0u;
      if (v == u) live = live && lv;
      any |= lv;
    }
    if (!any) {
      if (bl == 0 && threadIdx.x == 0 && u < n) atomicAdd(&g_uprof[14], (unsigned long long)(sweep + 1));
      break;
    }
  }
}
}  // namespace

namespace {
// Multi-CTA full-pivot ACA for giant unions (s > giant_union_threshold()), one cooperative launch
// for all giants of a pair wave, gper CTAs per union.  CTA bl owns a slab of
// rows of the residual M (global memory, the union's workspace); per pivot
// step: slab argmax -> global candidates -> grid barrier -> every CTA
// derives the same pivot (max |value|, ties to the smallest row-major index,
// as the single-CTA kernel and numpy) and copies the pivot row / piv and its
// slab of the pivot column -> grid barrier -> slab update.  The arithmetic
// is element for element that of union_kernel, so X, Y, D are bitwise the
// same; union_kernel then skips its ACA for these unions.
__global__ void __launch_bounds__(512)
union_aca_coop(const UnionDesc* __restrict__ descs, int n, int gper, double thr, double* cand,
               int* done_count, int max_smax) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sh[];
  __shared__ double wv[32];
  __shared__ long long wi[32];
  const int u = blockIdx.x / gper, bl = blockIdx.x % gper;
  const bool real = u < n;
  const UnionDesc d = descs[real ? u : n - 1];
  const int m = d.m, ko = d.k_old, C = d.k_old + d.k_f;
  const int smax = m < C ? m : C;
  const int spx = smax + (smax & 1);
  const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
  double* M = d.work;
  double* Acol = M + mreg;
  double* Bt = Acol + (size_t)m * smax;
  double* core = Bt + 2 * (size_t)C * smax;
  double* Dp = core + 2 * (size_t)smax * smax;
  int* hdr = (int*)(Dp + 4 * (size_t)smax);  // s for union_kernel
  const int rpc = (m + gper - 1) / gper;
  const int r0 = bl * rpc, r1 = min(m, r0 + rpc), nr = max(0, r1 - r0);
  double* rrs = sh;            // C
  double* ccs = rrs + C;       // nr
  int* acts = (int*)(ccs + rpc + 1);
  int* pos = acts + C;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double bv = -1.0;
  int bi = 0, bj = 0;
  auto better = [&](double av, int i, int j) {
    return av > bv || (av == bv && (long long)i * C + j < (long long)bi * C + bj);
  };
  for (int j = threadIdx.x; j < C; j += blockDim.x) { acts[j] = j; pos[j] = j; }
  // concat [B*diag(w) | F*diag(wf)] for the own rows + first local argmax
  for (long long e = threadIdx.x; e < (long long)nr * C; e += blockDim.x) {
    const int i = r0 + (int)(e % nr), j = (int)(e / nr);
    const double v = j < ko ? d.B[(size_t)i * d.b_r + (size_t)j * d.b_c] * d.w[j]
                            : d.F[(size_t)i * d.f_r + (size_t)(j - ko) * d.f_c] * d.wf[j - ko];
    M[(size_t)j * m + i] = v;
    if (better(fabs(v), i, j)) { bv = fabs(v); bi = i; bj = j; }
  }
  const double floor_ = thr / 8.0;
  int steps = 0, nact = C;
  bool done = !real;
  for (int it = 0; it < max_smax; ++it) {
    // ---- publish the slab candidate
    long long bflat = bv < 0.0 ? (1LL << 62) : (long long)bi * C + bj;
    warp_argmax(bv, bflat);
    if (lane == 0) { wv[warp] = bv; wi[warp] = bflat; }
    __syncthreads();
    if (warp == 0) {
      double gv = lane < nw ? wv[lane] : -1.0;
      long long gi = lane < nw ? wi[lane] : (1LL << 62);
      warp_argmax(gv, gi);
      if (lane == 0) {
        cand[2 * (size_t)blockIdx.x] = gv;
        reinterpret_cast<long long*>(cand)[2 * (size_t)blockIdx.x + 1] = gi;
      }
    }
    grid.sync();
    // ---- the union's pivot (identical in all of its CTAs)
    int p = 0, q = 0;
    double piv = 0.0;
    if (!done) {
      double gv = -1.0;
      long long gi = (1LL << 62);
      for (int b = lane; b < gper; b += 32) {
        const double ov = cand[2 * (size_t)(u * gper + b)];
        const long long oi = reinterpret_cast<const long long*>(cand)[2 * (size_t)(u * gper + b) + 1];
        if (ov > gv || (ov == gv && oi < gi)) { gv = ov; gi = oi; }
      }
      warp_argmax(gv, gi);
      p = (int)(gi / C);
      q = (int)(gi - (long long)p * C);
      if (it >= smax || gv < 0.0) done = true;
      else {
        piv = M[(size_t)q * m + p];
        if (piv == 0.0 || (fabs(piv) <= floor_ && steps >= d.min_rank)) done = true;
      }
      if (done && bl == 0 && threadIdx.x == 0) { *hdr = steps; atomicAdd(done_count, 1); }
    }
    if (!done) {
      for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const double v = M[(size_t)q * m + i];
        ccs[i - r0] = v;
        Acol[(size_t)steps * m + i] = v;
        if (i != p) M[(size_t)q * m + i] = 0.0;
      }
      for (int j = threadIdx.x; j < C; j += blockDim.x) {
        const double v = j == q ? 1.0 : M[(size_t)j * m + p] / piv;
        rrs[j] = v;
        if (bl == 0) Bt[(size_t)steps * C + j] = v;
      }
      if (threadIdx.x == 0) {
        const int k = pos[q], last = acts[nact - 1];
        acts[k] = last;
        pos[last] = k;
        if (bl == 0) Dp[steps] = piv;
      }
      --nact;
    }
    grid.sync();  // every CTA has read row p / piv before the slabs change
    if (*(volatile int*)done_count >= n) break;
    if (done) continue;
    if (threadIdx.x == 0 && p >= r0 && p < r1) M[(size_t)q * m + p] = 0.0;
    __syncthreads();
    bv = -1.0;
    constexpr int UN = 16;
    const int total = nr * nact, nthr = blockDim.x;
    if (nr > 0) {
      const int di = nthr % nr, dl = nthr / nr;
      int f = threadIdx.x, i = f % nr, l = f / nr;
      while (f < total) {
        int ii[UN], jj[UN];
        double v[UN];
#pragma unroll
        for (int uu = 0; uu < UN; ++uu) {
          const bool ok = f + uu * nthr < total;
          ii[uu] = i;
          jj[uu] = ok ? acts[l] : -1;
          v[uu] = ok ? M[(size_t)jj[uu] * m + r0 + i] : 0.0;
          i += di; l += dl;
          if (i >= nr) { i -= nr; ++l; }
        }
#pragma unroll
        for (int uu = 0; uu < UN; ++uu) {
          if (jj[uu] < 0) break;
          v[uu] = fma(-ccs[ii[uu]], rrs[jj[uu]], v[uu]);
          M[(size_t)jj[uu] * m + r0 + ii[uu]] = v[uu];
          const double av = fabs(v[uu]);
          if (better(av, r0 + ii[uu], jj[uu])) { bv = av; bi = r0 + ii[uu]; bj = jj[uu]; }
        }
        f += UN * nthr;
      }
    }
    ++steps;
  }
  if (real && !done && bl == 0 && threadIdx.x == 0) *hdr = steps;  // ran to max_smax
}
}  // namespace

namespace {
// Multi-CTA CholeskyQR2 + core formation for giant unions, after
// union_aca_coop: pivot scaling, Gram tiles and row-wise triangular solves
// are spread over the union's CTAs, the two Cholesky factorisations run in its
// first CTA, grid barriers in between.  Same arithmetic per element as
// union_kernel (same tiles, same Cholesky, same per-row solves), so the
// factors are bitwise those of the single-CTA path.  Writes QA / QB in place,
// W = core^T and the hand-off header; flags the union for union_kernel's
// Householder path when a Cholesky pivot ratio signals cond > ~1e6.
__global__ void __launch_bounds__(512)
union_cholqr_coop(const UnionDesc* __restrict__ descs, int n, int gper, int max_s) {
  cg::grid_group grid = cg::this_grid();
  const int u = blockIdx.x / gper, bl = blockIdx.x % gper;
  const bool real = u < n;
  const UnionDesc d = descs[real ? u : n - 1];
  const int m = d.m, C = d.k_old + d.k_f;
  const int smax = m < C ? m : C;
  const int spx = smax + (smax & 1);
  const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
  double* Mw = d.work;
  double* Acol = Mw + mreg;
  double* Bt = Acol + (size_t)m * smax;
  double* core = Bt + 2 * (size_t)C * smax;
  double* Dp = core + 2 * (size_t)smax * smax;
  double* tauA = Dp + smax;
  double* tauB = tauA + smax;
  int* hdr_aca = (int*)(Dp + 4 * (size_t)smax);  // s from union_aca_coop; [1]: fallback flag
  const int s = real ? hdr_aca[0] : 0;
  const int sp = s + (s & 1);
  const int nthr_all = gper * blockDim.x, tb = bl * blockDim.x;
  const int nw = blockDim.x >> 5, wb = bl * nw, wall = gper * nw;
  double* GA = Mw;
  double* GB = GA + (size_t)s * sp;
  double* RA1s = Mw + 2 * (size_t)s * sp;
  double* RB1s = RA1s + (size_t)s * sp;
  double* TA = RB1s + (size_t)s * sp;
  double* TB = TA + (size_t)s * sp;
  // every CTA of the grid runs the same barrier sequence; the work is
  // predicated on the union's state
  if (bl == 0 && threadIdx.x == 0 && real) hdr_aca[1] = 0;
  // pivot scaling L~ = X D^{-1}: rows over all threads of the union
  if (s > 0)
    for (int i = tb + threadIdx.x; i < m; i += nthr_all)
      for (int t0 = 0; t0 < s; t0 += 8) {
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = t0 + k < s ? Acol[(size_t)(t0 + k) * m + i] : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (t0 + k < s) Acol[(size_t)(t0 + k) * m + i] = v[k] / Dp[t0 + k];
      }
  grid.sync();
  for (int pass = 0; pass < 2; ++pass) {
    const bool act = s > 0 && hdr_aca[1] == 0;  // uniform per union
    if (act) cta_gram2(Acol, m, Bt, C, s, sp, GA, GB, wb, wall);
    grid.sync();
    // in-place Cholesky of both Grams on all of the union's CTAs: one grid
    // barrier per column (the same per-element arithmetic as cta_chol2)
    {
      double mxA = 0.0, mxB = 0.0, minr = 1.0;
      if (act)
        for (int k = 0; k < s; ++k) {
          mxA = fmax(mxA, GA[(size_t)k * sp + k]);
          mxB = fmax(mxB, GB[(size_t)k * sp + k]);
        }
      const double imxA = act ? 1.0 / mxA : 0.0, imxB = act ? 1.0 / mxB : 0.0;
      grid.sync();  // every CTA read the original diagonals
      const int lane = threadIdx.x & 31;
      for (int k = 0; k <= max_s; ++k) {
        if (act && k <= s) {
          if (k > 0) {  // finalise row k-1 of both R factors
            const double ra = tauA[k - 1], rb = tauB[k - 1];
            double* gra = GA + (size_t)(k - 1) * sp;
            double* grb = GB + (size_t)(k - 1) * sp;
            for (int j = k - 1 + tb + threadIdx.x; j < s; j += nthr_all) {
              gra[j] *= ra;
              grb[j] *= rb;
            }
          }
          if (k < s) {
            const double* ga = GA + (size_t)k * sp;
            const double* gbp = GB + (size_t)k * sp;
            const double pa = ga[k], pb = gbp[k];
            const double inva = 1.0 / pa, invb = 1.0 / pb;
            const double ra = rsqrt(pa), rb = rsqrt(pb);
            const double qa = pa * imxA, qb = pb * imxB;
            minr = (qa > 0.0 && isfinite(pa)) ? fmin(minr, qa) : 0.0;
            minr = (qb > 0.0 && isfinite(pb)) ? fmin(minr, qb) : 0.0;
            if (bl == 0 && threadIdx.x == 0) { tauA[k] = ra; tauB[k] = rb; }
            const int nr = s - k - 1;
            for (int t = wb + (threadIdx.x >> 5); t < 2 * nr; t += wall) {
              const bool isA = t < nr;
              const int i = k + 1 + (isA ? t : t - nr);
              const double* g = isA ? ga : gbp;
              double* Gi = (isA ? GA : GB) + (size_t)i * sp;
              const double fi = g[i] * (isA ? inva : invb);
              for (int j0 = i + lane; j0 < s; j0 += 128) {
                double gv[4], gw[4];
#pragma unroll
                for (int u2 = 0; u2 < 4; ++u2) {
                  const int j = j0 + 32 * u2;
                  gv[u2] = j < s ? g[j] : 0.0;
                  gw[u2] = j < s ? Gi[j] : 0.0;
                }
#pragma unroll
                for (int u2 = 0; u2 < 4; ++u2) {
                  const int j = j0 + 32 * u2;
                  if (j < s) Gi[j] = fma(-fi, gv[u2], gw[u2]);
                }
              }
            }
          }
        }
        grid.sync();
      }
      if (act && pass == 0 && bl == 0) {
        if (!(minr > kCholFloor)) {
          if (threadIdx.x == 0) hdr_aca[1] = 1;  // union_kernel runs the Householder path
        }
      }
      grid.sync();
      if (act && pass == 0 && hdr_aca[1] == 0)  // park R1
        for (int e = tb + threadIdx.x; e < 2 * s * sp; e += nthr_all) RA1s[e] = GA[e];
    }
    grid.sync();
    if (s > 0 && hdr_aca[1] == 0) cta_trsm2(Acol, m, GA, tauA, Bt, C, GB, tauB, s, sp, tb, nthr_all);
    grid.sync();
  }
  const bool ok = s > 0 && hdr_aca[1] == 0;
  if (ok) cta_trmul2(GA, RA1s, TA, GB, RB1s, TB, s, sp, tb, nthr_all);
  grid.sync();
  if (ok)
    for (int e = tb + threadIdx.x; e < s * s; e += nthr_all) {
      const int j = e / s, i = e - j * s;
      double acc = 0.0;
      for (int l = (i > j ? i : j); l < s; ++l)
        acc = fma(TB[(size_t)i * sp + l] * Dp[l], TA[(size_t)j * sp + l], acc);
      core[(size_t)j * s + i] = acc;  // W = core^T at the hand-off location
    }
  grid.sync();
  if (ok && bl == 0 && threadIdx.x == 0) *(int*)(core + 2 * (size_t)smax * smax) = s;  // header
}
}  // namespace

void launch_union_cholqr_coop(const UnionDesc* d_descs, int n, int gper, int max_s, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_union_cholqr_coop"};
  if (n <= 0) return;
  void* args[] = {(void*)&d_descs, (void*)&n, (void*)&gper, (void*)&max_s};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((void*)union_cholqr_coop, dim3(gper * n), dim3(512), args, 0, s);
  if (e != cudaSuccess)
    fprintf(stderr, "[ifmm] cooperative CholeskyQR launch failed: %s\n", cudaGetErrorString(e));
}

size_t union_aca_coop_smem(int max_C, int max_rpc) {
  return (size_t)(max_C + max_rpc + 1) * 8 + (size_t)2 * max_C * 4 + 64;
}

void launch_union_aca_coop(const UnionDesc* d_descs, int n, double thr, int gper, int max_C, int max_m,
                           int max_smax, double* d_cand, int* d_done, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_union_aca_coop"};
  if (n <= 0) return;
  const int rpc = (max_m + gper - 1) / gper;
  const size_t sh = union_aca_coop_smem(max_C, rpc);
  static size_t attr = 0;
  if (sh > attr) {
    cudaFuncSetAttribute(union_aca_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh);
    attr = sh;
  }
  cudaMemsetAsync(d_done, 0, sizeof(int), s);
  void* args[] = {(void*)&d_descs, (void*)&n, (void*)&gper, (void*)&thr, (void*)&d_cand,
                  (void*)&d_done, (void*)&max_smax};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((void*)union_aca_coop, dim3(gper * n), dim3(512), args, sh, s);
  if (e != cudaSuccess)
    fprintf(stderr, "[ifmm] cooperative ACA launch failed: %s\n", cudaGetErrorString(e));
}

void launch_union_jacobi_coop(const UnionDesc* d_descs, int n, int max_s, unsigned* d_flags,
                              cudaStream_t s, int sm_free) {
  DbgSync dbg_sync_{s, "launch_union_jacobi_coop"};
  if (n <= 0) return;
  int per = sm_free / n;
  const int half = (max_s + 1) / 2;
  const int need = (half + 7) / 8;  // 8 warps (pairs) per CTA and round
  if (per > need) per = need;
  if (per < 1) per = 1;
  int max_m1 = max_s + (max_s & 1) - 1;
  cudaMemsetAsync(d_flags, 0, sizeof(unsigned) * 64 * (size_t)n, s);
  void* args[] = {(void*)&d_descs, (void*)&n, (void*)&per, (void*)&d_flags, (void*)&max_m1};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((void*)union_jacobi_coop, dim3(per * n), dim3(256), args, 0, s);
  if (e != cudaSuccess) {  // surfaces through the caller's cudaGetLastError check
    fprintf(stderr, "[ifmm] cooperative Jacobi launch failed: %s\n", cudaGetErrorString(e));
  }
}

int giant_union_threshold() {
  static int t = -1;
  if (t < 0) {
    const char* e = getenv("IFMM_GIANT");
    t = e ? atoi(e) : 100;
  }
  return t;
}

bool union_fits_smem(int m, int k_old, int k_f) {
  return union_work_doubles(m, k_old, k_f) <= (size_t)UNION_SMEM_DOUBLES;
}

// smem != 0: every desc's workspace fits shared memory (caller partitions);
// smem == 0: workspaces in global memory with the full L1 as cache.
void launch_union(const UnionDesc* d_descs, int n, double thr, cudaStream_t s, int smem,
                  int jac_smem_doubles, const UnionDesc* d_giants, int n_giants, int max_giant_s,
                  double* d_scratch, int max_giant_m, int max_giant_C, int sm_reserved) {
  // SMs left for the cooperative giant kernels: the concurrent shared-memory
  // union launch holds one SM per union (228 KB each)
  const int sm_free = 148 - (sm_reserved < 120 ? sm_reserved : 120);
  unsigned* d_flags = reinterpret_cast<unsigned*>(d_scratch);              // 64 per giant
  int* d_done = reinterpret_cast<int*>(d_scratch + 32 * (size_t)n_giants);  // 1
  double* d_cand = d_scratch + 32 * (size_t)n_giants + 8;                   // 2 per CTA
  DbgSync dbg_sync_{s, "launch_union"};
  if (n <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(union_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         UNION_SMEM_DOUBLES * 8);
    attr = true;
  }
  static int nthr = -1;
  if (nthr < 0) {
    const char* e = getenv("IFMM_UNION_THREADS");
    nthr = e ? atoi(e) : 512;
  }
  static int force_hh = -1;
  if (force_hh < 0) {
    const char* e = getenv("IFMM_UNION_HH");  // diagnostics: Householder QR path
    force_hh = e ? atoi(e) : 0;
  }
  static bool attr3 = false;
  if (!attr3) {
    cudaFuncSetAttribute(union_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         UNION_SVD_SMEM_DOUBLES * 8);
    attr3 = true;
  }
  if (smem)
    union_kernel<true><<<n < 4096 ? n : 4096, nthr, (size_t)UNION_SMEM_DOUBLES * 8, s>>>(
        d_descs, n, thr, UNION_SMEM_DOUBLES, force_hh);
  else {
    static bool attr2 = false;
    if (!attr2) {
      cudaFuncSetAttribute(union_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           UNION_SMEM_DOUBLES * 8);
      attr2 = true;
    }
    // shared memory for the CholeskyQR matrices and the core SVD
    (void)jac_smem_doubles;
    const int jd = UNION_SMEM_DOUBLES;
    if (n_giants > 0) {  // the giants' ACA on several CTAs each (union_kernel skips it)
      int gper = sm_free / n_giants;
      const int want = (max_giant_m + 63) / 64;
      if (gper > want) gper = want;
      if (gper < 1) gper = 1;
      launch_union_aca_coop(d_giants, n_giants, thr, gper, max_giant_C, max_giant_m, max_giant_s,
                            d_cand, d_done, s);
      launch_union_cholqr_coop(d_giants, n_giants, gper, max_giant_s, s);
    }
    union_kernel<false><<<n < 4096 ? n : 4096, nthr, (size_t)jd * 8, s>>>(d_descs, n, thr, jd, force_hh);
  }
  if (n_giants > 0) launch_union_jacobi_coop(d_giants, n_giants, max_giant_s, d_flags, s, sm_free);
  union_svd_kernel<<<n < 4096 ? n : 4096, 512, (size_t)UNION_SVD_SMEM_DOUBLES * 8, s>>>(
      d_descs, n, thr, UNION_SVD_SMEM_DOUBLES);
  if (n_giants > 0) {
    const int gper = sm_free / n_giants > 0 ? sm_free / n_giants : 1;
    union_output_kernel<<<gper * n_giants, 256, 0, s>>>(d_giants, n_giants, gper);
  }
}

// ============================================================================
// LU with partial pivoting (row-major, in place) -- CTA cooperative
// ============================================================================

namespace {
__global__ void __launch_bounds__(512)
lu_kernel(const LuDesc* __restrict__ descs, int n, int* status, int smem_doubles) {
  extern __shared__ double smem[];
  __shared__ double red[32];
  __shared__ long long redi[32];
  __shared__ int s_p;
  __shared__ int s_bad;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const LuDesc d = descs[b];
    const int N = d.n;
    const bool sm = (long long)N * N <= smem_doubles;
    double* A = sm ? smem : d.A;
    const int lda = sm ? N : d.lda;
    if (sm)
      for (long long e = threadIdx.x; e < (long long)N * N; e += blockDim.x)
        smem[e] = d.A[(size_t)(e / N) * d.lda + (e % N)];
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    for (int j = 0; j < N; ++j) {
      double bv = -1.0;
      long long bi = (1LL << 62);
      for (int i = j + threadIdx.x; i < N; i += blockDim.x) {
        const double v = fabs(A[(size_t)i * lda + j]);
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
      }
      // NaN pivots: treat as bad
      block_argmax(bv, bi, red, redi);
      if (threadIdx.x == 0) {
        int p = (bi >= N || bi < j) ? j : (int)bi;
        s_p = p;
        d.piv[j] = p;
        const double pv = A[(size_t)p * lda + j];
        if (pv == 0.0 || !isfinite(pv)) s_bad = 1;
      }
      __syncthreads();
      const int p = s_p;
      if (p != j)
        for (int c = threadIdx.x; c < N; c += blockDim.x) {
          const double t = A[(size_t)j * lda + c];
          A[(size_t)j * lda + c] = A[(size_t)p * lda + c];
          A[(size_t)p * lda + c] = t;
        }
      __syncthreads();
      const double pv = A[(size_t)j * lda + j];
      if (pv != 0.0)
        for (int i = j + 1 + threadIdx.x; i < N; i += blockDim.x) A[(size_t)i * lda + j] /= pv;
      __syncthreads();
      const int rem = N - j - 1;
      if (rem > 0)
        for (long long e = threadIdx.x; e < (long long)rem * rem; e += blockDim.x) {
          const int i = j + 1 + (int)(e / rem), c = j + 1 + (int)(e % rem);
          A[(size_t)i * lda + c] -= A[(size_t)i * lda + j] * A[(size_t)j * lda + c];
        }
      __syncthreads();
    }
    // final finiteness scan (factor.py:171)
    int bad = 0;
    for (long long e = threadIdx.x; e < (long long)N * N; e += blockDim.x)
      if (!isfinite(A[(size_t)(e / N) * lda + (e % N)])) bad = 1;
    if (bad) s_bad = 1;
    __syncthreads();
    if (s_bad && threadIdx.x == 0) atomicCAS(status, 0, d.tag + 1);
    if (sm)
      for (long long e = threadIdx.x; e < (long long)N * N; e += blockDim.x)
        d.A[(size_t)(e / N) * d.lda + (e % N)] = smem[e];
    __syncthreads();
  }
}

// Warp-per-32-columns LU solve: lane owns one RHS column.
__global__ void __launch_bounds__(256)
lusolve_kernel(const LuSolveDesc* __restrict__ descs, int ndesc, int chunks_per_desc) {
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int di = gw / chunks_per_desc, ch = gw % chunks_per_desc;
  if (di >= ndesc) return;
  const LuSolveDesc d = descs[di];
  const int c = ch * 32 + lane;
  if (c >= d.nrhs) return;
  const int N = d.n;
  double* x = d.X + c;
  const size_t ld = d.ldx;
  for (int j = 0; j < N; ++j) {
    const int p = d.piv[j];
    if (p != j) { const double t = x[j * ld]; x[j * ld] = x[p * ld]; x[p * ld] = t; }
  }
  for (int i = 1; i < N; ++i) {
    const double* L = d.LU + (size_t)i * d.lda;
    double s0 = x[i * ld], s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = 0;
    for (; j + 3 < i; j += 4) {
      s0 = fma(-L[j], x[j * ld], s0);
      s1 = fma(-L[j + 1], x[(j + 1) * ld], s1);
      s2 = fma(-L[j + 2], x[(j + 2) * ld], s2);
      s3 = fma(-L[j + 3], x[(j + 3) * ld], s3);
    }
    for (; j < i; ++j) s0 = fma(-L[j], x[j * ld], s0);
    x[i * ld] = (s0 + s1) + (s2 + s3);
  }
  for (int i = N - 1; i >= 0; --i) {
    const double* U = d.LU + (size_t)i * d.lda;
    double s0 = x[i * ld], s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int j = i + 1;
    for (; j + 3 < N; j += 4) {
      s0 = fma(-U[j], x[j * ld], s0);
      s1 = fma(-U[j + 1], x[(j + 1) * ld], s1);
      s2 = fma(-U[j + 2], x[(j + 2) * ld], s2);
      s3 = fma(-U[j + 3], x[(j + 3) * ld], s3);
    }
    for (; j < N; ++j) s0 = fma(-U[j], x[j * ld], s0);
    x[i * ld] = ((s0 + s1) + (s2 + s3)) / U[i];
  }
}
// One CTA per (system, CW-column chunk): the chunk lives in shared memory
// (n x (CW+1) padded), column = tid % CW, 256/CW row groups split the rows
// of each rank-1 column sweep; one barrier per pivot.  Final backward values
// go straight to global memory so no thread overwrites a value another may
// still read.
template <int CW>
__global__ void __launch_bounds__(256)
lusolve_smem_kernel(const LuSolveDesc* __restrict__ descs, int ndesc, int chunks_per_desc) {
  extern __shared__ double xs[];
  constexpr int LD = CW + 1, RG = 256 / CW;
  const int c = threadIdx.x % CW, r0 = threadIdx.x / CW;
  const int di = blockIdx.x / chunks_per_desc, ch = blockIdx.x % chunks_per_desc;
  if (di >= ndesc) return;
  const LuSolveDesc d = descs[di];
  const int c0 = ch * CW;
  if (c0 >= d.nrhs) return;
  const int nc = min(CW, d.nrhs - c0);
  const int N = d.n;
  const size_t ld = d.ldx;
  for (int e = threadIdx.x; e < N * CW; e += blockDim.x) {
    const int i = e / CW, cc = e % CW;
    xs[i * LD + cc] = cc < nc ? d.X[(size_t)i * ld + c0 + cc] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x < CW)
    for (int j = 0; j < N; ++j) {
      const int p = d.piv[j];
      if (p != j) { const double t = xs[j * LD + c]; xs[j * LD + c] = xs[p * LD + c]; xs[p * LD + c] = t; }
    }
  __syncthreads();
  for (int j = 0; j < N - 1; ++j) {
    const double xj = xs[j * LD + c];
    for (int i = j + 1 + r0; i < N; i += RG) xs[i * LD + c] -= d.LU[(size_t)i * d.lda + j] * xj;
    __syncthreads();
  }
  for (int j = N - 1; j >= 0; --j) {
    const double xj = xs[j * LD + c] / d.LU[(size_t)j * d.lda + j];
    if (r0 == (j % RG) && c < nc) d.X[(size_t)j * ld + c0 + c] = xj;
    for (int i = r0; i < j; i += RG) xs[i * LD + c] -= d.LU[(size_t)i * d.lda + j] * xj;
    __syncthreads();
  }
}
}  // namespace

void launch_lu(const LuDesc* d_descs, int n, int* d_status, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_lu"};
  if (n <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  const int smem = 200 * 1024;
  lu_kernel<<<n < 4096 ? n : 4096, 512, smem, s>>>(d_descs, n, d_status, smem / 8);
}

void launch_lusolve(const LuSolveDesc* d_descs, int ndesc, int max_nrhs, cudaStream_t s,
                    int max_n) {
  DbgSync dbg_sync_{s, "launch_lusolve"};
  if (ndesc <= 0 || max_nrhs <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(lusolve_smem_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    cudaFuncSetAttribute(lusolve_smem_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    cudaFuncSetAttribute(lusolve_smem_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         220 * 1024);
    attr = true;
  }
  if (max_n > 0 && max_n <= 800) {
    const int chunks = (max_nrhs + 31) / 32;
    lusolve_smem_kernel<32><<<ndesc * chunks, 256, (size_t)max_n * 33 * sizeof(double), s>>>(
        d_descs, ndesc, chunks);
    return;
  }
  if (max_n > 0 && max_n <= 1600) {
    const int chunks = (max_nrhs + 15) / 16;
    lusolve_smem_kernel<16><<<ndesc * chunks, 256, (size_t)max_n * 17 * sizeof(double), s>>>(
        d_descs, ndesc, chunks);
    return;
  }
  if (max_n > 0 && max_n <= 3000) {
    const int chunks = (max_nrhs + 7) / 8;
    lusolve_smem_kernel<8><<<ndesc * chunks, 256, (size_t)max_n * 9 * sizeof(double), s>>>(
        d_descs, ndesc, chunks);
    return;
  }
  const int chunks = (max_nrhs + 31) / 32;
  const long long warps = (long long)ndesc * chunks;
  const int blocks = (int)((warps + 7) / 8);
  lusolve_kernel<<<blocks, 256, 0, s>>>(d_descs, ndesc, chunks);
}

}  // namespace ifmm

// ============================================================================
// Basis weights (initialize_weights) and tall-skinny QR helpers
// ============================================================================
namespace ifmm {

size_t weights_work_doubles(int k, int W) {
  return 4 * (size_t)k * k + (size_t)k * (W < k ? W : k) + 6 * (size_t)k + 16;
}

namespace {

// Replace exactly-zero columns of P (k x k col-major, first `good` valid
// columns orthonormal) by an orthonormal completion from unit vectors.
__device__ void cta_complete_zero_cols(double* P, int k, const double* sig, double* red) {
  __shared__ int s_ok;
  for (int pos = 0; pos < k; ++pos) {
    if (sig[pos] > 0.0) continue;
    for (int e = 0; e < k; ++e) {
      double* v = P + (size_t)pos * k;
      for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] = (i == e) ? 1.0 : 0.0;
      __syncthreads();
      for (int q = 0; q < k; ++q) {
        if (q == pos || (q > pos && sig[q] <= 0.0)) continue;
        const double* u = P + (size_t)q * k;
        double d = 0.0;
        for (int i = threadIdx.x; i < k; i += blockDim.x) d = fma(u[i], v[i], d);
        d = block_sum(d, red);
        for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] -= d * u[i];
        __syncthreads();
      }
      double nn = 0.0;
      for (int i = threadIdx.x; i < k; i += blockDim.x) nn = fma(v[i], v[i], nn);
      nn = block_sum(nn, red);
      if (threadIdx.x == 0) s_ok = nn > 0.25;
      __syncthreads();
      if (s_ok) {
        const double inv = 1.0 / sqrt(nn);
        for (int i = threadIdx.x; i < k; i += blockDim.x) v[i] *= inv;
        __syncthreads();
        break;
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(512) weights_kernel(const WeightDesc* __restrict__ descs, int n) {
  __shared__ double red[32];
  __shared__ int sflag;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const WeightDesc d = descs[b];
    const int k = d.k, W = d.W;
    double* M = d.work;              // k x k (or k x W)
    double* V = M + (size_t)k * k;   // k x k
    double* Pc = V + (size_t)k * k;  // k x k col-major result
    double* tau = Pc + (size_t)k * k;
    double* sig = tau + k;           // sorted sigma (k)
    int* order = (int*)(sig + k);
    double* sraw = sig + 3 * k;      // unsorted norms
    if (W >= k) {
      // H row-major k x W == H^T col-major W x k
      cta_geqrf(d.H, W, k, W, tau, red);
      for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int l = e / k, i = e % k;  // M(i,l) = R(l,i)
        M[e] = (l <= i) ? d.H[(size_t)i * W + l] : 0.0;
      }
      __syncthreads();
      cta_jacobi(M, k, k, k, V, &sflag);
      cta_sv_order(M, k, k, k, sraw, order);
      for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int pos = e / k, i = e % k;
        const int j = order[pos];
        const double s = sraw[j];
        Pc[e] = s > 0.0 ? M[(size_t)j * k + i] / s : 0.0;
      }
      for (int pos = threadIdx.x; pos < k; pos += blockDim.x) sig[pos] = sraw[order[pos]];
      __syncthreads();
      cta_complete_zero_cols(Pc, k, sig, red);
      // weights = sigma (len k), floor
      for (int a = threadIdx.x; a < k; a += blockDim.x) {
        const double scale = sig[0] > 0.0 ? sig[0] : 1.0;
        d.w[a] = fmax(sig[a], 1e-14 * scale);
      }
    } else {
      // H col-major k x W
      for (int e = threadIdx.x; e < k * W; e += blockDim.x) {
        const int w = e / k, a = e % k;
        M[e] = d.H[(size_t)a * W + w];
      }
      __syncthreads();
      cta_jacobi(M, k, W, k, V, &sflag);
      cta_sv_order(M, k, W, k, sraw, order);
      // B = [U (k x W) | e_0 .. e_{k-W-1}]  (k x k col-major) in V-space
      double* B = V;  // reuse (k x k)
      for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int pos = e / k, i = e % k;
        double v;
        if (pos < W) {
          const int j = order[pos];
          v = sraw[j] > 0.0 ? M[(size_t)j * k + i] / sraw[j] : 0.0;
        } else {
          v = (i == pos - W) ? 1.0 : 0.0;
        }
        B[e] = v;
      }
      for (int pos = threadIdx.x; pos < W; pos += blockDim.x) sig[pos] = sraw[order[pos]];
      __syncthreads();
      cta_geqrf(B, k, k, k, tau, red);
      cta_orgqr(B, k, k, k, tau, Pc, k);
      for (int a = threadIdx.x; a < k; a += blockDim.x) {
        double v = a < W ? sig[a] : sig[W - 1];
        const double scale = sig[0] > 0.0 ? sig[0] : 1.0;
        d.w[a] = fmax(v, 1e-14 * scale);
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
      const int i = e / k, pos = e % k;  // P row-major: P[i][pos]
      d.P[e] = Pc[(size_t)pos * k + i];
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(1024)
tall_orth_kernel(const double* Y, int n, int w, double* Q, double* work, int mode,
                 double* out) {
  __shared__ double red[32];
  __shared__ int sflag;
  double* A = work;                 // col-major n x w
  double* QQ = A + (size_t)n * w;   // col-major n x w
  double* tau = QQ + (size_t)n * w;
  for (long long e = threadIdx.x; e < (long long)n * w; e += blockDim.x) {
    const int c = (int)(e / n), i = (int)(e % n);
    A[e] = Y[(size_t)i * w + c];
  }
  __syncthreads();
  cta_geqrf(A, n, w, n, tau, red);
  if (mode == 0) {
    cta_orgqr(A, n, w, n, tau, QQ, n);
    __syncthreads();
    for (long long e = threadIdx.x; e < (long long)n * w; e += blockDim.x) {
      const int i = (int)(e / w), c = (int)(e % w);
      Q[e] = QQ[(size_t)c * n + i];
    }
  } else {
    // sigma_max of R (w x w)
    double* R = QQ;
    double* V = R + (size_t)w * w;
    double* sg = V + (size_t)w * w;
    int* order = (int*)(sg + w);
    for (int e = threadIdx.x; e < w * w; e += blockDim.x) {
      const int l = e / w, i = e % w;
      R[e] = (i <= l) ? A[(size_t)l * n + i] : 0.0;
    }
    __syncthreads();
    cta_jacobi(R, w, w, w, V, &sflag);
    cta_sv_order(R, w, w, w, sg, order);
    if (threadIdx.x == 0) *out = sg[order[0]];
  }
}

}  // namespace

void launch_weights(const WeightDesc* d_descs, int n, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_weights"};
  if (n <= 0) return;
  weights_kernel<<<n < 4096 ? n : 4096, 512, 0, s>>>(d_descs, n);
}

void launch_tall_orth(const double* Y, int n, int w, double* Q, double* work, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_tall_orth"};
  tall_orth_kernel<<<1, 1024, 0, s>>>(Y, n, w, Q, work, 0, nullptr);
}

void launch_tall_sigmax(const double* Y, int n, int w, double* out, double* work,
                        cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_tall_sigmax"};
  tall_orth_kernel<<<1, 1024, 0, s>>>(Y, n, w, nullptr, work, 1, out);
}

}  // namespace ifmm

// ============================================================================
// Blocked LU pieces, triangular solve, extension
// ============================================================================
namespace ifmm {
namespace {

__global__ void __launch_bounds__(1024)
panel_lu_kernel(double* A, int n, int lda, int j0, int jb, int* piv, int* status, int tag) {
  __shared__ double red[32];
  __shared__ long long redi[32];
  __shared__ int s_p;
  for (int j = j0; j < j0 + jb; ++j) {
    double bv = -1.0;
    long long bi = (1LL << 62);
    for (int i = j + threadIdx.x; i < n; i += blockDim.x) {
      const double v = fabs(A[(size_t)i * lda + j]);
      if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
    block_argmax(bv, bi, red, redi);
    if (threadIdx.x == 0) {
      const int p = (bi >= n || bi < j) ? j : (int)bi;
      s_p = p;
      piv[j] = p;
      const double pv = A[(size_t)p * lda + j];
      if (pv == 0.0 || !isfinite(pv)) atomicCAS(status, 0, tag + 1);
    }
    __syncthreads();
    const int p = s_p;
    if (p != j)
      for (int c = j0 + threadIdx.x; c < j0 + jb; c += blockDim.x) {
        const double t = A[(size_t)j * lda + c];
        A[(size_t)j * lda + c] = A[(size_t)p * lda + c];
        A[(size_t)p * lda + c] = t;
      }
    __syncthreads();
    const double pv = A[(size_t)j * lda + j];
    const int rem_c = j0 + jb - j - 1;
    if (pv != 0.0)
      for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
        double* row = A + (size_t)i * lda;
        const double l = row[j] / pv;
        row[j] = l;
        const double* prow = A + (size_t)j * lda;
        for (int c = 1; c <= rem_c; ++c) row[j + c] -= l * prow[j + c];
      }
    __syncthreads();
  }
}

__global__ void laswp_kernel(double* A, int n, int lda, int j0, int jb, const int* piv) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int ncols = n - jb;
  if (t >= ncols) return;
  const int c = t < j0 ? t : t + jb;
  for (int j = j0; j < j0 + jb; ++j) {
    const int p = piv[j];
    if (p != j) {
      const double x = A[(size_t)j * lda + c];
      A[(size_t)j * lda + c] = A[(size_t)p * lda + c];
      A[(size_t)p * lda + c] = x;
    }
  }
}

__global__ void trsm_lunit_kernel(const double* L, int ldl, int nb, double* X, int ldx,
                                  int ncols) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncols) return;
  for (int i = 1; i < nb; ++i) {
    double s = X[(size_t)i * ldx + c];
    const double* l = L + (size_t)i * ldl;
    for (int j = 0; j < i; ++j) s = fma(-l[j], X[(size_t)j * ldx + c], s);
    X[(size_t)i * ldx + c] = s;
  }
}

__global__ void finite_kernel(const double* A, int n, int lda, int* status, int tag) {
  const long long tot = (long long)n * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const double v = A[(size_t)(e / n) * lda + (e % n)];
    if (!isfinite(v)) atomicCAS(status, 0, tag + 1);
  }
}

__global__ void __launch_bounds__(512)
extend_kernel(double* NB, int m, int k, const double* G, int extra, double* NW, double thr,
              double* work) {
  __shared__ double red[32];
  __shared__ double s_w;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double* A = work;                      // col-major m x extra
  double* tau = A + (size_t)m * extra;
  double* Q = tau + extra;
  for (long long e = threadIdx.x; e < (long long)m * extra; e += blockDim.x) A[e] = G[e];
  double mx = 0.0;
  for (int a = threadIdx.x; a < k; a += blockDim.x) mx = fmax(mx, NW[a]);
  mx = warp_max(mx);
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t = fmax(t, red[w]);
    s_w = fmax(thr, 1e-14 * (k ? t : 1.0));
  }
  __syncthreads();
  // G -= B (B^T G), column by column (warp per column)
  for (int c = warp; c < extra; c += nw) {
    double* g = A + (size_t)c * m;
    for (int a = 0; a < k; ++a) {
      const double* b = NB + (size_t)a * m;
      double d = 0.0;
      for (int i = lane; i < m; i += 32) d = fma(b[i], G[(size_t)c * m + i], d);
      d = warp_sum(d);
      for (int i = lane; i < m; i += 32) g[i] -= d * b[i];
    }
  }
  __syncthreads();
  cta_geqrf(A, m, extra, m, tau, red);
  cta_orgqr(A, m, extra, m, tau, Q, m);
  __syncthreads();
  for (long long e = threadIdx.x; e < (long long)m * extra; e += blockDim.x)
    NB[(size_t)k * m + e] = Q[e];
  for (int a = threadIdx.x; a < extra; a += blockDim.x) NW[k + a] = s_w;
}

}  // namespace

void launch_panel_lu(double* A, int n, int lda, int j0, int jb, int* piv, int* status, int tag,
                     cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_panel_lu"};
  panel_lu_kernel<<<1, 1024, 0, s>>>(A, n, lda, j0, jb, piv, status, tag);
}
void launch_laswp(double* A, int n, int lda, int j0, int jb, const int* piv, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_laswp"};
  const int nc = n - jb;
  if (nc <= 0) return;
  laswp_kernel<<<(nc + 127) / 128, 128, 0, s>>>(A, n, lda, j0, jb, piv);
}
void launch_trsm_lunit(const double* L, int ldl, int nb, double* X, int ldx, int ncols,
                       cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_trsm_lunit"};
  if (ncols <= 0) return;
  trsm_lunit_kernel<<<(ncols + 127) / 128, 128, 0, s>>>(L, ldl, nb, X, ldx, ncols);
}
void launch_finite_check(const double* A, int n, int lda, int* status, int tag, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_finite_check"};
  finite_kernel<<<592, 256, 0, s>>>(A, n, lda, status, tag);
}
void launch_extend(double* NB, int m, int k, const double* G, int extra, double* NW, double thr,
                   double* work, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_extend"};
  extend_kernel<<<1, 512, 0, s>>>(NB, m, k, G, extra, NW, thr, work);
}

}  // namespace ifmm

// ============================================================================
// Randomized SVD pieces (lowrank.py:79-125) for large fills
// ============================================================================
namespace ifmm {
namespace {

__device__ __forceinline__ unsigned long long splitmix(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__global__ void randn_kernel(const RandDesc* __restrict__ descs, int n) {
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const RandDesc d = descs[b];
    for (int e = threadIdx.x; e < d.count; e += blockDim.x) {
      const unsigned long long r1 = splitmix(d.key ^ (2ull * e + 1ull) * 0x632be59bd9b4e019ULL);
      const unsigned long long r2 = splitmix(r1 ^ 0x85ebca6b2ull);
      const double u1 = ((r1 >> 11) + 1) * (1.0 / 9007199254740993.0);  // (0, 1]
      const double u2 = (r2 >> 11) * (1.0 / 9007199254740992.0);
      d.out[e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    }
  }
}

__global__ void __launch_bounds__(512) orth_kernel(const OrthDesc* __restrict__ descs, int n) {
  __shared__ double red[32];
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const OrthDesc d = descs[b];
    double* A = d.work;                 // copy of Y (reflectors)
    double* tau = A + (size_t)d.m * d.w;
    for (long long e = threadIdx.x; e < (long long)d.m * d.w; e += blockDim.x) A[e] = d.Y[e];
    __syncthreads();
    cta_geqrf(A, d.m, d.w, d.m, tau, red);
    cta_orgqr(A, d.m, d.w, d.m, tau, d.Y, d.m);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512)
rsvd_fin_kernel(const RsvdFinDesc* __restrict__ descs, int n, double thr) {
  __shared__ int sflag;
  for (int b = blockIdx.x; b < n; b += gridDim.x) {
    const RsvdFinDesc d = descs[b];
    const int w = d.w;
    double* Wb = d.work;                 // w x w
    double* sig = Wb + (size_t)w * w;
    int* order = (int*)(sig + w);
    // B^T = V S Wb^T  (one-sided Jacobi on the w columns of B^T)
    cta_jacobi(d.Bt, d.n, w, d.n, Wb, &sflag);
    cta_sv_order(d.Bt, d.n, w, d.n, sig, order);
    int keep = 0;
    for (int j = 0; j < w; ++j) keep += sig[order[j]] > thr;
    const int cap = d.full;
    if (keep > cap) keep = cap;
    // lowrank.py:104: stop if width >= full or k_try >= cap or s[k_try] <= thr
    const bool stop = w >= d.full || d.k_try >= cap || (w > d.k_try && sig[order[d.k_try]] <= thr);
    // U = Q Wb[:, order[:keep]]  (m x keep), V = B^T col / sigma
    for (long long e = threadIdx.x; e < (long long)d.m * keep; e += blockDim.x) {
      const int a = (int)(e / d.m), i = (int)(e % d.m);
      const double* wv = Wb + (size_t)order[a] * w;
      double acc = 0.0;
      for (int l = 0; l < w; ++l) acc = fma(d.Q[(size_t)l * d.m + i], wv[l], acc);
      d.U[(size_t)a * d.m + i] = acc;
    }
    for (long long e = threadIdx.x; e < (long long)d.n * keep; e += blockDim.x) {
      const int a = (int)(e / d.n), i = (int)(e % d.n);
      const int j = order[a];
      d.V[(size_t)a * d.n + i] = d.Bt[(size_t)j * d.n + i] / sig[j];
    }
    for (int a = threadIdx.x; a < keep; a += blockDim.x) d.S[a] = sig[order[a]];
    if (threadIdx.x == 0) { *d.rank = keep; *d.stop = stop ? 1 : 0; }
    __syncthreads();
  }
}

}  // namespace

void launch_randn(const RandDesc* d, int n, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_randn"};
  if (n > 0) randn_kernel<<<n < 4096 ? n : 4096, 256, 0, s>>>(d, n);
}
void launch_orth(const OrthDesc* d, int n, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_orth"};
  if (n > 0) orth_kernel<<<n < 4096 ? n : 4096, 512, 0, s>>>(d, n);
}
void launch_rsvd_fin(const RsvdFinDesc* d, int n, double thr, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_rsvd_fin"};
  if (n > 0) rsvd_fin_kernel<<<n < 4096 ? n : 4096, 512, 0, s>>>(d, n, thr);
}

}  // namespace ifmm

// ---- micro-benchmark of the CTA Jacobi SVD (diagnostics) -------------------
namespace ifmm {
namespace {
__global__ void __launch_bounds__(512) jacobi_bench_kernel(const double* A, int s, int reps,
                                                           unsigned long long* out, int variant) {
  extern __shared__ double sm[];
  __shared__ int sflag;
  double* W = sm;
  double* V = sm + (size_t)s * s;
  unsigned long long tot = 0;
  int sw = 0;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < s * s; e += blockDim.x) W[e] = A[e];
    __syncthreads();
    if (variant == 2) {  // CholeskyQR building block: in-place Cholesky of two s x s SPD copies
      const int sp = s + (s & 1);
      double* GA = sm;
      double* GB = sm + (size_t)s * sp;
      double* iv = sm + 2 * (size_t)s * sp;
      for (int e = threadIdx.x; e < s * s; e += blockDim.x) {
        const int i = e / s, j = e - i * s;
        GA[(size_t)i * sp + j] = A[e];
        GB[(size_t)i * sp + j] = A[e];
      }
      __syncthreads();
      const unsigned long long t0 = clock64();
      cta_chol2(GA, iv, GB, iv + s, s, sp);
      tot += clock64() - t0;
      sw += s;
      __syncthreads();
      continue;
    }
    const unsigned long long t0 = clock64();
    sw += variant ? cta_jacobi_wv(W, V, s) : cta_jacobi(W, s, s, s, V, &sflag);
    const unsigned long long t1 = clock64();
    tot += t1 - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = tot; out[1] = (unsigned long long)sw; }
}
}  // namespace
void jacobi_bench(const double* A, int s, int reps, int threads, unsigned long long* d_out,
                  cudaStream_t st) {
  cudaFuncSetAttribute(jacobi_bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       220 * 1024);
  jacobi_bench_kernel<<<1, threads & 0xffff, (size_t)(2 * (s + 1) * (s + 1) + s + 8) * 8, st>>>(A, s, reps, d_out,
                                                                          threads >> 16);
}
}  // namespace ifmm
