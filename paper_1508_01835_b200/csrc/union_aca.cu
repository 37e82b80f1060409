// Register-resident full-pivot ACA for the weighted basis union
// (aca_svd, lowrank.py:128-151; called from weighted_basis_union,
// lowrank.py:166-199).
//
// The residual R (m x C) lives in REGISTERS, spread over one CTA or over a
// thread-block cluster of G CTAs (G = 2, 4, 8 for the level-3/2 unions whose
// residual does not fit one SM): CTA g, warp w owns the rows
// i = (16 g + w) + 16 G a (a < ER), lane l the columns j = l + 32 b (b < EC).
// A warp therefore holds whole rows, so the pivot column of its rows is one
// warp shuffle away, and only the pivot row crosses warps.  Per pivot step:
//   update + local argmax (registers) -> warp argmax -> candidates to shared
//   memory -> barrier A -> every warp reduces the 16 G candidates (DSMEM
//   when G > 1) -> the owning warp stores row p into every CTA's row buffer
//   -> barrier B -> row factors / pivot column -> next update.
// Two barriers per step (cluster barriers when G > 1) instead of the global
// round trips of the shared-/global-memory residual.
//
// Arithmetic is element for element that of union_kernel's ACA (and of
// numpy up to the FMA in the rank-1 update): row factors R[p, j] / piv with
// R[p, q] / piv := 1, residual r = fma(-c_i, row_j, r), pivot = max |R| with
// ties to the smallest row-major index.  A pivoted column becomes exactly
// zero (fma(-x, 1, x) = 0) and stays zero, so no active-column list is
// needed; only strictly positive magnitudes become candidates, an all-zero
// residual ends the loop as numpy's piv == 0 does.
//
// Output (the global union workspace layout of union_kernel): Acol (m x s,
// col-major, the pivot columns before their update), Bt (C x s, row factors),
// Dp (s pivots), hdr[0] = s.  union_kernel (giant == 2) continues with the
// CholeskyQR2 / core formation.
#include "common.cuh"
#include "dense.h"
#include <climits>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace ifmm {

namespace {

IFMM_DEV void warp_argmax_i(double& v, int& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) { v = ov; idx = oi; }
  }
}

template <int G>
IFMM_DEV void aca_barrier() {
  if constexpr (G > 1) cg::this_cluster().sync();
  else __syncthreads();
}

// workspace offsets (union_kernel / union_aca_coop layout)
struct UnionWs {
  double* Acol;
  double* Bt;
  double* Dp;
  int* hdr;
};
IFMM_DEV UnionWs union_ws(const UnionDesc& d) {
  const int m = d.m, C = d.k_old + d.k_f;
  const int smax = m < C ? m : C;
  const int spx = smax + (smax & 1);
  const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
  UnionWs w;
  w.Acol = d.work + mreg;
  w.Bt = w.Acol + (size_t)m * smax;
  double* core = w.Bt + 2 * (size_t)C * smax;
  w.Dp = core + 2 * (size_t)smax * smax;
  w.hdr = (int*)(w.Dp + 4 * (size_t)smax);
  return w;
}

constexpr int ACA_THREADS = 512;
constexpr int ACA_WARPS = ACA_THREADS / 32;

template <int ER, int EC, int G>
__global__ void __launch_bounds__(ACA_THREADS, 1)
union_aca_reg(const UnionDesc* __restrict__ descs, int n, double thr) {
  __shared__ double candv[ACA_WARPS];
  __shared__ int candi[ACA_WARPS];
  __shared__ double prow[32 * EC];
  const int u = blockIdx.x / G;
  if (u >= n) return;  // whole clusters only (grid = n G)
  const int g = G > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const UnionDesc d = descs[u];
  if (d.giant < 2) return;  // uniform per cluster: giants / legacy-ACA unions
  const int m = d.m, ko = d.k_old, C = ko + d.k_f;
  const int smax = m < C ? m : C;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int ws = g * ACA_WARPS + w;
  constexpr int RS = ACA_WARPS * G;
  const UnionWs W = union_ws(d);

  // concat [B diag(w) | F diag(wf)] + first local argmax (row-major order of
  // the thread's elements: a-major, then b -> strict '>' keeps the first)
  double e[ER][EC];
  double bv = 0.0;
  int bi = INT_MAX;
#pragma unroll
  for (int a = 0; a < ER; ++a) {
    const int i = ws + a * RS;
#pragma unroll
    for (int b = 0; b < EC; ++b) {
      const int j = lane + 32 * b;
      double v = 0.0;
      if (i < m && j < C)
        v = j < ko ? d.B[(size_t)i * d.b_r + (size_t)j * d.b_c] * d.w[j]
                   : d.F[(size_t)i * d.f_r + (size_t)(j - ko) * d.f_c] * d.wf[j - ko];
      e[a][b] = v;
      const double av = fabs(v);
      if (av > bv) { bv = av; bi = i * C + j; }
    }
  }
  const double floor_ = thr / 8.0;
  int steps = 0;
  for (; steps < smax; ++steps) {
    // ---- candidates
    warp_argmax_i(bv, bi);
    if (lane == 0) { candv[w] = bv; candi[w] = bi; }
    aca_barrier<G>();  // A
    double gv = 0.0;
    int gi = INT_MAX;
    if constexpr (G > 1) {
      cg::cluster_group cl = cg::this_cluster();
      for (int c = lane; c < RS; c += 32) {
        const double* rv = cl.map_shared_rank(candv, c / ACA_WARPS);
        const int* ri = cl.map_shared_rank(candi, c / ACA_WARPS);
        const double ov = rv[c % ACA_WARPS];
        const int oi = ri[c % ACA_WARPS];
        if (ov > gv || (ov == gv && oi < gi)) { gv = ov; gi = oi; }
      }
    } else {
      if (lane < ACA_WARPS) { gv = candv[lane]; gi = candi[lane]; }
    }
    warp_argmax_i(gv, gi);
    if (gi == INT_MAX) break;  // all-zero residual (numpy: piv == 0), uniform
    const int p = gi / C, q = gi - p * C;
    // ---- the owning warp publishes row p (pre-update) to every CTA
    const int wsp = p % RS, ap = p / RS;
    if (ws == wsp) {
#pragma unroll
      for (int b = 0; b < EC; ++b) {
        double v = 0.0;
#pragma unroll
        for (int a = 0; a < ER; ++a) v = a == ap ? e[a][b] : v;
        const int j = lane + 32 * b;
        if constexpr (G > 1) {
          cg::cluster_group cl = cg::this_cluster();
#pragma unroll
          for (int r = 0; r < G; ++r) cl.map_shared_rank(prow, r)[j] = v;
        } else {
          prow[j] = v;
        }
      }
    }
    aca_barrier<G>();  // B
    const double piv = prow[q];
    if (fabs(piv) <= floor_ && steps >= d.min_rank) break;  // uniform
    // ---- pivot column of the own rows (one shuffle per row) and row factors
    const int bq = q >> 5, lq = q & 31;
    double c[ER];
#pragma unroll
    for (int a = 0; a < ER; ++a) {
      double v = 0.0;
#pragma unroll
      for (int b = 0; b < EC; ++b) v = b == bq ? e[a][b] : v;
      c[a] = __shfl_sync(0xffffffffu, v, lq);
    }
    double r[EC];
#pragma unroll
    for (int b = 0; b < EC; ++b) {
      const int j = lane + 32 * b;
      r[b] = j == q ? 1.0 : (j < C ? prow[j] / piv : 0.0);
    }
    if (lane == lq) {
#pragma unroll
      for (int a = 0; a < ER; ++a) {
        const int i = ws + a * RS;
        if (i < m) W.Acol[(size_t)steps * m + i] = c[a];
      }
    }
    if (ws == 0) {
#pragma unroll
      for (int b = 0; b < EC; ++b) {
        const int j = lane + 32 * b;
        if (j < C) W.Bt[(size_t)steps * C + j] = r[b];
      }
      if (lane == 0) W.Dp[steps] = piv;
    }
    // ---- rank-1 update + next local argmax
    bv = 0.0;
    bi = INT_MAX;
#pragma unroll
    for (int a = 0; a < ER; ++a) {
      const int ib = (ws + a * RS) * C;
#pragma unroll
      for (int b = 0; b < EC; ++b) {
        const double v = fma(-c[a], r[b], e[a][b]);
        e[a][b] = v;
        const double av = fabs(v);
        if (av > bv) { bv = av; bi = ib + lane + 32 * b; }
      }
    }
  }
  if (ws == 0 && lane == 0) W.hdr[0] = steps;
  // the other CTAs of the cluster may still read this CTA's candidates /
  // row buffer of the last step: keep shared memory alive until they are done
  if constexpr (G > 1) cg::this_cluster().sync();
}

template <int ER, int EC, int G>
void launch_g(const UnionDesc* d, int n, double thr, cudaStream_t s) {
  if constexpr (G == 1) {
    union_aca_reg<ER, EC, 1><<<n, ACA_THREADS, 0, s>>>(d, n, thr);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(n * G);
    cfg.blockDim = dim3(ACA_THREADS);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = G;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, union_aca_reg<ER, EC, G>, d, n, thr);
    if (e != cudaSuccess)
      fprintf(stderr, "[ifmm] cluster ACA launch (G=%d) failed: %s\n", G, cudaGetErrorString(e));
  }
}

template <int ER, int EC>
void launch_er(const UnionDesc* d, int n, double thr, int G, cudaStream_t s) {
  switch (G) {
    case 1: launch_g<ER, EC, 1>(d, n, thr, s); break;
    case 2: launch_g<ER, EC, 2>(d, n, thr, s); break;
    case 4: launch_g<ER, EC, 4>(d, n, thr, s); break;
    default: launch_g<ER, EC, 8>(d, n, thr, s); break;
  }
}

template <int EC>
void launch_ec(const UnionDesc* d, int n, double thr, int G, int ER, cudaStream_t s) {
  if (ER <= 4) launch_er<4, EC>(d, n, thr, G, s);
  else if (ER <= 8) launch_er<8, EC>(d, n, thr, G, s);
  else if constexpr (EC <= 2) launch_er<16, EC>(d, n, thr, G, s);
}

}  // namespace

// Register-tile class of a union (max_m rows, max_C columns): EC column
// slots per lane, ER rows per warp slot, G CTAs per cluster.  False when the
// residual does not fit a register tile of <= 32 elements per thread on up
// to 8 CTAs (the caller keeps union_kernel's own ACA).
bool union_aca_reg_class(int max_m, int max_C, int* G, int* ER, int* EC) {
  const int ec = (max_C + 31) / 32;
  if (ec < 1 || ec > 4 || max_m < 1) return false;
  const int er_max = ec <= 2 ? 16 : 8;  // ER * EC <= 32
  for (int g = 1; g <= 8; g *= 2) {
    const int er = (max_m + 16 * g - 1) / (16 * g);
    if (er <= er_max) {
      *G = g;
      *ER = er <= 4 ? 4 : er <= 8 ? 8 : 16;
      *EC = ec;
      return true;
    }
  }
  return false;
}

void launch_union_aca_reg(const UnionDesc* d_descs, int n, double thr, int G, int ER, int EC,
                          cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_union_aca_reg"};
  if (n <= 0) return;
  switch (EC) {
    case 1: launch_ec<1>(d_descs, n, thr, G, ER, s); break;
    case 2: launch_ec<2>(d_descs, n, thr, G, ER, s); break;
    case 3: launch_ec<3>(d_descs, n, thr, G, ER, s); break;
    default: launch_ec<4>(d_descs, n, thr, G, ER, s); break;
  }
}

}  // namespace ifmm
