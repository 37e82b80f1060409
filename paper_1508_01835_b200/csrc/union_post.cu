// Second half of the weighted basis union (weighted_basis_union,
// lowrank.py:166-199; aca_svd, lowrank.py:128-163) for the unions whose
// full-pivot ACA ran in registers (union_aca.cu): one CTA per union, every
// matrix of the orthonormalisation and of the core SVD in shared memory, the
// tall factors streamed through it in row chunks.
//
// Input (global union workspace, union_aca_reg's output): X (m x s, pivot
// columns), Y (C x s, row factors), D (s pivots).  With L = X D^-1:
//   pass 1   G_A = L^T L, G_B = Y^T Y          (DMMA 8x8x4 over row chunks)
//            R1 = chol(G)                      (packed upper triangles)
//            M = R1_B D R1_A^T                 (the core's transpose, s x s)
//   pass 2   Q1 = L R1^-1 row by row (teams of 16 lanes own a row in
//            registers), written back in place; E = Q1^T Q1 - I (DMMA)
//            The second CholeskyQR pass is first order in E (|E| ~ eps
//            cond(L)^2, below 1e-9 or the union falls back to the legacy
//            kernels): R2 = I + U, U = triu(E, 1) + diag(E) / 2, so
//            W = R2_B M R2_A^T = M + U_B M + M U_A^T and R2^-1 = I - U.
//   Jacobi   one-sided (Hestenes) on W with accumulated V, as union_svd_kernel
//   pass 3   new basis = Q1_A (I - U_A) phi_k, maps = Q1_B (I - U_B) sigma psi_k
//            / weights                          (DMMA over row chunks)
// Same algebra as union_kernel + union_svd_kernel (CholeskyQR2 of the
// pivot-scaled ACA factors, transposed-core Jacobi); results agree to
// rounding.  A union this kernel cannot take (s > 96, Cholesky breakdown,
// |E| > 1e-9) gets rank -1 and the host reruns it on the legacy path.
#include "common.cuh"
#include "dense.h"

namespace ifmm {

__device__ unsigned long long g_upprof[16];

void union_post_profile(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_upprof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(g_upprof, z, sizeof z);
  }
}

namespace {

constexpr int PT = 512;          // threads per CTA
constexpr int PW = PT / 32;      // warps
constexpr int P_SMAX = 96;       // largest ACA rank taken here
constexpr int P_SMEM = 29000;    // doubles of dynamic shared memory (232,000 B)
constexpr int P_EPT = 16;        // chunk elements staged per thread
constexpr int P_TILES = 5;       // Gram tiles per warp: 78 upper 8x8 tiles of a 96 x 96 Gram / 16
constexpr double kCholFloorP = 1e-12;
constexpr double kOrthFloor = 1e-9;
constexpr double kSkipRatio = 5e-3;

IFMM_DEV int tri_off(int i, int S) { return i * S - (i * (i + 1)) / 2; }  // + j, j >= i

// rows [r0, r0 + RC) of a col-major global matrix (ld ldg, nrows rows, S
// columns) -> registers; element e = threadIdx.x + u PT is (column e / RC,
// row e % RC); zero outside the matrix
IFMM_DEV void chunk_fetch(double (&reg)[P_EPT], const double* __restrict__ src, int ldg, int nrows,
                          int r0, int RC, int S) {
  int j = threadIdx.x / RC, r = threadIdx.x - j * RC;
  const int dj = PT / RC, dr = PT - dj * RC;
#pragma unroll
  for (int u = 0; u < P_EPT; ++u) {
    double v = 0.0;
    if (j < S && r0 + r < nrows) v = src[(size_t)j * ldg + r0 + r];
    reg[u] = v;
    j += dj; r += dr;
    if (r >= RC) { r -= RC; ++j; }
  }
}

// registers -> shared chunk (col-major, ld ldr, S8 columns); dv: optional
// per-column scales (reciprocals of the ACA pivots)
IFMM_DEV void chunk_store(const double (&reg)[P_EPT], double* chunk, int ldr, int RC, int S, int S8,
                          const double* dv) {
  int j = threadIdx.x / RC, r = threadIdx.x - j * RC;
  const int dj = PT / RC, dr = PT - dj * RC;
#pragma unroll
  for (int u = 0; u < P_EPT; ++u) {
    if (j < S8) chunk[j * ldr + r] = (dv && j < S) ? reg[u] * dv[j] : reg[u];
    j += dj; r += dr;
    if (r >= RC) { r -= RC; ++j; }
  }
}

// shared chunk -> rows [r0, r0 + RC) of the col-major global matrix
IFMM_DEV void chunk_writeback(const double* chunk, int ldr, int RC, double* dst, int ldg, int nrows,
                              int r0, int S) {
  int j = threadIdx.x / RC, r = threadIdx.x - j * RC;
  const int dj = PT / RC, dr = PT - dj * RC;
#pragma unroll
  for (int u = 0; u < P_EPT; ++u) {
    if (j < S && r0 + r < nrows) dst[(size_t)j * ldg + r0 + r] = chunk[j * ldr + r];
    j += dj; r += dr;
    if (r >= RC) { r -= RC; ++j; }
  }
}

// upper 8x8 tile t (column-block major): t = J (J + 1) / 2 + I, I <= J
IFMM_DEV void tile_ij(int t, int& I, int& J) {
  J = 0;
  while ((J + 1) * (J + 2) / 2 <= t) ++J;
  I = t - J * (J + 1) / 2;
}

// acc += chunk^T chunk over the chunk's rows (k4 steps of 4 rows).  Work item
// w = warp + 16 q is (upper tile w % nt, K group w / nt): KG groups split the
// 4-row steps of a tile (step k belongs to group k % KG) so that a warp
// carries several independent DMMA chains (DMMA 8x8x4 latency ~180 cycles);
// both operands come from the col-major chunk (A[i][k] = chunk[8 I + i][k],
// B[k][j] = chunk[8 J + j][k]).
IFMM_DEV void gram_accum(double (&acc)[P_TILES][2], const double* chunk, int ldr, int k4, int nt, int KG) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* pa[P_TILES];
  const double* pb[P_TILES];
  int k0[P_TILES];
#pragma unroll
  for (int q = 0; q < P_TILES; ++q) {
    const int w = warp + q * PW;
    int I = 0, J = 0;
    k0[q] = k4;
    if (w < nt * KG) {
      tile_ij(w % nt, I, J);
      k0[q] = w / nt;
    }
    pa[q] = chunk + (I * 8 + (lane >> 2)) * ldr + (lane & 3);
    pb[q] = chunk + (J * 8 + (lane >> 2)) * ldr + (lane & 3);
  }
  for (int k = 0; k < k4; k += KG) {
#pragma unroll
    for (int q = 0; q < P_TILES; ++q) {
      const int kk = k + k0[q];
      if (kk < k4) dmma_8x8x4(acc[q][0], acc[q][1], pa[q][4 * kk], pb[q][4 * kk]);
    }
  }
}

// accumulators -> packed upper triangle G (row i at tri_off(i) + j); the K
// groups of a tile are added in group order through `scratch` (64 doubles per
// work item; unused when KG == 1).  Ends with a barrier.
IFMM_DEV void gram_store(const double (&acc)[P_TILES][2], double* G, int S, int nt, int KG,
                         double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (KG == 1) {
#pragma unroll
    for (int q = 0; q < P_TILES; ++q) {
      const int t = warp + q * PW;
      if (t >= nt) continue;
      int I, J;
      tile_ij(t, I, J);
      const int i = I * 8 + (lane >> 2), j = J * 8 + 2 * (lane & 3);
      if (i < S) {
        if (j < S && i <= j) G[tri_off(i, S) + j] = acc[q][0];
        if (j + 1 < S && i <= j + 1) G[tri_off(i, S) + j + 1] = acc[q][1];
      }
    }
    __syncthreads();
    return;
  }
#pragma unroll
  for (int q = 0; q < P_TILES; ++q) {
    const int w = warp + q * PW;
    if (w < nt * KG) {
      scratch[w * 64 + 2 * lane] = acc[q][0];
      scratch[w * 64 + 2 * lane + 1] = acc[q][1];
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nt * 64; e += PT) {
    const int t = e >> 6, f = e & 63;
    double v = 0.0;
    for (int g = 0; g < KG; ++g) v += scratch[(g * nt + t) * 64 + f];
    int I, J;
    tile_ij(t, I, J);
    const int ln = f >> 1;
    const int i = I * 8 + (ln >> 2), j = J * 8 + 2 * (ln & 3) + (f & 1);
    if (i < S && j < S && i <= j) G[tri_off(i, S) + j] = v;
  }
  __syncthreads();
}

// In-place right-looking Cholesky G = R^T R of two packed SPD matrices at
// once, one barrier per step (step k eliminates with the unscaled row k and
// scales row k - 1).  rinv[k] = 1 / R[k][k].  Returns the smallest pivot ratio
// R_kk^2 / max_i G_ii of both (uniform; 0 on breakdown).
IFMM_DEV double chol2_packed(double* GA, double* ia, double* GB, double* ib, int S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double minr = 1.0, mxA = 0.0, mxB = 0.0;
  for (int k = 0; k < S; ++k) {
    mxA = fmax(mxA, GA[tri_off(k, S) + k]);
    mxB = fmax(mxB, GB[tri_off(k, S) + k]);
  }
  const double imxA = 1.0 / mxA, imxB = 1.0 / mxB;
  __syncthreads();
  for (int k = 0; k <= S; ++k) {
    if (k > 0) {
      const double ra = ia[k - 1], rb = ib[k - 1];
      double* gra = GA + tri_off(k - 1, S);
      double* grb = GB + tri_off(k - 1, S);
      for (int j = k - 1 + threadIdx.x; j < S; j += PT) {
        gra[j] *= ra;
        grb[j] *= rb;
      }
    }
    if (k < S) {
      const double* ga = GA + tri_off(k, S);
      const double* gb = GB + tri_off(k, S);
      const double pa = ga[k], pb = gb[k];
      const double inva = 1.0 / pa, invb = 1.0 / pb;
      const double ra = rsqrt(pa), rb = rsqrt(pb);
      const double qa = pa * imxA, qb = pb * imxB;
      minr = (qa > 0.0 && isfinite(pa)) ? fmin(minr, qa) : 0.0;
      minr = (qb > 0.0 && isfinite(pb)) ? fmin(minr, qb) : 0.0;
      if (threadIdx.x == 0) { ia[k] = ra; ib[k] = rb; }
      const int nr = S - k - 1;
      for (int t = wid; t < 2 * nr; t += PW) {
        const bool isA = t < nr;
        const int i = k + 1 + (isA ? t : t - nr);
        const double* g = isA ? ga : gb;
        double* Gi = (isA ? GA : GB) + tri_off(i, S);
        const double fi = g[i] * (isA ? inva : invb);
        for (int j = i + lane; j < S; j += 32) Gi[j] = fma(-fi, g[j], Gi[j]);
      }
    }
    __syncthreads();
  }
  return minr;
}

// chunk rows <- rows R^-1 (R packed upper, rinv = 1 / diag): a team of 16
// lanes owns one row in registers (lane l: columns l + 16 e); column j's
// solved entry is broadcast with one shuffle and eliminated from the later
// columns (right-looking), no barrier inside.
template <int NE>
IFMM_DEV void trsm_rows(double* chunk, int ldr, int rows, const double* __restrict__ R,
                        const double* __restrict__ rinv, int S) {
  const int l16 = threadIdx.x & 15, team = threadIdx.x >> 4;
  for (int rb = 0; rb < rows; rb += PT / 16) {
    const int r = rb + team;
    const bool on = r < rows;
    double a[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int col = l16 + 16 * e;
      a[e] = (on && col < S) ? chunk[col * ldr + r] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int jend = S - 16 * e < 16 ? S - 16 * e : 16;
      for (int jj = 0; jj < jend; ++jj) {
        const int j = 16 * e + jj;
        const double xj = __shfl_sync(0xffffffffu, a[e] * rinv[j], jj, 16);
        if (l16 == jj) a[e] = xj;
        const double* Rj = R + tri_off(j, S);
#pragma unroll
        for (int e2 = e; e2 < NE; ++e2) {
          const int col = l16 + 16 * e2;
          if (col > j && col < S) a[e2] = fma(-xj, Rj[col], a[e2]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int col = l16 + 16 * e;
      if (on && col < S) chunk[col * ldr + r] = a[e];
    }
  }
}

IFMM_DEV void trsm_chunk(double* chunk, int ldr, int rows, const double* R, const double* rinv, int S) {
  if (S <= 32) trsm_rows<2>(chunk, ldr, rows, R, rinv, S);
  else if (S <= 64) trsm_rows<4>(chunk, ldr, rows, R, rinv, S);
  else trsm_rows<6>(chunk, ldr, rows, R, rinv, S);
}

template <int T>
IFMM_DEV double team_sum_p(double v) {
#pragma unroll
  for (int o = T / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One round-robin Jacobi sweep on W (S columns of S rows, col-major ld) with
// the rotations accumulated in V.  A team of T lanes owns one column pair per
// round and holds NE rows per lane of all four columns in registers between
// the dot products and the rotation (T NE >= S); one barrier per round.
template <int T, int NE, bool VREG>
IFMM_DEV bool jac_sweep_p(double* W, double* V, int S, int ld, double tr2, double tc2) {
  const int tl = threadIdx.x & (T - 1), team = threadIdx.x / T;
  const int cp = S + (S & 1), half = cp >> 1, m1 = cp - 1;
  int p0 = team, q0 = team == 0 ? m1 : m1 - team;
  bool again = false;
  // warps whose teams never hold a pair leave the sweep's arithmetic (they
  // still take part in the barriers)
  const bool warp_on = ((threadIdx.x & ~31) / T) < half;
  for (int r = 0; r < m1; ++r) {
    if (warp_on) {
      const int lo = p0 < q0 ? p0 : q0, hi = p0 < q0 ? q0 : p0;
      const bool act = team < half && hi < S;
      double* x = W + (act ? lo : 0) * ld;
      double* y = W + (act ? hi : 0) * ld;
      double* vx = V + (act ? lo : 0) * ld;
      double* vy = V + (act ? hi : 0) * ld;
      double xr[NE], yr[NE], ur[VREG ? NE : 1], vr[VREG ? NE : 1];
      double a0 = 0.0, b0 = 0.0, g0 = 0.0, a1 = 0.0, b1 = 0.0, g1 = 0.0;
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        const int i = tl + e * T;
        const bool in = act && i < S;
        xr[e] = in ? x[i] : 0.0;
        yr[e] = in ? y[i] : 0.0;
        if constexpr (VREG) {
          ur[e] = in ? vx[i] : 0.0;
          vr[e] = in ? vy[i] : 0.0;
        }
      }
#pragma unroll
      for (int e = 0; e < NE; e += 2) {
        a0 = fma(xr[e], xr[e], a0); b0 = fma(yr[e], yr[e], b0); g0 = fma(xr[e], yr[e], g0);
        if (e + 1 < NE) {
          a1 = fma(xr[e + 1], xr[e + 1], a1); b1 = fma(yr[e + 1], yr[e + 1], b1);
          g1 = fma(xr[e + 1], yr[e + 1], g1);
        }
      }
      // every lane of the warp takes part in the shuffles (teams never straddle a warp)
      double a = a0 + a1, b = b0 + b1, g = g0 + g1;
#pragma unroll
      for (int o = T / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        g += __shfl_xor_sync(0xffffffffu, g, o);
      }
      const double ab = a * b, g2 = g * g;
      if (act && g != 0.0 && g2 > tr2 * ab) {
        // rotation angle theta with tan(2 theta) = gg / d, d = b - a, gg = 2 g, |theta| <= pi / 4:
        // with h = sqrt(d^2 + gg^2): cos^2 = (h + |d|) / 2h, sin cos = sign(d gg) |gg| / 2h
        // (two rsqrt chains instead of sqrt -> div -> rsqrt)
        const double d = b - a, gg = 2.0 * g;
        const double rh = rsqrt(fma(d, d, gg * gg));
        const double cc = fma(0.5 * fabs(d), rh, 0.5);
        const double rc = rsqrt(cc);
        const double c = cc * rc;
        const double sn = copysign(0.5 * fabs(gg) * rh * rc, d * gg);
#pragma unroll
        for (int e = 0; e < NE; ++e) {
          const int i = tl + e * T;
          if (i < S) {
            x[i] = fma(c, xr[e], -sn * yr[e]);
            y[i] = fma(sn, xr[e], c * yr[e]);
            if constexpr (VREG) {
              vx[i] = fma(c, ur[e], -sn * vr[e]);
              vy[i] = fma(sn, ur[e], c * vr[e]);
            }
          }
        }
        if constexpr (!VREG) {
          // V columns in batches of 4 rows per lane, all loads before the stores
#pragma unroll
          for (int e0 = 0; e0 < NE; e0 += 4) {
            double u4[4], v4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = tl + (e0 + e) * T;
              const bool in = e0 + e < NE && i < S;
              u4[e] = in ? vx[i] : 0.0;
              v4[e] = in ? vy[i] : 0.0;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int i = tl + (e0 + e) * T;
              if (e0 + e < NE && i < S) {
                vx[i] = fma(c, u4[e], -sn * v4[e]);
                vy[i] = fma(sn, u4[e], c * v4[e]);
              }
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

IFMM_DEV int jacobi_p(double* W, double* V, int S, int ld) {
  for (int e = threadIdx.x; e < S * ld; e += PT) {
    const int j = e / ld, i = e - j * ld;
    V[e] = (i == j) ? 1.0 : 0.0;
  }
  const double tol_rot = kEps;
  const double tol_conv = fmax(kEps * (double)(S > 4 ? S : 4), 1e-13);
  const double tr2 = tol_rot * tol_rot, tc2 = tol_conv * tol_conv;
  __syncthreads();
  if (S < 2) return 0;
  int sweep = 0;
  for (; sweep < 40; ++sweep) {
    bool ag;
    if (S <= 32) ag = jac_sweep_p<16, 2, true>(W, V, S, ld, tr2, tc2);
    else if (S <= 64) ag = jac_sweep_p<16, 4, true>(W, V, S, ld, tr2, tc2);
    else ag = jac_sweep_p<8, 12, false>(W, V, S, ld, tr2, tc2);
    if (!__syncthreads_or(ag)) break;
  }
  return sweep + 1;
}

// Column norms -> sig[j]; order[pos] = j sorted by sig desc (ties: lower j,
// NaN last).
IFMM_DEV void sv_order_p(const double* W, int S, int ld, double* sig, int* order) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < S; j += PW) {
    double a = 0.0;
    for (int i = lane; i < S; i += 32) { const double u = W[j * ld + i]; a = fma(u, u, a); }
    a = warp_sum(a);
    if (lane == 0) sig[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < S; j += PT) {
    const double sj = isnan(sig[j]) ? -1.0 : sig[j];
    int pos = 0;
    for (int l = 0; l < S; ++l) {
      const double sl = isnan(sig[l]) ? -1.0 : sig[l];
      pos += (sl > sj) || (sl == sj && l < j);
    }
    order[pos] = j;
  }
  __syncthreads();
}

// Z <- (I - U) Z in place for the S columns of Z (col-major ld), U packed
// strict upper + half diagonal: block rows of 8 top-down (row i reads rows
// l >= i, all still unmodified), values held in registers across the barrier.
IFMM_DEV void apply_inv_r2(double* Z, int ld, const double* U, int S) {
  for (int i0 = 0; i0 < S; i0 += 8) {
    const int nr = S - i0 < 8 ? S - i0 : 8;
    const int items = nr * S;  // (row i0 + ii, column c): ii fastest
    double out[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int it = threadIdx.x + q * PT;
      double acc = 0.0;
      if (it < items) {
        const int c = it / nr, i = i0 + (it - c * nr);
        const double* Ui = U + tri_off(i, S);
        const double* z = Z + c * ld;
        acc = z[i];
        for (int l = i; l < S; ++l) acc = fma(-Ui[l], z[l], acc);
      }
      out[q] = acc;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int it = threadIdx.x + q * PT;
      if (it < items) {
        const int c = it / nr, i = i0 + (it - c * nr);
        Z[c * ld + i] = out[q];
      }
    }
    __syncthreads();
  }
}

// Z[:, order[a]] <- R^-1 Z[:, order[a]] for a < k (R packed upper, rinv = 1 /
// diag): a team of 8 lanes owns one column in registers (lane l: rows l + 8 e)
// and back-substitutes from the last row up; each solved entry is broadcast
// with one shuffle and eliminated from the rows above it, no barrier inside.
template <int NE>
IFMM_DEV void backsolve_cols(double* Z, int ld, const int* order, int k, const double* __restrict__ R,
                             const double* __restrict__ rinv, int S) {
  const int l8 = threadIdx.x & 7, team = threadIdx.x >> 3;
  for (int cb = 0; cb < k; cb += PT / 8) {
    const int a = cb + team;
    const bool on = a < k;
    double* z = Z + order[on ? a : 0] * ld;
    double v[NE];
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int i = l8 + 8 * e;
      v[e] = (on && i < S) ? z[i] : 0.0;
    }
#pragma unroll
    for (int e = NE - 1; e >= 0; --e) {
      const int jtop = S - 8 * e < 8 ? S - 8 * e : 8;  // rows 8 e .. 8 e + jtop - 1 exist
      for (int jj = jtop - 1; jj >= 0; --jj) {
        const int i = 8 * e + jj;
        const double zi = __shfl_sync(0xffffffffu, v[e] * rinv[i], jj, 8);
        if (l8 == jj) v[e] = zi;
#pragma unroll
        for (int e2 = 0; e2 <= e; ++e2) {
          const int l = l8 + 8 * e2;
          if (l < i) v[e2] = fma(-zi, R[tri_off(l, S) + i], v[e2]);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int i = l8 + 8 * e;
      if (on && i < S) z[i] = v[e];
    }
  }
}

IFMM_DEV void backsolve(double* Z, int ld, const int* order, int k, const double* R, const double* rinv, int S) {
  if (S <= 32) backsolve_cols<4>(Z, ld, order, k, R, rinv, S);
  else if (S <= 64) backsolve_cols<8>(Z, ld, order, k, R, rinv, S);
  else backsolve_cols<12>(Z, ld, order, k, R, rinv, S);
}

// out(rows x k) = chunk(rows x S) Zsel(S x k) with Zsel's column a = column
// order[a] of Z; one warp per 8x8 output tile, DMMA over S8 / 4 steps.  The
// store callback receives (row in chunk, a, value).
template <class Store>
IFMM_DEV void out_tiles(const double* chunk, int ldr, int rows, const double* Z, int ld,
                        const int* order, int k, int S8, Store store) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rt = (rows + 7) >> 3, ct = (k + 7) >> 3;
  for (int t = warp; t < rt * ct; t += PW) {
    const int ti = t % rt, tj = t / rt;
    const int acol = tj * 8 + (lane >> 2);
    const double* pz = Z + order[acol < k ? acol : k - 1] * ld + (lane & 3);
    const double* pq = chunk + (lane & 3) * ldr + ti * 8 + (lane >> 2);
    double c0 = 0.0, c1 = 0.0;
    for (int l = 0; l < S8; l += 4) dmma_8x8x4(c0, c1, pq[l * ldr], pz[l]);
    const int row = ti * 8 + (lane >> 2), a = tj * 8 + 2 * (lane & 3);
    if (row < rows) {
      if (a < k) store(row, a, c0);
      if (a + 1 < k) store(row, a + 1, c1);
    }
  }
}

__global__ void __launch_bounds__(PT, 1)
union_post_kernel(const UnionDesc* __restrict__ descs, int n, double thr) {
  extern __shared__ double smem[];
  __shared__ double s_red[PW];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int bb = blockIdx.x; bb < n; bb += gridDim.x) {
    const UnionDesc d = descs[bb];
    if (d.giant != 3) continue;
    const int m = d.m, ko = d.k_old, C = d.k_old + d.k_f;
    const int smax = m < C ? m : C;
    const int spx = smax + (smax & 1);
    const size_t mreg = (size_t)m * C > 6 * (size_t)smax * spx ? (size_t)m * C : 6 * (size_t)smax * spx;
    double* gX = d.work + mreg;
    double* gY = gX + (size_t)m * smax;
    double* gD = gY + 2 * (size_t)C * smax + 2 * (size_t)smax * smax;
    const int S = *(const int*)(gD + 4 * (size_t)smax);
    __syncthreads();  // previous union's shared memory is dead
    if (S == 0) {
      if (threadIdx.x == 0) *d.rank = 0;
      continue;
    }
    if (S > P_SMAX) {
      if (threadIdx.x == 0) *d.rank = -1;
      continue;
    }
    unsigned long long t0 = clock64();
    const int nb8 = (S + 7) >> 3, S8 = nb8 * 8;
    const int nt = nb8 * (nb8 + 1) / 2;
    const int ld = S8;  // W / V column stride (rows S..S8-1 stay zero)
    const int tri = S * (S + 1) / 2;
    // ---- shared-memory layout
    double* Dv = smem;        // ACA pivots
    double* Di = Dv + S8;     // their reciprocals
    double* ia = Di + S8;
    double* ib = ia + S8;
    double* sig = ib + S8;
    int* order = (int*)(sig + S8);
    double* W = sig + 2 * S8;
    double* RA = W + S * ld;
    double* RB = RA + tri;
    double* V = RB + tri;
    double* fre = V + S * ld;
    const int n_fre = P_SMEM - (int)(fre - smem);
    // chunk buffers: passes 1 / 2 use V + the free tail; pass 3 the dead R
    // triangles or the free tail, whichever is larger
    auto chunk_rows = [&](int doubles, int nrows) {
      int rc = doubles / S8 - 4;
      const int cap = (PT * P_EPT) / S8;
      if (rc > cap) rc = cap;
      if (rc > 128) rc = 128;
      rc &= ~15;
      const int need = (nrows + 15) & ~15;
      if (rc > need) rc = need;
      return rc;
    };
    const int mc = m > C ? m : C;
    double* buf12 = V;
    const int RC12 = chunk_rows(S * ld + n_fre, mc);
    double* buf3 = 2 * tri >= n_fre ? RA : fre;
    const int RC3 = chunk_rows(2 * tri >= n_fre ? 2 * tri : n_fre, mc);
    if (RC12 < 16 || RC3 < 16) {  // cannot happen for S <= 96 (see P_SMEM)
      if (threadIdx.x == 0) *d.rank = -1;
      continue;
    }
    for (int j = threadIdx.x; j < S8; j += PT) {
      const double pv = j < S ? gD[j] : 1.0;
      Dv[j] = pv;
      Di[j] = 1.0 / pv;
    }
    __syncthreads();
    // K groups per Gram tile (independent DMMA chains per warp)
    const int KG = nt * 8 <= PW * P_TILES ? 8 : (PW * P_TILES) / nt;

    double reg[P_EPT];
    double acc[P_TILES][2];
    // ---- pass 1: Gram matrices of L = X D^-1 and of Y
    for (int side = 0; side < 2; ++side) {
      const double* src = side == 0 ? gX : gY;
      const int nrows = side == 0 ? m : C;
      const int RC = RC12, ldr = RC + 4;
#pragma unroll
      for (int q = 0; q < P_TILES; ++q) acc[q][0] = acc[q][1] = 0.0;
      unsigned long long q0 = clock64();
      chunk_fetch(reg, src, nrows, nrows, 0, RC, S);
      for (int r0 = 0; r0 < nrows; r0 += RC) {
        chunk_store(reg, buf12, ldr, RC, S, S8, side == 0 ? Di : nullptr);
        __syncthreads();
        unsigned long long q1 = clock64();
        if (r0 + RC < nrows) chunk_fetch(reg, src, nrows, nrows, r0 + RC, RC, S);
        const int rows = nrows - r0 < RC ? nrows - r0 : RC;
        gram_accum(acc, buf12, ldr, (rows + 3) >> 2, nt, KG);
        __syncthreads();
        unsigned long long q2 = clock64();
        if (threadIdx.x == 0) { atomicAdd(&g_upprof[12], q1 - q0); atomicAdd(&g_upprof[13], q2 - q1); }
        q0 = q2;
      }
      unsigned long long q3 = clock64();
      gram_store(acc, side == 0 ? RA : RB, S, nt, KG, buf12);
      if (threadIdx.x == 0) atomicAdd(&g_upprof[14], clock64() - q3);
    }
    unsigned long long t1 = clock64();
    const double r1 = chol2_packed(RA, ia, RB, ib, S);
    if (!(r1 > kCholFloorP)) {  // uniform: ill-conditioned factors -> legacy (Householder) path
      if (threadIdx.x == 0) *d.rank = -1;
      continue;
    }
    if (threadIdx.x == 0) atomicAdd(&g_upprof[15], clock64() - t1);
    // ---- M = R1_B D R1_A^T -> W (col-major: W[i + j ld] = M[i][j])
    for (int e = threadIdx.x; e < S * ld; e += PT) {
      const int j = e / ld, i = e - j * ld;
      double a = 0.0;
      if (i < S) {
        const double* rb = RB + tri_off(i, S);
        const double* ra = RA + tri_off(j, S);
        for (int l = (i > j ? i : j); l < S; ++l) a = fma(rb[l] * Dv[l], ra[l], a);
      }
      W[e] = a;
    }
    unsigned long long t2 = clock64();
    // Second CholeskyQR pass only when the Cholesky pivots do not already
    // bound the loss of orthogonality: |Q1^T Q1 - I| ~ eps cond(L)^2 and
    // 1 / r1 estimates cond(L)^2, so r1 >= kSkipRatio keeps it near 1e-13.
    // That perturbs the core's singular values by ~1e-13 |D_0| (D_0, the
    // first ACA pivot, is the core's scale); the single pass is taken only
    // when this stays below 1e-6 of the rank threshold, the margin the
    // two-pass path keeps at every epsilon (at eps = 1e-10 a single pass
    // moved 4 of ~20,000 rank decisions of the c2 configuration).
    const bool second = !(r1 >= kSkipRatio && 1e-13 * fabs(Dv[0]) <= 1e-6 * thr);
    if (second) {
    // ---- pass 2: Q1 = L R1^-1 (in place in global memory), E = Q1^T Q1 - I
    for (int side = 0; side < 2; ++side) {
      double* src = side == 0 ? gX : gY;
      const int nrows = side == 0 ? m : C;
      const double* R = side == 0 ? RA : RB;
      const double* ri = side == 0 ? ia : ib;
      const int RC = RC12, ldr = RC + 4;
      // side 1 reuses acc after side 0's accumulators moved to registers ea
#pragma unroll
      for (int q = 0; q < P_TILES; ++q) acc[q][0] = acc[q][1] = 0.0;
      chunk_fetch(reg, src, nrows, nrows, 0, RC, S);
      for (int r0 = 0; r0 < nrows; r0 += RC) {
        chunk_store(reg, buf12, ldr, RC, S, S8, side == 0 ? Di : nullptr);
        __syncthreads();
        if (r0 + RC < nrows) chunk_fetch(reg, src, nrows, nrows, r0 + RC, RC, S);
        const int rows = nrows - r0 < RC ? nrows - r0 : RC;
        trsm_chunk(buf12, ldr, rows, R, ri, S);
        __syncthreads();
        chunk_writeback(buf12, ldr, RC, src, nrows, nrows, r0, S);
        gram_accum(acc, buf12, ldr, (rows + 3) >> 2, nt, KG);
        __syncthreads();
      }
      // RA / RB are separate: side 0's G2 may replace its R1 right away
      gram_store(acc, side == 0 ? RA : RB, S, nt, KG, buf12);
    }
    // ---- U = triu(E, 1) + diag(E) / 2 in place; max |E|
    double emax = 0.0;
    for (int e = threadIdx.x; e < 2 * S; e += PT) {
      double* G = e < S ? RA : RB;
      const int i = e < S ? e : e - S;
      const double dd = G[tri_off(i, S) + i] - 1.0;
      emax = fmax(emax, fabs(dd));
      G[tri_off(i, S) + i] = 0.5 * dd;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 2 * tri; e += PT) {
      const double v = (e < tri ? RA : RB)[e < tri ? e : e - tri];
      emax = fmax(emax, fabs(v));  // diagonal entries are already halved: still a bound
    }
    emax = warp_max(emax);
    if (lane == 0) s_red[warp] = emax;
    __syncthreads();
    emax = 0.0;
    for (int w = 0; w < PW; ++w) emax = fmax(emax, s_red[w]);
    if (!(emax <= kOrthFloor)) {  // uniform
      if (threadIdx.x == 0) *d.rank = -1;
      continue;
    }
    // ---- W += U_B M + M U_A^T (first order in E), correction staged in V
    for (int e = threadIdx.x; e < S * ld; e += PT) {
      const int j = e / ld, i = e - j * ld;
      double a = 0.0;
      if (i < S) {
        const double* ub = RB + tri_off(i, S);
        for (int l = i; l < S; ++l) a = fma(ub[l], W[l + j * ld], a);
        const double* ua = RA + tri_off(j, S);
        for (int l = j; l < S; ++l) a = fma(W[i + l * ld], ua[l], a);
      }
      V[e] = a;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < S * ld; e += PT) W[e] += V[e];
    }  // second
    __syncthreads();
    unsigned long long t3 = clock64();
    // ---- core SVD
    const int nsw = jacobi_p(W, V, S, ld);
    unsigned long long t4 = clock64();
    sv_order_p(W, S, ld, sig, order);
    int kk = 0;
    for (int j = 0; j < S; ++j) kk += sig[order[j]] > thr;
    const int mr = d.min_rank < S ? d.min_rank : S;
    const int k = kk > mr ? kk : mr;
    if (second) {
      // Z_A = (I - U_A) phi (in V), Z_B = (I - U_B) sigma psi (in W); pass 3
      // multiplies the stored Q1
      apply_inv_r2(V, ld, RA, S);
      apply_inv_r2(W, ld, RB, S);
    } else {
      // Z_A = R1_A^-1 phi_k, Z_B = R1_B^-1 sigma psi_k; pass 3 multiplies L and Y
      backsolve(V, ld, order, k, RA, ia, S);
      backsolve(W, ld, order, k, RB, ib, S);
      __syncthreads();
    }
    unsigned long long t5 = clock64();
    // ---- pass 3: outputs
    if (k > 0) {
      for (int side = 0; side < 2; ++side) {
        const double* src = side == 0 ? gX : gY;
        const int nrows = side == 0 ? m : C;
        const double* Z = side == 0 ? V : W;
        const int RC = RC3, ldr = RC + 4;
        chunk_fetch(reg, src, nrows, nrows, 0, RC, S);
        for (int r0 = 0; r0 < nrows; r0 += RC) {
          chunk_store(reg, buf3, ldr, RC, S, S8, (!second && side == 0) ? Di : nullptr);
          __syncthreads();
          if (r0 + RC < nrows) chunk_fetch(reg, src, nrows, nrows, r0 + RC, RC, S);
          const int rows = nrows - r0 < RC ? nrows - r0 : RC;
          if (side == 0) {
            out_tiles(buf3, ldr, rows, Z, ld, order, k, S8, [&](int row, int a, double v) {
              d.NB[(size_t)(r0 + row) * d.nb_r + (size_t)a * d.nb_c] = v;
            });
          } else {
            out_tiles(buf3, ldr, rows, Z, ld, order, k, S8, [&](int row, int a, double v) {
              const int i = r0 + row;
              if (i < ko) d.OM[(size_t)a * ko + i] = v / d.w[i];
              else d.FM[(size_t)a * d.k_f + (i - ko)] = v / d.wf[i - ko];
            });
          }
          __syncthreads();
        }
      }
    }
    for (int a = threadIdx.x; a < k; a += PT) d.NW[a] = sig[order[a]];
    if (threadIdx.x == 0) {
      *d.rank = k;
      unsigned long long t6 = clock64();
      atomicAdd(&g_upprof[0], t1 - t0);  // Gram 1
      atomicAdd(&g_upprof[1], t2 - t1);  // Cholesky + M
      atomicAdd(&g_upprof[2], t3 - t2);  // TRSM + Gram 2 + corrections
      atomicAdd(&g_upprof[3], t4 - t3);  // Jacobi
      atomicAdd(&g_upprof[4], t5 - t4);  // order + Z
      atomicAdd(&g_upprof[5], t6 - t5);  // outputs
      atomicAdd(&g_upprof[6], 1ull);
      atomicAdd(&g_upprof[7], (unsigned long long)S);
      atomicAdd(&g_upprof[8], (unsigned long long)m);
      atomicAdd(&g_upprof[9], (unsigned long long)nsw);
      atomicAdd(&g_upprof[10], (unsigned long long)k);
      atomicAdd(&g_upprof[11], (unsigned long long)second);
    }

  }
}

}  // namespace

bool union_post_eligible(int m, int k_old, int k_f) {
  const int C = k_old + k_f;
  return (m < C ? m : C) <= P_SMAX;
}

void launch_union_post(const UnionDesc* d_descs, int n, double thr, cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_union_post"};
  if (n <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(union_post_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM * 8);
    attr = true;
  }
  union_post_kernel<<<n < 4096 ? n : 4096, PT, (size_t)P_SMEM * 8, s>>>(d_descs, n, thr);
}

}  // namespace ifmm
