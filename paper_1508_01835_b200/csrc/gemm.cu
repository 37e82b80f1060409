// Grouped fp64 GEMM on the FP64 tensor pipe (mma.sync m8n8k4 f64 -> DMMA) for
// the elimination's dense products (Schur fills factor.py:283-290, rebases
// factor.py:395-430, K rewrites factor.py:478-512, merges, blocked LU
// updates): C = alpha op(A) op(B) + beta C over a list of problems, one
// persistent CTA loop over the output tiles of the whole list.
//
// Operand tiles are staged global -> shared with cp.async (LDGSTS, 8-byte
// elements, zero-fill outside the matrix) through a 3-stage ring, one
// __syncthreads per 16-deep k tile.  Each operand tile is kept in the layout
// its global matrix is contiguous in -- [row][k] (ld 20) when k is the
// contiguous index, [k][row] (ld rows + 4) otherwise -- so the copies are
// coalesced and both layouts give conflict-free DMMA fragment reads (a
// half-warp's 16 (row, k) addresses fall in 16 different 8-byte banks).
// One tile shape, 64 x 64 (4 warps of 32 x 32, 3 CTAs per SM): a 128 x 128
// variant (8 warps of 32 x 64, 1 CTA per SM) measured no faster at any size
// and much slower on mid-size problems (wave quantisation), so it was removed.
#include "common.cuh"
#include "dense.h"
#include "runtime.h"

namespace ifmm {

namespace {

constexpr int G_BK = 16;      // k depth of a stage
constexpr int G_STAGES = 3;
constexpr int G_LDK = 20;     // [row][k] layout: row stride (20 mod 16 = 4)

IFMM_DEV void cp_async8(double* smem_dst, const double* gsrc, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gsrc), "r"(sz));
}
IFMM_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
IFMM_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// One operand tile (R rows x 16 k) of op(X) into a stage.  kcontig: X is
// stored [row][k] (k contiguous, leading dimension ld), else [k][row].
template <int R, int NT>
IFMM_DEV void stage_tile(double* dst, const double* __restrict__ X, int ld, bool kcontig, int r0,
                         int k0, int nrows, int nk) {
  const int t = threadIdx.x;
  if (kcontig) {
    const int k = t & 15, gk = k0 + k;
    const bool kv = gk < nk;
#pragma unroll
    for (int i = 0; i < R * 16 / NT; ++i) {
      const int r = (t >> 4) + i * (NT / 16), gr = r0 + r;
      const bool v = kv && gr < nrows;
      cp_async8(dst + r * G_LDK + k, v ? X + (size_t)gr * ld + gk : X, v);
    }
  } else {
    const int r = t % R, gr = r0 + r;
    const bool rv = gr < nrows;
#pragma unroll
    for (int i = 0; i < R * 16 / NT; ++i) {
      const int k = t / R + i * (NT / R), gk = k0 + k;
      const bool v = rv && gk < nk;
      cp_async8(dst + k * (R + 4) + r, v ? X + (size_t)gk * ld + gr : X, v);
    }
  }
}

template <int BM, int BN, int WM, int WN, int MINB>
__global__ void __launch_bounds__(WM * WN * 32, MINB)
gemm_grouped_kernel(const GemmDesc* __restrict__ descs, const int* __restrict__ tstart, int nprob,
                    int total) {
  constexpr int NT = WM * WN * 32;
  constexpr int TM = BM / WM / 8, TN = BN / WN / 8;  // 8x8 DMMA tiles per warp
  constexpr int SA = BM * G_LDK, SB = BN * G_LDK;    // doubles per stage (>= 16 (B? + 4))
  extern __shared__ double gsm[];
  double* As = gsm;
  double* Bs = gsm + G_STAGES * SA;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int fr = lane >> 2, fk = lane & 3;

  for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
    int lo = 0, hi = nprob - 1;  // largest p with tstart[p] <= tile
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tstart[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const GemmDesc d = descs[lo];
    const int local = tile - tstart[lo];
    const int tiles_n = (d.N + BN - 1) / BN;
    const int m0 = (local / tiles_n) * BM, n0 = (local % tiles_n) * BN;
    const bool ak = d.ta == 0, bk = d.tb != 0;  // k contiguous in the stored operand
    const int a_sr = ak ? G_LDK : 1, a_sk = ak ? 1 : BM + 4;
    const int b_sr = bk ? G_LDK : 1, b_sk = bk ? 1 : BN + 4;

    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nk = (d.K + G_BK - 1) / G_BK;
#pragma unroll
    for (int s = 0; s < G_STAGES - 1; ++s) {
      if (s < nk) {
        stage_tile<BM, NT>(As + s * SA, d.A, d.lda, ak, m0, s * G_BK, d.M, d.K);
        stage_tile<BN, NT>(Bs + s * SB, d.B, d.ldb, bk, n0, s * G_BK, d.N, d.K);
      }
      cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
      cp_async_wait<G_STAGES - 2>();
      __syncthreads();
      const int nxt = kt + G_STAGES - 1;
      if (nxt < nk) {
        const int s = nxt % G_STAGES;
        stage_tile<BM, NT>(As + s * SA, d.A, d.lda, ak, m0, nxt * G_BK, d.M, d.K);
        stage_tile<BN, NT>(Bs + s * SB, d.B, d.ldb, bk, n0, nxt * G_BK, d.N, d.K);
      }
      cp_async_commit();
      const double* a = As + (kt % G_STAGES) * SA + (wm * (BM / WM) + fr) * a_sr + fk * a_sk;
      const double* b = Bs + (kt % G_STAGES) * SB + (wn * (BN / WN) + fr) * b_sr + fk * b_sk;
#pragma unroll
      for (int k4 = 0; k4 < G_BK; k4 += 4) {
        double af[TM], bf[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) af[i] = a[i * 8 * a_sr + k4 * a_sk];
#pragma unroll
        for (int j = 0; j < TN; ++j) bf[j] = b[j * 8 * b_sr + k4 * b_sk];
        if (d.dscale) {
          const int gk = kt * G_BK + k4 + fk;
          const double sc = gk < d.K ? d.dscale[gk] : 0.0;
#pragma unroll
          for (int i = 0; i < TM; ++i) af[i] *= sc;
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    cp_async_wait<0>();
    // epilogue: lane holds C[fr][2 fk + {0, 1}] of each 8x8 tile
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int gm = m0 + wm * (BM / WM) + i * 8 + fr;
      if (gm >= d.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int gn = n0 + wn * (BN / WN) + j * 8 + 2 * fk + e;
          if (gn >= d.N) continue;
          double* c = d.C + (size_t)gm * d.ldc + gn;
          double v = d.alpha * acc[i][j][e];
          if (d.beta != 0.0) v += d.beta * (*c);
          *c = v;
        }
      }
    }
    __syncthreads();  // the next tile's prologue overwrites the ring
  }
}

template <int BM, int BN>
constexpr size_t gemm_smem_bytes() { return (size_t)G_STAGES * (BM + BN) * G_LDK * sizeof(double); }

}  // namespace

void gemm_tile_dims(int* bm, int* bn) {
  *bm = 64;
  *bn = 64;
}

void launch_gemm(const GemmDesc* d_descs, const int* d_tile_start, int nprob, int total_tiles,
                 cudaStream_t s) {
  DbgSync dbg_sync_{s, "launch_gemm"};
  if (total_tiles <= 0) return;
  static bool init = false;
  if (!init) {
    CUDA_CHECK(cudaFuncSetAttribute(gemm_grouped_kernel<64, 64, 2, 2, 3>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)gemm_smem_bytes<64, 64>()));
    init = true;
  }
  const int grid = total_tiles < 148 * 3 ? total_tiles : 148 * 3;  // 60 KB: 3 CTAs / SM
  gemm_grouped_kernel<64, 64, 2, 2, 3><<<grid, 128, gemm_smem_bytes<64, 64>(), s>>>(
      d_descs, d_tile_start, nprob, total_tiles);
}

}  // namespace ifmm
