// Batched small dense fp64 linear algebra on sm_100a: host-side launch API.
// All matrices are fp64; "row-major with leading dimension" unless stated.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ifmm {

// C[M,N] = alpha * op(A) * diag(dscale) * op(B) + beta * C   (row-major)
// op(A) is M x K: ta==0 -> A[m*lda+k], ta==1 -> A[k*lda+m]
// op(B) is K x N: tb==0 -> B[k*ldb+n], tb==1 -> B[n*ldb+k]
struct GemmDesc {
  const double* A;
  const double* B;
  double* C;
  const double* dscale;  // optional K-length column scale of op(A)
  int M, N, K;
  int lda, ldb, ldc;
  int ta, tb;
  double alpha, beta;
};

// Strided block copy / accumulate:  dst(i,j) = alpha*src(i,j) [+ dst(i,j)]
// src(i,j) = src[i*ss_r + j*ss_c]; dst(i,j) = dst[i*ds_r + j*ds_c].
// mode 0: copy, 1: add, 2: set to alpha*I (src ignored), 3: zero, 4: fill alpha.
struct CopyDesc {
  const double* src;
  double* dst;
  int rows, cols;
  int ss_r, ss_c, ds_r, ds_c;
  int mode;
  double alpha;
  const double* rscale;  // optional per-row scale (modes 0/1)
};

// Truncated SVD of a strided m x n block (fill compression, factor.py:329).
// Output: rank[0] = #{sigma > thr}; U (m x min) col-major ld m,
// S (min), V (n x min) col-major ld n.  Frobenius pre-filter: if
// ||F||_F <= thr*(1-1e-12) the rank is 0 without running Jacobi.
struct SvdDesc {
  const double* src;
  int m, n, s_r, s_c;
  double* U;
  double* S;
  double* V;
  int* rank;
  double* work;  // >= max(m,n)*min(m,n) + min^2 doubles (global fallback)
};

// Weighted basis union (lowrank.py:166-199) through full-pivot ACA +
// QR-QR-SVD (lowrank.py:128-163).  Old basis B(i,a) = B[i*b_r + a*b_c]
// (m x k_old), fill basis F(i,a) = F[i*f_r + a*f_c] (m x k_f).
// Output rank -> *rank; new basis written to NB(i,a) = NB[i*nb_r + a*nb_c]
// (capacity m x min(m, k_old+k_f)), weights NW, old_map OM (k_new x k_old,
// row-major ld k_old), fill_map FM (k_new x k_f, row-major ld k_f).
struct UnionDesc {
  const double* B;
  const double* w;
  const double* F;
  const double* wf;
  int m, k_old, k_f;
  int b_r, b_c, f_r, f_c;
  int min_rank;
  double* NB;
  int nb_r, nb_c;
  double* NW;
  double* OM;
  double* FM;
  int* rank;
  double* work;
  int giant;  // set by the launcher: 1 = multi-CTA giant path, 2 = register ACA ran, 3 = register ACA + union_post
};

__host__ __device__ size_t union_work_doubles(int m, int k_old, int k_f);
__host__ __device__ size_t svd_work_doubles(int m, int n);
// doubles of dynamic smem launch_svd uses for a given max_smem_dim (0: none)
size_t svd_smem_doubles(int max_smem_dim);

// Host launchers.  `descs` / side arrays must already be device-resident.
// (gemm.cu) d_tile_start: prefix sums of the problems' output-tile counts for
// the tile shape gemm_tile_dims reports (64 x 64).
void gemm_tile_dims(int* bm, int* bn);
void launch_gemm(const GemmDesc* d_descs, const int* d_tile_start, int nprob,
                 int total_tiles, cudaStream_t s);
void launch_copy(const CopyDesc* d_descs, int n, cudaStream_t s);
// rel_mode: thr is relative to sigma_max and rank >= 1 (h2.py:124-127).
void launch_svd(const SvdDesc* d_descs, int n, double thr, int max_smem_dim,
                cudaStream_t s, int rel_mode = 0);
bool union_fits_smem(int m, int k_old, int k_f);
// smem: all workspaces fit shared memory; otherwise jac_smem_doubles (<= 28500)
// of dynamic shared memory hold the core SVD when 2 s^2 fits.
// d_giants / n_giants: the subset (giant != 0) whose core SVD runs on several
// CTAs (cooperative launch between the two halves); d_flags: 64 uints per giant.
// d_scratch: union_giant_scratch_doubles(n_giants) doubles.
void launch_union(const UnionDesc* d_descs, int n, double thr, cudaStream_t s, int smem,
                  int jac_smem_doubles = 0, const UnionDesc* d_giants = nullptr, int n_giants = 0,
                  int max_giant_s = 0, double* d_scratch = nullptr, int max_giant_m = 0,
                  int max_giant_C = 0, int sm_reserved = 0);
// 64 flag words (32 doubles) per giant, the done counter (8 doubles), then 2
// candidate slots per CTA of the cooperative ACA grid: that grid has at most
// max(sm_free, n_giants) <= max(148, n_giants) CTAs.
inline int union_giant_scratch_doubles(int n_giants) {
  return 32 * n_giants + 8 + 2 * (n_giants > 148 ? n_giants : 148) + 8;
}
// giants per launch: beyond this the rest of a wave's large unions take the
// single-CTA global-workspace path (every cooperative grid stays co-resident)
constexpr int kMaxGiantsPerLaunch = 96;
// s_max above which a global-workspace union is "giant" (multi-CTA ACA,
// CholeskyQR, core SVD and output); IFMM_GIANT overrides (diagnostics)
int giant_union_threshold();
// Register-resident ACA (union_aca.cu) for the unions whose desc has giant ==
// 2 (union_kernel then starts at the CholeskyQR).  union_aca_reg_class picks
// the register tile (G CTAs per cluster, ER rows per warp slot, EC column
// slots per lane) for the batch's largest m / C; false: keep the legacy ACA.
bool union_aca_reg_class(int max_m, int max_C, int* G, int* ER, int* EC);
void launch_union_aca_reg(const UnionDesc* d_descs, int n, double thr, int G, int ER, int EC,
                          cudaStream_t s);
// Fused second half (union_post.cu) for the register-ACA unions with
// min(m, C) <= 96 (desc.giant == 3): CholeskyQR2 + core Jacobi + outputs, one
// CTA per union, everything on chip.  A union it cannot take gets rank -1
// (the host reruns it on the legacy path with giant = 0).
bool union_post_eligible(int m, int k_old, int k_f);
void launch_union_post(const UnionDesc* d_descs, int n, double thr, cudaStream_t s);
void union_post_profile(unsigned long long* out, int reset);

// LU with partial pivoting (getrf semantics) of row-major n x n matrices,
// in place; piv is 0-based (row j swapped with piv[j]).  status[0] is set to
// (tag+1) when a pivot is zero or non-finite (first error wins).
struct LuDesc {
  double* A;
  int n, lda;
  int* piv;
  int tag;
};
void launch_lu(const LuDesc* d_descs, int n, int* d_status, cudaStream_t s);

// Multi-RHS LU solve X <- P^{-1} X for row-major X (n x nrhs, ld ldx).
struct LuSolveDesc {
  const double* LU;
  const int* piv;
  int n, lda;
  double* X;
  int nrhs, ldx;
};
// max_n (largest system) <= 800 selects the shared-memory kernel.
void launch_lusolve(const LuSolveDesc* d_descs, int ndesc, int max_nrhs,
                    cudaStream_t s, int max_n = 0);

}  // namespace ifmm

namespace ifmm {

// initialize_weights, rigorous (h2.py:210-230): H = hstack_q K(j,q) stored
// row-major k x W.  Output P (k x k row-major, left singular vectors,
// completed to an orthogonal matrix as _complete_basis h2.py:234-239) and
// the padded weights w (k) (_pad_weights h2.py:242-247).  H is clobbered.
struct WeightDesc {
  double* H;
  int k, W;
  double* P;
  double* w;
  double* work;
};
size_t weights_work_doubles(int k, int W);
void launch_weights(const WeightDesc* d_descs, int n, cudaStream_t s);

// Orthonormal basis (Householder QR) of a tall row-major n x w matrix Y
// (np.linalg.qr(Y)[0], lowrank.py:74-76); single CTA.  work >= 2*n*w+2*w.
void launch_tall_orth(const double* Y, int n, int w, double* Q, double* work, cudaStream_t s);
// Largest singular value of a tall row-major n x w matrix; single CTA.
// the same on the whole grid (tall.cu: CholeskyQR2, w <= 12); *flag is raised
// on a Cholesky breakdown
bool tall_grid_supported(int w);
size_t tall_grid_work_doubles(int w);
void launch_tall_orth_grid(const double* Y, int n, int w, double* Q, double* work, int* flag,
                           cudaStream_t s);
void launch_tall_sigmax_grid(const double* Y, int n, int w, double* out, double* work,
                             cudaStream_t s);
void launch_tall_sigmax(const double* Y, int n, int w, double* out, double* work,
                        cudaStream_t s);

}  // namespace ifmm

namespace ifmm {
// Blocked right-looking LU pieces (row-major, panel width jb).
void launch_panel_lu(double* A, int n, int lda, int j0, int jb, int* piv, int* status, int tag,
                     cudaStream_t s);
void launch_laswp(double* A, int n, int lda, int j0, int jb, const int* piv, cudaStream_t s);
// X (nb x ncols, ld ldx) <- L^{-1} X with L unit lower (nb x nb, ld ldl)
void launch_trsm_lunit(const double* L, int ldl, int nb, double* X, int ldx, int ncols,
                       cudaStream_t s);
void launch_finite_check(const double* A, int n, int lda, int* status, int tag, cudaStream_t s);
// _extend_update core: append `extra` orthonormalised directions (from the
// Gaussian block G, col-major m x extra) to NB (col-major, first k columns
// orthonormal) and weights NW[k..] = max(thr, 1e-14*max(NW[0:k])).
void launch_extend(double* NB, int m, int k, const double* G, int extra, double* NW, double thr,
                   double* work, cudaStream_t s);
}  // namespace ifmm

namespace ifmm {
void union_profile(unsigned long long* out, int reset);
}

namespace ifmm {
// ---- randomized SVD pieces for large fills (lowrank.py:79-125) ----
// Gaussian sketch: out (n x w row-major) ~ N(0,1), counter-based (seed, tag)
struct RandDesc {
  double* out;
  int count;            // n * w
  unsigned long long key;
};
void launch_randn(const RandDesc* d, int n, cudaStream_t s);
// Orthonormal basis of a col-major m x w block, in place (Householder QR +
// explicit Q).  work >= m*w + w doubles per desc.
struct OrthDesc {
  double* Y;   // col-major m x w (ld m) -> overwritten with Q
  int m, w;
  double* work;
};
void launch_orth(const OrthDesc* d, int n, cudaStream_t s);
// SVD of B (w x n) given B^T col-major (n x w, ld n); U = Q Wb (m x keep,
// col-major ld m), S, V (n x keep col-major ld n).  rank = #{s > thr}
// (capped), flag[0] = 1 when the reference's doubling test says "stop"
// (width >= full or k_try >= cap or s[k_try] <= thr).
struct RsvdFinDesc {
  double* Bt;        // n x w col-major (clobbered)
  const double* Q;   // m x w col-major
  int m, n, w, k_try, full;
  double* U;
  double* S;
  double* V;
  int* rank;
  int* stop;
  double* work;      // >= w*w + 2w + 8
};
void launch_rsvd_fin(const RsvdFinDesc* d, int n, double thr, cudaStream_t s);
}  // namespace ifmm

namespace ifmm {
void jacobi_bench(const double* A, int s, int reps, int threads, unsigned long long* d_out,
                  cudaStream_t st);
}
