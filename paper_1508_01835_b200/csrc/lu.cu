// Blocked right-looking LU with partial pivoting for pivot blocks larger
// than one CTA's shared memory (upper-level clusters, top-level system).
#include "engine.h"

namespace ifmm {

void lu_blocked(Ctx& C, double* A, int n, int lda, int* piv, int tag) {
  const int nb = 32;
  for (int j0 = 0; j0 < n; j0 += nb) {
    const int jb = std::min(nb, n - j0);
    launch_panel_lu(A, n, lda, j0, jb, piv, C.d_status, tag, C.st);
    launch_laswp(A, n, lda, j0, jb, piv, C.st);
    const int rest = n - j0 - jb;
    if (rest > 0) {
      double* A12 = A + (size_t)j0 * lda + j0 + jb;
      launch_trsm_lunit(A + (size_t)j0 * lda + j0, lda, jb, A12, lda, rest, C.st);
      GemmBatch gb;
      gb.add(A + (size_t)(j0 + jb) * lda + j0, lda, 0, A12, lda, 0,
             A + (size_t)(j0 + jb) * lda + j0 + jb, lda, rest, rest, jb, -1.0, 1.0);
      gb.run(C);
    }
    C.launches += 3;
  }
  launch_finite_check(A, n, lda, C.d_status, tag, C.st);
  CUDA_CHECK(cudaGetLastError());
}

}  // namespace ifmm
