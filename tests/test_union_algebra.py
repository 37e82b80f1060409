"""CPU check of the algebra the CUDA union kernel uses (dense.cu union_kernel).

The kernel keeps the reference's full-pivot ACA (lowrank.py:128-151) but
factors its output differently from the reference's Householder QR-QR-SVD
(lowrank.py:153-163):

  * X = P L~ D (unit lower trapezoidal L~, pivots D) and Y are orthonormalised
    by two CholeskyQR passes of L~ and Y;
  * the core is R_A D R_B^T and its SVD is taken by one-sided Jacobi on the
    transpose, so the new basis is Q_A phi and the maps come from Q_B sigma psi.

This test restates those steps in numpy and checks them against the oracle's
reference-order union (oracle/ifmm_np.py basis_union) and the reference
known-answer vectors (tests/golden/kat_lowrank.npz): identical ranks, weights
to 1e-12 relative, and the same basis / maps up to column signs.
"""

import numpy as np
import pytest

from conftest import load_golden
from oracle import ifmm_np as O


def _aca_factors(M, thr, min_rank=0, margin=8.0):
    """Full-pivot ACA (same pivots as oracle.aca): residual columns and rows/pivot."""
    R = np.array(M, dtype=float, copy=True)
    cs, rs, piv = [], [], []
    for _ in range(min(M.shape)):
        p, q = np.unravel_index(np.argmax(np.abs(R)), R.shape)
        v = R[p, q]
        if v == 0.0 or (abs(v) <= thr / margin and len(cs) >= min_rank):
            break
        c = R[:, q].copy()
        r = R[p, :] / v
        cs.append(c)
        rs.append(r)
        piv.append(v)
        R -= np.outer(c, r)
    return np.column_stack(cs), np.vstack(rs).T, np.array(piv)


def _cholqr2(A):
    R1 = np.linalg.cholesky(A.T @ A).T
    Q1 = np.linalg.solve(R1.T, A.T).T
    R2 = np.linalg.cholesky(Q1.T @ Q1).T
    Q = np.linalg.solve(R2.T, Q1.T).T
    return Q, R2 @ R1


def kernel_union(B, w, F, wf, thr, min_rank=0):
    k0 = B.shape[1]
    M = np.hstack([B * w, F * wf])
    X, Y, D = _aca_factors(M, thr, min_rank)
    QA, RA = _cholqr2(X / D)
    QB, RB = _cholqr2(Y)
    coreT = RB @ np.diag(D) @ RA.T
    U, s, Vt = np.linalg.svd(coreT)          # coreT = psi S phi^T
    k = max(int(np.sum(s > thr)), min(min_rank, len(s)))
    basis = QA @ Vt[:k].T                   # Q_A phi
    smaps = QB @ (U[:, :k] * s[:k])         # Q_B sigma psi
    return basis, s[:k], smaps[:k0].T / w[None, :], smaps[k0:].T / wf[None, :], \
        np.linalg.cond(X / D), np.linalg.cond(Y)


def _match_signs(A, B):
    sg = np.sign(np.sum(A * B, axis=0))
    sg[sg == 0] = 1.0
    return B * sg


def _check(B, w, F, wf, thr):
    ref = O.basis_union(B, w, F, wf, thr)
    nb, nw, om, fm, cx, cy = kernel_union(B, w, F, wf, thr)
    assert nb.shape[1] == ref.rank
    np.testing.assert_allclose(nw, ref.weights, rtol=1e-12, atol=1e-14 * ref.weights[0])
    sg = np.sign(np.sum(nb * ref.basis, axis=0))
    np.testing.assert_allclose(nb * sg, ref.basis, atol=1e-9)
    np.testing.assert_allclose(om * sg[:, None], ref.old_map, atol=1e-9 * np.abs(ref.old_map).max())
    np.testing.assert_allclose(fm * sg[:, None], ref.fill_map, atol=1e-9 * np.abs(ref.fill_map).max())
    return cx, cy


def test_union_algebra_reference_kat():
    g = load_golden("kat_lowrank")
    thr = 1e-6 * float(np.max(g["w"]))
    _check(g["B"], g["w"], g["F"], g["wf"], thr)


@pytest.mark.parametrize("m,k0,kf,decay", [(64, 30, 6, 0.5), (120, 50, 12, 0.7), (300, 60, 8, 0.8),
                                           (40, 40, 10, 0.3)])
def test_union_algebra_graded(m, k0, kf, decay):
    rng = np.random.default_rng(m + k0)
    B, _ = np.linalg.qr(rng.standard_normal((m, k0)))
    F, _ = np.linalg.qr(rng.standard_normal((m, kf)))
    w = np.sort(decay ** np.arange(k0) * (1 + rng.random(k0)))[::-1]
    wf = np.sort(decay ** np.arange(kf) * (1 + rng.random(kf)))[::-1] * 0.3
    cx, cy = _check(B, w, F, wf, 1e-7 * w[0])
    # L~ and Y stay well conditioned (the premise of CholeskyQR)
    assert cx < 1e4 and cy < 1e4
