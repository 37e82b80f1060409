"""Low-rank primitives on the device (mirror of ``ifmm.lowrank``,
lowrank.py:1-199).

Public functions of the reference with the same arguments, results and
errors; the arithmetic runs in the engine's kernels -- the same ones the
factorization uses (``ifmm_dev_svd``: rank-revealing pivoted QR + one-sided
Jacobi; ``ifmm_dev_union``: full-pivot ACA + CholeskyQR2 + Jacobi core SVD;
``ifmm_dev_orth``: Householder QR).  Inputs and outputs are numpy arrays;
the sketch draws of ``randomized_svd`` come from the caller's numpy
Generator exactly as in the reference.  Truncation thresholds are absolute.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable

import numpy as np

from . import _native as N

ACA_MARGIN = 8.0  # the union kernel's fixed pivot floor: thr / 8 (lowrank.py:128)


@dataclass
class LowRankFactor:
    U: np.ndarray       # (m, k), orthonormal columns
    sigma: np.ndarray   # (k,), non-increasing, > 0
    V: np.ndarray       # (n, k), orthonormal columns

    @property
    def rank(self) -> int:
        return len(self.sigma)

    def matrix(self) -> np.ndarray:
        if self.rank == 0:
            return np.zeros((self.U.shape[0], self.V.shape[0]))
        return (self.U * self.sigma) @ self.V.T


@dataclass
class BasisUpdate:
    new_basis: np.ndarray    # (m, k_new), orthonormal
    new_weights: np.ndarray  # (k_new,)
    old_map: np.ndarray      # (k_new, k_old): old_basis ~= new_basis @ old_map
    fillin_map: np.ndarray   # (k_new, k_fill)

    @property
    def rank(self) -> int:
        return self.new_basis.shape[1]


def _empty(m, n):
    return LowRankFactor(np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0)))


def _torch():
    import torch
    return torch


def _dev(a):
    return _torch().from_numpy(np.ascontiguousarray(a, dtype=float)).cuda()


def _zeros(n, dtype=None):
    t = _torch()
    return t.zeros(max(int(n), 1), dtype=dtype or t.float64, device="cuda")


def _p(t):
    return C.c_void_p(t.data_ptr())


def _svd_all(M: np.ndarray, thr: float):
    """Device truncated SVD of a dense block: (U, s, V) of the triplets with
    s > thr (thr < 0: all of them)."""
    m, n = M.shape
    k = min(m, n)
    dA = _dev(M)
    dU, dS, dV = _zeros(m * k), _zeros(k), _zeros(n * k)
    dr = _zeros(1, _torch().int32)
    _torch().cuda.synchronize()
    N.check(N.lib().ifmm_dev_svd(N.ctx(), m, n, _p(dA), float(thr), _p(dU), _p(dS), _p(dV),
                                 _p(dr)))
    r = int(dr.item())
    U = dU.cpu().numpy()[:m * r].reshape(r, m).T.copy()
    V = dV.cpu().numpy()[:n * r].reshape(r, n).T.copy()
    return U, dS.cpu().numpy()[:r].copy(), V


def truncated_svd(M: np.ndarray, abs_threshold: float) -> LowRankFactor:
    """lowrank.py:54-61: exactly the triplets with sigma > threshold."""
    M = np.asarray(M, dtype=float)
    if M.size == 0:
        return _empty(*M.shape)
    U, s, V = _svd_all(M, abs_threshold)
    return LowRankFactor(U, s, V)


def rank_from_reference(sigmas: np.ndarray, epsilon: float, sigma0_ref: float) -> int:
    """lowrank.py:64-72: #{sigma > epsilon * sigma0_ref}."""
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must be in (0, 1)")
    if sigma0_ref <= 0.0:
        raise ValueError("sigma0_ref must be positive")
    return int(np.count_nonzero(np.asarray(sigmas, dtype=float) > epsilon * sigma0_ref))


def _orth(Y: np.ndarray) -> np.ndarray:
    n, w = Y.shape
    dY = _dev(Y)
    dQ = _zeros(n * w)
    _torch().cuda.synchronize()
    N.check(N.lib().ifmm_dev_orth(N.ctx(), n, w, _p(dY), _p(dQ)))
    return dQ.cpu().numpy()[:n * w].reshape(n, w)


def randomized_svd(apply: Callable, apply_t: Callable, m: int, n: int, abs_threshold: float,
                   oversample: int = 10, power_iters: int = 2,
                   rng: np.random.Generator | None = None, start_rank: int = 16,
                   max_rank: int | None = None) -> LowRankFactor:
    """lowrank.py:79-119: randomized SVD of an operator given by its
    (multi-column) products with M and M^T; the sketch width doubles until
    the smallest captured singular value is at or below the threshold.
    Orthonormalisation and the core SVD run on the device; the caller's
    ``apply`` / ``apply_t`` receive numpy blocks."""
    if oversample < 2:
        raise ValueError("oversample must be >= 2")
    if rng is None:
        rng = np.random.default_rng(0)
    full = min(m, n)
    if full == 0:
        return _empty(m, n)
    cap = full if max_rank is None else min(full, max_rank)
    k_try = min(start_rank, cap)
    while True:
        width = min(k_try + oversample, full)
        Y = np.asarray(apply(rng.standard_normal((n, width))), dtype=float)
        for _ in range(power_iters):
            Y = np.asarray(apply(np.asarray(apply_t(_orth(Y)), dtype=float)), dtype=float)
        Q = _orth(Y)
        B = np.asarray(apply_t(Q), dtype=float).T          # (width, n)
        Wb, s, V = _svd_all(B, -1.0)
        if width >= full or k_try >= cap or (len(s) > k_try and s[k_try] <= abs_threshold):
            break
        k_try = min(2 * k_try, cap)
    keep = min(int(np.count_nonzero(s > abs_threshold)), cap)
    if keep == 0:
        return _empty(m, n)
    return LowRankFactor(Q @ Wb[:, :keep], s[:keep].copy(), V[:, :keep].copy())


def randomized_svd_dense(M: np.ndarray, abs_threshold: float, **kw) -> LowRankFactor:
    """lowrank.py:122-125."""
    M = np.asarray(M, dtype=float)
    return randomized_svd(lambda X: M @ X, lambda X: M.T @ X, M.shape[0], M.shape[1],
                          abs_threshold, **kw)


def _union(B, w, F, wf, thr, min_rank):
    m, ko = B.shape
    kf = F.shape[1]
    cap = min(m, ko + kf)
    t = _torch()
    dB, dw, dF, dwf = _dev(B), _dev(w), _dev(F), _dev(wf)
    NB, NW, OM, FM = _zeros(m * cap), _zeros(cap), _zeros(cap * ko), _zeros(cap * kf)
    dr = _zeros(1, t.int32)
    t.cuda.synchronize()
    N.check(N.lib().ifmm_dev_union(N.ctx(), m, ko, kf, _p(dB), _p(dw), _p(dF), _p(dwf),
                                   float(thr), int(min_rank), _p(NB), _p(NW), _p(OM), _p(FM),
                                   _p(dr)))
    r = int(dr.item())
    return (NB.cpu().numpy()[:m * r].reshape(r, m).T.copy(), NW.cpu().numpy()[:r].copy(),
            OM.cpu().numpy()[:r * ko].reshape(r, ko).copy(),
            FM.cpu().numpy()[:r * kf].reshape(r, kf).copy())


def aca_svd(M: np.ndarray, abs_threshold: float, min_rank: int = 0,
            margin: float = ACA_MARGIN) -> LowRankFactor:
    """lowrank.py:128-163: full-pivot ACA down to threshold/margin, then
    QR-QR-SVD recompression truncated at the threshold (>= min_rank).  Runs
    the basis-union kernel on [M | 0] with unit weights (the zero column is
    never a pivot); the kernel's pivot margin is fixed at 8."""
    if margin != ACA_MARGIN:
        raise ValueError(f"the device ACA uses the reference's default margin {ACA_MARGIN}")
    M = np.asarray(M, dtype=float)
    m, n = M.shape
    if M.size == 0:
        return _empty(m, n)
    U, s, om, _ = _union(M, np.ones(n), np.zeros((m, 1)), np.ones(1), abs_threshold, min_rank)
    if len(s) == 0:
        return _empty(m, n)
    return LowRankFactor(U, s, (om / s[:, None]).T.copy())


def weighted_basis_union(old_basis: np.ndarray, old_weights: np.ndarray,
                         fill_basis: np.ndarray, fill_weights: np.ndarray,
                         abs_threshold: float, min_rank: int = 0) -> BasisUpdate:
    """lowrank.py:166-199: recompress [B diag(w) | F diag(wf)]; returns the
    new basis and weights and the maps r, r' with B ~= new r, F ~= new r'."""
    w = np.asarray(old_weights, dtype=float)
    wf = np.asarray(fill_weights, dtype=float)
    if old_basis.shape[1] != len(w):
        raise ValueError("old basis/weight size mismatch")
    if fill_basis.shape[1] != len(wf):
        raise ValueError("fill basis/weight size mismatch")
    if np.any(w <= 0.0) or np.any(wf <= 0.0):
        raise ValueError("weights must be positive")
    if fill_basis.shape[1] == 0:  # nothing to merge: aca of the weighted basis alone
        fac = aca_svd(np.asarray(old_basis, dtype=float) * w, abs_threshold, min_rank)
        scaled = fac.sigma[:, None] * fac.V.T
        return BasisUpdate(fac.U, fac.sigma.copy(), scaled / w[None, :],
                           np.zeros((fac.rank, 0)))
    U, s, om, fm = _union(np.asarray(old_basis, dtype=float), w,
                          np.asarray(fill_basis, dtype=float), wf, abs_threshold, min_rank)
    return BasisUpdate(U, s, om, fm)
