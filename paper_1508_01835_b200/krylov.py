"""FMM matvec and GMRES (mirror of ``ifmm.krylov``).

``h2_matvec`` (krylov.py:119-159) runs on the device (deterministic
block-sparse products).  ``gmres`` (krylov.py:32-116) is the reference's
non-restarted MGS/Givens loop.  With a CUDA torch ``b`` the Krylov basis V is
resident in HBM and the Arnoldi step (MGS projections + norm), the basis
normalisation and the final combination run in the engine's kernels
(``csrc/krylov.cu``); the Givens rotations and the k x k triangular solve stay
on the host, as in SURVEY A18.  A numpy ``b`` runs the same loop on the host
(the reference's own array path, for callers whose apply_A is host-side).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .h2 import H2Operators


@dataclass
class IterationTrace:
    residual_history: list = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    side: str = "none"


def h2_matvec(ops: H2Operators, x):
    """krylov.py:119-159 on the device; numpy or CUDA torch in, same out."""
    try:
        import torch
        is_t = isinstance(x, torch.Tensor)
    except Exception:
        is_t = False
    if is_t:
        if x.shape != (ops.dim,):
            raise ValueError("vector length mismatch")
        x = x.contiguous()
        y = torch.empty_like(x)
        torch.cuda.current_stream().synchronize()
        N.check(N.lib().ifmm_h2_matvec(ops._h, C.c_void_p(x.data_ptr()),
                                       C.c_void_p(y.data_ptr()), 1))
        return y
    x = np.ascontiguousarray(np.asarray(x, dtype=float))
    if len(x) != ops.dim:
        raise ValueError("vector length mismatch")
    y = np.empty_like(x)
    N.check(N.lib().ifmm_h2_matvec(ops._h, x.ctypes.data_as(C.c_void_p),
                                   y.ctypes.data_as(C.c_void_p), 0))
    return y


def gmres(apply_A, b, tol: float = 1e-10, max_iters: int = 500, precond=None,
          side: str = "right"):
    """krylov.py:32-116 (MGS Arnoldi + Givens least squares)."""
    if tol <= 0 or max_iters < 1:
        raise ValueError("tol must be > 0 and max_iters >= 1")
    if precond is None:
        side = "none"
    if side not in ("left", "right", "none"):
        raise ValueError("side must be 'left', 'right', or 'none'")
    trace = IterationTrace(side=side)
    try:
        import torch
        is_t = isinstance(b, torch.Tensor)
    except Exception:
        is_t = False
    if is_t and b.is_cuda:
        return _gmres_device(apply_A, b, tol, max_iters, precond, side, trace)
    if is_t:
        def dot(u, v): return float(torch.dot(u, v))
        def norm(u): return float(torch.linalg.vector_norm(u))
        zeros = lambda n: torch.zeros(n, dtype=b.dtype, device=b.device)  # noqa: E731
    else:
        b = np.asarray(b, dtype=float)
        def dot(u, v): return float(u @ v)
        def norm(u): return float(np.linalg.norm(u))
        zeros = lambda n: np.zeros(n)  # noqa: E731
    n = len(b)
    r0 = precond(b) if side == "left" else b
    beta = norm(r0)
    if beta == 0.0:
        trace.converged = True
        return zeros(n), trace
    V = [r0 / beta]
    H = np.zeros((max_iters + 1, max_iters))
    cs, sn = np.zeros(max_iters), np.zeros(max_iters)
    g = np.zeros(max_iters + 1)
    g[0] = beta
    k_done, breakdown = 0, False
    for k in range(max_iters):
        if side == "right":
            w = apply_A(precond(V[k]))
        elif side == "left":
            w = precond(apply_A(V[k]))
        else:
            w = apply_A(V[k])
        for i in range(k + 1):
            H[i, k] = dot(V[i], w)
            w = w - H[i, k] * V[i]
        h_sub = norm(w)
        H[k + 1, k] = h_sub
        for i in range(k):
            h0 = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = h0
        nu = np.hypot(H[k, k], H[k + 1, k])
        if nu == 0.0:
            k_done, breakdown = k, True
            break
        cs[k], sn[k] = H[k, k] / nu, H[k + 1, k] / nu
        H[k, k], H[k + 1, k] = nu, 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        rel = abs(g[k + 1]) / beta
        trace.residual_history.append(float(rel))
        k_done = k + 1
        if rel <= tol:
            trace.converged = True
            break
        if h_sub == 0.0:
            breakdown = True
            break
        V.append(w / h_sub)
    if breakdown and trace.residual_history:
        trace.converged = trace.residual_history[-1] <= tol
    k = k_done
    x = zeros(n)
    if k > 0:
        import scipy.linalg as sla
        y = sla.solve_triangular(H[:k, :k], g[:k])
        u = zeros(n)
        for i in range(k):
            u = u + float(y[i]) * V[i]
        x = precond(u) if side == "right" else u
    trace.iterations = k
    return x, trace


def _gmres_device(apply_A, b, tol, max_iters, precond, side, trace):
    """krylov.py:32-116 with V resident on the device (rows = Krylov vectors,
    grown by doubling up to the reference's (max_iters+1) x n), MGS / norm /
    normalisation / combination in ``csrc/krylov.cu``."""
    import torch
    import scipy.linalg as sla
    lib, ctx = N.lib(), N.ctx()
    b = b.to(torch.float64).contiguous()
    n = b.numel()

    def cur_sync():
        torch.cuda.current_stream().synchronize()

    def ptr(t):
        return C.c_void_p(t.data_ptr())

    r0 = (precond(b) if side == "left" else b).contiguous()
    cur_sync()
    hb = np.zeros(1)
    N.check(lib.ifmm_krylov_mgs(ctx, ptr(r0), n, 0, n, ptr(r0.clone()),
                                hb.ctypes.data_as(C.c_void_p)))
    beta = float(hb[0])
    if beta == 0.0:
        trace.converged = True
        return torch.zeros(n, dtype=torch.float64, device=b.device), trace
    cap = min(max_iters + 1, 32)
    V = torch.empty((cap, n), dtype=torch.float64, device=b.device)
    N.check(lib.ifmm_krylov_div(ctx, ptr(r0), n, beta, ptr(V[0])))
    H = np.zeros((max_iters + 1, max_iters))
    cs, sn = np.zeros(max_iters), np.zeros(max_iters)
    g = np.zeros(max_iters + 1)
    g[0] = beta
    hcol = np.zeros(max_iters + 2)
    k_done, breakdown = 0, False
    for k in range(max_iters):
        vk = V[k]
        if side == "right":
            w = apply_A(precond(vk))
        elif side == "left":
            w = precond(apply_A(vk))
        else:
            w = apply_A(vk)
        w = w.to(torch.float64).contiguous()
        if w.data_ptr() == vk.data_ptr():
            w = w.clone()
        cur_sync()
        N.check(lib.ifmm_krylov_mgs(ctx, ptr(V), n, k + 1, n, ptr(w),
                                    hcol.ctypes.data_as(C.c_void_p)))
        H[:k + 2, k] = hcol[:k + 2]
        h_sub = H[k + 1, k]
        for i in range(k):
            h0 = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = h0
        nu = np.hypot(H[k, k], H[k + 1, k])
        if nu == 0.0:
            k_done, breakdown = k, True
            break
        cs[k], sn[k] = H[k, k] / nu, H[k + 1, k] / nu
        H[k, k], H[k + 1, k] = nu, 0.0
        g[k + 1] = -sn[k] * g[k]
        g[k] = cs[k] * g[k]
        rel = abs(g[k + 1]) / beta
        trace.residual_history.append(float(rel))
        k_done = k + 1
        if rel <= tol:
            trace.converged = True
            break
        if h_sub == 0.0:
            breakdown = True
            break
        if k + 1 >= V.shape[0]:
            grown = torch.empty((min(max_iters + 1, 2 * V.shape[0]), n), dtype=torch.float64,
                                device=b.device)
            grown[:V.shape[0]].copy_(V)
            torch.cuda.current_stream().synchronize()
            V = grown
        N.check(lib.ifmm_krylov_div(ctx, ptr(w), n, float(h_sub), ptr(V[k + 1])))
    if breakdown and trace.residual_history:
        trace.converged = trace.residual_history[-1] <= tol
    k = k_done
    x = torch.zeros(n, dtype=torch.float64, device=b.device)
    if k > 0:
        y = np.ascontiguousarray(sla.solve_triangular(H[:k, :k], g[:k]))
        u = torch.empty(n, dtype=torch.float64, device=b.device)
        N.check(lib.ifmm_krylov_combine(ctx, ptr(V), n, k, y.ctypes.data_as(C.c_void_p), n,
                                        ptr(u)))
        x = precond(u) if side == "right" else u
    trace.iterations = k
    return x, trace


def exact_matvec(points, kernel, x):
    """y = A x with A_ij = kernel(|p_i - p_j|) evaluated on the device without
    storing A (replaces dense.dense_matrix(...) @ x of the reference's
    experiments._matvec_oracle, experiments.py:157-162, at any N)."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=float))
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError("points must be an (N, 3) array")
    kind, p0 = kernel.device_spec()
    x = np.ascontiguousarray(np.asarray(x, dtype=float))
    if len(x) != len(pts):
        raise ValueError("vector length mismatch")
    y = np.empty_like(x)
    N.check(N.lib().ifmm_exact_matvec(N.ctx(), kind, p0, len(pts), pts.ctypes.data_as(C.c_void_p),
                                      x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), 0))
    return y
