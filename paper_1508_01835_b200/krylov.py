"""FMM matvec and GMRES (mirror of ``ifmm.krylov``).

``h2_matvec`` (krylov.py:119-159) runs on the device (deterministic
block-sparse products).  ``gmres`` (krylov.py:32-116) is the reference's
non-restarted MGS/Givens loop.  With a CUDA torch ``b`` the Krylov basis V is
resident in HBM and the Arnoldi step (MGS projections + norm), the basis
normalisation and the final combination run in the engine's kernels
(``csrc/krylov.cu``); the Givens rotations and the k x k triangular solve stay
on the host, as in SURVEY A18.  A numpy ``b`` (the reference harness's call,
experiments.py:190-233) runs the same device loop: b is copied up once and
host-only operators are adapted per call (``_DeviceOperator``).
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
    import torch
    if isinstance(b, torch.Tensor) and b.is_cuda:
        return _gmres_device(apply_A, b, tol, max_iters, precond, side, trace)
    # Host operands (numpy b, or a CPU tensor): the Arnoldi loop still runs on
    # the device -- b is copied up once, the Krylov basis lives in HBM, and
    # the caller's operators are adapted per call (a device-capable operator
    # such as h2_matvec or IFMMFactorization.solve receives the CUDA vector
    # directly; a host-only one, e.g. ``lambda v: A @ v`` on numpy arrays, is
    # called with a numpy copy).  The result comes back in the caller's kind.
    if not torch.cuda.is_available():
        raise RuntimeError("gmres: the Arnoldi loop runs on the CUDA device and none is "
                           "visible (there is no CPU path)")
    host_tensor = isinstance(b, torch.Tensor)
    bh = b.detach().to(torch.float64).numpy() if host_tensor else np.asarray(b, dtype=float)
    bd = torch.from_numpy(np.ascontiguousarray(bh)).cuda()
    A_dev = _DeviceOperator(apply_A)
    P_dev = _DeviceOperator(precond) if precond is not None else None
    x, trace = _gmres_device(A_dev, bd, tol, max_iters, P_dev, side, trace)
    x = x.cpu()
    return (x if host_tensor else x.numpy()), trace


class _DeviceOperator:
    """Adapts a caller's operator to CUDA float64 vectors.  The first call
    probes whether the operator accepts a CUDA tensor (the package's own
    operators do); if it does not, every call goes through a host copy."""

    def __init__(self, fn):
        self.fn, self.mode = fn, None

    def __call__(self, v):
        import torch
        if self.mode != "host":
            try:
                out = self.fn(v)
                if isinstance(out, torch.Tensor) and out.is_cuda:
                    self.mode = "device"
                    return out
                if self.mode == "device":
                    raise TypeError("operator stopped returning CUDA tensors")
            except (TypeError, RuntimeError, ValueError, AttributeError):
                if self.mode == "device":
                    raise
            self.mode = "host"
        out = np.asarray(self.fn(v.cpu().numpy()), dtype=float)
        return torch.from_numpy(np.ascontiguousarray(out)).to(v.device)


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
    # k1 = 0: the kernel only forms ||w|| and never writes w, so r0 itself is
    # passed (no temporary whose producer runs on another stream)
    N.check(lib.ifmm_krylov_mgs(ctx, ptr(r0), n, 0, n, ptr(r0),
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
    experiments._matvec_oracle, experiments.py:157-162, at any N).  numpy or
    CUDA torch ``x``; the result is of the same kind."""
    pts = np.ascontiguousarray(np.asarray(points, dtype=float))
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError("points must be an (N, 3) array")
    kind, p0, p1 = kernel.device_spec()
    dim = len(pts) * kernel.block_dim
    try:
        import torch
        is_t = isinstance(x, torch.Tensor) and x.is_cuda
    except Exception:
        is_t = False
    if is_t:
        if x.shape != (dim,):
            raise ValueError("vector length mismatch")
        xd = x.to(torch.float64).contiguous()
        dp_ = torch.from_numpy(pts).to(xd.device)
        y = torch.empty_like(xd)
        torch.cuda.current_stream().synchronize()
        N.check(N.lib().ifmm_exact_matvec_k(N.ctx(), kind, p0, p1, len(pts), C.c_void_p(dp_.data_ptr()),
                                            C.c_void_p(xd.data_ptr()), C.c_void_p(y.data_ptr()), 1))
        return y
    x = np.ascontiguousarray(np.asarray(x, dtype=float))
    if len(x) != dim:
        raise ValueError("vector length mismatch")
    y = np.empty_like(x)
    N.check(N.lib().ifmm_exact_matvec_k(N.ctx(), kind, p0, p1, len(pts), pts.ctypes.data_as(C.c_void_p),
                                        x.ctypes.data_as(C.c_void_p), y.ctypes.data_as(C.c_void_p), 0))
    return y


class H2Matvec:
    """krylov.py:162-169: callable wrapper around h2_matvec."""

    def __init__(self, ops: H2Operators):
        self.ops = ops

    def __call__(self, x):
        return h2_matvec(self.ops, x)


class _BlockDiag:
    def __init__(self, handle, n):
        self._h, self.n = handle, n

    def __del__(self):
        try:
            N.lib().ifmm_blockdiag_destroy(self._h)
        except Exception:
            pass

    def __call__(self, v):
        import torch
        if isinstance(v, torch.Tensor) and v.is_cuda:
            v = v.to(torch.float64).contiguous()
            out = torch.empty_like(v)
            torch.cuda.current_stream().synchronize()
            N.check(N.lib().ifmm_blockdiag_apply(self._h, C.c_void_p(v.data_ptr()),
                                                 C.c_void_p(out.data_ptr()), 1))
            return out
        v = np.ascontiguousarray(np.asarray(v, dtype=float))
        if v.shape != (self.n,):
            raise ValueError("vector length mismatch")
        out = np.empty_like(v)
        N.check(N.lib().ifmm_blockdiag_apply(self._h, v.ctypes.data_as(C.c_void_p),
                                             out.ctypes.data_as(C.c_void_p), 0))
        return out


def block_diag_preconditioner(A, block_size: int):
    """krylov.py:172-196: factor the diagonal blocks of A once (device LU,
    partial pivoting), apply the block solves (one batched launch).  The
    last block is shorter when block_size does not divide the dimension."""
    try:
        import torch
        on_dev = isinstance(A, torch.Tensor) and A.is_cuda
    except Exception:
        on_dev = False
    if on_dev:
        A = A.to(torch.float64).contiguous()
        n = A.shape[0]
        ptr = C.c_void_p(A.data_ptr())
    else:
        A = np.ascontiguousarray(np.asarray(A, dtype=float))
        n = A.shape[0]
        ptr = A.ctypes.data_as(C.c_void_p)
    if block_size < 1 or block_size > n:
        raise ValueError("block_size must be in [1, n]")
    if on_dev:
        torch.cuda.current_stream().synchronize()
    h = N.lib().ifmm_blockdiag_create(N.ctx(), ptr, n, n, int(block_size), 1 if on_dev else 0)
    if not h:
        msg = N.last_error()
        if "diagonal block" in msg:
            a = int(msg.rsplit(" ", 1)[-1]) if msg.rsplit(" ", 1)[-1].isdigit() else 0
            raise ValueError(f"singular diagonal block [{a}:{min(n, a + block_size)}]")
        N.check_handle(h)
    return _BlockDiag(h, n)
