"""ctypes binding of the in-tree CUDA engine ``_ifmm_b200.so``.

There is deliberately no CPU fallback: if the library is missing, or no
CUDA device is visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ifmm_b200.so")

_lib = None
_lock = threading.RLock()
_ctx = None

E_VALUE, E_SINGULAR, E_CUDA, E_OOM, E_ASSERT = 1, 2, 3, 4, 5

vp, dp, ip, lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_longlong)

_SIGS = {
    "ifmm_abi_version": (C.c_int, []),
    "ifmm_last_error": (C.c_char_p, []),
    "ifmm_ctx_create": (vp, [C.c_int, C.c_ulonglong]),
    "ifmm_ctx_destroy": (None, [vp]),
    "ifmm_ctx_memory": (C.c_int, [vp, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]),
    "ifmm_tree_create": (vp, [vp, C.c_int, dp, ip, C.c_int, C.c_int, ip, ip, ip, ip, lp, dp,
                              dp, ip, ip]),
    "ifmm_tree_destroy": (None, [vp]),
    "ifmm_tree_topology_sizes": (C.c_int, [vp, lp, lp]),
    "ifmm_tree_topology": (C.c_int, [vp, lp, ip, lp, ip]),
    "ifmm_h2_build": (vp, [vp, C.c_int, C.c_double, C.c_int, C.c_double]),
    "ifmm_h2_weights_sampled": (C.c_int, [vp, vp, vp]),
    "ifmm_h2_build_k": (vp, [vp, C.c_int, C.c_double, C.c_double, C.c_int, C.c_double]),
    "ifmm_kernel_matrix_k": (C.c_int, [vp, C.c_int, C.c_double, C.c_double, C.c_int, vp, C.c_int, vp,
                                       vp, C.c_int]),
    "ifmm_exact_matvec_k": (C.c_int, [vp, C.c_int, C.c_double, C.c_double, C.c_int, vp, vp, vp,
                                      C.c_int]),
    "ifmm_h2_destroy": (None, [vp]),
    "ifmm_h2_ranks": (C.c_int, [vp, ip]),
    "ifmm_h2_weights": (C.c_int, [vp]),
    "ifmm_h2_block": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dp, ip, ip]),
    "ifmm_h2_matvec": (C.c_int, [vp, vp, vp, C.c_int]),
    "ifmm_h2_multipole_size": (C.c_int, [vp, C.POINTER(C.c_longlong)]),
    "ifmm_h2_matvec_part": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_longlong, C.c_longlong]),
    "ifmm_graph_build": (vp, [vp, C.c_int]),
    "ifmm_graph_destroy": (None, [vp]),
    "ifmm_graph_info": (C.c_int, [vp, lp, lp, lp]),
    "ifmm_graph_nodes": (C.c_int, [vp, ip, ip, ip]),
    "ifmm_graph_cluster_nodes": (C.c_int, [vp, ip, ip, ip]),
    "ifmm_graph_edges": (C.c_int, [vp, ip, ip, lp]),
    "ifmm_graph_block": (C.c_int, [vp, C.c_int, C.c_int, dp, ip, ip]),
    "ifmm_graph_copy": (vp, [vp]),
    "ifmm_graph_apply": (C.c_int, [vp, vp, vp, C.c_int, C.c_int]),
    "ifmm_graph_sigma0": (C.c_int, [vp, dp, C.c_int, C.c_int, dp]),
    "ifmm_factorize": (vp, [vp, C.c_double, C.c_double, C.c_int]),
    "ifmm_factorize_rng": (vp, [vp, C.c_double, C.c_double, C.c_int, vp, vp]),
    "ifmm_factorize_pcg64": (vp, [vp, C.c_double, C.c_double, C.c_int, C.POINTER(C.c_ulonglong)]),
    "ifmm_pcg64_normals": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_longlong, dp]),
    "ifmm_factor_level_times": (C.c_int, [vp, dp, C.c_int]),
    "ifmm_factor_events": (C.c_longlong, [vp, lp, C.c_longlong]),
    "ifmm_factor_layout": (C.c_int, [vp, ip, ip, ip, ip, ip, ip, ip]),
    "ifmm_kernel_matrix": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, vp, C.c_int, vp, vp,
                                     C.c_int]),
    "ifmm_blockdiag_create": (vp, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_int]),
    "ifmm_blockdiag_apply": (C.c_int, [vp, vp, vp, C.c_int]),
    "ifmm_blockdiag_destroy": (None, [vp]),
    "ifmm_factor_destroy": (None, [vp]),
    "ifmm_factor_stats": (C.c_int, [vp, lp, C.c_int]),
    "ifmm_factor_level_stats": (C.c_int, [vp, lp, C.c_int]),
    "ifmm_factor_level_ranks": (C.c_int, [vp, C.c_int, ip]),
    "ifmm_factor_timings": (C.c_int, [vp, dp, C.c_int]),
    "ifmm_solve": (C.c_int, [vp, vp, vp, C.c_int]),
    "ifmm_profile": (C.c_int, [dp, C.c_int]),
    "ifmm_ctx_event": (C.c_int, [vp, C.c_int]),
    "ifmm_ctx_elapsed": (C.c_int, [vp, C.c_int, C.c_int, dp]),
    "ifmm_ctx_launches": (C.c_longlong, [vp]),
    "ifmm_ktime": (C.c_int, [vp, C.c_int, dp, dp, lp, C.c_int]),
    "ifmm_union_profile": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    "ifmm_union_post_profile": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
    "ifmm_krylov_mgs": (C.c_int, [vp, vp, C.c_longlong, C.c_int, C.c_longlong, vp, vp]),
    "ifmm_krylov_div": (C.c_int, [vp, vp, C.c_longlong, C.c_double, vp]),
    "ifmm_krylov_combine": (C.c_int, [vp, vp, C.c_longlong, C.c_int, vp, C.c_longlong, vp]),
    "ifmm_dev_gemm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, vp, C.c_int,
                                C.c_int, vp, C.c_int, C.c_double, C.c_double]),
    "ifmm_dev_svd": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_double, vp, vp, vp, vp]),
    "ifmm_dev_lu_solve": (C.c_int, [vp, C.c_int, vp, vp, vp, C.c_int]),
    "ifmm_dev_union": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp, C.c_double,
                                 C.c_int, vp, vp, vp, vp, vp]),
    "ifmm_dev_orth": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
    "ifmm_dev_sync": (C.c_int, [vp]),
    "ifmm_dev_jacobi_bench": (C.c_int, [vp, C.c_int, vp, C.c_int, C.c_int, C.POINTER(C.c_ulonglong)]),
    "ifmm_exact_matvec": (C.c_int, [vp, C.c_int, C.c_double, C.c_int, vp, vp, vp, C.c_int]),
}


class NativeError(RuntimeError):
    pass


def lib():
    """Load the engine library (raises if it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"IFMM CUDA engine not built: {LIB_PATH} missing "
                        "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
                L = C.CDLL(LIB_PATH)
                for name, (res, args) in _SIGS.items():
                    f = getattr(L, name)
                    f.restype = res
                    f.argtypes = args
                _lib = L
    return _lib


def last_error() -> str:
    s = lib().ifmm_last_error()
    return s.decode() if s else ""


def check(status: int):
    """Map an ABI status to the reference's exception types."""
    if status == 0:
        return
    msg = last_error()
    if status == E_VALUE:
        raise ValueError(msg)
    if status == E_SINGULAR:
        from .factor import SingularPivotError
        raise SingularPivotError(msg)
    if status == E_OOM:
        raise MemoryError(msg)
    if status == E_ASSERT:
        raise AssertionError(msg)
    raise NativeError(msg)


def check_handle(h):
    if not h:
        msg = last_error()
        low = msg.lower()
        if "singular" in low or msg.startswith("cluster") or msg.startswith("top-level"):
            from .factor import SingularPivotError
            raise SingularPivotError(msg)
        if "epsilon" in low or "must be" in low or "unknown" in low or "basis weights" in low:
            raise ValueError(msg)
        if "arena exhausted" in low:
            raise MemoryError(msg)
        raise NativeError(msg or "native call failed")
    return h


def ctx():
    """Process-wide engine context (device arena + stream) on the current
    CUDA device.  IFMM_ARENA_GB sets the arena size (default: 60% of free)."""
    global _ctx
    if _ctx is None:
        with _lock:
            if _ctx is None:
                dev = 0
                try:
                    import torch
                    if torch.cuda.is_available():
                        dev = torch.cuda.current_device()
                except Exception:  # torch absent: device 0
                    pass
                gb = float(os.environ.get("IFMM_ARENA_GB", "0"))
                nbytes = int(gb * (1 << 30))
                if nbytes == 0:
                    nbytes = _default_arena(dev)
                h = lib().ifmm_ctx_create(dev, nbytes)
                _ctx = check_handle(h)
    return _ctx


def _default_arena(dev):
    try:
        import torch
        free, _ = torch.cuda.mem_get_info(dev)
        return int(free * 0.6)
    except Exception:
        return 0


def memory():
    a, b = C.c_ulonglong(), C.c_ulonglong()
    lib().ifmm_ctx_memory(ctx(), C.byref(a), C.byref(b))
    return a.value, b.value


def as_dp(a: np.ndarray):
    return a.ctypes.data_as(dp)


def as_ip(a: np.ndarray):
    return a.ctypes.data_as(ip)


def as_lp(a: np.ndarray):
    return a.ctypes.data_as(lp)


PROFILE_PHASES = ("lu", "xsolve", "schur", "add", "fillsvd", "union", "rebase", "newk", "merge",
                  "top", "host", "rsvd")


def profile():
    """Phase times of the last factorize (only populated with IFMM_PROFILE=1)."""
    out = np.zeros(len(PROFILE_PHASES))
    lib().ifmm_profile(as_dp(out), len(out))
    return dict(zip(PROFILE_PHASES, out.tolist()))


KCATS = ("gemm", "copy", "svd", "union", "lu", "lusolve", "spmv", "solve", "other")


def event(slot: int):
    check(lib().ifmm_ctx_event(ctx(), slot))


def elapsed_ms(a: int, b: int) -> float:
    out = C.c_double()
    check(lib().ifmm_ctx_elapsed(ctx(), a, b, C.byref(out)))
    return out.value


def launches() -> int:
    return int(lib().ifmm_ctx_launches(ctx()))


def ktime(enable: int = -1):
    """Per-category device kernel time / work / count; enable>=0 resets."""
    t, w = np.zeros(16), np.zeros(16)
    n = np.zeros(16, dtype=np.int64)
    lib().ifmm_ktime(ctx(), enable, as_dp(t), as_dp(w), as_lp(n), 16)
    return {k: (float(t[i]), float(w[i]), int(n[i])) for i, k in enumerate(KCATS)}
