"""Factorization and solve (mirror of ``ifmm.factor``).

``factorize`` (factor.py:176-230) runs the whole level-by-level
elimination in the CUDA engine and returns an ``IFMMFactorization`` whose
``solve`` (factor.py:99-157) replays the device event program.  ``solve``
accepts a numpy array (host in, host out -- copies are part of the call) or
a CUDA torch tensor (device in, device out).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .graph import ExtendedGraph, estimate_sigma0


class SingularPivotError(RuntimeError):
    """factor.py:32-35."""

    def __init__(self, what):
        super().__init__(f"singular pivot block during elimination: {what}")
        self.what = what


@dataclass
class FillinStats:
    level: int
    compressed_pairs: int = 0
    added: int = 0
    dropped_pairs: int = 0
    ranks: list = field(default_factory=list)
    compress_time: float = 0.0
    forced_rank_truncations: int = 0

    @property
    def max_rank(self):
        return max(self.ranks) if self.ranks else 0

    @property
    def mean_rank(self):
        return float(np.mean(self.ranks)) if self.ranks else 0.0


@dataclass
class FactorStats:
    levels: list = field(default_factory=list)
    peak_edges: int = 0
    n_clusters: int = 0
    max_basis_rank: int = 0
    max_fill_rank: int = 0
    forced_rank_truncations: int = 0

    @property
    def edge_bound_constant(self):
        return self.peak_edges / max(self.n_clusters, 1)


_TIMING_KEYS = ("lu_and_triangular_solves", "matmul_updates", "lowrank_approximations",
                "operator_transfer")


class IFMMFactorization:
    def __init__(self, graph: ExtendedGraph, handle, epsilon, sigma0, t_sigma0, t_total):
        self._h = handle
        self._graph = graph  # keeps tree / ops device data alive
        self.tree = graph.tree
        self.n_points = graph.tree.n_points
        self.block_dim = graph.block_dim
        self.perm = graph.tree.perm
        self.epsilon = epsilon
        self.sigma0 = sigma0
        L = N.lib()
        s = np.zeros(11, dtype=np.int64)
        N.check(L.ifmm_factor_stats(handle, N.as_lp(s), 11))
        nlev = int(s[5])
        lv = np.zeros(8 * max(nlev, 1), dtype=np.int64)
        N.check(L.ifmm_factor_level_stats(handle, N.as_lp(lv), nlev))
        levels = []
        for i in range(nlev):
            row = lv[8 * i:8 * i + 8]
            ranks = np.zeros(max(int(row[6]), 1), dtype=np.int32)
            N.check(L.ifmm_factor_level_ranks(handle, i, N.as_ip(ranks)))
            levels.append(FillinStats(int(row[0]), int(row[1]), int(row[2]), int(row[3]),
                                      ranks[:int(row[6])].tolist(), 0.0, int(row[7])))
        self.stats = FactorStats(levels, int(s[0]), int(s[1]), int(s[2]), int(s[3]), int(s[4]))
        self.event_counts = {"elim": int(s[6]), "rebase": int(s[7]), "merge": int(s[8])}
        self.top_nodes_count = int(s[9])
        self.top_dim = int(s[10])
        t = np.zeros(7)
        N.check(L.ifmm_factor_timings(handle, N.as_dp(t), 7))
        self.flops = {"gemm_lu_class": float(t[5]), "all": float(t[6])}
        self.timings = {k: 0.0 for k in _TIMING_KEYS}
        self.timings["sigma0_estimation"] = t_sigma0
        self.timings["elimination_total"] = float(t[4])

    def __del__(self):
        try:
            N.lib().ifmm_factor_destroy(self._h)
        except Exception:
            pass

    @property
    def dim(self):
        return self.n_points * self.block_dim

    @property
    def events(self):
        """Event tags (counts only; the log itself lives on the device)."""
        c = self.event_counts
        return [("elim",)] * c["elim"] + [("rebase",)] * c["rebase"] + [("merge",)] * c["merge"]

    def solve(self, b):
        """A x = b in the original point order (factor.py:99-157)."""
        try:
            import torch
            is_t = isinstance(b, torch.Tensor)
        except Exception:  # torch absent
            is_t = False
        if is_t:
            if not b.is_cuda or b.dtype != torch.float64 or b.shape != (self.dim,):
                raise ValueError(f"rhs must be a float64 CUDA tensor of shape ({self.dim},)")
            b = b.contiguous()
            x = torch.empty_like(b)
            torch.cuda.current_stream().synchronize()
            N.check(N.lib().ifmm_solve(self._h, C.c_void_p(b.data_ptr()),
                                       C.c_void_p(x.data_ptr()), 1))
            return x
        b = np.asarray(b, dtype=float)
        if b.shape != (self.dim,):
            raise ValueError(f"rhs must have shape ({self.dim},)")
        b = np.ascontiguousarray(b)
        x = np.empty_like(b)
        N.check(N.lib().ifmm_solve(self._h, b.ctypes.data_as(C.c_void_p),
                                   x.ctypes.data_as(C.c_void_p), 0))
        return x


def factorize(graph: ExtendedGraph, epsilon: float, seed: int = 0,
              sigma0: float | None = None, exact_order: bool | None = None
              ) -> IFMMFactorization:
    """factor.py:176-230.  Consumes the graph (like the reference's pops).

    ``exact_order`` processes the fill pairs of each elimination strictly in
    the reference's sorted order (one pair at a time).  The default groups
    cluster-disjoint pairs into concurrent waves, which commute up to
    rounding.  IFMM_EXACT_ORDER=1 sets the default."""
    import os
    if exact_order is None:
        exact_order = os.environ.get("IFMM_EXACT_ORDER", "0") == "1"
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must be in (0, 1)")
    if graph.consumed:
        raise ValueError("graph already factorized")
    t_s = 0.0
    if sigma0 is None:
        t0 = time.perf_counter()
        sigma0 = estimate_sigma0(graph, seed=seed)
        t_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    h = N.lib().ifmm_factorize(graph._h, float(epsilon), float(sigma0), 1 if exact_order else 0)
    graph.consumed = True
    h = N.check_handle(h)
    return IFMMFactorization(graph, h, epsilon, sigma0, t_s, time.perf_counter() - t0)
