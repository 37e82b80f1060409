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
        t = np.zeros(9)
        N.check(L.ifmm_factor_timings(handle, N.as_dp(t), 9))
        self.flops = {"gemm_lu_class": float(t[5]), "all": float(t[6])}
        self.rsvd = {"rounds": int(t[7]), "redraws": int(t[8])}
        # factor.py:71-72 buckets: device time attributed per bucket (events
        # on the engine stream at every bucket switch, csrc/runtime.h)
        self.timings = {k: float(v) for k, v in zip(_TIMING_KEYS, t[:4])}
        self.timings["sigma0_estimation"] = t_sigma0
        self.timings["elimination_total"] = float(t[4])
        ct = np.zeros(max(nlev, 1))
        N.check(L.ifmm_factor_level_times(handle, N.as_dp(ct), nlev))
        for lvl, c in zip(levels, ct):
            lvl.compress_time = float(c)

    def __del__(self):
        try:
            N.lib().ifmm_factor_destroy(self._h)
        except Exception:
            pass

    @property
    def dim(self):
        return self.n_points * self.block_dim

    def _layout(self):
        if getattr(self, "_lay", None) is None:
            L = N.lib()
            sz = np.zeros(3, dtype=np.int32)
            N.check(L.ifmm_factor_layout(self._h, N.as_ip(sz), None, None, None, None, None,
                                         None))
            nt, ni, nl = (int(v) for v in sz)
            tn, ts = np.zeros(max(nt, 1), np.int32), np.zeros(max(nt, 1), np.int32)
            isz = np.zeros(max(ni, 1), np.int32)
            ln, l0, l1 = (np.zeros(max(nl, 1), np.int32) for _ in range(3))
            N.check(L.ifmm_factor_layout(self._h, None, N.as_ip(tn), N.as_ip(ts), N.as_ip(isz),
                                         N.as_ip(ln), N.as_ip(l0), N.as_ip(l1)))
            self._lay = (tn[:nt].tolist(), ts[:nt].tolist(), isz[:ni].tolist(),
                         list(zip(ln[:nl].tolist(), l0[:nl].tolist(), l1[:nl].tolist())))
        return self._lay

    top_nodes = property(lambda self: list(self._layout()[0]))
    top_sizes = property(lambda self: list(self._layout()[1]))
    init_sizes = property(lambda self: list(self._layout()[2]))
    leaf_slices = property(lambda self: list(self._layout()[3]))

    @property
    def events(self):
        """The event log (factor.py:80) with the reference's tuple shapes and
        node ids; the numerical payload (LU factors, edge blocks, rebase maps)
        stays on the device and reads as None:
        ("elim", nx, nz, ny, size_x, size_z, None, [(b, None)..], [(a, None)..]),
        ("rebase", ny, None), ("merge", px, [(child_y, size)..])."""
        L = N.lib()
        n = int(L.ifmm_factor_events(self._h, None, 0))
        buf = np.zeros(max(n, 1), dtype=np.int64)
        L.ifmm_factor_events(self._h, N.as_lp(buf), n)
        v, out, i = buf[:n].tolist(), [], 0
        while i < n:
            t = v[i]
            if t == 0:
                nx, nz, ny, m, k, ns, nt = v[i + 1:i + 8]
                src = v[i + 8:i + 8 + ns]
                tgt = v[i + 8 + ns:i + 8 + ns + nt]
                out.append(("elim", nx, nz, ny, m, k, None, [(b, None) for b in src],
                            [(a, None) for a in tgt]))
                i += 8 + ns + nt
            elif t == 1:
                out.append(("rebase", v[i + 1], None))
                i += 2
            else:
                px, npart = v[i + 1], v[i + 2]
                pr = v[i + 3:i + 3 + 2 * npart]
                out.append(("merge", px, list(zip(pr[0::2], pr[1::2]))))
                i += 3 + 2 * npart
        return out

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


_NORMAL_SOURCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_longlong,
                             C.POINTER(C.c_double))


class _ReferenceStream:
    """The reference factorize rng -- ``np.random.Generator(PCG64(seed))``
    (factor.py:188) -- served to the engine as a stream of standard normals
    (ifmm_normal_source, include/ifmm_b200.h).  ``standard_normal((n, w))``
    is the next n*w deviates of one sequence, so the engine asks for flat
    runs of the sizes the reference draws, in the reference's order."""

    def __init__(self, seed):
        self.g = np.random.Generator(np.random.PCG64(seed))
        self.slots = {}
        self.drawn = 0
        self.error = None
        self.cb = _NORMAL_SOURCE(self._call)

    def _call(self, user, op, n, out):
        try:
            if op == 0:
                np.ctypeslib.as_array(out, shape=(n,))[:] = self.g.standard_normal(n)
                self.drawn += n
            elif op == 1:
                self.slots[n] = (self.g.bit_generator.state, self.drawn)
            elif op == 2:
                st, self.drawn = self.slots[n]
                self.g.bit_generator.state = st
            else:
                return 1
            return 0
        except Exception as e:  # surfaces as a ValueError from the engine
            self.error = e
            return 1


SCHEDULES = ("reference", "wavefront", "colored")


def pcg64_state(seed):
    """np.random.PCG64(seed)'s state as {state_hi, state_lo, inc_hi, inc_lo}."""
    st = np.random.PCG64(seed).state["state"]
    m = (1 << 64) - 1
    return (C.c_ulonglong * 4)(st["state"] >> 64, st["state"] & m, st["inc"] >> 64, st["inc"] & m)


def factorize(graph: ExtendedGraph, epsilon: float, seed: int = 0,
              sigma0: float | None = None, exact_order: bool | None = None,
              schedule: str | None = None) -> IFMMFactorization:
    """factor.py:176-230.  Consumes the graph (like the reference's pops).

    ``schedule``:
      * ``"reference"`` -- clusters are eliminated one at a time in the
        reference's Morton order, and every Gaussian the reference draws
        (rSVD sketches of fills with min(shape) > 64, lowrank.py:108) comes
        from the reference's own rng, ``Generator(PCG64(seed))``, in the
        reference's order.  Rank decisions and x then match the reference up
        to floating-point rounding.
      * ``"wavefront"`` -- clusters at Chebyshev distance >= 3 (no shared
        neighbour) are eliminated together in one batched stage, and the rSVD
        sketches come from a counter-based device generator.  Same
        algorithm; results differ from the reference the way the reference's
        own results differ between rng seeds.
      * ``"colored"`` -- the relaxed order of SURVEY.md 8e: 27 waves per
        level (9 in 2D), one per colour (x mod 3, y mod 3, z mod 3) of the
        cluster grid, every cluster of a colour eliminated in one batched
        stage.  The elimination ORDER differs from the reference's Morton
        order, so per-level fill statistics and x are not comparable with the
        reference's; this mode is validated by the residual criterion only
        (exact-matvec residual <= 2x the reference's, tests/test_gpu_large.py).
        Experimental: it is NOT robust on the hardest recipes -- at depth-5
        trees with a large absolute threshold (c4; the c5 recipe at
        N = 262,144) the relaxed order meets near-singular pivot blocks
        (SingularPivotError, or a preconditioner GMRES cannot use), where
        the reference order does not.
    The fill pairs of one elimination always run as waves of cluster-disjoint
    pairs (they commute); ``exact_order=True`` runs them one at a time
    (diagnostics).  Environment defaults: IFMM_SCHEDULE, IFMM_EXACT_ORDER."""
    import os
    if exact_order is None:
        exact_order = os.environ.get("IFMM_EXACT_ORDER", "0") == "1"
    if schedule is None:
        schedule = os.environ.get("IFMM_SCHEDULE", "reference")
    if schedule not in SCHEDULES:
        raise ValueError(f"schedule must be one of {SCHEDULES}")
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
    flags = (1 if exact_order else 0) | (8 if schedule == "colored" else 0)
    lib = N.lib()
    if schedule == "reference":
        # the reference's Generator(PCG64(seed)) (factor.py:188), run natively
        # in the engine (PCG64 + numpy's own ziggurat): bitwise the same draws
        h = lib.ifmm_factorize_pcg64(graph._h, float(epsilon), float(sigma0), flags | 4,
                                     pcg64_state(seed))
    else:
        h = lib.ifmm_factorize(graph._h, float(epsilon), float(sigma0), flags)
    graph.consumed = True
    h = N.check_handle(h)
    f = IFMMFactorization(graph, h, epsilon, sigma0, t_s, time.perf_counter() - t0)
    f.schedule = schedule
    return f
