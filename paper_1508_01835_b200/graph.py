"""Extended sparse graph on the device (mirror of ``ifmm.graph``).

``assemble_extended_graph`` (graph.py:219-229) builds the node/edge
store inside the engine (device blocks, host adjacency);
``estimate_sigma0`` (graph.py:232-241) draws the reference's Gaussian
sketch on the host -- exactly ``Generator(PCG64(seed)).standard_normal
((dim, 11))`` -- and runs the power iterations, QRs and the final SVD on the
device.
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Mapping

import numpy as np

from . import _native as N
from .h2 import H2Operators


X, Z, Y = "x", "z", "y"
_KIND = (X, Z, Y)


class _EdgeView(Mapping):
    """graph.edges: (target, source) -> block, fetched from the device on
    access (inspection and tests only)."""

    def __init__(self, g, keys):
        self._g, self._keys = g, keys

    def __getitem__(self, key):
        if key not in self._keys:
            raise KeyError(key)
        t, s = key
        r, c = C.c_int(), C.c_int()
        L = N.lib()
        N.check(L.ifmm_graph_block(self._g._h, int(t), int(s), None, C.byref(r), C.byref(c)))
        out = np.empty((r.value, c.value))
        N.check(L.ifmm_graph_block(self._g._h, int(t), int(s), N.as_dp(out), C.byref(r),
                                   C.byref(c)))
        return out

    def __iter__(self):
        return iter(sorted(self._keys))

    def __len__(self):
        return len(self._keys)

    def __contains__(self, key):
        return key in self._keys


class ExtendedGraph:
    """Device-resident extended sparse graph (graph.py:30-216).  The
    reference's inspection attributes (sizes, kinds, cluster_of, node_x/z/y,
    edges, row_sources, col_targets, peak_edges) are read-only host views of
    the device graph; ``apply`` / ``apply_transpose`` / ``copy`` run on the
    device.  ``rhs`` is host bookkeeping only: the factorization replays the
    event log from b in ``solve`` (factor.py:99-157), so the device graph
    carries no right-hand side."""

    def __init__(self, ops: H2Operators, handle, b=None):
        self.ops = ops
        self.tree = ops.tree
        self.topology = ops.topology
        self.block_dim = ops.block_dim
        self._h = handle
        self.consumed = False
        self._view = None
        self.rhs = {}
        self.set_rhs(b)

    def __del__(self):
        try:
            N.lib().ifmm_graph_destroy(self._h)
        except Exception:
            pass

    def _info(self):
        d, n, e = C.c_longlong(), C.c_longlong(), C.c_longlong()
        N.check(N.lib().ifmm_graph_info(self._h, C.byref(d), C.byref(n), C.byref(e)))
        return d.value, n.value, e.value

    def _live(self):
        if self.consumed:
            raise ValueError("graph already factorized (the factorization consumed it)")

    def _structure(self):
        self._live()
        if self._view is None:
            L = N.lib()
            _, nn, ne = self._info()
            size = np.zeros(nn, dtype=np.int32)
            kind = np.zeros(nn, dtype=np.int32)
            own = np.zeros(nn, dtype=np.int32)
            N.check(L.ifmm_graph_nodes(self._h, N.as_ip(size), N.as_ip(kind), N.as_ip(own)))
            nc = self.tree.n_clusters
            nx, nz, ny = (np.zeros(nc, dtype=np.int32) for _ in range(3))
            N.check(L.ifmm_graph_cluster_nodes(self._h, N.as_ip(nx), N.as_ip(nz), N.as_ip(ny)))
            t = np.zeros(max(ne, 1), dtype=np.int32)
            sv = np.zeros(max(ne, 1), dtype=np.int32)
            peak = C.c_longlong()
            N.check(L.ifmm_graph_edges(self._h, N.as_ip(t), N.as_ip(sv), C.byref(peak)))
            keys = list(zip(t[:ne].tolist(), sv[:ne].tolist()))
            rows = {i: set() for i in range(nn)}
            cols = {i: set() for i in range(nn)}
            for a, b in keys:
                rows[a].add(b)
                cols[b].add(a)
            self._view = dict(
                sizes=size.tolist(), kinds=[_KIND[k] for k in kind], cluster_of=own.tolist(),
                node_x={c: int(v) for c, v in enumerate(nx) if v >= 0},
                node_z={c: int(v) for c, v in enumerate(nz) if v >= 0},
                node_y={c: int(v) for c, v in enumerate(ny) if v >= 0},
                keys=set(keys), rows=rows, cols=cols, peak=int(peak.value))
        return self._view

    # ---- reference attributes (graph.py:30-60) ----
    sizes = property(lambda self: list(self._structure()["sizes"]))
    kinds = property(lambda self: list(self._structure()["kinds"]))
    cluster_of = property(lambda self: list(self._structure()["cluster_of"]))
    node_x = property(lambda self: dict(self._structure()["node_x"]))
    node_z = property(lambda self: dict(self._structure()["node_z"]))
    node_y = property(lambda self: dict(self._structure()["node_y"]))
    row_sources = property(lambda self: self._structure()["rows"])
    col_targets = property(lambda self: self._structure()["cols"])
    peak_edges = property(lambda self: self._structure()["peak"])
    eliminated = property(lambda self: set())

    @property
    def edges(self):
        return _EdgeView(self, self._structure()["keys"])

    def get_edge(self, t, s):
        return self.edges[(t, s)] if (t, s) in self._structure()["keys"] else None

    @property
    def dim(self) -> int:
        return self._info()[0]

    @property
    def num_edges(self) -> int:
        return self._info()[2]

    @property
    def sigma_u(self):
        return self.ops.sigma_u

    @property
    def sigma_v(self):
        return self.ops.sigma_v

    # ---- right-hand side bookkeeping (graph.py:123-140, 183-188) ----
    def set_rhs(self, b) -> None:
        self.rhs = {}
        if b is None:
            return
        bd = self.block_dim
        if len(b) != self.tree.n_points * bd:
            raise ValueError("rhs length mismatch")
        bt = np.asarray(b, dtype=float).reshape(self.tree.n_points, bd)[self.tree.perm].ravel()
        nx = self.node_x
        for cid in self.tree.leaves():
            c = self.tree.clusters[cid]
            self.rhs[nx[cid]] = bt[c.start * bd:c.stop * bd].copy()

    def _offsets(self):
        sz = self.sizes
        off = np.concatenate([[0], np.cumsum(sz)]).astype(np.int64)
        return off, int(off[-1])

    def full_rhs(self) -> np.ndarray:
        off, total = self._offsets()
        f = np.zeros(total)
        for nid, r in self.rhs.items():
            f[off[nid]:off[nid] + len(r)] = r
        return f

    # ---- whole-graph operator on the device (graph.py:157-181) ----
    def _apply(self, w, transpose):
        self._live()
        try:
            import torch
            is_t = isinstance(w, torch.Tensor) and w.is_cuda
        except Exception:
            is_t = False
        if is_t:
            w = w.to(torch.float64).contiguous()
            out = torch.empty_like(w)
            torch.cuda.current_stream().synchronize()
            N.check(N.lib().ifmm_graph_apply(self._h, C.c_void_p(w.data_ptr()),
                                             C.c_void_p(out.data_ptr()), int(transpose), 1))
            return out
        w = np.ascontiguousarray(np.asarray(w, dtype=float))
        if w.ndim == 2:  # multi-vector: one product per column
            return np.column_stack([self._apply(w[:, j], transpose) for j in range(w.shape[1])])
        if len(w) != self.dim:
            raise ValueError("vector length mismatch")
        out = np.empty_like(w)
        N.check(N.lib().ifmm_graph_apply(self._h, w.ctypes.data_as(C.c_void_p),
                                         out.ctypes.data_as(C.c_void_p), int(transpose), 0))
        return out

    def apply(self, w):
        return self._apply(w, False)

    def apply_transpose(self, w):
        return self._apply(w, True)

    def dense_matrix(self) -> np.ndarray:
        """graph.py:172-178 (small problems): blocks gathered from the device."""
        off, total = self._offsets()
        E = np.zeros((total, total))
        for (t, s), blk in self.edges.items():
            E[off[t]:off[t] + blk.shape[0], off[s]:off[s] + blk.shape[1]] = blk
        return E

    def sparsity_pattern(self) -> dict:
        """graph.py:183-188: JSON-able node list and sorted edge keys."""
        v = self._structure()
        nodes = [{"id": i, "kind": v["kinds"][i], "cluster": v["cluster_of"][i],
                  "size": v["sizes"][i]} for i in range(len(v["sizes"]))]
        return {"nodes": nodes, "edges": [list(k) for k in sorted(v["keys"])]}

    def copy(self) -> "ExtendedGraph":
        """graph.py:190-216: deep copy on the device (new blocks)."""
        self._live()
        h = N.check_handle(N.lib().ifmm_graph_copy(self._h))
        g = ExtendedGraph.__new__(ExtendedGraph)
        g.ops, g.tree, g.topology, g.block_dim = self.ops, self.tree, self.topology, self.block_dim
        g._h, g.consumed, g._view = h, False, None
        g.rhs = {k: v.copy() for k, v in self.rhs.items()}
        return g


def assemble_extended_graph(ops: H2Operators, topology=None, b=None,
                            consume: bool = False) -> ExtendedGraph:
    """graph.py:219-229.  ``b`` (original point order) is kept as host
    bookkeeping (``graph.rhs``); the device graph carries no right-hand side
    because the solve replays the event log from b (factor.py:99-157).
    ``consume=True`` moves the operator blocks into the graph (no copy; the
    operators cannot be used afterwards) -- for problems near device memory."""
    if ops.tree.depth >= 2 and not ops._weighted:
        raise ValueError("operators have no basis weights; run initialize_weights first")
    if b is not None and len(b) != ops.tree.n_points * ops.block_dim:
        raise ValueError("rhs length mismatch")
    h = N.lib().ifmm_graph_build(ops._h, 1 if consume else 0)
    return ExtendedGraph(ops, N.check_handle(h), b)


def estimate_sigma0(graph: ExtendedGraph, seed: int = 0, oversample: int = 10,
                    power_iters: int = 2) -> float:
    """graph.py:232-241 -> lowrank.randomized_svd(start_rank=1, max_rank=1)."""
    if oversample < 2:
        raise ValueError("oversample must be >= 2")
    if graph.consumed:
        raise ValueError("graph already factorized")
    rng = np.random.Generator(np.random.PCG64(seed))
    dim = graph.dim
    width = min(1 + oversample, dim)
    omega = np.ascontiguousarray(rng.standard_normal((dim, width)))
    out = C.c_double()
    N.check(N.lib().ifmm_graph_sigma0(graph._h, N.as_dp(omega), width, int(power_iters),
                                      C.byref(out)))
    return float(out.value)


def h2_dense(ops: H2Operators) -> np.ndarray:
    """graph.py:244-292 (test support, small N): the dense matrix the
    operators represent, in tree point order.  Far field composed level by
    level, F_l = K_l + T_u F_{l-1} T_v, then A = near + U F_L V^T; the blocks
    are read from the device through the operator views."""
    tree, bd = ops.tree, ops.block_dim
    F, prev = None, []
    coupling = ops.coupling
    for level in range(2, tree.depth + 1):
        ids = tree.levels[level]
        offs = np.cumsum([0] + [ops.rank[c] for c in ids])
        pos = {c: i for i, c in enumerate(ids)}
        Fl = np.zeros((offs[-1], offs[-1]))
        for (i, j) in coupling:
            if i in pos and j in pos:
                Fl[offs[pos[i]]:offs[pos[i] + 1], offs[pos[j]]:offs[pos[j] + 1]] = coupling[(i, j)]
        if F is not None:
            poffs = np.cumsum([0] + [ops.rank[c] for c in prev])
            ppos = {c: i for i, c in enumerate(prev)}
            Tu = np.zeros((offs[-1], poffs[-1]))
            Tv = np.zeros((poffs[-1], offs[-1]))
            tu, tv = ops.transfer_u, ops.transfer_vt
            for c in ids:
                r, q = pos[c], ppos[tree.clusters[c].parent]
                Tu[offs[r]:offs[r + 1], poffs[q]:poffs[q + 1]] = tu[c]
                Tv[poffs[q]:poffs[q + 1], offs[r]:offs[r + 1]] = tv[c]
            Fl = Fl + Tu @ F @ Tv
        F, prev = Fl, ids
    dim = tree.n_points * bd
    A = np.zeros((dim, dim))
    cl = tree.clusters
    near = ops.near
    for (i, j) in near:
        A[cl[i].start * bd:cl[i].stop * bd, cl[j].start * bd:cl[j].stop * bd] = near[(i, j)]
    if F is not None:
        offs = np.cumsum([0] + [ops.rank[c] for c in prev])
        pos = {c: i for i, c in enumerate(prev)}
        U = np.zeros((dim, offs[-1]))
        Vt = np.zeros((offs[-1], dim))
        lu, lv = ops.leaf_u, ops.leaf_v
        for c in tree.leaves():
            a, b, r = cl[c].start * bd, cl[c].stop * bd, pos[c]
            U[a:b, offs[r]:offs[r + 1]] = lu[c]
            Vt[offs[r]:offs[r + 1], a:b] = lv[c].T
        A = A + U @ F @ Vt
    return A
