"""TEST INFRASTRUCTURE ONLY: numpy restatement of the reference IFMM path.

Checker for the CUDA product (``paper_1508_01835_b200``); imported only by
tests, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs.  All
citations are ``/root/reference/pkg/src/ifmm/<file>:<line>``.

Data model (deliberately not the reference's classes):

* ``Tree``      flat per-cluster arrays + python lists for children / levels.
* ``Topo``      sorted neighbour / interaction id lists per cluster.
* ``Ops``       dict-of-blocks H2 operators (same keys as the reference).
* ``Graph``     extended sparse graph: node tables + ``{(t, s): block}``.
* ``Factor``    replay log + top LU, with ``solve``.

The numerics follow the reference operation by operation (same operand
order, same LAPACK drivers via numpy/scipy) so that results agree to
rounding.  The one deliberate addition is the gesdd->gesvd retry in
``_svd`` (numpy's bundled OpenBLAS gesdd sometimes fails to converge on
benign input).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla


# --------------------------------------------------------------------------
# small LAPACK wrappers
# --------------------------------------------------------------------------

def _svd(M, full_matrices=False):
    """np.linalg.svd with a gesvd retry (numpy gesdd defect)."""
    try:
        return np.linalg.svd(M, full_matrices=full_matrices)
    except np.linalg.LinAlgError:
        return sla.svd(M, full_matrices=full_matrices, lapack_driver="gesvd")


class SingularPivotError(RuntimeError):
    """factor.py:32-35."""

    def __init__(self, what):
        super().__init__(f"singular pivot block during elimination: {what}")
        self.what = what


class DegenerateGeometryError(ValueError):
    """tree.py:22-23."""


# --------------------------------------------------------------------------
# kernels (kernels.py:22-56 plugin contract: block(P, Q) -> (m, n) fp64)
# --------------------------------------------------------------------------

def _pair_dist(P, Q):
    # scipy cdist 'euclidean' (kernels.py:19,48) -- same routine for parity
    from scipy.spatial.distance import cdist
    return cdist(P, Q)


def exp_block(P, Q):
    """A_ij = exp(-|x_i - x_j|)  (BASELINE configs 1-2)."""
    return np.exp(-_pair_dist(P, Q))


def imq_block(h):
    """A_ij = 1/sqrt(|x_i - x_j|^2 + h^2)  (BASELINE configs 3-5)."""
    h2 = float(h) * float(h)

    def block(P, Q):
        r = _pair_dist(P, Q)
        return 1.0 / np.sqrt(r ** 2 + h2)
    return block


def benchmark_block(d):
    """kernels.py:42-56: 1 at r=0, r/d below d, d/r beyond."""
    def block(P, Q):
        r = _pair_dist(P, Q)
        out = np.empty_like(r)
        lt = r < d
        out[lt] = r[lt] / d
        out[~lt] = d / r[~lt]
        out[r == 0.0] = 1.0
        return out
    return block


# --------------------------------------------------------------------------
# tree + topology (tree.py:83-239)
# --------------------------------------------------------------------------

@dataclass
class Tree:
    points: np.ndarray          # Morton-sorted points
    perm: np.ndarray            # points[i] = original[perm[i]]
    depth: int
    center: np.ndarray
    half_width: float
    level: np.ndarray           # (nc,) int
    cell: np.ndarray            # (nc, 3) int64
    ccenter: np.ndarray         # (nc, 3)
    chw: np.ndarray             # (nc,)
    start: np.ndarray
    stop: np.ndarray
    parent: np.ndarray          # -1 for root
    children: list
    levels: list                # ids per level, Morton order

    @property
    def n_clusters(self):
        return len(self.level)

    def leaves(self):
        return self.levels[self.depth]


def cell_coords(points, center, hw, level):
    """tree.py:92-99: ceil((p - lo)/h) - 1, clipped; boundary -> lower cell."""
    ncell = 1 << level
    h = 2.0 * hw / ncell
    idx = np.ceil((points - (center - hw)) / h).astype(np.int64) - 1
    return np.clip(idx, 0, ncell - 1)


def morton(cells, nbits):
    """tree.py:83-89: bit b of axis a lands at bit 3b+a."""
    c = cells.astype(np.int64)
    key = np.zeros(len(c), dtype=np.int64)
    for b in range(nbits):
        for a in range(3):
            key |= ((c[:, a] >> b) & 1) << (3 * b + a)
    return key


def build_tree(points, leaf_target, depth=None, root_box=None, max_depth=12):
    """tree.py:107-196."""
    pts = np.asarray(points, dtype=float)
    if pts.ndim != 2 or pts.shape[1] != 3:
        raise ValueError("points must be an (N, 3) array")
    if len(pts) == 0:
        raise ValueError("points must be non-empty")
    if leaf_target < 1:
        raise ValueError("leaf_target must be >= 1")
    if root_box is not None:
        center = np.asarray(root_box[0], dtype=float)
        hw = float(root_box[1])
    else:
        lo, hi = pts.min(axis=0), pts.max(axis=0)
        center = 0.5 * (lo + hi)
        hw = 0.5 * float((hi - lo).max())
    if hw <= 0.0:
        raise DegenerateGeometryError("all points coincide; zero bounding box")
    if depth is None:                                   # tree.py:140-145
        depth = 2
        while depth < max_depth:
            occ = len(np.unique(morton(cell_coords(pts, center, hw, depth), depth)))
            if len(pts) / occ <= leaf_target:
                break
            depth += 1
    elif depth < 0:
        raise ValueError("depth must be >= 0")

    cells = cell_coords(pts, center, hw, depth)
    keys = morton(cells, depth)
    perm = np.argsort(keys, kind="stable")              # tree.py:151
    skeys = keys[perm]
    scells = cells[perm]
    ukeys, first = np.unique(skeys, return_index=True)
    last = np.append(first[1:], len(pts))

    lev, cel, st, sp, par, kids = [], [], [], [], [], []
    levels = [[] for _ in range(depth + 1)]
    for a, b in zip(first, last):                       # leaves, Morton order
        levels[depth].append(len(lev))
        lev.append(depth); cel.append(tuple(int(v) for v in scells[a]))
        st.append(int(a)); sp.append(int(b)); par.append(-1); kids.append([])
    cur_ids, cur_keys = list(levels[depth]), [int(k) for k in ukeys]
    for lv in range(depth - 1, -1, -1):                 # tree.py:168-193
        groups = {}
        for cid, key in zip(cur_ids, cur_keys):
            groups.setdefault(key >> 3, []).append(cid)
        nxt_ids, nxt_keys = [], []
        for pk in sorted(groups):
            ch = groups[pk]
            pid = len(lev)
            lev.append(lv); cel.append(tuple(v >> 1 for v in cel[ch[0]]))
            st.append(st[ch[0]]); sp.append(sp[ch[-1]]); par.append(-1)
            kids.append(list(ch))
            for c in ch:
                par[c] = pid
            levels[lv].append(pid)
            nxt_ids.append(pid); nxt_keys.append(pk)
        cur_ids, cur_keys = nxt_ids, nxt_keys

    level = np.array(lev, dtype=np.int64)
    cell = np.array(cel, dtype=np.int64).reshape(-1, 3)
    hws = hw / (1 << level).astype(float)
    # tree.py:199-202 cell centre: lo + h*(cell + 0.5)
    hcell = (2.0 * hw / (1 << level).astype(float))[:, None]
    ccenter = (center - hw) + hcell * (cell.astype(float) + 0.5)
    return Tree(pts[perm], perm, depth, center, hw, level, cell, ccenter, hws,
                np.array(st), np.array(sp), np.array(par), kids, levels)


@dataclass
class Topo:
    neighbors: list
    interactions: list
    nbr_sets: list

    def adjacent(self, i, j):
        return j in self.nbr_sets[i]


def build_topology(tree: Tree) -> Topo:
    """tree.py:205-239."""
    n = tree.n_clusters
    nbrs = [[] for _ in range(n)]
    inter = [[] for _ in range(n)]
    for ids in tree.levels:
        where = {tuple(tree.cell[c]): c for c in ids}
        for c in ids:
            x, y, z = tree.cell[c]
            found = []
            for dx in (-1, 0, 1):
                for dy in (-1, 0, 1):
                    for dz in (-1, 0, 1):
                        o = where.get((x + dx, y + dy, z + dz))
                        if o is not None:
                            found.append(o)
            nbrs[c] = sorted(found)
    sets = [set(v) for v in nbrs]
    for lv in range(2, tree.depth + 1):
        for c in tree.levels[lv]:
            cand = []
            for pn in nbrs[tree.parent[c]]:
                cand.extend(tree.children[pn])
            inter[c] = sorted(q for q in cand if q not in sets[c])
    return Topo(nbrs, inter, sets)


# --------------------------------------------------------------------------
# Chebyshev H2 operators (h2.py:29-182)
# --------------------------------------------------------------------------

def cheb_nodes(n):
    """h2.py:29-31."""
    return np.cos((2.0 * np.arange(n) + 1.0) * np.pi / (2.0 * n))


def cheb_weights(t, n):
    """h2.py:34-49: S[t, m] = 1/n + 2/n sum_k T_k(t) T_k(x_m)."""
    xm = cheb_nodes(n)
    tc = np.clip(t, -1.0, 1.0)
    S = np.full((len(tc), n), 1.0 / n)
    if n > 1:
        k = np.arange(1, n)[None, :]
        Tt = np.cos(np.arccos(tc)[:, None] * k)
        Tx = np.cos(np.arccos(xm)[:, None] * k)
        S += (2.0 / n) * Tt @ Tx.T
    return S


def cheb_grid(center, hw, n):
    """h2.py:52-57: n^3 x 3, x index slowest."""
    g = cheb_nodes(n)
    X, Yg, Z = np.meshgrid(g, g, g, indexing="ij")
    return center + hw * np.column_stack([X.ravel(), Yg.ravel(), Z.ravel()])


def interp_matrix(pts, center, hw, n):
    """h2.py:60-67."""
    rel = (pts - center) / hw
    Sx, Sy, Sz = (cheb_weights(rel[:, a], n) for a in range(3))
    return np.einsum("pi,pj,pk->pijk", Sx, Sy, Sz).reshape(len(pts), n ** 3)


@dataclass
class Ops:
    tree: Tree
    topo: Topo
    block: object
    n_cheb: int
    rank: dict
    leaf_u: dict
    leaf_v: dict
    transfer_u: dict
    transfer_vt: dict
    coupling: dict
    near: dict
    sigma_u: dict = field(default_factory=dict)
    sigma_v: dict = field(default_factory=dict)

    @property
    def dim(self):
        return len(self.tree.points)


def h2_operators(tree: Tree, topo: Topo, block, n, epsilon=0.0) -> Ops:
    """h2.py:104-182 (block_dim 1, symmetric kernel)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rel = max(epsilon, 1e-13)

    def reduce(M):                                      # h2.py:124-127
        W, s, Zt = _svd(M)
        k = max(1, int(np.sum(s > rel * s[0])))
        return W[:, :k], s[:k, None] * Zt[:k]

    rank, leaf_u, tu, G, grids = {}, {}, {}, {}, {}

    def grid_of(c):
        if c not in grids:
            grids[c] = cheb_grid(tree.ccenter[c], tree.chw[c], n)
        return grids[c]

    for c in tree.leaves():
        P = interp_matrix(tree.points[tree.start[c]:tree.stop[c]],
                          tree.ccenter[c], tree.chw[c], n)
        B, G[c] = reduce(P)
        leaf_u[c] = B
        rank[c] = B.shape[1]
    for lv in range(tree.depth - 1, 1, -1):             # h2.py:137-152
        for p in tree.levels[lv]:
            stack = [G[c] @ interp_matrix(grid_of(c), tree.ccenter[p], tree.chw[p], n)
                     for c in tree.children[p]]
            B, G[p] = reduce(np.vstack(stack))
            rank[p] = B.shape[1]
            off = 0
            for c in tree.children[p]:
                tu[c] = B[off:off + rank[c]]
                off += rank[c]
    coupling = {}
    for lv in range(2, tree.depth + 1):                 # h2.py:154-164
        for i in tree.levels[lv]:
            gi = grid_of(i)
            for j in topo.interactions[i]:
                if (i, j) in coupling:
                    continue
                K = G[i] @ block(gi, grid_of(j)) @ G[j].T
                coupling[(i, j)] = K
                coupling[(j, i)] = K.T
    near = {}
    for i in tree.leaves():                             # h2.py:166-177
        pi = tree.points[tree.start[i]:tree.stop[i]]
        for j in topo.neighbors[i]:
            if (i, j) in near:
                continue
            S = block(pi, tree.points[tree.start[j]:tree.stop[j]])
            near[(i, j)] = S
            if j != i:
                near[(j, i)] = S.T
    leaf_v = {c: U.copy() for c, U in leaf_u.items()}
    tvt = {c: T.T.copy() for c, T in tu.items()}
    return Ops(tree, topo, block, n, rank, leaf_u, leaf_v, tu, tvt, coupling, near)


def basis_weights(ops: Ops) -> Ops:
    """h2.py:185-231, rigorous mode, symmetric kernel (P == Q)."""
    tree, topo = ops.tree, ops.topo
    for lv in range(2, tree.depth + 1):
        for j in tree.levels[lv]:
            k = ops.rank[j]
            il = topo.interactions[j]
            if not il:
                ops.sigma_u[j] = np.ones(k)
                ops.sigma_v[j] = np.ones(k)
                continue
            P, s, _ = _svd(np.hstack([ops.coupling[(j, q)] for q in il]))
            if P.shape[1] < k:                          # h2.py:234-239
                P = np.linalg.qr(np.hstack([P, np.eye(k)]))[0][:, :k]
            else:
                P = P[:, :k]
            ops.sigma_u[j] = _weights_from(s, k)
            ops.sigma_v[j] = ops.sigma_u[j].copy()
            # h2.py:265-290 rotations
            if tree.children[j]:
                for c in tree.children[j]:
                    ops.transfer_u[c] = ops.transfer_u[c] @ P
            else:
                ops.leaf_u[j] = ops.leaf_u[j] @ P
            for q in il:
                ops.coupling[(j, q)] = P.T @ ops.coupling[(j, q)]
            if j in ops.transfer_u:
                ops.transfer_u[j] = P.T @ ops.transfer_u[j]
            if tree.children[j]:
                for c in tree.children[j]:
                    ops.transfer_vt[c] = P.T @ ops.transfer_vt[c]
            else:
                ops.leaf_v[j] = ops.leaf_v[j] @ P
            for q in il:
                ops.coupling[(q, j)] = ops.coupling[(q, j)] @ P
            if j in ops.transfer_vt:
                ops.transfer_vt[j] = ops.transfer_vt[j] @ P
    return ops


def _weights_from(s, k):
    """h2.py:242-247."""
    if len(s) == 0:
        return np.ones(k)
    w = np.concatenate([s[:k], np.full(max(0, k - len(s)), s[min(len(s), k) - 1])])
    return np.maximum(w, 1e-14 * (w[0] if w[0] > 0 else 1.0))


# --------------------------------------------------------------------------
# extended sparse graph (graph.py:30-241)
# --------------------------------------------------------------------------

class Graph:
    """graph.py:30-216.  Node ids: leaf x (Morton), then per level 2..L a
    (z, y) pair per cluster; merged parent x nodes appended later."""

    def __init__(self, ops: Ops, b=None):
        tree = ops.tree
        self.ops, self.tree, self.topo = ops, tree, ops.topo
        self.sizes, self.kinds, self.owner = [], [], []
        self.nx, self.nz, self.ny = {}, {}, {}
        self.E = {}
        self.rows, self.cols = {}, {}
        self.rhs = {}
        self.dead = set()
        self.su = {c: w.copy() for c, w in ops.sigma_u.items()}
        self.sv = {c: w.copy() for c, w in ops.sigma_v.items()}
        self.peak_edges = 0
        for c in tree.leaves():
            self.nx[c] = self.add_node(int(tree.stop[c] - tree.start[c]), "x", c)
        for lv in range(2, tree.depth + 1):
            for c in tree.levels[lv]:
                self.nz[c] = self.add_node(ops.rank[c], "z", c)
                self.ny[c] = self.add_node(ops.rank[c], "y", c)
        for (i, j), S in ops.near.items():             # graph.py:63-84
            self.put(self.nx[i], self.nx[j], S.copy())
        if tree.depth >= 2:
            for c in tree.leaves():
                self.put(self.nx[c], self.nz[c], ops.leaf_u[c].copy())
                self.put(self.nz[c], self.nx[c], ops.leaf_v[c].T.copy())
        for lv in range(2, tree.depth + 1):
            for c in tree.levels[lv]:
                k = ops.rank[c]
                self.put(self.nz[c], self.ny[c], -np.eye(k))
                self.put(self.ny[c], self.nz[c], -np.eye(k))
        for (i, j), K in ops.coupling.items():
            self.put(self.ny[i], self.ny[j], K.copy())
        for c, T in ops.transfer_u.items():
            self.put(self.ny[c], self.nz[tree.parent[c]], T.copy())
        for c, Tt in ops.transfer_vt.items():
            self.put(self.nz[tree.parent[c]], self.ny[c], Tt.copy())
        self.load_rhs(b)

    def add_node(self, size, kind, owner):
        nid = len(self.sizes)
        self.sizes.append(size); self.kinds.append(kind); self.owner.append(owner)
        self.rows[nid] = set(); self.cols[nid] = set()
        self.rhs[nid] = np.zeros(size)
        return nid

    def put(self, t, s, blk):
        if (t, s) not in self.E:
            self.rows[t].add(s); self.cols[s].add(t)
        self.E[(t, s)] = blk
        self.peak_edges = max(self.peak_edges, len(self.E))

    def accumulate(self, t, s, blk):
        if (t, s) in self.E:
            self.E[(t, s)] = self.E[(t, s)] + blk
        else:
            self.put(t, s, blk)

    def take(self, t, s):
        blk = self.E.pop((t, s))
        self.rows[t].discard(s); self.cols[s].discard(t)
        return blk

    def load_rhs(self, b):
        for nid in self.rhs:
            self.rhs[nid] = np.zeros(self.sizes[nid])
        if b is None:
            return
        b = np.asarray(b, dtype=float)
        if len(b) != len(self.tree.points):
            raise ValueError("rhs length mismatch")
        bt = b[self.tree.perm]
        for c in self.tree.leaves():
            self.rhs[self.nx[c]] = bt[self.tree.start[c]:self.tree.stop[c]].copy()

    def offsets(self):
        off = np.concatenate([[0], np.cumsum(self.sizes)]).astype(int)
        return off[:-1], int(off[-1])

    def apply(self, w, transpose=False):
        """graph.py:157-170."""
        off, tot = self.offsets()
        out = np.zeros((tot,) + w.shape[1:])
        for (t, s), B in self.E.items():
            if transpose:
                out[off[s]:off[s] + B.shape[1]] += B.T @ w[off[t]:off[t] + B.shape[0]]
            else:
                out[off[t]:off[t] + B.shape[0]] += B @ w[off[s]:off[s] + B.shape[1]]
        return out

    def dense(self):
        off, tot = self.offsets()
        A = np.zeros((tot, tot))
        for (t, s), B in self.E.items():
            A[off[t]:off[t] + B.shape[0], off[s]:off[s] + B.shape[1]] = B
        return A


# --------------------------------------------------------------------------
# low-rank primitives (lowrank.py:22-199)
# --------------------------------------------------------------------------

@dataclass
class LR:
    U: np.ndarray
    s: np.ndarray
    V: np.ndarray

    @property
    def rank(self):
        return len(self.s)


def _lr_empty(m, n):
    return LR(np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0)))


def svd_trunc(M, thr):
    """lowrank.py:54-61 (absolute threshold)."""
    if M.size == 0:
        return _lr_empty(*M.shape)
    U, s, Vt = _svd(M)
    k = int(np.sum(s > thr))
    return LR(U[:, :k].copy(), s[:k].copy(), Vt[:k].T.copy())


def rsvd(apply, apply_t, m, n, thr, oversample=10, power_iters=2, rng=None,
         start_rank=16, max_rank=None):
    """lowrank.py:79-119 (doubling sketch)."""
    if rng is None:
        rng = np.random.default_rng(0)
    full = min(m, n)
    if full == 0:
        return _lr_empty(m, n)
    cap = full if max_rank is None else min(full, max_rank)
    kt = min(start_rank, cap)
    while True:
        width = min(kt + oversample, full)
        Y = apply(rng.standard_normal((n, width)))
        for _ in range(power_iters):
            Y = apply(apply_t(np.linalg.qr(Y)[0]))
        Q = np.linalg.qr(Y)[0]
        Wb, s, Vt = _svd(apply_t(Q).T)
        if width >= full or kt >= cap or (len(s) > kt and s[kt] <= thr):
            break
        kt = min(2 * kt, cap)
    keep = min(int(np.sum(s > thr)), cap)
    if keep == 0:
        return _lr_empty(m, n)
    return LR(Q @ Wb[:, :keep], s[:keep].copy(), Vt[:keep].T.copy())


def aca(M, thr, min_rank=0, margin=8.0):
    """lowrank.py:128-163: full-pivot ACA to thr/margin, then QR-QR-SVD."""
    m, n = M.shape
    if M.size == 0:
        return _lr_empty(m, n)
    floor = thr / margin
    R = np.array(M, dtype=float, copy=True)
    cs, rs = [], []
    for _ in range(min(m, n)):
        p, q = np.unravel_index(np.argmax(np.abs(R)), R.shape)
        piv = R[p, q]
        if piv == 0.0 or (abs(piv) <= floor and len(cs) >= min_rank):
            break
        c = R[:, q].copy()
        r = R[p, :] / piv
        cs.append(c); rs.append(r)
        R -= np.outer(c, r)
    if not cs:
        return _lr_empty(m, n)
    QA, RA = np.linalg.qr(np.column_stack(cs))
    QB, RB = np.linalg.qr(np.vstack(rs).T)
    W, s, Zt = _svd(RA @ RB.T, full_matrices=True)
    k = max(int(np.sum(s > thr)), min(min_rank, len(s)))
    if k == 0:
        return _lr_empty(m, n)
    return LR(QA @ W[:, :k], s[:k].copy(), QB @ Zt[:k].T)


@dataclass
class Union:
    basis: np.ndarray
    weights: np.ndarray
    old_map: np.ndarray
    fill_map: np.ndarray

    @property
    def rank(self):
        return self.basis.shape[1]


def basis_union(B, w, F, wf, thr, min_rank=0):
    """lowrank.py:166-199."""
    w = np.asarray(w, dtype=float)
    wf = np.asarray(wf, dtype=float)
    if B.shape[1] != len(w) or F.shape[1] != len(wf):
        raise ValueError("basis/weight size mismatch")
    if np.any(w <= 0.0) or np.any(wf <= 0.0):
        raise ValueError("weights must be positive")
    k0 = B.shape[1]
    f = aca(np.hstack([B * w, F * wf]), thr, min_rank=min_rank)
    sc = f.s[:, None] * f.V.T
    return Union(f.U, f.s.copy(), sc[:, :k0] / w[None, :], sc[:, k0:] / wf[None, :])


# --------------------------------------------------------------------------
# sigma0 (graph.py:232-241)
# --------------------------------------------------------------------------

def sigma0_estimate(g: Graph, seed=0, oversample=10, power_iters=2):
    rng = np.random.Generator(np.random.PCG64(seed))
    _, dim = g.offsets()
    f = rsvd(lambda w: g.apply(w), lambda w: g.apply(w, transpose=True), dim, dim,
             0.0, oversample=oversample, power_iters=power_iters, rng=rng,
             start_rank=1, max_rank=1)
    return float(f.s[0])


# --------------------------------------------------------------------------
# factorization (factor.py:38-578)
# --------------------------------------------------------------------------

@dataclass
class LevelStats:
    """factor.py:38-54."""
    level: int
    compressed_pairs: int = 0
    added: int = 0
    dropped_pairs: int = 0
    ranks: list = field(default_factory=list)
    forced_rank_truncations: int = 0

    @property
    def max_rank(self):
        return max(self.ranks) if self.ranks else 0


def _lu(P, what):
    """factor.py:166-173."""
    if P.shape[0] == 0:
        return None
    lu, piv = sla.lu_factor(P, check_finite=False)
    d = np.abs(np.diag(lu))
    if not np.all(np.isfinite(lu)) or (d.size and d.min() == 0.0):
        raise SingularPivotError(what)
    return lu, piv


def _lusolve(f, rhs):
    """factor.py:160-163."""
    if f is None:
        return rhs[:0]
    return sla.lu_solve(f, rhs)


class Factor:
    """factor.py:75-157 replay log."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    def solve(self, b):
        b = np.asarray(b, dtype=float)
        if b.shape != (self.n_points,):
            raise ValueError(f"rhs must have shape ({self.n_points},)")
        bt = b[self.perm]
        r = {nid: np.zeros(s) for nid, s in enumerate(self.init_sizes)}
        for nxid, a, e in self.leaf_slices:
            r[nxid] = bt[a:e].copy()
        for ev in self.events:                        # forward (factor.py:111-126)
            if ev[0] == "elim":
                _, nxid, nzid, nyid, m, k, f, src, tgt = ev
                g = _lusolve(f, np.concatenate([r[nxid], np.zeros(k)]))
                for a, B in tgt:
                    r[a] = r[a] - B @ g[:m]
                r[nyid] = r[nyid] + g[m:]
            elif ev[0] == "rebase":
                r[ev[1]] = ev[2] @ r[ev[1]]
            else:
                _, px, parts = ev
                r[px] = np.concatenate([r[cy] for cy, _ in parts]) if parts else np.zeros(0)
        sol = {}
        if self.top_nodes:                            # factor.py:129-135
            y = _lusolve(self.top_lu, np.concatenate([r[t] for t in self.top_nodes]))
            off = 0
            for t, s in zip(self.top_nodes, self.top_sizes):
                sol[t] = y[off:off + s]
                off += s
        for ev in reversed(self.events):              # backward (factor.py:137-152)
            if ev[0] == "elim":
                _, nxid, nzid, nyid, m, k, f, src, tgt = ev
                rx = r[nxid].copy()
                for bn, B in src:
                    rx -= B @ sol[bn]
                xz = _lusolve(f, np.concatenate([rx, sol[nyid]]))
                sol[nxid], sol[nzid] = xz[:m], xz[m:]
            elif ev[0] == "merge":
                off = 0
                for cy, s in ev[2]:
                    sol[cy] = sol[ev[1]][off:off + s]
                    off += s
        xt = np.concatenate([sol[nxid] for nxid, _, _ in self.leaf_slices])
        x = np.empty_like(xt)
        x[self.perm] = xt
        return x


def factorize(g: Graph, epsilon, seed=0, sigma0=None, exact_fill_svd=False):
    """factor.py:176-230.  ``exact_fill_svd`` swaps the rSVD branch of
    factor.py:329-332 for a plain truncated SVD (the CUDA path's choice)."""
    if not 0.0 < epsilon < 1.0:
        raise ValueError("epsilon must be in (0, 1)")
    tree = g.tree
    rng = np.random.Generator(np.random.PCG64(seed))
    t0 = time.perf_counter()
    if sigma0 is None:
        sigma0 = sigma0_estimate(g, seed=seed)
    t_sigma0 = time.perf_counter() - t0
    thr = epsilon * sigma0
    init_sizes = list(g.sizes)
    leaf_slices = [(g.nx[c], int(tree.start[c]), int(tree.stop[c])) for c in tree.leaves()]
    events, levels = [], []
    ctx = dict(thr=thr, rng=rng, events=events, exact=exact_fill_svd)
    for lv in range(tree.depth, 1, -1):
        st = LevelStats(lv)
        for c in tree.levels[lv]:
            eliminate_one(g, c, st, ctx)
        levels.append(st)
        if lv > 2:
            merge_level(g, lv, events)
    top = ([g.ny[c] for c in tree.levels[2]] if tree.depth >= 2
           else [g.nx[c] for c in tree.leaves()])
    tsz = [g.sizes[t] for t in top]
    top_lu = _top_lu(g, top, tsz)
    return Factor(n_points=len(tree.points), perm=tree.perm, init_sizes=init_sizes,
                  leaf_slices=leaf_slices, events=events, top_nodes=top,
                  top_sizes=tsz, top_lu=top_lu, epsilon=epsilon, sigma0=sigma0,
                  levels=levels, peak_edges=g.peak_edges,
                  max_basis_rank=max((len(w) for w in g.su.values()), default=0),
                  forced=sum(s.forced_rank_truncations for s in levels),
                  t_sigma0=t_sigma0)


def _top_lu(g, top, tsz):
    """factor.py:233-246."""
    off = np.concatenate([[0], np.cumsum(tsz)]).astype(int)
    pos = {t: i for i, t in enumerate(top)}
    if off[-1] == 0:
        return None
    M = np.zeros((off[-1], off[-1]))
    for (t, s), B in g.E.items():
        if t in pos and s in pos:
            M[off[pos[t]]:off[pos[t]] + B.shape[0], off[pos[s]]:off[pos[s]] + B.shape[1]] = B
    return _lu(M, "top-level system")


TRACE = None  # optional list collecting per-pair decisions (triage only)


def _tr(*a):
    if TRACE is not None:
        TRACE.append(" ".join(str(int(v)) if not isinstance(v, str) else v for v in a))


def eliminate_one(g: Graph, c, st: LevelStats, ctx, compress_ws=True):
    """factor.py:259-326."""
    nxid, nzid, nyid = g.nx[c], g.nz[c], g.ny[c]
    _tr("E", c, g.sizes[nxid], g.sizes[nzid])
    m, k = g.sizes[nxid], g.sizes[nzid]
    D = g.take(nxid, nxid)
    U = g.take(nxid, nzid)
    Vt = g.take(nzid, nxid)
    g.take(nzid, nyid)
    g.take(nyid, nzid)
    f = _lu(np.block([[D, U], [Vt, np.zeros((k, k))]]), f"cluster {c}")
    src = [(b, g.take(nxid, b)) for b in sorted(g.rows[nxid])]
    tgt = [(a, g.take(a, nxid)) for a in sorted(g.cols[nxid])]
    if g.rows[nzid] or g.cols[nzid]:
        raise AssertionError("z node unexpectedly has extra edges")
    ctx["events"].append(("elim", nxid, nzid, nyid, m, k, f, src, tgt))
    g.dead.add(c)
    X = {b: _lusolve(f, np.vstack([B, np.zeros((k, B.shape[1]))])) for b, B in src}
    X[nyid] = _lusolve(f, np.vstack([np.zeros((m, k)), -np.eye(k)]))
    gr = _lusolve(f, np.concatenate([g.rhs[nxid], np.zeros(k)]))
    for a, B in tgt:
        g.rhs[a] = g.rhs[a] - B @ gr[:m]
    g.rhs[nyid] = g.rhs[nyid] + gr[m:]
    stash = {}
    for a, Ea in tgt + [(nyid, None)]:
        ca = g.owner[a]
        for b in [b for b, _ in src] + [nyid]:
            F = X[b][m:, :] if a == nyid else -(Ea @ X[b][:m, :])
            cb = g.owner[b]
            if (not compress_ws) or (ca in g.dead and cb in g.dead) or g.topo.adjacent(ca, cb):
                g.accumulate(a, b, F)
                st.added += 1
            else:
                stash[(ca, cb)] = F
    for cj, ck in sorted({(min(p), max(p)) for p in stash}):
        redirect(g, cj, ck, stash.get((ck, cj)), stash.get((cj, ck)), st, ctx)


def _compress(M, ctx):
    """factor.py:329-332."""
    if min(M.shape) > 64 and not ctx["exact"]:
        return rsvd(lambda X: M @ X, lambda X: M.T @ X, M.shape[0], M.shape[1],
                    ctx["thr"], rng=ctx["rng"])
    return svd_trunc(M, ctx["thr"])


def _pad_union(u: Union, kt, floor, rng):
    """factor.py:340-358."""
    m, k = u.basis.shape
    extra = min(kt, m) - k
    if extra <= 0:
        return u
    G = rng.standard_normal((m, extra))
    G -= u.basis @ (u.basis.T @ G)
    Q = np.linalg.qr(G)[0]
    w = max(floor, 1e-14 * (u.weights.max() if k else 1.0))
    return Union(np.hstack([u.basis, Q[:, :extra]]),
                 np.concatenate([u.weights, np.full(extra, w)]),
                 np.vstack([u.old_map, np.zeros((extra, u.old_map.shape[1]))]),
                 np.vstack([u.fill_map, np.zeros((extra, u.fill_map.shape[1]))]))


def _cut_union(u: Union, k):
    return Union(u.basis[:, :k], u.weights[:k], u.old_map[:k], u.fill_map[:k])


def unions_for(g: Graph, c, fu, wu, fv, wv, st, ctx):
    """factor.py:366-392."""
    thr, rng = ctx["thr"], ctx["rng"]
    Uc = g.E[(g.nx[c], g.nz[c])]
    Vc = g.E[(g.nz[c], g.nx[c])].T
    su, sv = g.su[c], g.sv[c]

    def one(B, w, F, wf, mr=0):
        if F is not None and F.shape[1]:
            return basis_union(B, w, F, wf, thr, min_rank=mr)
        return Union(B, w.copy(), np.eye(B.shape[1]), np.zeros((B.shape[1], 0)))

    uu, uv = one(Uc, su, fu, wu), one(Vc, sv, fv, wv)
    if uu.rank != uv.rank:
        kk = max(uu.rank, uv.rank)
        if uu.rank < kk and fu is not None and fu.shape[1]:
            uu = basis_union(Uc, su, fu, wu, thr, min_rank=kk)
        if uv.rank < kk and fv is not None and fv.shape[1]:
            uv = basis_union(Vc, sv, fv, wv, thr, min_rank=kk)
        if uu.rank < kk:
            uu = _pad_union(uu, kk, thr, rng)
        if uv.rank < kk:
            uv = _pad_union(uv, kk, thr, rng)
        if uu.rank != uv.rank:
            kk = min(uu.rank, uv.rank)
            uu, uv = _cut_union(uu, kk), _cut_union(uv, kk)
            st.forced_rank_truncations += 1
    return uu, uv


def rebase(g: Graph, c, uu: Union, uv: Union, partner, events):
    """factor.py:395-430."""
    nxid, nzid, nyid = g.nx[c], g.nz[c], g.ny[c]
    _tr("R", c, uu.old_map.shape[1], uu.rank, uv.rank)
    py = g.ny[partner]
    r, t = uu.old_map, uv.old_map
    kn = uu.rank
    g.put(nxid, nzid, uu.basis)
    g.put(nzid, nxid, uv.basis.T)
    g.su[c], g.sv[c] = uu.weights, uv.weights
    for b in sorted(g.rows[nyid]):
        if b not in (nzid, py):
            g.put(nyid, b, r @ g.E[(nyid, b)])
    for a in sorted(g.cols[nyid]):
        if a not in (nzid, py):
            g.put(a, nyid, g.E[(a, nyid)] @ t.T)
    g.take(nzid, nyid)
    g.take(nyid, nzid)
    g.sizes[nzid] = kn
    g.sizes[nyid] = kn
    g.put(nzid, nyid, -np.eye(kn))
    g.put(nyid, nzid, -np.eye(kn))
    g.rhs[nyid] = r @ g.rhs[nyid]
    if not (r.shape[0] == r.shape[1] and np.array_equal(r, np.eye(r.shape[0]))):
        events.append(("rebase", nyid, r))


def redirect(g: Graph, cj, ck, F_kj, F_jk, st: LevelStats, ctx):
    """factor.py:433-522."""
    ej, ek = cj in g.dead, ck in g.dead
    if ej and ek:
        raise AssertionError("both-eliminated fills are added, not redirected")
    f_kj = _compress(F_kj, ctx) if F_kj is not None else None
    f_jk = _compress(F_jk, ctx) if F_jk is not None else None
    r1 = f_kj.rank if f_kj is not None else 0
    r2 = f_jk.rank if f_jk is not None else 0
    if r1 == 0 and r2 == 0:
        st.dropped_pairs += 1
        _tr("D", cj, ck)
        return
    st.compressed_pairs += 1
    st.ranks.append(max(r1, r2))
    _tr("P", cj, ck, r1, r2, ej, ek)
    yj, yk = g.ny[cj], g.ny[ck]
    old_kj = g.E.get((yk, yj))
    old_jk = g.E.get((yj, yk))
    if old_kj is None:
        old_kj = np.zeros((g.sizes[yk], g.sizes[yj]))
    if old_jk is None:
        old_jk = np.zeros((g.sizes[yj], g.sizes[yk]))

    def split(f, m, n):
        if f is None or f.rank == 0:
            return np.zeros((m, 0)), np.zeros(0), np.zeros((n, 0))
        return f.U, f.s, f.V

    ev = ctx["events"]
    if not ej and not ek:
        mj, mk = g.sizes[g.nx[cj]], g.sizes[g.nx[ck]]
        Ukj, skj, Vkj = split(f_kj, mk, mj)
        Ujk, sjk, Vjk = split(f_jk, mj, mk)
        uj, vj = unions_for(g, cj, Ujk, sjk, Vkj, skj, st, ctx)
        uk, vk = unions_for(g, ck, Ukj, skj, Vjk, sjk, st, ctx)
        rebase(g, cj, uj, vj, ck, ev)
        rebase(g, ck, uk, vk, cj, ev)
        g.put(yk, yj, uk.old_map @ old_kj @ vj.old_map.T + (uk.fill_map * skj) @ vj.fill_map.T)
        g.put(yj, yk, uj.old_map @ old_jk @ vk.old_map.T + (uj.fill_map * sjk) @ vk.fill_map.T)
    else:
        live, dead = (ck, cj) if ej else (cj, ck)
        fu, fv = (f_kj, f_jk) if ej else (f_jk, f_kj)
        ml = g.sizes[g.nx[live]]
        nd = g.sizes[g.ny[dead]]
        Ul, sl, Wl = split(fu, ml, nd)
        Ud, sd, Vl = split(fv, nd, ml)
        uu, uv = unions_for(g, live, Ul, sl, Vl, sd, st, ctx)
        rebase(g, live, uu, uv, dead, ev)
        old_ld = old_kj if live == ck else old_jk
        old_dl = old_jk if live == ck else old_kj
        K_ld = (sl[:, None] * Wl.T) if len(sl) else np.zeros((0, nd))
        K_dl = (Ud * sd) if len(sd) else np.zeros((nd, 0))
        g.put(g.ny[live], g.ny[dead], uu.old_map @ old_ld + uu.fill_map @ K_ld)
        g.put(g.ny[dead], g.ny[live], old_dl @ uv.old_map.T + K_dl @ uv.fill_map.T)


def merge_level(g: Graph, lv, events):
    """factor.py:525-578."""
    tree = g.tree
    px_of, off_of, owner = {}, {}, {}
    for p in tree.levels[lv - 1]:
        parts, o = [], 0
        for c in tree.children[p]:
            cy = g.ny[c]
            off_of[cy] = o
            parts.append((cy, g.sizes[cy]))
            owner[cy] = p
            o += g.sizes[cy]
        px = g.add_node(o, "x", p)
        g.nx[p] = px
        px_of[p] = px
        g.rhs[px] = np.concatenate([g.rhs[cy] for cy, _ in parts]) if parts else np.zeros(0)
        events.append(("merge", px, parts))
    for (t, s) in [e for e in g.E if e[0] in owner or e[1] in owner]:
        B = g.take(t, s)
        if t in owner and s in owner:
            a, b = px_of[owner[t]], px_of[owner[s]]
            if (a, b) not in g.E:
                g.put(a, b, np.zeros((g.sizes[a], g.sizes[b])))
            g.E[(a, b)][off_of[t]:off_of[t] + B.shape[0], off_of[s]:off_of[s] + B.shape[1]] += B
        elif t in owner:
            a = px_of[owner[t]]
            if (a, s) not in g.E:
                g.put(a, s, np.zeros((g.sizes[a], g.sizes[s])))
            g.E[(a, s)][off_of[t]:off_of[t] + B.shape[0], :] += B
        else:
            b = px_of[owner[s]]
            if (t, b) not in g.E:
                g.put(t, b, np.zeros((g.sizes[t], g.sizes[b])))
            g.E[(t, b)][:, off_of[s]:off_of[s] + B.shape[1]] += B


# --------------------------------------------------------------------------
# FMM matvec + GMRES (krylov.py:32-159)
# --------------------------------------------------------------------------

def h2_matvec(ops: Ops, x):
    """krylov.py:119-159."""
    tree, topo = ops.tree, ops.topo
    x = np.asarray(x, dtype=float)
    if len(x) != len(tree.points):
        raise ValueError("vector length mismatch")
    xt = x[tree.perm]
    up = {c: ops.leaf_v[c].T @ xt[tree.start[c]:tree.stop[c]] for c in tree.leaves()}
    for lv in range(tree.depth - 1, 1, -1):
        for p in tree.levels[lv]:
            up[p] = sum(ops.transfer_vt[c] @ up[c] for c in tree.children[p])
    down = {}
    for lv in range(2, tree.depth + 1):
        for c in tree.levels[lv]:
            acc = np.zeros(ops.rank[c])
            for q in topo.interactions[c]:
                acc += ops.coupling[(c, q)] @ up[q]
            if lv > 2:
                acc += ops.transfer_u[c] @ down[tree.parent[c]]
            down[c] = acc
    out = np.zeros_like(xt)
    for c in tree.leaves():
        a, e = tree.start[c], tree.stop[c]
        seg = np.zeros(e - a)
        for q in topo.neighbors[c]:
            seg += ops.near[(c, q)] @ xt[tree.start[q]:tree.stop[q]]
        if tree.depth >= 2:
            seg += ops.leaf_u[c] @ down[c]
        out[a:e] = seg
    res = np.empty_like(out)
    res[tree.perm] = out
    return res


def gmres(apply_A, b, tol=1e-10, max_iters=500, precond=None, side="right"):
    """krylov.py:32-116: MGS Arnoldi + Givens.  Returns (x, its, hist, conv)."""
    if tol <= 0 or max_iters < 1:
        raise ValueError("tol must be > 0 and max_iters >= 1")
    if precond is None:
        side = "none"
    n = len(b)
    r0 = precond(b) if side == "left" else b
    beta = np.linalg.norm(r0)
    hist = []
    if beta == 0.0:
        return np.zeros(n), 0, hist, True
    V = np.zeros((max_iters + 1, n))
    H = np.zeros((max_iters + 1, max_iters))
    cs, sn = np.zeros(max_iters), np.zeros(max_iters)
    gv = np.zeros(max_iters + 1)
    gv[0] = beta
    V[0] = r0 / beta
    kd, brk, conv = 0, False, False
    for k in range(max_iters):
        if side == "right":
            w = apply_A(precond(V[k]))
        elif side == "left":
            w = precond(apply_A(V[k]))
        else:
            w = apply_A(V[k])
        for i in range(k + 1):
            H[i, k] = V[i] @ w
            w = w - H[i, k] * V[i]
        hs = np.linalg.norm(w)
        H[k + 1, k] = hs
        for i in range(k):
            h0 = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
            H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
            H[i, k] = h0
        nu = np.hypot(H[k, k], H[k + 1, k])
        if nu == 0.0:
            kd, brk = k, True
            break
        cs[k], sn[k] = H[k, k] / nu, H[k + 1, k] / nu
        H[k, k], H[k + 1, k] = nu, 0.0
        gv[k + 1] = -sn[k] * gv[k]
        gv[k] = cs[k] * gv[k]
        rel = abs(gv[k + 1]) / beta
        hist.append(float(rel))
        kd = k + 1
        if rel <= tol:
            conv = True
            break
        if hs == 0.0:
            brk = True
            break
        V[k + 1] = w / hs
    if brk and hist:
        conv = hist[-1] <= tol
    x = np.zeros(n)
    if kd > 0:
        y = sla.solve_triangular(H[:kd, :kd], gv[:kd])
        u = V[:kd].T @ y
        x = precond(u) if side == "right" else u
    return x, kd, hist, conv


# --------------------------------------------------------------------------
# pinned BASELINE inputs and a one-call pipeline
# --------------------------------------------------------------------------

CONFIGS = {
    # name: (N, dim, seed, kernel, leaf_target, n_cheb, eps)
    "c1": (4096, 2, 0, "exp", 32, 4, 1e-8),
    "c2": (65536, 2, 1, "exp", 64, 6, 1e-10),
    "c3": (262144, 3, 2, "imq", 64, 4, 1e-6),
    "c4": (1048576, 3, 3, "imq", 64, 4, 1e-6),
}


def config_inputs(name, n_override=None):
    """Pinned points, rhs, kernel for a BASELINE config."""
    N, dim, seed, kern, leaf, n, eps = CONFIGS[name]
    if n_override is not None:
        N = n_override
    g = np.random.Generator(np.random.PCG64(seed))
    if dim == 2:
        p2 = g.uniform(0.0, 1.0, size=(N, 2))
        pts = np.column_stack([p2, np.zeros(N)])
    else:
        pts = g.uniform(0.0, 1.0, size=(N, 3))
    gb = np.random.Generator(np.random.PCG64(seed + 1))
    b = gb.uniform(-1.0, 1.0, N) if dim == 2 else gb.standard_normal(N)
    if kern == "exp":
        block, kd = exp_block, ("exp", {})
    else:
        h = N ** (-1.0 / 3.0)
        block, kd = imq_block(h), ("imq", {"h": h})
    return dict(points=pts, b=b, block=block, kernel=kd, leaf=leaf, n=n, eps=eps, N=N)


def pipeline(points, block, leaf, n, eps):
    tree = build_tree(points, leaf)
    topo = build_topology(tree)
    ops = h2_operators(tree, topo, block, n, epsilon=eps)
    basis_weights(ops)
    return tree, topo, ops
