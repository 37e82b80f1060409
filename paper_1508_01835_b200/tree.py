"""Octree, Morton order and cluster topology (mirror of ``ifmm.tree``).

``build_octree`` reproduces the reference tree bit for bit
(tree.py:107-196): data-derived root cube, depth = smallest L >= 2 whose
mean occupied-leaf population is <= leaf_target, cell index
ceil((p - lo)/h) - 1 clipped, 3L-bit Morton keys (x bit lowest), stable
argsort, leaves numbered in Morton order and parents appended bottom-up.
The tree is integer/byte host work on O(N) data; the topology
(tree.py:205-239) is computed by the native engine and handed back as the
reference's list-of-lists.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as N


class DegenerateGeometryError(ValueError):
    """Raised when all input points coincide (tree.py:22-23)."""


@dataclass
class Cluster:
    level: int
    cell: tuple
    center: np.ndarray
    half_width: float
    start: int
    stop: int
    parent: int | None = None
    children: list = field(default_factory=list)

    @property
    def size(self) -> int:
        return self.stop - self.start

    @property
    def is_leaf(self) -> bool:
        return not self.children


@dataclass
class Octree:
    points: np.ndarray
    perm: np.ndarray
    depth: int
    root_center: np.ndarray
    root_half_width: float
    clusters: list
    levels: list
    _handle: object = field(default=None, repr=False)

    @property
    def n_points(self) -> int:
        return len(self.points)

    @property
    def n_clusters(self) -> int:
        return len(self.clusters)

    def leaves(self):
        return self.levels[self.depth]

    def inverse_perm(self):
        inv = np.empty_like(self.perm)
        inv[self.perm] = np.arange(len(self.perm))
        return inv

    # device-side tree (points, permutation, topology) -- created lazily
    def handle(self):
        if self._handle is None:
            self._handle = _TreeHandle(self, device=True)
        return self._handle


@dataclass
class ClusterTopology:
    neighbors: list
    interactions: list
    neighbor_sets: list

    def are_neighbors(self, i: int, j: int) -> bool:
        return j in self.neighbor_sets[i]


def _morton_key(cells: np.ndarray, depth: int) -> np.ndarray:
    """Interleave cell-coordinate bits, axis a of bit b at 3b+a (tree.py:83-89)."""
    c = np.asarray(cells, dtype=np.int64)
    key = np.zeros(len(c), dtype=np.int64)
    for b in range(depth):
        for a in range(3):
            key |= ((c[:, a] >> b) & 1) << (3 * b + a)
    return key


def _cell_indices(points, center, half_width, level):
    """tree.py:92-99: boundary points go to the lower cell."""
    n_cells = 1 << level
    h = 2.0 * half_width / n_cells
    rel = points - (center - half_width)
    idx = np.ceil(rel / h).astype(np.int64) - 1
    return np.clip(idx, 0, n_cells - 1)


def _cell_center(root_center, root_half_width, level, cell):
    h = 2.0 * root_half_width / (1 << level)
    return (root_center - root_half_width) + h * (np.array(cell, dtype=float) + 0.5)


def build_octree(points, leaf_target: int, depth: int | None = None,
                 root_box=None, max_depth: int = 12):
    """Mirror of ifmm.tree.build_octree (tree.py:107-196)."""
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
    if depth is None:
        depth = 2
        while depth < max_depth:
            occ = len(np.unique(_morton_key(_cell_indices(pts, center, hw, depth), depth)))
            if len(pts) / occ <= leaf_target:
                break
            depth += 1
    elif depth < 0:
        raise ValueError("depth must be >= 0")

    cells = _cell_indices(pts, center, hw, depth)
    keys = _morton_key(cells, depth)
    perm = np.argsort(keys, kind="stable")
    skeys = keys[perm]
    scells = cells[perm]
    ukeys, starts = np.unique(skeys, return_index=True)
    stops = np.append(starts[1:], len(pts))

    clusters: list = []
    levels: list = [[] for _ in range(depth + 1)]
    leaf_cells = scells[starts]
    for i in range(len(ukeys)):
        cell = (int(leaf_cells[i, 0]), int(leaf_cells[i, 1]), int(leaf_cells[i, 2]))
        clusters.append(Cluster(depth, cell, _cell_center(center, hw, depth, cell),
                                hw / (1 << depth), int(starts[i]), int(stops[i])))
        levels[depth].append(i)
    ids = np.arange(len(ukeys))
    ckeys = ukeys.copy()
    for lv in range(depth - 1, -1, -1):
        pk = ckeys >> 3
        # children are Morton-sorted, so equal parent keys are contiguous
        uniq, first = np.unique(pk, return_index=True)
        last = np.append(first[1:], len(pk))
        new_ids = []
        for u, a, b in zip(uniq, first, last):
            kids = [int(x) for x in ids[a:b]]
            c0 = clusters[kids[0]]
            cell = tuple(v >> 1 for v in c0.cell)
            pid = len(clusters)
            clusters.append(Cluster(lv, cell, _cell_center(center, hw, lv, cell),
                                    hw / (1 << lv), c0.start, clusters[kids[-1]].stop,
                                    children=kids))
            for k in kids:
                clusters[k].parent = pid
            levels[lv].append(pid)
            new_ids.append(pid)
        ids = np.array(new_ids, dtype=np.int64)
        ckeys = uniq
    tree = Octree(pts[perm], perm, depth, center, hw, clusters, levels)
    return tree, perm


class _TreeHandle:
    """Native copy of the tree: sorted points + permutation on the device,
    and compute_topology (tree.py:205-239) in C++."""

    def __init__(self, tree: Octree, device: bool):
        cl = tree.clusters
        nc = len(cl)
        level = np.array([c.level for c in cl], dtype=np.int32)
        parent = np.array([-1 if c.parent is None else c.parent for c in cl], dtype=np.int32)
        start = np.array([c.start for c in cl], dtype=np.int32)
        stop = np.array([c.stop for c in cl], dtype=np.int32)
        cell = np.array([c.cell for c in cl], dtype=np.int64).reshape(nc, 3)
        center = np.array([c.center for c in cl], dtype=float).reshape(nc, 3)
        hwa = np.array([c.half_width for c in cl], dtype=float)
        cptr = np.zeros(nc + 1, dtype=np.int32)
        cptr[1:] = np.cumsum([len(c.children) for c in cl])
        cidx = np.array([k for c in cl for k in c.children] or [0], dtype=np.int32)
        pts = np.ascontiguousarray(tree.points, dtype=float)
        perm = np.ascontiguousarray(tree.perm, dtype=np.int32)
        self.lib = N.lib()
        h = self.lib.ifmm_tree_create(N.ctx() if device else None, len(pts), N.as_dp(pts), N.as_ip(perm), tree.depth,
                                      nc, N.as_ip(level), N.as_ip(parent), N.as_ip(start),
                                      N.as_ip(stop), N.as_lp(cell), N.as_dp(center),
                                      N.as_dp(hwa), N.as_ip(cptr), N.as_ip(cidx))
        self.h = N.check_handle(h)
        self.n_clusters = nc

    def topology_arrays(self):
        import ctypes as C
        a, b = C.c_longlong(), C.c_longlong()
        self.lib.ifmm_tree_topology_sizes(self.h, C.byref(a), C.byref(b))
        nptr = np.zeros(self.n_clusters + 1, dtype=np.int64)
        iptr = np.zeros(self.n_clusters + 1, dtype=np.int64)
        nidx = np.zeros(max(a.value, 1), dtype=np.int32)
        iidx = np.zeros(max(b.value, 1), dtype=np.int32)
        self.lib.ifmm_tree_topology(self.h, N.as_lp(nptr), N.as_ip(nidx), N.as_lp(iptr),
                                    N.as_ip(iidx))
        return nptr, nidx, iptr, iidx

    def __del__(self):
        try:
            self.lib.ifmm_tree_destroy(self.h)
        except Exception:
            pass


def compute_topology(tree: Octree) -> ClusterTopology:
    """Neighbour / interaction lists (tree.py:205-239), computed natively."""
    hd = tree._handle if tree._handle is not None else _TreeHandle(tree, device=False)
    nptr, nidx, iptr, iidx = hd.topology_arrays()
    nbrs = [nidx[nptr[i]:nptr[i + 1]].tolist() for i in range(tree.n_clusters)]
    inter = [iidx[iptr[i]:iptr[i + 1]].tolist() for i in range(tree.n_clusters)]
    return ClusterTopology(nbrs, inter, [set(v) for v in nbrs])
