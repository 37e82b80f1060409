"""H2 operators on the device (mirror of ``ifmm.h2``).

``chebyshev_operators`` (h2.py:104-182) and ``initialize_weights``
(h2.py:185-231, rigorous mode) run entirely in the CUDA engine; the
returned ``H2Operators`` holds the device handle.  The dict-of-blocks
attributes of the reference (``leaf_u``, ``coupling``, ``near`` ...) are
read-only views that copy one block to the host on access (tests and
inspection only).
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Mapping

import numpy as np

from . import _native as N
from .kernels import Kernel
from .tree import ClusterTopology, Octree

_WHICH = {"leaf_u": 0, "leaf_v": 1, "transfer_u": 2, "transfer_vt": 3, "coupling": 4,
          "near": 5, "sigma_u": 6, "sigma_v": 7}


class _BlockView(Mapping):
    def __init__(self, ops, which, keys):
        self._ops, self._w, self._keys = ops, which, keys

    def _fetch(self, key):
        i, j = key if isinstance(key, tuple) else (key, 0)
        r, c = C.c_int(), C.c_int()
        h = self._ops._h
        N.check(N.lib().ifmm_h2_block(h, self._w, int(i), int(j), None, C.byref(r), C.byref(c)))
        if r.value < 0:
            raise KeyError(key)
        out = np.empty((r.value, c.value))
        N.check(N.lib().ifmm_h2_block(h, self._w, int(i), int(j), N.as_dp(out), C.byref(r),
                                      C.byref(c)))
        return out[0] if self._w in (6, 7) else out

    def __getitem__(self, key):
        if key not in self._keys:
            raise KeyError(key)
        return self._fetch(key)

    def __iter__(self):
        return iter(self._keys)

    def __len__(self):
        return len(self._keys)

    def __contains__(self, key):
        return key in self._keys


class H2Operators:
    """Device-resident operators; attribute views mirror h2.py:76-101."""

    def __init__(self, tree: Octree, topology: ClusterTopology, kernel: Kernel, n_cheb: int,
                 handle):
        self.tree, self.topology, self.kernel, self.n_cheb = tree, topology, kernel, n_cheb
        self._h = handle
        self._tree_handle = tree.handle()  # keep the device tree alive
        nc = tree.n_clusters
        r = np.zeros(nc, dtype=np.int32)
        N.check(N.lib().ifmm_h2_ranks(handle, N.as_ip(r)))
        self.rank = {c: int(r[c]) for c in range(nc) if r[c] >= 0}
        self._weighted = False

    def __del__(self):
        try:
            N.lib().ifmm_h2_destroy(self._h)
        except Exception:
            pass

    @property
    def block_dim(self):
        return self.kernel.block_dim

    @property
    def dim(self):
        return self.tree.n_points * self.kernel.block_dim

    def max_rank(self):
        return max(self.rank.values()) if self.rank else 0

    # ---- reference-shaped read-only views ----
    def _leaf_keys(self):
        return self.tree.leaves() if self.tree.depth >= 2 else []

    @property
    def leaf_u(self):
        return _BlockView(self, 0, set(self._leaf_keys()))

    @property
    def leaf_v(self):
        return _BlockView(self, 1, set(self._leaf_keys()))

    @property
    def transfer_u(self):
        cl = self.tree.clusters
        return _BlockView(self, 2, {c for c in range(len(cl)) if cl[c].level >= 3})

    @property
    def transfer_vt(self):
        cl = self.tree.clusters
        return _BlockView(self, 3, {c for c in range(len(cl)) if cl[c].level >= 3})

    @property
    def coupling(self):
        keys = {(i, j) for lv in range(2, self.tree.depth + 1) for i in self.tree.levels[lv]
                for j in self.topology.interactions[i]}
        return _BlockView(self, 4, keys)

    @property
    def near(self):
        keys = {(i, j) for i in self.tree.leaves() for j in self.topology.neighbors[i]}
        return _BlockView(self, 5, keys)

    @property
    def sigma_u(self):
        return _BlockView(self, 6, set(self.rank) if self._weighted else set())

    @property
    def sigma_v(self):
        return _BlockView(self, 7, set(self.rank) if self._weighted else set())


def chebyshev_operators(tree: Octree, topology: ClusterTopology, kernel: Kernel, n: int,
                        epsilon: float = 0.0) -> H2Operators:
    """h2.py:104-182 on the device."""
    if n < 1:
        raise ValueError("n must be >= 1")
    kind, p0, p1 = kernel.device_spec()
    h = N.lib().ifmm_h2_build_k(tree.handle().h, kind, p0, p1, int(n), float(epsilon))
    return H2Operators(tree, topology, kernel, n, N.check_handle(h))


def initialize_weights(ops: H2Operators, topology: ClusterTopology, mode: str = "rigorous",
                       sample_size: int = 64, seed: int = 0) -> H2Operators:
    """h2.py:185-231 (rigorous mode) on the device, in place."""
    if mode not in ("rigorous", "sampled"):
        raise ValueError("mode must be 'rigorous' or 'sampled'")
    if mode == "sampled":
        # the row samples of every cluster's basis, drawn on the host in the
        # reference's loop order from its Generator(PCG64(seed)) (h2.py:200,
        # 250-262); the Gram products, SVDs and rotations run on the device
        rng = np.random.Generator(np.random.PCG64(seed))
        tree, bd = ops.tree, ops.block_dim
        rank = ops.rank
        ptr = np.zeros(tree.n_clusters + 1, dtype=np.int64)
        chunks = []
        order = [j for level in range(2, tree.depth + 1) for j in tree.levels[level]]
        sizes = {}
        for j in order:
            if not topology.interactions[j]:
                continue
            cl = tree.clusters[j]
            m = (cl.stop - cl.start) * bd if not cl.children else sum(rank[c] for c in cl.children)
            s = min(int(sample_size), m)
            if s < 1:
                raise ValueError("sample_size must be >= 1")
            idx = np.sort(rng.choice(m, size=s, replace=False)) if s < m else np.arange(m)
            sizes[j] = np.asarray(idx, dtype=np.int32)
        for j in range(tree.n_clusters):
            ptr[j + 1] = ptr[j] + (len(sizes[j]) if j in sizes else 0)
            if j in sizes:
                chunks.append(sizes[j])
        idx_all = np.ascontiguousarray(np.concatenate(chunks) if chunks else np.zeros(1, dtype=np.int32))
        N.check(N.lib().ifmm_h2_weights_sampled(ops._h, ptr.ctypes.data_as(C.c_void_p),
                                                idx_all.ctypes.data_as(C.c_void_p)))
        ops._weighted = True
        return ops
    N.check(N.lib().ifmm_h2_weights(ops._h))
    ops._weighted = True
    return ops
