"""c4 (BASELINE configs[3], the headline: 3D N = 1,048,576 IMQ, leaves <= 64,
4^3 Chebyshev nodes, eps = 1e-6) structure golden from the UNMODIFIED
reference.  The reference cannot factorize c4 in this container (SURVEY.md
8d: >= 6 h, tens of GB), so this pins what it can produce in minutes:

  * build_octree / compute_topology (tree.py:107-239): depth, permutation
    checksum, per-cluster point ranges checksum, neighbour / interaction
    list sizes and an order-sensitive checksum of the lists;
  * the H2 ranks of every cluster from the reference's own leaf and transfer
    reductions (h2.py:121-150 -- the first two loops of chebyshev_operators,
    executed here statement for statement with the reference's _interp_matrix,
    _grid and _kron_bd; the M2L / P2P loops that follow do not change ranks).

Run in the build container:
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_c4.py
Writes tests/golden/large/c4_structure.npz."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_shim  # noqa: E402


def list_checksum(lists):
    """Order-sensitive checksum of a list of int lists (mod 2^61 - 1)."""
    M = (1 << 61) - 1
    acc = 0
    for i, l in enumerate(lists):
        a = np.asarray(l, dtype=np.int64)
        if len(a):
            acc = (acc + (i + 1) * int(((a + 1) * np.arange(1, len(a) + 1)).sum() % M)) % M
    return acc


def main():
    ifmm = ref_shim.import_reference()
    from ifmm import h2 as H
    N, seed, leaf, n, eps = 1048576, 3, 64, 4, 1e-6
    pts = np.random.Generator(np.random.PCG64(seed)).uniform(0.0, 1.0, size=(N, 3))
    t0 = time.perf_counter()
    tree, perm = ifmm.build_octree(pts, leaf)
    topo = ifmm.compute_topology(tree)
    t_tree = time.perf_counter() - t0
    cl = tree.clusters
    floor = max(eps, 1e-13)

    def _reduce(M):  # h2.py:124-127
        W, s, Zt = np.linalg.svd(M, full_matrices=False)
        k = max(1, int(np.sum(s > floor * s[0])))
        return W[:, :k], s[:k, None] * Zt[:k]

    rank, reduce_map, grids = {}, {}, {}
    t0 = time.perf_counter()
    for cid in tree.leaves():  # h2.py:129-135
        c = cl[cid]
        Pm = H._interp_matrix(tree.points[c.start:c.stop], c.center, c.half_width, n)
        basis, G = _reduce(H._kron_bd(Pm, 1))
        reduce_map[cid] = G
        rank[cid] = basis.shape[1]
    for level in range(tree.depth - 1, 1, -1):  # h2.py:137-150
        for pid in tree.levels[level]:
            p = cl[pid]
            blocks = []
            for c in p.children:
                child_grid = grids.setdefault(c, H._grid(cl[c].center, cl[c].half_width, n))
                T = H._interp_matrix(child_grid, p.center, p.half_width, n)
                blocks.append(reduce_map[c] @ H._kron_bd(T, 1))
            basis, G = _reduce(np.vstack(blocks))
            reduce_map[pid] = G
            rank[pid] = basis.shape[1]
    t_rank = time.perf_counter() - t0
    nc = tree.n_clusters
    out = os.path.join(HERE, "large", "c4_structure.npz")
    np.savez_compressed(
        out, N=N, seed=seed, leaf=leaf, n=n, eps=eps, depth=tree.depth, n_clusters=nc,
        perm_checksum=int((np.asarray(perm, dtype=np.int64) * np.arange(1, N + 1)).sum()),
        range_checksum=int(sum((i + 1) * (c.start + 3 * c.stop) for i, c in enumerate(cl)) % ((1 << 61) - 1)),
        n_neighbors=np.array([len(x) for x in topo.neighbors], dtype=np.int16),
        n_interactions=np.array([len(x) for x in topo.interactions], dtype=np.int16),
        neighbors_checksum=list_checksum(topo.neighbors),
        interactions_checksum=list_checksum(topo.interactions),
        ranks=np.array([rank.get(c, -1) for c in range(nc)], dtype=np.int16),
        t_tree=t_tree, t_rank=t_rank)
    print("c4 structure: depth", tree.depth, "clusters", nc, "rank sum", sum(rank.values()),
          "tree+topology %.1f s, reductions %.1f s" % (t_tree, t_rank), "->", out)


if __name__ == "__main__":
    main()
