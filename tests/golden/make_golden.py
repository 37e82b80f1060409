"""Generate golden vectors from the UNMODIFIED reference ``ifmm`` package.

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py
Writes ``tests/golden/<case>.npz``.  Each case records, for a seeded input,
the reference's tree (perm, levels, cluster ranges), topology (CSR
neighbour / interaction lists), H2 ranks and basis weights, sigma0, the
per-level fill statistics of ``factorize`` and the solution x of one rhs,
plus the H2 matvec of that rhs.  The numpy restatement (oracle/ifmm_np.py)
is pinned against these in tests/test_oracle_golden.py.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref_shim  # noqa: E402

ifmm = ref_shim.import_reference()

# name: (N, dim, point seed, kernel, leaf, n_cheb, eps)
CASES = {
    "exp2d_n1024": (1024, 2, 0, "exp", 32, 4, 1e-8),
    "c1_exp2d_n4096": (4096, 2, 0, "exp", 32, 4, 1e-8),
    "imq3d_n2048": (2048, 3, 2, "imq", 64, 4, 1e-6),
    "imq3d_n4096_leaf32": (4096, 3, 2, "imq", 32, 4, 1e-6),
    "exp2d_n2048_n6": (2048, 2, 1, "exp", 64, 6, 1e-10),
    "imq3d_n1500_lossless": (1500, 3, 7, "imq", 24, 3, 1e-13),
}


def inputs(N, dim, seed, kern):
    g = np.random.Generator(np.random.PCG64(seed))
    if dim == 2:
        pts = np.column_stack([g.uniform(0.0, 1.0, size=(N, 2)), np.zeros(N)])
    else:
        pts = g.uniform(0.0, 1.0, size=(N, 3))
    gb = np.random.Generator(np.random.PCG64(seed + 1))
    b = gb.uniform(-1.0, 1.0, N) if dim == 2 else gb.standard_normal(N)
    from scipy.spatial.distance import cdist
    if kern == "exp":
        block = lambda P, Q: np.exp(-cdist(P, Q))  # noqa: E731
        h = 0.0
    else:
        h = N ** (-1.0 / 3.0)
        block = lambda P, Q: 1.0 / np.sqrt(cdist(P, Q) ** 2 + h * h)  # noqa: E731
    return pts, b, ifmm.Kernel(kern, 1, {"h": h}, block), h


def csr(lists):
    ptr = np.zeros(len(lists) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(x) for x in lists])
    idx = np.array([v for x in lists for v in x], dtype=np.int64)
    return ptr, idx


def run(name, N, dim, seed, kern, leaf, n, eps):
    pts, b, K, h = inputs(N, dim, seed, kern)
    tree, perm = ifmm.build_octree(pts, leaf)
    topo = ifmm.compute_topology(tree)
    ops = ifmm.chebyshev_operators(tree, topo, K, n, epsilon=eps)
    ifmm.initialize_weights(ops, topo)
    y_h2 = ifmm.h2_matvec(ops, b)
    graph = ifmm.assemble_extended_graph(ops)
    sigma0 = ifmm.estimate_sigma0(graph, seed=0)
    fct = ifmm.factorize(graph, eps, seed=0, sigma0=sigma0)
    x = fct.solve(b)
    cl = tree.clusters
    nptr, nidx = csr(topo.neighbors)
    iptr, iidx = csr(topo.interactions)
    lv = fct.stats.levels
    ranks = np.array([ops.rank.get(c, -1) for c in range(len(cl))])
    su_keys = sorted(ops.sigma_u)
    su = [ops.sigma_u[c] for c in su_keys]
    out = dict(
        N=N, dim=dim, seed=seed, kernel=kern, h=h, leaf=leaf, n=n, eps=eps,
        points=pts, b=b, perm=perm, depth=tree.depth,
        cl_level=np.array([c.level for c in cl]),
        cl_start=np.array([c.start for c in cl]),
        cl_stop=np.array([c.stop for c in cl]),
        cl_parent=np.array([-1 if c.parent is None else c.parent for c in cl]),
        cl_cell=np.array([c.cell for c in cl]),
        nbr_ptr=nptr, nbr_idx=nidx, int_ptr=iptr, int_idx=iidx,
        ranks=ranks,
        su_keys=np.array(su_keys), su_ptr=csr(su)[0],
        su_val=np.concatenate(su) if su else np.zeros(0),
        sigma0=sigma0,
        lv_level=np.array([s.level for s in lv]),
        lv_compressed=np.array([s.compressed_pairs for s in lv]),
        lv_dropped=np.array([s.dropped_pairs for s in lv]),
        lv_added=np.array([s.added for s in lv]),
        lv_ranksum=np.array([sum(s.ranks) for s in lv]),
        lv_maxrank=np.array([s.max_rank for s in lv]),
        peak_edges=fct.stats.peak_edges,
        max_basis_rank=fct.stats.max_basis_rank,
        top_sizes=np.array(fct.top_sizes),
        n_rebase=sum(1 for e in fct.events if e[0] == "rebase"),
        x=x, y_h2=y_h2,
    )
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "depth", tree.depth, "sigma0", sigma0, "compressed",
          out["lv_compressed"].tolist(), "dropped", out["lv_dropped"].tolist())


def kat_lowrank():
    """Known-answer vectors for ACA / basis union / truncated SVD."""
    rng = np.random.Generator(np.random.PCG64(11))
    A = rng.standard_normal((40, 6)) @ np.diag(10.0 ** -np.arange(6)) @ rng.standard_normal((6, 30))
    fa = ifmm.aca_svd(A, 1e-3)
    B, _ = np.linalg.qr(rng.standard_normal((50, 12)))
    w = np.sort(rng.uniform(0.01, 3.0, 12))[::-1]
    F, _ = np.linalg.qr(rng.standard_normal((50, 3)))
    wf = np.array([0.5, 0.05, 0.002])
    bu = ifmm.weighted_basis_union(B, w, F, wf, 1e-2)
    ts = ifmm.truncated_svd(A, 1e-2)
    np.savez_compressed(os.path.join(HERE, "kat_lowrank.npz"), A=A, aca_s=fa.sigma,
                        aca_U=fa.U, aca_V=fa.V, B=B, w=w, F=F, wf=wf,
                        bu_basis=bu.new_basis, bu_w=bu.new_weights,
                        bu_old=bu.old_map, bu_fill=bu.fillin_map, ts_s=ts.sigma)


if __name__ == "__main__":
    kat_lowrank()
    only = sys.argv[1:]
    for name, spec in CASES.items():
        if only and name not in only:
            continue
        run(name, *spec)
