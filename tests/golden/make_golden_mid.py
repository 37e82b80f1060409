"""Mid-size golden cases from the UNMODIFIED reference ``ifmm`` package.

Run in the build container (needs /root/reference; minutes of CPU each):
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_mid.py <case>
Writes ``tests/golden/mid/<case>.npz``.

These pin what the small cases of make_golden.py cannot: fill compression at
*merged* (non-leaf) levels of 3D inverse-multiquadric problems, and the full
c2 configuration.  Points are not stored (they are regenerated from the
seeded recipe); stored are the tree checksums, the H2
ranks, sigma0, per-level fill statistics, peak edges, the solution x of one
rhs, and the reference's per-pair decision log: for every call of
``redirect_fillin`` (factor.py:433) in call order, (level, cj, ck, r1, r2),
where r1/r2 are the ranks ``_compress_fill`` (factor.py:329) returned for
F_kj/F_jk (-1 = absent), and for every ``weighted_basis_union``
(lowrank.py:166) call (m, k_old, k_fill, min_rank, rank).  The log is
recorded by wrapping those two module functions; the reference's arithmetic
and rng stream are untouched.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref_shim  # noqa: E402

# name: (N, dim, point seed, kernel, leaf, n_cheb, eps)
CASES = {
    "imq3d_n32768": (32768, 3, 2, "imq", 64, 4, 1e-6),
    "imq3d_n32768_leaf8": (32768, 3, 2, "imq", 8, 4, 1e-6),
    "imq3d_n16384_leaf16": (16384, 3, 2, "imq", 16, 4, 1e-6),
    "c2_exp2d_n65536": (65536, 2, 1, "exp", 64, 6, 1e-10),
    # c3 itself (BASELINE configs[2]); about an hour of CPU
    "c3_imq3d_n262144": (262144, 3, 2, "imq", 64, 4, 1e-6),
    # the c3 recipe on a slab [0,1]^2 x [0,1/4]: depth 4 with 64-point leaves
    # (compression at the leaf level AND at merged levels, as in c3) at 1/4 of
    # c3's size
    "imq_slab_n65536": (65536, 3, 2, "imq", 64, 4, 1e-6),
}
SLAB = {"imq_slab_n65536": 0.25}


def inputs(N, dim, seed, kern, zscale=1.0):
    g = np.random.Generator(np.random.PCG64(seed))
    if dim == 2:
        pts = np.column_stack([g.uniform(0.0, 1.0, size=(N, 2)), np.zeros(N)])
    else:
        pts = g.uniform(0.0, 1.0, size=(N, 3))
        if zscale != 1.0:
            pts[:, 2] *= zscale
    gb = np.random.Generator(np.random.PCG64(seed + 1))
    b = gb.uniform(-1.0, 1.0, N) if dim == 2 else gb.standard_normal(N)
    return pts, b


def run(name, N, dim, seed, kern, leaf, n, eps):
    ifmm = ref_shim.import_reference()
    import ifmm.factor as F
    import ifmm.lowrank as L
    from scipy.spatial.distance import cdist
    zs = SLAB.get(name, 1.0)
    pts, b = inputs(N, dim, seed, kern, zs)
    if kern == "exp":
        h = 0.0
        block = lambda P, Q: np.exp(-cdist(P, Q))  # noqa: E731
    else:
        h = N ** (-1.0 / 3.0)
        block = lambda P, Q: 1.0 / np.sqrt(cdist(P, Q) ** 2 + h * h)  # noqa: E731
    K = ifmm.Kernel(kern, 1, {"h": h}, block)

    pair_log, union_log, cur = [], [], {"level": 0, "r": []}
    orig_compress, orig_redirect = F._compress_fill, F.redirect_fillin
    orig_union = F.weighted_basis_union
    orig_level = F.eliminate_level

    def compress(M, threshold, rng):
        fac = orig_compress(M, threshold, rng)
        cur["r"].append(fac.rank)
        return fac

    def redirect(graph, cj, ck, F_kj, F_jk, *a, **kw):
        cur["r"] = []
        out = orig_redirect(graph, cj, ck, F_kj, F_jk, *a, **kw)
        rr = list(cur["r"])
        r1 = rr.pop(0) if F_kj is not None else -1
        r2 = rr.pop(0) if F_jk is not None else -1
        pair_log.append((cur["level"], cj, ck, r1, r2))
        return out

    def union(old_basis, old_weights, fill_basis, fill_weights, thr, min_rank=0):
        bu = orig_union(old_basis, old_weights, fill_basis, fill_weights, thr, min_rank=min_rank)
        union_log.append((cur["level"], old_basis.shape[0], old_basis.shape[1],
                          fill_basis.shape[1], min_rank, bu.rank))
        return bu

    def level(graph, lv, *a, **kw):
        cur["level"] = lv
        return orig_level(graph, lv, *a, **kw)

    F._compress_fill, F.redirect_fillin = compress, redirect
    F.weighted_basis_union, F.eliminate_level = union, level
    t0 = time.perf_counter()
    tree, perm = ifmm.build_octree(pts, leaf)
    topo = ifmm.compute_topology(tree)
    ops = ifmm.chebyshev_operators(tree, topo, K, n, epsilon=eps)
    ifmm.initialize_weights(ops, topo)
    graph = ifmm.assemble_extended_graph(ops)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    sigma0 = ifmm.estimate_sigma0(graph, seed=0)
    fct = ifmm.factorize(graph, eps, seed=0, sigma0=sigma0)
    t_fact = time.perf_counter() - t0
    t0 = time.perf_counter()
    x = fct.solve(b)
    t_solve = time.perf_counter() - t0
    cl = tree.clusters
    lv = fct.stats.levels
    ranks = np.array([ops.rank.get(c, -1) for c in range(len(cl))], dtype=np.int32)
    out = dict(
        N=N, dim=dim, seed=seed, kernel=kern, h=h, leaf=leaf, n=n, eps=eps, zscale=zs,
        depth=tree.depth, n_clusters=len(cl),
        perm_checksum=np.int64((perm.astype(np.int64) * np.arange(1, N + 1)).sum()),
        cl_start=np.array([c.start for c in cl], dtype=np.int32),
        cl_level=np.array([c.level for c in cl], dtype=np.int8),
        n_neighbors=np.array([len(x) for x in topo.neighbors], dtype=np.int16),
        n_interactions=np.array([len(x) for x in topo.interactions], dtype=np.int16),
        ranks=ranks, sigma0=sigma0,
        lv_level=np.array([s.level for s in lv]),
        lv_compressed=np.array([s.compressed_pairs for s in lv]),
        lv_dropped=np.array([s.dropped_pairs for s in lv]),
        lv_added=np.array([s.added for s in lv]),
        lv_ranksum=np.array([sum(s.ranks) for s in lv]),
        lv_maxrank=np.array([s.max_rank for s in lv]),
        lv_forced=np.array([s.forced_rank_truncations for s in lv]),
        peak_edges=fct.stats.peak_edges, max_basis_rank=fct.stats.max_basis_rank,
        top_sizes=np.array(fct.top_sizes, dtype=np.int32),
        n_rebase=sum(1 for e in fct.events if e[0] == "rebase"),
        pairs=np.array(pair_log, dtype=np.int32).reshape(-1, 5),
        unions=np.array(union_log, dtype=np.int32).reshape(-1, 6),
        x=x, b=b,
        t_setup=t_setup, t_factorize=t_fact, t_solve=t_solve,
    )
    os.makedirs(os.path.join(HERE, "mid"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "mid", name + ".npz"), **out)
    print(name, "depth", tree.depth, "sigma0", sigma0, "compressed",
          out["lv_compressed"].tolist(), "dropped", out["lv_dropped"].tolist(),
          "t_fact %.1f s" % t_fact, flush=True)


if __name__ == "__main__":
    for name in sys.argv[1:] or CASES:
        run(name, *CASES[name])
