"""initialize_weights(mode="sampled") goldens (h2.py:197-225, 250-262) from
the UNMODIFIED reference.  Run in the build container:
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_sampled.py
Writes tests/golden/sampled/sampled.npz: per case the points, b, the sampled
weights of every cluster, h2_matvec(b), sigma0, per-level fill statistics and
x of the factorization built on the sampled weights."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_shim  # noqa: E402

ifmm = ref_shim.import_reference()
from scipy.spatial.distance import cdist  # noqa: E402

CASES = {
    # name: (N, dim, kernel, leaf, n, eps, sample_size, weight seed)
    "exp2d_n2048_s16": (2048, 2, "exp", 32, 4, 1e-8, 16, 0),
    "imq3d_n4096_s24": (4096, 3, "imq", 32, 3, 1e-6, 24, 7),
}
out = {}
for name, (N, dim, kern, leaf, n, eps, ss, wseed) in CASES.items():
    g = np.random.Generator(np.random.PCG64(11))
    pts = (np.column_stack([g.uniform(0, 1, size=(N, 2)), np.zeros(N)]) if dim == 2
           else g.uniform(0, 1, size=(N, 3)))
    b = np.random.Generator(np.random.PCG64(12)).standard_normal(N)
    h = N ** (-1.0 / 3.0)
    K = (ifmm.Kernel("exp", 1, {}, lambda P, Q: np.exp(-cdist(P, Q))) if kern == "exp"
         else ifmm.Kernel("imq", 1, {"h": h}, lambda P, Q: 1.0 / np.sqrt(cdist(P, Q) ** 2 + h * h)))
    tree, perm = ifmm.build_octree(pts, leaf)
    topo = ifmm.compute_topology(tree)
    ops = ifmm.chebyshev_operators(tree, topo, K, n, epsilon=eps)
    ifmm.initialize_weights(ops, topo, mode="sampled", sample_size=ss, seed=wseed)
    mv = ifmm.h2_matvec(ops, b)
    graph = ifmm.assemble_extended_graph(ops)
    s0 = ifmm.estimate_sigma0(graph, seed=0)
    fct = ifmm.factorize(graph, eps, seed=0, sigma0=s0)
    x = fct.solve(b)
    st = fct.stats
    ids = sorted(ops.sigma_u)
    pre = name + "__"
    out.update({pre + "points": pts, pre + "b": b, pre + "kernel": kern, pre + "h": h, pre + "leaf": leaf,
                pre + "n": n, pre + "eps": eps, pre + "sample_size": ss, pre + "wseed": wseed,
                pre + "sigma_ids": np.array(ids),
                pre + "sigma_ptr": np.cumsum([0] + [len(ops.sigma_u[c]) for c in ids]),
                pre + "sigma_u": np.concatenate([ops.sigma_u[c] for c in ids]),
                pre + "h2_matvec": mv, pre + "sigma0": s0, pre + "x": x, pre + "peak_edges": st.peak_edges,
                pre + "lv_compressed": np.array([s.compressed_pairs for s in st.levels]),
                pre + "lv_dropped": np.array([s.dropped_pairs for s in st.levels]),
                pre + "lv_ranksum": np.array([sum(s.ranks) for s in st.levels])})
    print(name, "depth", tree.depth, "levels", [(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks))
                                                 for s in st.levels])
os.makedirs(os.path.join(HERE, "sampled"), exist_ok=True)
np.savez_compressed(os.path.join(HERE, "sampled", "sampled.npz"), **out)
