"""block_dim = 3 goldens (Rotne-Prager-Yamakawa mobility, kernels.py:59-91)
from the UNMODIFIED reference, run in the build container:
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_rpy.py
Writes tests/golden/rpy/rpy.npz (pipeline cases) and tests/golden/rpy/rpy_reports.json
(run_stokes reports).

Pipeline cases: points, b, H2 ranks, h2_matvec(b), sigma0, per-level fill
statistics, peak edges and the solution x of
    build_octree -> compute_topology -> chebyshev_operators(rpy) ->
    initialize_weights -> assemble_extended_graph -> factorize -> solve,
plus the dense kernel matrix checksum and A @ b (dense.dense_matrix)."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_shim  # noqa: E402

ifmm = ref_shim.import_reference()
from ifmm.dense import dense_matrix  # noqa: E402
from ifmm.experiments import RunConfig, run_stokes  # noqa: E402
from ifmm.kernels import cube_uniform, rpy_kernel, sphere_lattice  # noqa: E402

# name: (points, radius, leaf_target, n_cheb, eps_ops, eps_fact)
CASES = {
    # tests/test_factor.py:285-301 test_rpy_lossless
    "rpy_lossless": (cube_uniform(120, seed=8).points * 3.0, 0.05, 8, 2, 0.0, 1e-13),
    # a compressing case: 2x2x2 lattice of icospheres (42 vertices each), overlapping regime
    "rpy_lattice": (sphere_lattice(2, 2, 2, subdivision=1, spacing=4.0).points, 0.25, 20, 2, 1e-3, 1e-3),
    # depth 3 (512 leaves): fills are compressed at the leaf level and at the merged level
    "rpy_cube3000": (cube_uniform(3000, seed=3).points * 4.0, 0.1, 6, 2, 1e-4, 1e-4),
}
out = {}
for name, (pts, a, leaf, n, eps_ops, eps) in CASES.items():
    kern = rpy_kernel(a)
    N = len(pts)
    b = np.random.default_rng(9).standard_normal(3 * N)
    tree, perm = ifmm.build_octree(pts, leaf_target=leaf)
    topo = ifmm.compute_topology(tree)
    ops = ifmm.chebyshev_operators(tree, topo, kern, n, epsilon=eps_ops)
    ifmm.initialize_weights(ops, topo)
    mv = ifmm.h2_matvec(ops, b)
    A = dense_matrix(pts, kern)
    graph = ifmm.assemble_extended_graph(ops)
    s0 = ifmm.estimate_sigma0(graph, seed=0)
    fct = ifmm.factorize(graph, eps, seed=0, sigma0=s0)
    x = fct.solve(b)
    st = fct.stats
    pre = name + "__"
    out.update({pre + "points": pts, pre + "b": b, pre + "radius": a, pre + "leaf": leaf, pre + "n": n,
                pre + "eps_ops": eps_ops, pre + "eps": eps, pre + "depth": tree.depth,
                pre + "ranks": np.array([ops.rank.get(c, -1) for c in range(tree.n_clusters)]),
                pre + "h2_matvec": mv, pre + "dense_matvec": A @ b,
                pre + "dense_fro": np.linalg.norm(A), pre + "dense_corner": A[:6, :9].copy(),
                pre + "sigma0": s0, pre + "x": x, pre + "peak_edges": st.peak_edges,
                pre + "lv_level": np.array([s.level for s in st.levels]),
                pre + "lv_compressed": np.array([s.compressed_pairs for s in st.levels]),
                pre + "lv_dropped": np.array([s.dropped_pairs for s in st.levels]),
                pre + "lv_ranksum": np.array([sum(s.ranks) for s in st.levels]),
                pre + "top_sizes": np.array(fct.top_sizes)})
    print(name, "N", N, "depth", tree.depth, "ranks sum", sum(ops.rank.values()), "levels",
          [(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in st.levels],
          "resid", np.linalg.norm(A @ x - b) / np.linalg.norm(b))
os.makedirs(os.path.join(HERE, "rpy"), exist_ok=True)
np.savez_compressed(os.path.join(HERE, "rpy", "rpy.npz"), **out)

reports = {}
BASE = dict(kernel="rpy", n_points=0, distribution="lattice", cheb_nodes=2, epsilon=1e-3,
            leaf_target=20, seed=0, mode="gmres", precond="ifmm", lattice_shape=(2, 2, 1),
            subdivision=1, gmres_tol=1e-8)
for name, kw in {"stokes_lattice_ifmm": dict(BASE), "stokes_lattice_blockdiag": dict(BASE, precond="blockdiag", blockdiag_size=126),
                 "stokes_shells_ifmm": dict(BASE, distribution="shells", shell_subdivisions=(1, 2), shell_radii=(1.0, 2.0))}.items():
    try:
        cfg = RunConfig(**kw)
    except TypeError as e:
        print("skip", name, e)
        continue
    rep = run_stokes(cfg).to_dict()
    reports[name] = {"kwargs": {k: (list(v) if isinstance(v, tuple) else v) for k, v in kw.items()},
                     "report": rep}
    print(name, rep["errors"], (rep["iteration"] or {}).get("iterations"))
json.dump(reports, open(os.path.join(HERE, "rpy", "rpy_reports.json"), "w"), indent=1)
