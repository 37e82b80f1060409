"""c5 recipe (BASELINE configs[4]) at reduced N from the UNMODIFIED reference:
points on the unit sphere (kernels.sphere_surface(N, seed=4)), inverse
multiquadric with h = sqrt(4 pi / N), leaves <= 64, 4^3 Chebyshev nodes,
eps = 1e-3; IFMM as right preconditioner for GMRES on the H2 matvec to a
relative residual of 1e-10.  Records GMRES iteration counts
and residual histories.  Run in the build container:
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_sphere.py 16384
Writes tests/golden/sphere/c5_n<N>.npz."""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_shim  # noqa: E402


def run(N):
    ifmm = ref_shim.import_reference()
    from scipy.spatial.distance import cdist
    pts = ifmm.sphere_surface(N, 4).points
    h = float(np.sqrt(4.0 * np.pi / N))
    K = ifmm.Kernel("imq", 1, {"h": h}, lambda P, Q: 1.0 / np.sqrt(cdist(P, Q) ** 2 + h * h))
    b = np.random.Generator(np.random.PCG64(5)).standard_normal(N)
    eps = 1e-3
    t0 = time.perf_counter()
    tree, _ = ifmm.build_octree(pts, 64)
    topo = ifmm.compute_topology(tree)
    ops = ifmm.chebyshev_operators(tree, topo, K, 4, epsilon=eps)
    ifmm.initialize_weights(ops, topo)
    graph = ifmm.assemble_extended_graph(ops)
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    s0 = ifmm.estimate_sigma0(graph, seed=0)
    fct = ifmm.factorize(graph, eps, seed=0, sigma0=s0)
    t_fact = time.perf_counter() - t0
    t0 = time.perf_counter()
    x, tr = ifmm.gmres(lambda v: ifmm.h2_matvec(ops, v), b, tol=1e-10, max_iters=500,
                       precond=fct.solve, side="right")
    t_gmres = time.perf_counter() - t0
    x0, tr0 = ifmm.gmres(lambda v: ifmm.h2_matvec(ops, v), b, tol=1e-10, max_iters=500)
    os.makedirs(os.path.join(HERE, "sphere"), exist_ok=True)
    np.savez_compressed(os.path.join(HERE, "sphere", f"c5_n{N}.npz"), N=N, h=h, eps=eps,
                        depth=tree.depth, sigma0=s0, iterations=tr.iterations,
                        converged=tr.converged, history=np.array(tr.residual_history),
                        iterations_none=tr0.iterations, history_none=np.array(tr0.residual_history),
                        x=x, lv_compressed=np.array([s.compressed_pairs for s in fct.stats.levels]),
                        t_setup=t_setup, t_factorize=t_fact, t_gmres=t_gmres)
    print(N, "depth", tree.depth, "its", tr.iterations, "(none:", tr0.iterations, ")",
          "t_fact %.1f t_gmres %.1f" % (t_fact, t_gmres), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        run(int(a))
