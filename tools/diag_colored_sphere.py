import os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1508_01835_b200 as P
from test_gpu_sphere import c5_problem
for N in [int(a) for a in sys.argv[1:]] or (4096, 16384, 65536):
    pts, K, b = c5_problem(P, N)
    tree, _ = P.build_octree(pts, 64)
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, K, 4, epsilon=1e-3)
    P.initialize_weights(ops, topo)
    for sch in ("wavefront", "colored"):
        graph = P.assemble_extended_graph(ops)
        s0 = P.estimate_sigma0(graph, seed=0)
        fct = P.factorize(graph, 1e-3, seed=0, sigma0=s0, schedule=sch)
        db = torch.from_numpy(b).cuda()
        x1 = fct.solve(db); x2 = fct.solve(db)
        u = torch.from_numpy(np.random.default_rng(1).standard_normal(N)).cuda()
        lin = float(torch.linalg.norm(fct.solve(db + u) - x1 - fct.solve(u)) / torch.linalg.norm(x1))
        r = float(torch.linalg.norm(P.h2_matvec(ops, x1) - db) / torch.linalg.norm(db))
        x, tr = P.gmres(lambda v: P.h2_matvec(ops, v), db, tol=1e-10, max_iters=500, precond=fct.solve, side="right")
        rt = float(torch.linalg.norm(P.h2_matvec(ops, x) - db) / torch.linalg.norm(db))
        print(f"N={N} {sch}: depth {tree.depth} replay equal {bool(torch.equal(x1, x2))} linearity {lin:.1e} direct residual {r:.2e} "
              f"gmres its {tr.iterations} true residual {rt:.2e} levels {[(s.level, s.compressed_pairs, s.dropped_pairs) for s in fct.stats.levels]}", flush=True)
