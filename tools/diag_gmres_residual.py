"""Diagnostics: true vs recurrence residual of the IFMM-preconditioned GMRES
on the c5 recipe at reduced N, and the linearity defect of the replay solve.

    python tools/diag_gmres_residual.py [N]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1508_01835_b200 as P  # noqa: E402
from test_gpu_sphere import c5_problem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
pts, K, b = c5_problem(P, N)
tree, _ = P.build_octree(pts, 64)
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, K, 4, epsilon=1e-3)
P.initialize_weights(ops, topo)
graph = P.assemble_extended_graph(ops)
fct = P.factorize(graph, 1e-3, seed=0, schedule="wavefront")
db = torch.from_numpy(b).cuda()
nb = float(torch.linalg.norm(db))
rng = np.random.default_rng(0)
u = torch.from_numpy(rng.standard_normal(N)).cuda()
v = torch.from_numpy(rng.standard_normal(N)).cuda()
su, sv, suv = fct.solve(u), fct.solve(v), fct.solve(u + v)
print("solve linearity defect |S(u+v) - S(u) - S(v)| / |S(u+v)| = %.2e" %
      float(torch.linalg.norm(suv - su - sv) / torch.linalg.norm(suv)))
print("|S(u)| / |u| = %.2e" % float(torch.linalg.norm(su) / torch.linalg.norm(u)))
for tol in (1e-6, 1e-8, 1e-10, 1e-12):
    x, tr = P.gmres(lambda w: P.h2_matvec(ops, w), db, tol=tol, max_iters=500, precond=fct.solve,
                    side="right")
    r = float(torch.linalg.norm(P.h2_matvec(ops, x) - db)) / nb
    print(f"tol {tol:g}: its {tr.iterations} recurrence {tr.residual_history[-1]:.2e} true {r:.2e}")
x, tr = P.gmres(lambda w: P.h2_matvec(ops, w), b, tol=1e-10, max_iters=500, precond=fct.solve, side="right")
print("numpy-b path: its", tr.iterations, "true %.2e" % (np.linalg.norm(P.h2_matvec(ops, x) - b) / nb))
