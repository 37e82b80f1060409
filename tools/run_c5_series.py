"""c5 recipe (sphere, IMQ h = sqrt(4 pi / N), eps = 1e-3, IFMM-preconditioned
GMRES on the H2 matvec, tol 1e-10) at N = 2^12 ... through the CUDA path:
setup / factorize / GMRES device times and iteration counts (SURVEY.md 8d's
reduced-N series for the configuration whose full size needs 8 GPUs).

    python tools/run_c5_series.py [log2N ...] [--schedule wavefront]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1508_01835_b200 as P  # noqa: E402
from test_gpu_sphere import c5_problem  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
sched = "wavefront"
if "--schedule" in sys.argv:
    sched = sys.argv[sys.argv.index("--schedule") + 1]
    args = [a for a in args if a != sched]
logs = [int(a) for a in args] or [12, 14, 16, 17, 18]
free, _ = torch.cuda.mem_get_info()
os.environ.setdefault("IFMM_ARENA_GB", f"{max(0.5 * free, free - 22 * 2**30) / 2**30:.1f}")
SPH = os.path.join(ROOT, "tests", "golden", "sphere")
for lg in logs:
    N = 1 << lg
    pts, K, b = c5_problem(P, N)
    t0 = time.perf_counter()
    tree, _ = P.build_octree(pts, 64)
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, K, 4, epsilon=1e-3)
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    s0 = P.estimate_sigma0(graph, seed=0)
    fct = P.factorize(graph, 1e-3, seed=0, sigma0=s0, schedule=sched)
    torch.cuda.synchronize()
    t_fact = time.perf_counter() - t0
    db = torch.from_numpy(b).cuda()
    t0 = time.perf_counter()
    x, tr = P.gmres(lambda v: P.h2_matvec(ops, v), db, tol=1e-10, max_iters=500,
                    precond=fct.solve, side="right")
    torch.cuda.synchronize()
    t_gm = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(5):
        y = P.h2_matvec(ops, db)
    torch.cuda.synchronize()
    t_mv = (time.perf_counter() - t0) / 5
    r = float(torch.linalg.norm(P.h2_matvec(ops, x) - db) / torch.linalg.norm(db))
    ref = ""
    gp = os.path.join(SPH, f"c5_n{N}.npz")
    if os.path.exists(gp):
        g = np.load(gp)
        ref = (f" | reference its {int(g['iterations'])} t_fact {float(g['t_factorize']):.1f}s "
               f"t_gmres {float(g['t_gmres']):.1f}s")
    print(f"N=2^{lg}={N} depth {tree.depth} leaves {len(tree.leaves())} schedule {sched}: setup {t_setup:.2f}s "
          f"factorize {t_fact:.2f}s gmres {t_gm:.3f}s its {tr.iterations} converged {tr.converged} "
          f"h2 residual {r:.2e} matvec {t_mv * 1e3:.2f} ms solve/iter {1e3 * (t_gm / max(tr.iterations, 1) - t_mv):.2f} ms"
          f" compressed {[s.compressed_pairs for s in fct.stats.levels]}{ref}", flush=True)
    del fct, ops, graph, x
