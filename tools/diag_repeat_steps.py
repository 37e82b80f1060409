"""Diagnostics: the same factorize+solve step several times in ONE process
(operators rebuilt and consumed per step, as bench.py does at N >= 500k), with
per-level wall times (IFMM_MEMTRACE) and arena statistics -- does a step slow
down once the arena has been through a full factorization?

    python tools/diag_repeat_steps.py c4 3"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IFMM_MEMTRACE", "1")
import bench  # noqa: E402
import paper_1508_01835_b200 as P  # noqa: E402
from paper_1508_01835_b200 import _native as NN  # noqa: E402
import torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
free, _ = torch.cuda.mem_get_info()
os.environ.setdefault("IFMM_ARENA_GB", f"{max(0.5 * free, free - 22 * 2**30) / 2**30:.1f}")
inp = bench.inputs(cfg)
K = P.exp_kernel() if inp["kern"] == "exp" else P.imq_kernel(inp["h"])
tree, _ = P.build_octree(inp["pts"], inp["leaf"])
topo = P.compute_topology(tree)
consume = inp["N"] >= 500000
ops = None
for r in range(reps):
    t0 = time.perf_counter()
    if ops is None or consume:
        ops = P.chebyshev_operators(tree, topo, K, inp["nc"], epsilon=inp["eps"])
        P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops, consume=consume)
    t1 = time.perf_counter()
    s0 = P.estimate_sigma0(graph)
    t2 = time.perf_counter()
    f = P.factorize(graph, inp["eps"], sigma0=s0, schedule="wavefront")
    t3 = time.perf_counter()
    x = f.solve(inp["b"])
    t4 = time.perf_counter()
    print(f"step {r}: setup {t1 - t0:.1f}s sigma0 {t2 - t1:.2f}s factorize {t3 - t2:.1f}s solve {t4 - t3:.2f}s "
          f"arena (in use, peak) GB {tuple(round(v / 2**30, 1) for v in NN.memory())}", flush=True)
    del f, x, graph
