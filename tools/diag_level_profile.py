"""Per-level kernel-category profile of one factorize at a BASELINE config.

    IFMM_MEMTRACE=1 python tools/diag_level_profile.py c4 [N]
Prints, after each level, arena usage and cumulative device time per kernel
category (CUDA events per launch -- diagnostics, not bench numbers)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("IFMM_MEMTRACE", "1")
import bench  # noqa: E402  (seeded inputs)
import paper_1508_01835_b200 as P  # noqa: E402
from paper_1508_01835_b200 import _native as NN  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n_override = int(sys.argv[2]) if len(sys.argv) > 2 else None
import torch  # noqa: E402
free, _ = torch.cuda.mem_get_info()
os.environ.setdefault("IFMM_ARENA_GB", f"{max(0.5 * free, free - 22 * 2**30) / 2**30:.1f}")
inp = bench.inputs(cfg, n_override)
K = P.exp_kernel() if inp["kern"] == "exp" else P.imq_kernel(inp["h"])
t0 = time.perf_counter()
tree, _ = P.build_octree(inp["pts"], inp["leaf"])
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, K, inp["nc"], epsilon=inp["eps"])
P.initialize_weights(ops, topo)
graph = P.assemble_extended_graph(ops, consume=inp["N"] >= 500000)
print(f"setup {time.perf_counter() - t0:.1f}s", flush=True)
t0 = time.perf_counter()
s0 = P.estimate_sigma0(graph)
print(f"sigma0 {s0:.6g} in {time.perf_counter() - t0:.2f}s", flush=True)
if os.environ.get("IFMM_DIAG_SIGMA0_ONLY"):
    sys.exit(0)
NN.ktime(1)
t0 = time.perf_counter()
f = P.factorize(graph, inp["eps"], sigma0=s0)
tf = time.perf_counter() - t0
t0 = time.perf_counter()
x = f.solve(inp["b"])
ts = time.perf_counter() - t0
kt = NN.ktime(0)
print(f"factorize {tf:.1f}s solve {ts:.2f}s unknowns/s {inp['N'] / (tf + ts):.1f}")
print({k: (round(v[0], 2), v[2]) for k, v in kt.items() if v[2]})
print("levels", [(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in f.stats.levels])
print("flops", f.flops)
print("phases", {k: round(v, 2) for k, v in NN.profile().items()})
if os.environ.get("IFMM_DIAG_RESIDUAL"):
    b = inp["b"]
    t0 = time.perf_counter()
    res = np.linalg.norm(P.exact_matvec(inp["pts"], K, x) - b) / np.linalg.norm(b)
    print(f"schedule {f.schedule} exact-matvec residual {res:.4e} ({time.perf_counter() - t0:.1f}s)")
