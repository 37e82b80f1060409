"""Solve timing (diagnostics): factorize a c3-recipe problem, then time the
first solve (direct launches) and graph replays on device-resident b, and
check that every solve is bitwise identical.

    python tools/time_solve.py [N] [schedule]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1508_01835_b200 as P  # noqa: E402
from paper_1508_01835_b200 import _native as NN  # noqa: E402
from oracle.ifmm_np import config_inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else None
sch = sys.argv[2] if len(sys.argv) > 2 else "wavefront"
inp = config_inputs("c3", n)
tree, _ = P.build_octree(inp["points"], inp["leaf"])
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, P.imq_kernel(inp["kernel"][1]["h"]), inp["n"], epsilon=inp["eps"])
P.initialize_weights(ops, topo)
g = P.assemble_extended_graph(ops, consume=True)
f = P.factorize(g, inp["eps"], sigma0=P.estimate_sigma0(g), schedule=sch)
print("top", sum(f.top_sizes), "events", f.event_counts, "IFMM_SOLVE_PARTS", os.environ.get("IFMM_SOLVE_PARTS"))
b = torch.from_numpy(inp["b"]).cuda()
NN.ktime(1)
xs, ts = [], []
for i in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = f.solve(b)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    xs.append(x.cpu().numpy())
kt = NN.ktime(0)
print("solve wall s:", [round(t, 4) for t in ts])
print("solve kernel:", kt["solve"], "GB/s (algorithmic, mean over launches):",
      kt["solve"][1] / max(kt["solve"][0], 1e-12) / 1e9)
print("bitwise identical:", all(np.array_equal(xs[0], x) for x in xs))
xh = f.solve(inp["b"])
print("host-b solve identical:", np.array_equal(xh, xs[0]))
