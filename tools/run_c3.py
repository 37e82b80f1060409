"""c3 (3D N=262,144 IMQ, eps=1e-6) through the CUDA path with a chosen
schedule; prints per-level fill statistics against the reference-semantics
golden (tests/golden/large/c3_stats.json) and |x - x_ref|.

    IFMM_TRACE=gpurun_out/c3_trace.txt python tools/run_c3.py [reference|wavefront]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1508_01835_b200 as P  # noqa: E402
from oracle.ifmm_np import config_inputs  # noqa: E402  (seeded inputs only)

sch = sys.argv[1] if len(sys.argv) > 1 else "reference"
G = os.path.join(ROOT, "tests", "golden", "large")
st = json.load(open(os.path.join(G, "c3_stats.json")))
inp = config_inputs("c3")
t0 = time.perf_counter()
tree, _ = P.build_octree(inp["points"], inp["leaf"])
topo = P.compute_topology(tree)
K = P.imq_kernel(inp["kernel"][1]["h"])
ops = P.chebyshev_operators(tree, topo, K, inp["n"], epsilon=inp["eps"])
P.initialize_weights(ops, topo)
graph = P.assemble_extended_graph(ops, consume=True)
print("setup %.1f s, ranks sum %d (ref %d)" % (time.perf_counter() - t0, sum(ops.rank.values()),
                                               st["ranks_sum"]), flush=True)
t0 = time.perf_counter()
if sch == "morton_devrng":  # diagnostics: Morton one-at-a-time order with the device generator
    from paper_1508_01835_b200 import _native as NN
    from paper_1508_01835_b200.factor import IFMMFactorization
    h = NN.check_handle(NN.lib().ifmm_factorize(graph._h, float(inp["eps"]), float(st["sigma0"]), 4))
    graph.consumed = True
    fct = IFMMFactorization(graph, h, inp["eps"], st["sigma0"], 0.0, 0.0)
    fct.schedule = sch
else:
    fct = P.factorize(graph, inp["eps"], seed=int(os.environ.get("IFMM_C3_SEED", "0")), sigma0=st["sigma0"],
                      schedule=sch)
tf = time.perf_counter() - t0
print("schedule", sch, "factorize %.2f s" % tf, "rsvd", fct.rsvd,
      {k: round(v, 2) for k, v in fct.timings.items()}, flush=True)
for s, r in zip(fct.stats.levels, st["levels"]):
    print(f"level {s.level}: ours comp {s.compressed_pairs} drop {s.dropped_pairs} add {s.added} "
          f"Σr {sum(s.ranks)} | ref {r}")
print("peak edges", fct.stats.peak_edges, "ref", st["peak_edges"])
x = fct.solve(inp["b"])
xr = np.load(os.path.join(G, "c3_x.npy"))
print("|x - x_ref|/|x_ref| = %.3e" % (np.linalg.norm(x - xr) / np.linalg.norm(xr)))
b = inp["b"]
res = np.linalg.norm(P.exact_matvec(inp["points"], K, x) - b) / np.linalg.norm(b)
print("exact residual %.4e" % res)
np.save(os.path.join(ROOT, "gpurun_out", f"c3_x_{sch}.npy"), x)
