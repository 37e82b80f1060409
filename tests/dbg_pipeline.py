import sys, numpy as np, json
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from conftest import load_golden
import paper_1508_01835_b200 as P
g = load_golden(sys.argv[1])
eps = float(g["eps"])
K = P.exp_kernel() if str(g["kernel"]) == "exp" else P.imq_kernel(float(g["h"]))
tree, _ = P.build_octree(g["points"], int(g["leaf"]))
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, K, int(g["n"]), epsilon=eps)
P.initialize_weights(ops, topo)
su = {c: ops.sigma_u[c].tolist() for c in list(ops.rank)[:50] if tree.clusters[c].level >= 2}
graph = P.assemble_extended_graph(ops)
f = P.factorize(graph, eps, sigma0=float(g["sigma0"]))
x = f.solve(g["b"])
out = {"ranks": [s.ranks for s in f.stats.levels], "err": float(np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])),
       "events": f.event_counts, "su": {int(k): v for k, v in su.items()}}
json.dump(out, open(f"gpurun_out/dbg_{sys.argv[1]}.json", "w"))
print(out["err"], out["events"])
