"""c3 parity triage: x vs the reference-semantics oracle fixture for
fill-truncation / ordering variants (IFMM_FILL_DELTA, EXACT=1)."""
import json, os, sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import GOLDEN
import paper_1508_01835_b200 as P
from oracle.ifmm_np import config_inputs
st = json.load(open(os.path.join(GOLDEN, "large", "c3_stats.json")))
x_ref = np.load(os.path.join(GOLDEN, "large", "c3_x.npy"))
inp = config_inputs("c3")
tree, _ = P.build_octree(inp["points"], inp["leaf"])
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, P.imq_kernel(inp["kernel"][1]["h"]), 4, epsilon=1e-6)
P.initialize_weights(ops, topo)
gr = P.assemble_extended_graph(ops)
f = P.factorize(gr, 1e-6, sigma0=st["sigma0"], exact_order=os.environ.get("EXACT") == "1")
x = f.solve(inp["b"])
y = P.h2_matvec(ops, x)
print(sys.argv[1:], "rel_x", np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref),
      "res_h2", np.linalg.norm(y - inp["b"]) / np.linalg.norm(inp["b"]),
      "ref_res_h2", np.linalg.norm(P.h2_matvec(ops, x_ref) - inp["b"]) / np.linalg.norm(inp["b"]),
      [(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in f.stats.levels], flush=True)
