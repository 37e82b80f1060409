"""Host-side phase profile of one c3 factorize (IFMM_PROFILE=2: host time per
engine phase, no synchronisation; IFMM_PROFILE=1: stream-synchronised phase
times).  Diagnostics only.

    IFMM_PROFILE=2 python tools/profile_phases.py [reference|wavefront] [N]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1508_01835_b200 as P  # noqa: E402
from paper_1508_01835_b200 import _native as NN  # noqa: E402
from oracle.ifmm_np import config_inputs  # noqa: E402

sch = sys.argv[1] if len(sys.argv) > 1 else "reference"
inp = config_inputs("c3", int(sys.argv[2]) if len(sys.argv) > 2 else None)
tree, _ = P.build_octree(inp["points"], inp["leaf"])
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, P.imq_kernel(inp["kernel"][1]["h"]), inp["n"], epsilon=inp["eps"])
P.initialize_weights(ops, topo)
graph = P.assemble_extended_graph(ops, consume=True)
s0 = P.estimate_sigma0(graph)
t0 = time.perf_counter()
f = P.factorize(graph, inp["eps"], sigma0=s0, schedule=sch)
print(f"PROFILE={os.environ.get('IFMM_PROFILE')} schedule {sch} factorize {time.perf_counter() - t0:.2f}s")
print({k: round(v, 2) for k, v in NN.profile().items()})
