"""Kernel-category and basis-union phase profile of one c3 factorize
(diagnostics: CUDA events per launch and clock64 phase counters perturb the
run; never bench numbers).

    python tools/profile_c3.py [reference|wavefront] [N]
"""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("IFMM_MEMTRACE", "1")
import paper_1508_01835_b200 as P  # noqa: E402
from paper_1508_01835_b200 import _native as NN  # noqa: E402
from oracle.ifmm_np import config_inputs  # noqa: E402  (seeded inputs only)

sch = sys.argv[1] if len(sys.argv) > 1 else "reference"
n_over = int(sys.argv[2]) if len(sys.argv) > 2 else None
inp = config_inputs("c3", n_over)
K = P.imq_kernel(inp["kernel"][1]["h"])
tree, _ = P.build_octree(inp["points"], inp["leaf"])
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, K, inp["n"], epsilon=inp["eps"])
P.initialize_weights(ops, topo)
graph = P.assemble_extended_graph(ops, consume=True)
s0 = P.estimate_sigma0(graph)
NN.ktime(1)
up = (C.c_ulonglong * 48)()
NN.lib().ifmm_union_profile(up, 1)
t0 = time.perf_counter()
f = P.factorize(graph, inp["eps"], sigma0=s0, schedule=sch)
tf = time.perf_counter() - t0
kt = NN.ktime(0)
NN.lib().ifmm_union_profile(up, 1)
u = list(up)
print(f"schedule {sch} factorize {tf:.2f}s launches {NN.launches()}")
print("kernel s (count):", {k: (round(v[0], 2), v[2]) for k, v in kt.items() if v[2]})
print("timings", {k: round(v, 2) for k, v in f.timings.items()})
print("levels", [(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in f.stats.levels])
ghz = 1.965e9


def cls(base, name):
    n = u[base + 6]
    if not n:
        return
    print(f"unions {name}: n={n} avg m={u[base + 7] / n:.0f} C={u[base + 8] / n:.0f} s={u[base + 5] / n:.0f} | "
          f"s total: aca {u[base + 0] / ghz:.2f} cholqr {u[base + 1] / ghz:.2f} jacobi+order {u[base + 3] / ghz:.2f} "
          f"out {u[base + 4] / ghz:.2f}")


cls(0, "all")
cls(16, "128<m<=400")
cls(25, ">400")
print("jacobi sweeps", u[11], "householder fallbacks", u[13], "giant jacobi sweeps", u[14])
