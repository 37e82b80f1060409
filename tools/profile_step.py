"""One setup + factorize + solve at a given N (c3 recipe), for ncu captures.

    python tools/profile_step.py 32768
Under ncu use -k / --launch-skip to select kernels; timings printed here are
never bench values."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_01835_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
g = np.random.Generator(np.random.PCG64(2))
pts = g.uniform(0.0, 1.0, size=(N, 3))
b = np.random.Generator(np.random.PCG64(3)).standard_normal(N)
tree, _ = P.build_octree(pts, 64)
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, P.imq_kernel(N ** (-1.0 / 3.0)), 4, epsilon=1e-6)
P.initialize_weights(ops, topo)
graph = P.assemble_extended_graph(ops)
s0 = P.estimate_sigma0(graph)
t0 = time.perf_counter()
f = P.factorize(graph, 1e-6, sigma0=s0)
x = f.solve(b)
print(f"N={N} factorize+solve {time.perf_counter() - t0:.2f}s")
y = P.h2_matvec(ops, b)
print("h2 residual %.3e" % (np.linalg.norm(P.h2_matvec(ops, x) - b) / np.linalg.norm(b)))
