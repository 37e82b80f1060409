"""Small end-to-end factorize + solve exercising every kernel family, with the
giant-union cooperative kernels forced on (IFMM_GIANT=20) for fault / race
hunting: IFMM_DEBUG_SYNC=1 synchronises and checks after every launch, and
the printed solution hashes must agree between runs (a race shows up as
nondeterminism).  (compute-sanitizer is not available on the GPU pool.)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_01835_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
g = np.random.Generator(np.random.PCG64(2))
pts = g.uniform(0.0, 1.0, size=(N, 3))
b = np.random.Generator(np.random.PCG64(3)).standard_normal(N)
K = P.imq_kernel(N ** (-1.0 / 3.0))
tree, _ = P.build_octree(pts, 24)
topo = P.compute_topology(tree)
ops = P.chebyshev_operators(tree, topo, K, 3, epsilon=1e-6)
P.initialize_weights(ops, topo)
for sch in ("reference", "wavefront"):
    graph = P.assemble_extended_graph(ops)
    f = P.factorize(graph, 1e-6, sigma0=P.estimate_sigma0(graph), schedule=sch)
    x = f.solve(b)
    x2 = f.solve(b)
    y = P.h2_matvec(ops, x)
    import hashlib
    print("XHASH", sch, hashlib.sha256(x.tobytes()).hexdigest())
    print(sch, "depth", tree.depth, "levels", [(s.level, s.compressed_pairs) for s in f.stats.levels],
          "h2 residual %.3e" % (np.linalg.norm(y - b) / np.linalg.norm(b)), "replay equal", np.array_equal(x, x2))
