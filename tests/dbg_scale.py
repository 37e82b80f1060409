"""Scale probe: time each stage of the pipeline at a given N (c3/c4 recipe)."""
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1508_01835_b200 as P
from paper_1508_01835_b200 import _native as NN
N = int(sys.argv[1]); leaf = int(sys.argv[2]) if len(sys.argv) > 2 else 64
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 2
g = np.random.Generator(np.random.PCG64(seed))
pts = g.uniform(0.0, 1.0, size=(N, 3))
b = np.random.Generator(np.random.PCG64(seed + 1)).standard_normal(N)
h = N ** (-1.0 / 3.0)
t = time.perf_counter(); tree, _ = P.build_octree(pts, leaf); topo = P.compute_topology(tree)
print(f"N={N} depth={tree.depth} leaves={len(tree.leaves())} tree {time.perf_counter()-t:.2f}s", flush=True)
t = time.perf_counter(); ops = P.chebyshev_operators(tree, topo, P.imq_kernel(h), 4, epsilon=1e-6)
print(f"h2 build {time.perf_counter()-t:.2f}s max rank {ops.max_rank()}", flush=True)
t = time.perf_counter(); P.initialize_weights(ops, topo); print(f"weights {time.perf_counter()-t:.2f}s", flush=True)
t = time.perf_counter(); gr = P.assemble_extended_graph(ops); print(f"graph {time.perf_counter()-t:.2f}s dim {gr.dim} edges {gr.num_edges}", flush=True)
t = time.perf_counter(); s0 = P.estimate_sigma0(gr); print(f"sigma0 {s0:.10g} {time.perf_counter()-t:.2f}s", flush=True)
import os
if os.environ.get("KT") == "1": NN.ktime(1)
l0 = NN.launches()
t = time.perf_counter(); f = P.factorize(gr, 1e-6, sigma0=s0); tf = time.perf_counter() - t
print("launches", NN.launches() - l0)
import ctypes as CC
up = (CC.c_ulonglong * 48)()
NN.lib().ifmm_union_profile(up, 1)
u = list(up); n_ = max(u[6], 1)
print("union prof: per-union Mcycles aca %.3f qr %.3f q %.3f jac %.3f out %.3f | steps %.1f m %.1f C %.1f smem %d/%d sweeps/union %.2f" % (
    u[0]/n_/1e6, u[1]/n_/1e6, u[2]/n_/1e6, u[3]/n_/1e6, u[4]/n_/1e6, u[5]/n_, u[7]/n_, u[8]/n_, u[9], u[6], u[10]/n_))
print("union core jacobi: sweeps/union %.2f  Mcycles/union %.3f" % (u[11]/n_, u[12]/n_/1e6))
for lo, hi, b in ((128, 400, 16), (400, 1 << 30, 25)):
    nb = max(u[b + 6], 1)
    print("unions %d < m <= %s: n %d  Mcycles aca %.3f cholqr %.3f sweeps %.2f jac %.3f out %.3f | steps %.1f m %.1f C %.1f" % (
        lo, hi if hi < 1 << 30 else "inf", u[b + 6], u[b]/nb/1e6, u[b + 1]/nb/1e6, u[b + 2]/nb, u[b + 3]/nb/1e6,
        u[b + 4]/nb/1e6, u[b + 5]/nb, u[b + 7]/nb, u[b + 8]/nb))
print("householder fallbacks", u[13])
nq = max(u[39], 1)
print("large-union CholeskyQR Mcycles: scale+gram1+chol1 %.3f trsm1+park %.3f gram2 %.3f chol2 %.3f trsm2+trmul %.3f" % (
    u[38]/nq/1e6, u[34]/nq/1e6, u[35]/nq/1e6, u[36]/nq/1e6, u[37]/nq/1e6))
if os.environ.get("KT") == "1":
    kt = NN.ktime(0); print("ktime", {k: (round(v[0], 3), v[2]) for k, v in kt.items() if v[2]}, "sum", round(sum(v[0] for v in kt.values()), 3))
print(f"factorize {tf:.2f}s stats peak_edges={f.stats.peak_edges} events={f.event_counts} flops={f.flops}", flush=True)
print("profile", {k: round(v, 3) for k, v in NN.profile().items()}, flush=True)
print("levels", [(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in f.stats.levels], flush=True)
t = time.perf_counter(); x = f.solve(b); ts = time.perf_counter() - t
t = time.perf_counter(); x = f.solve(b); ts2 = time.perf_counter() - t
y = P.h2_matvec(ops, x)
print(f"solve {ts:.3f}s / {ts2:.3f}s  rel res (H2) {np.linalg.norm(y-b)/np.linalg.norm(b):.3e}  unknowns/s {N/(tf+ts2):.1f}")
print("arena in_use/peak GB", [v / 2**30 for v in NN.memory()])
