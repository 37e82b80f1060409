"""Micro-benchmark: cycles per Jacobi round for s x s graded matrices.

variant 0: generic cta_jacobi (fill SVD / weights); variant 1: the union-core
layout Z = [A; V] with one-pass rounds (cta_jacobi_z)."""
import ctypes as C
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_01835_b200 import _native as N
N.ctx()
for s in (16, 40, 86, 110):
    rng = np.random.default_rng(s)
    U, _ = np.linalg.qr(rng.standard_normal((s, s)))
    V, _ = np.linalg.qr(rng.standard_normal((s, s)))
    A = (U * 10.0 ** -np.linspace(0, 10, s)) @ V.T
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
    for var in (0, 1):
        for thr in (256, 512):
            out = (C.c_ulonglong * 2)()
            N.check(N.lib().ifmm_dev_jacobi_bench(N.ctx(), s, C.c_void_p(dA.data_ptr()), 5,
                                                  thr | (var << 16), out))
            cyc, sw = out[0] / 5, out[1] / 5
            rounds = sw * (s + (s & 1) - 1)
            print(f"variant={var} s={s:4d} threads={thr:4d} sweeps={sw:5.1f} cycles={cyc:10.0f} "
                  f"cycles/round={cyc / max(rounds, 1):8.0f}", flush=True)

# real union cores (transposed, as the kernel sees them) from oracle unions of
# the c3 recipe at N=32768 (tools/micro/union_cores.npz)
cores = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "micro", "union_cores.npz"))
for name in sorted(cores.files):
    A = cores[name]
    s = A.shape[0]
    dA = torch.from_numpy(np.asfortranarray(A).ravel(order="F").copy()).cuda()
    out = (C.c_ulonglong * 2)()
    N.check(N.lib().ifmm_dev_jacobi_bench(N.ctx(), s, C.c_void_p(dA.data_ptr()), 5, 512 | (1 << 16), out))
    cyc, sw = out[0] / 5, out[1] / 5
    print(f"real core {name}: s={s} sweeps={sw:.1f} cycles={cyc:.0f} cycles/round={cyc / max(sw * (s + (s & 1) - 1), 1):.0f}",
          flush=True)

# in-place Cholesky (CholeskyQR building block): cycles per column step
for s in (40, 64, 88, 120):
    rng = np.random.default_rng(s)
    X = rng.standard_normal((3 * s, s))
    G = X.T @ X
    dG = torch.from_numpy(G.ravel().copy()).cuda()
    out = (C.c_ulonglong * 2)()
    N.check(N.lib().ifmm_dev_jacobi_bench(N.ctx(), s, C.c_void_p(dG.data_ptr()), 5, 512 | (2 << 16), out))
    print(f"chol2 s={s}: cycles={out[0] / 5:.0f} per column step={out[0] / 5 / (s + 1):.0f}", flush=True)
