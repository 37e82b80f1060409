"""Micro-benchmark (diagnostics): one weighted basis union on the device at
synthetic sizes up to the giant level-2 unions of c3/c4, with the kernel's
phase counters.  B and F are orthonormal, weights graded like the engine's
(geometric decay), thr at 1e-6 of the largest weight.

    python tools/bench_union.py [m k_old k_f] ..."""
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_01835_b200 import _native as N  # noqa: E402

N.ctx()
sizes = [(120, 30, 8), (230, 45, 10), (530, 80, 12), (620, 110, 14), (620, 240, 28),
         (1200, 330, 40), (2000, 450, 50)]
if len(sys.argv) > 3:
    a = list(map(int, sys.argv[1:]))
    sizes = [tuple(a[i:i + 3]) for i in range(0, len(a) - 2, 3)]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ptr(t):
    return C.c_void_p(t.data_ptr())


for m, ko, kf in sizes:
    rng = np.random.default_rng(m + ko)
    B, _ = np.linalg.qr(rng.standard_normal((m, ko)))
    F, _ = np.linalg.qr(rng.standard_normal((m, kf)))
    w = np.sort(10.0 ** (-9 * rng.random(ko)))[::-1]
    wf = np.sort(10.0 ** (-9 * rng.random(kf)))[::-1] * 0.5
    thr = 1e-6 * w[0]
    cap = min(m, ko + kf)
    dB, dw, dF, dwf = dev(B.ravel()), dev(w), dev(F.ravel()), dev(wf)
    NB = torch.zeros(m * cap, dtype=torch.float64, device="cuda")
    NW = torch.zeros(cap, dtype=torch.float64, device="cuda")
    OM = torch.zeros(cap * ko, dtype=torch.float64, device="cuda")
    FM = torch.zeros(cap * kf, dtype=torch.float64, device="cuda")
    dr = torch.zeros(1, dtype=torch.int32, device="cuda")
    up = (C.c_ulonglong * 48)()
    for rep in range(2):
        N.lib().ifmm_union_profile(up, 1)
        N.lib().ifmm_union_post_profile((C.c_ulonglong * 16)(), 1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        N.check(N.lib().ifmm_dev_union(N.ctx(), m, ko, kf, ptr(dB), ptr(dw), ptr(dF), ptr(dwf), thr, 0,
                                       ptr(NB), ptr(NW), ptr(OM), ptr(FM), ptr(dr)))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    N.lib().ifmm_union_profile(up, 1)
    u = list(up)
    s = u[5]
    print(f"m={m:5d} C={ko + kf:4d} s={s:4d} rank={int(dr.item()):4d} wall {dt * 1e3:8.2f} ms | Mcycles "
          f"aca {u[0] / 1e6:7.2f} cholqr {u[1] / 1e6:7.2f} jacobi {u[3] / 1e6:7.2f} (sweeps {u[11]}) "
          f"out {u[4] / 1e6:6.2f}", flush=True)
    vp = (C.c_ulonglong * 16)()
    N.lib().ifmm_union_post_profile(vp, 1)
    v = list(vp)
    if v[6]:
        print(f"   fused second half: s={v[7]} k={v[10]} sweeps {v[9]} pass2 {v[11]} | kcycles gram1 {v[0] / 1e3:.1f} chol+M {v[1] / 1e3:.1f} "
              f"trsm+gram2+corr {v[2] / 1e3:.1f} jacobi {v[3] / 1e3:.1f} order+Z {v[4] / 1e3:.1f} out {v[5] / 1e3:.1f}"
              f" | gram1: fetch+store {v[12] / 1e3:.1f} accum {v[13] / 1e3:.1f} reduce {v[14] / 1e3:.1f}; chol only {v[15] / 1e3:.1f}", flush=True)
    if u[39]:
        print(f"   cholqr parts (m>400): scale+gram1+chol1 {u[38] / 1e6:.3f} trsm1 {u[34] / 1e6:.3f} "
              f"gram2 {u[35] / 1e6:.3f} chol2 {u[36] / 1e6:.3f} trsm2+trmul {u[37] / 1e6:.3f}", flush=True)
