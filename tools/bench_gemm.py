"""Micro-benchmark (diagnostics): the grouped DMMA GEMM on single problems of
the elimination's shapes (Schur product, rebase) against cuBLAS DGEMM.

    python tools/bench_gemm.py [M N K] ..."""
import ctypes as C
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1508_01835_b200 import _native as N  # noqa: E402

N.ctx()
sizes = [(512, 512, 512), (2048, 2048, 256), (7000, 7000, 280), (4096, 4096, 4096), (280, 7000, 280),
         (64, 64, 40), (40, 200, 40)]
if len(sys.argv) > 3:
    a = list(map(int, sys.argv[1:]))
    sizes = [tuple(a[i:i + 3]) for i in range(0, len(a) - 2, 3)]


def ptr(t):
    return C.c_void_p(t.data_ptr())


for M, Nn, K in sizes:
    for ta, tb in ((0, 0), (1, 0), (0, 1)):
        A = torch.randn((K, M) if ta else (M, K), dtype=torch.float64, device="cuda")
        B = torch.randn((Nn, K) if tb else (K, Nn), dtype=torch.float64, device="cuda")
        Cm = torch.zeros((M, Nn), dtype=torch.float64, device="cuda")
        reps = max(3, min(50, int(2e11 / (2.0 * M * Nn * K))))
        for it in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(reps):
                N.check(N.lib().ifmm_dev_gemm(N.ctx(), M, Nn, K, ptr(A), A.shape[1], ta, ptr(B),
                                              B.shape[1], tb, ptr(Cm), Nn, 1.0, 0.0))
            N.check(N.lib().ifmm_dev_sync(N.ctx()))
            dt = (time.perf_counter() - t0) / reps
        ref = (A.T if ta else A) @ (B.T if tb else B)
        err = float((Cm - ref).abs().max() / ref.abs().max())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            ref = torch.matmul(A.T if ta else A, B.T if tb else B)
        torch.cuda.synchronize()
        dc = (time.perf_counter() - t0) / reps
        fl = 2.0 * M * Nn * K
        print(f"M={M:5d} N={Nn:5d} K={K:5d} ta={ta} tb={tb}: ours {dt * 1e6:9.1f} us {fl / dt / 1e12:6.2f} TF/s | "
              f"cuBLAS {dc * 1e6:9.1f} us {fl / dc / 1e12:6.2f} TF/s | err {err:.1e}", flush=True)
