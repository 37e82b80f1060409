"""Micro-benchmark of the device MGS Arnoldi step (csrc/krylov.cu) at the c5
vector length: achieved HBM GB/s of ifmm_krylov_mgs against MEASURED_PEAKS.

Algorithmic bytes of one call with k1 basis vectors (8-byte elements):
pass 0 reads V_0 and w (16 n); passes 1..k1-1 read V_{i-1}, V_i, w and write w
(32 n); the norm pass reads V_{k1-1}, w and writes w (24 n).

    python tools/bench_gmres.py [--n 8388608] [--k 10 50 100]
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1508_01835_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_388_608)
    ap.add_argument("--k", type=int, nargs="+", default=[10, 50, 100])
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = None
    n = a.n
    kmax = max(a.k)
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn((kmax, n), dtype=torch.float64, device="cuda", generator=g)
    V /= V.norm(dim=1, keepdim=True)
    w0 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    h = np.zeros(kmax + 1)
    lib, ctx = N.lib(), N.ctx()
    for k1 in a.k:
        nbytes = 16 * n + 32 * n * (k1 - 1) + 24 * n
        ts = []
        for r in range(a.reps + 1):
            w = w0.clone()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            N.check(lib.ifmm_krylov_mgs(ctx, C.c_void_p(V.data_ptr()), n, k1, n,
                                        C.c_void_p(w.data_ptr()), h.ctypes.data_as(C.c_void_p)))
            ts.append(time.perf_counter() - t0)
        t = min(ts[1:])
        gbs = nbytes / t / 1e9
        print(json.dumps({"kernel": "ifmm_krylov_mgs", "n": n, "k1": k1, "ms": t * 1e3,
                          "alg_bytes": nbytes, "achieved_gbs": round(gbs, 1), "peak_gbs": peak,
                          "frac": round(gbs / peak, 3) if peak else None,
                          "timing": "host clock around the synchronous ABI call (includes "
                                    "one cooperative launch + the h readback)"}))


if __name__ == "__main__":
    main()
