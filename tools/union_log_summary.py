"""Summarise an IFMM_UNION_LOG file (one line per union launch: n_smem
n_global max_m max_C max_rank device_ms pre_ms gap_ms) by max-m bucket.
Diagnostics only.    python tools/union_log_summary.py <log>"""
import sys

import numpy as np

a = np.loadtxt(sys.argv[1])
n = a[:, 0] + a[:, 1]
m = a[:, 2]
ms = a[:, 5]
gap = a[:, 7]
print(f"{len(a)} launches, device {ms.sum() / 1e3:.2f} s, host gaps {gap.sum() / 1e3:.2f} s, "
      f"unions {int(n.sum())}")
for lo, hi in [(0, 128), (128, 256), (256, 400), (400, 600), (600, 1e9)]:
    s = (m > lo) & (m <= hi)
    if s.any():
        print(f"max m in ({lo}, {hi:.0f}]: {s.sum():6d} launches, {ms[s].sum() / 1e3:7.2f} s, "
              f"mean {ms[s].mean():6.3f} ms, unions/launch {n[s].mean():5.2f}, "
              f"mean max C {a[s, 3].mean():6.1f}, mean max rank {a[s, 4].mean():6.1f}")
