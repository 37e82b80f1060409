"""Fault and race hunting without compute-sanitizer (closed on the GPU pool):
the small end-to-end case of tools/sanitize_small.py with the multi-CTA
cooperative giant-union kernels forced on (IFMM_GIANT=20) and a sync +
error check after every launch (IFMM_DEBUG_SYNC=1), run twice in fresh
processes -- every solution must be bitwise identical across runs (grid
barriers, last-block tickets and fixed-order reductions are deterministic
only if race-free)."""

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_small.py"), "3000"],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return {ln.split()[1]: ln.split()[2] for ln in out.stdout.splitlines() if ln.startswith("XHASH")}


def test_giant_path_debug_sync_deterministic():
    a = _run({"IFMM_GIANT": "20", "IFMM_DEBUG_SYNC": "1"})
    b = _run({"IFMM_GIANT": "20"})
    c = _run({"IFMM_GIANT": "20"})
    assert set(a) == {"reference", "wavefront"}
    assert a == b == c
