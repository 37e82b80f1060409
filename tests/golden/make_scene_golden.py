"""Scene generators and the RPY kernel from the UNMODIFIED reference, as
small fixtures (kernels.py:59-203).  Run in the build container:
    python tests/golden/make_scene_golden.py
Writes tests/golden/scenes.npz."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_shim  # noqa: E402

ifmm = ref_shim.import_reference()
rng = np.random.Generator(np.random.PCG64(3))
P = rng.uniform(-1, 1, (6, 3))
Q = np.vstack([P[:2], P[2:4] + 0.01, rng.uniform(-1, 1, (3, 3))])
out = {f"ico{s}": ifmm.icosphere(s) for s in range(4)}
out["lattice"] = ifmm.sphere_lattice(2, 3, 2, 1, 4.0, 1.5).points
out["shells"] = ifmm.concentric_shells([0, 1, 2], [1.0, 2.0, 3.5]).points
out["rpy_P"], out["rpy_Q"] = P, Q
out["rpy"] = ifmm.rpy_kernel(0.3, 0.7).block(P, Q)
out["sphere"] = ifmm.sphere_surface(50, 4).points
out["cube"] = ifmm.cube_uniform(50, 4).points
np.savez_compressed(os.path.join(HERE, "scenes.npz"), **out)
print({k: v.shape for k, v in out.items()})
