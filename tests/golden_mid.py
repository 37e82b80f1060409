"""Loader for the mid-size reference goldens (tests/golden/mid/, written by
tests/golden/make_golden_mid.py from the unmodified reference).  Points are
regenerated from the seeded recipe."""
import os

import numpy as np

MID = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "mid")


def mid_names():
    return sorted(f[:-4] for f in os.listdir(MID) if f.endswith(".npz"))


def load_mid(name):
    return dict(np.load(os.path.join(MID, name + ".npz"), allow_pickle=False))


def mid_points(g):
    N, dim, seed = int(g["N"]), int(g["dim"]), int(g["seed"])
    r = np.random.Generator(np.random.PCG64(seed))
    if dim == 2:
        return np.column_stack([r.uniform(0.0, 1.0, size=(N, 2)), np.zeros(N)])
    pts = r.uniform(0.0, 1.0, size=(N, 3))
    zs = float(g["zscale"]) if "zscale" in g else 1.0
    if zs != 1.0:
        pts[:, 2] *= zs
    return pts


def mid_inputs(P, g):
    """(points, b, Kernel) of a mid case for the package P."""
    pts = mid_points(g)
    K = P.exp_kernel() if str(g["kernel"]) == "exp" else P.imq_kernel(float(g["h"]))
    return pts, g["b"], K
