"""Kernel plugin type and scenes (mirror of ``ifmm.kernels``).

The reference's plugin is ``Kernel(name, block_dim, params, block,
symmetric)`` with a Python ``block(P, Q)`` callable (kernels.py:22-39).  A
Python callable cannot run on the device, so the engine recognises kernels
by ``name`` + ``params`` and evaluates them in-register inside its fused
kernel-evaluation CUDA kernels.  ``block`` is kept (numpy) for callers and
tests that want the reference semantics on the host; it is never used by
the engine.  Kernels without a device implementation raise ValueError --
there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import numpy as np

KIND = {"exp": 1, "imq": 2, "inverse_multiquadric": 2, "benchmark": 3, "zero": 4}


def _dist(P, Q):
    P = np.atleast_2d(np.asarray(P, dtype=float))
    Q = np.atleast_2d(np.asarray(Q, dtype=float))
    d = P[:, None, :] - Q[None, :, :]
    return np.sqrt(np.sum(d * d, axis=-1))


@dataclass
class Kernel:
    name: str
    block_dim: int
    params: dict
    block: Callable = field(repr=False, default=None)
    symmetric: bool = True

    def evaluate(self, ri, rj):
        return self.block(np.atleast_2d(ri), np.atleast_2d(rj))

    def device_spec(self):
        """(kind, p0) understood by the CUDA engine, or ValueError."""
        if self.block_dim != 1:
            raise ValueError(f"kernel '{self.name}': block_dim {self.block_dim} has no device "
                             "implementation yet (scalar kernels only)")
        if not self.symmetric:
            raise ValueError("non-symmetric kernels are not supported by the engine")
        kind = KIND.get(self.name)
        if kind is None:
            raise ValueError(f"kernel '{self.name}' has no device implementation; "
                             f"supported: {sorted(KIND)}")
        if kind == 2:
            return kind, float(self.params["h"])
        if kind == 3:
            return kind, float(self.params["d"])
        return kind, 0.0


def exp_kernel() -> Kernel:
    """A_ij = exp(-|x_i - x_j|) (BASELINE configs 1-2)."""
    return Kernel("exp", 1, {}, lambda P, Q: np.exp(-_dist(P, Q)))


def imq_kernel(h: float) -> Kernel:
    """A_ij = 1/sqrt(|x_i - x_j|^2 + h^2) (BASELINE configs 3-5)."""
    if h <= 0:
        raise ValueError("h must be positive")
    h = float(h)
    return Kernel("imq", 1, {"h": h}, lambda P, Q: 1.0 / np.sqrt(_dist(P, Q) ** 2 + h * h))


def benchmark_kernel(d: float) -> Kernel:
    """kernels.py:42-56: 1 at r=0, r/d for 0<r<d, d/r for r>=d."""
    if d <= 0:
        raise ValueError("d must be positive")

    def block(P, Q):
        r = _dist(P, Q)
        out = np.empty_like(r)
        near = r < d
        out[near] = r[near] / d
        out[~near] = d / r[~near]
        out[r == 0.0] = 1.0
        return out

    return Kernel("benchmark", 1, {"d": d}, block)


def zero_kernel() -> Kernel:
    return Kernel("zero", 1, {}, lambda P, Q: np.zeros((len(np.atleast_2d(P)),
                                                         len(np.atleast_2d(Q)))))


def scaled_d(base: float, n_points: int, exponent: float) -> float:
    """kernels.py:94-98."""
    if n_points < 1:
        raise ValueError("n_points must be >= 1")
    return base * (n_points / 1000.0) ** exponent


@dataclass
class Scene:
    points: np.ndarray
    description: str


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def sphere_surface(n: int, seed: int) -> Scene:
    """kernels.py:111-122: normalised PCG64 Gaussians on the unit sphere."""
    if n < 1:
        raise ValueError("n must be >= 1")
    g = _rng(seed).standard_normal((n, 3))
    norms = np.linalg.norm(g, axis=1, keepdims=True)
    while np.any(norms == 0.0):
        bad = norms[:, 0] == 0.0
        g[bad] = _rng(seed + 1).standard_normal((bad.sum(), 3))
        norms = np.linalg.norm(g, axis=1, keepdims=True)
    return Scene(g / norms, f"sphere_surface(n={n}, seed={seed})")


def cube_uniform(n: int, seed: int) -> Scene:
    """kernels.py:125-130: uniform in [-1, 1]^3."""
    if n < 1:
        raise ValueError("n must be >= 1")
    return Scene(_rng(seed).uniform(-1.0, 1.0, size=(n, 3)), f"cube_uniform(n={n}, seed={seed})")
