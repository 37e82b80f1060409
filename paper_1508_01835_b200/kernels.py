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

KIND = {"exp": 1, "imq": 2, "inverse_multiquadric": 2, "benchmark": 3, "zero": 4, "rpy": 5}


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
        """(kind, p0, p1) understood by the CUDA engine, or ValueError.
        kind 5 (RPY, block_dim 3): p0 = radius a, p1 = 1 / (6 pi eta a)."""
        if not self.symmetric:
            raise ValueError("non-symmetric kernels are not supported by the engine")
        kind = KIND.get(self.name)
        if kind is None:
            raise ValueError(f"kernel '{self.name}' has no device implementation; "
                             f"supported: {sorted(KIND)}")
        if self.block_dim != (3 if kind == 5 else 1):
            raise ValueError(f"kernel '{self.name}': block_dim {self.block_dim} has no device "
                             "implementation")
        if kind == 2:
            spec = (kind, float(self.params["h"]), 0.0)
        elif kind == 3:
            spec = (kind, float(self.params["d"]), 0.0)
        elif kind == 5:
            a = float(self.params["radius"])
            spec = (kind, a, 1.0 / (6.0 * np.pi * float(self.params["viscosity"]) * a))
        else:
            spec = (kind, 0.0, 0.0)
        self._check_block_matches(kind)
        return spec

    def _check_block_matches(self, kind):
        """The engine evaluates the kernel from ``name`` / ``params``; a plugin
        whose ``block`` computes something else under a known name (e.g.
        ``Kernel("exp", 1, {}, other_fn)``) must not be silently replaced by
        the built-in formula.  A fixed 5 x 4 probe (incl. a coincident pair)
        compares ``block`` with the built-in of the same name and parameters."""
        if self.block is None or getattr(self, "_probed", False):
            return
        ref = {1: lambda: exp_kernel(), 2: lambda: imq_kernel(self.params["h"]),
               3: lambda: benchmark_kernel(self.params["d"]), 4: lambda: zero_kernel(),
               5: lambda: rpy_kernel(self.params["radius"], self.params["viscosity"])}[kind]()
        g = np.random.Generator(np.random.PCG64(20150807))
        Pp = g.uniform(-1.0, 1.0, size=(5, 3))
        Qq = np.vstack([g.uniform(-1.0, 1.0, size=(3, 3)), Pp[:1]])
        mine = np.asarray(self.block(Pp, Qq), dtype=float)
        want = np.asarray(ref.block(Pp, Qq), dtype=float)
        if mine.shape != want.shape or not np.allclose(mine, want, rtol=1e-12, atol=1e-14):
            raise ValueError(f"kernel '{self.name}': block() differs from the engine's device "
                             f"implementation of '{self.name}' with these params; a custom "
                             "kernel function has no device implementation")
        object.__setattr__(self, "_probed", True)


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


def rpy_kernel(radius: float, viscosity: float = 1.0) -> Kernel:
    """kernels.py:59-91: Rotne-Prager-Yamakawa 3x3 mobility blocks
    f(r) I + g(r) r^ r^T with c = 1/(6 pi eta a); far field (r > 2a)
    f = c(3a/4r + a^3/2r^3), g = c(3a/4r - 3a^3/2r^3); overlap f = c(1 - 9r/32a),
    g = c(3r/32a); self f = c, g = 0.  The host ``block`` gives the
    reference's point-major (3m x 3n) layout; the engine evaluates the same
    blocks in ``csrc/h2_kernels.cu`` (rpy_block, kernel kind 5)."""
    if radius <= 0 or viscosity <= 0:
        raise ValueError("radius and viscosity must be positive")
    a = float(radius)
    c0 = 1.0 / (6.0 * np.pi * viscosity * a)

    def block(P, Q):
        P = np.atleast_2d(np.asarray(P, dtype=float))
        Q = np.atleast_2d(np.asarray(Q, dtype=float))
        dv = P[:, None, :] - Q[None, :, :]
        r = np.sqrt(np.einsum("ijk,ijk->ij", dv, dv))
        safe = np.where(r == 0.0, 1.0, r)
        inv, inv3 = 1.0 / safe, 1.0 / safe ** 3
        far = r > 2.0 * a
        f = np.where(far, c0 * (0.75 * a * inv + 0.5 * a ** 3 * inv3), c0 * (1.0 - 9.0 * r / (32.0 * a)))
        g = np.where(far, c0 * (0.75 * a * inv - 1.5 * a ** 3 * inv3), c0 * (3.0 * r / (32.0 * a)))
        g = np.where(r == 0.0, 0.0, g)
        u = dv * inv[..., None]
        out = g[..., None, None] * (u[..., :, None] * u[..., None, :])
        out += f[..., None, None] * np.eye(3)
        m, n = len(P), len(Q)
        return out.transpose(0, 2, 1, 3).reshape(3 * m, 3 * n)

    return Kernel("rpy", 3, {"radius": a, "viscosity": float(viscosity)}, block)


def icosphere(subdivision: int) -> np.ndarray:
    """kernels.py:133-167: vertices of a unit icosphere (10*4^s + 2).

    Recursive 4-way face split of the regular icosahedron; each new vertex
    is the normalised edge midpoint, numbered in first-visit order.  Vertex
    and face orders follow the reference so the point sets are identical."""
    if subdivision < 0:
        raise ValueError("subdivision must be >= 0")
    t = (1.0 + np.sqrt(5.0)) / 2.0
    base = [(-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0), (0, -1, t), (0, 1, t),
            (0, -1, -t), (0, 1, -t), (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1)]
    V = [np.asarray(v, dtype=float) / np.linalg.norm(v) for v in base]
    F = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
         (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
         (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivision):
        seen = {}

        def midpoint(i, j):
            e = (i, j) if i < j else (j, i)
            if e not in seen:
                v = V[i] + V[j]
                V.append(v / np.linalg.norm(v))
                seen[e] = len(V) - 1
            return seen[e]

        nf = []
        for i, j, k in F:
            ij, jk, ki = midpoint(i, j), midpoint(j, k), midpoint(k, i)
            nf.extend([(i, ij, ki), (j, jk, ij), (k, ki, jk), (ij, jk, ki)])
        F = nf
    return np.array(V)


def sphere_lattice(nx: int, ny: int, nz: int, subdivision: int, spacing: float,
                   body_radius: float = 1.0) -> Scene:
    """kernels.py:170-182: an nx x ny x nz lattice of icosphere bodies (x
    slowest, z fastest)."""
    body = icosphere(subdivision) * body_radius
    shifts = [spacing * np.array([i, j, k], dtype=float)
              for i in range(nx) for j in range(ny) for k in range(nz)]
    pts = np.vstack([body + s for s in shifts]) if shifts else np.zeros((0, 3))
    return Scene(pts, f"sphere_lattice({nx}x{ny}x{nz}, subdivision={subdivision}, "
                      f"spacing={spacing}, body_radius={body_radius})")


def concentric_shells(subdivisions, radii) -> Scene:
    """kernels.py:185-192: one icosphere shell per (subdivision, radius)."""
    if len(subdivisions) != len(radii):
        raise ValueError("subdivisions and radii must have equal length")
    pts = np.vstack([icosphere(s) * r for s, r in zip(subdivisions, radii)])
    return Scene(pts, f"concentric_shells(subdivisions={list(subdivisions)}, "
                      f"radii={list(radii)})")


def scene_to_text(scene: Scene, path) -> None:
    """kernels.py:195-196: x y z per line, round-trip precision."""
    np.savetxt(path, scene.points, fmt="%.17g")


def scene_from_text(path, description: str = "imported") -> Scene:
    """kernels.py:199-203."""
    pts = np.loadtxt(path, ndmin=2)
    if pts.shape[1] != 3:
        raise ValueError("expected three columns (x y z)")
    return Scene(pts, description)
