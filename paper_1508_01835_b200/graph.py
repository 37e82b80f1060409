"""Extended sparse graph on the device (mirror of ``ifmm.graph``).

``assemble_extended_graph`` (graph.py:219-229) builds the node/edge
store inside the engine (device blocks, host adjacency);
``estimate_sigma0`` (graph.py:232-241) draws the reference's Gaussian
sketch on the host -- exactly ``Generator(PCG64(seed)).standard_normal
((dim, 11))`` -- and runs the power iterations, QRs and the final SVD on the
device.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .h2 import H2Operators


class ExtendedGraph:
    def __init__(self, ops: H2Operators, handle):
        self.ops = ops
        self.tree = ops.tree
        self.topology = ops.topology
        self.block_dim = ops.block_dim
        self._h = handle
        self.consumed = False

    def __del__(self):
        try:
            N.lib().ifmm_graph_destroy(self._h)
        except Exception:
            pass

    def _info(self):
        d, n, e = C.c_longlong(), C.c_longlong(), C.c_longlong()
        N.check(N.lib().ifmm_graph_info(self._h, C.byref(d), C.byref(n), C.byref(e)))
        return d.value, n.value, e.value

    @property
    def dim(self) -> int:
        return self._info()[0]

    @property
    def num_edges(self) -> int:
        return self._info()[2]


def assemble_extended_graph(ops: H2Operators, topology=None, b=None,
                            consume: bool = False) -> ExtendedGraph:
    """graph.py:219-229.  The right-hand side is not carried by the device
    graph: the solve replays the event log from b (factor.py:99-157).
    ``consume=True`` moves the operator blocks into the graph (no copy; the
    operators cannot be used afterwards) -- for problems near device memory."""
    if ops.tree.depth >= 2 and not ops._weighted:
        raise ValueError("operators have no basis weights; run initialize_weights first")
    h = N.lib().ifmm_graph_build(ops._h, 1 if consume else 0)
    return ExtendedGraph(ops, N.check_handle(h))


def estimate_sigma0(graph: ExtendedGraph, seed: int = 0, oversample: int = 10,
                    power_iters: int = 2) -> float:
    """graph.py:232-241 -> lowrank.randomized_svd(start_rank=1, max_rank=1)."""
    if oversample < 2:
        raise ValueError("oversample must be >= 2")
    if graph.consumed:
        raise ValueError("graph already factorized")
    rng = np.random.Generator(np.random.PCG64(seed))
    dim = graph.dim
    width = min(1 + oversample, dim)
    omega = np.ascontiguousarray(rng.standard_normal((dim, width)))
    out = C.c_double()
    N.check(N.lib().ifmm_graph_sigma0(graph._h, N.as_dp(omega), width, int(power_iters),
                                      C.byref(out)))
    return float(out.value)
