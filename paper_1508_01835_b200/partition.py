"""Morton-range partitioning of the FMM matvec over ranks.

The reference (``ifmm.krylov.h2_matvec``, krylov.py:119-159) is a single
process.  Here every rank owns a contiguous Morton range of whole leaves --
the points [p_lo, p_hi) of the tree order -- and the product runs as

  phase 0  (device)  partial multipoles y of every cluster meeting the range
                      (P2M of the own leaves, M2M over the children in range);
  all-reduce(y)       NCCL over NVLink: the upper tree levels, whose clusters
                      span ranks, are summed; the vector is small (sum of the
                      cluster ranks, ~15 MB at c4);
  phase 1  (device)  M2L from the full y, L2L, and the rows of the own leaves:
                      L2P + P2P over the neighbour leaves' x (the x halo);
  all-reduce(rows)    the disjoint row ranges are assembled on every rank.

Each rank does the work of its own targets only; the operator blocks are
those of ``chebyshev_operators`` on the rank's device.  GMRES (c5) calls this
as its ``apply_A``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def morton_partition(leaf_start, leaf_stop, world: int):
    """Split Morton-ordered leaves (point ranges [start, stop)) into `world`
    contiguous groups with balanced point counts.  Returns [(p_lo, p_hi)]."""
    if world < 1:
        raise ValueError("world must be >= 1")
    starts = np.asarray(leaf_start, dtype=np.int64)
    stops = np.asarray(leaf_stop, dtype=np.int64)
    n = int(stops[-1]) if len(stops) else 0
    cuts = [0]
    for r in range(1, world):
        target = r * n / world
        # first leaf boundary at or after the target (leaf starts are sorted)
        k = int(np.searchsorted(starts, target, side="left"))
        b = int(starts[k]) if k < len(starts) else n
        cuts.append(max(b, cuts[-1]))
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def tree_partition(tree, world: int):
    leaves = tree.levels[tree.depth]
    return morton_partition([tree.clusters[c].start for c in leaves],
                            [tree.clusters[c].stop for c in leaves], world)


def distributed_matvec(x_sorted, n_multipole, p_range, phase_fn, allreduce, zeros):
    """The rank-local protocol shared by the device path and the CPU tests.

    x_sorted: the full input in tree order (the halo is the whole vector);
    phase_fn(xs, ys, yv, phase, p_lo, p_hi) runs one phase of this rank;
    allreduce(v) sums v over the ranks in place; zeros(n) allocates."""
    p_lo, p_hi = p_range
    yv = zeros(n_multipole)
    ys = zeros(len(x_sorted))
    phase_fn(x_sorted, ys, yv, 0, p_lo, p_hi)
    allreduce(yv)
    phase_fn(x_sorted, ys, yv, 1, p_lo, p_hi)
    allreduce(ys)
    return ys


def h2_matvec_distributed(ops, x, group=None):
    """h2_matvec over the ranks of `group` (torch.distributed, NCCL on the
    GPU); x is the full CUDA vector in original point order on every rank, the
    full product is returned on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise ValueError("h2_matvec_distributed takes a CUDA tensor")
    if x.shape != (ops.dim,):
        raise ValueError("vector length mismatch")
    perm = torch.as_tensor(np.asarray(ops.tree.perm), device=x.device)
    ranges = tree_partition(ops.tree, world)
    ms = C.c_longlong()
    N.check(N.lib().ifmm_h2_multipole_size(ops._h, C.byref(ms)))

    def phase_fn(xs, ys, yv, phase, lo, hi):
        torch.cuda.current_stream().synchronize()
        N.check(N.lib().ifmm_h2_matvec_part(ops._h, C.c_void_p(xs.data_ptr()),
                                            C.c_void_p(ys.data_ptr()), C.c_void_p(yv.data_ptr()),
                                            phase, lo, hi))

    def allreduce(v):
        if world > 1:
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)

    xs = x.contiguous()[perm].contiguous()
    ys = distributed_matvec(xs, max(ms.value, 1), ranges[rank], phase_fn, allreduce,
                            lambda n: torch.zeros(n, dtype=torch.float64, device=x.device))
    y = torch.empty_like(ys)
    y[perm] = ys
    return y
