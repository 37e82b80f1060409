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

``HaloPlan`` / ``distributed_matvec_halo`` replace the two full-length
all-reduces by what the product needs: x stays distributed
(every rank holds its own range), the x of the neighbour leaves owned by
other ranks and the multipoles of the interaction-list clusters owned by
other ranks travel point to point (grouped isend / irecv: NCCL over NVLink on
the GPUs, gloo in the CPU tests), and only the few upper-level clusters whose
point range spans several ranks are all-reduced.  The result stays
distributed too (own rows).
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


class HaloPlan:
    """Who needs what for one rank of the Morton-range partitioned matvec.

    start / stop / level: per-cluster point ranges and levels; children,
    neighbors, interactions: the tree's lists; off / rank: offset and length
    of every cluster's segment in the multipole vector (-1 / 0 if absent);
    ranges: [(p_lo, p_hi)] of all ranks; me: this rank.

    Built once per (operators, world).  Attributes:
      x_send[r] / x_recv[r]   point ranges (a, e) of x sent to / received from r
      y_send[r] / y_recv[r]   multipole segments (o, k) sent to / received from r
      shared                  multipole segments (o, k) of the clusters that span
                              ranks (summed over ranks by an all-reduce)"""

    def __init__(self, start, stop, level, depth, leaves, neighbors, interactions, off, rank,
                 ranges, me):
        self.ranges, self.me = list(ranges), int(me)
        world = len(self.ranges)
        nc = len(start)

        def owner(c):  # rank whose range contains the cluster, or -1 if it spans ranks
            for r, (lo, hi) in enumerate(self.ranges):
                if start[c] >= lo and stop[c] <= hi and stop[c] > start[c]:
                    return r
            return -1

        own = [owner(c) for c in range(nc)]
        self.owner = own
        meets = [[c for c in range(nc) if level[c] >= 2 and start[c] < hi and stop[c] > lo]
                 for (lo, hi) in self.ranges]
        self.shared = sorted((off[c], rank[c]) for c in range(nc)
                             if level[c] >= 2 and own[c] == -1 and off[c] >= 0 and rank[c] > 0)
        # x halo: neighbour leaves of a rank's own leaves that another rank owns
        need_x = [set() for _ in range(world)]
        for c in leaves:
            r = own[c]
            for q in neighbors[c]:
                if own[q] != r:
                    need_x[r].add(q)
        # multipole halo: interaction-list clusters of every cluster meeting the range
        need_y = [set() for _ in range(world)]
        for r in range(world):
            for c in meets[r]:
                for q in interactions[c]:
                    if own[q] >= 0 and own[q] != r and off[q] >= 0 and rank[q] > 0:
                        need_y[r].add(q)
        self.x_recv = {r: sorted((start[q], stop[q]) for q in need_x[self.me] if own[q] == r)
                       for r in range(world) if r != self.me}
        self.x_send = {r: sorted((start[q], stop[q]) for q in need_x[r] if own[q] == self.me)
                       for r in range(world) if r != self.me}
        self.y_recv = {r: sorted((off[q], rank[q]) for q in need_y[self.me] if own[q] == r)
                       for r in range(world) if r != self.me}
        self.y_send = {r: sorted((off[q], rank[q]) for q in need_y[r] if own[q] == self.me)
                       for r in range(world) if r != self.me}
        for d in (self.x_recv, self.x_send, self.y_recv, self.y_send):
            for r in [r for r, v in d.items() if not v]:
                del d[r]
        # segments of the multipole vector this rank may read in phase 1 (tests poison the rest)
        mine = {(off[c], rank[c]) for c in meets[self.me] if off[c] >= 0 and rank[c] > 0}
        self.y_valid = sorted(mine | set(self.shared) | {s for v in self.y_recv.values() for s in v})
        lo, hi = self.ranges[self.me]
        self.x_valid = sorted({(lo, hi)} | {s for v in self.x_recv.values() for s in v})

    @classmethod
    def from_tree(cls, tree, topology, rank_of, world, me):
        """Plan for ``tree`` / ``topology`` (package types) and the H2 ranks
        ``rank_of`` (dict cluster -> rank)."""
        cl = tree.clusters
        nc = len(cl)
        off, rk, tot = [-1] * nc, [0] * nc, 0
        for c in range(nc):
            k = int(rank_of.get(c, 0) or 0)
            if cl[c].level >= 2 and k > 0:
                off[c], rk[c] = tot, k
                tot += k
        plan = cls([c.start for c in cl], [c.stop for c in cl], [c.level for c in cl], tree.depth,
                   list(tree.levels[tree.depth]), topology.neighbors, topology.interactions, off, rk,
                   tree_partition(tree, world), me)
        plan.n_multipole = tot
        return plan

    def volume(self):
        """Doubles this rank sends per matvec: (x halo, multipole halo, shared all-reduce)."""
        return (sum(e - a for v in self.x_send.values() for a, e in v),
                sum(k for v in self.y_send.values() for _, k in v),
                sum(k for _, k in self.shared))


def _pack(buf, segs, cat, as_len=False):
    parts = [buf[a:(a + b) if as_len else b] for a, b in segs]
    return cat(parts)


def distributed_matvec_halo(x_own, n_points, n_multipole, plan, phase_fn, exchange, allreduce, zeros,
                            cat, poison=None):
    """One rank of the halo-exchange protocol.  x_own: this rank's range of x
    (tree order); returns this rank's rows of the product.

    phase_fn as in ``distributed_matvec`` (full-length address space: only the
    own range, the halo and the needed multipole segments hold data);
    exchange(send: {peer: 1-D buffer}, recv_len: {peer: n}) -> {peer: buffer}
    moves the packed halos point to point; allreduce sums in place over the
    ranks; cat concatenates 1-D buffers; poison (tests): value written to
    every entry the protocol did not deliver before phase 1."""
    lo, hi = plan.ranges[plan.me]
    xs = zeros(n_points)
    xs[lo:hi] = x_own
    # ---- x halo ----
    got = exchange({r: _pack(xs, segs, cat) for r, segs in plan.x_send.items()},
                   {r: sum(e - a for a, e in segs) for r, segs in plan.x_recv.items()})
    for r, segs in plan.x_recv.items():
        o = 0
        for a, e in segs:
            xs[a:e] = got[r][o:o + e - a]
            o += e - a
    yv = zeros(n_multipole)
    ys = zeros(n_points)
    phase_fn(xs, ys, yv, 0, lo, hi)
    # ---- clusters spanning ranks: all-reduce of their partial multipoles ----
    if plan.shared:
        sh = _pack(yv, plan.shared, cat, as_len=True)
        allreduce(sh)
        o = 0
        for a, k in plan.shared:
            yv[a:a + k] = sh[o:o + k]
            o += k
    # ---- multipole halo ----
    got = exchange({r: _pack(yv, segs, cat, as_len=True) for r, segs in plan.y_send.items()},
                   {r: sum(k for _, k in segs) for r, segs in plan.y_recv.items()})
    for r, segs in plan.y_recv.items():
        o = 0
        for a, k in segs:
            yv[a:a + k] = got[r][o:o + k]
            o += k
    if poison is not None:
        keep = zeros(n_multipole)
        for a, k in plan.y_valid:
            keep[a:a + k] = 1.0
        yv[keep == 0] = poison
        keepx = zeros(n_points)
        for a, e in plan.x_valid:
            keepx[a:e] = 1.0
        xs[keepx == 0] = poison
    phase_fn(xs, ys, yv, 1, lo, hi)
    return ys[lo:hi]


def torch_exchange(group=None):
    """exchange() for ``distributed_matvec_halo`` over torch.distributed:
    one grouped batch of isend / irecv (ncclSend / ncclRecv under NCCL)."""
    import torch
    import torch.distributed as dist

    def exchange(send, recv_len):
        if not send and not recv_len:
            return {}
        ref = next(iter(send.values())) if send else None
        ops_, out = [], {}
        for r, n in recv_len.items():
            out[r] = torch.empty(n, dtype=torch.float64, device=ref.device if ref is not None else "cpu")
            ops_.append(dist.P2POp(dist.irecv, out[r], r, group=group))
        for r, b in send.items():
            ops_.append(dist.P2POp(dist.isend, b.contiguous(), r, group=group))
        for w in dist.batch_isend_irecv(ops_):
            w.wait()
        return out
    return exchange


def h2_matvec_halo(ops, x_own, plan, group=None):
    """The halo-exchange matvec on the GPUs: x_own is this rank's Morton range
    of x in TREE order (a CUDA tensor); returns this rank's rows in tree order.
    plan = HaloPlan.from_tree(ops.tree, ops.topology, ops.rank, world, rank)."""
    import torch
    import torch.distributed as dist

    if not (isinstance(x_own, torch.Tensor) and x_own.is_cuda):
        raise ValueError("h2_matvec_halo takes a CUDA tensor")
    lo, hi = plan.ranges[plan.me]
    if x_own.shape != (hi - lo,):
        raise ValueError("x_own must hold this rank's point range")
    world = len(plan.ranges)

    def phase_fn(xs, ys, yv, phase, p_lo, p_hi):
        torch.cuda.current_stream().synchronize()
        N.check(N.lib().ifmm_h2_matvec_part(ops._h, C.c_void_p(xs.data_ptr()),
                                            C.c_void_p(ys.data_ptr()), C.c_void_p(yv.data_ptr()),
                                            phase, p_lo, p_hi))

    def allreduce(v):
        if world > 1:
            dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)

    exchange = torch_exchange(group) if world > 1 else (lambda send, recv_len: {})
    return distributed_matvec_halo(
        x_own.contiguous(), ops.tree.n_points, max(plan.n_multipole, 1), plan, phase_fn, exchange,
        allreduce, lambda n: torch.zeros(n, dtype=torch.float64, device=x_own.device), torch.cat)


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
