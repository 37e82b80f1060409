"""Morton-range partitioned FMM matvec (paper_1508_01835_b200/partition.py):
the partition plan and the rank protocol (partial multipoles -> all-reduce ->
locals + own rows -> all-reduce) on world-size 2 and 3 gloo groups on CPU.

The device phases (H2::matvec_part) are replaced here by a numpy restatement
of the same per-rank phase semantics over the oracle's operators, and the
assembled product must equal the oracle's single-process h2_matvec
(krylov.py:119-159).  The GPU test (test_gpu_pipeline.py) checks the device
phases against the single-device matvec."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1508_01835_b200.partition import (HaloPlan, distributed_matvec, distributed_matvec_halo,
                                             morton_partition, torch_exchange)


def test_morton_partition_balanced_whole_leaves():
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 60, size=200)
    stops = np.cumsum(sizes)
    starts = stops - sizes
    for world in (1, 2, 3, 8):
        rr = morton_partition(starts, stops, world)
        assert rr[0][0] == 0 and rr[-1][1] == stops[-1]
        assert all(a[1] == b[0] for a, b in zip(rr, rr[1:]))
        bounds = set(starts.tolist()) | {int(stops[-1])}
        assert all(lo in bounds and hi in bounds for lo, hi in rr)
        n = stops[-1]
        assert max(hi - lo for lo, hi in rr) <= n / world + sizes.max()
    with pytest.raises(ValueError):
        morton_partition(starts, stops, 0)


def _oracle_setup():
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import ifmm_np as O
    g = np.random.Generator(np.random.PCG64(2))
    pts = g.uniform(size=(3000, 3))
    tree, topo, ops = O.pipeline(pts, O.imq_block(3000 ** (-1 / 3)), 32, 3, 1e-6)
    return O, tree, topo, ops


def _offsets(tree, ops):
    off, tot = {}, 0
    for c in range(tree.n_clusters):
        if tree.level[c] >= 2 and ops.rank.get(c, 0) > 0:
            off[c] = tot
            tot += ops.rank[c]
    return off, tot


def _np_phase(tree, topo, ops, off):
    """numpy restatement of H2::matvec_part (h2.cu) for one rank."""
    def meets(c, lo, hi):
        return tree.start[c] < hi and tree.stop[c] > lo

    def inside(c, lo, hi):
        return tree.start[c] >= lo and tree.stop[c] <= hi

    def phase_fn(xs, ys, yv, phase, lo, hi):
        if phase == 0:
            for c in tree.leaves():
                if inside(c, lo, hi):
                    yv[off[c]:off[c] + ops.rank[c]] = ops.leaf_v[c].T @ xs[tree.start[c]:tree.stop[c]]
            for lv in range(tree.depth - 1, 1, -1):
                for p in tree.levels[lv]:
                    if meets(p, lo, hi):
                        acc = np.zeros(ops.rank[p])
                        for c in tree.children[p]:
                            if meets(c, lo, hi):
                                acc += ops.transfer_vt[c] @ yv[off[c]:off[c] + ops.rank[c]]
                        yv[off[p]:off[p] + ops.rank[p]] = acc
            return
        z = {}
        for lv in range(2, tree.depth + 1):
            for c in tree.levels[lv]:
                if not meets(c, lo, hi):
                    continue
                acc = np.zeros(ops.rank[c])
                for q in topo.interactions[c]:
                    acc += ops.coupling[(c, q)] @ yv[off[q]:off[q] + ops.rank[q]]
                if lv > 2:
                    acc += ops.transfer_u[c] @ z[tree.parent[c]]
                z[c] = acc
        for c in tree.leaves():
            if not inside(c, lo, hi):
                continue
            a, e = tree.start[c], tree.stop[c]
            seg = np.zeros(e - a)
            for q in topo.neighbors[c]:
                seg += ops.near[(c, q)] @ xs[tree.start[q]:tree.stop[q]]
            seg += ops.leaf_u[c] @ z[c]
            ys[a:e] = seg
    return phase_fn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O, tree, topo, ops = _oracle_setup()
    off, tot = _offsets(tree, ops)
    leaves = tree.leaves()
    ranges = morton_partition(tree.start[leaves], tree.stop[leaves], world)
    x = np.random.Generator(np.random.PCG64(5)).standard_normal(len(tree.points))
    xs = x[tree.perm]

    def allreduce(v):
        t = torch.from_numpy(v)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    ys = distributed_matvec(xs, tot, ranges[rank], _np_phase(tree, topo, ops, off), allreduce,
                            lambda n: np.zeros(n))
    y = np.empty_like(ys)
    y[tree.perm] = ys
    ref = O.h2_matvec(ops, x)
    q.put((rank, float(np.linalg.norm(y - ref) / np.linalg.norm(ref)), ranges[rank]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_matvec_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, rel, rng_ in out:
        assert rel < 1e-13, (rank, rel)
    # the ranges tile the points
    assert out[0][2][0] == 0 and all(out[i][2][1] == out[i + 1][2][0] for i in range(world - 1))


def _halo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    O, tree, topo, ops = _oracle_setup()
    off, tot = _offsets(tree, ops)
    leaves = list(tree.leaves())
    ranges = morton_partition(tree.start[leaves], tree.stop[leaves], world)
    nc = tree.n_clusters
    offs = [off.get(c, -1) for c in range(nc)]
    rks = [int(ops.rank.get(c, 0)) if c in off else 0 for c in range(nc)]
    plan = HaloPlan(tree.start, tree.stop, tree.level, tree.depth, leaves, topo.neighbors,
                    topo.interactions, offs, rks, ranges, rank)
    x = np.random.Generator(np.random.PCG64(5)).standard_normal(len(tree.points))
    xs = x[tree.perm]
    lo, hi = ranges[rank]
    tex = torch_exchange()

    def exchange(send, recv_len):  # numpy buffers over the torch point-to-point batch
        got = tex({r: torch.from_numpy(np.ascontiguousarray(b)) for r, b in send.items()}, recv_len)
        return {r: t.numpy() for r, t in got.items()}

    def allreduce(v):
        t = torch.from_numpy(v)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)

    # NaN poison: phase 1 may only read what the protocol delivered
    ys_own = distributed_matvec_halo(xs[lo:hi].copy(), len(xs), tot, plan,
                                     _np_phase(tree, topo, ops, off), exchange, allreduce,
                                     lambda n: np.zeros(n), np.concatenate, poison=np.nan)
    ref = O.h2_matvec(ops, x)[tree.perm][lo:hi]
    rel = float(np.linalg.norm(ys_own - ref) / np.linalg.norm(ref))
    q.put((rank, rel, plan.volume(), len(xs), tot, sorted(plan.x_send), sorted(plan.x_recv)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_matvec_gloo(world):
    """Halo-exchange protocol (HaloPlan / distributed_matvec_halo): x and the
    result stay distributed; neighbour-leaf x and interaction-list multipoles
    travel point to point, only the clusters spanning ranks are all-reduced.
    Everything the protocol did not deliver is NaN before phase 1, so a finite
    exact result proves the plan is sufficient; the traffic must be a fraction
    of the two full-length all-reduces it replaces."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_halo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for rank, rel, vol, n, tot, snd, rcv in out:
        assert np.isfinite(rel) and rel < 1e-13, (rank, rel)
        assert snd == rcv  # neighbour relation is symmetric
        assert 0 < vol[0] < n and vol[1] < tot and vol[2] < tot
    # sends and receives match pairwise
    total_sent = sum(o[2][0] + o[2][1] for o in out)
    assert total_sent > 0


def test_halo_plan_single_rank_is_empty():
    O, tree, topo, ops = _oracle_setup()
    off, tot = _offsets(tree, ops)
    nc = tree.n_clusters
    leaves = list(tree.leaves())
    plan = HaloPlan(tree.start, tree.stop, tree.level, tree.depth, leaves, topo.neighbors,
                    topo.interactions, [off.get(c, -1) for c in range(nc)],
                    [int(ops.rank.get(c, 0)) if c in off else 0 for c in range(nc)],
                    [(0, len(tree.points))], 0)
    assert plan.volume() == (0, 0, 0) and not plan.shared and not plan.x_recv and not plan.y_recv
