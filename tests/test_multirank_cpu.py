"""World-size-2 gloo test of the bench's multi-rank timing reduction
(max over ranks) and of replica independence (each rank's host-side tree is
identical)."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import reduce_max
    import paper_1508_01835_b200 as P
    t = reduce_max([1.0 + rank, 5.0 - rank], device="cpu")
    pts = np.random.Generator(np.random.PCG64(1)).uniform(size=(2000, 3))
    tree, perm = P.build_octree(pts, 32)
    q.put((rank, t, int(perm[:50].sum()), tree.depth))
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert out[0][1] == out[1][1] == [2.0, 5.0]
    assert out[0][2:] == out[1][2:]
