"""BASELINE-size parity: c3 (3D N=262,144 IMQ, eps=1e-6) against the
UNMODIFIED reference run on the same seeded inputs (tests/golden/mid/
c3_imq3d_n262144.npz, make_golden_mid.py: 42 min of CPU).

Gates: tree (perm checksum, neighbour / interaction counts), H2 ranks and
the leaf-level fill statistics exact; levels 3 and 2 within 3x the
reference's own variability (its compressed-pair count moves by 43 at level
3 between factorize rng seeds, tests/golden/large/c3_seed1_stats.json);
|x - x_ref| within 2x the reference's seed-to-seed |x| variability (9.4e-3,
tests/golden/large/c3_seed1_x.npy); relative residual against the EXACT
matvec within 2x the reference's (north star)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN
from golden_mid import load_mid, mid_inputs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("schedule", ["reference"])
def test_c3_parity_against_reference(schedule):
    import paper_1508_01835_b200 as P
    g = load_mid("c3_imq3d_n262144")
    pts, b, K = mid_inputs(P, g)
    eps = float(g["eps"])
    tree, perm = P.build_octree(pts, int(g["leaf"]))
    assert tree.depth == int(g["depth"])
    assert int((np.asarray(perm, dtype=np.int64) * np.arange(1, len(perm) + 1)).sum()) == int(g["perm_checksum"])
    topo = P.compute_topology(tree)
    np.testing.assert_array_equal([len(x) for x in topo.neighbors], g["n_neighbors"])
    np.testing.assert_array_equal([len(x) for x in topo.interactions], g["n_interactions"])
    ops = P.chebyshev_operators(tree, topo, K, int(g["n"]), epsilon=eps)
    np.testing.assert_array_equal([ops.rank.get(c, -1) for c in range(tree.n_clusters)], g["ranks"])
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops, consume=True)
    fct = P.factorize(graph, eps, seed=0, sigma0=float(g["sigma0"]), schedule=schedule)
    lv = fct.stats.levels
    assert (lv[0].level, lv[0].compressed_pairs, lv[0].dropped_pairs, lv[0].added, sum(lv[0].ranks)) == \
        (int(g["lv_level"][0]), int(g["lv_compressed"][0]), int(g["lv_dropped"][0]),
         int(g["lv_added"][0]), int(g["lv_ranksum"][0]))
    assert fct.stats.peak_edges == int(g["peak_edges"])
    seed1 = json.load(open(os.path.join(GOLDEN, "large", "c3_seed1_stats.json")))
    s0 = json.load(open(os.path.join(GOLDEN, "large", "c3_stats.json")))
    for i in (1, 2):
        spread = abs(seed1["levels"][i][1] - s0["levels"][i][1])
        assert abs(lv[i].compressed_pairs - int(g["lv_compressed"][i])) <= 3 * max(spread, 10), \
            (lv[i].level, lv[i].compressed_pairs, int(g["lv_compressed"][i]), spread)
    x = fct.solve(b)
    x_s1 = np.load(os.path.join(GOLDEN, "large", "c3_seed1_x.npy"))
    var_ref = float(np.linalg.norm(x_s1 - g["x"]) / np.linalg.norm(g["x"]))
    rel = float(np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]))
    nb = np.linalg.norm(b)
    res = float(np.linalg.norm(P.exact_matvec(pts, K, x) - b) / nb)
    res_ref = float(np.linalg.norm(P.exact_matvec(pts, K, g["x"]) - b) / nb)
    print(f"c3 {schedule}: |x - x_ref|/|x_ref| = {rel:.3e} (reference seed0 vs seed1: {var_ref:.3e}); "
          f"exact residual ours {res:.4e} ref {res_ref:.4e}; levels ours "
          f"{[(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in lv]} "
          f"ref {g['lv_compressed'].tolist()} / {g['lv_ranksum'].tolist()}")
    assert res <= 2.0 * res_ref, (res, res_ref)
    assert rel <= 2.0 * var_ref, (rel, var_ref)


def test_c3_colored_schedule_residual():
    """c3 through schedule="colored" (relaxed elimination order):
    gated by the north-star residual criterion only (exact-matvec residual <=
    2x the unmodified reference's)."""
    import paper_1508_01835_b200 as P
    g = load_mid("c3_imq3d_n262144")
    pts, b, K = mid_inputs(P, g)
    eps = float(g["eps"])
    tree, perm = P.build_octree(pts, int(g["leaf"]))
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, K, int(g["n"]), epsilon=eps)
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops, consume=True)
    fct = P.factorize(graph, eps, seed=0, sigma0=float(g["sigma0"]), schedule="colored")
    assert fct.stats.peak_edges == int(g["peak_edges"])
    x = fct.solve(b)
    nb = np.linalg.norm(b)
    res = float(np.linalg.norm(P.exact_matvec(pts, K, x) - b) / nb)
    res_ref = float(np.linalg.norm(P.exact_matvec(pts, K, g["x"]) - b) / nb)
    print(f"c3 colored: exact residual ours {res:.4e} ref {res_ref:.4e}; levels "
          f"{[(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in fct.stats.levels]}")
    assert res <= 2.0 * res_ref, (res, res_ref)


def _list_checksum(lists):
    M = (1 << 61) - 1
    acc = 0
    for i, l in enumerate(lists):
        a = np.asarray(l, dtype=np.int64)
        if len(a):
            acc = (acc + (i + 1) * int(((a + 1) * np.arange(1, len(a) + 1)).sum() % M)) % M
    return acc


def test_c4_structure_and_ranks_against_reference():
    """c4 (the BASELINE headline config, N = 1,048,576): the reference cannot
    factorize it in the build container, so parity is pinned on what it does
    produce (tests/golden/make_golden_c4.py, unmodified reference): the tree
    and the interaction lists bit-exact, and every cluster's H2 rank from the
    reference's leaf / transfer reductions (h2.py:121-150) exact.  The engine
    then factorizes and solves it once; the size-independent properties the
    domain offers are checked: the leaf level drops every fill (Frobenius
    pre-filter == compression decision), repeated solves are bitwise equal, the
    solve is linear, and the exact-matvec residual is reported."""
    import torch
    import paper_1508_01835_b200 as P
    g = np.load(os.path.join(GOLDEN, "large", "c4_structure.npz"))
    N, eps = int(g["N"]), float(g["eps"])
    _, total = torch.cuda.mem_get_info()
    if total < 170 * 2**30:
        pytest.skip("c4 needs ~136 GB of device memory (arena + dedicated allocations)")
    pts = np.random.Generator(np.random.PCG64(int(g["seed"]))).uniform(0.0, 1.0, size=(N, 3))
    b = np.random.Generator(np.random.PCG64(int(g["seed"]) + 1)).standard_normal(N)
    tree, perm = P.build_octree(pts, int(g["leaf"]))
    assert tree.depth == int(g["depth"]) and tree.n_clusters == int(g["n_clusters"])
    assert int((np.asarray(perm, dtype=np.int64) * np.arange(1, N + 1)).sum()) == int(g["perm_checksum"])
    assert int(sum((i + 1) * (c.start + 3 * c.stop) for i, c in enumerate(tree.clusters))
               % ((1 << 61) - 1)) == int(g["range_checksum"])
    topo = P.compute_topology(tree)
    np.testing.assert_array_equal([len(x) for x in topo.neighbors], g["n_neighbors"])
    np.testing.assert_array_equal([len(x) for x in topo.interactions], g["n_interactions"])
    assert _list_checksum(topo.neighbors) == int(g["neighbors_checksum"])
    assert _list_checksum(topo.interactions) == int(g["interactions_checksum"])
    K = P.imq_kernel(N ** (-1.0 / 3.0))
    ops = P.chebyshev_operators(tree, topo, K, int(g["n"]), epsilon=eps)
    np.testing.assert_array_equal([ops.rank.get(c, -1) for c in range(tree.n_clusters)], g["ranks"])
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops, consume=True)
    fct = P.factorize(graph, eps, seed=0, schedule="wavefront")
    lv = fct.stats.levels
    assert lv[0].level == 5 and lv[0].compressed_pairs == 0 and lv[0].dropped_pairs > 4_000_000
    db = torch.from_numpy(b).cuda()
    x1, x2 = fct.solve(db), fct.solve(db)
    assert torch.equal(x1, x2)
    u = torch.from_numpy(np.random.default_rng(7).standard_normal(N)).cuda()
    lin = float(torch.linalg.norm(fct.solve(db + 0.5 * u) - x1 - 0.5 * fct.solve(u)) / torch.linalg.norm(x1))
    assert lin <= 1e-9, lin
    x = x1.cpu().numpy()
    res = float(np.linalg.norm(P.exact_matvec(pts, K, x) - b) / np.linalg.norm(b))
    print(f"c4: levels {[(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in lv]}; "
          f"exact-matvec residual {res:.3e} (eps*sigma0 = {eps * fct.sigma0:.3g}: the direct solve at this "
          f"absolute threshold is a preconditioner, not a solver); solve linearity defect {lin:.1e}")
    assert np.isfinite(res)
