"""The reference's own public-API behaviours (pkg/tests/test_factor.py,
test_h2.py, test_lowrank.py, graph.py attributes) through the drop-in, on the
device: lossless factorization equals the dense H2 solve, single-leaf trees
are a dense LU, zero rhs / linearity, bitwise determinism across
REFACTORIZATIONS of a copied graph, SingularPivotError through factorize,
graph inspection views, event log tags, and the lowrank primitives against
the reference's known answers."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _setup(P, n_points=400, seed=5, d=1e-2, n=2, leaf_target=12, depth=None, eps=0.0):
    pts = P.cube_uniform(n_points, seed=seed).points
    kern = P.benchmark_kernel(d)
    tree, _ = P.build_octree(pts, leaf_target, depth=depth)
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, kern, n, epsilon=eps)
    P.initialize_weights(ops, topo)
    return pts, kern, tree, topo, ops


@pytest.mark.parametrize("schedule", ["reference", "wavefront", "colored"])
@pytest.mark.parametrize("n_points,leaf_target", [(400, 12), (500, 3)])
def test_lossless_equals_h2_dense_solve(n_points, leaf_target, schedule):
    """test_factor.py:37-46."""
    import paper_1508_01835_b200 as P
    pts, kern, tree, topo, ops = _setup(P, n_points, leaf_target=leaf_target)
    fct = P.factorize(P.assemble_extended_graph(ops), epsilon=1e-13, seed=0, schedule=schedule)
    b = np.random.default_rng(1).standard_normal(n_points)
    x = fct.solve(b)
    xt = np.linalg.solve(P.h2_dense(ops), b[tree.perm])
    x_ref = np.empty_like(xt)
    x_ref[tree.perm] = xt
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-9


def test_single_leaf_is_dense_lu():
    """test_factor.py:68-76."""
    import paper_1508_01835_b200 as P
    pts, kern, tree, topo, ops = _setup(P, 100, depth=0, leaf_target=500)
    fct = P.factorize(P.assemble_extended_graph(ops), epsilon=1e-3, seed=0)
    b = np.random.default_rng(3).standard_normal(100)
    x = fct.solve(b)
    from paper_1508_01835_b200.dense import dense_matrix
    x_ref = np.linalg.solve(dense_matrix(pts, kern), b)
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) < 1e-10
    assert fct.top_sizes == [100] and len(fct.events) == 0


def test_zero_rhs_and_linearity():
    """test_factor.py:79-92."""
    import paper_1508_01835_b200 as P
    pts, kern, tree, topo, ops = _setup(P, 300)
    fct = P.factorize(P.assemble_extended_graph(ops), epsilon=1e-4, seed=0)
    assert np.array_equal(fct.solve(np.zeros(300)), np.zeros(300))
    b1, b2 = np.random.default_rng(4).standard_normal((2, 300))
    lhs = fct.solve(1.7 * b1 - 0.3 * b2)
    rhs = 1.7 * fct.solve(b1) - 0.3 * fct.solve(b2)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(lhs) < 1e-10


@pytest.mark.parametrize("schedule", ["reference", "wavefront", "colored"])
def test_refactorization_bitwise_deterministic(schedule):
    """test_factor.py:95-106: an independent factorize with the same seed is
    bitwise identical (here: of a device copy of the graph, and of a freshly
    assembled one)."""
    import paper_1508_01835_b200 as P
    pts, kern, tree, topo, ops = _setup(P, 2000, leaf_target=20, n=3, d=1e-3)
    b1, b2 = np.random.default_rng(5).standard_normal((2, 2000))
    g = P.assemble_extended_graph(ops)
    g2 = g.copy()
    f1 = P.factorize(g, epsilon=1e-6, seed=7, schedule=schedule)
    x1, x2 = f1.solve(b1), f1.solve(b2)
    assert np.array_equal(f1.solve(b1), x1)
    f2 = P.factorize(g2, epsilon=1e-6, seed=7, schedule=schedule)
    assert np.array_equal(f2.solve(b1), x1) and np.array_equal(f2.solve(b2), x2)
    f3 = P.factorize(P.assemble_extended_graph(ops), epsilon=1e-6, seed=7, schedule=schedule)
    assert np.array_equal(f3.solve(b1), x1)
    assert [s.compressed_pairs for s in f3.stats.levels] == [s.compressed_pairs for s in f1.stats.levels]


def test_singular_pivot_through_factorize():
    """test_factor.py:303-316: a zero kernel raises SingularPivotError."""
    import paper_1508_01835_b200 as P
    pts = P.cube_uniform(200, seed=10).points
    tree, _ = P.build_octree(pts, leaf_target=20)
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, P.zero_kernel(), 1)
    P.initialize_weights(ops, topo)
    with pytest.raises(P.SingularPivotError) as ei:
        P.factorize(P.assemble_extended_graph(ops), epsilon=1e-3, seed=0)
    assert "cluster" in str(ei.value.what) or "top-level" in str(ei.value.what)


def test_dropped_fill_means_no_rebase_and_peak_edges():
    """test_factor.py:319-338."""
    import paper_1508_01835_b200 as P
    pts, kern, tree, topo, ops = _setup(P, 300, leaf_target=6)
    fct = P.factorize(P.assemble_extended_graph(ops), epsilon=0.9, seed=0)
    assert all(ev[0] != "rebase" for ev in fct.events)
    assert all(ls.compressed_pairs == 0 for ls in fct.stats.levels)
    pts, kern, tree, topo, ops = _setup(P, 400, leaf_target=8)
    g = P.assemble_extended_graph(ops)
    initial = g.num_edges
    fct = P.factorize(g, epsilon=1e-4, seed=0)
    assert initial <= fct.stats.peak_edges <= 400 * tree.n_clusters
    assert fct.stats.n_clusters == tree.n_clusters
    tags = {ev[0] for ev in fct.events}
    assert tags <= {"elim", "rebase", "merge"} and "elim" in tags
    n_elim = sum(1 for ev in fct.events if ev[0] == "elim")
    assert n_elim == sum(len(tree.levels[l]) for l in range(2, tree.depth + 1))
    assert sum(fct.timings[k] for k in ("lu_and_triangular_solves", "matmul_updates",
                                        "lowrank_approximations", "operator_transfer")) > 0


def test_graph_views_match_oracle():
    """graph.py:30-216 attributes vs the numpy oracle's graph of the same
    operators (structure exact, blocks to rounding), apply vs dense_matrix."""
    import paper_1508_01835_b200 as P
    from oracle import ifmm_np as O
    g0 = load_golden("imq3d_n2048")
    tree, _ = P.build_octree(g0["points"], int(g0["leaf"]))
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, P.imq_kernel(float(g0["h"])), int(g0["n"]),
                                epsilon=float(g0["eps"]))
    P.initialize_weights(ops, topo)
    g = P.assemble_extended_graph(ops, b=g0["b"])
    ot, otp, oops = O.pipeline(g0["points"], O.imq_block(float(g0["h"])), int(g0["leaf"]),
                               int(g0["n"]), float(g0["eps"]))
    og = O.Graph(oops)
    assert g.sizes == list(og.sizes)
    assert set(g.edges.keys()) == set(og.E.keys())
    assert g.num_edges == len(og.E) and g.dim == sum(og.sizes)
    assert g.kinds[:3] == ["x", "x", "x"] and g.kinds[-1] == "y"
    for c, nid in g.node_x.items():
        assert g.cluster_of[nid] == c and g.sizes[nid] == tree.clusters[c].size
    w = np.random.default_rng(2).standard_normal(g.dim)
    E = g.dense_matrix()
    np.testing.assert_allclose(g.apply(w), E @ w, rtol=0, atol=1e-12 * np.abs(E @ w).max())
    np.testing.assert_allclose(g.apply_transpose(w), E.T @ w, rtol=0,
                               atol=1e-12 * np.abs(E.T @ w).max())
    assert np.count_nonzero(g.full_rhs()) == 2048
    pat = g.sparsity_pattern()
    assert len(pat["nodes"]) == len(g.sizes) and len(pat["edges"]) == g.num_edges
    gc = g.copy()
    np.testing.assert_array_equal(gc.dense_matrix(), E)
    P.factorize(g, 1e-6)
    with pytest.raises(ValueError):
        g.sizes


def test_lowrank_primitives_known_answers():
    """lowrank.py public functions vs the reference's KATs (kat_lowrank) and
    test_lowrank.py properties."""
    import paper_1508_01835_b200 as P
    k = load_golden("kat_lowrank")
    fa = P.aca_svd(k["A"], 1e-3)
    np.testing.assert_allclose(fa.sigma, k["aca_s"], rtol=1e-9)
    np.testing.assert_allclose(fa.matrix(), (k["aca_U"] * k["aca_s"]) @ k["aca_V"].T, atol=1e-10)
    bu = P.weighted_basis_union(k["B"], k["w"], k["F"], k["wf"], 1e-2)
    assert bu.rank == k["bu_basis"].shape[1]
    np.testing.assert_allclose(bu.new_weights, k["bu_w"], rtol=1e-10)
    np.testing.assert_allclose(bu.new_basis @ bu.old_map, k["bu_basis"] @ k["bu_old"], atol=1e-10)
    np.testing.assert_allclose(bu.new_basis @ bu.fillin_map, k["bu_basis"] @ k["bu_fill"],
                               atol=1e-10)
    ts = P.truncated_svd(k["A"], 1e-2)
    np.testing.assert_allclose(ts.sigma, k["ts_s"], rtol=1e-10)
    np.testing.assert_allclose(ts.U.T @ ts.U, np.eye(ts.rank), atol=1e-12)
    assert P.truncated_svd(np.zeros((4, 0)), 1.0).rank == 0
    rng = np.random.Generator(np.random.PCG64(7))
    M = rng.standard_normal((120, 9)) @ np.diag(10.0 ** -np.arange(9)) @ rng.standard_normal((9, 90))
    f = P.randomized_svd_dense(M, 1e-6, rng=np.random.Generator(np.random.PCG64(1)))
    s = np.linalg.svd(M, compute_uv=False)
    assert f.rank == int(np.sum(s > 1e-6))
    np.testing.assert_allclose(f.sigma, s[:f.rank], rtol=1e-8)
    assert np.linalg.norm(M - f.matrix(), 2) <= 1e-5
    assert P.rank_from_reference(np.array([3.0, 1.0, 0.1]), 0.1, 5.0) == 2
    with pytest.raises(ValueError):
        P.rank_from_reference(np.ones(2), 1.5, 1.0)
    with pytest.raises(ValueError):
        P.weighted_basis_union(k["B"], -k["w"], k["F"], k["wf"], 1e-2)
    with pytest.raises(ValueError):
        P.randomized_svd(lambda X: X, lambda X: X, 3, 3, 0.1, oversample=1)


def test_block_diag_preconditioner_and_dense():
    """krylov.py:172-196 and dense.py on the device."""
    import paper_1508_01835_b200 as P
    pts = P.cube_uniform(300, seed=2).points
    K = P.benchmark_kernel(1e-2)
    from paper_1508_01835_b200.dense import dense_matrix
    A = dense_matrix(pts, K)
    np.testing.assert_allclose(A, K.block(pts, pts), rtol=1e-14, atol=1e-15)
    pre = P.block_diag_preconditioner(A, 64)
    v = np.random.default_rng(0).standard_normal(300)
    out = pre(v)
    for a in range(0, 300, 64):
        b = min(300, a + 64)
        np.testing.assert_allclose(A[a:b, a:b] @ out[a:b], v[a:b], atol=1e-10)
    with pytest.raises(ValueError):
        P.block_diag_preconditioner(A, 0)
    prob = P.assemble_dense(P.cube_uniform(200, seed=3), K, seed=1)
    x = P.dense_solve(prob)
    assert np.linalg.norm(x - prob.x_true) / np.linalg.norm(prob.x_true) < 1e-8
    with pytest.raises(ValueError):
        P.assemble_dense(P.cube_uniform(200, seed=3), K, cap=100)
