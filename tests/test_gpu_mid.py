"""Mid-size parity against the UNMODIFIED reference (tests/golden/mid/,
make_golden_mid.py): fill compression at merged (non-leaf) 3D levels and the
full c2 configuration.

Both schedules: on the 3D cases every per-level statistic is exact and
|x - x_ref| <= 10 eps.  c2 (eps = 1e-10): every statistic exact; x is
within 2e-6 of the reference's (10 eps = 1e-9 is below the rounding
amplification of this problem -- the reference's own x moves by 1.8e-5
between factorize rng seeds, tests/golden/mid_seed1/).  The slab (the c3
recipe on [0,1]^2 x [0,1/4]: leaf-level AND merged-level compression at 1/4
of c3's size) is exact at the leaf level; above it the reference itself is
chaotic -- rerun with 4 BLAS threads it changes 428 decisions and its x by
188 % (tests/golden/mid_seed1/imq_slab_n65536_blas4.npz) -- so only the leaf
level and the structure are gated there."""

import os

import numpy as np
import pytest

from golden_mid import MID, load_mid, mid_inputs

pytestmark = pytest.mark.gpu

CASES_3D = ["imq3d_n16384_leaf16", "imq3d_n32768", "imq3d_n32768_leaf8"]


def _run(name, schedule):
    import paper_1508_01835_b200 as P
    g = load_mid(name)
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
    graph = P.assemble_extended_graph(ops)
    fct = P.factorize(graph, eps, seed=0, sigma0=float(g["sigma0"]), schedule=schedule)
    x = fct.solve(b)
    return g, fct, x


@pytest.mark.parametrize("schedule", ["reference", "wavefront"])
@pytest.mark.parametrize("name", CASES_3D)
def test_mid_3d_exact(name, schedule):
    g, fct, x = _run(name, schedule)
    st = fct.stats
    np.testing.assert_array_equal([s.level for s in st.levels], g["lv_level"])
    np.testing.assert_array_equal([s.compressed_pairs for s in st.levels], g["lv_compressed"])
    np.testing.assert_array_equal([s.dropped_pairs for s in st.levels], g["lv_dropped"])
    np.testing.assert_array_equal([s.added for s in st.levels], g["lv_added"])
    np.testing.assert_array_equal([sum(s.ranks) for s in st.levels], g["lv_ranksum"])
    np.testing.assert_array_equal([s.max_rank for s in st.levels], g["lv_maxrank"])
    assert st.peak_edges == int(g["peak_edges"])
    assert st.max_basis_rank == int(g["max_basis_rank"])
    assert fct.top_sizes == g["top_sizes"].tolist()
    assert sum(1 for e in fct.events if e[0] == "rebase") == int(g["n_rebase"])
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    assert rel <= 10 * float(g["eps"]), rel


@pytest.mark.parametrize("schedule", ["reference", "wavefront"])
def test_c2_full_exact_statistics(schedule):
    g, fct, x = _run("c2_exp2d_n65536", schedule)
    st = fct.stats
    np.testing.assert_array_equal([s.compressed_pairs for s in st.levels], g["lv_compressed"])
    np.testing.assert_array_equal([s.dropped_pairs for s in st.levels], g["lv_dropped"])
    np.testing.assert_array_equal([sum(s.ranks) for s in st.levels], g["lv_ranksum"])
    assert st.peak_edges == int(g["peak_edges"])
    s1 = dict(np.load(os.path.join(os.path.dirname(MID), "mid_seed1", "c2_exp2d_n65536.npz")))
    var = np.linalg.norm(s1["x"] - g["x"]) / np.linalg.norm(g["x"])
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    print(f"c2 {schedule}: |x - x_ref| = {rel:.3e}; reference seed0 vs seed1 {var:.3e}")
    assert rel <= 2e-6, (rel, var)


@pytest.mark.parametrize("schedule", ["reference", "wavefront"])
def test_slab_leaf_level_exact(schedule):
    g, fct, x = _run("imq_slab_n65536", schedule)
    st = fct.stats
    lv = st.levels[0]
    assert lv.level == int(g["lv_level"][0])
    assert (lv.compressed_pairs, lv.dropped_pairs, lv.added, sum(lv.ranks)) == \
        (int(g["lv_compressed"][0]), int(g["lv_dropped"][0]), int(g["lv_added"][0]),
         int(g["lv_ranksum"][0]))
    assert [s.added for s in st.levels] == g["lv_added"].tolist()
    assert st.peak_edges == int(g["peak_edges"])


@pytest.mark.parametrize("name", CASES_3D + ["c2_exp2d_n65536"])
def test_colored_schedule_residual_criterion(name):
    """schedule="colored" (SURVEY.md 8e relaxed mode: one batched stage per
    colour of the cluster grid) changes the elimination ORDER, so statistics
    and x are not comparable with the reference's; it is held to the
    north-star residual criterion: the exact-matvec residual of its solution is
    within 2x the residual of the unmodified reference's solution, and the
    structure that does not depend on the order (peak edge count, top-level
    system) matches."""
    import paper_1508_01835_b200 as P
    g, fct, x = _run(name, "colored")
    pts, b, K = mid_inputs(P, g)
    nb = np.linalg.norm(b)
    res = float(np.linalg.norm(P.exact_matvec(pts, K, x) - b) / nb)
    res_ref = float(np.linalg.norm(P.exact_matvec(pts, K, g["x"]) - b) / nb)
    print(f"{name} colored: exact residual {res:.3e} (reference {res_ref:.3e}); compressed "
          f"{[s.compressed_pairs for s in fct.stats.levels]} ref {g['lv_compressed'].tolist()}")
    assert res <= 2.0 * res_ref + 1e-12, (res, res_ref)
    assert fct.stats.peak_edges == int(g["peak_edges"])
    x2 = _run(name, "colored")[2]
    assert np.array_equal(x, x2), "colored schedule is not run-to-run deterministic"
