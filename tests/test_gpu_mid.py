"""Mid-size parity against the UNMODIFIED reference (tests/golden/mid/,
make_golden_mid.py): fill compression at merged (non-leaf) 3D levels and the
full c2 configuration.

schedule="reference" (Morton cluster order, the reference's PCG64 sketch
stream): on the 3D cases every per-level statistic is exact and
|x - x_ref| <= 10 eps.  c2 (eps = 1e-10) has decisions that the reference
itself flips between rng seeds (tests/golden/mid_seed1/: 192 of 16,314 pair
decisions and |x_seed0 - x_seed1| = 1.8e-5); there the gate is the
reference's own variability: statistics within its seed spread and
|x - x_ref| <= 2 x |x_seed0 - x_seed1|."""

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
def test_c2_full_within_reference_variability(schedule):
    g, fct, x = _run("c2_exp2d_n65536", schedule)
    s1 = dict(np.load(os.path.join(os.path.dirname(MID), "mid_seed1", "c2_exp2d_n65536.npz")))
    var = np.linalg.norm(s1["x"] - g["x"]) / np.linalg.norm(g["x"])
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    print(f"c2 {schedule}: |x - x_ref| = {rel:.3e}; reference seed0 vs seed1 {var:.3e}")
    assert rel <= 2.0 * var, (rel, var)
    st = fct.stats
    # leaf level: exact; merged levels: within the reference's seed spread
    assert st.levels[0].compressed_pairs == int(g["lv_compressed"][0])
    assert sum(st.levels[0].ranks) == int(g["lv_ranksum"][0])
    for i in range(1, len(st.levels)):
        spread = abs(int(s1["lv_compressed"][i]) - int(g["lv_compressed"][i]))
        assert abs(st.levels[i].compressed_pairs - int(g["lv_compressed"][i])) <= 4 * max(spread, 1)
        rspread = abs(int(s1["lv_ranksum"][i]) - int(g["lv_ranksum"][i]))
        assert abs(sum(st.levels[i].ranks) - int(g["lv_ranksum"][i])) <= 4 * max(rspread, 1)
    assert st.peak_edges == int(g["peak_edges"])
