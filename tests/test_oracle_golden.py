"""Pin the numpy oracle (oracle/ifmm_np.py) against the reference's own
outputs (tests/golden/*.npz written by tests/golden/make_golden.py)."""

import numpy as np
import pytest

from conftest import csr_lists, golden_names, load_golden
from oracle import ifmm_np as O

CASES = golden_names()


def _block(g):
    if str(g["kernel"]) == "exp":
        return O.exp_block
    return O.imq_block(float(g["h"]))


@pytest.mark.parametrize("name", CASES)
def test_tree_topology_bitexact(name):
    g = load_golden(name)
    tree = O.build_tree(g["points"], int(g["leaf"]))
    topo = O.build_topology(tree)
    assert tree.depth == int(g["depth"])
    np.testing.assert_array_equal(tree.perm, g["perm"])
    np.testing.assert_array_equal(tree.level, g["cl_level"])
    np.testing.assert_array_equal(tree.start, g["cl_start"])
    np.testing.assert_array_equal(tree.stop, g["cl_stop"])
    np.testing.assert_array_equal(tree.parent, g["cl_parent"])
    np.testing.assert_array_equal(tree.cell, g["cl_cell"])
    assert topo.neighbors == csr_lists(g["nbr_ptr"], g["nbr_idx"])
    assert topo.interactions == csr_lists(g["int_ptr"], g["int_idx"])


@pytest.mark.parametrize("name", CASES)
def test_factorize_solve_matches_reference(name):
    g = load_golden(name)
    eps = float(g["eps"])
    tree, topo, ops = O.pipeline(g["points"], _block(g), int(g["leaf"]), int(g["n"]), eps)
    ranks = np.array([ops.rank.get(c, -1) for c in range(tree.n_clusters)])
    np.testing.assert_array_equal(ranks, g["ranks"])
    for i, c in enumerate(g["su_keys"]):
        w = g["su_val"][g["su_ptr"][i]:g["su_ptr"][i + 1]]
        np.testing.assert_allclose(ops.sigma_u[int(c)], w, rtol=1e-9, atol=1e-12 * w[0])
    y = O.h2_matvec(ops, g["b"])
    assert np.linalg.norm(y - g["y_h2"]) <= 1e-12 * np.linalg.norm(g["y_h2"])
    graph = O.Graph(ops)
    s0 = O.sigma0_estimate(graph, seed=0)
    assert abs(s0 - float(g["sigma0"])) <= 1e-9 * s0
    fct = O.factorize(graph, eps, seed=0, sigma0=float(g["sigma0"]))
    np.testing.assert_array_equal([s.level for s in fct.levels], g["lv_level"])
    np.testing.assert_array_equal([s.compressed_pairs for s in fct.levels], g["lv_compressed"])
    np.testing.assert_array_equal([s.dropped_pairs for s in fct.levels], g["lv_dropped"])
    np.testing.assert_array_equal([s.added for s in fct.levels], g["lv_added"])
    np.testing.assert_array_equal([sum(s.ranks) for s in fct.levels], g["lv_ranksum"])
    assert fct.peak_edges == int(g["peak_edges"])
    np.testing.assert_array_equal(fct.top_sizes, g["top_sizes"])
    x = fct.solve(g["b"])
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    assert rel <= 10 * max(eps, 1e-12), rel


def test_lowrank_kats():
    k = load_golden("kat_lowrank")
    fa = O.aca(k["A"], 1e-3)
    np.testing.assert_allclose(fa.s, k["aca_s"], rtol=1e-12)
    np.testing.assert_allclose(np.abs(fa.U.T @ k["aca_U"]), np.eye(len(fa.s)), atol=1e-9)
    u = O.basis_union(k["B"], k["w"], k["F"], k["wf"], 1e-2)
    np.testing.assert_allclose(u.weights, k["bu_w"], rtol=1e-12)
    np.testing.assert_allclose(u.basis @ u.old_map, k["bu_basis"] @ k["bu_old"], atol=1e-12)
    np.testing.assert_allclose(u.basis @ u.fill_map, k["bu_basis"] @ k["bu_fill"], atol=1e-12)
    np.testing.assert_allclose(O.svd_trunc(k["A"], 1e-2).s, k["ts_s"], rtol=1e-12)
