"""BASELINE-size parity (c3: 3D N=262,144 IMQ, eps=1e-6) against the oracle
run with reference semantics (tests/golden/large/, written by
tests/golden/make_large_stats.py -- 53 min on one CPU core).

Gates: tree, H2 ranks (sum), leaf-level fill statistics and peak edges
exact; relative residual against the EXACT matvec within 2x the
reference's (north star); x within the reference's own variability.

Why not "x within 10 eps" at this size: the reference's x itself moves by
9.4e-3 between factorize rng seeds 0 and 1 (rSVD sketches of fills with
min(shape) > 64, factor.py:329-332), see tests/golden/large/c3_seed1_*.
Upper-level fill statistics are reported, not gated, for the same reason."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c3_parity_against_reference_semantics():
    import paper_1508_01835_b200 as P
    from oracle.ifmm_np import config_inputs  # seeded inputs only
    st = json.load(open(os.path.join(GOLDEN, "large", "c3_stats.json")))
    x_ref = np.load(os.path.join(GOLDEN, "large", "c3_x.npy"))
    inp = config_inputs("c3")
    tree, _ = P.build_octree(inp["points"], inp["leaf"])
    assert tree.depth == st["depth"]
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, P.imq_kernel(inp["kernel"][1]["h"]), inp["n"],
                                epsilon=inp["eps"])
    assert sum(ops.rank.values()) == st["ranks_sum"]
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops, consume=True)
    fct = P.factorize(graph, inp["eps"], seed=0, sigma0=st["sigma0"])
    lv = fct.stats.levels
    leaf = st["levels"][0]
    assert [lv[0].level, lv[0].compressed_pairs, lv[0].dropped_pairs, lv[0].added,
            sum(lv[0].ranks)] == leaf[:5]
    assert fct.stats.peak_edges == st["peak_edges"]
    x = fct.solve(inp["b"])
    b = inp["b"]
    K = P.imq_kernel(inp["kernel"][1]["h"])
    res = float(np.linalg.norm(P.exact_matvec(inp["points"], K, x) - b) / np.linalg.norm(b))
    res_ref = float(np.linalg.norm(P.exact_matvec(inp["points"], K, x_ref) - b) / np.linalg.norm(b))
    x_s1 = np.load(os.path.join(GOLDEN, "large", "c3_seed1_x.npy"))
    var_ref = float(np.linalg.norm(x_s1 - x_ref) / np.linalg.norm(x_ref))
    rel = float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
    print(f"c3 |x - x_ref|/|x_ref| = {rel:.3e} (reference seed0 vs seed1: {var_ref:.3e}); "
          f"exact residual ours {res:.4e} ref {res_ref:.4e}; levels ours "
          f"{[(s.level, s.compressed_pairs, s.dropped_pairs, sum(s.ranks)) for s in lv]} "
          f"ref {[tuple(v[:3]) + (v[4],) for v in st['levels']]}")
    assert res <= 2.0 * res_ref, (res, res_ref)
    assert rel <= 5.0 * var_ref, (rel, var_ref)
