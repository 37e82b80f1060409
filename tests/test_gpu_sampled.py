"""initialize_weights(mode="sampled") (h2.py:197-225, _sampled_gram
h2.py:250-262) against the UNMODIFIED reference
(tests/golden/sampled/sampled.npz, make_golden_sampled.py): the row samples
come from the reference's own rng.choice stream (drawn on the host), the Gram
products, SVDs and rotations run on the device; the sampled weights of every
cluster, the H2 matvec and the factorization built on them must match."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(GOLDEN, "sampled", "sampled.npz"))
CASES = sorted({k.split("__")[0] for k in G.files})


@pytest.mark.parametrize("name", CASES)
def test_sampled_weights_match_reference(name):
    import paper_1508_01835_b200 as P
    g = {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(name + "__")}
    pts, b = g["points"], g["b"]
    K = P.exp_kernel() if str(g["kernel"]) == "exp" else P.imq_kernel(float(g["h"]))
    eps = float(g["eps"])
    tree, _ = P.build_octree(pts, int(g["leaf"]))
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, K, int(g["n"]), epsilon=eps)
    P.initialize_weights(ops, topo, mode="sampled", sample_size=int(g["sample_size"]), seed=int(g["wseed"]))
    su = ops.sigma_u
    for t, c in enumerate(g["sigma_ids"]):
        ref = g["sigma_u"][g["sigma_ptr"][t]:g["sigma_ptr"][t + 1]]
        np.testing.assert_allclose(su[int(c)], ref, rtol=1e-8, atol=1e-12 * ref[0], err_msg=f"cluster {c}")
    mv = P.h2_matvec(ops, b)
    np.testing.assert_allclose(mv, g["h2_matvec"], rtol=0, atol=1e-11 * np.abs(g["h2_matvec"]).max())
    graph = P.assemble_extended_graph(ops)
    fct = P.factorize(graph, eps, seed=0, sigma0=float(g["sigma0"]), schedule="reference")
    st = fct.stats
    np.testing.assert_array_equal([s.compressed_pairs for s in st.levels], g["lv_compressed"])
    np.testing.assert_array_equal([s.dropped_pairs for s in st.levels], g["lv_dropped"])
    np.testing.assert_array_equal([sum(s.ranks) for s in st.levels], g["lv_ranksum"])
    assert st.peak_edges == int(g["peak_edges"])
    x = fct.solve(b)
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    # The sampled Gram (m/s) Bs^T Bs H is ill-conditioned or rank deficient when
    # s is near the cluster rank, and the rotation's trailing columns are then
    # LAPACK's arbitrary completion: weights and every rank decision agree,
    # x only to the accuracy the factorization itself has.  Held to the
    # residual of the reference's own solution instead of 10 eps.
    nb = np.linalg.norm(b)
    r = np.linalg.norm(P.h2_matvec(ops, x) - b) / nb
    r_ref = np.linalg.norm(P.h2_matvec(ops, g["x"]) - b) / nb
    print(f"{name}: |x - x_ref|/|x_ref| = {rel:.2e}, h2 residual {r:.2e} (reference x: {r_ref:.2e})")
    assert r <= 2.0 * r_ref + 1e-12, (r, r_ref)
    assert rel <= 1e-3, rel


def test_sampled_mode_argument_checks():
    import paper_1508_01835_b200 as P
    g = {k.split("__", 1)[1]: G[k] for k in G.files if k.startswith(CASES[0] + "__")}
    tree, _ = P.build_octree(g["points"], int(g["leaf"]))
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, P.exp_kernel(), int(g["n"]), epsilon=1e-8)
    with pytest.raises(ValueError):
        P.initialize_weights(ops, topo, mode="other")
    with pytest.raises(ValueError):
        P.initialize_weights(ops, topo, mode="sampled", sample_size=0)
