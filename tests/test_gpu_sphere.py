"""c5 recipe (BASELINE configs[4]: points on the unit sphere, IMQ with
h = sqrt(4 pi / N), leaves <= 64, 4^3 Chebyshev nodes, eps = 1e-3; IFMM as
right preconditioner of GMRES on the H2 matvec, tol 1e-10) at reduced N
against the UNMODIFIED reference (tests/golden/sphere/, make_golden_sphere.py):
the device Arnoldi loop converges in the reference's iteration count (the
eps = 1e-3 preconditioner's randomised fills allow +-1), the residual history
follows the reference's, and the solution agrees to the GMRES tolerance."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sphere")


def c5_problem(P, N):
    pts = P.sphere_surface(N, 4).points
    h = float(np.sqrt(4.0 * np.pi / N))
    K = P.imq_kernel(h)
    b = np.random.Generator(np.random.PCG64(5)).standard_normal(N)
    return pts, K, b


def c5_solve(P, pts, K, b, eps=1e-3, schedule="reference", sigma0=None, device_rhs=True):
    import torch
    tree, _ = P.build_octree(pts, 64)
    topo = P.compute_topology(tree)
    ops = P.chebyshev_operators(tree, topo, K, 4, epsilon=eps)
    P.initialize_weights(ops, topo)
    graph = P.assemble_extended_graph(ops)
    if sigma0 is None:
        sigma0 = P.estimate_sigma0(graph, seed=0)
    fct = P.factorize(graph, eps, seed=0, sigma0=sigma0, schedule=schedule)
    rhs = torch.from_numpy(np.ascontiguousarray(b)).cuda() if device_rhs else b
    x, tr = P.gmres(lambda v: P.h2_matvec(ops, v), rhs, tol=1e-10, max_iters=500,
                    precond=fct.solve, side="right")
    if device_rhs:
        x = x.cpu().numpy()
    return tree, ops, fct, x, tr


@pytest.mark.parametrize("schedule", ["reference", "wavefront"])
@pytest.mark.parametrize("N", [4096, 16384])
def test_c5_reduced_matches_reference(N, schedule):
    import paper_1508_01835_b200 as P
    g = np.load(os.path.join(SPH, f"c5_n{N}.npz"))
    pts, K, b = c5_problem(P, N)
    tree, ops, fct, x, tr = c5_solve(P, pts, K, b, schedule=schedule, sigma0=float(g["sigma0"]))
    assert tree.depth == int(g["depth"])
    assert [s.compressed_pairs for s in fct.stats.levels] == g["lv_compressed"].tolist()
    assert tr.converged and bool(g["converged"])
    assert abs(tr.iterations - int(g["iterations"])) <= 1, (tr.iterations, int(g["iterations"]))
    k = min(len(tr.residual_history), len(g["history"])) - 1
    np.testing.assert_allclose(tr.residual_history[:k], g["history"][:k], rtol=0.5)
    # true residual of the returned x (GMRES stops on its recurrence residual;
    # the attainable true residual is set by the problem's conditioning) held
    # against the true residual of the reference's own solution
    nb = np.linalg.norm(b)
    r = np.linalg.norm(P.h2_matvec(ops, x) - b) / nb
    r_ref = np.linalg.norm(P.h2_matvec(ops, g["x"]) - b) / nb
    rel = np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"])
    print(f"c5 N={N} {schedule}: iterations {tr.iterations} (reference {int(g['iterations'])}), "
          f"|x - x_ref|/|x_ref| = {rel:.2e}, h2 residual {r:.2e} (reference x: {r_ref:.2e})")
    # the replay's compensated row sums keep the preconditioner linear to
    # rounding, so the true residual follows the recurrence residual as in the
    # reference (plain FMA sums left it at 1e-8 at N = 16,384)
    assert r <= 3.0 * max(r_ref, 1e-10), (r, r_ref)
    assert rel <= 1e-6, rel


def test_c5_host_rhs_same_iterations():
    """numpy b in, numpy x out (the reference harness's call, experiments.py:190-233)
    runs the same device loop."""
    import paper_1508_01835_b200 as P
    g = np.load(os.path.join(SPH, "c5_n4096.npz"))
    pts, K, b = c5_problem(P, 4096)
    _, ops, _, x, tr = c5_solve(P, pts, K, b, sigma0=float(g["sigma0"]), device_rhs=False)
    assert isinstance(x, np.ndarray)
    assert abs(tr.iterations - int(g["iterations"])) <= 1
    assert np.linalg.norm(x - g["x"]) <= 1e-6 * np.linalg.norm(g["x"])
