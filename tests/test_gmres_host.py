"""gmres (krylov.py:32-116) called with numpy operands -- the reference
harness's call -- vs the oracle's restatement (the Arnoldi loop runs on the
device, so these are GPU tests), and its argument errors (CPU)."""

import numpy as np
import pytest


@pytest.mark.gpu
@pytest.mark.parametrize("side", ["none", "right", "left"])
def test_gmres_numpy_matches_oracle(side):
    import paper_1508_01835_b200 as P
    from oracle import ifmm_np as O
    rng = np.random.default_rng(5)
    n = 120
    A = rng.standard_normal((n, n)) / np.sqrt(n) + 2.0 * np.eye(n)
    d = 1.0 / np.diag(A)
    b = rng.standard_normal(n)
    pre = (lambda v: d * v) if side != "none" else None
    x_ref, its, hist, conv = O.gmres(lambda v: A @ v, b, tol=1e-12, max_iters=100, precond=pre,
                                     side=side)
    x, tr = P.gmres(lambda v: A @ v, b, tol=1e-12, max_iters=100, precond=pre, side=side)
    assert tr.iterations == its and tr.converged == conv
    np.testing.assert_allclose(tr.residual_history, hist, rtol=1e-8, atol=1e-15)
    assert np.linalg.norm(x - x_ref) <= 1e-12 * np.linalg.norm(x_ref)
    assert np.linalg.norm(A @ x - b) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.gpu
def test_gmres_zero_rhs_and_breakdown():
    import paper_1508_01835_b200 as P
    x, tr = P.gmres(lambda v: 2.0 * v, np.zeros(5))
    assert tr.converged and tr.iterations == 0 and not x.any()
    # A = 2I: the Krylov space is exhausted after one step (exact solve)
    b = np.arange(1.0, 6.0)
    x, tr = P.gmres(lambda v: 2.0 * v, b)
    assert tr.converged and tr.iterations == 1
    np.testing.assert_allclose(x, b / 2.0, rtol=1e-15)


def test_gmres_argument_errors():
    import paper_1508_01835_b200 as P
    with pytest.raises(ValueError):
        P.gmres(lambda v: v, np.ones(3), tol=0.0)
    with pytest.raises(ValueError):
        P.gmres(lambda v: v, np.ones(3), max_iters=0)
    with pytest.raises(ValueError):
        P.gmres(lambda v: v, np.ones(3), precond=lambda v: v, side="middle")
