"""Device GMRES (csrc/krylov.cu, krylov.py:32-116) vs numpy and the oracle's
gmres (oracle/ifmm_np.py, checker only) on the same seeded inputs (GPU only)."""

import ctypes as C

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _p(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("k1,n", [(0, 1), (1, 7), (5, 1000), (40, 65536 + 3), (3, 2_000_000),
                                  (0, 5_000_001), (4, 5_000_001)])
def test_mgs_step(k1, n):
    """h_i = <V_i, w>; w -= h_i V_i in order (krylov.py:73-75), h[k1] = ||w||
    (krylov.py:76), vs the same loop in numpy."""
    from paper_1508_01835_b200 import _native as N
    rng = np.random.default_rng(k1 * 31 + n)
    V = rng.standard_normal((max(k1, 1), n))
    if k1:
        V = np.linalg.qr(V.T)[0].T.copy() if n >= k1 else V
    w = rng.standard_normal(n)
    ref_w, ref_h = w.copy(), np.zeros(k1 + 1)
    for i in range(k1):
        ref_h[i] = V[i] @ ref_w
        ref_w = ref_w - ref_h[i] * V[i]
    ref_h[k1] = np.linalg.norm(ref_w)
    dV, dw = torch.from_numpy(V).cuda(), torch.from_numpy(w).cuda()
    h = np.zeros(k1 + 1)
    torch.cuda.synchronize()
    N.check(N.lib().ifmm_krylov_mgs(N.ctx(), _p(dV), n, k1, n, _p(dw), h.ctypes.data_as(C.c_void_p)))
    scale = np.linalg.norm(w)
    np.testing.assert_allclose(h, ref_h, rtol=0, atol=1e-13 * scale * max(1, np.sqrt(n) / 100))
    np.testing.assert_allclose(dw.cpu().numpy(), ref_w, rtol=0, atol=1e-13 * scale)
    # deterministic: a second run is bitwise identical
    dw2 = torch.from_numpy(w).cuda()
    h2 = np.zeros(k1 + 1)
    N.check(N.lib().ifmm_krylov_mgs(N.ctx(), _p(dV), n, k1, n, _p(dw2), h2.ctypes.data_as(C.c_void_p)))
    np.testing.assert_array_equal(h, h2)
    assert torch.equal(dw, dw2)


def test_div_combine_bitwise():
    """w / h (krylov.py:104) is bitwise numpy's; the combination
    (krylov.py:113) is the sequential sum u + y_i V_i, bitwise."""
    from paper_1508_01835_b200 import _native as N
    rng = np.random.default_rng(3)
    n, k = 4099, 9
    V, y, w = rng.standard_normal((k, n)), rng.standard_normal(k), rng.standard_normal(n)
    dV, dw = torch.from_numpy(V).cuda(), torch.from_numpy(w).cuda()
    out, u = torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty_like(dw)
    torch.cuda.synchronize()
    N.check(N.lib().ifmm_krylov_div(N.ctx(), _p(dw), n, 1.7, _p(out)))
    np.testing.assert_array_equal(out.cpu().numpy(), w / 1.7)
    N.check(N.lib().ifmm_krylov_combine(N.ctx(), _p(dV), n, k, y.ctypes.data_as(C.c_void_p), n,
                                        _p(u)))
    ref = np.zeros(n)
    for i in range(k):
        ref = ref + y[i] * V[i]
    np.testing.assert_array_equal(u.cpu().numpy(), ref)


def test_mgs_rejects_bad_arguments():
    from paper_1508_01835_b200 import _native as N
    h = np.zeros(2)
    d = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        N.check(N.lib().ifmm_krylov_mgs(N.ctx(), _p(d), 4, 1, 8, _p(d), h.ctypes.data_as(C.c_void_p)))


@pytest.mark.parametrize("side", ["none", "right", "left"])
def test_gmres_dense_vs_oracle(side):
    """Same SPD-ish system, same loop: iteration count and residual history
    match the oracle's numpy gmres; x within 1e-10 relative."""
    import paper_1508_01835_b200 as P
    from oracle import ifmm_np as O
    rng = np.random.default_rng(11)
    n = 300
    A = rng.standard_normal((n, n)) / np.sqrt(n) + 2.0 * np.eye(n)
    D = np.diag(1.0 / np.diag(A))
    b = rng.standard_normal(n)
    pre = (lambda v: D @ v) if side != "none" else None
    ref = O.gmres(lambda v: A @ v, b, tol=1e-12, max_iters=200, precond=pre, side=side)
    x_ref, its_ref, hist_ref = ref[0], ref[1], ref[2]
    dA, dD, db = (torch.from_numpy(a).cuda() for a in (A, D, b))
    dpre = (lambda v: dD @ v) if side != "none" else None
    x, tr = P.gmres(lambda v: dA @ v, db, tol=1e-12, max_iters=200, precond=dpre, side=side)
    assert tr.iterations == its_ref
    np.testing.assert_allclose(tr.residual_history, hist_ref, rtol=1e-6, atol=1e-15)
    assert tr.converged
    x = x.cpu().numpy()
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)


def test_gmres_ifmm_preconditioned_h2():
    """The c5 recipe in miniature: GMRES on h2_matvec, right-preconditioned by
    an IFMM factorization, device path vs the oracle loop with the same
    device operators applied through numpy."""
    import paper_1508_01835_b200 as P
    from oracle import ifmm_np as O
    g = load_golden("imq3d_n2048")
    tree, _ = P.build_octree(g["points"], int(g["leaf"]))
    topo = P.compute_topology(tree)
    kern = P.imq_kernel(float(g["h"])) if str(g["kernel"]) != "exp" else P.exp_kernel()
    ops = P.chebyshev_operators(tree, topo, kern, int(g["n"]), epsilon=1e-10)
    P.initialize_weights(ops, topo)
    fct = P.factorize(P.assemble_extended_graph(_weighted(P, tree, topo, kern, g)), 1e-3)
    b = g["b"]
    ref = O.gmres(lambda v: P.h2_matvec(ops, v), b, tol=1e-10, max_iters=100, precond=fct.solve,
                  side="right")
    db = torch.from_numpy(np.ascontiguousarray(b)).cuda()
    x, tr = P.gmres(lambda v: P.h2_matvec(ops, v), db, tol=1e-10, max_iters=100,
                    precond=fct.solve, side="right")
    assert tr.converged and ref[3]
    assert abs(tr.iterations - ref[1]) <= 1
    x = x.cpu().numpy()
    r = np.linalg.norm(P.h2_matvec(ops, x) - b) / np.linalg.norm(b)
    assert r <= 2e-10, r
    assert np.linalg.norm(x - ref[0]) <= 1e-8 * np.linalg.norm(ref[0])


def _weighted(P, tree, topo, kern, g):
    ops = P.chebyshev_operators(tree, topo, kern, int(g["n"]), epsilon=1e-3)
    P.initialize_weights(ops, topo)
    return ops
