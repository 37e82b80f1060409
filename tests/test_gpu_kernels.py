"""Device micro-kernels vs numpy / the oracle (GPU only)."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _p(t):
    return C.c_void_p(t.data_ptr())


@pytest.fixture(scope="module")
def N():
    from paper_1508_01835_b200 import _native
    _native.ctx()
    return _native


@pytest.mark.parametrize("M,Nn,K,ta,tb", [(1, 1, 1, 0, 0), (7, 5, 3, 0, 0), (64, 64, 64, 0, 0),
                                          (100, 37, 129, 1, 0), (65, 130, 17, 0, 1),
                                          (300, 200, 150, 1, 1), (513, 257, 96, 0, 0),
                                          (1500, 1300, 70, 0, 0), (1301, 1407, 33, 1, 1),
                                          (1400, 1290, 131, 0, 1), (1290, 1400, 50, 1, 0)])
def test_gemm(N, M, Nn, K, ta, tb):
    rng = np.random.default_rng(M * 7 + Nn)
    A = rng.standard_normal((K, M) if ta else (M, K))
    B = rng.standard_normal((Nn, K) if tb else (K, Nn))
    Cm = rng.standard_normal((M, Nn))
    ref = 1.5 * (A.T if ta else A) @ (B.T if tb else B) - 0.5 * Cm
    dA, dB, dC = _dev(A), _dev(B), _dev(Cm)
    N.check(N.lib().ifmm_dev_gemm(N.ctx(), M, Nn, K, _p(dA), A.shape[1], ta, _p(dB), B.shape[1],
                                  tb, _p(dC), Nn, 1.5, -0.5))
    N.check(N.lib().ifmm_dev_sync(N.ctx()))
    np.testing.assert_allclose(dC.cpu().numpy(), ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("m,n", [(1, 1), (5, 3), (3, 5), (40, 40), (64, 60), (60, 97), (150, 40)])
def test_svd(N, m, n):
    rng = np.random.default_rng(m + 100 * n)
    k = min(m, n)
    s_true = 10.0 ** -np.linspace(0, 12, k)
    U, _ = np.linalg.qr(rng.standard_normal((m, k)))
    V, _ = np.linalg.qr(rng.standard_normal((n, k)))
    A = (U * s_true) @ V.T
    thr = 1e-7
    dA = _dev(A)
    dU = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    dS = torch.zeros(k, dtype=torch.float64, device="cuda")
    dV = torch.zeros(n * k, dtype=torch.float64, device="cuda")
    dr = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().ifmm_dev_svd(N.ctx(), m, n, _p(dA), thr, _p(dU), _p(dS), _p(dV), _p(dr)))
    r = int(dr.item())
    s_ref = np.linalg.svd(A, compute_uv=False)
    assert r == int(np.sum(s_ref > thr))
    S = dS.cpu().numpy()[:r]
    np.testing.assert_allclose(S, s_ref[:r], rtol=1e-10, atol=1e-14)
    Uo = dU.cpu().numpy()[:m * r].reshape(r, m).T
    Vo = dV.cpu().numpy()[:n * r].reshape(r, n).T
    Ar = (U[:, :r] * s_true[:r]) @ V[:, :r].T
    np.testing.assert_allclose((Uo * S) @ Vo.T, Ar, atol=1e-9)
    np.testing.assert_allclose(Uo.T @ Uo, np.eye(r), atol=1e-12)


@pytest.mark.parametrize("n,nrhs", [(1, 1), (17, 3), (90, 40), (160, 70), (161, 5), (400, 33),
                                    (1000, 40), (2000, 9)])
def test_lu_solve(N, n, nrhs):
    rng = np.random.default_rng(n)
    A = rng.standard_normal((n, n)) + n * 0.05 * np.eye(n)
    X = rng.standard_normal((n, nrhs))
    ref = np.linalg.solve(A, X)
    dA, dX = _dev(A), _dev(X)
    dp = torch.zeros(n, dtype=torch.int32, device="cuda")
    N.check(N.lib().ifmm_dev_lu_solve(N.ctx(), n, _p(dA), _p(dp), _p(dX), nrhs))
    np.testing.assert_allclose(dX.cpu().numpy(), ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def test_lu_singular(N):
    A = np.zeros((8, 8))
    dA = _dev(A)
    dp = torch.zeros(8, dtype=torch.int32, device="cuda")
    dX = _dev(np.ones((8, 1)))
    with pytest.raises(Exception):
        N.check(N.lib().ifmm_dev_lu_solve(N.ctx(), 8, _p(dA), _p(dp), _p(dX), 1))


def test_union_matches_oracle(N):
    from conftest import load_golden
    from oracle import ifmm_np as O
    k = load_golden("kat_lowrank")
    B, w, F, wf = k["B"], k["w"], k["F"], k["wf"]
    m, ko = B.shape
    kf = F.shape[1]
    thr = 1e-2
    ref = O.basis_union(B, w, F, wf, thr)
    cap = min(m, ko + kf)
    dB, dw, dF, dwf = _dev(B), _dev(w), _dev(F), _dev(wf)
    NB = torch.zeros(m * cap, dtype=torch.float64, device="cuda")
    NW = torch.zeros(cap, dtype=torch.float64, device="cuda")
    OM = torch.zeros(cap * ko, dtype=torch.float64, device="cuda")
    FM = torch.zeros(cap * kf, dtype=torch.float64, device="cuda")
    dr = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().ifmm_dev_union(N.ctx(), m, ko, kf, _p(dB), _p(dw), _p(dF), _p(dwf), thr, 0,
                                   _p(NB), _p(NW), _p(OM), _p(FM), _p(dr)))
    r = int(dr.item())
    assert r == ref.rank
    nb = NB.cpu().numpy()[:m * r].reshape(r, m).T
    np.testing.assert_allclose(NW.cpu().numpy()[:r], ref.weights, rtol=1e-10)
    om = OM.cpu().numpy()[:r * ko].reshape(r, ko)
    fm = FM.cpu().numpy()[:r * kf].reshape(r, kf)
    np.testing.assert_allclose(nb @ om, ref.basis @ ref.old_map, atol=1e-10)
    np.testing.assert_allclose(nb @ fm, ref.basis @ ref.fill_map, atol=1e-10)


@pytest.mark.parametrize("m,n,decay,r_cut", [(480, 480, 0.5, 12), (480, 100, 0.3, 13),
                                              (100, 480, 0.3, 13), (200, 300, 0.05, 60),
                                              (64, 64, 0.2, 40), (500, 450, 0.02, 100),
                                              (450, 480, 0.01, 300)])
def test_fill_svd_large(N, m, n, decay, r_cut):
    """Rank-revealing fill compression vs numpy on large blocks (global path);
    the threshold sits between two singular values."""
    rng = np.random.default_rng(m * 3 + n)
    k = min(m, n)
    s_true = 10.0 ** (-decay * np.arange(k))
    thr = float(np.sqrt(s_true[r_cut - 1] * s_true[r_cut]))
    U, _ = np.linalg.qr(rng.standard_normal((m, k)))
    V, _ = np.linalg.qr(rng.standard_normal((n, k)))
    A = (U * s_true) @ V.T
    s_ref = np.linalg.svd(A, compute_uv=False)
    dA = _dev(A)
    dU = torch.zeros(m * k, dtype=torch.float64, device="cuda")
    dS = torch.zeros(k, dtype=torch.float64, device="cuda")
    dV = torch.zeros(n * k, dtype=torch.float64, device="cuda")
    dr = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().ifmm_dev_svd(N.ctx(), m, n, _p(dA), thr, _p(dU), _p(dS), _p(dV), _p(dr)))
    r = int(dr.item())
    assert r == int(np.sum(s_ref > thr))
    S = dS.cpu().numpy()[:r]
    np.testing.assert_allclose(S, s_ref[:r], rtol=1e-9, atol=1e-6 * thr)
    Uo = dU.cpu().numpy()[:m * r].reshape(r, m).T
    Vo = dV.cpu().numpy()[:n * r].reshape(r, n).T
    Ar = (U[:, :r] * s_true[:r]) @ V[:, :r].T
    assert np.linalg.norm((Uo * S) @ Vo.T - Ar) <= 1e-8 * np.linalg.norm(Ar) + 1e-5 * thr


def test_exact_matvec_matches_dense(N):
    import paper_1508_01835_b200 as P
    rng = np.random.default_rng(5)
    pts = rng.uniform(size=(1500, 3))
    x = rng.standard_normal(1500)
    for K in (P.imq_kernel(0.05), P.exp_kernel(), P.benchmark_kernel(0.2)):
        A = K.block(pts, pts)
        y = P.exact_matvec(pts, K, x)
        np.testing.assert_allclose(y, A @ x, rtol=1e-11, atol=1e-11 * np.abs(A @ x).max())


def test_union_giant_matches_oracle(N):
    """A giant union (min(m, C) above the giant threshold): cooperative multi-CTA
    ACA, CholeskyQR2 and block-cyclic Jacobi."""
    from oracle import ifmm_np as O
    rng = np.random.default_rng(11)
    m, ko, kf = 420, 190, 24
    B, _ = np.linalg.qr(rng.standard_normal((m, ko)))
    F, _ = np.linalg.qr(rng.standard_normal((m, kf)))
    w = np.sort(10.0 ** (-7 * rng.random(ko)))[::-1]
    wf = np.sort(10.0 ** (-7 * rng.random(kf)))[::-1] * 0.5
    thr = 1e-6 * w[0]
    ref = O.basis_union(B, w, F, wf, thr)
    assert min(m, ko + kf) > 160
    cap = min(m, ko + kf)
    dB, dw, dF, dwf = _dev(B), _dev(w), _dev(F), _dev(wf)
    NB = torch.zeros(m * cap, dtype=torch.float64, device="cuda")
    NW = torch.zeros(cap, dtype=torch.float64, device="cuda")
    OM = torch.zeros(cap * ko, dtype=torch.float64, device="cuda")
    FM = torch.zeros(cap * kf, dtype=torch.float64, device="cuda")
    dr = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().ifmm_dev_union(N.ctx(), m, ko, kf, _p(dB), _p(dw), _p(dF), _p(dwf), thr, 0,
                                   _p(NB), _p(NW), _p(OM), _p(FM), _p(dr)))
    r = int(dr.item())
    assert r == ref.rank
    nb = NB.cpu().numpy()[:m * r].reshape(r, m).T
    np.testing.assert_allclose(NW.cpu().numpy()[:r], ref.weights, rtol=1e-10, atol=1e-13 * w[0])
    om = OM.cpu().numpy()[:r * ko].reshape(r, ko)
    fm = FM.cpu().numpy()[:r * kf].reshape(r, kf)
    np.testing.assert_allclose(nb @ om, ref.basis @ ref.old_map, atol=1e-9)
    np.testing.assert_allclose(nb @ fm, ref.basis @ ref.fill_map, atol=1e-9)


@pytest.mark.parametrize("m,ko,kf,decay", [(12, 5, 3, 3), (64, 20, 6, 6), (97, 41, 9, 7),
                                           (120, 30, 8, 9), (230, 45, 10, 9), (255, 64, 17, 8),
                                           (530, 80, 12, 9), (700, 70, 26, 5), (60, 70, 20, 6),
                                           (400, 88, 8, 2), (1000, 60, 30, 12)])
def test_union_fused_second_half_matches_oracle(N, m, ko, kf, decay):
    """Register ACA + union_post_kernel (CholeskyQR2 with a first-order second
    pass, shared-memory Jacobi, DMMA outputs) against the oracle union: same
    rank, weights to 1e-10, the same represented operators, orthonormal basis."""
    import ctypes as C
    from oracle import ifmm_np as O
    rng = np.random.default_rng(m + 7 * ko)
    B, _ = np.linalg.qr(rng.standard_normal((m, min(ko, m))))
    ko = B.shape[1]
    F, _ = np.linalg.qr(rng.standard_normal((m, min(kf, m))))
    kf = F.shape[1]
    w = np.sort(10.0 ** (-decay * rng.random(ko)))[::-1]
    wf = np.sort(10.0 ** (-decay * rng.random(kf)))[::-1] * 0.5
    thr = 1e-6 * w[0]
    ref = O.basis_union(B, w, F, wf, thr)
    cap = min(m, ko + kf)
    dB, dw, dF, dwf = _dev(B), _dev(w), _dev(F), _dev(wf)
    NB = torch.zeros(m * cap, dtype=torch.float64, device="cuda")
    NW = torch.zeros(cap, dtype=torch.float64, device="cuda")
    OM = torch.zeros(cap * ko, dtype=torch.float64, device="cuda")
    FM = torch.zeros(cap * kf, dtype=torch.float64, device="cuda")
    dr = torch.zeros(1, dtype=torch.int32, device="cuda")
    up = (C.c_ulonglong * 16)()
    N.lib().ifmm_union_post_profile(up, 1)
    N.check(N.lib().ifmm_dev_union(N.ctx(), m, ko, kf, _p(dB), _p(dw), _p(dF), _p(dwf), thr, 0,
                                   _p(NB), _p(NW), _p(OM), _p(FM), _p(dr)))
    N.lib().ifmm_union_post_profile(up, 0)
    assert up[6] == 1, "the fused second half did not take this union"
    r = int(dr.item())
    assert r == ref.rank
    nb = NB.cpu().numpy()[:m * r].reshape(r, m).T
    np.testing.assert_allclose(NW.cpu().numpy()[:r], ref.weights, rtol=1e-10, atol=1e-13 * w[0])
    np.testing.assert_allclose(nb.T @ nb, np.eye(r), atol=1e-12)
    om = OM.cpu().numpy()[:r * ko].reshape(r, ko)
    fm = FM.cpu().numpy()[:r * kf].reshape(r, kf)
    np.testing.assert_allclose(nb @ om, ref.basis @ ref.old_map, atol=1e-9)
    np.testing.assert_allclose(nb @ fm, ref.basis @ ref.fill_map, atol=1e-9)
