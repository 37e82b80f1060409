"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports
every symbol include/ifmm_b200.h declares, fails loudly without a GPU, and
its host-side topology matches the oracle / reference goldens bit for bit."""

import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, csr_lists, golden_names, load_golden

HEADER = os.path.join(ROOT, "include", "ifmm_b200.h")


def _declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(ifmm_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1508_01835_b200 import _native
    lib = _native.lib()
    names = _declared()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    assert lib.ifmm_abi_version() == 1
    # every declared symbol is bound with a signature in the ctypes layer
    missing = [n for n in names if n not in _native._SIGS]
    assert not missing, missing


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1508_01835_b200 import _native
    h = _native.lib().ifmm_ctx_create(0, 1 << 20)
    assert not h
    assert "no CUDA device" in _native.last_error()


@pytest.mark.parametrize("name", golden_names())
def test_host_tree_topology_bitexact(name):
    import paper_1508_01835_b200 as P
    g = load_golden(name)
    tree, perm = P.build_octree(g["points"], int(g["leaf"]))
    topo = P.compute_topology(tree)
    assert tree.depth == int(g["depth"])
    np.testing.assert_array_equal(perm, g["perm"])
    np.testing.assert_array_equal([c.level for c in tree.clusters], g["cl_level"])
    np.testing.assert_array_equal([c.start for c in tree.clusters], g["cl_start"])
    np.testing.assert_array_equal([c.stop for c in tree.clusters], g["cl_stop"])
    np.testing.assert_array_equal([-1 if c.parent is None else c.parent for c in tree.clusters],
                                  g["cl_parent"])
    np.testing.assert_array_equal([c.cell for c in tree.clusters], g["cl_cell"])
    assert topo.neighbors == csr_lists(g["nbr_ptr"], g["nbr_idx"])
    assert topo.interactions == csr_lists(g["int_ptr"], g["int_idx"])


def _grid_points(k):
    h = 1.0 / k
    return np.array([((i + .5) * h, (j + .5) * h, (l + .5) * h)
                     for i in range(k) for j in range(k) for l in range(k)])


def test_corner_and_interior_list_sizes():
    """Reference KATs (test_tree.py:92-114): corner |N|=8, |I|=56; interior
    |N|=27, |I|=189 on a full 8^3 leaf grid."""
    import paper_1508_01835_b200 as P
    pts = _grid_points(8)
    tree, _ = P.build_octree(pts, 1, depth=3, root_box=(np.array([.5, .5, .5]), .5))
    topo = P.compute_topology(tree)
    cells = {tree.clusters[c].cell: c for c in tree.leaves()}
    corner, interior = cells[(0, 0, 0)], cells[(3, 4, 3)]
    assert len(topo.neighbors[corner]) == 8 and len(topo.interactions[corner]) == 56
    assert len(topo.neighbors[interior]) == 27 and len(topo.interactions[interior]) == 189


def test_tree_edge_cases_match_oracle():
    import paper_1508_01835_b200 as P
    from oracle import ifmm_np as O
    rng = np.random.default_rng(3)
    cases = [
        (rng.uniform(-1, 1, (257, 3)), dict(leaf_target=5)),
        (rng.uniform(0, 1, (100, 3)), dict(leaf_target=500, depth=0)),
        (rng.uniform(0, 1, (300, 3)), dict(leaf_target=4, depth=1)),
        (np.column_stack([rng.uniform(0, 1, (500, 2)), np.zeros(500)]), dict(leaf_target=8)),
        (np.repeat(rng.uniform(0, 1, (20, 3)), 7, axis=0), dict(leaf_target=3)),  # duplicates
        (_grid_points(4), dict(leaf_target=1, root_box=(np.array([.5, .5, .5]), .5))),
    ]
    for pts, kw in cases:
        t, perm = P.build_octree(pts, **kw)
        to = O.build_tree(pts, **kw)
        np.testing.assert_array_equal(perm, to.perm)
        assert t.depth == to.depth
        assert [c.children for c in t.clusters] == to.children
        topo, otopo = P.compute_topology(t), O.build_topology(to)
        assert topo.neighbors == otopo.neighbors
        assert topo.interactions == otopo.interactions


def test_tree_errors():
    import paper_1508_01835_b200 as P
    with pytest.raises(ValueError):
        P.build_octree(np.zeros((5, 2)), 4)
    with pytest.raises(ValueError):
        P.build_octree(np.zeros((0, 3)), 4)
    with pytest.raises(ValueError):
        P.build_octree(np.random.rand(5, 3), 0)
    with pytest.raises(P.DegenerateGeometryError):
        P.build_octree(np.ones((5, 3)), 4)


def test_kernel_plugin_contract():
    import paper_1508_01835_b200 as P
    from oracle import ifmm_np as O
    rng = np.random.default_rng(0)
    A, B = rng.uniform(size=(7, 3)), rng.uniform(size=(5, 3))
    np.testing.assert_allclose(P.exp_kernel().block(A, B), O.exp_block(A, B), rtol=1e-14)
    np.testing.assert_allclose(P.imq_kernel(0.1).block(A, B), O.imq_block(0.1)(A, B), rtol=1e-14)
    np.testing.assert_allclose(P.benchmark_kernel(0.3).block(A, B), O.benchmark_block(0.3)(A, B),
                               rtol=1e-14)
    assert P.imq_kernel(0.1).device_spec() == (2, 0.1, 0.0)
    k, a, c0 = P.rpy_kernel(0.25, 2.0).device_spec()
    assert (k, a) == (5, 0.25) and abs(c0 - 1.0 / (6.0 * np.pi * 2.0 * 0.25)) < 1e-16
    with pytest.raises(ValueError):
        P.Kernel("custom", 1, {}, lambda P_, Q: None).device_spec()
    # a known name with a different function is refused, not silently replaced (kernels.py:22-39)
    with pytest.raises(ValueError, match="differs"):
        P.Kernel("exp", 1, {}, lambda A_, B_: np.ones((len(A_), len(B_)))).device_spec()
    from scipy.spatial.distance import cdist
    ref_style = P.Kernel("imq", 1, {"h": 0.2}, lambda A_, B_: 1.0 / np.sqrt(cdist(A_, B_) ** 2 + 0.04))
    assert ref_style.device_spec() == (2, 0.2, 0.0)


@pytest.mark.parametrize("seed", [0, 1, 123456789])
def test_native_pcg64_stream_is_numpys(seed):
    """The engine's reference stream (native PCG64 + numpy's ziggurat from
    libnpyrandom, factor.cu) is bitwise np.random.Generator(PCG64(seed))
    .standard_normal -- the draws of the reference's factorize rng
    (factor.py:188, lowrank.py:108)."""
    import ctypes as C
    from paper_1508_01835_b200 import _native as N
    from paper_1508_01835_b200.factor import pcg64_state
    n = 2_000_003
    out = np.empty(n)
    N.check(N.lib().ifmm_pcg64_normals(pcg64_state(seed), n, N.as_dp(out)))
    ref = np.random.Generator(np.random.PCG64(seed)).standard_normal(n)
    assert np.array_equal(out, ref)
