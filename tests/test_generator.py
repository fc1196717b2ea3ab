"""Generator (h2gen) checks: kd-tree partition/balance, admissibility examples, Chebyshev closed
forms, and the structure counts that reproduce the paper's printed sparsity constants."""
import numpy as np
import pytest

from h2gen import build_cluster_tree, dual_traversal
from h2gen.tree import grid_points, uniform_points
from h2gen.structure import admissible
from h2gen.h2data import cheb_nodes_1d, _lagrange_1d, _box_nodes, _tensor_lagrange, _tensor_points


def test_kd_tree_collinear():
    tr = build_cluster_tree(np.array([[3.0], [0.0], [2.0], [1.0]]), 1)
    assert tr.q == 2
    assert list(tr.perm) == [1, 3, 2, 0]


def test_kd_tree_partition_balance():
    tr = build_cluster_tree(uniform_points(1000, 2, 1), 16)
    assert tr.q == 6
    assert sorted(tr.perm) == list(range(1000))
    sizes = np.diff(tr.leaf_ptr)
    assert sizes.max() - sizes.min() <= 1 and sizes.max() <= 16
    for l in range(tr.q):
        # children partition the parent's range
        assert np.array_equal(tr.starts[l], tr.starts[l + 1][::2])


def test_admissibility_examples():
    c = lambda *v: np.array([v], dtype=float)
    d = np.array([np.sqrt(2.0)])
    assert not admissible(c(0, 0), d, c(0, 0), d, 0.9)        # same box
    assert admissible(c(0, 0), d, c(10, 0), d, 0.9)           # 9 >= sqrt 2
    assert not admissible(c(0, 0), d, c(1, 0), d, 0.9)        # 0.9 < sqrt 2


def test_chebyshev_closed_forms():
    assert np.allclose(cheb_nodes_1d(1), [0.0])
    assert np.allclose(cheb_nodes_1d(2), [np.sqrt(0.5), -np.sqrt(0.5)])
    n3 = _box_nodes(np.array([[0.0, 0.0]]), np.array([[2.0, 2.0]]), 3)[0, 0]
    assert np.allclose(n3, [1 + np.cos(np.pi / 6), 1.0, 1 - np.cos(np.pi / 6)])


def test_lagrange_cardinality_and_partition_of_unity():
    nodes = _box_nodes(np.array([[0.0, 0.0]]), np.array([[1.0, 2.0]]), 4)
    pts = _tensor_points(nodes, 4, 2)                      # (1, 16, 2)
    L = _tensor_lagrange(nodes, pts, 4)[0]
    assert np.allclose(L, np.eye(16), atol=1e-13)
    x = np.random.default_rng(0).random((1, 50, 2))
    assert np.allclose(_tensor_lagrange(nodes, x, 4)[0].sum(axis=1), 1.0)


def test_transfer_identity_same_box():
    from h2gen.h2data import _tensor_lagrange
    nodes = _box_nodes(np.array([[0.0, 0.0]]), np.array([[1.0, 1.0]]), 3)
    pts = _tensor_points(nodes, 3, 2)
    assert np.allclose(_tensor_lagrange(nodes, pts, 3)[0], np.eye(9), atol=1e-13)


def test_structure_counts_cfg1_cfg2():
    """SURVEY.md App. A counts (exact rules of App. B)."""
    tr = build_cluster_tree(uniform_points(4096, 2, 210905451), 32)
    st = dual_traversal(tr, 0.9)
    assert (tr.q, st.n_S, st.csp(), st.n_D) == (7, 1608, 14, 982)
    tr = build_cluster_tree(grid_points((64, 64)), 32)
    st = dual_traversal(tr, 0.9)
    assert (st.n_S, st.csp(), st.n_D) == (1314, 17, 808)


def test_paper_csp_2d(golden):
    """The paper's 2D set (2^19 points, m=64, eta=0.9) reproduces C_sp = 17."""
    tr = build_cluster_tree(grid_points((1024, 512)), 64)
    st = dual_traversal(tr, 0.9)
    assert tr.q == 13
    assert st.csp() == golden["csp_2d"]["value"]
    assert (st.n_S, st.n_D) == (202914, 40576)


@pytest.mark.slow
def test_paper_csp_3d(golden):
    """3D set (2^19 points, m=64) with eta = 1.1 (reading R5) reproduces C_sp = 30."""
    tr = build_cluster_tree(grid_points((64, 64, 128)), 64)
    st = dual_traversal(tr, 1.1)
    assert st.csp() == golden["csp_3d"]["value"]


def test_levels_536M(golden):
    from h2gen.tree import tree_depth
    assert tree_depth(1 << 29, 64) == golden["levels_536M"]["value"]


def test_flop_convention_matches_paper(golden):
    """2 nv (stored operator scalars) per point for the paper's 2D set agrees with the paper-implied
    4524 flop/point/vector within 1.5%, from structure counts alone."""
    tr = build_cluster_tree(grid_points((1024, 512)), 64)
    st = dual_traversal(tr, 0.9)
    k, m, q, N = 64, 64, tr.q, tr.N
    ops = st.n_D * m * m + st.n_S * k * k + 2 * N * k + 2 * (2 ** (q + 1) - 2) * k * k
    per_pt = 2 * ops / N
    ref = golden["flop_per_point_per_vector_paper"]["value"]
    assert abs(per_pt - ref) / ref < 0.015


def test_fd_kernel_and_diffusivity():
    """FD operator (reading R10): K_ij = -2 a(x_i, x_j) / |x_j - x_i|^(2+2beta),
    K_ii = 0, a = sqrt(kappa_i kappa_j), kappa = 1 + f(x1; 0, 1.5) f(x2; 0, 2.0)."""
    import numpy as np
    from h2gen.kernels import Kernel, fd_kappa
    k = Kernel("fd", beta=0.75)
    x = np.array([[0.9, 0.9], [0.9, -0.1], [0.0, 0.0]])
    assert np.isclose(fd_kappa(x[:1])[0], 1.0) and np.isclose(fd_kappa(x[2:])[0], 1.0 + np.exp(-2.0))
    K = k(x[:, None, :], x[None, :, :])
    assert K[0, 1] == -2.0                          # kappa = 1 at both, distance 1
    assert np.all(np.diag(K) == 0.0)
    r = np.linalg.norm(x[0] - x[2])
    assert np.isclose(K[0, 2], -2.0 * np.sqrt(1.0 + np.exp(-2.0)) / r ** 3.5)
    assert np.allclose(K, K.T)
