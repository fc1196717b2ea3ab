"""Pins of the CPU oracle (oracle/h2_oracle.c) to things other than itself:
brute-force dense assembly, closed forms, the all-dense degenerate case, paper-printed values,
invariants.  All CPU (-m "not gpu")."""
import numpy as np
import pytest

import oracle
from h2gen import build_cluster_tree, dual_traversal, random_h2_data, make_xy, poly_kernel_apply
from h2gen.tree import grid_points, uniform_points
from h2gen.kernels import Kernel
from h2gen.h2data import build_h2
from tests.dense_assembly import assemble


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def colmax_rel(a, b):
    return max(np.linalg.norm(a[i] - b[i]) / np.linalg.norm(b[i]) for i in range(a.shape[0]))


def small_random(N=700, m=16, dim=2, eta=0.9, ranks=None, seed=3, symmetric=False, grid=None):
    pts = grid_points(grid) if grid else uniform_points(N, dim, seed)
    tr = build_cluster_tree(pts, m)
    st = dual_traversal(tr, eta)
    if ranks is None:
        ranks = [((3 * l + 5) % 7) + 4 for l in range(tr.q + 1)]   # varies by level
    return random_h2_data(tr, st, ranks, seed + 100, symmetric=symmetric)


@pytest.mark.parametrize("N,m,eta,seed", [(700, 16, 0.9, 3), (1000, 24, 0.7, 5), (333, 8, 1.5, 9)])
def test_dense_assembly_random_h2(N, m, eta, seed):
    """Whole oracle vs brute force on RANDOM unsymmetric H² data with ragged leaves and per-level
    ranks: a transposed operand, a swapped k^l/k^{l-1}, a dropped level or term fails this."""
    h = small_random(N, m, eta=eta, seed=seed)
    assert h.n_S > 0 and h.n_D > 0
    A, cover = assemble(h)
    assert np.all(cover == 1), "partition property (SPEC.md:71)"
    X = make_xy(h.perm, 3, seed, -1.0, 1.0)
    Y0 = make_xy(h.perm, 3, seed, -1.0, 1.0, stream=1)
    alpha, beta = -0.7, 0.3
    Y = oracle.matvec(h, X, alpha, beta, Y0)
    Yref = alpha * (X @ A.T) + beta * Y0
    assert colmax_rel(Y, Yref) < 1e-13


def test_ragged_leaf_sizes_present():
    h = small_random(700, 16)
    sizes = np.diff(h.leaf_ptr)
    assert sizes.min() < sizes.max() <= h.m


def test_all_dense_degenerate_case():
    """eta -> 'never admissible': A~ = K entrywise, Y = K X by a plain library product."""
    pts = uniform_points(512, 2, 11)
    tr = build_cluster_tree(pts, 16)
    st = dual_traversal(tr, 0.9, all_dense=True)
    assert st.n_S == 0
    kern = Kernel("exp", ell=0.1)
    h = build_h2(tr, st, kern, 3)
    X = make_xy(h.perm, 2, 4)
    K = kern(h.points[:, None, :], h.points[None, :, :])
    Y = oracle.matvec(h, X)
    assert rel(Y, X @ K.T) < 1e-13


@pytest.mark.parametrize("dim,p,grid", [(2, 4, (40, 37)), (2, 5, None), (3, 3, (11, 12, 10))])
def test_polynomial_kernel_closed_form(dim, p, grid):
    """K = (1 + x.y)^(p-1) is reproduced exactly by order-p Chebyshev interpolation, so the oracle
    on generated H² data must equal the O(N #monomials) moment closed form to rounding."""
    pts = grid_points(grid) if grid else uniform_points(2000, dim, 21)
    tr = build_cluster_tree(pts, 32)
    st = dual_traversal(tr, 0.9)
    assert st.n_S > 0
    h = build_h2(tr, st, Kernel("poly", p=p), p)
    X = make_xy(h.perm, 2, 6)
    Y = oracle.matvec(h, X)
    Yc = poly_kernel_apply(h.points, X, p)
    assert colmax_rel(Y, Yc) < 1e-12


def test_upsweep_closed_form_chebyshev():
    """x^_s^l[b] = sum_{i in s} L^s_b(p_i) x_i: nested Chebyshev interpolation (degree p-1) reproduces
    the parent's Lagrange polynomials exactly, checked at every level."""
    from h2gen.h2data import _box_nodes, _tensor_lagrange
    pts = uniform_points(1500, 2, 8)
    tr = build_cluster_tree(pts, 24)
    st = dual_traversal(tr, 0.9)
    p = 4
    h = build_h2(tr, st, Kernel("exp", ell=0.1), p)
    X = make_xy(h.perm, 2, 2)
    xh, _ = oracle.trees(h, X)
    for l in range(h.q + 1):
        nodes = _box_nodes(tr.lo[l], tr.hi[l], p)
        for i in range(0, 1 << l, max(1, (1 << l) // 8)):
            a, b = tr.starts[l][i], tr.starts[l][i + 1]
            L = _tensor_lagrange(nodes[i:i + 1], tr.points[None, a:b], p)[0]   # (rows, k)
            ref = X[:, a:b] @ L                                                 # (nv, k)
            assert np.allclose(xh[l][i], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_coupling_tree_against_naive_loop():
    """y^_t^l = sum_s S_ts x^_s on random data, from the oracle's own x^ tree."""
    h = small_random(600, 16, seed=4)
    X = make_xy(h.perm, 2, 3)
    xh, yh = oracle.trees(h, X)
    for l in range(h.q + 1):
        for t in range(1 << l):
            ref = np.zeros((2, h.ranks[l]))
            for b in range(h.S_rowptr[l][t], h.S_rowptr[l][t + 1]):
                ref += xh[l][h.S_col[l][b]] @ h.S[l][b]      # stored S^T -> (x^T S^T)
            assert np.allclose(yh[l][t], ref, rtol=1e-13, atol=1e-14)


def test_linearity_and_columns():
    h = small_random(800, 16, seed=12)
    X1 = make_xy(h.perm, 4, 1, -1, 1)
    X2 = make_xy(h.perm, 4, 2, -1, 1)
    a, b = 0.37, -1.9
    lhs = oracle.matvec(h, a * X1 + b * X2)
    rhs = a * oracle.matvec(h, X1) + b * oracle.matvec(h, X2)
    assert rel(lhs, rhs) < 1e-13
    # nv = 4 equals 4 independent nv = 1 calls, column by column
    Y4 = oracle.matvec(h, X1)
    for c in range(4):
        assert np.array_equal(Y4[c:c + 1], oracle.matvec(h, X1[c:c + 1]))


def test_alpha_beta_semantics():
    h = small_random(400, 16, seed=13)
    X = make_xy(h.perm, 2, 1)
    Y0 = make_xy(h.perm, 2, 2, stream=1)
    assert np.array_equal(oracle.matvec(h, X, 0.0, 0.5, Y0), 0.5 * Y0)   # alpha = 0 -> beta Y exactly
    Ynan = np.full_like(Y0, np.nan)
    Y = oracle.matvec(h, X, 1.0, 0.0, Ynan)                              # beta = 0 -> Y not read
    assert np.all(np.isfinite(Y))
    assert np.array_equal(Y, oracle.matvec(h, X))


def test_symmetry_invariant():
    """Symmetric data (U=V, E=F, S_st = S_ts^T, D_st = D_ts^T): y^T (A x) = x^T (A y)."""
    from h2gen import build_config
    h = build_h2(build_cluster_tree(uniform_points(1200, 2, 5), 32),
                 dual_traversal(build_cluster_tree(uniform_points(1200, 2, 5), 32), 0.9),
                 Kernel("exp", ell=0.1), 4)
    x = make_xy(h.perm, 1, 1, -1, 1)
    y = make_xy(h.perm, 1, 2, -1, 1)
    Ax, Ay = oracle.matvec(h, x), oracle.matvec(h, y)
    lhs, rhs = float((y @ Ax.T)[0, 0]), float((x @ Ay.T)[0, 0])
    scale = np.linalg.norm(x) * np.linalg.norm(y) * np.linalg.norm(Ax) / np.linalg.norm(x)
    assert abs(lhs - rhs) <= 1e-12 * scale


def test_sampled_rows_equal_full():
    """Sampled-row oracle: restricted to the sampled leaves it equals the full
    result exactly (same arithmetic, same order)."""
    h = small_random(900, 16, seed=14)
    X = make_xy(h.perm, 3, 1)
    Y0 = make_xy(h.perm, 3, 2, stream=1)
    full = oracle.matvec(h, X, 1.3, -0.2, Y0)
    mask = np.zeros(1 << h.q, dtype=bool)
    mask[::7] = True
    mask[-1] = True
    part = oracle.matvec(h, X, 1.3, -0.2, Y0, leaf_mask=mask)
    rows = np.concatenate([np.arange(h.leaf_ptr[i], h.leaf_ptr[i + 1]) for i in np.flatnonzero(mask)])
    assert np.array_equal(part[:, rows], full[:, rows])
    other = np.setdiff1d(np.arange(h.N), rows)
    assert np.array_equal(part[:, other], Y0[:, other])


def test_paper_accuracy_2d(golden):
    """2D grid, exp ell=0.1a, m=64, eta=0.9, k=64 (p=8): relative accuracy < 1e-7 on
    10% sampled rows with uniform random x.  Checked at N = 4096 (64 x 64 grid) to the order of
    magnitude (reading R17 in DESIGN.md: our first-kind Chebyshev construction gives 5.3e-7 at
    64x64, 1.1e-7 at 512x256; the paper's node family/order is not stated)."""
    tr = build_cluster_tree(grid_points((64, 64)), 64)
    st = dual_traversal(tr, 0.9)
    kern = Kernel("exp", ell=0.1)
    h = build_h2(tr, st, kern, 8)
    x = make_xy(h.perm, 1, 99)
    y = oracle.matvec(h, x)
    rows = np.random.default_rng(1).choice(h.N, h.N // 10, replace=False)
    K = kern(h.points[rows][:, None, :], h.points[None, :, :])
    ref = (K @ x[0])
    err = np.linalg.norm(y[0, rows] - ref) / np.linalg.norm(ref)
    assert err < 10 * golden["accuracy_2d"]["value"]


def test_paper_accuracy_3d_order(golden):
    """3D exp ell=0.2a, k=64 (tricubic p=4), accuracy ~1e-3 (eta=1.1, reading R5)."""
    tr = build_cluster_tree(grid_points((16, 16, 16)), 64)
    st = dual_traversal(tr, 1.1)
    kern = Kernel("exp", ell=0.2)
    h = build_h2(tr, st, kern, 4)
    x = make_xy(h.perm, 1, 98)
    y = oracle.matvec(h, x)
    rows = np.random.default_rng(2).choice(h.N, h.N // 10, replace=False)
    K = kern(h.points[rows][:, None, :], h.points[None, :, :])
    ref = K @ x[0]
    err = np.linalg.norm(y[0, rows] - ref) / np.linalg.norm(ref)
    v = golden["accuracy_3d"]["value"]
    assert v / 30 < err < v * 30, err


def test_openmp_threads_bitwise_equal():
    """The OpenMP oracle keeps a fixed per-output order: 1 thread and all host
    threads give bitwise-identical results, in the full and in the sampled-row mode."""
    h = small_random(3000, 16, seed=21)
    X = make_xy(h.perm, 5, 21, -1.0, 1.0)
    Y0 = make_xy(h.perm, 5, 22, -1.0, 1.0, stream=1)
    mask = (np.arange(1 << h.q) % 3) == 0
    try:
        oracle.set_threads(1)
        a = oracle.matvec(h, X, -0.7, 0.3, Y0)
        am = oracle.matvec(h, X, -0.7, 0.3, Y0, leaf_mask=mask)
        ta = oracle.trees(h, X)
        n = oracle.set_threads(max(4, len(__import__("os").sched_getaffinity(0))))
        assert n >= 2
        b = oracle.matvec(h, X, -0.7, 0.3, Y0)
        bm = oracle.matvec(h, X, -0.7, 0.3, Y0, leaf_mask=mask)
        tb = oracle.trees(h, X)
    finally:
        oracle.set_threads(0)
    assert np.array_equal(a, b) and np.array_equal(am, bm)
    for u, v in zip(ta[0] + ta[1], tb[0] + tb[1]):
        assert np.array_equal(u, v)
