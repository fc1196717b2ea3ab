"""Fractional-diffusion solve.

CPU (-m "not gpu"): the oracle side pinned to things other than itself -- D from the oracle's
K^ 1 against brute-force direct summation over the extended grid (PAPER.md:766 definition of
D_ii), the stencil C's structure, the PCG routine against a dense solve, SPD probes of
A = h^2 (D + K + C).  GPU: h2_fd_diag + h2_pcg against the oracle's PCG on the same inputs."""
import numpy as np
import pytest

import oracle
from oracle import fd as ofd
from h2gen.fd import fd_problem, build_fd_operators
from h2gen.kernels import fd_kappa


@pytest.fixture(scope="module")
def ops():
    return build_fd_operators(20, m=32)


def test_D_by_khat_matches_direct_sum(ops):
    """D_ii = sum_{j != i} 2 a(x_i, y_j)/|y_j - x_i|^(2+2beta) over Omega u Omega_0,
    brute force, vs the product K^ 1: exact (1e-12) when K^ is stored dense
    (all-dense structure: pins the index map, sign and point sets), and within the Chebyshev
    k = 36 approximation (2e-2 here; no paper value: "parity unpinned" for the approximation)
    for the H² K^."""
    from h2gen.tree import build_cluster_tree
    from h2gen.structure import dual_traversal
    from h2gen.kernels import Kernel
    from h2gen.h2data import build_h2
    pr = ops.prob
    tE = build_cluster_tree(pr.extended, 32)
    hE = build_h2(tE, dual_traversal(tE, 0.9, all_dense=True), Kernel("fd", beta=pr.beta, sign=1.0), 2)
    assert hE.n_S == 0
    inv = np.empty_like(tE.perm)
    inv[tE.perm] = np.arange(tE.perm.size)
    invK = np.empty_like(ops.K.perm)
    invK[ops.K.perm] = np.arange(ops.K.perm.size)
    idx_dense = inv[pr.ext_interior[ops.K.perm]]
    D_exact = ofd.fd_diag(hE, idx_dense)
    D = ofd.fd_diag(ops.Khat, ops.idx)                    # tree order of K
    x = ops.K.points                                      # interior, tree order
    y = pr.extended
    kx = fd_kappa(x)[:, None]
    ky = fd_kappa(y)[None, :]
    r2 = ((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)
    with np.errstate(divide="ignore"):
        t = np.where(r2 > 0, 2.0 * np.sqrt(kx * ky) / r2 ** (1.0 + pr.beta), 0.0)
    Dref = t.sum(1)
    assert np.max(np.abs(D_exact - Dref) / Dref) < 1e-12
    assert np.all(D > 0)
    assert np.max(np.abs(D - Dref) / Dref) < 2e-2


def test_stencil_C():
    pr = fd_problem(12)
    n = 12
    Cd = np.zeros((n * n, n * n))
    for i in range(n * n):
        a, b = pr.C_rowptr[i], pr.C_rowptr[i + 1]
        Cd[i, pr.C_col[a:b]] = pr.C_val[a:b]
    assert np.array_equal(Cd, Cd.T)
    assert np.all(np.diag(Cd) > 0) and np.all(Cd - np.diag(np.diag(Cd)) <= 0)
    assert np.diff(pr.C_rowptr).max() == 5
    # the corner row (kappa == 1 on its whole stencil): (-1, -1, 4) h^(-2b-2), two of the four
    # edges lead to Omega_0 (u = 0) and stay on the diagonal
    k = fd_kappa(pr.interior)
    assert k[0] == 1.0 and abs(k[1] - 1.0) < 1e-3 and abs(k[n] - 1.0) < 1e-3
    row = Cd[0][Cd[0] != 0] / pr.h ** (-2 * pr.beta - 2)
    assert np.allclose(sorted(row), [-1, -1, 4], rtol=1e-3)
    assert np.linalg.eigvalsh(Cd).min() > 0               # Omega_0 rows make it definite


def test_pcg_against_dense_solve():
    rng = np.random.default_rng(3)
    M = rng.standard_normal((60, 60))
    A = M @ M.T + 60 * np.eye(60)
    b = rng.standard_normal(60)
    x, it, hist = ofd.pcg(lambda v: A @ v, b, 1.0 / np.diag(A), 1e-12, 200)
    assert np.linalg.norm(x - np.linalg.solve(A, b)) / np.linalg.norm(x) < 1e-10
    assert it <= 60 and hist[-1] <= 1e-12


def test_fd_operator_spd_and_solve(ops):
    D = ofd.fd_diag(ops.Khat, ops.idx)
    h = ops.prob.h
    rng = np.random.default_rng(5)
    u, v = rng.standard_normal((2, D.size))

    def A(w):
        return h * h * (D * w + oracle.matvec(ops.K, w[None, :], 1.0, 0.0)[0] +
                        ofd.csr_apply(ops.C_rowptr, ops.C_col, ops.C_val, w))
    assert abs(u @ A(v) - v @ A(u)) <= 1e-9 * np.linalg.norm(u) * np.linalg.norm(A(v))
    for _ in range(5):
        w = rng.standard_normal(D.size)
        assert w @ A(w) > 0
    x, it, hist = ofd.fd_solve(ops.K, D, ops.C_rowptr, ops.C_col, ops.C_val, h, ops.b, 1e-8, 300)
    assert hist[-1] <= 1e-8 and it < 300
    assert np.linalg.norm(A(x) - ops.b) / np.linalg.norm(ops.b) <= 1e-8


@pytest.mark.gpu
def test_gpu_fd_solve_matches_oracle(ops):
    import torch
    from paper_2109_05451_b200 import operator_from_h2data, load_library
    from paper_2109_05451_b200.fd import solve_fd
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    load_library()
    opK = operator_from_h2data(ops.K, nv_max=1)
    opE = operator_from_h2data(ops.Khat, nv_max=1)
    u, it, hist, D = solve_fd(opK, opE, ops.idx, ops.C_rowptr, ops.C_col, ops.C_val, ops.C_diag, ops.prob.h,
                              ops.b, rtol=1e-8, maxit=300)
    opK.close()
    opE.close()
    Dref = ofd.fd_diag(ops.Khat, ops.idx)
    assert np.max(np.abs(D - Dref) / Dref) <= 1e-12
    x, it_ref, hist_ref = ofd.fd_solve(ops.K, Dref, ops.C_rowptr, ops.C_col, ops.C_val, ops.prob.h, ops.b, 1e-8, 300)
    assert abs(it - it_ref) <= 1
    assert hist[-1] <= 1e-8
    assert np.linalg.norm(u - x) / np.linalg.norm(x) <= 1e-7
    assert np.allclose(hist[:5], hist_ref[:5], rtol=1e-8)
