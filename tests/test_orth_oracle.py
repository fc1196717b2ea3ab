"""Pins of the basis-orthogonalization oracle (oracle/orth.py, NEXT-3's first step)
to things other than itself: the operator is unchanged (brute-force dense assembly), every implied
level basis has orthonormal columns (explicit expansion of the transfer recursion), and each R^l_t
equals the textbook QR factor of the ORIGINAL explicit level basis (not the recursion).  CPU."""
import numpy as np
import pytest

from h2gen import build_cluster_tree, dual_traversal, random_h2_data
from h2gen.tree import uniform_points
from h2gen.configs import build_config
from oracle.orth import orthogonalize, qr_pos
from tests.dense_assembly import assemble, explicit_bases


def _case(N, m, ranks_fn, seed, eta=0.9):
    tr = build_cluster_tree(uniform_points(N, 2, seed), m)
    st = dual_traversal(tr, eta)
    return random_h2_data(tr, st, [ranks_fn(l) for l in range(tr.q + 1)], seed + 100)


CASES = {
    "uniform-k8": lambda: _case(900, 32, lambda l: 8, 3),
    "ranks-by-level": lambda: _case(1100, 32, lambda l: 6 + (l % 3), 5),   # 2 k^l >= k^{l-1}
    "cfg1-chebyshev": lambda: build_config("cfg1"),
}


@pytest.fixture(scope="module", params=sorted(CASES))
def orth(request):
    h = CASES[request.param]()
    g, RU, RV = orthogonalize(h)
    return h, g, RU, RV


def test_operator_unchanged(orth):
    h, g, _, _ = orth
    A, _ = assemble(h)
    B, _ = assemble(g)
    assert np.linalg.norm(A - B) <= 1e-12 * np.linalg.norm(A)


@pytest.mark.parametrize("which", ["U", "V"])
def test_level_bases_orthonormal(orth, which):
    _, g, _, _ = orth
    for (l, i), B in explicit_bases(g, which).items():
        k = B.shape[1]
        assert np.abs(B.T @ B - np.eye(k)).max() <= 1e-12, (l, i)


@pytest.mark.parametrize("which", ["U", "V"])
def test_R_is_qr_of_explicit_basis(orth, which):
    """R^l_t (from the upsweep recursion) == R factor of the original explicit basis U^l_t."""
    h, _, RU, RV = orth
    R = RU if which == "U" else RV
    for (l, i), B in explicit_bases(h, which).items():
        if B.shape[0] < B.shape[1]:
            continue                                   # rank-deficient leaf: R not unique
        _, Rt = qr_pos(B)
        Rr = R[l][i].T
        assert np.abs(Rr - Rt).max() <= 1e-10 * max(1.0, np.abs(Rt).max()), (l, i)
        assert np.allclose(np.tril(Rr, -1), 0.0) and (np.diag(Rr) >= 0).all()


def _rows(h, l, i):
    sh = h.q - l
    return h.leaf_ptr[i << sh], h.leaf_ptr[(i + 1) << sh]


def test_reweigh_R_is_cholesky_of_block_row_gram(orth):
    """Reweighing downsweep: R^l_i^T R^l_i == B^l_iT B^l_i, with B^l_iT = U^lT_i
    A^l_i built by brute force -- A^l_i = the rows of cluster i of every low-rank block at levels
    <= l (the coarser blocks restricted to i's rows and the level-l blocks of row i) -- and, where
    that Gram matrix is well conditioned, R^l_i == its Cholesky factor (unique, positive diagonal)."""
    from oracle.orth import reweigh_R
    _, g, _, _ = orth
    R = reweigh_R(g)
    UB, VB = explicit_bases(g, "U"), explicit_bases(g, "V")
    A = np.zeros((g.N, g.N))
    for l in range(g.q + 1):
        rp, col = g.S_rowptr[l], g.S_col[l]
        for t in range(len(rp) - 1):
            r0, r1 = _rows(g, l, t)
            for b in range(rp[t], rp[t + 1]):
                s = col[b]
                c0, c1 = _rows(g, l, s)
                A[r0:r1, c0:c1] += UB[(l, t)] @ g.S[l][b].T @ VB[(l, s)].T
        for i in range(1 << l):
            r0, r1 = _rows(g, l, i)
            Bt = UB[(l, i)].T @ A[r0:r1]                 # k x N
            G = Bt @ Bt.T
            Ri = R[l][i].T
            scale = max(np.abs(G).max(), 1e-300)
            assert np.abs(Ri.T @ Ri - G).max() <= 1e-10 * scale, (l, i)
            assert np.allclose(np.tril(Ri, -1), 0.0) and (np.diag(Ri) >= 0).all()
            w = np.linalg.eigvalsh(G)
            if w.min() > 1e-8 * w.max():
                Lc = np.linalg.cholesky(G)
                assert np.abs(Ri - Lc.T).max() <= 1e-8 * max(1.0, np.abs(Lc).max()), (l, i)
