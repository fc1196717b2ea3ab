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
