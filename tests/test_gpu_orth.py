"""GPU parity of the basis orthogonalization (h2_orthogonalize, NEXT-3 step 1)
against the oracle (oracle/orth.py, pinned in test_orth_oracle.py): every new array element by
element -- leaf bases, transfers, coupling blocks (QR factors are unique with diag R >= 0) -- and
the operator unchanged (matvec after orthogonalization vs the oracle of the ORIGINAL operator)."""
import numpy as np
import pytest

import oracle
from oracle.orth import orthogonalize
from h2gen import make_xy
from tests.gpu_util import gpu_matvec, colmax_rel
from tests.test_orth_oracle import CASES

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", sorted(CASES))
def test_orthogonalize_parity(name):
    from paper_2109_05451_b200 import operator_from_h2data
    from paper_2109_05451_b200._binding import H2_EXPORT_S, H2_EXPORT_U, H2_EXPORT_VT, H2_EXPORT_E, H2_EXPORT_FT
    h = CASES[name]()
    g, _, _ = orthogonalize(h)
    nv = 4
    op = operator_from_h2data(h, nv_max=nv)
    X = make_xy(h.perm, nv, 11, -1.0, 1.0)
    Y0 = make_xy(h.perm, nv, 12, -1.0, 1.0, stream=1)
    before = gpu_matvec(op, X, 0.8, -0.3, Y0)            # also captures the graph before the change
    op.orthogonalize()
    q, m, kq = h.q, h.m, h.ranks[h.q]
    nleaf = 1 << q
    U = op.export(H2_EXPORT_U, q, nleaf * m * kq).reshape(nleaf, kq, m)
    assert _rel(U, g.U_leaf) <= 1e-10
    Vt = op.export(H2_EXPORT_VT, q, nleaf * m * kq).reshape(nleaf, m, kq)
    assert _rel(np.transpose(Vt, (0, 2, 1)), g.V_leaf) <= 1e-10
    for l in range(1, q + 1):
        kl, kp = h.ranks[l], h.ranks[l - 1]
        E = op.export(H2_EXPORT_E, l, (1 << l) * kl * kp).reshape(1 << l, kp, kl)
        assert _rel(E, g.E[l]) <= 1e-10, l
        Ft = op.export(H2_EXPORT_FT, l, (1 << l) * kl * kp).reshape(1 << l, kl, kp)
        assert _rel(np.transpose(Ft, (0, 2, 1)), g.F[l]) <= 1e-10, l
    for l in range(q + 1):
        nb, k = g.S[l].shape[0], h.ranks[l]
        if nb == 0:
            continue
        S = op.export(H2_EXPORT_S, l, nb * k * k).reshape(nb, k, k)
        assert _rel(S, g.S[l]) <= 1e-10, l
    after = gpu_matvec(op, X, 0.8, -0.3, Y0)
    ref = oracle.matvec(h, X, 0.8, -0.3, Y0)
    assert colmax_rel(before, ref) <= 1e-12
    assert colmax_rel(after, ref) <= 1e-12
    op.close()


def test_orthogonalize_rejects_unsupported():
    from paper_2109_05451_b200 import operator_from_h2data
    from paper_2109_05451_b200._binding import H2Error
    h = CASES["uniform-k8"]()
    op = operator_from_h2data(h.astype(np.float32), dtype="f32", nv_max=1)
    with pytest.raises(H2Error):
        op.orthogonalize()
    op.close()


@pytest.mark.parametrize("name", sorted(CASES))
def test_reweigh_parity(name):
    """h2_reweigh after h2_orthogonalize vs the oracle's reweighing downsweep (pinned against the
    brute-force block-row Gram matrices in test_orth_oracle.py): every R^l_i element by element
    (rows whose stack is rank deficient compared through R^T R, the unique part)."""
    import torch
    from paper_2109_05451_b200 import operator_from_h2data
    from oracle.orth import reweigh_R
    h = CASES[name]()
    g, _, _ = orthogonalize(h)
    Rref = reweigh_R(g)
    op = operator_from_h2data(h, nv_max=1)
    op.orthogonalize()
    n = sum((1 << l) * h.ranks[l] ** 2 for l in range(h.q + 1))
    Rd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
    op.reweigh(Rd)
    R = Rd.cpu().numpy()
    off = 0
    for l in range(h.q + 1):
        k = h.ranks[l]
        got = R[off:off + (1 << l) * k * k].reshape(1 << l, k, k)
        off += (1 << l) * k * k
        for i in range(1 << l):
            a, b = got[i].T, Rref[l][i].T
            scale = max(np.abs(b).max(), 1e-300)
            G = b.T @ b
            assert np.abs(a.T @ a - G).max() <= 1e-10 * max(np.abs(G).max(), 1e-300), (l, i)
            w = np.linalg.eigvalsh(G) if scale > 1e-300 else np.zeros(1)
            if w.min() > 1e-8 * max(w.max(), 1e-300):
                assert np.abs(a - b).max() <= 1e-9 * scale, (l, i)
    op.close()


def test_reweigh_and_export_argument_checks():
    """Wrong sizes and unknown arrays are rejected (H2_ERR_ARG), nothing is written."""
    import torch
    from paper_2109_05451_b200 import operator_from_h2data
    from paper_2109_05451_b200._binding import H2Error, H2_EXPORT_S
    h = CASES["uniform-k8"]()
    op = operator_from_h2data(h, nv_max=1)
    n = sum((1 << l) * h.ranks[l] ** 2 for l in range(h.q + 1))
    with pytest.raises(H2Error):
        op.reweigh(torch.zeros(n - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        op.reweigh(torch.zeros(n, dtype=torch.float32, device="cuda"))
    with pytest.raises(H2Error):
        op.export(H2_EXPORT_S, h.q, 1)                          # wrong count
    with pytest.raises(H2Error):
        op.export(99, 0, 1)                                     # unknown array
    with pytest.raises(H2Error):
        op.export(H2_EXPORT_S, h.q + 1, 1)                      # level out of range
    op.close()
