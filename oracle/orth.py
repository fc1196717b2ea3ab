"""Basis orthogonalization and the reweighing downsweep of an H² matrix (PAPER.md:540-608,
§"Algebraic Matrix Compression") — CPU oracle, TEST INFRASTRUCTURE (only tests/ may import it; the
product path never does).

The paper's pre-processing step of the recompression: "Orthogonalizing a
basis involves performing QR on the finest level basis and then going up the tree to compute new
transfer matrices that allow higher level nodes to satisfy the orthogonality condition ... an
upsweep pass that is very similar to the one described above for truncation, but replacing the
SVD operations by QR operations", written out step by step in the paper's order:

  leaves (level q):    U_t = Q_t R_t                         (QR of the m x k^q leaf basis)
                       U'_t = Q_t
  level l -> l-1:      M_p = [R_{c1} E_{c1}; R_{c2} E_{c2}]  (2 k^l x k^{l-1}, children c1, c2 of p;
                       M_p = Q_p R_p                          the transfer recursion of PAPER.md:135-142
                       E'_{c1} = Q_p[:k^l], E'_{c2} = Q_p[k^l:]  applied to U_c = Q_c R_c)
  the same for V with F, then every coupling block is re-expressed in the new bases (the projection
  of PAPER.md:610-613 with exact, untruncated bases):
                       S'_ts = R^U_t S_ts (R^V_s)^T
so U'_t S'_ts V'_s^T = U_t S_ts V_s^T: the operator is unchanged, every implied level basis
U'^l_t has orthonormal columns, and R^l_t is the R factor of the explicit level basis U^l_t.

Reading R21: QR factors are normalised to a non-negative diagonal of R (unique for
full-rank bases), the convention both this oracle and the GPU path use.  numpy.linalg.qr
(LAPACK Householder) is the library primitive of each step.  Requires m >= k^q and
2 k^l >= k^{l-1} (the QRs are reduced / thin).

Storage follows h2gen.H2Data (column-major batches: an r x c matrix is stored as (c, r)).
"""
import numpy as np


def qr_pos(A):
    """Thin QR with R's diagonal made non-negative (column signs of Q flipped to match)."""
    Q, R = np.linalg.qr(A, mode="reduced")
    s = np.where(np.diag(R) < 0, -1.0, 1.0)
    return Q * s[None, :], R * s[:, None]


def _orth_tree(leaf, T, q, ranks):
    """QR upsweep of one basis tree.  leaf: (2^q, k^q, m) stored; T[l]: (2^l, k^{l-1}, k^l)
    stored.  Returns (new leaf, new T, R) with R[l]: (2^l, k^l, k^l) stored column-major."""
    new_leaf = np.empty_like(leaf)
    new_T = [None] + [np.empty_like(T[l]) for l in range(1, q + 1)]
    R = [None] * (q + 1)
    kq = ranks[q]
    R[q] = np.empty((1 << q, kq, kq))
    for t in range(1 << q):
        Qt, Rt = qr_pos(leaf[t].T)                  # m x k^q
        new_leaf[t] = Qt.T
        R[q][t] = Rt.T
    for l in range(q, 0, -1):
        kl, kp = ranks[l], ranks[l - 1]
        R[l - 1] = np.empty((1 << (l - 1), kp, kp))
        for p in range(1 << (l - 1)):
            c1, c2 = 2 * p, 2 * p + 1
            M = np.vstack([R[l][c1].T @ T[l][c1].T,  # R_c E_c: (k^l x k^l)(k^l x k^{l-1})
                           R[l][c2].T @ T[l][c2].T])
            Qp, Rp = qr_pos(M)                      # 2 k^l x k^{l-1}
            new_T[l][c1] = Qp[:kl].T
            new_T[l][c2] = Qp[kl:].T
            R[l - 1][p] = Rp.T
    return new_leaf, new_T, R


def orthogonalize(h):
    """Orthogonalized copy of h (U, V, E, F, S replaced; D unchanged) and the R factors
    (RU, RV: per level, stored column-major)."""
    import copy
    assert h.m >= h.ranks[h.q] and all(2 * h.ranks[l] >= h.ranks[l - 1] for l in range(1, h.q + 1))
    U, E, RU = _orth_tree(h.U_leaf, h.E, h.q, h.ranks)
    V, F, RV = _orth_tree(h.V_leaf, h.F, h.q, h.ranks)
    S = []
    for l in range(h.q + 1):
        Sl = np.empty_like(h.S[l])
        rp, col = h.S_rowptr[l], h.S_col[l]
        for t in range(len(rp) - 1):
            for b in range(rp[t], rp[t + 1]):
                s = col[b]
                Sl[b] = (RU[l][t].T @ h.S[l][b].T @ RV[l][s]).T      # R^U_t S (R^V_s)^T
        S.append(Sl)
    g = copy.copy(h)
    g.U_leaf, g.V_leaf, g.E, g.F, g.S = U, V, E, F, S
    return g, RU, RV


def reweigh_R(g):
    """The reweighing downsweep of the recompression, on an H² matrix g whose
    V basis is orthogonal (the output of orthogonalize): for every node i of every level, root to
    leaves, the R factor of the stacked small matrix of Eq. (Btq),

        B^l_i -> [ R^{l-1}_{i+} E^{lT}_i ; S^{lT}_{ij_1} ; ... ; S^{lT}_{ij_b} ]

    (the parent part absent at the root; an empty stack gives R = 0).  Returns R[l]: (2^l, k^l, k^l)
    stored column-major (R^l_i = R[l][i].T, upper triangular, diag >= 0).  The new basis of level l
    is U^l_i R^{lT}_i."""
    q, k = g.q, g.ranks
    R = [None] * (q + 1)
    for l in range(q + 1):
        kl = k[l]
        R[l] = np.zeros((1 << l, kl, kl))
        for i in range(1 << l):
            parts = []
            if l >= 1:
                parts.append(R[l - 1][i >> 1].T @ g.E[l][i])            # R_{i+} (k^{l-1} sq) E_i^T
            rp, col = g.S_rowptr[l], g.S_col[l]
            for b in range(rp[i], rp[i + 1]):
                parts.append(g.S[l][b])                                 # stored (k, k) col-major = S^T
            if not parts:
                continue
            M = np.vstack(parts)
            _, Ri = qr_pos(M)                                           # (min(rows, k), k)
            Rf = np.zeros((kl, kl))
            Rf[:Ri.shape[0]] = Ri
            R[l][i] = Rf.T
    return R
