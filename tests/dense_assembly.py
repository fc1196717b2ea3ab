"""Brute-force dense assembly of A~ from its definition (test helper, independent of oracle/):

    A~ = A_de + <U, S, V^T>,  every block (t, s) at level l assembled as U^l_t S^l_ts V^l_s^T
    (PAPER.md:145-150), with the inner bases expanded explicitly by the transfer recursion
    U^{l-1}_i = diag(U^l_{i1}, U^l_{i2}) [E^l_{i1}; E^l_{i2}].

Also returns the coverage count of every (i, j) (partition property)."""
import numpy as np


def explicit_bases(h, which="U"):
    """{(l, i): (rows, k^l) explicit basis over the cluster's real rows}"""
    leaf = h.U_leaf if which == "U" else h.V_leaf
    T = h.E if which == "U" else h.F
    q = h.q
    out = {}
    for i in range(1 << q):
        n = h.leaf_ptr[i + 1] - h.leaf_ptr[i]
        out[(q, i)] = leaf[i].T[:n, :]                 # stored (k, m) -> m x k, real rows
    for l in range(q, 0, -1):
        for i in range(1 << (l - 1)):
            c0, c1 = 2 * i, 2 * i + 1
            E0 = T[l][c0].T                            # stored (k^{l-1}, k^l) -> k^l x k^{l-1}
            E1 = T[l][c1].T
            out[(l - 1, i)] = np.vstack([out[(l, c0)] @ E0, out[(l, c1)] @ E1])
    return out


def assemble(h):
    N, q = h.N, h.q
    lp = h.leaf_ptr
    Ub = explicit_bases(h, "U")
    Vb = explicit_bases(h, "V") if h.V_leaf is not h.U_leaf or any(
        a is not b for a, b in zip(h.E, h.F)) else Ub
    A = np.zeros((N, N))
    cover = np.zeros((N, N), dtype=np.int32)

    def rng(l, i):
        a = lp[i << (q - l)]
        b = lp[(i + 1) << (q - l)]
        return a, b

    for l in range(q + 1):
        rp, col, S = h.S_rowptr[l], h.S_col[l], h.S[l]
        for t in range(1 << l):
            r0, r1 = rng(l, t)
            for b in range(rp[t], rp[t + 1]):
                s = col[b]
                c0, c1 = rng(l, s)
                A[r0:r1, c0:c1] += Ub[(l, t)] @ S[b].T @ Vb[(l, s)].T
                cover[r0:r1, c0:c1] += 1
    for t in range(1 << q):
        r0, r1 = lp[t], lp[t + 1]
        for b in range(h.D_rowptr[t], h.D_rowptr[t + 1]):
            s = h.D_col[b]
            c0, c1 = lp[s], lp[s + 1]
            A[r0:r1, c0:c1] += h.D[b].T[: r1 - r0, : c1 - c0]
            cover[r0:r1, c0:c1] += 1
    return A, cover
