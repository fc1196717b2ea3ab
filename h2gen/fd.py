"""Input side of the fractional-diffusion solve:

    h^2 (D + K + C) u = b ,   b = 1 on Omega = [-1, 1]^2,  u = 0 on Omega_0 = [-3, 3]^2 \\ Omega

* interior grid: n x n points x = -1 + (i+1) h, h = 2 / (n+1) (reading R10)
* K: the H² operator of the FD kernel -2 a(x, y) / |x - y|^(2+2beta), K_ii = 0, on the interior points
  (workload cfg4's operator; built with h2gen.build_h2)
* D: D_ii = sum_{j != i, y_j in Omega u Omega_0} 2 a(x_i, y_j) / |y_j - x_i|^(2+2beta), recast as
  K^ 1 on the extended grid of Omega u Omega_0 at the same spacing -- the matvec is
  the method's; this module only builds the extended point set and the interior index map
* C: the sparse correction with the footprint of a 5-point Laplacian.  The paper
  defers its entries to a companion paper; we use SPEC.md:506's stand-in (reading R19): the
  5-point discretisation of -div(kappa grad u) with harmonic-mean edge coefficients, scaled by
  h^(-2 beta - 2), Omega_0 neighbours contributing to the diagonal only (u = 0 there).

No arithmetic of the matvec or the solver lives here."""
from dataclasses import dataclass

import numpy as np

from .kernels import fd_kappa


@dataclass
class FDProblem:
    n: int
    h: float
    beta: float
    interior: np.ndarray      # (n^2, 2) row-major grid order (i fastest along axis 0)
    extended: np.ndarray      # (ne^2, 2) extended grid, row-major
    ext_interior: np.ndarray  # (n^2,) index of each interior point in `extended`
    C_rowptr: np.ndarray      # CSR of C in the interior's row-major order
    C_col: np.ndarray
    C_val: np.ndarray
    b: np.ndarray             # (n^2,) right-hand side (ones)


def fd_problem(n, beta=0.75):
    h = 2.0 / (n + 1)
    ax = -1.0 + h * np.arange(1, n + 1)
    gi, gj = np.meshgrid(ax, ax, indexing="ij")
    interior = np.stack([gi.reshape(-1), gj.reshape(-1)], axis=1)
    # extended grid: -1 + j h for every j with the point inside [-3, 3]: j = -(n+1) .. 2(n+1)
    J = np.arange(-(n + 1), 2 * (n + 1) + 1)
    ex = -1.0 + h * J
    ne = ex.size
    ei, ej = np.meshgrid(ex, ex, indexing="ij")
    extended = np.stack([ei.reshape(-1), ej.reshape(-1)], axis=1)
    off = n + 1                                   # extended index of interior j = 1 is off + 1
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    ext_interior = ((ii + 1 + off) * ne + (jj + 1 + off)).reshape(-1)
    # C: 5-point stencil of -div(kappa grad u), harmonic-mean edge coefficients, x h^(-2 beta - 2)
    kap = fd_kappa(interior).reshape(n, n)
    scale = h ** (-2.0 * beta - 2.0)
    rows, cols, vals = [], [], []
    idx = np.arange(n * n).reshape(n, n)
    diag = np.zeros((n, n))
    for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        # neighbour coordinates and its kappa (outside Omega: on Omega_0, kappa from the field)
        pi, pj = ii + di, jj + dj
        inside = (pi >= 0) & (pi < n) & (pj >= 0) & (pj < n)
        nb = np.stack([-1.0 + h * (pi + 1), -1.0 + h * (pj + 1)], axis=-1)
        kn = fd_kappa(nb)
        ke = 2.0 * kap * kn / (kap + kn)
        diag += ke
        rows.append(idx[inside])
        cols.append(idx[pi[inside], pj[inside]])
        vals.append(-ke[inside])
    rows.append(idx.reshape(-1))
    cols.append(idx.reshape(-1))
    vals.append(diag.reshape(-1))
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    v = np.concatenate(vals) * scale
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rowptr = np.zeros(n * n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n * n), out=rowptr[1:])
    return FDProblem(n, h, beta, interior, extended, ext_interior, rowptr, c.astype(np.int32), v,
                     np.ones(n * n))


def permute_csr(rowptr, col, val, perm):
    """CSR of P C P^T for tree order: new row r = old row perm[r]; columns mapped likewise."""
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    counts = np.diff(rowptr)[perm]
    nrp = np.zeros(perm.size + 1, dtype=np.int64)
    np.cumsum(counts, out=nrp[1:])
    take = np.concatenate([np.arange(rowptr[p], rowptr[p + 1]) for p in perm]) if perm.size else np.zeros(0, int)
    ncol = inv[col[take]].astype(np.int32)
    nval = val[take]
    # keep columns ascending within a row
    for rr in range(perm.size):
        a, b = nrp[rr], nrp[rr + 1]
        o = np.argsort(ncol[a:b], kind="stable")
        ncol[a:b] = ncol[a:b][o]
        nval[a:b] = nval[a:b][o]
    return nrp, ncol, nval


@dataclass
class FDOperators:
    prob: FDProblem
    K: object            # H2Data of K on the interior points (tree order)
    Khat: object         # H2Data of K^ on the extended grid (tree order)
    idx: np.ndarray      # K tree position -> K^ tree position of the same point
    C_rowptr: np.ndarray  # C in K's tree order (diagonal included)
    C_col: np.ndarray
    C_val: np.ndarray
    C_diag: np.ndarray
    b: np.ndarray        # tree order


def build_fd_operators(n, m=64, p=6, eta=0.9, beta=0.75):
    """Inputs of the FD solve at grid side n: K (kernel sign -1) on the interior points and K^
    (sign +1) on the extended grid as Chebyshev H² data (reading R8/R10), the index map between
    their tree orders, C permuted to K's tree order, b = 1."""
    from .tree import build_cluster_tree
    from .structure import dual_traversal
    from .kernels import Kernel
    from .h2data import build_h2
    prob = fd_problem(n, beta)
    tK = build_cluster_tree(prob.interior, m)
    hK = build_h2(tK, dual_traversal(tK, eta), Kernel("fd", beta=beta, sign=-1.0), p)
    tE = build_cluster_tree(prob.extended, m)
    hE = build_h2(tE, dual_traversal(tE, eta), Kernel("fd", beta=beta, sign=1.0), p)
    invE = np.empty_like(tE.perm)
    invE[tE.perm] = np.arange(tE.perm.size)
    idx = invE[prob.ext_interior[tK.perm]]
    rp, col, val = permute_csr(prob.C_rowptr, prob.C_col, prob.C_val, tK.perm)
    rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    cdiag = np.zeros(rp.size - 1)
    np.add.at(cdiag, rows[col == rows], val[col == rows])
    return FDOperators(prob, hK, hE, idx.astype(np.int64), rp, col, val, cdiag, prob.b[tK.perm])
