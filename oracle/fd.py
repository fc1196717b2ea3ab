"""Oracle of the fractional-diffusion solve (TEST INFRASTRUCTURE):

    A u = h^2 (D + K + C) u = b,   D = diag(K^ 1) restricted to the interior

K and K^ applied with the oracle's own H² matvec (oracle.matvec), C as given (CSR), and the
textbook preconditioned conjugate gradient method (Saad, Iterative Methods, Alg. 9.1)
with the Jacobi preconditioner diag(A), in that order and nothing fused.  Plain numpy, FP64."""
import numpy as np

from . import matvec


def fd_diag(hkhat, idx):
    """D_ii = (K^ 1)[idx[i]]: one oracle H² matvec of the extended-grid operator with ones."""
    ones = np.ones((1, hkhat.N))
    return matvec(hkhat, ones, 1.0, 0.0)[0][np.asarray(idx)]


def csr_apply(rp, col, val, x):
    y = np.zeros_like(x)
    for i in range(rp.size - 1):
        a, b = rp[i], rp[i + 1]
        y[i] = np.dot(val[a:b], x[col[a:b]])
    return y


def pcg(apply_A, b, minv, rtol, maxit, x0=None):
    """Preconditioned CG (Alg. 9.1): returns (x, iterations, relative residual history)."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - apply_A(x)
    z = minv * r
    p = z.copy()
    rz = float(r @ z)
    bn = float(np.linalg.norm(b)) or 1.0
    hist = [float(np.linalg.norm(r)) / bn]
    it = 0
    while it < maxit and hist[-1] > rtol:
        q = apply_A(p)
        alpha = rz / float(p @ q)
        x = x + alpha * p
        r = r - alpha * q
        z = minv * r
        rz_new = float(r @ z)
        p = z + (rz_new / rz) * p
        rz = rz_new
        it += 1
        hist.append(float(np.linalg.norm(r)) / bn)
    return x, it, hist


def fd_solve(hK, D, C_rowptr, C_col, C_val, h, b, rtol=1e-8, maxit=500):
    """Solve h^2 (D + K + C) u = b; C's diagonal is part of C (CSR with its diagonal)."""
    cdiag = np.zeros(b.size)
    for i in range(b.size):
        a, e = C_rowptr[i], C_rowptr[i + 1]
        m = C_col[a:e] == i
        cdiag[i] = C_val[a:e][m].sum()

    def apply_A(u):
        Ku = matvec(hK, u[None, :], 1.0, 0.0)[0]
        return h * h * (D * u + Ku + csr_apply(C_rowptr, C_col, C_val, u))
    minv = 1.0 / (h * h * (D + cdiag))
    return pcg(apply_A, b, minv, rtol, maxit)
