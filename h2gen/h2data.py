"""H² data: explicit leaf bases U, V (m x k^q), interlevel transfers
E, F (k^l x k^{l-1}), per-level coupling blocks S^l_ts (k^l x k^l) on the admissible blocks,
and dense leaf blocks A_de (m x m) on the inadmissible leaf pairs.

Chebyshev construction (reading R8): first-kind nodes cos(pi(2i+1)/(2p))
mapped to each cluster's bounding box, tensor Lagrange leaf bases, transfer (a,b) =
L^parent_b(xi^child_a), coupling (a,b) = K(xi^t_a, xi^s_b); U = V, E = F for symmetric
kernels.  Tensor index a = sum_d a_d p^d (dimension 0 fastest).

Column-major storage: a batch of r x c matrices is an array of shape (batch, c, r)."""
from dataclasses import dataclass
import itertools
import math
import os
from concurrent.futures import ThreadPoolExecutor
import numpy as np

from .tree import ClusterTree
from .structure import BlockStructure
from .kernels import Kernel


@dataclass
class H2Data:
    dim: int
    N: int
    m: int
    q: int
    ranks: list            # k^l, l = 0..q
    perm: np.ndarray       # tree position -> original point id
    points: np.ndarray     # (N, dim) tree order
    leaf_ptr: np.ndarray   # (2^q + 1,) int64
    U_leaf: np.ndarray     # (2^q, k^q, m)   col-major m x k^q per leaf, rows >= leaf size are 0
    V_leaf: np.ndarray
    E: list                # [q+1]; E[0] None; E[l]: (2^l, k^{l-1}, k^l) col-major k^l x k^{l-1}
    F: list
    S_rowptr: list         # [q+1] int64
    S_col: list            # [q+1] int32
    S: list                # [q+1]; (nblk_l, k^l, k^l) col-major
    D_rowptr: np.ndarray
    D_col: np.ndarray
    D: np.ndarray          # (n_D, m, m) col-major
    eta: float = 0.0
    kernel: object = None

    @property
    def n_S(self):
        return int(sum(c.size for c in self.S_col))

    @property
    def n_D(self):
        return int(self.D_col.size)

    def csp(self):
        return max(int(np.diff(rp).max(initial=0)) for rp in self.S_rowptr)

    def operator_scalars(self):
        """Stored operator scalars (U, V, E, F counted separately): SURVEY.md §8(d) `ops`."""
        n = self.U_leaf.size + self.V_leaf.size + self.D.size
        n += sum(e.size for e in self.E[1:]) + sum(f.size for f in self.F[1:])
        n += sum(s.size for s in self.S)
        return int(n)

    def flops(self, nv):
        """Paper's flop convention (pinned to 1%): 2 nv ops."""
        return 2.0 * nv * self.operator_scalars()

    def nbytes(self, nv, wbytes=8, beta_nonzero=False):
        """Algorithmic bytes per matvec: operator once + X read + Y write
        (+ Y read if beta != 0) + x^ / y^ trees written and read once each."""
        tree = sum((1 << l) * self.ranks[l] for l in range(self.q + 1))
        vec = self.N * (2 + (1 if beta_nonzero else 0)) + 4 * tree
        return wbytes * (self.operator_scalars() + nv * vec)

    def astype(self, dt):
        """Copy with every float array cast to dt (used for the FP32 path and its oracle input)."""
        c = lambda a: None if a is None else a.astype(dt)
        sym_u = self.U_leaf is self.V_leaf
        U = c(self.U_leaf)
        E = [c(e) for e in self.E]
        sym_e = all(a is b for a, b in zip(self.E, self.F))
        return H2Data(self.dim, self.N, self.m, self.q, list(self.ranks), self.perm, self.points,
                      self.leaf_ptr, U, U if sym_u else c(self.V_leaf), E,
                      E if sym_e else [c(f) for f in self.F], self.S_rowptr, self.S_col,
                      [c(s) for s in self.S], self.D_rowptr, self.D_col, c(self.D), self.eta,
                      self.kernel)


# ----------------------------------------------------------------------------------------
# Chebyshev tensor interpolation (generator side)

def cheb_nodes_1d(p):
    i = np.arange(p, dtype=np.float64)
    return np.cos(np.pi * (2 * i + 1) / (2 * p))


def _box_nodes(lo, hi, p):
    """lo, hi: (n, dim) -> 1D nodes per dim (n, dim, p) mapped to the boxes.  A zero extent is
    widened to 1e-3 x the box's largest half-extent (or 1e-12) so the Lagrange basis exists
    (interpolation stays exact for any positive width; reading R8)."""
    c = 0.5 * (lo + hi)
    h = 0.5 * (hi - lo)
    hmax = np.max(h, axis=1, keepdims=True)
    floor = np.maximum(1e-3 * hmax, 1e-12)
    h = np.where(h > 0, h, floor)
    return c[:, :, None] + h[:, :, None] * cheb_nodes_1d(p)[None, None, :]


def _lagrange_1d(nodes, x):
    """nodes (n, p), x (n, r) -> L (n, r, p), L[.., r, a] = prod_{b != a} (x_r - n_b)/(n_a - n_b)."""
    n, p = nodes.shape
    L = np.ones(x.shape + (p,))
    for a in range(p):
        for b in range(p):
            if a != b:
                L[..., a] *= (x - nodes[:, b:b + 1]) / (nodes[:, a:a + 1] - nodes[:, b:b + 1])
    return L


def _tensor_index(p, dim):
    """multi-indices a (k, dim) with a = sum_d a_d p^d (dim 0 fastest)."""
    k = p ** dim
    idx = np.arange(k)
    return np.stack([(idx // p ** d) % p for d in range(dim)], axis=1)


def _tensor_points(nodes1d, p, dim):
    """nodes1d (n, dim, p) -> tensor Chebyshev points (n, k, dim)."""
    mi = _tensor_index(p, dim)
    return np.stack([nodes1d[:, d, :][:, mi[:, d]] for d in range(dim)], axis=2)


def _tensor_lagrange(nodes1d, x, p):
    """nodes1d (n, dim, p), x (n, r, dim) -> (n, r, k) tensor Lagrange values."""
    n, dim, _ = nodes1d.shape
    mi = _tensor_index(p, dim)
    out = None
    for d in range(dim):
        Ld = _lagrange_1d(nodes1d[:, d, :], x[:, :, d])   # (n, r, p)
        Ld = Ld[:, :, mi[:, d]]
        out = Ld if out is None else out * Ld
    return out


def _leaf_point_index(leaf_ptr, m):
    """(2^q, m) tree-order point index per leaf row, -1 for padding rows."""
    nleaf = leaf_ptr.size - 1
    idx = leaf_ptr[:-1, None] + np.arange(m)[None, :]
    return np.where(idx < leaf_ptr[1:, None], idx, -1)


def build_h2(tree: ClusterTree, st: BlockStructure, kernel: Kernel, p: int, chunk=2048):
    dim, q, m = tree.dim, tree.q, tree.m
    k = p ** dim
    ranks = [k] * (q + 1)
    nodes = [_box_nodes(tree.lo[l], tree.hi[l], p) for l in range(q + 1)]   # (2^l, dim, p)
    chebpts = [_tensor_points(nodes[l], p, dim) for l in range(q + 1)]       # (2^l, k, dim)
    # leaf bases: U[s, a, i] = L^s_a(x_i)
    pidx = _leaf_point_index(tree.leaf_ptr, m)
    lp = tree.points[np.maximum(pidx, 0)]                                   # (2^q, m, dim)
    U = _tensor_lagrange(nodes[q], lp, p)                                   # (2^q, m, k)
    U[pidx < 0] = 0.0
    U = np.ascontiguousarray(U.transpose(0, 2, 1))                          # (2^q, k, m)
    # transfers: E_c (k x k col-major), E_c[a, b] = L^parent_b(xi^child_a) -> stored [c, b, a]
    E = [None]
    for l in range(1, q + 1):
        par = np.arange(1 << l) // 2
        vals = _tensor_lagrange(nodes[l - 1][par], chebpts[l], p)          # (2^l, k_child a, k_par b)
        E.append(np.ascontiguousarray(vals.transpose(0, 2, 1)))
    pool = ThreadPoolExecutor(max(1, min(16, len(os.sched_getaffinity(0)))))
    # couplings S_ts[a, b] = K(xi^t_a, xi^s_b) -> stored [blk, b, a]
    S = []
    for l in range(q + 1):
        rp, col = st.S_rowptr[l], st.S_col[l]
        rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
        out = np.empty((col.size, k, k))

        def fill_s(b0, l=l, rows=rows, col=col, out=out):
            b1 = min(col.size, b0 + chunk)
            xt = chebpts[l][rows[b0:b1]]                                    # (nb, k, dim)
            xs = chebpts[l][col[b0:b1]]
            out[b0:b1] = kernel(xs[:, :, None, :], xt[:, None, :, :])       # [b, beta, alpha]
        list(pool.map(fill_s, range(0, col.size, chunk)))
        S.append(out)
    # dense D_ts[i, j] = K(x_i, x_j) -> stored [blk, j, i]; zero on padding rows/cols
    rows = np.repeat(np.arange(st.D_rowptr.size - 1), np.diff(st.D_rowptr))
    D = np.empty((st.n_D, m, m))

    def fill_d(b0):
        b1 = min(st.n_D, b0 + chunk)
        it, js = pidx[rows[b0:b1]], pidx[st.D_col[b0:b1]]
        xi = tree.points[np.maximum(it, 0)]
        xj = tree.points[np.maximum(js, 0)]
        v = kernel(xj[:, :, None, :], xi[:, None, :, :])                    # [b, j, i]
        v *= (js >= 0)[:, :, None] & (it >= 0)[:, None, :]
        D[b0:b1] = v
    list(pool.map(fill_d, range(0, st.n_D, chunk)))
    pool.shutdown()
    return H2Data(dim, tree.N, m, q, ranks, tree.perm, tree.points, tree.leaf_ptr, U, U, E, E,
                  st.S_rowptr, st.S_col, S, st.D_rowptr, st.D_col, D, st.eta, kernel)


def random_h2_data(tree: ClusterTree, st: BlockStructure, ranks, seed, symmetric=False):
    """Random H² data on a real block structure: U != V, E != F, unsymmetric S and D, and
    per-level ranks k^l that may differ between levels.  Independent uniform(-1, 1) entries,
    transfers scaled by 1/sqrt(k^l) so the x^ / y^ trees stay O(1).  A transposed operand or
    a swapped k^l / k^{l-1} anywhere changes the result (used by parity tests)."""
    rng = np.random.default_rng(seed)
    q, m = tree.q, tree.m
    ranks = list(ranks)
    assert len(ranks) == q + 1
    u = lambda *shape: rng.uniform(-1.0, 1.0, size=shape)
    pidx = _leaf_point_index(tree.leaf_ptr, m)
    pad = (pidx < 0)[:, None, :]
    U = u(1 << q, ranks[q], m) / math.sqrt(m)
    U[np.broadcast_to(pad, U.shape)] = 0.0
    V = U if symmetric else u(1 << q, ranks[q], m) / math.sqrt(m)
    if not symmetric:
        V[np.broadcast_to(pad, V.shape)] = 0.0
    E, F = [None], [None]
    for l in range(1, q + 1):
        e = u(1 << l, ranks[l - 1], ranks[l]) / math.sqrt(ranks[l])
        E.append(e)
        F.append(e if symmetric else u(1 << l, ranks[l - 1], ranks[l]) / math.sqrt(ranks[l]))
    S = [u(st.S_col[l].size, ranks[l], ranks[l]) / ranks[l] for l in range(q + 1)]
    D = u(st.n_D, m, m) / m
    rows_pad = np.broadcast_to(pad, (1 << q, m, m))   # leaf row i of padding -> zero
    if st.n_D:
        rows = np.repeat(np.arange(1 << q), np.diff(st.D_rowptr))
        D *= ~(pidx[st.D_col] < 0)[:, :, None]          # padding columns j
        D *= ~(pidx[rows] < 0)[:, None, :]              # padding rows i
    return H2Data(tree.dim, tree.N, m, q, ranks, tree.perm, tree.points, tree.leaf_ptr, U, V,
                  E, F, st.S_rowptr, st.S_col, S, st.D_rowptr, st.D_col, D, st.eta, None)


def poly_kernel_apply(points, X, p):
    """Closed form of Y = K X for K(x, y) = (1 + x.y)^(p-1), O(N x #monomials):
    K(x, y) = sum_{|a| <= p-1} c_a x^a y^a with multinomial c_a = (p-1)! / (a! (p-1-|a|)!),
    so y_i = sum_a c_a x_i^a M_a with moments M_a = sum_j x_j^a X_j.
    points (N, dim), X (nv, N) -> (nv, N).  Independent of the H² machinery (pin only)."""
    N, dim = points.shape
    n = p - 1
    Y = np.zeros_like(X)
    for a in itertools.product(range(n + 1), repeat=dim):
        if sum(a) > n:
            continue
        c = math.factorial(n) / (math.prod(math.factorial(ai) for ai in a) * math.factorial(n - sum(a)))
        mono = np.prod(points ** np.array(a)[None, :], axis=1)     # (N,)
        M = X @ mono                                               # (nv,)
        Y += c * M[:, None] * mono[None, :]
    return Y
