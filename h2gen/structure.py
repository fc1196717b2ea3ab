"""Block structure of the matrix tree by dual-tree traversal with the geometric
admissibility condition  eta * ||C_t - C_s|| >= (D_t + D_s) / 2  (
reading R4: bounding boxes of the point sets, equality admissible, child pairs of
inadmissible pairs starting from (root, root), inadmissible leaf pairs -> dense)."""
from dataclasses import dataclass
import numpy as np


@dataclass
class BlockStructure:
    q: int
    eta: float
    S_rowptr: list      # [q+1] int64 (2^l + 1,)  coupling block rows per level (level 0 always empty)
    S_col: list         # [q+1] int32 column node index (within level) per block, ascending per row
    D_rowptr: np.ndarray  # (2^q + 1,) int64
    D_col: np.ndarray     # int32 leaf column index per dense block, ascending per row

    @property
    def n_S(self):
        return int(sum(c.size for c in self.S_col))

    @property
    def n_D(self):
        return int(self.D_col.size)

    def csp(self):
        """Sparsity constant: max blocks in any block row at any level."""
        best = 0
        for rp in self.S_rowptr:
            if rp.size > 1:
                best = max(best, int(np.diff(rp).max(initial=0)))
        return best

    def csp_per_level(self):
        return [int(np.diff(rp).max(initial=0)) for rp in self.S_rowptr]


def _csr(rows, cols, nrows):
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=nrows), out=rowptr[1:])
    return rowptr, cols.astype(np.int32)


def admissible(ct, dt, cs, ds, eta):
    return eta * np.linalg.norm(ct - cs, axis=-1) >= 0.5 * (dt + ds)


def dual_traversal(tree, eta, all_dense=False):
    """all_dense=True marks every pair inadmissible (the degenerate all-dense case of
    SURVEY.md §8(c): A~ = K entrywise)."""
    q = tree.q
    S_rowptr = [np.zeros(2, dtype=np.int64)]
    S_col = [np.zeros(0, dtype=np.int32)]
    t = np.zeros(1, dtype=np.int64)
    s = np.zeros(1, dtype=np.int64)
    for l in range(q):
        # the 4 child pairs of every inadmissible pair at level l
        ct = (2 * t[:, None] + np.array([0, 0, 1, 1])[None, :]).reshape(-1)
        cs = (2 * s[:, None] + np.array([0, 1, 0, 1])[None, :]).reshape(-1)
        if all_dense:
            adm = np.zeros(ct.size, dtype=bool)
        else:
            C = tree.center(l + 1)
            D = tree.diameter(l + 1)
            adm = admissible(C[ct], D[ct], C[cs], D[cs], eta)
        rp, col = _csr(ct[adm], cs[adm], 1 << (l + 1))
        S_rowptr.append(rp)
        S_col.append(col)
        t, s = ct[~adm], cs[~adm]
    D_rowptr, D_col = _csr(t, s, 1 << q)
    return BlockStructure(q, eta, S_rowptr, S_col, D_rowptr, D_col)
