"""Cluster tree T_I ("hierarchical clusterings of these index sets";
k-d tree PAPER.md:769).  Readings R6/R7 of DESIGN.md: median split on the longest
bounding-box extent, ties -> lowest axis; stable order; balanced sizes
(ceil(n/2), floor(n/2)); depth q = ceil(log2(N/m)); all leaves on level q."""
from dataclasses import dataclass
import math
import numpy as np


@dataclass
class ClusterTree:
    dim: int
    N: int
    m: int
    q: int
    points: np.ndarray      # (N, dim) in TREE order
    perm: np.ndarray        # (N,) tree position -> original point index
    starts: list            # starts[l]: (2^l + 1,) int64 row offsets of level-l nodes
    lo: list                # lo[l]: (2^l, dim) bounding-box lower corners
    hi: list                # hi[l]: (2^l, dim) bounding-box upper corners

    @property
    def leaf_ptr(self):
        return self.starts[self.q]

    def center(self, l):
        return 0.5 * (self.lo[l] + self.hi[l])

    def diameter(self, l):
        return np.linalg.norm(self.hi[l] - self.lo[l], axis=1)


def tree_depth(N, m):
    if N <= m:
        return 0
    return int(math.ceil(math.log2(N / m) - 1e-12))


def build_cluster_tree(points, m):
    points = np.ascontiguousarray(points, dtype=np.float64)
    if points.ndim != 2 or points.shape[0] < 1:
        raise ValueError("structural error: empty point cloud")
    N, dim = points.shape
    if m < 1:
        raise ValueError("leaf size must be >= 1")
    q = tree_depth(N, m)
    if N < (1 << q):
        raise ValueError("structural error: fewer points than leaves")
    perm = np.arange(N, dtype=np.int64)
    starts = [np.array([0, N], dtype=np.int64)]
    for l in range(q):
        st = starts[l]
        sizes = np.diff(st)
        nn = sizes.size
        node_of = np.repeat(np.arange(nn), sizes)
        pts = points[perm]
        lo = np.minimum.reduceat(pts, st[:-1], axis=0)
        hi = np.maximum.reduceat(pts, st[:-1], axis=0)
        axis = np.argmax(hi - lo, axis=1)            # first max -> lowest axis on ties
        key = pts[np.arange(N), axis[node_of]]
        order = np.lexsort((key, node_of))           # stable: node-major, then key
        perm = perm[order]
        half = (sizes + 1) // 2                      # ceil(n/2) to the first child
        nst = np.empty(2 * nn + 1, dtype=np.int64)
        nst[0:-1:2] = st[:-1]
        nst[1::2] = st[:-1] + half
        nst[-1] = N
        starts.append(nst)
    pts = points[perm]
    los, his = [], []
    for l in range(q + 1):
        st = starts[l]
        los.append(np.minimum.reduceat(pts, st[:-1], axis=0))
        his.append(np.maximum.reduceat(pts, st[:-1], axis=0))
    return ClusterTree(dim, N, m, q, pts, perm, starts, los, his)


def grid_points(dims):
    """Integer lattice `dims` in meshgrid(indexing='ij') order, scaled so the longest side is 1
    (SURVEY.md App. B.1)."""
    axes = [np.arange(d, dtype=np.float64) for d in dims]
    g = np.meshgrid(*axes, indexing="ij")
    pts = np.stack([a.reshape(-1) for a in g], axis=1)
    return pts / (max(dims) - 1)


def uniform_points(n, dim, seed):
    return np.random.default_rng(seed).random((n, dim))


def fd_grid_points(n):
    """n x n interior vertex grid of Omega = [-1, 1]^2: x_i = -1 + (i+1) h, h = 2 / (n+1)
    ("N points with spacing h in Omega"; reading R10), meshgrid(ij) order."""
    h = 2.0 / (n + 1)
    ax = -1.0 + h * np.arange(1, n + 1, dtype=np.float64)
    g = np.meshgrid(ax, ax, indexing="ij")
    return np.stack([a.reshape(-1) for a in g], axis=1)
