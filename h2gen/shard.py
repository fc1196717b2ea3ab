"""Shard-aware generation for multi-GPU weak scaling: build only the operator arrays one rank
holds (its branch of the block rows; top levels replicated) without ever
materialising the global arrays.  Output is the same per-rank view as
paper_2109_05451_b200.operator.shard_arrays(build_h2(...), rank, P) — the tests check that."""
import numpy as np

from .h2data import (_box_nodes, _tensor_points, _tensor_lagrange, _leaf_point_index)


def _held(l, rank, P):
    C = P.bit_length() - 1
    if l < C:
        return 0, 1 << l
    w = 1 << (l - C)
    return rank * w, (rank + 1) * w


def build_h2_shard(tree, st, kernel, p, rank, P, chunk=2048):
    """Per-rank h2_create keyword arrays (host numpy, FP64) + (r0, r1) global row range."""
    from concurrent.futures import ThreadPoolExecutor
    import os
    dim, q, m = tree.dim, tree.q, tree.m
    k = p ** dim
    nodes = [_box_nodes(tree.lo[l], tree.hi[l], p) for l in range(q + 1)]
    chebpts = [_tensor_points(nodes[l], p, dim) for l in range(q + 1)]
    pidx = _leaf_point_index(tree.leaf_ptr, m)
    la, lb = _held(q, rank, P)
    lp = np.asarray(tree.leaf_ptr, dtype=np.int64)
    r0, r1 = int(lp[la]), int(lp[lb])
    lpts = tree.points[np.maximum(pidx[la:lb], 0)]
    U = _tensor_lagrange(nodes[q][la:lb], lpts, p)
    U[pidx[la:lb] < 0] = 0.0
    U = np.ascontiguousarray(U.transpose(0, 2, 1))
    E = [None]
    for l in range(1, q + 1):
        a, b = _held(l, rank, P)
        par = np.arange(a, b) // 2
        vals = _tensor_lagrange(nodes[l - 1][par], chebpts[l][a:b], p)
        E.append(np.ascontiguousarray(vals.transpose(0, 2, 1)))
    pool = ThreadPoolExecutor(max(1, min(16, len(os.sched_getaffinity(0)))))
    Srp, Scol, S = [], [], []
    for l in range(q + 1):
        a, b = _held(l, rank, P)
        rp = st.S_rowptr[l]
        b0, b1 = int(rp[a]), int(rp[b])
        col = st.S_col[l][b0:b1]
        rows = np.repeat(np.arange(a, b), np.diff(rp[a:b + 1]))
        out = np.empty((col.size, k, k))

        def fill(c0, l=l, rows=rows, col=col, out=out):
            c1 = min(col.size, c0 + chunk)
            xt = chebpts[l][rows[c0:c1]]
            xs = chebpts[l][col[c0:c1]]
            out[c0:c1] = kernel(xs[:, :, None, :], xt[:, None, :, :])
        list(pool.map(fill, range(0, col.size, chunk)))
        Srp.append(rp[a:b + 1] - b0)
        Scol.append(col)
        S.append(out)
    drp = st.D_rowptr
    d0, d1 = int(drp[la]), int(drp[lb])
    dcol = st.D_col[d0:d1]
    rows = np.repeat(np.arange(la, lb), np.diff(drp[la:lb + 1]))
    D = np.empty((dcol.size, m, m))

    def filld(c0):
        c1 = min(dcol.size, c0 + chunk)
        it, js = pidx[rows[c0:c1]], pidx[dcol[c0:c1]]
        xi = tree.points[np.maximum(it, 0)]
        xj = tree.points[np.maximum(js, 0)]
        v = kernel(xj[:, :, None, :], xi[:, None, :, :])
        v *= (js >= 0)[:, :, None] & (it >= 0)[:, None, :]
        D[c0:c1] = v
    list(pool.map(filld, range(0, dcol.size, chunk)))
    pool.shutdown()
    kw = dict(depth=q, leaf_size=m, level_rank=np.full(q + 1, k, dtype=np.int32),
              leaf_ptr=lp[la:lb + 1] - r0, U_leaf=U, V_leaf=U, E=E, F=E, S_rowptr=Srp, S_col=Scol,
              S=S, D_rowptr=drp[la:lb + 1] - d0, D_col=dcol, D=D, n_local=r1 - r0, rank=rank,
              nranks=P)
    return kw, (r0, r1)
