"""Helpers for the GPU parity tests (test infrastructure)."""
import numpy as np

import oracle
from h2gen import build_cluster_tree, dual_traversal, random_h2_data, make_xy
from h2gen.tree import uniform_points, grid_points


def colmax_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return max(np.linalg.norm(a[i] - b[i]) / max(np.linalg.norm(b[i]), 1e-300) for i in range(a.shape[0]))


def random_case(N, m, ranks_fn, seed, eta=0.9, dim=2, grid=None):
    pts = grid_points(grid) if grid else uniform_points(N, dim, seed)
    tr = build_cluster_tree(pts, m)
    st = dual_traversal(tr, eta)
    ranks = [ranks_fn(l) for l in range(tr.q + 1)]
    return random_h2_data(tr, st, ranks, seed + 1000)


def gpu_matvec(op, X, alpha, beta, Y0, dtype="f64"):
    import torch
    tdt = torch.float64 if dtype == "f64" else torch.float32
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to("cuda", tdt)
    Yd = torch.from_numpy(np.ascontiguousarray(Y0)).to("cuda", tdt)
    op.matvec(Xd, Yd, alpha, beta)
    torch.cuda.synchronize()
    return Yd.double().cpu().numpy()


def with_root_coupling(h, seed=77):
    """The same H² data plus one coupling block at the root (level 0): a valid operator
    A + U_0 S_00 V_0^T (the matvec does not need the partition property) whose top tree holds a
    coupling at every P >= 2 -- at P = 2 the only level above the C-level is the root."""
    import dataclasses
    rng = np.random.default_rng(seed)
    k0 = h.ranks[0]
    Srp = [np.array([0, 1], dtype=np.int64)] + list(h.S_rowptr[1:])
    Scol = [np.array([0], dtype=np.int32)] + list(h.S_col[1:])
    S = [rng.uniform(-1.0, 1.0, size=(1, k0, k0)) / k0] + list(h.S[1:])
    return dataclasses.replace(h, S_rowptr=Srp, S_col=Scol, S=S)
