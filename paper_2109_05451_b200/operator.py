"""Block-row distribution of a global H² description into one rank's h2_desc view
(levels l >= C = log2 P split into branches, rank p owns branch p; levels
l < C replicated, reading R16), and construction of the rank's H2Operator.

Host-side marshalling only (slicing index ranges of the global arrays); no matvec arithmetic."""
import numpy as np

from ._binding import H2Operator, H2Group


def c_level(P):
    C = 0
    while (1 << C) < P:
        C += 1
    if (1 << C) != P:
        raise ValueError("P must be a power of two")
    return C


def held_range(l, rank, P):
    """[a, b) global node indices of level l held by `rank` (all nodes above the C-level)."""
    C = c_level(P)
    if l < C:
        return 0, 1 << l
    w = 1 << (l - C)
    return rank * w, (rank + 1) * w


def shard_arrays(h, rank=0, P=1):
    """Per-rank arrays for h2_create from a global description `h` (attributes as in
    h2gen.H2Data: q, m, ranks, leaf_ptr, U_leaf, V_leaf, E, F, S_rowptr, S_col, S, D_rowptr,
    D_col, D).  Returns (kwargs, row_range)."""
    q = h.q
    C = c_level(P)
    if C > q:
        raise ValueError("P too large for depth")
    la, lb = held_range(q, rank, P)
    lp = np.asarray(h.leaf_ptr, dtype=np.int64)
    r0, r1 = int(lp[la]), int(lp[lb])
    E, F, Srp, Scol, S = [None], [None], [], [], []
    for l in range(q + 1):
        a, b = held_range(l, rank, P)
        if l >= 1:
            E.append(h.E[l][a:b])
            F.append(h.F[l][a:b])
        rp = np.asarray(h.S_rowptr[l], dtype=np.int64)
        b0, b1 = int(rp[a]), int(rp[b])
        Srp.append(rp[a:b + 1] - b0)
        Scol.append(np.asarray(h.S_col[l])[b0:b1])
        S.append(h.S[l][b0:b1])
    drp = np.asarray(h.D_rowptr, dtype=np.int64)
    d0, d1 = int(drp[la]), int(drp[lb])
    kw = dict(depth=q, leaf_size=h.m, level_rank=np.asarray(h.ranks, dtype=np.int32),
              leaf_ptr=lp[la:lb + 1] - r0, U_leaf=h.U_leaf[la:lb], V_leaf=h.V_leaf[la:lb],
              E=E, F=F, S_rowptr=Srp, S_col=Scol, S=S, D_rowptr=drp[la:lb + 1] - d0,
              D_col=np.asarray(h.D_col)[d0:d1], D=h.D[d0:d1], n_local=r1 - r0, rank=rank, nranks=P)
    return kw, (r0, r1)


def broadcast_nccl_id(device):
    """A fresh NCCL unique id (each h2_create needs its own) generated on rank 0 and broadcast
    with torch.distributed (plumbing only)."""
    import torch
    import torch.distributed as dist
    from ._binding import nccl_unique_id
    t = torch.zeros(128, dtype=torch.uint8, device=device)
    if dist.get_rank() == 0:
        t.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(t, 0)
    return bytes(t.cpu().numpy().tolist())


def operator_from_h2data(h, rank=0, nranks=1, nccl_id=None, dtype="f64", nv_max=16, device=False,
                         torch_device=None, symmetric=False):
    """H2Operator for `rank` of `nranks`.  device=True uploads the floating arrays as CUDA torch
    tensors that the handle adopts (H2_MEM_DEVICE); otherwise h2_create copies host arrays."""
    kw, rows = shard_arrays(h, rank, nranks)
    npdt = np.float64 if dtype == "f64" else np.float32
    cast = lambda a: None if a is None else np.ascontiguousarray(a, dtype=npdt)
    for key in ("U_leaf", "V_leaf", "D"):
        kw[key] = cast(kw[key])
    for key in ("E", "F", "S"):
        kw[key] = [cast(a) for a in kw[key]]
    if device:
        import torch
        dev = torch_device or torch.device("cuda", torch.cuda.current_device())
        up = lambda a: None if a is None else torch.from_numpy(a).to(dev)
        for key in ("U_leaf", "V_leaf", "D"):
            kw[key] = up(kw[key])
        for key in ("E", "F", "S"):
            kw[key] = [up(a) for a in kw[key]]
    if symmetric:
        kw["V_leaf"] = kw["U_leaf"]        # the same array (H2_SYMMETRIC asserts U = V)
        kw["F"] = kw["E"]
    op = H2Operator(dtype=dtype, nv_max=nv_max, nccl_id=nccl_id, symmetric=symmetric, **kw)
    op.row_range = rows
    return op


def group_from_h2data(h, P, dtype="f64", nv_max=16):
    """Loopback group of P emulated ranks on the current GPU (tests): returns (H2Group, row
    ranges).  Host arrays, copied by h2_group_create."""
    npdt = np.float64 if dtype == "f64" else np.float32
    cast = lambda a: None if a is None else np.ascontiguousarray(a, dtype=npdt)
    views, rows = [], []
    for o in range(P):
        kw, rr = shard_arrays(h, o, P)
        for key in ("U_leaf", "V_leaf", "D"):
            kw[key] = cast(kw[key])
        for key in ("E", "F", "S"):
            kw[key] = [cast(a) for a in kw[key]]
        views.append(kw)
        rows.append(rr)
    return H2Group(views, dtype=dtype, nv_max=nv_max), rows
