"""The oracle's own reader of the `.h2m` flat file (TEST INFRASTRUCTURE, like the rest of oracle/).

Layout: SPEC.md:156 ("header {N, m, depth, level ranks}, then level-ordered arrays") as fixed in
h2gen/h2m.py's docstring: a 512-byte little-endian header, then 64-byte-aligned sections.  This
reader shares no code with the generator's writer or the CUDA library's reader; it returns an
object with the attributes oracle.matvec reads (N, m, q, ranks, leaf_ptr, U_leaf, V_leaf, E, F,
S_rowptr, S_col, S, D_rowptr, D_col, D) plus dim, perm, points, eta, seed."""
from types import SimpleNamespace

import numpy as np


def read_h2m(path):
    raw = np.fromfile(path, dtype=np.uint8)
    if raw[:8].tobytes() != b"H2MFLAT1":
        raise ValueError("not an .h2m file (magic)")
    u32 = raw[8:40].view("<u4")
    version, dtype, dim, m, q, flags, kernel_id = (int(v) for v in u32[:7])
    if version != 1:
        raise ValueError(f"unsupported .h2m version {version}")
    N, n_D, seed = (int(v) for v in raw[40:64].view("<u8"))
    f64 = raw[64:104].view("<f8")
    ranks = [int(v) for v in raw[128:256].view("<i4")[: q + 1]]
    n_S = [int(v) for v in raw[256:512].view("<i8")[: q + 1]]
    fl = np.dtype("<f8") if dtype == 0 else np.dtype("<f4")
    pos = [512]

    def take(n, dt, shape):
        dt = np.dtype(dt)
        off = (pos[0] + 63) // 64 * 64
        end = off + n * dt.itemsize
        if end > raw.size:
            raise ValueError(".h2m file truncated")
        pos[0] = end
        return raw[off:end].view(dt).reshape(shape).astype(dt.newbyteorder("="), copy=True)

    nleaf = 1 << q
    points = take(N * dim, "<f8", (N, dim))
    perm = take(N, "<i8", (N,))
    leaf_ptr = take(nleaf + 1, "<i8", (nleaf + 1,))
    U = take(nleaf * ranks[q] * m, fl, (nleaf, ranks[q], m))
    V = U if flags & 1 else take(nleaf * ranks[q] * m, fl, (nleaf, ranks[q], m))
    E = [None] + [take((1 << l) * ranks[l - 1] * ranks[l], fl, (1 << l, ranks[l - 1], ranks[l]))
                  for l in range(1, q + 1)]
    F = E if flags & 2 else [None] + [take((1 << l) * ranks[l - 1] * ranks[l], fl, (1 << l, ranks[l - 1], ranks[l]))
                                      for l in range(1, q + 1)]
    Srp, Scol, S = [], [], []
    for l in range(q + 1):
        Srp.append(take((1 << l) + 1, "<i8", ((1 << l) + 1,)))
        Scol.append(take(n_S[l], "<i4", (n_S[l],)))
        S.append(take(n_S[l] * ranks[l] * ranks[l], fl, (n_S[l], ranks[l], ranks[l])))
    Drp = take(nleaf + 1, "<i8", (nleaf + 1,))
    Dcol = take(n_D, "<i4", (n_D,))
    D = take(n_D * m * m, fl, (n_D, m, m))
    return SimpleNamespace(N=N, m=m, q=q, dim=dim, ranks=ranks, perm=perm, points=points, leaf_ptr=leaf_ptr,
                           U_leaf=U, V_leaf=V, E=E, F=F, S_rowptr=Srp, S_col=Scol, S=S, D_rowptr=Drp, D_col=Dcol,
                           D=D, eta=float(f64[0]), seed=seed, kernel_id=kernel_id, kernel_par=list(f64[1:5]),
                           dtype="f64" if dtype == 0 else "f32")
