"""Writer of the `.h2m` flat file ("header {N, m, depth, level ranks}, then
level-ordered arrays"; SURVEY.md §8(b) "Flat file .h2m").  Generator side: it serialises an
H2Data; the CUDA library (h2_create_from_file) and the oracle (oracle/h2m.py) each read it with
their own reader.

Layout (little-endian; every section starts at a multiple of 64 bytes):

  header, 512 bytes
    0   char[8]  magic "H2MFLAT1"
    8   u32      version (1), dtype (0 = f64, 1 = f32), dim, m, q, flags, kernel_id, reserved
                 flags bit 0: V_leaf aliases U_leaf (no V section); bit 1: F aliases E (no F sections)
                 kernel_id: 0 exp, 1 gaussian, 2 poly, 3 fd, 255 other / random data
    40  u64      N, n_D, seed
    64  f64      eta, kernel parameters[4] (exp / gaussian: ell; poly: p; fd: beta)
    128 i32[32]  level_rank k^l, l = 0..q
    256 i64[32]  n_S^l coupling blocks per level, l = 0..q
  sections, in order
    points    f64 [N][dim]          tree order
    perm      i64 [N]               tree position -> original point id
    leaf_ptr  i64 [2^q + 1]
    U_leaf    T   [2^q][k^q][m]     (m x k^q column-major per leaf)
    V_leaf    T   [2^q][k^q][m]     (absent when flags bit 0)
    E^l       T   [2^l][k^{l-1}][k^l]   l = 1..q (k^l x k^{l-1} column-major)
    F^l       T   same              (absent when flags bit 1)
    for l = 0..q:  S_rowptr^l i64 [2^l + 1], S_col^l i32 [n_S^l], S^l T [n_S^l][k^l][k^l]
    D_rowptr  i64 [2^q + 1];  D_col i32 [n_D];  D T [n_D][m][m]
"""
import numpy as np

MAGIC = b"H2MFLAT1"
HEADER = 512
KERNEL_IDS = {"exp": 0, "gaussian": 1, "poly": 2, "fd": 3}


def _pad(f):
    pos = f.tell()
    if pos % 64:
        f.write(b"\0" * (64 - pos % 64))


def write_h2m(path, h, seed=0):
    """Write H2Data `h` (FP64 or FP32 floating arrays) to `path`."""
    dt = np.dtype(h.U_leaf.dtype)
    if dt not in (np.float64, np.float32):
        raise ValueError("floating arrays must be float64 or float32")
    q = int(h.q)
    if q + 1 > 32:
        raise ValueError("depth > 31 not representable")
    sym_u = h.V_leaf is h.U_leaf
    sym_e = all(a is b for a, b in zip(h.E[1:], h.F[1:]))
    kern = getattr(h, "kernel", None)
    kid, kpar = 255, [0.0] * 4
    if kern is not None and kern.name in KERNEL_IDS:
        kid = KERNEL_IDS[kern.name]
        kpar[0] = {"exp": kern.ell, "gaussian": kern.ell, "poly": float(kern.p), "fd": kern.beta}[kern.name]
    hdr = bytearray(HEADER)
    hdr[0:8] = MAGIC
    np.frombuffer(hdr, dtype="<u4", count=8, offset=8)[:] = [
        1, 0 if dt == np.float64 else 1, int(h.dim), int(h.m), q, (1 if sym_u else 0) | (2 if sym_e else 0), kid, 0]
    np.frombuffer(hdr, dtype="<u8", count=3, offset=40)[:] = [int(h.N), int(h.n_D), int(seed)]
    np.frombuffer(hdr, dtype="<f8", count=5, offset=64)[:] = [float(h.eta)] + kpar
    np.frombuffer(hdr, dtype="<i4", count=32, offset=128)[: q + 1] = h.ranks
    np.frombuffer(hdr, dtype="<i8", count=32, offset=256)[: q + 1] = [c.size for c in h.S_col]
    fl = "<f8" if dt == np.float64 else "<f4"
    with open(path, "wb") as f:
        f.write(bytes(hdr))

        def sec(a, dtype):
            _pad(f)
            f.write(np.ascontiguousarray(a, dtype=dtype).tobytes())
        sec(h.points, "<f8")
        sec(h.perm, "<i8")
        sec(h.leaf_ptr, "<i8")
        sec(h.U_leaf, fl)
        if not sym_u:
            sec(h.V_leaf, fl)
        for l in range(1, q + 1):
            sec(h.E[l], fl)
        if not sym_e:
            for l in range(1, q + 1):
                sec(h.F[l], fl)
        for l in range(q + 1):
            sec(h.S_rowptr[l], "<i8")
            sec(h.S_col[l], "<i4")
            sec(h.S[l], fl)
        sec(h.D_rowptr, "<i8")
        sec(h.D_col, "<i4")
        sec(h.D, fl)
        _pad(f)
