"""Fractional-diffusion solve on the GPU: argument
marshalling for h2_fd_diag / h2_pcg (include/h2.h); every arithmetic step runs in the library.

    A u = h^2 (D + K + C) u = b,  D = diag(K^ 1) on the interior, Jacobi-PCG."""
import ctypes as C

import numpy as np

from ._binding import load_library, _check


def solve_fd(opK, opKhat, idx, C_rowptr, C_col, C_val, C_diag, h, b, rtol=1e-8, maxit=500):
    """opK / opKhat: H2Operator handles (FP64, one rank) of K (interior) and K^ (extended grid);
    idx: K tree position -> K^ tree position; C (CSR, K's tree order, diagonal included, C_diag its
    diagonal); b in tree order.  Returns (u, iterations, relative residual history, D)."""
    import torch
    lib = load_library()
    lib.h2_fd_diag.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
    lib.h2_fd_diag.restype = C.c_int
    lib.h2_pcg.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_double)]
    lib.h2_pcg.restype = C.c_int
    dev = torch.device("cuda", torch.cuda.current_device())
    n = int(opK.n_local)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
    d_idx, d_cd = t(idx, np.int64), t(C_diag, np.float64)
    diag = torch.empty(n, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    _check(lib.h2_fd_diag(opKhat.handle, d_idx.data_ptr(), d_cd.data_ptr(), n, diag.data_ptr()))
    D = (diag - d_cd).cpu().numpy()
    rp, col, val, bb = t(C_rowptr, np.int64), t(C_col, np.int32), t(C_val, np.float64), t(b, np.float64)
    u = torch.zeros(n, dtype=torch.float64, device=dev)
    hist = (C.c_double * (maxit + 1))()
    it = C.c_int()
    _check(lib.h2_pcg(opK.handle, float(h * h), diag.data_ptr(), rp.data_ptr(), col.data_ptr(), val.data_ptr(),
                      bb.data_ptr(), u.data_ptr(), float(rtol), int(maxit), C.byref(it), hist))
    return u.cpu().numpy(), it.value, list(hist)[: it.value + 1], D
