"""CPU oracle of the H² matvec — TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The product path (paper_2109_05451_b200) never imports it and the two
share no code; see h2_oracle.c's header for the algorithm and its citations.

The oracle takes h2gen.H2Data (FP64 arrays in the column-major storage convention) and
X / Y as (nv, N) C-contiguous arrays (== N x nv column-major, tree order).
"""
import ctypes as C
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "h2_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-fopenmp", "-shared", "-fPIC",
                               "-o", _LIB, _SRC])
    return _LIB


class _Input(C.Structure):
    _fields_ = [
        ("N", C.c_int64), ("m", C.c_int32), ("q", C.c_int32),
        ("ranks", C.POINTER(C.c_int32)), ("leaf_ptr", C.POINTER(C.c_int64)),
        ("U_leaf", C.c_void_p), ("V_leaf", C.c_void_p),
        ("E", C.POINTER(C.c_void_p)), ("F", C.POINTER(C.c_void_p)),
        ("S_rowptr", C.POINTER(C.c_void_p)), ("S_col", C.POINTER(C.c_void_p)),
        ("S", C.POINTER(C.c_void_p)),
        ("D_rowptr", C.POINTER(C.c_int64)), ("D_col", C.POINTER(C.c_int32)), ("D", C.c_void_p),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.h2o_matvec.restype = C.c_int
        _lib.h2o_matvec.argtypes = [C.POINTER(_Input), C.c_int, C.c_double, C.c_void_p,
                                    C.c_double, C.c_void_p, C.c_void_p]
        _lib.h2o_trees.restype = C.c_int
        _lib.h2o_trees.argtypes = [C.POINTER(_Input), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.h2o_set_threads.restype = C.c_int
        _lib.h2o_set_threads.argtypes = [C.c_int]
    return _lib


def set_threads(n=0):
    """OpenMP threads of later oracle calls (n < 1: all host cores the process may use).
    Returns the count in effect.  The result does not depend on it (fixed per-output order)."""
    import os
    if n is None or n < 1:
        n = len(os.sched_getaffinity(0))
    return _load().h2o_set_threads(int(n))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class _Pinned:
    """Keeps FP64 contiguous copies alive for the duration of a call."""

    def __init__(self, h):
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
        self.keep = []
        q = h.q
        self.ranks = i32(h.ranks)
        self.leaf_ptr = i64(h.leaf_ptr)
        self.U = f(h.U_leaf); self.V = f(h.V_leaf)
        self.E = [f(e) for e in h.E]; self.F = [f(x) for x in h.F]
        self.Srp = [i64(r) for r in h.S_rowptr]; self.Scol = [i32(c) for c in h.S_col]
        self.S = [f(s) for s in h.S]
        self.Drp = i64(h.D_rowptr); self.Dcol = i32(h.D_col); self.D = f(h.D)
        arr = lambda lst: (C.c_void_p * (q + 1))(*[a.ctypes.data if a is not None else None for a in lst])
        self.Ea, self.Fa = arr(self.E), arr(self.F)
        self.Srpa, self.Scola, self.Sa = arr(self.Srp), arr(self.Scol), arr(self.S)
        self.inp = _Input(h.N, h.m, q, self.ranks.ctypes.data_as(C.POINTER(C.c_int32)),
                          self.leaf_ptr.ctypes.data_as(C.POINTER(C.c_int64)), _ptr(self.U), _ptr(self.V),
                          self.Ea, self.Fa, self.Srpa, self.Scola, self.Sa,
                          self.Drp.ctypes.data_as(C.POINTER(C.c_int64)),
                          self.Dcol.ctypes.data_as(C.POINTER(C.c_int32)), _ptr(self.D))


def matvec(h2, X, alpha=1.0, beta=0.0, Y=None, leaf_mask=None, prepared=None):
    """Y := alpha A~ X + beta Y (FP64).  X, Y: (nv, N).  Returns the new Y (a fresh array).
    leaf_mask: optional bool (2^q,) -> only those leaves' rows are computed (others keep Y's
    input value, or 0 when Y is None)."""
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float64)
    nv, N = X.shape
    assert N == h2.N
    Yo = np.zeros((nv, N)) if Y is None else np.array(Y, dtype=np.float64, order="C", copy=True)
    p = prepared if prepared is not None else _Pinned(h2)
    mask = None if leaf_mask is None else np.ascontiguousarray(leaf_mask, dtype=np.uint8)
    rc = lib.h2o_matvec(C.byref(p.inp), nv, float(alpha), _ptr(X), float(beta), _ptr(Yo), _ptr(mask))
    if rc != 0:
        raise RuntimeError("oracle h2o_matvec failed")
    return Yo


def prepare(h2):
    """Pre-marshal the input once (for repeated timed calls)."""
    return _Pinned(h2)


def trees(h2, X):
    """Per-level x^ (after the upsweep) and y^ (after the coupling multiply): lists over levels
    of arrays (2^l, nv, k^l)."""
    lib = _load()
    X = np.ascontiguousarray(X, dtype=np.float64)
    nv, N = X.shape
    total = sum((1 << l) * h2.ranks[l] * nv for l in range(h2.q + 1))
    xh = np.zeros(total); yh = np.zeros(total)
    p = _Pinned(h2)
    if lib.h2o_trees(C.byref(p.inp), nv, _ptr(X), _ptr(xh), _ptr(yh)) != 0:
        raise RuntimeError("oracle h2o_trees failed")
    outx, outy, off = [], [], 0
    for l in range(h2.q + 1):
        sz = (1 << l) * h2.ranks[l] * nv
        outx.append(xh[off:off + sz].reshape(1 << l, nv, h2.ranks[l]))
        outy.append(yh[off:off + sz].reshape(1 << l, nv, h2.ranks[l]))
        off += sz
    return outx, outy
