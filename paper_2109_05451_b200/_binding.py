"""ctypes binding of include/h2.h (argument marshalling only: every step of the matvec runs in
the CUDA kernels of libh2b200.so).  Loading fails loudly when the library is missing; there is
no CPU fallback."""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libh2b200.so")

H2_OK, H2_ERR_ARG, H2_ERR_SHAPE, H2_ERR_STRUCT, H2_ERR_CUDA, H2_ERR_NCCL, H2_ERR_OOM, H2_ERR_STATE = \
    0, -1, -2, -3, -4, -5, -6, -7
H2_F64, H2_F32 = 0, 1
H2_MEM_HOST, H2_MEM_DEVICE = 0, 1
H2_SYMMETRIC = 1

EXPORTS = ["h2_create", "h2_matvec", "h2_matvec_ld", "h2_matvec_host", "h2_set_stream", "h2_stats",
           "h2_group_create", "h2_group_matvec", "h2_file_info", "h2_create_from_file", "h2_group_create_from_file", "h2_n_local", "h2_fd_diag", "h2_pcg",
           "h2_set_profiling", "h2_phase_times", "h2_phase_stats",
           "h2_plan_counts", "h2_plan_census", "h2_destroy", "h2_nccl_unique_id", "h2_last_error", "h2_version",
           "h2_orthogonalize", "h2_export", "h2_reweigh"]
H2_EXPORT_S, H2_EXPORT_U, H2_EXPORT_VT, H2_EXPORT_E, H2_EXPORT_FT, H2_EXPORT_XHAT, H2_EXPORT_YHAT = 0, 1, 2, 3, 4, 5, 6
PHASES = ["up_leaf", "up_transfer", "exchange_top", "coupling_diag", "coupling_offdiag",
          "down_transfer", "leaf_u", "dense", "coupling_leaf"]
KERNEL_OF_PHASE = {"up_leaf": "k_up_leaf", "up_transfer": "k_sweep<WRITE>", "exchange_top": "k_pack + k_tree",
                   "coupling_diag": "k_rows<WRITE>", "coupling_offdiag": "k_rows<ACCUM>",
                   "down_transfer": "k_sweep<ACCUM>",
                   "leaf_u": "k_leaf_dense (last transfer + leaf expansion + dense near field + epilogue)",
                   "dense": "k_leaf_dense", "coupling_leaf": "k_rows<WRITE>"}


class H2Error(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"h2 error {code}: {msg}")
        self.code = code


class h2_desc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("mem", C.c_int32), ("depth", C.c_int32), ("leaf_size", C.c_int32),
        ("rank", C.c_int32), ("nranks", C.c_int32), ("n_local", C.c_int64),
        ("level_rank", C.c_void_p), ("leaf_ptr", C.c_void_p),
        ("U_leaf", C.c_void_p), ("V_leaf", C.c_void_p),
        ("E", C.c_void_p), ("F", C.c_void_p),
        ("S_rowptr", C.c_void_p), ("S_col", C.c_void_p), ("S", C.c_void_p),
        ("D_rowptr", C.c_void_p), ("D_col", C.c_void_p), ("D", C.c_void_p),
        ("flags", C.c_int32),
    ]


_lib = None


def load_library(path=None):
    """Load libh2b200.so (raises if absent: build with python -m paper_2109_05451_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} not built (run python -m paper_2109_05451_b200.build); "
                          "there is no CPU fallback")
    lib = C.CDLL(path)
    vp, i32, i64, d = C.c_void_p, C.c_int, C.c_int64, C.c_double
    sig = {
        "h2_create": ([C.POINTER(h2_desc), i32, vp, C.POINTER(vp)], i32),
        "h2_matvec": ([vp, d, vp, d, vp, i32], i32),
        "h2_matvec_ld": ([vp, d, vp, i64, d, vp, i64, i32], i32),
        "h2_matvec_host": ([vp, d, vp, d, vp, i32], i32),
        "h2_set_stream": ([vp, vp], i32),
        "h2_stats": ([vp, i32, C.POINTER(d), C.POINTER(d), C.POINTER(d), C.POINTER(i32)], i32),
        "h2_plan_counts": ([vp, C.POINTER(C.c_int64)], i32),
        "h2_plan_census": ([C.POINTER(h2_desc), i32, vp, vp, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], i32),
        "h2_set_profiling": ([vp, i32], i32),
        "h2_phase_times": ([vp, C.POINTER(d), C.POINTER(C.c_int64)], i32),
        "h2_phase_stats": ([vp, i32, C.POINTER(d), C.POINTER(d)], i32),
        "h2_destroy": ([vp], i32),
        "h2_orthogonalize": ([vp], i32),
        "h2_export": ([vp, i32, i32, vp, i64], i32),
        "h2_reweigh": ([vp, vp, i64], i32),
        "h2_group_create_from_file": ([C.c_char_p, i32, i32, C.POINTER(vp)], i32),
        "h2_n_local": ([vp, C.POINTER(C.c_int64)], i32),
        "h2_file_info": ([C.c_char_p, C.POINTER(C.c_int64)], i32),
        "h2_create_from_file": ([C.c_char_p, i32, i32, i32, vp, C.POINTER(vp)], i32),
        "h2_group_create": ([C.POINTER(C.POINTER(h2_desc)), i32, i32, C.POINTER(vp)], i32),
        "h2_group_matvec": ([C.POINTER(vp), i32, d, C.POINTER(vp), d, C.POINTER(vp), i32], i32),
        "h2_nccl_unique_id": ([vp], i32),
        "h2_last_error": ([], C.c_char_p),
        "h2_version": ([], C.c_char_p),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes, f.restype = args, res
    _lib = lib
    return lib


def _check(rc):
    if rc != H2_OK:
        raise H2Error(rc, _lib.h2_last_error().decode())


def nccl_unique_id():
    lib = load_library()
    buf = (C.c_uint8 * 128)()
    _check(lib.h2_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return bytes(buf)


def _is_torch(a):
    return type(a).__module__.startswith("torch")


class _Desc:
    """Marshals one rank's arrays into an h2_desc (keeps the buffers alive)."""

    def __init__(self, *, depth, leaf_size, level_rank, leaf_ptr, U_leaf, V_leaf, E, F, S_rowptr,
                 S_col, S, D_rowptr, D_col, D, n_local, rank=0, nranks=1, dtype="f64", symmetric=False):
        self.dtype = {"f64": H2_F64, "f32": H2_F32}[dtype]
        self.np_dtype = np.float64 if self.dtype == H2_F64 else np.float32
        fl = [U_leaf, V_leaf, D] + [a for a in list(E) + list(F) + list(S) if a is not None]
        self.device = device = any(_is_torch(a) and a.is_cuda for a in fl)
        self.keep = []

        def size(a):
            return 0 if a is None else (a.numel() if _is_torch(a) else a.size)

        def fptr(a):
            if a is None or size(a) == 0:
                return None
            if device:
                if not (_is_torch(a) and a.is_cuda and a.is_contiguous()):
                    raise ValueError("device mode needs contiguous CUDA tensors for every float array")
                want = "torch.float64" if self.dtype == H2_F64 else "torch.float32"
                if str(a.dtype) != want:
                    raise ValueError(f"float arrays must be {want}")
                self.keep.append(a)
                return a.data_ptr()
            a = np.ascontiguousarray(a, dtype=self.np_dtype)
            self.keep.append(a)
            return a.ctypes.data

        def iptr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self.keep.append(a)
            return a.ctypes.data

        q = int(depth)
        arr = lambda vals: (C.c_void_p * (q + 1))(*vals)
        self.E = arr([fptr(e) for e in E])
        self.F = arr([fptr(f) for f in F])
        self.Srp = arr([iptr(r, np.int64) for r in S_rowptr])
        self.Scol = arr([iptr(c, np.int32) for c in S_col])
        self.S = arr([fptr(s) for s in S])
        d = h2_desc()
        d.dtype, d.mem, d.depth, d.leaf_size = self.dtype, H2_MEM_DEVICE if device else H2_MEM_HOST, q, int(leaf_size)
        d.rank, d.nranks, d.n_local = int(rank), int(nranks), int(n_local)
        d.level_rank = iptr(level_rank, np.int32)
        d.leaf_ptr = iptr(leaf_ptr, np.int64)
        d.U_leaf, d.V_leaf = fptr(U_leaf), fptr(V_leaf)
        d.E, d.F = C.cast(self.E, C.c_void_p), C.cast(self.F, C.c_void_p)
        d.S_rowptr, d.S_col, d.S = (C.cast(self.Srp, C.c_void_p), C.cast(self.Scol, C.c_void_p),
                                    C.cast(self.S, C.c_void_p))
        d.D_rowptr, d.D_col = iptr(D_rowptr, np.int64), iptr(D_col, np.int32)
        d.D = fptr(D)
        d.flags = H2_SYMMETRIC if symmetric else 0
        self.desc = d


def file_info(path):
    """Header facts of an .h2m file (no GPU): N, dim, m, q, dtype, n_S (all levels), n_D, k^q."""
    lib = load_library()
    info = (C.c_int64 * 8)()
    _check(lib.h2_file_info(os.fsencode(path), info))
    return dict(zip(["N", "dim", "m", "q", "dtype", "n_S", "n_D", "k"], list(info)))


def plan_census(level, **kw):
    """Host-only compressed off-diagonal node lists (pid, nodes_ptr, nodes) of one rank's view
    (PAPER.md:454-468); level -1 = dense halo leaves.  No GPU needed."""
    lib = load_library()
    kw = dict(kw)
    for key in ("dtype", "nv_max", "nccl_id"):
        kw.pop(key, None)
    ds = _Desc(**kw)
    npid, nn = C.c_int64(), C.c_int64()
    _check(lib.h2_plan_census(C.byref(ds.desc), int(level), None, None, None, C.byref(npid), C.byref(nn)))
    pid = np.zeros(npid.value, dtype=np.int64)
    ptr = np.zeros(npid.value + 1, dtype=np.int64)
    nodes = np.zeros(nn.value, dtype=np.int64)
    _check(lib.h2_plan_census(C.byref(ds.desc), int(level), pid.ctypes.data, ptr.ctypes.data,
                              nodes.ctypes.data, C.byref(npid), C.byref(nn)))
    return pid, ptr, nodes


class H2Operator:
    """One rank's H² operator on the GPU (h2_create / h2_matvec / h2_destroy).

    Floating arrays: numpy arrays (HOST: copied) or CUDA torch tensors (DEVICE: adopted and
    kept alive by this object); all of one kind.  Integer arrays: numpy.  Shapes follow
    include/h2.h (column-major small matrices)."""

    def __init__(self, *, dtype="f64", nv_max=16, nccl_id=None, **kw):
        lib = load_library()
        self._lib = lib
        ds = _Desc(dtype=dtype, **kw)
        self.dtype, self.np_dtype = ds.dtype, ds.np_dtype
        self.n_local, self.nv_max = int(kw["n_local"]), int(nv_max)
        self.rank, self.nranks = int(kw.get("rank", 0)), int(kw.get("nranks", 1))
        idbuf = None
        if self.nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nccl_id (128 bytes) required when nranks > 1")
            idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        _check(lib.h2_create(C.byref(ds.desc), int(nv_max), C.cast(idbuf, C.c_void_p) if idbuf else None,
                             C.byref(h)))
        self.handle = h
        self._keep = ds.keep if ds.device else []   # host arrays were copied by h2_create
        self.device_index = None
        try:
            import torch
            if torch.cuda.is_available():
                self.device_index = torch.cuda.current_device()
        except Exception:
            pass

    @classmethod
    def from_file(cls, path, *, nv_max=16, rank=0, nranks=1, nccl_id=None):
        """h2_create_from_file: this rank's view of an .h2m file (host reads, copied to the GPU)."""
        lib = load_library()
        self = cls.__new__(cls)
        self._lib = lib
        info = file_info(path)
        self.dtype = H2_F64 if info["dtype"] == 0 else H2_F32
        self.np_dtype = np.float64 if self.dtype == H2_F64 else np.float32
        self.rank, self.nranks, self.nv_max = int(rank), int(nranks), int(nv_max)
        idbuf = None
        if self.nranks > 1:
            if nccl_id is None or len(nccl_id) != 128:
                raise ValueError("nccl_id (128 bytes) required when nranks > 1")
            idbuf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        h = C.c_void_p()
        _check(lib.h2_create_from_file(os.fsencode(path), self.rank, self.nranks, self.nv_max,
                                       C.cast(idbuf, C.c_void_p) if idbuf else None, C.byref(h)))
        self.handle = h
        self._keep = []
        nl = C.c_int64()
        _check(lib.h2_n_local(h, C.byref(nl)))
        self.n_local = int(nl.value)
        self.device_index = None
        try:
            import torch
            if torch.cuda.is_available():
                self.device_index = torch.cuda.current_device()
        except Exception:
            pass
        return self

    # -- calls
    def set_stream(self, stream_ptr):
        _check(self._lib.h2_set_stream(self.handle, C.c_void_p(int(stream_ptr))))

    def _check_vectors(self, X, Y, want_cuda):
        """Shape / dtype / device / layout checks before raw pointers cross the C ABI."""
        want = "torch.float64" if self.dtype == H2_F64 else "torch.float32"
        nv = X.shape[0] if len(X.shape) == 2 else -1
        if len(X.shape) != 2 or tuple(X.shape) != (nv, self.n_local) or tuple(Y.shape) != tuple(X.shape):
            raise ValueError(f"X, Y must both have shape (nv, n_local={self.n_local})")
        if not 1 <= nv <= self.nv_max:
            raise ValueError(f"nv must be in [1, nv_max={self.nv_max}]")
        for name, a in (("X", X), ("Y", Y)):
            if _is_torch(a):
                if str(a.dtype) != want:
                    raise ValueError(f"{name} must be {want} (handle dtype)")
                if not a.is_contiguous():
                    raise ValueError(f"{name} must be contiguous")
                if a.is_cuda != want_cuda:
                    raise ValueError(f"{name} must be a {'CUDA' if want_cuda else 'host'} tensor")
                if want_cuda and self.device_index is not None and a.device.index != self.device_index:
                    raise ValueError(f"{name} is on cuda:{a.device.index}, the handle on cuda:{self.device_index}")
            else:
                if want_cuda:
                    raise ValueError(f"{name} must be a CUDA tensor")
                if a.dtype != self.np_dtype or not a.flags["C_CONTIGUOUS"]:
                    raise ValueError(f"{name} must be a C-contiguous {np.dtype(self.np_dtype).name} array")
                if name == "Y" and not a.flags["WRITEABLE"]:
                    raise ValueError("Y must be writeable")
        return nv

    def matvec(self, X, Y, alpha=1.0, beta=0.0, stream=None):
        """Y := alpha A X + beta Y.  X, Y: CUDA tensors of shape (nv, n_local) (contiguous ==
        n_local x nv column-major).  Asynchronous on `stream` (default: torch's current stream)."""
        import torch
        nv = self._check_vectors(X, Y, True)
        st = stream if stream is not None else torch.cuda.current_stream(X.device)
        self.set_stream(st.cuda_stream)
        _check(self._lib.h2_matvec(self.handle, float(alpha), X.data_ptr(), float(beta), Y.data_ptr(), nv))
        return Y

    def matvec_ld(self, X, ldx, Y, ldy, nv, alpha=1.0, beta=0.0, stream=None):
        """h2_matvec_ld: X, Y are 1-D CUDA tensors holding nv columns of n_local rows with leading
        dimensions ldx, ldy (>= n_local): column n of X starts at element n * ldx."""
        import torch
        want = torch.float64 if self.dtype == H2_F64 else torch.float32
        for name, a, ld in (("X", X, ldx), ("Y", Y, ldy)):
            if not (_is_torch(a) and a.is_cuda and a.dtype == want and a.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous CUDA {want} tensor")
            if ld < self.n_local or a.numel() < (nv - 1) * ld + self.n_local:
                raise ValueError(f"{name} too small for nv={nv}, ld={ld}")
        st = stream if stream is not None else torch.cuda.current_stream(X.device)
        self.set_stream(st.cuda_stream)
        _check(self._lib.h2_matvec_ld(self.handle, float(alpha), X.data_ptr(), int(ldx), float(beta),
                                      Y.data_ptr(), int(ldy), int(nv)))
        return Y

    def matvec_host(self, X, Y, alpha=1.0, beta=0.0, stream=None):
        """End-to-end: X, Y host arrays (nv, n_local) (numpy or pinned CPU torch tensors)."""
        ptr = lambda a: a.data_ptr() if _is_torch(a) else a.ctypes.data
        nv = self._check_vectors(X, Y, False)
        if stream is not None:
            self.set_stream(stream.cuda_stream)
        _check(self._lib.h2_matvec_host(self.handle, float(alpha), ptr(X), float(beta), ptr(Y), nv))
        return Y

    def stats(self, nv):
        f, b, x, n = C.c_double(), C.c_double(), C.c_double(), C.c_int()
        _check(self._lib.h2_stats(self.handle, int(nv), C.byref(f), C.byref(b), C.byref(x), C.byref(n)))
        return {"flops": f.value, "bytes": b.value, "xchg_bytes": x.value, "launches": n.value}

    def set_profiling(self, on=True):
        _check(self._lib.h2_set_profiling(self.handle, 1 if on else 0))

    def phase_times(self):
        """Mean ms per phase per call since the last read (dict incl. 'total'), and the call count."""
        ms, n = (C.c_double * 10)(), C.c_int64()
        _check(self._lib.h2_phase_times(self.handle, ms, C.byref(n)))
        out = dict(zip(PHASES + ["total"], list(ms)))
        return out, n.value

    def phase_stats(self, nv):
        b, f = (C.c_double * 10)(), (C.c_double * 10)()
        _check(self._lib.h2_phase_stats(self.handle, int(nv), b, f))
        return dict(zip(PHASES + ["total"], list(b))), dict(zip(PHASES + ["total"], list(f)))

    def plan_counts(self):
        c = (C.c_int64 * 8)()
        _check(self._lib.h2_plan_counts(self.handle, c))
        keys = ["diag_S", "offdiag_S", "root_S", "diag_D", "offdiag_D", "peers", "recv_nodes", "recv_leaves"]
        return dict(zip(keys, list(c)))

    def orthogonalize(self):
        """Basis orthogonalization in place (h2_orthogonalize; FP64, one GPU, full storage)."""
        _check(self._lib.h2_orthogonalize(self.handle))

    def reweigh(self, R_out):
        """Reweighing downsweep (h2_reweigh) into the device tensor R_out (sum_l 2^l k_l^2 doubles)."""
        import torch
        if not (isinstance(R_out, torch.Tensor) and R_out.is_cuda and R_out.dtype == torch.float64
                and R_out.is_contiguous()):
            raise ValueError("R_out must be a contiguous CUDA float64 tensor")
        _check(self._lib.h2_reweigh(self.handle, C.c_void_p(R_out.data_ptr()), int(R_out.numel())))

    def export(self, what, level, count):
        """Host copy (1-D, count elements) of one operator array (h2_export; H2_EXPORT_*)."""
        out = np.empty(int(count), dtype=self.np_dtype)
        _check(self._lib.h2_export(self.handle, int(what), int(level), out.ctypes.data, int(count)))
        return out

    def close(self):
        if getattr(self, "handle", None):
            _check(self._lib.h2_destroy(self.handle))
            self.handle = None
            self._keep = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class H2Group:
    """P ranks emulated in ONE process on the current GPU (h2_group_create; test entry point):
    the multi-rank path with the per-call exchange done by device copies instead of NCCL.
    views: list of P per-rank keyword dicts (operator.shard_arrays output, rank o at index o)."""

    def __init__(self, views, *, dtype="f64", nv_max=16, path=None, P=None):
        lib = load_library()
        self._lib = lib
        if path is not None:                  # h2_group_create_from_file: every view read from an .h2m file
            self.P = int(P)
            hs = (C.c_void_p * self.P)()
            _check(lib.h2_group_create_from_file(os.fsencode(path), self.P, int(nv_max), hs))
            self.handles, self.nv_max = hs, int(nv_max)
            self.dtype = H2_F64 if file_info(path)["dtype"] == 0 else H2_F32
            self.n_local = []
            for o in range(self.P):
                nl = C.c_int64()
                _check(lib.h2_n_local(hs[o], C.byref(nl)))
                self.n_local.append(int(nl.value))
            return
        self.P = len(views)
        self._descs = [_Desc(dtype=dtype, **v) for v in views]
        self.n_local = [int(v["n_local"]) for v in views]
        self.dtype = self._descs[0].dtype
        arr = (C.POINTER(h2_desc) * self.P)(*[C.pointer(ds.desc) for ds in self._descs])
        hs = (C.c_void_p * self.P)()
        _check(lib.h2_group_create(arr, self.P, int(nv_max), hs))
        self.handles = hs
        self.nv_max = int(nv_max)

    def matvec(self, Xs, Ys, alpha=1.0, beta=0.0, stream=None):
        """Ys[o] := alpha A Xs[o] + beta Ys[o]: CUDA tensors (nv, n_local[o]) of the handle dtype."""
        import torch
        want = torch.float64 if self.dtype == H2_F64 else torch.float32
        nv = Xs[0].shape[0]
        for o in range(self.P):
            for a in (Xs[o], Ys[o]):
                if not (a.is_cuda and a.dtype == want and a.is_contiguous() and tuple(a.shape) == (nv, self.n_local[o])):
                    raise ValueError(f"rank {o}: X, Y must be contiguous CUDA {want} of shape (nv, {self.n_local[o]})")
        st = stream if stream is not None else torch.cuda.current_stream(Xs[0].device)
        _check(self._lib.h2_set_stream(self.handles[0], C.c_void_p(st.cuda_stream)))
        xp = (C.c_void_p * self.P)(*[x.data_ptr() for x in Xs])
        yp = (C.c_void_p * self.P)(*[y.data_ptr() for y in Ys])
        _check(self._lib.h2_group_matvec(self.handles, self.P, float(alpha), xp, float(beta), yp, nv))
        return Ys

    def plan_counts(self, o):
        c = (C.c_int64 * 8)()
        _check(self._lib.h2_plan_counts(self.handles[o], c))
        keys = ["diag_S", "offdiag_S", "root_S", "diag_D", "offdiag_D", "peers", "recv_nodes", "recv_leaves"]
        return dict(zip(keys, list(c)))

    def close(self):
        if getattr(self, "handles", None) is not None:
            for o in range(self.P):
                if self.handles[o]:
                    _check(self._lib.h2_destroy(self.handles[o]))
                    self.handles[o] = None
            self.handles = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
