"""B200-native eNMF hot path (arxiv 2605.19325) -- thin Python binding of libenmf.so.

Argument marshalling only: every step of the method runs in the sm_100a kernels behind the
C-ABI declared in include/enmf.h.  There is no CPU fallback: importing this package fails
loudly when the in-tree libenmf.so is missing.

torch is used for device memory and streams only.  Matrices are fp32, row-major, on the
handle's CUDA device: X (m x n, this rank's rows), U (rows x r), V (n x r).
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libenmf.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python __graft_entry__.py build`")
_lib = ctypes.CDLL(LIB_PATH)

ENMF_MAX_RANK = 128
PREC_AUTO, PREC_FP64, PREC_TC = 0, 1, 2
STATUS = {0: "ok", -1: "invalid argument", -2: "invalid shape", -3: "X has a negative entry",
          -4: "X has rank 0", -5: "non-finite value", -6: "CUDA error", -7: "NCCL error",
          -8: "out of device memory", -9: "call out of order"}


class EnmfError(RuntimeError):
    def __init__(self, code, where):
        super().__init__(f"{where}: {STATUS.get(code, code)} ({code})")
        self.code = code


class Problem(ctypes.Structure):
    _fields_ = [("m_global", ctypes.c_int64), ("n", ctypes.c_int64), ("r", ctypes.c_int64),
                ("row_begin", ctypes.c_int64), ("row_count", ctypes.c_int64),
                ("world_size", ctypes.c_int), ("rank", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p)]


class Options(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("oversample", ctypes.c_int),
                ("power_iters", ctypes.c_int), ("admm_iters", ctypes.c_int),
                ("admm_rho", ctypes.c_double), ("lift_steps", ctypes.c_int),
                ("pbcd_eps", ctypes.c_double), ("pbcd_max_iter", ctypes.c_int),
                ("precision", ctypes.c_int), ("step_rule", ctypes.c_int),
                ("descent", ctypes.c_int)]


class InitInfo(ctypes.Structure):
    _fields_ = [("sigma", ctypes.c_double * ENMF_MAX_RANK), ("rank_deficient", ctypes.c_int),
                ("negativity_svd", ctypes.c_double), ("negativity_rot", ctypes.c_double),
                ("orth_residual", ctypes.c_double), ("admm_third_branch", ctypes.c_int64),
                ("lambda_u", ctypes.c_double), ("lambda_v", ctypes.c_double),
                ("xnorm2", ctypes.c_double)]


class IterInfo(ctypes.Structure):
    _fields_ = [("ascent_sweeps", ctypes.c_int), ("hals_sweeps", ctypes.c_int),
                ("feasible", ctypes.c_int), ("pbcd_iters_u", ctypes.c_int),
                ("pbcd_iters_v", ctypes.c_int), ("hals_fallback_rows", ctypes.c_int)]


class Kkt(ctypes.Structure):
    _fields_ = [(k, ctypes.c_double) for k in ("min_u", "min_v", "comp_max", "comp_sum",
                                               "delta_w", "sigma_w", "dual_viol", "xnorm2",
                                               "rms_cross")]


_H = ctypes.c_void_p
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.POINTER(ctypes.c_double)
_sigs = {
    "enmf_default_options": (None, [ctypes.POINTER(Options)]),
    "enmf_create": (ctypes.c_int, [ctypes.POINTER(Problem), ctypes.POINTER(Options),
                                   ctypes.POINTER(_H)]),
    "enmf_destroy": (ctypes.c_int, [_H]),
    "enmf_set_data": (ctypes.c_int, [_H, _P, _I64]),
    "enmf_set_data_csr": (ctypes.c_int, [_H, _P, _P, _P, _I64]),
    "enmf_set_data_masked": (ctypes.c_int, [_H, _P, _P, _P, _I64]),
    "enmf_softimpute": (ctypes.c_int, [_H, _P, _I64, ctypes.c_int, _P, _I64, _P, _I64, _D]),
    "enmf_svd": (ctypes.c_int, [_H, _P, _I64, _P, _I64, _D]),
    "enmf_rotate": (ctypes.c_int, [_H, _P, _I64, _P, _I64, ctypes.POINTER(InitInfo)]),
    "enmf_init": (ctypes.c_int, [_H, _P, _I64, _P, _I64, _P, _I64, ctypes.POINTER(InitInfo)]),
    "enmf_rotate_rsr": (ctypes.c_int, [_H, _P, _I64, _P, _I64, ctypes.POINTER(InitInfo), _D]),
    "enmf_set_stage": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_double, ctypes.c_double]),
    "enmf_get_stage": (ctypes.c_int, [_H, ctypes.POINTER(ctypes.c_int), _D, _D]),
    "enmf_project": (ctypes.c_int, [_H, _P, _I64, _P, _I64]),
    "enmf_set_ablation": (ctypes.c_int, [_H, ctypes.c_int, ctypes.c_int]),
    "enmf_iterate": (ctypes.c_int, [_H, _P, _I64, _P, _I64, ctypes.c_int, _D,
                                    ctypes.POINTER(IterInfo)]),
    "enmf_iterate_host": (ctypes.c_int, [_H, _P, _P, ctypes.c_int, _D,
                                         ctypes.POINTER(IterInfo)]),
    "enmf_objective": (ctypes.c_int, [_H, _P, _I64, _P, _I64, ctypes.c_int, _D]),
    "enmf_kkt_residual": (ctypes.c_int, [_H, _P, _I64, _P, _I64, ctypes.POINTER(Kkt)]),
    "enmf_cross_terms": (ctypes.c_int, [_H, _P, _I64, _P, _I64, _P, _P]),
    "enmf_solve_host": (ctypes.c_int, [_H, _P, _P, _P, ctypes.c_int, _D,
                                       ctypes.POINTER(InitInfo)]),
    "enmf_launch_count": (ctypes.c_int64, [_H]),
    "enmf_set_profiling": (ctypes.c_int, [_H, ctypes.c_int]),
    "enmf_get_profile": (ctypes.c_int, [_H, _D, ctypes.POINTER(ctypes.c_int64)]),
    "enmf_set_host_allreduce": (ctypes.c_int, [_H, ctypes.c_void_p, ctypes.c_void_p]),
    "enmf_nccl_unique_id": (ctypes.c_int, [_P]),
    "enmf_precision_name": (ctypes.c_char_p, [_H]),
    "enmf_status_string": (ctypes.c_char_p, [ctypes.c_int]),
}
_HOST_AR = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                            ctypes.c_int64, ctypes.c_int)

for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)


def _check(code, where):
    if code != 0:
        raise EnmfError(code, where)


def default_options(**kw):
    o = Options()
    _lib.enmf_default_options(ctypes.byref(o))
    for k, v in kw.items():
        if not hasattr(o, k):
            raise TypeError(f"unknown option {k}")
        setattr(o, k, v)
    return o


def _mat(t, cols, name):
    """(device pointer, leading dim) of a 2-D fp32 CUDA tensor with unit column stride."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float32:
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    if t.dim() != 2 or t.shape[1] != cols or (t.shape[0] > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be (rows x {cols}) with unit column stride")
    return t.data_ptr(), max(t.stride(0), cols)


def _info_dict(s):
    out = {}
    for f, _ in s._fields_:
        v = getattr(s, f)
        out[f] = list(v) if hasattr(v, "__len__") else v
    return out


class Enmf:
    """One eNMF problem on the current CUDA device (one rank of a row-sharded job)."""

    def __init__(self, m, n, r, *, row_begin=0, row_count=None, world_size=1, rank=0,
                 nccl_id=None, stream=None, **options):
        import torch
        self.m, self.n, self.r = int(m), int(n), int(r)
        self.row_begin = int(row_begin)
        self.rows = int(row_count if row_count is not None else m)
        self._stream = stream if stream is not None else torch.cuda.current_stream()
        self._uid = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be the 128-byte ncclUniqueId")
            self._uid = ctypes.create_string_buffer(bytes(nccl_id), 128)
        # world_size > 1 without nccl_id: collectives via set_host_allreduce
        prob = Problem(self.m, self.n, self.r, self.row_begin, self.rows, int(world_size),
                       int(rank), ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None,
                       self._stream.cuda_stream)
        self.options = default_options(**options)
        h = _H()
        _check(_lib.enmf_create(ctypes.byref(prob), ctypes.byref(self.options), ctypes.byref(h)),
               "enmf_create")
        self._h = h
        self._X = None

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None) and _lib is not None:   # _lib is None at interpreter exit
            _lib.enmf_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def launch_count(self):
        return int(_lib.enmf_launch_count(self._h))

    @property
    def precision(self):
        return _lib.enmf_precision_name(self._h).decode()

    def set_profiling(self, on=True):
        _check(_lib.enmf_set_profiling(self._h, int(bool(on))), "enmf_set_profiling")

    def profile(self):
        """{'xv': (ms, passes), 'xtu': (ms, passes)} since set_profiling."""
        ms = (ctypes.c_double * 2)()
        cnt = (ctypes.c_int64 * 2)()
        _check(_lib.enmf_get_profile(self._h, ms, cnt), "enmf_get_profile")
        return {"xv": (ms[0], cnt[0]), "xtu": (ms[1], cnt[1])}

    # -- calls
    def set_data(self, X):
        px, ldx = _mat(X, self.n, "X")
        self._X = X
        _check(_lib.enmf_set_data(self._h, px, ldx), "enmf_set_data")

    def set_data_csr(self, row_ptr, col_idx, vals):
        """Bind this rank's rows of a sparse X as CSR CUDA tensors (row_ptr int64 of length
        row_count + 1, col_idx int32 ascending per row, vals float32); see enmf_set_data_csr."""
        import torch
        for t, dt, name in ((row_ptr, torch.int64, "row_ptr"), (col_idx, torch.int32, "col_idx"),
                            (vals, torch.float32, "vals")):
            if not (t.is_cuda and t.dtype == dt and t.is_contiguous()):
                raise TypeError(f"{name}: contiguous CUDA {dt} tensor required")
        if row_ptr.numel() != self.rows + 1 or col_idx.numel() != vals.numel():
            raise ValueError("row_ptr / col_idx / vals sizes")
        self._X = (row_ptr, col_idx, vals)
        _check(_lib.enmf_set_data_csr(self._h, row_ptr.data_ptr(), col_idx.data_ptr() or None,
                                      vals.data_ptr() or None, int(vals.numel())),
               "enmf_set_data_csr")

    def rotate_rsr(self, U, V):
        """RSR-ADMM (App. A) from (U*, V*) in place: returns (init-info dict, Lambda)."""
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        info = InitInfo()
        lam = np.zeros(self.r)
        _check(_lib.enmf_rotate_rsr(self._h, pu, ldu, pv, ldv, ctypes.byref(info),
                                    lam.ctypes.data_as(_D)), "enmf_rotate_rsr")
        return _info_dict(info), lam

    def set_data_masked(self, row_ptr, col_idx, vals):
        """eNMC: bind the OBSERVED entries of X as CSR CUDA tensors (same layout as
        set_data_csr); unlisted entries are missing (enmf_set_data_masked)."""
        import torch
        for t, dt, name in ((row_ptr, torch.int64, "row_ptr"), (col_idx, torch.int32, "col_idx"),
                            (vals, torch.float32, "vals")):
            if not (t.is_cuda and t.dtype == dt and t.is_contiguous()):
                raise TypeError(f"{name}: contiguous CUDA {dt} tensor required")
        if row_ptr.numel() != self.rows + 1 or col_idx.numel() != vals.numel():
            raise ValueError("row_ptr / col_idx / vals sizes")
        self._X = (row_ptr, col_idx, vals)
        _check(_lib.enmf_set_data_masked(self._h, row_ptr.data_ptr(), col_idx.data_ptr() or None,
                                         vals.data_ptr() or None, int(vals.numel())),
               "enmf_set_data_masked")

    def softimpute(self, U0, iters, U, V):
        """softImpute-ALS (lambda = 0) from the start U0: writes A into U, B into V; returns D."""
        p0, ld0 = _mat(U0, self.r, "U0")
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        d = np.zeros(self.r)
        _check(_lib.enmf_softimpute(self._h, p0, ld0, int(iters), pu, ldu, pv, ldv,
                                    d.ctypes.data_as(_D)), "enmf_softimpute")
        return d

    def svd(self, U, V):
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        sig = np.zeros(self.r)
        _check(_lib.enmf_svd(self._h, pu, ldu, pv, ldv, sig.ctypes.data_as(_D)), "enmf_svd")
        return sig

    def rotate(self, U, V):
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        info = InitInfo()
        _check(_lib.enmf_rotate(self._h, pu, ldu, pv, ldv, ctypes.byref(info)), "enmf_rotate")
        return _info_dict(info)

    def init(self, X, U, V):
        px, ldx = _mat(X, self.n, "X")
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        self._X = X
        info = InitInfo()
        _check(_lib.enmf_init(self._h, px, ldx, pu, ldu, pv, ldv, ctypes.byref(info)), "enmf_init")
        d = _info_dict(info)
        d["sigma"] = d["sigma"][: self.r]
        return d

    def set_stage(self, stage, lambda_u=0.0, lambda_v=0.0):
        _check(_lib.enmf_set_stage(self._h, int(stage), float(lambda_u), float(lambda_v)),
               "enmf_set_stage")

    def get_stage(self):
        s = ctypes.c_int()
        lu, lv = ctypes.c_double(), ctypes.c_double()
        _check(_lib.enmf_get_stage(self._h, ctypes.byref(s), ctypes.byref(lu), ctypes.byref(lv)),
               "enmf_get_stage")
        return s.value, lu.value, lv.value

    def project(self, U, V):
        """Post-rotation variant 'projection + HALS': U, V <- max(0, .)
        in place and the HALS stage."""
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        _check(_lib.enmf_project(self._h, pu, ldu, pv, ldv), "enmf_project")

    def set_ablation(self, step_rule=0, descent=0):
        """Ablation variants (R29): fixed ascent step 1/lambda_max, projected-gradient descent."""
        _check(_lib.enmf_set_ablation(self._h, int(step_rule), int(descent)), "enmf_set_ablation")

    def iterate(self, U, V, n_iters, trace=True):
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        f = np.zeros(max(int(n_iters), 1))
        info = IterInfo()
        _check(_lib.enmf_iterate(self._h, pu, ldu, pv, ldv, int(n_iters),
                                 f.ctypes.data_as(_D) if trace else None, ctypes.byref(info)),
               "enmf_iterate")
        return f[: int(n_iters)], _info_dict(info)

    def set_host_allreduce(self, fn):
        """Multi-rank handle without an NCCL id: fn(buf, op) reduces the float64 numpy array
        buf in place across the ranks (op 'sum' | 'min' | 'max'); see enmf_set_host_allreduce.
        Typically a torch.distributed (gloo) all_reduce on torch.from_numpy(buf)."""
        ops = {0: "sum", 1: "min", 2: "max"}

        def tramp(ctx, buf, count, op):
            try:
                arr = np.ctypeslib.as_array(buf, shape=(count,))
                fn(arr, ops[op])
                return 0
            except Exception:           # noqa: BLE001 -- reported as ENMF_ERR_NCCL
                import traceback
                traceback.print_exc()
                return 1

        self._host_ar = _HOST_AR(tramp)        # keep the callback alive with the handle
        _check(_lib.enmf_set_host_allreduce(self._h, ctypes.cast(self._host_ar, ctypes.c_void_p),
                                            None), "enmf_set_host_allreduce")

    def iterate_host(self, U, V, n_iters, trace=True):
        """enmf_iterate_host: U (row_count x r) and V (n x r) are contiguous fp32 CPU tensors
        (pinned for asynchronous copies) or numpy arrays, updated in place."""
        for name, A, rows in (("U", U, self.rows), ("V", V, self.n)):
            shape = tuple(A.shape)
            dev = getattr(A, "device", None)
            contig = A.is_contiguous() if hasattr(A, "is_contiguous") else \
                A.flags["C_CONTIGUOUS"]
            if shape != (rows, self.r) or (dev is not None and dev.type != "cpu") or not contig:
                raise EnmfError(-1, f"iterate_host: {name} must be a contiguous CPU "
                                    f"({rows}, {self.r}) array")
            if str(getattr(A, "dtype", "")) not in ("torch.float32", "float32"):
                raise EnmfError(-1, f"iterate_host: {name} must be float32")
        pu = U.data_ptr() if hasattr(U, "data_ptr") else U.ctypes.data
        pv = V.data_ptr() if hasattr(V, "data_ptr") else V.ctypes.data
        f = np.zeros(max(int(n_iters), 1))
        info = IterInfo()
        _check(_lib.enmf_iterate_host(self._h, ctypes.c_void_p(pu), ctypes.c_void_p(pv),
                                      int(n_iters), f.ctypes.data_as(_D) if trace else None,
                                      ctypes.byref(info)), "enmf_iterate_host")
        return f[: int(n_iters)], _info_dict(info)

    def objective(self, U, V, exact=False):
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        f = ctypes.c_double()
        _check(_lib.enmf_objective(self._h, pu, ldu, pv, ldv, int(bool(exact)), ctypes.byref(f)),
               "enmf_objective")
        return f.value

    def cross_terms(self, U, V):
        """(P, Q) = (X V, X^T U) as float64 CUDA tensors (the two X passes of a sweep)."""
        import torch
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        P = torch.empty(self.rows, self.r, dtype=torch.float64, device="cuda")
        Q = torch.empty(self.n, self.r, dtype=torch.float64, device="cuda")
        _check(_lib.enmf_cross_terms(self._h, pu, ldu, pv, ldv, P.data_ptr(), Q.data_ptr()),
               "enmf_cross_terms")
        return P, Q

    def kkt(self, U, V):
        pu, ldu = _mat(U, self.r, "U")
        pv, ldv = _mat(V, self.r, "V")
        k = Kkt()
        _check(_lib.enmf_kkt_residual(self._h, pu, ldu, pv, ldv, ctypes.byref(k)),
               "enmf_kkt_residual")
        return _info_dict(k)

    def solve_host(self, X_host, n_iters):
        """End to end from host memory: X_host (m x n float32 numpy, C order)."""
        X_host = np.ascontiguousarray(X_host, dtype=np.float32)
        if X_host.shape != (self.m, self.n):
            raise ValueError("X_host shape mismatch")
        U = np.zeros((self.m, self.r), np.float32)
        V = np.zeros((self.n, self.r), np.float32)
        f = np.zeros(max(int(n_iters), 1))
        info = InitInfo()
        _check(_lib.enmf_solve_host(self._h, X_host.ctypes.data, U.ctypes.data, V.ctypes.data,
                                    int(n_iters), f.ctypes.data_as(_D), ctypes.byref(info)),
               "enmf_solve_host")
        return U, V, f[: int(n_iters)], _info_dict(info)


def nccl_unique_id():
    # torch first: its libtorch_cuda.so binds the NCCL it ships (2.28); libenmf.so dlopens
    # "libnccl.so.2", which then resolves to that already-loaded copy instead of loading the
    # system one (2.27), which torch's later import would fail to link against
    import torch  # noqa: F401
    buf = ctypes.create_string_buffer(128)
    _check(_lib.enmf_nccl_unique_id(buf), "enmf_nccl_unique_id")
    return buf.raw


def row_partition(m, world_size, rank):
    """Rows [begin, begin+count) of rank `rank` in the row-sharded layout:
    contiguous blocks, the first m % world_size ranks one row longer."""
    base, extra = divmod(int(m), int(world_size))
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)
