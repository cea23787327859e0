"""ctypes binding of the fp64 CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package
paper_2605_19325_b200.  All arrays are numpy; X is float32 (the exact input bytes),
factors are float64 row-major.  See oracle.h for the cited passages.
"""
import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_F = ctypes.POINTER(ctypes.c_float)
_U8 = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64


class Options(ctypes.Structure):
    _fields_ = [("r", ctypes.c_int), ("oversample", ctypes.c_int), ("svd_tol", ctypes.c_double),
                ("svd_max_iter", ctypes.c_int), ("admm_iters", ctypes.c_int),
                ("admm_rho", ctypes.c_double), ("lift_steps", ctypes.c_int),
                ("pbcd_eps", ctypes.c_double), ("pbcd_max_iter", ctypes.c_int),
                ("round_f32", ctypes.c_int), ("step_rule", ctypes.c_int),
                ("descent", ctypes.c_int)]


class State(ctypes.Structure):
    _fields_ = [("stage", ctypes.c_int), ("lambda_u", ctypes.c_double),
                ("lambda_v", ctypes.c_double), ("sweeps_done", ctypes.c_int)]


def options(r, oversample=10, svd_tol=1e-13, svd_max_iter=500, admm_iters=100, admm_rho=0.0,
            lift_steps=10, pbcd_eps=1e-2, pbcd_max_iter=50, round_f32=0, step_rule=0,
            descent=0):
    """round_f32=1: factor state stored in fp32 at block boundaries, as the C-ABI stores
    U and V (reading R26); the arithmetic itself stays fp64.  step_rule / descent select the
    ablation variants (fixed 1/lambda_max ascent step; projected-gradient descent; R29)."""
    return Options(r, oversample, svd_tol, svd_max_iter, admm_iters, admm_rho, lift_steps,
                   pbcd_eps, pbcd_max_iter, round_f32, step_rule, descent)


def lib():
    global _lib
    if _lib is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python __graft_entry__.py build`")
        L = ctypes.CDLL(path)
        L.or_xv.argtypes = [_F, _i64, _i64, _D, ctypes.c_int, _D]
        L.or_xtu.argtypes = [_F, _i64, _i64, _D, ctypes.c_int, _D]
        L.or_gram.argtypes = [_D, _i64, ctypes.c_int, _D]
        for f in ("or_frob2_direct", "or_frob2_trace"):
            getattr(L, f).argtypes = [_F, _i64, _i64, _D, _D, ctypes.c_int]
            getattr(L, f).restype = ctypes.c_double
        L.or_xnorm2.argtypes = [_F, _i64, _i64]
        L.or_xnorm2.restype = ctypes.c_double
        L.or_project.argtypes = [_D, _i64]
        L.or_project.restype = None
        L.or_negativity.argtypes = [_D, _i64]
        L.or_negativity.restype = ctypes.c_double
        L.or_svd_jacobi.argtypes = [_D, _i64, ctypes.c_int, _D, _D, _D]
        L.or_svd_jacobi.restype = ctypes.c_int
        L.or_orthonormalise.argtypes = [_D, _i64, ctypes.c_int]
        L.or_truncated_svd.argtypes = [_F, _i64, _i64, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.c_int, _D, _D, _D]
        L.or_truncated_svd.restype = ctypes.c_int
        L.or_zprox.argtypes = [ctypes.c_double, ctypes.c_double]
        L.or_zprox.restype = ctypes.c_double
        L.or_procrustes.argtypes = [_D, _D, _i64, ctypes.c_int, _D]
        L.or_admm_rotate.argtypes = [_D, _i64, ctypes.c_int, ctypes.c_double, ctypes.c_int, _D, _D]
        L.or_admm_rotate.restype = _i64
        L.or_lift.argtypes = [_D, _i64, ctypes.c_double]
        L.or_lift_constant.argtypes = [_D, _i64, ctypes.c_int]
        L.or_lift_constant.restype = ctypes.c_double
        L.or_pbcd.argtypes = [_D, _i64, ctypes.c_int, _D, _D, _U8, ctypes.c_double, ctypes.c_int,
                              _D, _D]
        L.or_pbcd.restype = ctypes.c_int
        L.or_hals.argtypes = [_D, _i64, ctypes.c_int, _D, _D]
        L.or_pbcd_step.argtypes = [_D, _i64, ctypes.c_int, _D, _D, _U8, ctypes.c_double,
                                   ctypes.c_int, ctypes.c_double, _D, _D]
        L.or_pbcd_step.restype = ctypes.c_int
        L.or_pgd.argtypes = [_D, _i64, ctypes.c_int, _D, _D, ctypes.c_double]
        L.or_pgd.restype = None
        L.or_lambda_max.argtypes = [_D, ctypes.c_int]
        L.or_lambda_max.restype = ctypes.c_double
        L.or_sweep.argtypes = [_F, _i64, _i64, _D, _D, ctypes.POINTER(Options),
                               ctypes.POINTER(State), ctypes.POINTER(ctypes.c_int)]
        L.or_sweep.restype = ctypes.c_int
        L.or_enmf.argtypes = [_F, _i64, _i64, ctypes.POINTER(Options), ctypes.c_int, _D, _D, _D,
                              _D, ctypes.POINTER(State)]
        L.or_enmf.restype = ctypes.c_int
        L.or_kkt.argtypes = [_F, _i64, _i64, _D, _D, ctypes.c_int, _D]
        _I64P = ctypes.POINTER(ctypes.c_int64)
        _I32P = ctypes.POINTER(ctypes.c_int32)
        L.or_nmc_objective.argtypes = [_I64P, _I32P, _F, _i64, _D, _D, ctypes.c_int]
        L.or_nmc_objective.restype = ctypes.c_double
        L.or_nmc_grad.argtypes = [_I64P, _I32P, _F, _i64, _D, _D, ctypes.c_int, _D]
        L.or_nmc_grad.restype = None
        L.or_nmc_pbcd.argtypes = [_I64P, _I32P, _F, _i64, _D, _D, ctypes.c_int, _U8,
                                  ctypes.c_double, ctypes.c_int, _D, _D]
        L.or_nmc_pbcd.restype = ctypes.c_int
        L.or_csr_transpose.argtypes = [_I64P, _I32P, _F, _i64, _i64, _I64P, _I32P, _F]
        L.or_csr_transpose.restype = None
        L.or_nmc_sweep.argtypes = [_I64P, _I32P, _F, _I64P, _I32P, _F, _i64, _i64, _D, _D,
                                   ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_int)]
        L.or_nmc_sweep.restype = None
        L.or_softimpute.argtypes = [_I64P, _I32P, _F, _i64, _i64, ctypes.c_int, _D,
                                    ctypes.c_int, _D, _D, _D]
        L.or_softimpute.restype = ctypes.c_int
        _lib = L
    return _lib


def _f32(X):
    X = np.ascontiguousarray(X, dtype=np.float32)
    return X, X.ctypes.data_as(_F)


def _f64(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    return A, A.ctypes.data_as(_D)


def _out(shape):
    A = np.zeros(shape, dtype=np.float64)
    return A, A.ctypes.data_as(_D)


def xv(X, V):
    X, px = _f32(X)
    V, pv = _f64(V)
    P, pp = _out((X.shape[0], V.shape[1]))
    lib().or_xv(px, X.shape[0], X.shape[1], pv, V.shape[1], pp)
    return P


def xtu(X, U):
    X, px = _f32(X)
    U, pu = _f64(U)
    Q, pq = _out((X.shape[1], U.shape[1]))
    lib().or_xtu(px, X.shape[0], X.shape[1], pu, U.shape[1], pq)
    return Q


def gram(A):
    A, pa = _f64(A)
    G, pg = _out((A.shape[1], A.shape[1]))
    lib().or_gram(pa, A.shape[0], A.shape[1], pg)
    return G


def frob2_direct(X, U, V):
    X, px = _f32(X)
    U, pu = _f64(U)
    V, pv = _f64(V)
    return lib().or_frob2_direct(px, X.shape[0], X.shape[1], pu, pv, U.shape[1])


def frob2_trace(X, U, V):
    X, px = _f32(X)
    U, pu = _f64(U)
    V, pv = _f64(V)
    return lib().or_frob2_trace(px, X.shape[0], X.shape[1], pu, pv, U.shape[1])


def xnorm2(X):
    X, px = _f32(X)
    return lib().or_xnorm2(px, X.shape[0], X.shape[1])


def negativity(A):
    A, pa = _f64(A)
    return lib().or_negativity(pa, A.size)


def project(A):
    """Post-rotation variant (ii) of the ablation: max(0, A) on a copy."""
    A = np.array(A, dtype=np.float64, order="C")
    lib().or_project(A.ctypes.data_as(_D), A.size)
    return A


def svd_jacobi(A):
    A, pa = _f64(A)
    rows, k = A.shape
    U, pu = _out((rows, k))
    s, ps = _out((k,))
    V, pv = _out((k, k))
    lib().or_svd_jacobi(pa, rows, k, pu, ps, pv)
    return U, s, V


def orthonormalise(Y):
    Y = np.array(Y, dtype=np.float64, order="C")
    lib().or_orthonormalise(Y.ctypes.data_as(_D), Y.shape[0], Y.shape[1])
    return Y


def truncated_svd(X, r, p=10, tol=1e-13, max_iter=500):
    X, px = _f32(X)
    m, n = X.shape
    Us, pu = _out((m, r))
    Vs, pv = _out((n, r))
    s, ps = _out((r,))
    it = lib().or_truncated_svd(px, m, n, r, p, tol, max_iter, pu, pv, ps)
    return Us, Vs, s, it


def zprox(b, rho):
    return lib().or_zprox(b, rho)


def procrustes(W, B):
    W, pw = _f64(W)
    B, pb = _f64(B)
    r = W.shape[1]
    R, pr = _out((r, r))
    lib().or_procrustes(pw, pb, W.shape[0], r, pr)
    return R


def admm_rotate(W, T=100, rho=0.0):
    W, pw = _f64(W)
    r = W.shape[1]
    R, pr = _out((r, r))
    neg, pn = _out((T,))
    third = lib().or_admm_rotate(pw, W.shape[0], r, rho, T, pr, pn)
    return R, neg, third


def lift(A, lam):
    A = np.array(A, dtype=np.float64, order="C")
    lib().or_lift(A.ctypes.data_as(_D), A.size, lam)
    return A


def lift_constant(A, L=10):
    A, pa = _f64(A)
    return lib().or_lift_constant(pa, A.size, L)


def pbcd(F, C, G, M, eps=1e-2, max_iter=50):
    F = np.array(F, dtype=np.float64, order="C")
    C, pc = _f64(C)
    G, pg = _f64(G)
    M = np.ascontiguousarray(M, dtype=np.uint8)
    g0 = ctypes.c_double()
    g1 = ctypes.c_double()
    it = lib().or_pbcd(F.ctypes.data_as(_D), F.shape[0], F.shape[1], pc, pg,
                       M.ctypes.data_as(_U8), eps, max_iter, ctypes.byref(g0), ctypes.byref(g1))
    return F, it, g0.value, g1.value


def pbcd_step(F, C, G, M, step, eps=1e-2, max_iter=50):
    F = np.array(F, dtype=np.float64, order="C")
    C, pc = _f64(C)
    G, pg = _f64(G)
    M = np.ascontiguousarray(M, dtype=np.uint8)
    g0 = ctypes.c_double()
    g1 = ctypes.c_double()
    it = lib().or_pbcd_step(F.ctypes.data_as(_D), F.shape[0], F.shape[1], pc, pg,
                            M.ctypes.data_as(_U8), eps, max_iter, step, ctypes.byref(g0),
                            ctypes.byref(g1))
    return F, it, g0.value, g1.value


def pgd(F, C, G, step):
    F = np.array(F, dtype=np.float64, order="C")
    C, pc = _f64(C)
    G, pg = _f64(G)
    lib().or_pgd(F.ctypes.data_as(_D), F.shape[0], F.shape[1], pc, pg, step)
    return F


def lambda_max(G):
    G, pg = _f64(G)
    return lib().or_lambda_max(pg, G.shape[0])


def hals(F, C, G):
    F = np.array(F, dtype=np.float64, order="C")
    C, pc = _f64(C)
    G, pg = _f64(G)
    lib().or_hals(F.ctypes.data_as(_D), F.shape[0], F.shape[1], pc, pg)
    return F


@dataclass
class SweepState:
    stage: int = 0
    lambda_u: float = 0.0
    lambda_v: float = 0.0
    sweeps_done: int = 0


def sweep(X, U, V, state: SweepState, opts=None):
    """One eNMF sweep in place on copies; returns (U, V, stage, (iters_u, iters_v))."""
    X, px = _f32(X)
    U = np.array(U, dtype=np.float64, order="C")
    V = np.array(V, dtype=np.float64, order="C")
    opts = opts or options(U.shape[1])
    st = State(state.stage, state.lambda_u, state.lambda_v, state.sweeps_done)
    it = (ctypes.c_int * 2)()
    stage = lib().or_sweep(px, X.shape[0], X.shape[1], U.ctypes.data_as(_D), V.ctypes.data_as(_D),
                           ctypes.byref(opts), ctypes.byref(st), it)
    state.stage, state.sweeps_done = st.stage, st.sweeps_done
    return U, V, stage, (it[0], it[1])


def enmf(X, r, n_sweeps, opts=None):
    """Alg. 3 end to end: returns (U, V, sigma, f_trace, SweepState)."""
    X, px = _f32(X)
    m, n = X.shape
    opts = opts or options(r)
    U, pu = _out((m, r))
    V, pv = _out((n, r))
    s, ps = _out((r,))
    f, pf = _out((max(n_sweeps, 1),))
    st = State()
    rc = lib().or_enmf(px, m, n, ctypes.byref(opts), n_sweeps, pu, pv, ps, pf, ctypes.byref(st))
    if rc != 0:
        raise ValueError(f"or_enmf failed: {rc}")
    return U, V, s, f[:n_sweeps], SweepState(st.stage, st.lambda_u, st.lambda_v, st.sweeps_done)


KKT_FIELDS = ("min_u", "min_v", "comp_max", "comp_sum", "delta_w", "sigma_w", "dual_viol",
              "xnorm2", "rms_cross")


def kkt(X, U, V):
    X, px = _f32(X)
    U, pu = _f64(U)
    V, pv = _f64(V)
    out, po = _out((9,))
    lib().or_kkt(px, X.shape[0], X.shape[1], pu, pv, U.shape[1], po)
    return dict(zip(KKT_FIELDS, out.tolist()))


# ---------------------------------------------------------------- eNMC (oracle_nmc.c)
class Observed:
    """Observed entries of an m x n X (eNMC) as CSR lists plus the
    transposed (CSC) lists the V block reads; built from a dense X and a boolean mask."""

    def __init__(self, X, mask):
        X = np.asarray(X, dtype=np.float32)
        mask = np.asarray(mask, dtype=bool)
        self.m, self.n = X.shape
        rows, cols = np.nonzero(mask)            # row-major order: columns ascend per row
        self.ptr = np.zeros(self.m + 1, dtype=np.int64)
        np.add.at(self.ptr, rows + 1, 1)
        self.ptr = np.cumsum(self.ptr).astype(np.int64)
        self.idx = cols.astype(np.int32)
        self.val = X[rows, cols].astype(np.float32)
        self.tptr = np.zeros(self.n + 1, dtype=np.int64)
        self.tidx = np.zeros(len(self.idx), dtype=np.int32)
        self.tval = np.zeros(len(self.idx), dtype=np.float32)
        lib().or_csr_transpose(*self._csr(), self.m, self.n, _p64(self.tptr), _p32(self.tidx),
                               self.tval.ctypes.data_as(_F))

    def _csr(self):
        return _p64(self.ptr), _p32(self.idx), self.val.ctypes.data_as(_F)

    def _csc(self):
        return _p64(self.tptr), _p32(self.tidx), self.tval.ctypes.data_as(_F)


def _p64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _p32(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def nmc_objective(obs, U, V):
    U, pu = _f64(U)
    V, pv = _f64(V)
    return lib().or_nmc_objective(*obs._csr(), obs.m, pu, pv, U.shape[1])


def nmc_grad(obs, U, V, block="U"):
    """grad_U f^ = (M_E o (U V^T - X)) V, or grad_V (block="V") from the transposed lists."""
    U, pu = _f64(U)
    V, pv = _f64(V)
    if block == "U":
        G, pg = _out(U.shape)
        lib().or_nmc_grad(*obs._csr(), obs.m, pu, pv, U.shape[1], pg)
    else:
        G, pg = _out(V.shape)
        lib().or_nmc_grad(*obs._csc(), obs.n, pv, pu, V.shape[1], pg)
    return G


def nmc_pbcd(obs, F, O, M, block="U", eps=1e-2, max_iter=50):
    """PBCD of one block (F = U with O = V for block "U", F = V with O = U for "V");
    returns (F_new, iterations, pg0, pg_last)."""
    F = np.array(F, dtype=np.float64, order="C")
    O, po = _f64(O)
    M = np.ascontiguousarray(M, dtype=np.uint8)
    g0, g1 = ctypes.c_double(), ctypes.c_double()
    lists = obs._csr() if block == "U" else obs._csc()
    rows = obs.m if block == "U" else obs.n
    it = lib().or_nmc_pbcd(*lists, rows, F.ctypes.data_as(_D), po, F.shape[1],
                           M.ctypes.data_as(_U8), eps, max_iter, ctypes.byref(g0),
                           ctypes.byref(g1))
    return F, it, g0.value, g1.value


def nmc_sweep(obs, U, V, lambda_u, lambda_v, eps=1e-2, max_iter=50, round_f32=1):
    """One eNMC sweep (Alg. NMC loop body); returns (U, V, (iters_u, iters_v))."""
    U = np.array(U, dtype=np.float64, order="C")
    V = np.array(V, dtype=np.float64, order="C")
    it = (ctypes.c_int * 2)()
    lib().or_nmc_sweep(*obs._csr(), *obs._csc(), obs.m, obs.n, U.ctypes.data_as(_D),
                       V.ctypes.data_as(_D), U.shape[1], lambda_u, lambda_v, eps, max_iter,
                       round_f32, it)
    return U, V, (it[0], it[1])


def softimpute(obs, U0, iters):
    """softImpute-ALS, lambda = 0 (reading R31): returns (A, B, d)."""
    U0, pu = _f64(U0)
    r = U0.shape[1]
    A, pa = _out((obs.m, r))
    B, pb = _out((obs.n, r))
    d, pd = _out((r,))
    rc = lib().or_softimpute(*obs._csr(), obs.m, obs.n, r, pu, iters, pa, pb, pd)
    if rc != 0:
        raise ValueError("softimpute: a half-step product has a zero singular value")
    return A, B, d
