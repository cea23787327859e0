"""Pins of the fp64 oracle against what the paper and mathematics fix.

None of these compare the oracle with itself: each uses a closed form, a library routine
(LAPACK via numpy, allowed in tests only), a brute-force search, a hand-computed example
or an invariant of the method.  Citations are PAPER.md lines.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def rand_orth(r, seed):
    q, rr = np.linalg.qr(np.random.default_rng(seed).standard_normal((r, r)))
    return q * np.sign(np.diag(rr))


# ---------------------------------------------------------------- P6 objective (Eq.1)
def test_objective_direct_matches_definition_and_trace():
    X = synth.x_full(synth.C1)
    g = np.random.default_rng(1)
    U, V = g.random((200, 5)), g.random((100, 5))
    f_lib = float(((X.astype(np.float64) - U @ V.T) ** 2).sum())   # numpy as a library step
    f_d = oracle.frob2_direct(X, U, V)
    f_t = oracle.frob2_trace(X, U, V)
    assert rel(f_d, f_lib) < 1e-12
    # trace form agrees up to its conditioning ||X||^2/f (Hard part 2)
    assert rel(f_t, f_d) < 1e-15 * oracle.xnorm2(X) / f_d * 50


def test_objective_zero_at_exact_factorization():
    g = np.random.default_rng(2)
    U = g.integers(0, 4, (9, 3)).astype(np.float64)
    V = g.integers(0, 4, (7, 3)).astype(np.float64)
    X = (U @ V.T).astype(np.float32)          # small integers: exact in fp32
    assert oracle.frob2_direct(X, U, V) == 0.0
    assert oracle.frob2_trace(X, U, V) == 0.0


def test_objective_level_set_invariance():
    """f(UR, VR) = f(U, V) for R^T R = I (Eq.(2) 135-138)."""
    X = synth.x_full(synth.C1)
    g = np.random.default_rng(3)
    U, V = g.standard_normal((200, 5)), g.standard_normal((100, 5))
    R = rand_orth(5, 4)
    assert rel(oracle.frob2_direct(X, U @ R, V @ R), oracle.frob2_direct(X, U, V)) < 1e-12


def test_negativity_hand_example():
    assert oracle.negativity(np.array([[-1.0, 2.0], [-3.0, 0.0]])) == 4.0


# ---------------------------------------------------------------- P1 truncated SVD
@pytest.mark.parametrize("cfg", [synth.C1, synth.C3.scaled(160, 700, 12, 12)])
def test_svd_eckart_young_against_lapack(cfg):
    X = synth.x_full(cfg)
    r = cfg.r
    Us, Vs, s, it = oracle.truncated_svd(X, r)
    assert it > 0, "subspace iteration did not converge"
    Ul, sl, Vlt = np.linalg.svd(X.astype(np.float64), full_matrices=False)
    assert np.allclose(s, sl[:r], rtol=1e-10, atol=0)
    f_ey = float((sl[r:] ** 2).sum())
    assert rel(oracle.frob2_direct(X, Us, Vs), f_ey) < 1e-9
    # balanced scaling U* = U S^1/2, V* = V S^1/2
    assert np.allclose(np.linalg.norm(Us, axis=0), np.sqrt(s), rtol=1e-10)
    assert np.allclose(np.linalg.norm(Vs, axis=0), np.sqrt(s), rtol=1e-10)
    # singular directions equal LAPACK's up to sign; sign rule R5
    for k in range(r):
        u = Us[:, k] / np.sqrt(s[k])
        assert abs(abs(u @ Ul[:, k]) - 1) < 1e-9
        assert u[np.argmax(np.abs(u))] > 0


def test_svd_diag_example():
    """X = diag(3,2,1), r = 2 -> sigma = (3,2), residual 1."""
    X = np.diag([3.0, 2.0, 1.0]).astype(np.float32)
    Us, Vs, s, _ = oracle.truncated_svd(X, 2)
    assert np.allclose(s, [3.0, 2.0], rtol=1e-12)
    assert abs(oracle.frob2_direct(X, Us, Vs) - 1.0) < 1e-12


def test_svd_known_factor_map():
    """App. A.1: for X = U0 V0^T of rank r, A = S^-1/2 U_r^T U0 gives
    U* A = U0 and V* A^-T = V0."""
    g = np.random.default_rng(5)
    U0 = g.integers(0, 3, (30, 4)).astype(np.float64)
    V0 = g.integers(0, 3, (25, 4)).astype(np.float64)
    X = (U0 @ V0.T).astype(np.float32)
    Us, Vs, s, _ = oracle.truncated_svd(X, 4)
    Ur = Us / np.sqrt(s)
    A = np.diag(s ** -0.5) @ Ur.T @ U0
    assert np.abs(Us @ A - U0).max() < 1e-9
    assert np.abs(Vs @ np.linalg.inv(A).T - V0).max() < 1e-9


# ---------------------------------------------------------------- P2 rotation (Alg. 1)
def test_zprox_is_the_eq7_minimiser():
    """Eq.(7) PAPER.md:182-190 vs brute-force grid minimisation of h(z) + rho/2 (z-b)^2."""
    assert oracle.zprox(0.5, 1.0) == 0.5 and oracle.zprox(-0.5, 1.0) == 0.0
    assert oracle.zprox(-2.0, 1.0) == -1.0
    zs = np.linspace(-6, 6, 240001)
    for rho in (0.5, 1.0, 3.0):
        for b in np.linspace(-5, 5, 41):
            obj = np.maximum(0, -zs) + rho / 2 * (zs - b) ** 2
            assert abs(oracle.zprox(b, rho) - zs[np.argmin(obj)]) < 1e-4


def test_procrustes_recovers_planted_rotation():
    g = np.random.default_rng(6)
    W = g.standard_normal((50, 6))
    Q = rand_orth(6, 7)
    assert np.abs(oracle.procrustes(W, W @ Q) - Q).max() < 1e-10


def test_procrustes_beats_angle_sweep():
    """R = C D^T minimises ||B - W R||_F over the orthogonal group."""
    g = np.random.default_rng(8)
    W, B = g.standard_normal((40, 2)), g.standard_normal((40, 2))
    R = oracle.procrustes(W, B)
    best = np.inf
    for th in np.linspace(0, 2 * np.pi, 3600, endpoint=False):
        c, s = np.cos(th), np.sin(th)
        for Rt in (np.array([[c, -s], [s, c]]), np.array([[c, s], [s, -c]])):
            best = min(best, np.linalg.norm(B - W @ Rt))
    assert np.linalg.norm(B - W @ R) <= best + 1e-12
    assert np.abs(R.T @ R - np.eye(2)).max() < 1e-13


def _rotated_c1():
    X = synth.x_full(synth.C1)
    Us, Vs, s, _ = oracle.truncated_svd(X, 5)
    return X, Us, Vs, s


def test_admm_orthogonal_invariant_and_projection_regime():
    X, Us, Vs, _ = _rotated_c1()
    W = np.vstack([Us, Vs])
    R, neg, third = oracle.admm_rotate(W, T=100)
    assert third == 0                                       # reading R7
    assert np.abs(R.T @ R - np.eye(5)).max() < 1e-12
    f0 = oracle.frob2_direct(X, Us, Vs)
    assert rel(oracle.frob2_direct(X, Us @ R, Vs @ R), f0) < 1e-12
    assert neg[-1] < 0.01 * oracle.negativity(W)
    # in the projection regime the scaled iteration does not depend on rho (R7)
    wmax = np.abs(W).max()
    R2, _, third2 = oracle.admm_rotate(W, T=100, rho=1e-4 / wmax)
    assert third2 == 0 and np.abs(R2 - R).max() < 1e-10


def test_admm_reaches_orthant_on_dense_synthetic_analog():
    """Scaled analog of the paper's dense synthetic family (Table 3):
    rotation alone reaches the orthant, so eNMF ends at the unconstrained optimum
    (relative error 1.00)."""
    g = np.random.default_rng(9)
    Wt, H = g.random((500, 100)), g.random((100, 500))
    S = Wt @ H
    sig = np.sqrt((S ** 2).mean() / 10 ** (40 / 10))
    X = (S + sig * g.standard_normal(S.shape)).astype(np.float32)
    r = 10
    Us, Vs, s, _ = oracle.truncated_svd(X, r)
    # the step count is not the paper's 1-5 (reading R8): this analog needs ~104 steps
    R, neg, third = oracle.admm_rotate(np.vstack([Us, Vs]), T=200)
    assert third == 0 and neg[-1] == 0.0
    U, V, sig2, f, st = oracle.enmf(X, r, 5, oracle.options(r, admm_iters=200))
    f_ey = oracle.frob2_direct(X, Us, Vs)
    assert st.stage == 1 and rel(f[-1], f_ey) < 1e-9


# ---------------------------------------------------------------- P3 lift (Eq.6/7)
def test_lift_examples():
    assert oracle.lift(np.array([[-0.3]]), 0.1)[0, 0] == pytest.approx(-0.2, abs=1e-15)
    g = np.random.default_rng(10)
    A = g.standard_normal((30, 7))
    B = oracle.lift(A, 0.05)
    assert ((B != A) == (A < 0)).all()
    assert (B[A >= 0] == A[A >= 0]).all()


def test_lift_constant_gives_exactly_L_lifts():
    g = np.random.default_rng(11)
    A = g.standard_normal((40, 6))
    lam = oracle.lift_constant(A, 10)
    B = A.copy()
    for t in range(1, 11):
        B = oracle.lift(B, lam)
        assert (B.min() >= 0) == (t == 10)


# ---------------------------------------------------------------- P4 step size (Eq.10, App. B)
def _golden(phi, lo, hi, iters=200):
    gr = (np.sqrt(5) - 1) / 2
    a, b = lo, hi
    for _ in range(iters):
        c, d = b - gr * (b - a), a + gr * (b - a)
        if phi(c) < phi(d):
            b = d
        else:
            a = c
    return (a + b) / 2


def test_pbcd_step_is_exact_line_minimiser():
    """App. B: d* minimises ||X_i - (U_i - d g_i) V^T||^2."""
    g = np.random.default_rng(12)
    n, r = 60, 5
    for trial in range(10):
        V = g.random((n, r))
        x = g.random(n) * 3
        u = 5 + g.random(r)                                   # far from 0: no projection
        P = (x @ V)[None, :]
        G = V.T @ V
        mask = np.ones((1, r), dtype=np.uint8)
        unew, it, _, _ = oracle.pbcd(u[None, :], P, G, mask, eps=0.0, max_iter=1)
        grad = (np.outer(u, 1) @ np.ones((1, 1))).ravel() * 0 + ((u @ V.T - x) @ V)  # literal (uV^T - x) V
        d_or = float(np.median((u - unew[0]) / grad))
        phi = lambda d: float(((x - (u - d * grad) @ V.T) ** 2).sum())
        d_gs = _golden(phi, 0.0, 10 * d_or + 1.0)
        assert rel(d_or, d_gs) < 1e-8


def test_pbcd_step_scaled_orthonormal():
    """V with orthonormal columns scaled by c gives d* = 1/c^2."""
    q, _ = np.linalg.qr(np.random.default_rng(13).standard_normal((20, 4)))
    c = 2.5
    V = c * q
    x = V @ np.array([1.0, 2.0, 3.0, 4.0])        # minimiser inside the orthant: no clipping
    u = np.full(4, 50.0)
    grad = (u @ V.T - x) @ V
    unew, _, _, _ = oracle.pbcd(u[None, :], (x @ V)[None, :], V.T @ V, np.ones((1, 4), np.uint8),
                                eps=0.0, max_iter=1)
    assert np.allclose((u - unew[0]) / grad, 1 / c ** 2, rtol=1e-12)


def test_pbcd_gradient_literal_and_stopping_rule():
    """Alg. 2 line 235 uses M o ((U V^T - X) V) and stops at the first sweep with
    projected_grad < eps * initial."""
    g = np.random.default_rng(15)
    m, n, r = 30, 20, 4
    X = g.random((m, n)).astype(np.float32)
    U, V = g.standard_normal((m, r)), g.random((n, r))
    M = (U >= 0).astype(np.uint8)
    lit = M * ((U @ V.T - X.astype(np.float64)) @ V)
    P, G = X.astype(np.float64) @ V, V.T @ V
    _, it, pg0, pg = oracle.pbcd(U, P, G, M, eps=1e-2, max_iter=500)
    assert rel(pg0, np.linalg.norm(lit)) < 1e-12
    assert 1 < it < 500 and pg < 1e-2 * pg0
    Uk, _, _, pgk = oracle.pbcd(U, P, G, M, eps=0.0, max_iter=it - 1)
    assert pgk >= 1e-2 * pg0
    # masked entries untouched bit for bit, free entries projected to >= 0
    Un, _, _, _ = oracle.pbcd(U, P, G, M, eps=1e-2, max_iter=500)
    assert (Un[M == 0] == U[M == 0]).all() and (Un[M == 1] >= 0).all()


def test_pbcd_state_rounding_sensitivity():
    """Why reading R26 exists: on the image-like data the ascent stage amplifies a 1e-7
    perturbation of the factor state by >= 1e3 (projection active sets change), so the GPU
    (fp32 state) is compared with the oracle rounding its state to fp32 at the same points."""
    from tests.gpu_common import rotated_point, rel_fro
    cfg = synth.C2.scaled(150, 700, 49, 49)
    X = synth.x_full(cfg)
    U0, V0, lu, lv = rotated_point(X, 49)
    a = oracle.sweep(X, U0, V0, oracle.SweepState(0, lu, lv, 0))
    g = np.random.default_rng(1)
    b = oracle.sweep(X, U0 * (1 + 1e-7 * g.standard_normal(U0.shape)), V0,
                     oracle.SweepState(0, lu, lv, 0))
    assert rel_fro(b[1], a[1]) > 1e3 * 1e-7
    c = oracle.sweep(X, U0, V0, oracle.SweepState(0, lu, lv, 0), oracle.options(49, round_f32=1))
    assert np.array_equal(c[0], c[0].astype(np.float32).astype(np.float64))
    assert np.array_equal(c[1], c[1].astype(np.float32).astype(np.float64))


# ---------------------------------------------------------------- P5 HALS
def test_project_is_the_bounded_least_squares_solution():
    """or_project (ablation variant (ii)) against the Euclidean projection
    onto {Y >= 0} computed by a bounded least-squares solver (scipy lsq_linear on the identity
    system, bounds [0, inf)) -- a different algorithm for the same minimiser -- plus the
    special cases: idempotent, fixes the orthant, zero on the negative orthant."""
    from scipy.optimize import lsq_linear
    g = np.random.default_rng(11)
    A = g.normal(size=(6, 5))
    P = oracle.project(A)
    ref = lsq_linear(np.eye(A.size), A.ravel(), bounds=(0.0, np.inf), tol=1e-14).x
    assert np.allclose(P.ravel(), ref, atol=1e-12)
    assert np.array_equal(oracle.project(P), P)
    B = np.abs(A)
    assert np.array_equal(oracle.project(B), B)
    assert np.array_equal(oracle.project(-B), np.zeros_like(B))


def _block_f(F, C, G):
    """f(F) - const = 1/2 tr(F G F^T) - tr(F^T C) for the block problem min 1/2 ||X - F W^T||^2
    with C = X W, G = W^T W."""
    return 0.5 * np.sum((F @ G) * F) - np.sum(F * C)


def test_lambda_max_against_eigvalsh():
    g = np.random.default_rng(21)
    for r in (1, 5, 33):
        A = g.random((60, r))
        G = A.T @ A
        assert abs(oracle.lambda_max(G) - np.linalg.eigvalsh(G)[-1]) <= 1e-12 * np.linalg.eigvalsh(G)[-1]


def test_pgd_descent_lemma_and_nnls_fixed_point():
    """or_pgd (ablation 'standard gradient descent', reading R29): with step 1/lambda_max(G)
    the projected-gradient step cannot increase the block objective (descent lemma + the
    projection's non-expansiveness), and the exact per-row NNLS solution (scipy nnls, an
    active-set method) is a fixed point."""
    from scipy.optimize import nnls
    g = np.random.default_rng(22)
    X = g.random((40, 30))
    W = g.random((30, 6))
    C, G = X @ W, W.T @ W
    L = oracle.lambda_max(G)
    F = g.normal(size=(40, 6))
    f_prev = _block_f(np.maximum(F, 0), C, G)
    F = np.maximum(F, 0)
    for _ in range(20):
        F = oracle.pgd(F, C, G, 1.0 / L)
        f = _block_f(F, C, G)
        assert f <= f_prev + 1e-12 * abs(f_prev)
        f_prev = f
    Fs = np.array([nnls(W, X[i])[0] for i in range(X.shape[0])])
    assert np.allclose(oracle.pgd(Fs, C, G, 1.0 / L), Fs, atol=1e-9)


def test_pbcd_fixed_step_is_monotone():
    """or_pbcd_step with the fixed step 1/lambda_max(G) (ablation 'fixed step size', R29) and
    every entry free: the block objective is non-increasing over the inner iterations, and
    step <= 0 reproduces or_pbcd (Eq.(10))."""
    g = np.random.default_rng(23)
    X = g.random((25, 20))
    W = g.random((20, 5))
    C, G = X @ W, W.T @ W
    F0 = np.abs(g.normal(size=(25, 5)))
    M = np.ones_like(F0, dtype=np.uint8)
    L = oracle.lambda_max(G)
    f_prev = _block_f(F0, C, G)
    F = F0
    for _ in range(10):
        F, it, _, _ = oracle.pbcd_step(F, C, G, M, 1.0 / L, eps=0.0, max_iter=1)
        f = _block_f(F, C, G)
        assert f <= f_prev + 1e-12 * abs(f_prev)
        f_prev = f
    a = oracle.pbcd(F0, C, G, M, max_iter=7)
    b = oracle.pbcd_step(F0, C, G, M, 0.0, max_iter=7)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]


def test_hals_matches_textbook_residual_form():
    """HALS (cited Cichocki & Phan): column k is the projected
    least-squares solution max(0, (X - sum_{l!=k} U_l V_l^T) V_k / ||V_k||^2)."""
    g = np.random.default_rng(16)
    m, n, r = 25, 18, 4
    X = g.random((m, n)).astype(np.float32)
    U, V = g.random((m, r)), g.random((n, r))
    Uo = oracle.hals(U, X.astype(np.float64) @ V, V.T @ V)
    Ut = U.copy()
    Xd = X.astype(np.float64)
    for k in range(r):
        Rk = Xd - Ut @ V.T + np.outer(Ut[:, k], V[:, k])
        Ut[:, k] = np.maximum(0, Rk @ V[:, k] / (V[:, k] @ V[:, k]))
    assert np.abs(Uo - Ut).max() < 1e-12


def test_hals_sweeps_monotone():
    X, Us, Vs, _ = _rotated_c1()
    U, V = np.abs(Us), np.abs(Vs)
    st = oracle.SweepState(stage=1)
    f_prev = oracle.frob2_direct(X, U, V)
    for _ in range(20):
        U, V, stage, _ = oracle.sweep(X, U, V, st)
        f = oracle.frob2_direct(X, U, V)
        assert stage == 1 and f <= f_prev * (1 + 1e-13)
        f_prev = f


# ---------------------------------------------------------------- P7 KKT
def test_kkt_hand_example():
    X = np.eye(2, dtype=np.float32)
    U = np.array([[1.0], [0.0]])
    V = np.array([[0.5], [0.0]])
    k = oracle.kkt(X, U, V)
    # grad_U = U V^T V - X V = [-0.25, 0]; grad_V = V U^T U - X^T U = [-0.5, 0]
    assert k["min_u"] == 0 and k["min_v"] == 0
    assert k["comp_max"] == 0.25 and k["comp_sum"] == 0.5
    assert k["delta_w"] == 0.0 and k["sigma_w"] == -0.5 and k["dual_viol"] == 0.5


def test_kkt_reached_at_convergence_c1():
    X = synth.x_full(synth.C1)
    U, V, _, f, st = oracle.enmf(X, 5, 3000)
    k = oracle.kkt(X, U, V)
    assert k["min_u"] >= 0 and k["min_v"] >= 0
    assert k["comp_sum"] / k["xnorm2"] < 1e-6
    assert k["dual_viol"] / k["rms_cross"] < 1e-6


# ---------------------------------------------------------------- P8 brute force exact NMF
def _brute_force_exact_nmf(X, r):
    """Enumerate r-subsets of X's columns as U (separable model), solve the NNLS for V by
    active-set enumeration; return every zero-residual factorisation."""
    m, n = X.shape
    sols = []
    for cols in itertools.combinations(range(n), r):
        U = X[:, cols].astype(np.float64)
        V = np.zeros((n, r))
        ok = True
        for j in range(n):
            best = None
            for act in itertools.product([0, 1], repeat=r):
                idx = [a for a in range(r) if act[a]]
                v = np.zeros(r)
                if idx:
                    sol, *_ = np.linalg.lstsq(U[:, idx], X[:, j].astype(np.float64), rcond=None)
                    if (sol < -1e-12).any():
                        continue
                    v[idx] = sol
                res = np.linalg.norm(X[:, j] - U @ v)
                if best is None or res < best[0]:
                    best = (res, v)
            V[j] = best[1]
            ok &= best[0] < 1e-9
        if ok:
            sols.append((U, V))
    return sols


def test_exact_recovery_tiny_separable():
    """Exact-NMF instance with identity blocks in U0 and V0 (unique up to permutation and
    scale): brute force finds it, and eNMF reaches it."""
    U0 = np.array([[1, 0], [0, 1], [1, 2], [2, 1], [3, 1], [1, 3], [2, 2], [0, 2]], float)
    V0 = np.array([[1, 0], [0, 1], [2, 1], [1, 1], [1, 3], [3, 2], [2, 3]], float)
    X = (U0 @ V0.T).astype(np.float32)
    sols = _brute_force_exact_nmf(X, 2)
    assert sols, "brute force found no exact factorisation"
    U, V, _, f, _ = oracle.enmf(X, 2, 2000)
    F0 = oracle.xnorm2(X)
    assert f[-1] <= 1e-12 * F0
    Ub = sols[0][0]
    cos = (U / np.linalg.norm(U, axis=0)).T @ (Ub / np.linalg.norm(Ub, axis=0))
    assert np.sort(cos.max(axis=1)).min() > 1 - 1e-6


# ---------------------------------------------------------------- P9 ascent-descent sandwich
def test_ascent_descent_sandwich_c1():
    """Ascent raises the error above the rotated SVD point, HALS descends
    (324); with reading R9 exactly L = 10 ascent sweeps; feasibility gap <= 12 % (Fig. 5)."""
    X, Us, Vs, _ = _rotated_c1()
    W = np.vstack([Us, Vs])
    R, _, _ = oracle.admm_rotate(W, T=100)
    U, V = Us @ R, Vs @ R
    f_rot = oracle.frob2_direct(X, U, V)
    st = oracle.SweepState(0, oracle.lift_constant(U), oracle.lift_constant(V), 0)
    stages, fs = [], []
    for _ in range(200):
        U, V, stage, _ = oracle.sweep(X, U, V, st)
        stages.append(stage)
        fs.append(oracle.frob2_direct(X, U, V))
    assert stages[:10] == [0] * 10 and all(s == 1 for s in stages[10:])
    f_feas = fs[9]
    assert f_feas >= f_rot and fs[-1] <= f_feas
    assert all(b <= a * (1 + 1e-13) for a, b in zip(fs[10:], fs[11:]))
    assert f_feas <= 1.12 * fs[-1]
