"""Pins of the RSR-ADMM oracle (oracle/rsr.py; App. A): every closed-form
update against a generic numerical minimisation of the subproblem it claims to solve, the
lambda root choice against a dense search, Procrustes against a planted rotation and random
orthogonal matrices, the exact invariant U V^T = U* V*^T, and the paper's qualitative claim
that on a small exact-NMF instance the general RSR form reaches (almost) exact nonnegative
factors where the single rotation of Alg. 1 stalls (Fig. ICML_ap_fig4)."""
import numpy as np
from scipy.optimize import minimize

import oracle
from oracle import rsr


def test_zprox_is_the_grid_minimiser():
    t = 0.7
    z = np.linspace(-10, 10, 200001)
    for b in (-5.0, -1.0 / t - 0.3, -1.0 / t + 0.2, -0.1, 0.0, 0.4, 3.0):
        h = np.maximum(0.0, -z) + 0.5 * t * (z - b) ** 2
        assert abs(rsr.zprox(np.array(b), t) - z[h.argmin()]) < 2e-4


def test_w1_and_w2_closed_forms_minimise_their_subproblems():
    """W11 / W12 and W21 / W22 are the exact minimisers
    of their quadratic pieces of f1 and f2, written out here from the cost functions of
    PAPER.md:889-899 and minimised by BFGS."""
    g = np.random.default_rng(0)
    k, r = 6, 3
    rho, gamma, t = 0.7, 1.3, 0.4
    lam = 0.5 + g.random(r)
    UR, M1, W21, N1 = (g.standard_normal((k, r)) for _ in range(4))
    W31, P1 = g.standard_normal((k, r)), g.standard_normal((k, r))
    R2 = np.linalg.qr(g.standard_normal((r, r)))[0]
    # W11: rho/2 ||W11 - U* R1 + M1||^2 + gamma/2 ||W21 - W11 Lambda + N1||^2
    f = lambda w: (0.5 * rho * np.sum((w.reshape(k, r) - UR + M1) ** 2) +
                   0.5 * gamma * np.sum((W21 - w.reshape(k, r) * lam + N1) ** 2))
    w_num = minimize(f, np.zeros(k * r), method="BFGS", options={"gtol": 1e-12}).x.reshape(k, r)
    w_cf = (rho * (UR - M1) + gamma * lam * (W21 + N1)) / (rho + gamma * lam ** 2)
    assert np.abs(w_num - w_cf).max() < 1e-6
    # W12 with Lambda^-1
    f = lambda w: (0.5 * rho * np.sum((w.reshape(k, r) - UR + M1) ** 2) +
                   0.5 * gamma * np.sum((W21 - w.reshape(k, r) / lam + N1) ** 2))
    w_num = minimize(f, np.zeros(k * r), method="BFGS", options={"gtol": 1e-12}).x.reshape(k, r)
    w_cf = (rho * (UR - M1) + (gamma / lam) * (W21 + N1)) / (rho + gamma / lam ** 2)
    assert np.abs(w_num - w_cf).max() < 1e-6
    # W21: gamma/2 ||W21 - W11 Lambda + N1||^2 + t/2 ||W31 - W21 R2 + P1||^2
    W11 = g.standard_normal((k, r))
    f = lambda w: (0.5 * gamma * np.sum((w.reshape(k, r) - W11 * lam + N1) ** 2) +
                   0.5 * t * np.sum((W31 - w.reshape(k, r) @ R2 + P1) ** 2))
    w_num = minimize(f, np.zeros(k * r), method="BFGS", options={"gtol": 1e-12}).x.reshape(k, r)
    w_cf = (gamma * W11 * lam - gamma * N1 + t * (W31 + P1) @ R2.T) / (gamma + t)
    assert np.abs(w_num - w_cf).max() < 1e-6


def test_lambda_update_is_the_global_minimiser():
    """The quartic's chosen root (reading R37) is the global minimiser of the lambda_i
    objective over (0, inf): dense log grid plus a local refinement."""
    g = np.random.default_rng(1)
    for trial in range(20):
        w11, w21, n1 = (g.standard_normal(7) for _ in range(3))
        w12, w22, n2 = (g.standard_normal(5) for _ in range(3))
        lam = rsr.lambda_update(w11, w21, n1, w12, w22, n2, 1.0, 1.0)
        grid = np.exp(np.linspace(np.log(1e-4), np.log(1e4), 200001))
        vals = np.array([rsr.lambda_objective(x, w11, w21, n1, w12, w22, n2, 1.0) for x in
                         grid[::50]])
        best = grid[::50][vals.argmin()]
        res = minimize(lambda x: rsr.lambda_objective(abs(x[0]), w11, w21, n1, w12, w22, n2, 1.0),
                       [best], method="Nelder-Mead", options={"xatol": 1e-13, "fatol": 1e-15})
        ref = abs(res.x[0])
        assert rsr.lambda_objective(lam, w11, w21, n1, w12, w22, n2, 1.0) <= \
            rsr.lambda_objective(ref, w11, w21, n1, w12, w22, n2, 1.0) + 1e-10
        assert abs(lam - ref) < 1e-5 * ref


def test_procrustes_planted_and_optimal():
    g = np.random.default_rng(2)
    A = g.standard_normal((30, 4))
    Q = np.linalg.qr(g.standard_normal((4, 4)))[0]
    assert np.abs(rsr.procrustes(A, A @ Q) - Q).max() < 1e-12
    B = g.standard_normal((30, 4))
    R = rsr.procrustes(A, B)
    assert np.abs(R.T @ R - np.eye(4)).max() < 1e-12
    best = np.linalg.norm(A @ R - B)
    for _ in range(2000):
        O = np.linalg.qr(g.standard_normal((4, 4)))[0]
        assert best <= np.linalg.norm(A @ O - B) + 1e-12


def exact_instance(seed=0, m=40, n=50, r=10):
    """Exact NMF X = W H^T with half of W's and H's entries zero (the App. A synthetic family,
    PAPER.md:836-840, at its small size)."""
    g = np.random.default_rng(seed)
    W = g.random((m, r)) * (g.random((m, r)) < 0.5)
    H = g.random((n, r)) * (g.random((n, r)) < 0.5)
    return (W @ H.T).astype(np.float32)


def test_rsr_preserves_the_product_and_orthogonality():
    X = exact_instance()
    Us, Vs, _, _ = oracle.truncated_svd(X, 10)
    R1, R2, lam, U, V = rsr.rsr_admm(Us, Vs, 50)
    assert np.abs(R1.T @ R1 - np.eye(10)).max() < 1e-12
    assert np.abs(R2.T @ R2 - np.eye(10)).max() < 1e-12
    assert np.all(lam > 0)
    assert np.abs(U @ V.T - Us @ Vs.T).max() < 1e-12 * np.abs(Us @ Vs.T).max()
    assert np.allclose(U, (Us @ R1) * lam @ R2) and np.allclose(V, (Vs @ R1) / lam @ R2)


def test_rsr_reaches_the_orthant_where_alg1_stalls():
    """PAPER.md:836-842 and Fig. ICML_ap_fig4: on small exact instances the ADMM for Eq. eq5
    yields almost exact nonnegative factors, while the single rotation (Alg. 1, R1 = Lambda =
    I) stays away from the orthant."""
    X = exact_instance()
    Us, Vs, _, _ = oracle.truncated_svd(X, 10)
    neg0 = oracle.negativity(np.vstack([Us, Vs]))
    trace = []
    rsr.rsr_admm(Us, Vs, 2000, trace=trace)
    _, neg1, _ = oracle.admm_rotate(np.vstack([Us, Vs]), T=2000)
    print(f"negativity: SVD {neg0:.3f}, Alg. 1 {neg1[-1]:.3f}, RSR-ADMM {trace[-1]:.4f}")
    assert trace[-1] < 0.01 * neg0
    assert neg1[-1] > 0.1 * neg0
