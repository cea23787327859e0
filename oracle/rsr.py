"""RSR-ADMM oracle: the rotation-scale-rotation ADMM of App. A (Alg. "ADMM
for (eq:admm_form_2)", label alg:rsr) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Plain numpy in fp64, written in the paper's order and notation; it shares nothing with the
CUDA path.  Problem (Eq. eq5): find orthogonal R1, R2 and a positive
diagonal Lambda such that U* R1 Lambda R2 >= 0 and V* R1 Lambda^-1 R2 >= 0, minimising the
negativity h.  The split: W1 = W_svd R1, W2 = [W11 Lambda; W12 Lambda^-1],
W3 = W2 R2, objective sum h(W3).

Readings: R1 orientation -- U* is the top (m x r) block of W_svd, V* the bottom
(n x r) block (the paper's sum limits i = 1..n / 1..m in Eq. eq5 are transposed); R34 --
rho = gamma = t = 1e-3 / max|W_svd| (the projection regime of reading R7: every negative b
lands in the middle branch of the W3 prox); R35 -- R1 = R2 = I, Lambda = I, W1 = W2 = W3 =
W_svd, M = N = P = 0; R36 -- a fixed number of iterations T, last iterate; R37 -- lambda_i is
the positive real root of the quartic with the smallest value of the
lambda_i objective; lambda_i is kept when ||W11(:,i)|| = 0 or
||W12(:,i)|| = 0 (the objective then has no minimiser in (0, inf)).
"""
import numpy as np


def zprox(b, t):
    """W3 update: argmin_z h(z) + t/2 (z - b)^2, h(q) = max(0, -q)."""
    return np.where(b > 0, b, np.where(b >= -1.0 / t, 0.0, b + 1.0 / t))


def procrustes(A, B):
    """argmin_{R^T R = I} ||A R - B||_F = C D^T from the SVD A^T B = C S D^T (Eqs.
    eq:updateR_1 / eq:updateR_2)."""
    C, _, Dt = np.linalg.svd(A.T @ B)
    return C @ Dt


def lambda_objective(lam, w11, w21, n1, w12, w22, n2, gamma):
    """The lambda_i subproblem."""
    return 0.5 * gamma * (np.sum((w21 - lam * w11 + n1) ** 2) +
                          np.sum((w22 - w12 / lam + n2) ** 2))


def lambda_update(w11, w21, n1, w12, w22, n2, gamma, lam_old):
    """Reading R37: roots of lambda^4 ||w11||^2 - lambda^3 (w21 + n1)^T w11
    + lambda (w22 + n2)^T w12 - ||w12||^2 = 0, the positive real one with
    the smallest subproblem value."""
    a = float(w11 @ w11)
    d = float(w12 @ w12)
    if a == 0.0 or d == 0.0:
        return lam_old
    b = float((w21 + n1) @ w11)
    c = float((w22 + n2) @ w12)
    roots = np.roots([a, -b, 0.0, c, -d])
    cand = [float(z.real) for z in roots if abs(z.imag) <= 1e-9 * abs(z) and z.real > 0]
    if not cand:
        return lam_old
    vals = [lambda_objective(x, w11, w21, n1, w12, w22, n2, gamma) for x in cand]
    return cand[int(np.argmin(vals))]


def rsr_admm(Us, Vs, T, rho=None, gamma=None, t=None, trace=None):
    """Alg. alg:rsr from W_svd = [U*; V*] for T iterations.  Returns
    (R1, R2, lam, U, V) with U = U* R1 Lambda R2, V = V* R1 Lambda^-1 R2 (Eq. gen_2, so that
    U V^T = U* V*^T).  trace (list, optional) receives the negativity of [U; V] per iteration."""
    Us = np.asarray(Us, np.float64)
    Vs = np.asarray(Vs, np.float64)
    m, r = Us.shape
    Ws = np.vstack([Us, Vs])
    scale = 1e-3 / max(np.abs(Ws).max(), 1e-300)
    rho = scale if rho is None else rho
    gamma = scale if gamma is None else gamma
    t = scale if t is None else t
    R1 = np.eye(r)
    R2 = np.eye(r)
    lam = np.ones(r)
    W1, W2, W3 = Ws.copy(), Ws.copy(), Ws.copy()
    M = np.zeros_like(Ws)
    N = np.zeros_like(Ws)
    P = np.zeros_like(Ws)
    for _ in range(T):
        # (W1, W3) <- argmin f1  (separable)
        W3 = zprox(W2 @ R2 - P, t)
        UR = Ws[:m] @ R1
        VR = Ws[m:] @ R1
        W11 = (rho * (UR - M[:m]) + gamma * lam * (W2[:m] + N[:m])) / (rho + gamma * lam ** 2)
        W12 = (rho * (VR - M[m:]) + (gamma / lam) * (W2[m:] + N[m:])) / (rho + gamma / lam ** 2)
        W1 = np.vstack([W11, W12])
        # (W2, R1) <- argmin f2
        R1n = procrustes(Ws, W1 + M)
        G = (W3 + P) @ R2.T
        W21 = (gamma * W11 * lam - gamma * N[:m] + t * G[:m]) / (gamma + t)
        W22 = (gamma * W12 / lam - gamma * N[m:] + t * G[m:]) / (gamma + t)
        W2 = np.vstack([W21, W22])
        R1 = R1n
        # (R2, Lambda) <- argmin f3
        R2 = procrustes(W2, W3 + P)
        lam = np.array([lambda_update(W11[:, i], W21[:, i], N[:m, i], W12[:, i], W22[:, i],
                                      N[m:, i], gamma, lam[i]) for i in range(r)])
        # multipliers
        M = M + W1 - Ws @ R1
        N = N + W2 - np.vstack([W11 * lam, W12 / lam])
        P = P + W3 - W2 @ R2
        if trace is not None:
            U = Us @ R1 * lam @ R2
            V = Vs @ R1 / lam @ R2
            trace.append(float(np.maximum(0.0, -np.vstack([U, V])).sum()))
    U = (Us @ R1) * lam @ R2
    V = (Vs @ R1) / lam @ R2
    return R1, R2, lam, U, V
