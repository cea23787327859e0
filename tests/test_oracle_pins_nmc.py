"""Pins of the eNMC oracle (oracle_nmc.c; App. C) against what the
mathematics fixes: finite differences, special cases that reduce to the (pinned) eNMF oracle
or to a LAPACK routine, a brute-force line search, and exact recovery of a completable
low-rank matrix.  None compares the oracle with itself."""
import numpy as np

import oracle
import synth


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def planted(m, n, r, density, seed, noise=0.0):
    g = np.random.default_rng(seed)
    A, B = g.random((m, r)), g.random((n, r))
    X = A @ B.T + noise * np.abs(g.standard_normal((m, n)))
    mask = g.random((m, n)) < density
    return X.astype(np.float32), mask, g


def test_transposed_lists_match_column_enumeration():
    X, M, _ = planted(13, 9, 2, 0.4, 0)
    obs = oracle.Observed(X, M)
    for j in range(9):
        rows = np.nonzero(M[:, j])[0]
        lo, hi = obs.tptr[j], obs.tptr[j + 1]
        assert np.array_equal(obs.tidx[lo:hi], rows)
        assert np.array_equal(obs.tval[lo:hi], X[rows, j])


def test_masked_objective_full_mask_is_eq1():
    """With every entry observed f^ is Eq.(1)'s ||X - U V^T||^2 (the pinned eNMF oracle)."""
    X, _, g = planted(40, 30, 3, 1.0, 1, noise=0.1)
    U, V = g.standard_normal((40, 3)), g.standard_normal((30, 3))
    obs = oracle.Observed(X, np.ones(X.shape, bool))
    assert rel(oracle.nmc_objective(obs, U, V), oracle.frob2_direct(X, U, V)) < 1e-13


def test_masked_objective_sums_only_observed_entries():
    """Changing an unobserved entry of X changes nothing; a missing row contributes 0."""
    X, M, g = planted(20, 15, 2, 0.5, 2)
    M[4] = False
    U, V = g.random((20, 2)), g.random((15, 2))
    f0 = oracle.nmc_objective(oracle.Observed(X, M), U, V)
    X2 = X.copy()
    X2[~M] = 1e6
    assert oracle.nmc_objective(oracle.Observed(X2, M), U, V) == f0


def test_masked_gradient_against_finite_differences():
    """grad_U (1/2 f^) = (M_E o (U V^T - X)) V and grad_V likewise, checked
    by central differences of the objective, entry by entry."""
    X, M, g = planted(12, 10, 3, 0.5, 3, noise=0.05)
    obs = oracle.Observed(X, M)
    U, V = g.standard_normal((12, 3)), g.standard_normal((10, 3))
    GU, GV = oracle.nmc_grad(obs, U, V, "U"), oracle.nmc_grad(obs, U, V, "V")
    h = 1e-6
    for F, G, which in ((U, GU, 0), (V, GV, 1)):
        for idx in np.ndindex(F.shape):
            Fp, Fm = F.copy(), F.copy()
            Fp[idx] += h
            Fm[idx] -= h
            args_p = (Fp, V) if which == 0 else (U, Fp)
            args_m = (Fm, V) if which == 0 else (U, Fm)
            fd = (oracle.nmc_objective(obs, *args_p) - oracle.nmc_objective(obs, *args_m)) / (4 * h)
            assert abs(fd - G[idx]) < 1e-6 * max(1.0, abs(G[idx]))


def test_masked_gradient_full_mask_is_u_gv_minus_xv():
    X, _, g = planted(25, 18, 4, 1.0, 4, noise=0.1)
    U, V = g.standard_normal((25, 4)), g.standard_normal((18, 4))
    obs = oracle.Observed(X, np.ones(X.shape, bool))
    ref = U @ oracle.gram(V) - oracle.xv(X, V)
    assert np.abs(oracle.nmc_grad(obs, U, V) - ref).max() < 1e-11 * np.abs(ref).max()


def test_masked_pbcd_step_is_exact_line_minimiser():
    """Reading R30: one inner iteration moves every row to the minimiser of f^ along its
    masked gradient (before the projection): with all entries free and a start far from the
    orthant's boundary, the row after one iteration equals u_i - d* grad_i with d* from a
    golden-section search of the row's observed residual."""
    X, M, g = planted(6, 40, 3, 0.5, 5, noise=0.1)
    obs = oracle.Observed(X, M)
    U = 5.0 + g.random((6, 3))
    V = g.random((40, 3))
    free = np.ones(U.shape, np.uint8)
    U1, it, _, _ = oracle.nmc_pbcd(obs, U, V, free, "U", eps=0.0, max_iter=1)
    assert it == 1
    G = oracle.nmc_grad(obs, U, V)
    for i in range(6):
        obs_j = np.nonzero(M[i])[0]

        def phi(d):
            u = U[i] - d * G[i]
            return float(((X[i, obs_j].astype(np.float64) - V[obs_j] @ u) ** 2).sum())

        a, b = 0.0, 10.0
        gr = (np.sqrt(5) - 1) / 2
        for _ in range(200):
            c, d_ = b - gr * (b - a), a + gr * (b - a)
            if phi(c) < phi(d_):
                b = d_
            else:
                a = c
        dstar = 0.5 * (a + b)
        assert np.allclose(U1[i], np.maximum(0.0, U[i] - dstar * G[i]), rtol=1e-7, atol=1e-10)


def test_masked_pbcd_full_mask_is_alg2():
    """With every entry observed the eNMC PBCD is Alg. 2 of eNMF (the pinned or_pbcd): same
    iterate and the same stopping index."""
    X, _, g = planted(30, 25, 3, 1.0, 6, noise=0.1)
    obs = oracle.Observed(X, np.ones(X.shape, bool))
    U = g.standard_normal((30, 3))
    V = g.random((25, 3))
    U = oracle.lift(U, 0.5 * abs(U.min()))
    M = (U >= 0).astype(np.uint8)
    U_nmc, it_nmc, _, _ = oracle.nmc_pbcd(obs, U, V, M, "U")
    U_nmf, it_nmf, _, _ = oracle.pbcd(U, oracle.xv(X, V), oracle.gram(V), M)
    assert it_nmc == it_nmf
    assert np.abs(U_nmc - U_nmf).max() < 1e-10 * np.abs(U_nmf).max()


def test_masked_sweep_full_mask_is_enmf_ascent_sweep():
    """One eNMC sweep with every entry observed equals one eNMF ascent sweep (or_sweep,
    stage 0) from the same point with the same lift constants.  max_iter = 3: over longer
    runs Alg. 2 amplifies rounding ~15x per inner iteration in its unstable rows (DESIGN.md
    R33), and the two formulations of the same gradient (observed-entry sums vs U G - X V)
    round differently; after 3 iterations they agree to 1e-10."""
    cfg = synth.C1
    X = synth.x_full(cfg)
    obs = oracle.Observed(X, np.ones(X.shape, bool))
    Us, Vs, _, _ = oracle.truncated_svd(X, cfg.r)
    lu, lv = oracle.lift_constant(Us), oracle.lift_constant(Vs)
    Un, Vn, its = oracle.nmc_sweep(obs, Us, Vs, lu, lv, max_iter=3, round_f32=0)
    Ue, Ve, st, ite = oracle.sweep(X, Us, Vs, oracle.SweepState(0, lu, lv, 0),
                                   oracle.options(cfg.r, pbcd_max_iter=3))
    assert st == 0 and its == ite
    assert np.abs(Un - Ue).max() < 1e-10 * np.abs(Ue).max()
    assert np.abs(Vn - Ve).max() < 1e-10 * np.abs(Ve).max()


def test_softimpute_full_mask_is_eckart_young():
    """With every entry observed softImpute-ALS (lambda = 0) is block power iteration on X:
    A B^T converges to the rank-r truncated SVD (LAPACK), d^2 to its singular values."""
    X, _, g = planted(40, 30, 3, 1.0, 7, noise=0.05)
    obs = oracle.Observed(X, np.ones(X.shape, bool))
    A, B, d = oracle.softimpute(obs, g.standard_normal((40, 3)), 300)
    u, s, vt = np.linalg.svd(X.astype(np.float64))
    best = (u[:, :3] * s[:3]) @ vt[:3]
    assert np.abs(A @ B.T - best).max() < 1e-9 * np.abs(best).max()
    assert np.allclose(d ** 2, s[:3], rtol=1e-10)
    # balanced output, sign rule R5 on A
    assert np.allclose(np.linalg.norm(A, axis=0), np.linalg.norm(B, axis=0), rtol=1e-10)
    assert np.all(A[np.abs(A).argmax(0), np.arange(3)] > 0)


def test_softimpute_completes_a_low_rank_matrix():
    """An exactly rank-3 X observed on 60 % of its entries: the completion A B^T equals X on
    the MISSING entries too (matrix completion; the masked objective's global minimum 0)."""
    X, M, g = planted(40, 30, 3, 0.6, 8)
    obs = oracle.Observed(X, M)
    A, B, _ = oracle.softimpute(obs, g.standard_normal((40, 3)), 400)
    err = np.abs(A @ B.T - X.astype(np.float64))
    assert err[~M].max() < 1e-5 * np.abs(X).max()
    assert oracle.nmc_objective(obs, A, B) < 1e-12 * float((X[M].astype(np.float64) ** 2).sum())


def test_softimpute_objective_monotone():
    """softImpute-ALS with lambda = 0 is an EM / majorise-minimise iteration: f^ of the model
    A B^T never increases from one iteration to the next (Hastie et al. 2015, Sec. 4)."""
    X, M, g = planted(30, 25, 4, 0.5, 9, noise=0.2)
    obs = oracle.Observed(X, M)
    U0 = g.standard_normal((30, 4))
    f = [oracle.nmc_objective(obs, *oracle.softimpute(obs, U0, t)[:2]) for t in range(1, 12)]
    assert all(b <= a * (1 + 1e-12) for a, b in zip(f, f[1:])), f
