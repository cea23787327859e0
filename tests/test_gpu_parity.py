"""GPU path (libenmf.so through the C-ABI) vs the fp64 oracle on the same seeded inputs.

Tolerances are BASELINE.json:5's: one update from identical (U, V) <= 1e-5 relative Frobenius
per factor; objective trajectory over the first 50 sweeps <= 1e-4 relative; final objective
<= 1e-3; factors after permutation matching.

Every test here holds those numbers directly.  The exterior stages (ADMM rotation, lift +
PBCD ascent) take discrete decisions (k*, masks, stage switch) that a rounding-level difference
can flip; their parity is checked in the well-posed form of tests/test_gpu_shadow.py (the
oracle repeats each GPU sweep from the GPU's own state with the GPU's k*; the rotation step by
step).  The tests below that run an ascent sweep use that form too.
"""
import itertools

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import (iterate_direct, make, rel_fro, rotated_point, to_dev, to_np,
                               trace_bar_applies)

pytestmark = pytest.mark.gpu

FP64, TC = 1, 2

# small parity shapes spanning several tiles, CPL boundaries and ragged tails
CASES = [
    synth.C1,
    synth.C2.scaled(150, 700, 49, 49),
    synth.C3.scaled(160, 900, 32, 32),
    synth.C4.scaled(300, 250, 20, 0),
    synth.C1.scaled(257, 131, 33, 33, name="planted-ragged-r33"),
    synth.C1.scaled(130, 97, 1, 1, name="planted-r1"),
    synth.C5.scaled(400, 300, 128, 128, name="C5-shape-r128"),
]
IDS = [c.name for c in CASES]
TC_CASES = [CASES[0], CASES[4], CASES[6], synth.C5.scaled(700, 650, 128, 128, name="C5-700x650")]
TC_IDS = [c.name for c in TC_CASES]


def F32STATE(r):
    """Oracle options with the factor state stored in fp32 at block boundaries, as the C-ABI
    stores U and V (reading R26)."""
    return oracle.options(r, round_f32=1)


def oracle_sweeps(X, U, V, st, n, r):
    f = []
    for _ in range(n):
        U, V, _, _ = oracle.sweep(X, U, V, st, F32STATE(r))
        f.append(oracle.frob2_direct(X, U, V))
    return U, V, np.array(f)


# ----------------------------------------------------------------------------- HALS stage
@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_one_hals_sweep(cfg, prec):
    h, X, _ = make(cfg, precision=prec)
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U0, V0 = np.abs(U0), np.abs(V0)           # a feasible point: HALS stage
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    f, info = h.iterate(U, V, 1)
    Uo, Vo, stage, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1), F32STATE(cfg.r))
    assert info["hals_sweeps"] == 1 and stage == 1
    eu, ev = rel_fro(to_np(U), Uo), rel_fro(to_np(V), Vo)
    print(f"{cfg.name} prec={h.precision}: U {eu:.2e} V {ev:.2e}")
    assert eu < 1e-5 and ev < 1e-5


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [CASES[1], CASES[6]], ids=[IDS[1], IDS[6]])
def test_hals_sweep_rows_outgrowing_digit_scale(cfg, prec):
    """Every third row of U scaled by 1e-6: the sweep grows it by ~1e6, past the digit scale
    tc_hals_kernel chose from the old row (|u| su >= 64 after the first 32-column block), so
    those rows finish with the kernel's sequential fp64 fallback.  Same bar as one sweep."""
    h, X, _ = make(cfg, precision=prec)
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U0, V0 = np.abs(U0), np.abs(V0)
    U0[::3] *= np.float32(1e-6)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    _, info = h.iterate(U, V, 1)
    if prec == TC:   # the fallback really ran
        assert info["hals_fallback_rows"] > 0, info
    else:
        assert info["hals_fallback_rows"] == 0
    Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1), F32STATE(cfg.r))
    eu, ev = rel_fro(to_np(U), Uo), rel_fro(to_np(V), Vo)
    eu3 = rel_fro(to_np(U)[::3], Uo[::3])
    print(f"{cfg.name} prec={h.precision}: U {eu:.2e} (scaled rows {eu3:.2e}) V {ev:.2e} "
          f"fallback rows {info['hals_fallback_rows']}")
    assert eu < 1e-5 and ev < 1e-5 and eu3 < 1e-5


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
def test_hals_keeps_tiny_positive_entries(prec):
    """The HALS projection is max(0, .): legitimately tiny positive entries
    survive.  Planted X = U0 V0^T (fp32) with a quarter of U0's entries at 2^-19 of their row's
    maximum, started at the planted point (a fixed point of the exact update): after one
    sweep every tiny entry is still positive and within 2^-21 of its row maximum of the
    oracle's value (the tensor-core path's operands carry ~2^-22 of their scale group's
    maximum; its HALS zero snap, reading R28, acts only below 2^-22 of the row maximum --
    the round-1 snap at 2^-18 zeroed these entries), and the factors match at 1e-5."""
    g = np.random.default_rng(5)
    m, n, r = 300, 260, 16
    U0 = 0.5 + g.random((m, r))
    V0 = 0.5 + g.random((n, r))
    tiny = g.random((m, r)) < 0.25
    U0[tiny] *= 2.0 ** -19
    U0 = U0.astype(np.float32).astype(np.float64)
    V0 = V0.astype(np.float32).astype(np.float64)
    X = (U0 @ V0.T).astype(np.float32)
    h, _, _ = make(X.astype(np.float64), r, precision=prec)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    h.iterate(U, V, 1)
    Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1), F32STATE(r))
    Ug, Vg = to_np(U), to_np(V)
    rowmax = np.abs(Uo).max(axis=1, keepdims=True) * np.ones((1, r))
    dev = np.abs(Ug - Uo)[tiny] / rowmax[tiny]
    print(f"prec={h.precision}: {tiny.sum()} tiny entries, min gpu {Ug[tiny].min():.3e}, max "
          f"deviation {dev.max():.2e} of the row max; U {rel_fro(Ug, Uo):.2e} V {rel_fro(Vg, Vo):.2e}")
    assert np.all(Ug[tiny] > 0)
    assert dev.max() < 2.0 ** -21
    assert rel_fro(Ug, Uo) < 1e-5 and rel_fro(Vg, Vo) < 1e-5


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [CASES[0], CASES[4], CASES[6]], ids=[IDS[0], IDS[4], IDS[6]])
def test_projection_then_hals(cfg, prec):
    """Post-rotation variant (ii) of the ablation: enmf_project on the
    rotated (infeasible) point, then HALS sweeps, against oracle.project + oracle HALS sweeps.
    The projection is exact (bitwise); the sweeps are held to the HALS bars (one sweep 1e-5,
    10-sweep f trajectory 1e-4)."""
    h, X, _ = make(cfg, precision=prec)
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U, V = to_dev(U0), to_dev(V0)
    h.project(U, V)
    Up, Vp = oracle.project(U0), oracle.project(V0)
    assert np.array_equal(to_np(U), Up.astype(np.float32)) and \
        np.array_equal(to_np(V), Vp.astype(np.float32))
    assert h.get_stage()[0] == 1
    f_tr, f_gpu, info, asc = iterate_direct(h, U, V, 10)
    assert info["hals_sweeps"] == 1 and asc == 0
    U1, V1, _, _ = oracle.sweep(X, Up, Vp, oracle.SweepState(stage=1), F32STATE(cfg.r))
    Uo, Vo, f_or = oracle_sweeps(X, Up, Vp, oracle.SweepState(stage=1), 10, cfg.r)
    err = np.abs(f_gpu - f_or) / f_or
    etr = np.abs(f_tr - f_gpu) / f_gpu
    print(f"{cfg.name} prec={h.precision}: projection + 10 HALS sweeps, max direct f err "
          f"{err.max():.2e}, trace vs direct {etr.max():.2e}")
    assert np.all(err < 1e-4), err
    if trace_bar_applies(prec == TC, X, f_or):
        assert np.all(etr < 1e-4), etr
    # one sweep from the projected point: BASELINE's per-update bar
    h2, _, _ = make(cfg, precision=prec)
    U, V = to_dev(U0), to_dev(V0)
    h2.project(U, V)
    h2.iterate(U, V, 1)
    assert rel_fro(to_np(U), U1) < 1e-5 and rel_fro(to_np(V), V1) < 1e-5


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [CASES[0], CASES[4], CASES[6]], ids=[IDS[0], IDS[4], IDS[6]])
def test_ablation_gradient_descent(cfg, prec):
    """Descent-stage variant 'standard gradient descent' of the ablation (options.descent = 1,
    PAPER.md:2096-2099, reading R29): projected-gradient sweeps with step 1/lambda_max(G)
    from a shared feasible point -- one sweep within 1e-5 of the oracle, 10-sweep f trajectory
    at the HALS-stage bars."""
    h, X, _ = make(cfg, precision=prec, descent=1)
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U0, V0 = np.abs(U0), np.abs(V0)
    opts = oracle.options(cfg.r, round_f32=1, descent=1)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    h.iterate(U, V, 1)
    Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1), opts)
    eu, ev = rel_fro(to_np(U), Uo), rel_fro(to_np(V), Vo)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    f_tr, f_gpu, info, _ = iterate_direct(h, U, V, 10)
    st = oracle.SweepState(stage=1)
    Ua, Va, f_or = U0, V0, []
    for _ in range(10):
        Ua, Va, _, _ = oracle.sweep(X, Ua, Va, st, opts)
        f_or.append(oracle.frob2_direct(X, Ua, Va))
    f_or = np.array(f_or)
    err = np.abs(f_gpu - f_or) / f_or
    etr = np.abs(f_tr - f_gpu) / f_gpu
    print(f"{cfg.name} prec={h.precision}: PGD sweep U {eu:.2e} V {ev:.2e}, 10-sweep direct f "
          f"err {err.max():.2e}, trace vs direct {etr.max():.2e}")
    assert eu < 1e-5 and ev < 1e-5
    assert info["hals_sweeps"] == 1 and np.all(err < 1e-4)
    if trace_bar_applies(prec == TC, X, f_or):
        assert np.all(etr < 1e-4), etr
    # the same variant switched on a handle created with the defaults (enmf_set_ablation)
    h2, _, _ = make(cfg, precision=prec)
    h2.set_ablation(0, 1)
    U, V = to_dev(U0), to_dev(V0)
    h2.set_stage(1)
    f2, _ = h2.iterate(U, V, 10)
    assert np.array_equal(f2, f_tr)


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [CASES[1], CASES[6]], ids=[IDS[1], IDS[6]])
def test_ablation_fixed_step_ascent(cfg, prec):
    """Feasibility-stage variant 'fixed step size' (options.step_rule = 1, PAPER.md:2160-2165,
    reading R29): one lift + PBCD sweep with the step 1/lambda_max(G) for every row from an
    infeasible start, repeated by the oracle in the well-posed form of test_gpu_shadow.py
    (U block from the shared start, V block from the GPU's U_new, the GPU's k* inner
    iterations): 1e-5 per factor away from 0 (R20), no mask flips."""
    from tests.test_gpu_shadow import f32, r20, start_point
    h, X, _ = make(cfg, precision=prec, step_rule=1)
    U0, V0, lu, lv = start_point(X, cfg.r, want_infeasible=True)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(0, lu, lv)
    _, info = h.iterate(U, V, 1)
    assert info["ascent_sweeps"] == 1
    Un, Vn = to_np(U), to_np(V)
    out = []
    for F, other, up, lam, k in ((U0, V0, True, lu, info["pbcd_iters_u"]),
                                 (V0, Un, False, lv, info["pbcd_iters_v"])):
        C = oracle.xv(X, other) if up else oracle.xtu(X, other)
        G = oracle.gram(other)
        Fl = oracle.lift(F, lam)
        M = Fl >= 0
        step = 1.0 / oracle.lambda_max(G)
        _, own, _, _ = oracle.pbcd_step(Fl, C, G, M, step, 1e-2, 50)
        Fo, _, _, _ = oracle.pbcd_step(Fl, C, G, M, step, 0.0, k)
        out.append((f32(Fo), own, k))
    (eu, fu), (ev, fv) = r20(Un, out[0][0]), r20(Vn, out[1][0])
    print(f"{cfg.name} prec={h.precision}: fixed-step ascent U {eu:.2e} V {ev:.2e}, flips "
          f"{fu}/{fv}, k* gpu {out[0][2]}/{out[1][2]} oracle rule {out[0][1]}/{out[1][1]}")
    assert eu < 1e-5 and ev < 1e-5 and fu + fv == 0


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", CASES[:4] + [CASES[6]], ids=IDS[:4] + [IDS[6]])
def test_hals_trajectory_50_sweeps(cfg, prec):
    """50 HALS sweeps from a shared feasible point, both sides along their own trajectories
    (the HALS stage has no discrete decisions): final factors within 1e-4 and the direct
    objective (enmf_objective(exact=1)) within 1e-4 at every sweep; the trace-form f that
    enmf_iterate reports within 1e-4 of the direct one where gpu_common.trace_bar_applies."""
    h, X, _ = make(cfg, precision=prec)
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U0, V0 = np.abs(U0), np.abs(V0)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    f_tr, f_gpu, info, _ = iterate_direct(h, U, V, 50)
    Uo, Vo, f_or = oracle_sweeps(X, U0, V0, oracle.SweepState(stage=1), 50, cfg.r)
    err = np.abs(f_gpu - f_or) / f_or
    etr = np.abs(f_tr - f_gpu) / f_gpu
    cond = oracle.xnorm2(X) / f_or
    print(f"{cfg.name} prec={h.precision}: max direct f err {err.max():.2e}, trace vs direct "
          f"{etr.max():.2e} (max ||X||^2/f {cond.max():.1e})")
    assert np.all(err < 1e-4), err
    if trace_bar_applies(prec == TC, X, f_or):
        assert np.all(etr < 1e-4), etr
    assert abs(h.objective(U, V, exact=True) - f_or[-1]) / f_or[-1] < 1e-4
    assert rel_fro(to_np(U), Uo) < 1e-4 and rel_fro(to_np(V), Vo) < 1e-4


# ----------------------------------------------------------------------------- init
@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [synth.C1, synth.C3.scaled(160, 900, 32, 32),
                                 synth.C5.scaled(600, 500, 16, 16, name="C5-shape-r16"),
                                 synth.C5.scaled(700, 650, 128, 128, name="C5-shape-r128")],
                         ids=["C1", "C3-scaled", "C5-shape-r16", "C5-shape-r128"])
def test_randomised_svd_matches_converged_svd(cfg, prec):
    """Randomised range finder (q = 2) vs the oracle's converged subspace iteration on gapped
    spectra: singular values and balanced factors U* = U S^1/2, V* = V S^1/2.  prec=tc runs the
    2q + 2 X passes as tensor-core column-block products (tc_xf; l = 138 > 128 at r = 128 takes
    two blocks)."""
    X = synth.x_full(cfg)
    import paper_2605_19325_b200 as E
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=prec)
    h.set_data(to_dev(X))
    U = to_dev(np.zeros((cfg.m, cfg.r)))
    V = to_dev(np.zeros((cfg.n, cfg.r)))
    sig = h.svd(U, V)
    Us, Vs, s, _ = oracle.truncated_svd(X, cfg.r)
    assert np.allclose(sig, s, rtol=1e-6)
    assert rel_fro(to_np(U), Us) < 1e-5 and rel_fro(to_np(V), Vs) < 1e-5


@pytest.mark.parametrize("cfg", CASES[:3], ids=IDS[:3])
def test_rotation_from_shared_point(cfg):
    """Alg. 1 (T_admm = 100, reading R8) from the same fp32 [U*; V*]: the invariants -- R
    orthogonal, f unchanged (level set), no third-branch Z entries (R7) -- and
    the negativity reached, printed beside the oracle's.  After ~100 steps the iteration's
    sensitivity to rounding makes factor parity ill posed (the oracle moves by O(1) under a
    1e-7 perturbation of its input on C2/C3, R26); the step-by-step parity of the
    same iteration is test_gpu_shadow.test_admm_stepwise_from_shared_point."""
    X = synth.x_full(cfg)
    Us, Vs, _, _ = oracle.truncated_svd(X, cfg.r)
    U0 = Us.astype(np.float32).astype(np.float64)
    V0 = Vs.astype(np.float32).astype(np.float64)
    h, _, _ = make(X, cfg.r)
    U, V = to_dev(U0), to_dev(V0)
    info = h.rotate(U, V)

    R, neg, _ = oracle.admm_rotate(np.vstack([U0, V0]), T=100)
    Ug, Vg = to_np(U), to_np(V)
    f0 = oracle.frob2_direct(X, U0, V0)
    assert info["admm_third_branch"] == 0 and info["orth_residual"] < 1e-12
    assert abs(oracle.frob2_direct(X, Ug, Vg) - f0) / f0 < 1e-5
    neg0 = oracle.negativity(np.vstack([U0, V0]))
    neg_gpu = oracle.negativity(np.vstack([Ug, Vg]))
    print(f"{cfg.name}: negativity [U*;V*] {neg0:.4g} -> gpu {neg_gpu:.4g}, oracle {neg[-1]:.4g}; "
          f"U vs oracle {rel_fro(Ug, U0 @ R):.2e}")
    assert neg_gpu < neg0


# ----------------------------------------------------------------------------- objective, KKT
@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", CASES[:3] + [CASES[6]], ids=IDS[:3] + [IDS[6]])
def test_objective_and_kkt(cfg, prec):
    h, X, _ = make(cfg, precision=prec)
    g = np.random.default_rng(0)
    U0 = g.random((cfg.m, cfg.r)).astype(np.float32).astype(np.float64)
    V0 = g.random((cfg.n, cfg.r)).astype(np.float32).astype(np.float64)
    U, V = to_dev(U0), to_dev(V0)
    f_d = oracle.frob2_direct(X, U0, V0)
    assert abs(h.objective(U, V, exact=True) - f_d) / f_d < 1e-12
    # trace form: fp64 path -- conditioning ||X||^2 / f times the contraction's relative
    # accuracy; tensor-core path -- the trace form of the quantised operands: first-order
    # error 2 <E, X - U V^T> with |E| <= 2^-22 of the scale groups' maxima (<~ 2^-21 f), plus
    # the dropped digit products' noise (~1e-10 ||X||^2 at these K)
    f_t = h.objective(U, V, exact=False)
    if prec == FP64:
        assert abs(f_t - f_d) / f_d < 1e-15 * oracle.xnorm2(X) / f_d + 1e-12
    else:
        assert abs(f_t - f_d) < 1e-6 * f_d + 1e-10 * oracle.xnorm2(X)
    k = h.kkt(U, V)
    ko = oracle.kkt(X, U0, V0)
    rtol = 1e-9 if prec == FP64 else 1e-5
    for key in ("min_u", "min_v", "comp_max", "comp_sum", "delta_w", "sigma_w", "dual_viol",
                "xnorm2", "rms_cross"):
        assert abs(k[key] - ko[key]) <= rtol * max(abs(ko[key]), 1e-300) + 1e-12 * ko["xnorm2"], key


@pytest.mark.parametrize("pair", ["0", "1"], ids=["cta1", "cta2"])
@pytest.mark.parametrize("signed", [False, True], ids=["nonneg", "signed"])
@pytest.mark.parametrize("cfg", TC_CASES, ids=TC_IDS)
def test_tc_contractions_match_oracle(cfg, signed, pair, monkeypatch):
    """The tensor-core X passes (3 base-2^8 int8 digit planes, exact int32 TMEM accumulation)
    element by element against the oracle's fp64 X V and X^T U.  Error budget: operands
    rounded to 2^-16 of a scale group maximum in [63, 126) (<= 2^-23 relative to that maximum),
    dropped products of weight <= 2^-24 (unbiased), so |err| <= ~5e-7 |X||V| entrywise and the
    normwise error is ~1e-8.  pair=1 runs the cta_group::2 kernel (ENMF_TC_PAIR, read when X is
    bound); the shapes include odd 128-row tile counts, whose missing pair partner is not
    stored."""
    monkeypatch.setenv("ENMF_TC_PAIR", pair)
    h, X, _ = make(cfg, precision=TC)
    assert h.precision.startswith("tc")
    g = np.random.default_rng(3)
    U0 = g.random((cfg.m, cfg.r))
    V0 = g.random((cfg.n, cfg.r))
    if signed:
        U0, V0 = U0 - 0.4, V0 - 0.4
    U0 = U0.astype(np.float32).astype(np.float64)
    V0 = V0.astype(np.float32).astype(np.float64)
    P, Q = h.cross_terms(to_dev(U0), to_dev(V0))
    P, Q = to_np(P), to_np(Q)
    Xa = np.abs(X.astype(np.float64))
    Pr, Qr = oracle.xv(X, V0), oracle.xtu(X, U0)
    ep = np.abs(P - Pr) / (Xa @ np.abs(V0))
    eq = np.abs(Q - Qr) / (Xa.T @ np.abs(U0))
    print(f"{cfg.name} {'signed' if signed else 'nonneg'}: P normwise {rel_fro(P, Pr):.2e} "
          f"max {ep.max():.2e}; Q normwise {rel_fro(Q, Qr):.2e} max {eq.max():.2e}")
    assert ep.max() < 2e-6 and eq.max() < 2e-6
    if not signed:
        assert rel_fro(P, Pr) < 1e-7 and rel_fro(Q, Qr) < 1e-7
    # the trace-form objective of the quantised operands (tc_gemm.cu): first-order error
    # 2 <E, X - U V^T> with |E| <= 2^-22 of the scale groups' maxima, plus the dropped
    # products' noise -- the bound test_objective_and_kkt states
    f_d = oracle.frob2_direct(X, U0, V0)
    f_t = h.objective(to_dev(U0), to_dev(V0), exact=False)
    assert abs(f_t - f_d) < 1e-6 * f_d + 1e-10 * oracle.xnorm2(X)


# ----------------------------------------------------------------------------- edges
def test_edge_cases():
    import torch
    import paper_2605_19325_b200 as E
    with pytest.raises(E.EnmfError):
        E.Enmf(10, 5, 6)                            # r > min(m, n)
    with pytest.raises(E.EnmfError):
        E.Enmf(10, 5, 0)
    with pytest.raises(E.EnmfError):
        E.Enmf(300, 300, 129)                       # r > ENMF_MAX_RANK
    h = E.Enmf(8, 6, 2)
    X = torch.rand(8, 6, device="cuda")
    X[3, 2] = -1e-3
    with pytest.raises(E.EnmfError) as ei:
        h.set_data(X)
    assert ei.value.code == -3
    X[3, 2] = float("nan")
    with pytest.raises(E.EnmfError) as ei:
        h.set_data(X)
    assert ei.value.code == -5
    U = torch.zeros(8, 2, device="cuda")
    V = torch.zeros(6, 2, device="cuda")
    with pytest.raises(E.EnmfError) as ei:
        h.iterate(U, V, 1)                          # no data bound
    assert ei.value.code == -9
    with pytest.raises(E.EnmfError) as ei:
        h.init(torch.zeros(8, 6, device="cuda"), U, V)   # X = 0: rank 0
    assert ei.value.code == -4


def test_zero_sweeps_and_launch_count():
    h, X, _ = make(synth.C1)
    U0, V0, lu, lv = rotated_point(X, 5)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(0, lu, lv)
    n0 = h.launch_count
    f, info = h.iterate(U, V, 0)
    assert len(f) == 0 and np.array_equal(to_np(U), U0)
    h.iterate(U, V, 2)
    assert h.launch_count > n0


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
def test_rank_deficient_init_rotation(prec):
    """X of exact rank 2 (small integers: exact in fp32) with r = 4: the SVD zero-fills the two
    deficient columns, so the ADMM Procrustes matrix W^T B is singular -- the
    Newton polar iteration reports failure and the gated Jacobi-SVD path with basis completion
    computes R (kernels_small.cu).  R must stay orthogonal: the rotated U V^T equals the SVD
    point's, which reproduces X (f = ||X||^2 - sum sigma^2 = 0)."""
    import paper_2605_19325_b200 as E
    g = np.random.default_rng(11)
    m, n, r = 300, 220, 4
    A, B = g.integers(0, 8, (m, 2)), g.integers(0, 8, (n, 2))
    X = (A @ B.T).astype(np.float64)
    h = E.Enmf(m, n, r, precision=prec)
    U, V = to_dev(np.zeros((m, r))), to_dev(np.zeros((n, r)))
    info = h.init(to_dev(X), U, V)
    Ur, Vr = to_np(U), to_np(V)
    assert info["rank_deficient"] == 2
    assert np.all(np.isfinite(Ur)) and np.all(np.isfinite(Vr))
    err = rel_fro(Ur @ Vr.T, X)
    print(f"prec={h.precision}: |U V^T - X| / |X| = {err:.2e}")
    assert err < 1e-6


def test_iterate_host_matches_iterate():
    """enmf_iterate_host (factor state in pinned host memory, overlapped transfers) gives
    bit-identical factors and objective trace to enmf_iterate on device copies, through the
    ascent -> HALS transition, with one call per sweep and with one multi-sweep call."""
    import torch
    cfg = synth.C1
    h1, X, _ = make(cfg)
    h2, _, _ = make(cfg)
    U0, V0, lu, lv = rotated_point(X, cfg.r)
    Ud, Vd = to_dev(U0), to_dev(V0)
    Uh = torch.from_numpy(U0.astype(np.float32)).pin_memory()
    Vh = torch.from_numpy(V0.astype(np.float32)).pin_memory()
    h1.set_stage(0, lu, lv)
    h2.set_stage(0, lu, lv)
    f1, i1 = h1.iterate(Ud, Vd, 14)
    f2 = [h2.iterate_host(Uh, Vh, 1)[0][0] for _ in range(12)]
    f3, i3 = h2.iterate_host(Uh, Vh, 2)
    assert np.array_equal(np.array(f2 + list(f3)), f1)
    assert np.array_equal(Uh.numpy(), to_np(Ud).astype(np.float32))
    assert np.array_equal(Vh.numpy(), to_np(Vd).astype(np.float32))
    assert i1["ascent_sweeps"] == 10 and h2.get_stage()[0] == 1


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
def test_graph_replay_matches_eager(prec, monkeypatch):
    """Sweeps 1 .. n-1 of an enmf_iterate call are captured once as a CUDA graph and replayed
    (enmf_capi.cu replay_sweeps): bitwise the same factors, objective trace, stage counts and
    k* as the eager launch sequence (ENMF_GRAPH=0), through the ascent -> HALS transition."""
    cfg = CASES[1]
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("ENMF_GRAPH", mode)
        h, X, _ = make(cfg, precision=prec)
        U0, V0, lu, lv = rotated_point(X, cfg.r)
        U, V = to_dev(U0), to_dev(V0)
        h.set_stage(0, lu, lv)
        f, info = h.iterate(U, V, 14)
        out[mode] = (f, to_np(U), to_np(V), info["ascent_sweeps"], info["pbcd_iters_u"])
    a, b = out["0"], out["1"]
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert a[3:] == b[3:] and a[3] == 10


def test_solve_host_matches_device_calls():
    """enmf_solve_host (X, U, V in host memory: X staged through pinned buffers, init, sweeps,
    U and V copied back) gives exactly what enmf_init + enmf_iterate give on device copies."""
    import paper_2605_19325_b200 as E
    cfg = CASES[0]
    X = synth.x_full(cfg)
    h1 = E.Enmf(cfg.m, cfg.n, cfg.r)
    Uh, Vh, fh, info = h1.solve_host(X, 30)
    h2 = E.Enmf(cfg.m, cfg.n, cfg.r)
    U = to_dev(np.zeros((cfg.m, cfg.r)))
    V = to_dev(np.zeros((cfg.n, cfg.r)))
    h2.init(to_dev(X), U, V)
    fd, _ = h2.iterate(U, V, 30)
    assert np.array_equal(fh, fd)
    assert np.array_equal(Uh.astype(np.float64), to_np(U)) and np.array_equal(Vh.astype(np.float64), to_np(V))
