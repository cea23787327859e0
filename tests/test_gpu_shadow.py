"""Well-posed per-sweep parity of the GPU path against the fp64 oracle ("shadow" runs).

The exterior stages of eNMF take discrete decisions: the stage switch, the PBCD
stopping index k* of Alg. 2's global rule pg < eps pg0 and the mask M = [F >= 0]
(PAPER.md:217).  A tolerance on a multi-sweep comparison from a shared starting point would
have to absorb whatever a rounding-level difference does to those decisions.  These tests
instead compare what is well posed:

* every sweep is repeated by the oracle from the GPU's OWN state (U_t, V_t); the V block from
  the GPU's U_{t+1} (the V update uses U^(k+1));
* in the ascent stage the oracle runs the GPU's k* inner iterations (its own eps rule is
  evaluated too: a k* mismatch is accepted only where the stopping test sits within the
  arithmetic's precision of its threshold, and is counted and printed);
* factors are compared per entry away from 0: an entry at or below 1e-6 of the
  factor's maximum on exactly one side is a mask flip, counted and required to be
  <= 1e-6 rows r (i.e. none at these sizes); the rest at BASELINE.json:5's 1e-5 relative
  Frobenius per factor and update;
* in a PBCD block many rows are ILL-CONDITIONED: 50 inner iterations of Alg. 2 amplify an
  input perturbation by 1e3 .. 1e10 (measured in the oracle alone; the extreme rows are those
  where the Eq.(10) step, computed from the whole masked gradient including entries the
  projection holds at 0, exceeds 2 / G_kk on a free entry, so that entry oscillates with
  growing amplitude into a period-2 orbit; R33).  What such a row ends at is
  decided by rounding, not by the method.  Rows whose oracle output moves by more than 1e-6
  when the block's inputs (F, C, G) are perturbed at the path's arithmetic precision (1e-15
  on the fp64 path; 2^-22, the relative rounding of the tensor-core path's digit operands,
  on the tc path) are counted, printed and excluded, and every other row is held to 1e-5.
  The excluded fraction is computed from the oracle alone (it does not depend on the GPU's
  result), so a GPU error cannot hide in it; it grows through the ascent stage (fp64: 0-3 %
  in the first sweep, up to ~50 % of a block in later sweeps of the C5-shape case; tc: most
  rows of these small cases, since the X passes alone perturb C by ~1e-8);
* objective trajectories compare the DIRECT objective ||X - U V^T||^2 (enmf_objective(exact=1),
  oracle.frob2_direct) at 1e-4 per sweep, with the oracle replaying the GPU's discrete
  decisions along its own trajectory; the GPU's trace-form f (what enmf_iterate reports) is
  held to the direct objective of the same state at 1e-4 as well.

Both contraction paths run every case: fp64 (SIMT) and tc (tensor-core int8 digits).
"""
import itertools

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import make, rel_fro, rotated_point, to_dev, to_np, trace_bar_applies

pytestmark = pytest.mark.gpu

FP64, TC = 1, 2
PRECS = [FP64, TC]
PIDS = ["fp64", "tc"]
EPS, MAX_ITER = 1e-2, 50          # Alg. 2 defaults (reading R10)

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


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def r20(gpu, ora, rel_zero=1e-6):
    """(relative Frobenius error over the entries that are not mask flips, flips).
    A flip is an entry at or below rel_zero * max|ora| on exactly one side."""
    thr = rel_zero * max(float(np.abs(ora).max()), 1e-300)
    flip = (np.abs(gpu) <= thr) ^ (np.abs(ora) <= thr)
    d = np.where(flip, 0.0, gpu - ora)
    return float(np.linalg.norm(d) / max(np.linalg.norm(ora), 1e-300)), int(flip.sum())


DELTA = {FP64: 1e-15, TC: 2.0 ** -22}   # the paths' arithmetic precision (see above)


def oracle_block(X, F, other, upper, ascent, lam=0.0, kstar=None, delta=0.0):
    """One block update of the oracle (Alg. 3) from F with the other factor
    fixed: upper -> U block (C = X V, G = V^T V), else V block (C = X^T U, G = U^T U).
    HALS, or lift + mask + PBCD (Alg. 2) with `kstar` inner iterations (eps = 0 runs exactly
    that many; None: the eps rule).  Returns (F_new rounded to fp32 as the C-ABI stores it,
    reading R26; the oracle's own k*; pg after kstar / pg0; ill-conditioned rows (bool per
    row, PBCD with delta > 0 only: the row moved by > 1e-6 under two random relative
    perturbations of size delta of F, C and G, mask kept))."""
    C = oracle.xv(X, other) if upper else oracle.xtu(X, other)
    G = oracle.gram(other)
    if not ascent:
        return f32(oracle.hals(F, C, G)), 0, 0.0, None
    Fl = oracle.lift(F, lam)
    M = Fl >= 0
    _, own, _, _ = oracle.pbcd(Fl, C, G, M, EPS, MAX_ITER)
    k = own if kstar is None else kstar
    Fn, _, g0, g1 = oracle.pbcd(Fl, C, G, M, 0.0, k)
    ill = None
    if delta > 0:
        g = np.random.default_rng(99)
        spread = np.zeros(len(Fn))
        nrm = np.maximum(np.linalg.norm(Fn, axis=1), 1e-300)
        for _ in range(2):
            Fp = Fl * (1.0 + delta * g.standard_normal(Fl.shape))
            Cp = C * (1.0 + delta * g.standard_normal(C.shape))
            Gp = G * (1.0 + delta * g.standard_normal(G.shape))
            Fq, _, _, _ = oracle.pbcd(Fp, Cp, 0.5 * (Gp + Gp.T), M, 0.0, k)
            spread = np.maximum(spread, np.linalg.norm(Fq - Fn, axis=1) / nrm)
        ill = spread > 1e-6
    return f32(Fn), own, (g1 / g0 if g0 > 0 else 0.0), ill


def kstar_margin(X, F, other, upper, lam, k_gpu, k_own):
    """|pg(k)/pg0 - eps| / eps at the earlier of the two stopping indices: how close the
    oracle's own stopping test is to its threshold where the GPU decided differently."""
    _, _, ratio, _ = oracle_block(X, F, other, upper, True, lam, min(k_gpu, k_own))
    return abs(ratio - EPS) / EPS


def start_point(X, r, want_infeasible):
    """The oracle's rotated point (Alg. 3, fp32); where that is already feasible
    (the paper's one-shot case) and an ascent start is wanted, the un-rotated SVD point
    U* = U S^1/2, V* = V S^1/2 -- infeasible for every r > 1."""
    U0, V0, lu, lv = rotated_point(X, r)
    if want_infeasible and U0.min() >= 0 and V0.min() >= 0:
        Us, Vs, _, _ = oracle.truncated_svd(X, r)
        U0, V0 = f32(Us), f32(Vs)
        lu, lv = oracle.lift_constant(U0), oracle.lift_constant(V0)
    return U0, V0, lu, lv


class Shadow:
    """Accumulates the per-sweep comparison of one run."""

    def __init__(self, rows_u, rows_v, r):
        self.eu = self.ev = 0.0
        self.flips = 0
        self.ill = 0              # ill-posed PBCD rows excluded (all blocks)
        self.ill_frac = 0.0       # worst fraction of one block
        self.kmis = []            # (sweep, block, k_gpu, k_own, margin)
        self.hals_flips = 0
        self.limit_flips = 1e-6 * (rows_u + rows_v) * r

    def block(self, gpu, ora, ill=None, pbcd=True):
        if ill is not None and ill.all():        # nothing well conditioned to compare
            self.ill += int(ill.sum())
            self.ill_frac = 1.0
            return 0.0
        """PBCD blocks: R20 error over the well-conditioned rows, flips counted.  HALS blocks
        (well conditioned, no active-set dynamics): the plain relative Frobenius error over
        every entry -- a near-zero entry that differs only by sitting on the other side of
        the R20 threshold contributes its (tiny) difference; flips are counted, not limited."""
        if ill is not None and ill.any():
            self.ill += int(ill.sum())
            self.ill_frac = max(self.ill_frac, float(ill.mean()))
            gpu, ora = gpu[~ill], ora[~ill]
        e, fl = r20(gpu, ora)
        if pbcd:
            self.flips += fl
            return e
        self.hals_flips += fl
        return float(np.linalg.norm(gpu - ora) / max(np.linalg.norm(ora), 1e-300))


def shadow_sweep(sh, X, Ut, Vt, Un, Vn, info, lu, lv, prec, t):
    """Oracle repeat of one GPU sweep from the GPU's state (Ut, Vt) -> (Un, Vn)."""
    ascent = info["ascent_sweeps"] == 1
    # the stage decision of PAPER.md:334 from the sweep's entry state
    assert ascent == (Ut.min() < 0 or Vt.min() < 0), (t, ascent)
    ku = info["pbcd_iters_u"] if ascent else None
    kv = info["pbcd_iters_v"] if ascent else None
    Uo, own_u, _, illu = oracle_block(X, Ut, Vt, True, ascent, lu, ku, DELTA[prec])
    Vo, own_v, _, illv = oracle_block(X, Vt, Un, False, ascent, lv, kv, DELTA[prec])
    sh.eu = max(sh.eu, sh.block(Un, Uo, illu, ascent))
    sh.ev = max(sh.ev, sh.block(Vn, Vo, illv, ascent))
    if ascent:
        for blk, kg, ko, F, other, up, lam in (("U", ku, own_u, Ut, Vt, True, lu),
                                               ("V", kv, own_v, Vt, Un, False, lv)):
            if kg != ko:
                sh.kmis.append((t, blk, kg, ko, kstar_margin(X, F, other, up, lam, kg, ko)))
    return ascent


# ----------------------------------------------------------------------------- HALS stage
@pytest.mark.parametrize("prec", PRECS, ids=PIDS)
@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_shadow_hals_50_sweeps(cfg, prec):
    """50 HALS sweeps from a shared feasible point, every one repeated by the oracle from the
    GPU's own state: per-update parity 1e-5 (relative Frobenius); the trace-form f of every
    sweep within 1e-4 of the direct objective of the same state (where
    gpu_common.trace_bar_applies); the GPU's direct objective equal to the oracle's to
    1e-12."""
    h, X, _ = make(cfg, precision=prec)
    U0, V0, _, _ = rotated_point(X, cfg.r)
    Ut, Vt = np.abs(U0), np.abs(V0)
    U, V = to_dev(Ut), to_dev(Vt)
    h.set_stage(1)
    sh = Shadow(cfg.m, cfg.n, cfg.r)
    ftr = 0.0
    fds = []
    for t in range(50):
        f, info = h.iterate(U, V, 1)
        assert info["hals_sweeps"] == 1
        Un, Vn = to_np(U), to_np(V)
        shadow_sweep(sh, X, Ut, Vt, Un, Vn, info, 0.0, 0.0, prec, t)
        fd = oracle.frob2_direct(X, Un, Vn)
        fds.append(fd)
        ftr = max(ftr, abs(f[0] - fd) / fd)
        Ut, Vt = Un, Vn
    fx = h.objective(U, V, exact=True)
    print(f"{cfg.name} prec={h.precision}: 50 HALS sweeps, per-update U {sh.eu:.2e} "
          f"V {sh.ev:.2e}, R20 flips {sh.hals_flips}; trace f vs direct {ftr:.2e}; direct "
          f"{abs(fx - fd) / fd:.1e}")
    assert sh.eu < 1e-5 and sh.ev < 1e-5
    assert abs(fx - fd) / fd < 1e-12
    if trace_bar_applies(prec == TC, X, fds):
        assert ftr < 1e-4


# ----------------------------------------------------------------------------- ascent stage
@pytest.mark.parametrize("prec", PRECS, ids=PIDS)
@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_shadow_ascent_sweeps(cfg, prec):
    """The ascent stage (lift + mask + PBCD on both blocks, Alg. 2/3) sweep by sweep until the
    GPU reaches the orthant, plus 3 HALS sweeps, each repeated by the oracle from the GPU's
    state with the GPU's k*: per-update parity 1e-5 (R20) on the well-conditioned rows (see
    the module doc; their fraction is printed), no flips there, the stage decision
    identical, and every k* equal to the oracle's own eps rule -- or, where not, the
    oracle's stopping test within 1e-6 (fp64) / 1e-3 (tc) of its threshold."""
    h, X, _ = make(cfg, precision=prec)
    Ut, Vt, lu, lv = start_point(X, cfg.r, want_infeasible=True)
    if Ut.min() >= 0 and Vt.min() >= 0:
        pytest.skip("rank 1: the SVD point is already feasible")
    U, V = to_dev(Ut), to_dev(Vt)
    h.set_stage(0, lu, lv)
    sh = Shadow(cfg.m, cfg.n, cfg.r)
    n_asc = n_hals = 0
    for t in range(40):
        _, info = h.iterate(U, V, 1)
        Un, Vn = to_np(U), to_np(V)
        if shadow_sweep(sh, X, Ut, Vt, Un, Vn, info, lu, lv, prec, t):
            n_asc += 1
        else:
            n_hals += 1
        Ut, Vt = Un, Vn
        if n_hals == 3:
            break
    tol_margin = 1e-6 if prec == FP64 else 1e-3
    print(f"{cfg.name} prec={h.precision}: {n_asc} ascent + {n_hals} HALS sweeps, per-update "
          f"U {sh.eu:.2e} V {sh.ev:.2e}, flips {sh.flips}, ill-posed rows {sh.ill} (worst "
          f"block {100 * sh.ill_frac:.1f} %), k* mismatches {sh.kmis}")
    assert n_asc >= 1 and n_hals == 3
    assert sh.eu < 1e-5 and sh.ev < 1e-5
    assert sh.flips <= sh.limit_flips
    assert all(m[4] < tol_margin for m in sh.kmis), sh.kmis


@pytest.mark.parametrize("cfg", CASES[:5] + [CASES[6]], ids=IDS[:5] + [IDS[6]])
def test_shadow_tc_pbcd_one_iteration_all_rows(cfg):
    """The tensor-core PBCD kernel against Alg. 2 on EVERY row: with max_iter = 1 (eps = 0, so
    k* = 1) the inner iteration cannot amplify the X passes' ~6e-9 into the R33 orbits, so one
    lift + PBCD step per block -- the oracle from the GPU's own start state, on the exact X V
    and X^T U_new -- must agree per update at 1e-5 over all rows, for 3 ascent sweeps.  This
    separates the kernel's arithmetic (digit MMAs, byte digits, the Eq.(10) step, the
    projection) from the method's own ill-conditioning, which removes most rows of the
    tensor-core cases from test_shadow_ascent_sweeps at 50 iterations.  The rows that
    test_shadow_ascent_sweeps would exclude (perturbation 2^-22) are counted and printed."""
    h, X, _ = make(cfg, precision=TC, pbcd_max_iter=1, pbcd_eps=0.0)
    Ut, Vt, lu, lv = start_point(X, cfg.r, want_infeasible=True)
    U, V = to_dev(Ut), to_dev(Vt)
    h.set_stage(0, lu, lv)
    eu = ev = 0.0
    flips = ill = 0
    for t in range(3):
        _, info = h.iterate(U, V, 1)
        assert info["ascent_sweeps"] == 1
        assert info["pbcd_iters_u"] == 1 and info["pbcd_iters_v"] == 1
        Un, Vn = to_np(U), to_np(V)
        Uo, _, _, illu = oracle_block(X, Ut, Vt, True, True, lu, 1, DELTA[TC])
        Vo, _, _, illv = oracle_block(X, Vt, Un, False, True, lv, 1, DELTA[TC])
        for gpu, ora, il in ((Un, Uo, illu), (Vn, Vo, illv)):
            e, fl = r20(gpu, ora)
            flips += fl
            ill += int(il.sum())
        eu, ev = max(eu, r20(Un, Uo)[0]), max(ev, r20(Vn, Vo)[0])
        Ut, Vt = Un, Vn
    print(f"{cfg.name} tc PBCD x1, all rows: per-update U {eu:.2e} V {ev:.2e}, flips {flips} "
          f"({ill} rows would count as ill-conditioned at 2^-22)")
    assert eu < 1e-5 and ev < 1e-5
    assert flips <= 1e-6 * (cfg.m + cfg.n) * cfg.r * 3


# ----------------------------------------------------------------------------- trajectories
@pytest.mark.parametrize("prec", PRECS, ids=PIDS)
@pytest.mark.parametrize("cfg", CASES[:4] + [CASES[6]], ids=IDS[:4] + [IDS[6]])
def test_direct_objective_trajectory_50_sweeps(cfg, prec):
    """The first 50 sweeps of the method from its rotated point (ascent, then HALS).  The
    ascent sweeps are ill-conditioned (module doc; the oracle's own 50-sweep trajectory moves
    by ~1e-2 in f under a one-ulp perturbation of its start, test_pbcd_state_rounding_
    sensitivity), so their per-update parity is test_shadow_ascent_sweeps' (well-conditioned
    rows); here the direct objective of the GPU's ascent sweeps against the oracle's repeat
    of each is printed, and from the GPU's first feasible point on the oracle runs its OWN
    HALS trajectory: the direct objective (enmf_objective(exact=1) vs oracle.frob2_direct)
    within 1e-4 at every remaining sweep.  The GPU's trace-form f within 1e-4 of its direct
    objective where gpu_common.trace_bar_applies."""
    h, X, _ = make(cfg, precision=prec)
    U0, V0, lu, lv = start_point(X, cfg.r, want_infeasible=False)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(0, lu, lv)
    Ut, Vt = U0, V0
    e_asc = e_hals = ftr = 0.0
    n_asc = 0
    Uo = Vo = None
    fgs = []
    for t in range(50):
        f, info = h.iterate(U, V, 1)
        Un, Vn = to_np(U), to_np(V)
        fg = h.objective(U, V, exact=True)
        fgs.append(fg)
        ftr = max(ftr, abs(f[0] - fg) / fg)
        if info["ascent_sweeps"] == 1:
            n_asc += 1
            Ua, _, _, _ = oracle_block(X, Ut, Vt, True, True, lu, info["pbcd_iters_u"])
            Va, _, _, _ = oracle_block(X, Vt, Un, False, True, lv, info["pbcd_iters_v"])
            fa = oracle.frob2_direct(X, Ua, Va)
            e_asc = max(e_asc, abs(fg - fa) / fa)
        else:
            if Uo is None:                       # the oracle's HALS trajectory starts here
                Uo, Vo = Ut, Vt
            Uo, _, _, _ = oracle_block(X, Uo, Vo, True, False)
            Vo, _, _, _ = oracle_block(X, Vo, Uo, False, False)
            fo = oracle.frob2_direct(X, Uo, Vo)
            e_hals = max(e_hals, abs(fg - fo) / fo)
        Ut, Vt = Un, Vn
    print(f"{cfg.name} prec={h.precision}: 50 sweeps ({n_asc} ascent, shadowed: direct f "
          f"{e_asc:.2e}; then the oracle's own HALS trajectory: direct f {e_hals:.2e}), trace "
          f"vs direct {ftr:.2e}")
    assert e_hals < 1e-4
    if trace_bar_applies(prec == TC, X, fgs):
        assert ftr < 1e-4


# ----------------------------------------------------------------------------- end to end
@pytest.mark.parametrize("prec", PRECS, ids=PIDS)
def test_final_objective_and_factors_c1(prec):
    """Full C1 schedule (SVD init + rotation + 200 sweeps, nothing shared) on both sides: final
    f within 1e-3 and factors equal after permutation matching (reading R19) within 1e-3, on
    the fp64 and the tensor-core paths."""
    import paper_2605_19325_b200 as E
    cfg = synth.C1
    X = synth.x_full(cfg)
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=prec)
    U = to_dev(np.zeros((cfg.m, cfg.r)))
    V = to_dev(np.zeros((cfg.n, cfg.r)))
    info = h.init(to_dev(X), U, V)
    f_gpu, it = h.iterate(U, V, cfg.sweeps)
    Uo, Vo, s, f_or, st = oracle.enmf(X, cfg.r, cfg.sweeps, oracle.options(cfg.r, round_f32=1))
    assert np.allclose(info["sigma"][:cfg.r], s, rtol=1e-6)
    assert it["ascent_sweeps"] == 10 and it["hals_sweeps"] == cfg.sweeps - 10
    fx = h.objective(U, V, exact=True)
    Ug, Vg = to_np(U), to_np(V)
    cu = (Ug / np.linalg.norm(Ug, axis=0)).T @ (Uo / np.linalg.norm(Uo, axis=0))
    perm = max(itertools.permutations(range(cfg.r)),
               key=lambda p: sum(cu[p[i], i] for i in range(cfg.r)))
    Ug, Vg = Ug[:, list(perm)], Vg[:, list(perm)]

    def bal(Uf, Vf):
        a = np.sqrt(np.linalg.norm(Vf, axis=0) / np.linalg.norm(Uf, axis=0))
        return Uf * a, Vf / a

    Ug, Vg = bal(Ug, Vg)
    Ub, Vb = bal(Uo, Vo)
    print(f"C1 final prec={h.precision}: f gpu {fx:.8g} (trace {f_gpu[-1]:.8g}) oracle "
          f"{f_or[-1]:.8g}; U {rel_fro(Ug, Ub):.2e} V {rel_fro(Vg, Vb):.2e}")
    assert abs(fx - f_or[-1]) / f_or[-1] < 1e-3
    if trace_bar_applies(prec == TC, X, f_or):
        assert abs(f_gpu[-1] - f_or[-1]) / f_or[-1] < 1e-3
    assert rel_fro(Ug, Ub) < 1e-3 and rel_fro(Vg, Vb) < 1e-3


# ----------------------------------------------------------------------------- rotation
@pytest.mark.parametrize("cfg", CASES[:3] + [CASES[6]], ids=IDS[:3] + [IDS[6]])
def test_admm_stepwise_from_shared_point(cfg):
    """Alg. 1 from the same fp32 [U*; V*]: after T = 1, 2, 3 and 5 ADMM steps
    the GPU's rotated factors equal the oracle's.  Every step is a continuous map (the Z-prox
    of Eq.(7) is piecewise linear and continuous; R = polar(W^T B) is smooth where W^T B is
    nonsingular), so the two agree to rounding: the stored fp32 factors to about one fp32 ulp
    (2e-7 relative), the fp64 negativity to 1e-9."""
    import paper_2605_19325_b200 as E
    X = synth.x_full(cfg)
    Us, Vs, _, _ = oracle.truncated_svd(X, cfg.r)
    U0, V0 = f32(Us), f32(Vs)
    for T in (1, 2, 3, 5):
        h = E.Enmf(cfg.m, cfg.n, cfg.r, admm_iters=T)
        h.set_data(to_dev(X))
        U, V = to_dev(U0), to_dev(V0)
        info = h.rotate(U, V)
        R, neg, third = oracle.admm_rotate(np.vstack([U0, V0]), T=T)
        eu, ev = rel_fro(to_np(U), f32(U0 @ R)), rel_fro(to_np(V), f32(V0 @ R))
        print(f"{cfg.name}: T={T} U {eu:.2e} V {ev:.2e} negativity gpu "
              f"{info['negativity_rot']:.6g} oracle {neg[-1]:.6g}")
        assert info["admm_third_branch"] == 0 and third == 0
        assert eu < 2e-7 and ev < 2e-7
        assert abs(info["negativity_rot"] - neg[-1]) <= 1e-9 * max(neg[-1], 1e-300) + 1e-12
