"""eNMC (App. C; Alg. NMC) on the GPU (enmf_set_data_masked,
enmf_softimpute, enmf_rotate, enmf_iterate) against the eNMC oracle (oracle_nmc.c), on
C4-recipe ratings matrices: the stored ratings are the OBSERVED entries, the zeros missing
(the MovieLens-1M setting of PAPER.md:1369-1371; no MovieLens data is used).  The sweep
parity uses the well-posed form of test_gpu_shadow.py (oracle from the GPU's state with the
GPU's k*, R20 flips, ill-conditioned PBCD rows excluded at the fp64 precision)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import rel_fro, to_dev, to_np
from tests.test_gpu_shadow import r20

pytestmark = pytest.mark.gpu

EPS, MAX_ITER = 1e-2, 50


def ratings(m, n, r, name):
    cfg = synth.C4.scaled(m, n, r, 0, name=name)
    X = synth.x_full(cfg)
    return cfg, X, X > 0


CASES = [ratings(1200, 900, 10, "C4-1200x900-r10"), ratings(700, 560, 20, "C4-700x560-r20"),
         ratings(400, 333, 37, "C4-400x333-r37")]
IDS = [c[0].name for c in CASES]


def bind(X, M, r):
    import torch
    import paper_2605_19325_b200 as E
    obs = oracle.Observed(X, M)
    m, n = X.shape
    h = E.Enmf(m, n, r)
    dev = (torch.from_numpy(obs.ptr).cuda(), torch.from_numpy(obs.idx).cuda(),
           torch.from_numpy(obs.val).cuda())
    h.set_data_masked(*dev)
    h._keep = dev
    assert h.precision == "nmc-f64"
    return h, obs


def start(m, r, seed=0):
    return np.random.default_rng(seed).standard_normal((m, r)).astype(np.float32)


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_softimpute_matches_oracle(case):
    """softImpute-ALS (lambda = 0, reading R31) from the same start, 40 iterations: the rank-r
    model A B^T on every entry (observed and missing) and D within 1e-8 relative; the masked
    objective of the GPU's output equals the oracle's f^ of it (1e-12)."""
    cfg, X, M = case
    h, obs = bind(X, M, cfg.r)
    U0 = start(cfg.m, cfg.r)
    U, V = to_dev(np.zeros((cfg.m, cfg.r))), to_dev(np.zeros((cfg.n, cfg.r)))
    d = h.softimpute(to_dev(U0), 40, U, V)
    A, B, do = oracle.softimpute(obs, U0.astype(np.float64), 40)
    Ag, Bg = to_np(U), to_np(V)
    em = rel_fro(Ag @ Bg.T, A @ B.T)
    ed = np.abs(d / do - 1).max()
    fg = h.objective(U, V)
    fo = oracle.nmc_objective(obs, Ag, Bg)
    print(f"{cfg.name}: {obs.val.size} observed, model A B^T {em:.2e}, D {ed:.2e}, "
          f"f^ {fo:.6g}, A {rel_fro(Ag, A):.2e} B {rel_fro(Bg, B):.2e}")
    assert em < 1e-6 and ed < 1e-8        # fp32 outputs: A, B rounded to 2^-24
    assert abs(fg - fo) <= 1e-12 * fo


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_nmc_sweeps_shadowed(case):
    """softImpute (40 iterations) -> Alg. 1 rotation -> 12 eNMC sweeps; every sweep repeated
    by the oracle from the GPU's state with the GPU's k* (U block from (U_t, V_t), V block from
    the GPU's U_t+1): 1e-5 per factor on the well-conditioned rows (R20, ill-conditioned rows
    <= 10 %), no flips, f^ of the GPU's state equal to the oracle's f^ of it."""
    cfg, X, M = case
    h, obs = bind(X, M, cfg.r)
    U0 = start(cfg.m, cfg.r)
    U, V = to_dev(np.zeros((cfg.m, cfg.r))), to_dev(np.zeros((cfg.n, cfg.r)))
    h.softimpute(to_dev(U0), 40, U, V)
    info = h.rotate(U, V)
    lu, lv = info["lambda_u"], info["lambda_v"]
    Ut, Vt = to_np(U), to_np(V)
    worst = [0.0, 0.0]
    flips = ill = 0
    ill_frac = 0.0
    kmis = []
    g = np.random.default_rng(3)
    for t in range(12):
        f, it = h.iterate(U, V, 1)
        Un, Vn = to_np(U), to_np(V)
        for b, (F, O, lam, k, gpu, blk) in enumerate(((Ut, Vt, lu, it["pbcd_iters_u"], Un, "U"),
                                                      (Vt, Un, lv, it["pbcd_iters_v"], Vn, "V"))):
            Fl = oracle.lift(F, lam)
            Msk = Fl >= 0
            _, own, _, _ = oracle.nmc_pbcd(obs, Fl, O, Msk, blk, EPS, MAX_ITER)
            Fo, _, _, _ = oracle.nmc_pbcd(obs, Fl, O, Msk, blk, 0.0, k)
            if own != k:
                kmis.append((t, blk, k, own))
            # rows ill-conditioned at fp64 precision: moved by > 1e-6 under 1e-15 perturbations
            spread = np.zeros(len(Fo))
            nrm = np.maximum(np.linalg.norm(Fo, axis=1), 1e-300)
            for _ in range(2):
                Fp = Fl * (1 + 1e-15 * g.standard_normal(Fl.shape))
                Op = O * (1 + 1e-15 * g.standard_normal(O.shape))
                Fq, _, _, _ = oracle.nmc_pbcd(obs, Fp, Op, Msk, blk, 0.0, k)
                spread = np.maximum(spread, np.linalg.norm(Fq - Fo, axis=1) / nrm)
            bad = spread > 1e-6
            ill += int(bad.sum())
            ill_frac = max(ill_frac, float(bad.mean()))
            e, fl = r20(gpu[~bad], Fo.astype(np.float32).astype(np.float64)[~bad])
            worst[b] = max(worst[b], e)
            flips += fl
        fo = oracle.nmc_objective(obs, Un, Vn)
        assert abs(f[0] - fo) <= 1e-12 * fo
        Ut, Vt = Un, Vn
    print(f"{cfg.name}: 12 eNMC sweeps, per-update U {worst[0]:.2e} V {worst[1]:.2e}, flips "
          f"{flips}, ill-conditioned rows {ill} (worst block {100 * ill_frac:.1f} %), k* "
          f"mismatches {kmis}, f^ {f[0]:.6g}, min U {Ut.min():.3g} V {Vt.min():.3g}")
    assert worst[0] < 1e-5 and worst[1] < 1e-5
    assert flips == 0 and ill_frac <= 0.10


def test_nmc_full_mask_equals_enmf_ascent():
    """With every entry observed the eNMC sweep is the eNMF ascent sweep (App. C reduces to
    Alg. 3's feasibility stage): the GPU's eNMC sweep from a shared infeasible point against
    the GPU's dense fp64 eNMF ascent sweep with the same lift constants, to 1e-9 with 3 inner
    iterations (beyond that Alg. 2 amplifies the two formulations' rounding, R33)."""
    import paper_2605_19325_b200 as E
    cfg = synth.C1
    X = synth.x_full(cfg)
    r = cfg.r
    h, obs = bind(X, np.ones(X.shape, bool), r)
    Us, Vs, _, _ = oracle.truncated_svd(X, r)
    U0, V0 = Us.astype(np.float32), Vs.astype(np.float32)
    lu, lv = oracle.lift_constant(U0), oracle.lift_constant(V0)
    h2 = E.Enmf(cfg.m, cfg.n, r, precision=E.PREC_FP64, pbcd_max_iter=3)
    h2.set_data(to_dev(X))
    h3 = E.Enmf(cfg.m, cfg.n, r, pbcd_max_iter=3)
    dev = h._keep
    h3.set_data_masked(*dev)
    U, V = to_dev(U0), to_dev(V0)
    U2, V2 = to_dev(U0), to_dev(V0)
    h3.set_stage(0, lu, lv)
    h2.set_stage(0, lu, lv)
    _, i3 = h3.iterate(U, V, 1)
    _, i2 = h2.iterate(U2, V2, 1)
    eu, ev = rel_fro(to_np(U), to_np(U2)), rel_fro(to_np(V), to_np(V2))
    print(f"full mask: eNMC vs eNMF ascent sweep U {eu:.2e} V {ev:.2e}, k* {i3['pbcd_iters_u']}/"
          f"{i2['pbcd_iters_u']}")
    assert eu < 1e-9 and ev < 1e-9


def test_nmc_edge_cases():
    """Rows / columns with no observed entry keep their values (their masked gradient is 0);
    a wrong call order and a multi-rank / r > 64 handle are rejected."""
    import torch
    import paper_2605_19325_b200 as E
    g = np.random.default_rng(5)
    m, n, r = 90, 70, 4
    X = (g.random((m, r)) @ g.random((n, r)).T).astype(np.float32)
    M = g.random((m, n)) < 0.5
    M[7] = False
    M[:, 11] = False
    h, obs = bind(X, M, r)
    U0 = g.random((m, r)).astype(np.float32)
    V0 = g.random((n, r)).astype(np.float32)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(0, 0.0, 0.0)
    h.iterate(U, V, 2)
    assert np.array_equal(to_np(U)[7], U0[7].astype(np.float64))
    assert np.array_equal(to_np(V)[11], V0[11].astype(np.float64))
    with pytest.raises(E.EnmfError) as ei:
        h.kkt(U, V)
    assert ei.value.code == -9
    h2 = E.Enmf(m, n, r)
    with pytest.raises(E.EnmfError) as ei:
        h2.softimpute(to_dev(U0), 5, U, V)          # not bound as masked
    assert ei.value.code == -9
    h3 = E.Enmf(200, 150, 65)
    with pytest.raises(E.EnmfError) as ei:
        h3.set_data_masked(*[torch.zeros(201, dtype=torch.int64, device="cuda"),
                             torch.zeros(0, dtype=torch.int32, device="cuda"),
                             torch.zeros(0, dtype=torch.float32, device="cuda")])
    assert ei.value.code == -2
