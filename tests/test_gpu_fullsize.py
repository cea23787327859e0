"""Full-size parity at BASELINE's largest config (C5: 200000 x 50000, r = 128, 40 GB X) in the
launch configuration bench.py times (tensor-core path, one GPU).  The oracle cannot run a
whole C5 sweep in seconds, but block updates are row-independent: sampled rows
of the GPU's U block are recomputed by the oracle from X's sampled rows, and sampled rows of
the V block from X's sampled columns and the GPU's U_new.  Tolerance: BASELINE's 1e-5
relative per update (HALS stage), max(1e-5, 10 x oracle floor) is not needed here because
the HALS stage is well conditioned."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _mem_ok():
    import torch
    free, _ = torch.cuda.mem_get_info()
    return free > 110e9


def test_c5_fullsize_hals_sweep_sampled():
    import torch
    import paper_2605_19325_b200 as E
    if not _mem_ok():
        pytest.skip("needs ~110 GB of free device memory")
    cfg = synth.C5
    m, n, r = cfg.m, cfg.n, cfg.r
    X = torch.empty(m, n, device="cuda")
    synth.x_rows_device(cfg, 0, m, X)
    # a feasible, data-scaled start: the planted factors' generator rows with a mild skew
    g = np.random.default_rng(7)
    U0 = (0.5 + g.random((m, r))).astype(np.float32)
    V0 = (0.5 + g.random((n, r))).astype(np.float32)
    U, V = torch.from_numpy(U0).cuda(), torch.from_numpy(V0).cuda()
    h = E.Enmf(m, n, r, precision=E.PREC_TC)
    h.set_data(X)
    assert h.precision.startswith("tc")
    h.set_stage(1)
    f, info = h.iterate(U, V, 1)
    assert info["hals_sweeps"] == 1
    # the trace-form f enmf_iterate reports (tensor-core path: the quantised operands' trace
    # form, tc_gemm.cu) against the direct objective of the same state, at the bench's scale
    fx = h.objective(U, V, exact=True)
    etr = abs(f[0] - fx) / fx
    Ug, Vg = U.cpu().numpy().astype(np.float64), V.cpu().numpy().astype(np.float64)
    del X
    torch.cuda.empty_cache()
    # U block on 48 sampled rows: P_i = X_i V0, G = V0^T V0
    r0 = int(g.integers(0, m - 48))
    rows = np.arange(r0, r0 + 48)
    V0d = V0.astype(np.float64)
    G = V0d.T @ V0d
    Xr = synth.x_block(cfg, r0, 48, 0, n)
    Pr = oracle.xv(Xr, V0d)
    Uo = oracle.hals(U0[rows].astype(np.float64), Pr, G)
    Uo = Uo.astype(np.float32).astype(np.float64)
    eu = np.linalg.norm(Ug[rows] - Uo) / np.linalg.norm(Uo)
    # V block on 24 sampled rows: Q_j = X[:, j]^T U_new (the GPU's U_new), H = U_new^T U_new
    c0 = int(g.integers(0, n - 24))
    cols = np.arange(c0, c0 + 24)
    H = Ug.T @ Ug
    Xc = synth.x_block(cfg, 0, m, c0, 24)
    Qc = oracle.xtu(Xc, Ug)
    Vo = oracle.hals(V0[cols].astype(np.float64), Qc, H).astype(np.float32).astype(np.float64)
    ev = np.linalg.norm(Vg[cols] - Vo) / np.linalg.norm(Vo)
    print(f"C5 full size, sampled HALS update: U rows {eu:.2e}, V rows {ev:.2e}; trace f vs "
          f"direct {etr:.2e}")
    assert eu < 1e-5 and ev < 1e-5
    assert etr < 1e-6


def test_c5_fullsize_ascent_sweep_sampled():
    """One ascent sweep (lift + tensor-core PBCD on both blocks) at C5 full size.  PBCD rows
    are independent given (C, G) and the global iteration count k* (Alg. 2's stopping rule
    sums over all rows), so sampled rows are recomputed by the oracle running exactly the
    GPU's k* iterations (eps = 0), the V rows from the GPU's U_new (the well-posed form of
    test_gpu_shadow.py): 1e-5 per factor over the entries away from 0, no mask
    flips."""
    import torch
    import paper_2605_19325_b200 as E
    from tests.test_gpu_shadow import r20
    if not _mem_ok():
        pytest.skip("needs ~110 GB of free device memory")
    cfg = synth.C5
    m, n, r = cfg.m, cfg.n, cfg.r
    X = torch.empty(m, n, device="cuda")
    synth.x_rows_device(cfg, 0, m, X)
    g = np.random.default_rng(11)
    U0 = (g.random((m, r)) - 0.15).astype(np.float32)
    V0 = (g.random((n, r)) - 0.15).astype(np.float32)
    lu = 1.001 * abs(float(U0.min())) / 10.0          # R9 lift constants
    lv = 1.001 * abs(float(V0.min())) / 10.0
    U, V = torch.from_numpy(U0).cuda(), torch.from_numpy(V0).cuda()
    h = E.Enmf(m, n, r, precision=E.PREC_TC)
    h.set_data(X)
    h.set_stage(0, lu, lv)
    f, info = h.iterate(U, V, 1)
    assert info["ascent_sweeps"] == 1
    ku, kv = info["pbcd_iters_u"], info["pbcd_iters_v"]
    Ug, Vg = U.cpu().numpy().astype(np.float64), V.cpu().numpy().astype(np.float64)
    del X
    torch.cuda.empty_cache()

    def block(F0, C, G, lam, k):
        Fl = oracle.lift(F0.astype(np.float64), lam)
        M = (Fl >= 0).astype(np.uint8)
        out, _, _, _ = oracle.pbcd(Fl, C, G, M, eps=0.0, max_iter=k)
        return out.astype(np.float32).astype(np.float64)

    # U block on 48 sampled rows: P_i = X_i V0, G = V0^T V0 (the V the U block saw)
    r0 = int(g.integers(0, m - 48))
    rows = np.arange(r0, r0 + 48)
    V0d = V0.astype(np.float64)
    G = V0d.T @ V0d
    Pr = oracle.xv(synth.x_block(cfg, r0, 48, 0, n), V0d)
    Uo = block(U0[rows], Pr, G, lu, ku)
    eu, fu = r20(Ug[rows], Uo)
    # V block on 16 sampled rows: Q_j = X[:, j]^T U_new (the GPU's), H = U_new^T U_new
    c0 = int(g.integers(0, n - 16))
    cols = np.arange(c0, c0 + 16)
    H = Ug.T @ Ug
    Qc = oracle.xtu(synth.x_block(cfg, 0, m, c0, 16), Ug)
    Vo = block(V0[cols], Qc, H, lv, kv)
    ev, fv = r20(Vg[cols], Vo)
    print(f"C5 full size, sampled ascent update (k* = {ku}/{kv}): U rows {eu:.2e} "
          f"({fu} flips), V rows {ev:.2e} ({fv} flips)")
    assert eu < 1e-5 and ev < 1e-5 and fu + fv == 0
