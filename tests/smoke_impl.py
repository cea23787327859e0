"""__graft_entry__.smoke(): one small eNMF invocation on cuda:0 vs the oracle."""
import numpy as np


def run_smoke():
    import torch

    import oracle
    import paper_2605_19325_b200 as E
    import synth

    assert torch.cuda.is_available(), "smoke() needs a CUDA device"
    torch.cuda.set_device(0)
    cfg = synth.C1
    X = synth.x_full(cfg)
    h = E.Enmf(cfg.m, cfg.n, cfg.r)
    U = torch.zeros(cfg.m, cfg.r, device="cuda")
    V = torch.zeros(cfg.n, cfg.r, device="cuda")
    # (1) Alg. 3 on the GPU: randomised SVD + ADMM rotation + 20 sweeps (ascent -> HALS)
    info = h.init(torch.from_numpy(X).cuda(), U, V)
    Us, Vs, s, _ = oracle.truncated_svd(X, cfg.r)
    assert np.allclose(info["sigma"], s, rtol=1e-6), (info["sigma"], s)
    f_gpu, it = h.iterate(U, V, 20)
    assert it["ascent_sweeps"] == 10 and it["hals_sweeps"] == 10, it
    assert float(U.min()) >= 0 and float(V.min()) >= 0
    # (2) 5 more HALS sweeps from the GPU's feasible point on both sides
    U0 = U.cpu().numpy().astype(np.float64)
    V0 = V.cpu().numpy().astype(np.float64)
    f_gpu, _ = h.iterate(U, V, 5)
    st = oracle.SweepState(stage=1)
    f_or = []
    for _ in range(5):
        U0, V0, _, _ = oracle.sweep(X, U0, V0, st, oracle.options(cfg.r, round_f32=1))
        f_or.append(oracle.frob2_direct(X, U0, V0))
    rel = np.abs(f_gpu - np.array(f_or)) / np.array(f_or)
    assert rel.max() < 1e-4, rel
    # (3) one HALS sweep through the tcgen05 tensor-core contraction path
    c5 = synth.C5.scaled(400, 300, 128, 128)
    X5 = synth.x_full(c5)
    h5 = E.Enmf(c5.m, c5.n, c5.r, precision=E.PREC_TC)
    h5.set_data(torch.from_numpy(X5).cuda())
    g = np.random.default_rng(0)
    U5 = g.random((c5.m, c5.r)).astype(np.float32)
    V5 = g.random((c5.n, c5.r)).astype(np.float32)
    Ud, Vd = torch.from_numpy(U5).cuda(), torch.from_numpy(V5).cuda()
    h5.set_stage(1)
    h5.iterate(Ud, Vd, 1)
    Uo, Vo, _, _ = oracle.sweep(X5, U5.astype(np.float64), V5.astype(np.float64),
                                oracle.SweepState(stage=1), oracle.options(c5.r, round_f32=1))
    eu = np.linalg.norm(Ud.cpu().numpy() - Uo) / np.linalg.norm(Uo)
    ev = np.linalg.norm(Vd.cpu().numpy() - Vo) / np.linalg.norm(Vo)
    assert eu < 1e-5 and ev < 1e-5, (eu, ev)
    # (4) one ascent sweep (lift + PBCD) with the tensor-core PBCD kernel, repeated by the
    # oracle from the GPU's own state with the GPU's k* (the well-posed parity of
    # tests/test_gpu_shadow.py): 1e-5 per factor on the rows that are well conditioned at the
    # path's 2^-22 operand rounding (reading R33), no mask flips (R20)
    from tests.test_gpu_shadow import TC, Shadow, shadow_sweep, start_point
    c4 = synth.C4.scaled(300, 250, 20, 0)
    X4 = synth.x_full(c4)
    Ur, Vr, lu, lv = start_point(X4, c4.r, want_infeasible=True)
    ht = E.Enmf(c4.m, c4.n, c4.r, precision=E.PREC_TC)
    ht.set_data(torch.from_numpy(X4).cuda())
    Ut = torch.from_numpy(Ur.astype(np.float32)).cuda()
    Vt = torch.from_numpy(Vr.astype(np.float32)).cuda()
    ht.set_stage(0, lu, lv)
    _, it4 = ht.iterate(Ut, Vt, 1)
    assert it4["ascent_sweeps"] == 1, it4
    sh = Shadow(c4.m, c4.n, c4.r)
    shadow_sweep(sh, X4, Ur, Vr, Ut.cpu().numpy().astype(np.float64),
                 Vt.cpu().numpy().astype(np.float64), it4, lu, lv, TC, 0)
    ea, eb = sh.eu, sh.ev
    assert ea < 1e-5 and eb < 1e-5 and sh.flips == 0, (ea, eb, sh.flips, sh.ill)
    print(f"smoke ok: HALS f rel err {rel.max():.2e}; tc path ({h5.precision}) U {eu:.2e} "
          f"V {ev:.2e}; tc ascent (k* {it4['pbcd_iters_u']}/{it4['pbcd_iters_v']}) U {ea:.2e} "
          f"V {eb:.2e} ({sh.ill} ill-conditioned rows excluded, 0 flips); "
          f"launches {h.launch_count + h5.launch_count + ht.launch_count}")
