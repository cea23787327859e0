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
    Xd = torch.from_numpy(X).cuda()
    U = torch.zeros(cfg.m, cfg.r, device="cuda")
    V = torch.zeros(cfg.n, cfg.r, device="cuda")
    # (1) init on the GPU (randomised SVD + ADMM) vs the oracle's converged SVD
    info = h.init(Xd, U, V)
    Us, Vs, s, _ = oracle.truncated_svd(X, cfg.r)
    assert np.allclose(info["sigma"], s, rtol=1e-6), (info["sigma"], s)
    # (2) 20 sweeps (10 ascent + 10 HALS) from the oracle's rotated point on both sides
    R, _, _ = oracle.admm_rotate(np.vstack([Us, Vs]), T=100)
    U0 = (Us @ R).astype(np.float32)
    V0 = (Vs @ R).astype(np.float32)
    U.copy_(torch.from_numpy(U0))
    V.copy_(torch.from_numpy(V0))
    lu = oracle.lift_constant(U0.astype(np.float64))
    lv = oracle.lift_constant(V0.astype(np.float64))
    h.set_stage(0, lu, lv)
    f_gpu, it = h.iterate(U, V, 20)
    st = oracle.SweepState(0, lu, lv, 0)
    Uo, Vo = U0.astype(np.float64), V0.astype(np.float64)
    f_or = []
    for _ in range(20):
        Uo, Vo, _, _ = oracle.sweep(X, Uo, Vo, st, oracle.options(cfg.r, round_f32=1))
        f_or.append(oracle.frob2_direct(X, Uo, Vo))
    rel = np.abs(f_gpu - np.array(f_or)) / np.array(f_or)
    assert rel.max() < 1e-4, rel
    assert it["ascent_sweeps"] == 10 and it["hals_sweeps"] == 10, it
    assert h.launch_count > 0
    print(f"smoke ok: f[19] gpu={f_gpu[-1]:.8g} oracle={f_or[-1]:.8g} max rel={rel.max():.2e} "
          f"launches={h.launch_count}")
