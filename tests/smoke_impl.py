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
    info = h.init(Xd, U, V)
    f_gpu, it = h.iterate(U, V, 20)
    Uo, Vo, s, f_or, st = oracle.enmf(X, cfg.r, 20)
    rel = np.abs(f_gpu - f_or) / f_or
    assert np.allclose(info["sigma"], s, rtol=1e-6), (info["sigma"], s)
    assert rel.max() < 1e-4, rel
    assert it["ascent_sweeps"] + it["hals_sweeps"] == 20
    assert h.launch_count > 0
    print(f"smoke ok: f[19] gpu={f_gpu[-1]:.8g} oracle={f_or[-1]:.8g} max rel={rel.max():.2e} "
          f"launches={h.launch_count}")
