import numpy as np, torch, sys
sys.path.insert(0, '.')
import oracle, synth
from tests.gpu_common import rel_fro, rotated_point, to_dev, to_np
import paper_2605_19325_b200 as E
cfg = synth.C6.scaled(257, 131, 33, 33, density=0.004, name="sparse-ragged-empty-rows")
X = synth.x_full(cfg)
U0, V0, _, _ = rotated_point(X, cfg.r)
U0, V0 = np.abs(U0), np.abs(V0)
print("U0 col norms", np.round(np.linalg.norm(U0, axis=0)[:8], 3), "V0 max", np.abs(V0).max(), "min nonzero", np.abs(V0[V0 != 0]).min())
import os
for mode in ("dense", "dense-tc", "csr"):
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=2 if mode == "dense-tc" else 0)
    if mode.startswith("dense"):
        h.set_data(to_dev(X))
    else:
        rp, ci, v = synth.csr_rows(cfg)
        dev = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda())
        h.set_data_csr(*dev)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    _, info = h.iterate(U, V, 1)
    Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1), oracle.options(cfg.r, round_f32=1))
    Vg = to_np(V)
    err = np.abs(Vg - Vo).max(axis=1)
    bad = np.argsort(-err)[:5]
    print(mode, h.precision, "fallback", info["hals_fallback_rows"], "U", rel_fro(to_np(U), Uo), "V", rel_fro(Vg, Vo), "|Vo|", np.linalg.norm(Vo))
    for b in bad:
        print("  row", b, "err", err[b], "gpu max", np.abs(Vg[b]).max(), "or max", np.abs(Vo[b]).max(), "V0 max", np.abs(V0[b]).max())
