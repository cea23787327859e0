import numpy as np, torch, sys, os
sys.path.insert(0, '.')
import oracle, synth
from tests.gpu_common import rel_fro, rotated_point, to_dev, to_np
import paper_2605_19325_b200 as E
cfg = synth.C6.scaled(257, 131, 33, 33, density=0.004)
X = synth.x_full(cfg)
U0, V0, _, _ = rotated_point(X, cfg.r)
U0, V0 = np.abs(U0), np.abs(V0)
rp, ci, v = synth.csr_rows(cfg)
dev = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda())
h = E.Enmf(cfg.m, cfg.n, cfg.r)
h.set_data_csr(*dev)
U, V = to_dev(U0), to_dev(V0)
h.set_stage(1)
_, info = h.iterate(U, V, 1)
Ug, Vg = to_np(U), to_np(V)
Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1), oracle.options(cfg.r, round_f32=1))
print(os.environ.get("ENMF_TC_HALS"), "fallback", info["hals_fallback_rows"], "U", rel_fro(Ug, Uo), "V", rel_fro(Vg, Vo))
# V block inputs as the GPU saw them: Q = X^T U_gpu, G = U_gpu^T U_gpu
Q = X.astype(np.float64).T @ Ug
G = Ug.T @ Ug
np.set_printoptions(precision=3, linewidth=200)
err = np.abs(Vg - Vo).max(axis=1)
for b in np.argsort(-err)[:2]:
    print("row", b, "Q row max", np.abs(Q[b]).max(), "X col nnz", (X[:, b] != 0).sum())
    print(" V0 ", V0[b][:33])
    print(" gpu", Vg[b][:33])
    print(" or ", Vo[b][:33])
print("G diag", np.diag(G))
