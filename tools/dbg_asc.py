import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import synth, oracle
from tests.gpu_common import make, rotated_point, to_dev, to_np, rel_fro
cfg = synth.C1
h, X, _ = make(cfg, precision=2)
U0, V0, lu, lv = rotated_point(X, cfg.r)
U, V = to_dev(U0), to_dev(V0)
h.set_stage(0, lu, lv)
f, info = h.iterate(U, V, 1)
torch.cuda.synchronize()
Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(0, lu, lv, 0), oracle.options(cfg.r, round_f32=1))
print("U err", rel_fro(to_np(U), Uo), "V err", rel_fro(to_np(V), Vo), info)
print(to_np(U)[:3], Uo[:3])
