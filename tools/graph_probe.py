import sys; sys.path.insert(0,'.')
import numpy as np, torch, synth, paper_2605_19325_b200 as E
from tests.gpu_common import make, rotated_point, to_dev
for prec in (1,2):
    cfg = synth.C5.scaled(400, 300, 128, 128, name="x")
    h, X, _ = make(cfg, precision=prec)
    U0, V0, lu, lv = rotated_point(X, cfg.r)
    U, V = to_dev(np.abs(U0)), to_dev(np.abs(V0))
    h.set_stage(1)
    try:
        f, i = h.iterate(U, V, 5); print(prec, "hals ok", f)
    except Exception as e: print(prec, "hals fail", e)
    U, V = to_dev(U0), to_dev(V0)
    h2, _, _ = make(cfg, precision=prec)
    h2.set_stage(0, lu, lv)
    try:
        f, i = h2.iterate(U, V, 5); print(prec, "asc ok", f)
    except Exception as e: print(prec, "asc fail", e)
