"""C5: trace-form f vs the direct objective after the bench schedule's first sweeps, and the
HALS sweep rate of the tensor-core path."""
import time

import numpy as np
import torch

import paper_2605_19325_b200 as E
import synth

cfg = synth.C5
m, n, r = cfg.m, cfg.n, cfg.r
X = torch.empty(m, n, device="cuda")
synth.x_rows_device(cfg, 0, m, X)
h = E.Enmf(m, n, r, precision=E.PREC_TC)
U = torch.empty(m, r, device="cuda")
V = torch.empty(n, r, device="cuda")
h.init(X, U, V)
out = []
for k in (10, 20, 30):
    f, info = h.iterate(U, V, 10)
    fx = h.objective(U, V, exact=True)
    out.append((k, f[-1], fx, abs(f[-1] - fx) / fx, info["hals_sweeps"]))
torch.cuda.synchronize()
t = time.time()
f, info = h.iterate(U, V, 20)
torch.cuda.synchronize()
dt = time.time() - t
fx = h.objective(U, V, exact=True)
out.append((50, f[-1], fx, abs(f[-1] - fx) / fx, info["hals_sweeps"]))
print("HALS sweeps/s %.2f" % (20 / dt))
for o in out:
    print("after %d sweeps: f_trace %.12e f_direct %.12e rel %.2e (hals %d)" % o)
