import sys, numpy as np
sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else "/root/repo")
sys.path.insert(1, "/root/repo")
import oracle, synth
import paper_2605_19325_b200 as E
from tests.gpu_common import to_dev, to_np, rel_fro
cfg = synth.C3.scaled(160, 900, 32, 32)
X = synth.x_full(cfg)
h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=2)
h.set_data(to_dev(X))
g = np.random.default_rng(3)
U0 = g.random((cfg.m, cfg.r)).astype(np.float32).astype(np.float64)
V0 = g.random((cfg.n, cfg.r)).astype(np.float32).astype(np.float64)
P, Q = h.cross_terms(to_dev(U0), to_dev(V0))
P, Q = to_np(P), to_np(Q)
Pr, Qr = oracle.xv(X, V0), oracle.xtu(X, U0)
print(E.__file__, "P", rel_fro(P, Pr), "Q", rel_fro(Q, Qr), "xnorm", h.objective(to_dev(U0), to_dev(V0), exact=False), oracle.frob2_direct(X, U0, V0))
