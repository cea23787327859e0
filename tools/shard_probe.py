"""Per-GPU work of one rank at N GPUs on one GPU (no collectives): C5 with m / N rows.
The V block is not sharded here (every rank would update n / N rows), so this is an upper
bound on the per-rank compute time of a sweep; comm time is not included."""
import sys
import time

import torch

import paper_2605_19325_b200 as E
import synth

for N in (int(a) for a in sys.argv[1:] or ["1", "2", "4", "8"]):
    cfg = synth.C5.scaled(synth.C5.m // N, synth.C5.n)
    X = torch.empty(cfg.m, cfg.n, device="cuda")
    synth.x_rows_device(cfg, 0, cfg.m, X)
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=E.PREC_TC)
    U = torch.empty(cfg.m, cfg.r, device="cuda")
    V = torch.empty(cfg.n, cfg.r, device="cuda")
    h.init(X, U, V)
    h.iterate(U, V, 12)                       # through the ascent stage
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, info = h.iterate(U, V, 20)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    print(f"N={N}: rows {cfg.m}, HALS sweep {ms:.3f} ms ({info['hals_sweeps']} HALS), "
          f"ideal {15.2 / N:.3f} ms", flush=True)
    del X, h, U, V
    torch.cuda.empty_cache()
