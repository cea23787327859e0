"""k* (Alg. 2 inner iterations actually used) per ascent sweep at C5 through the public API,
and the time of each sweep (CUDA events)."""
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2605_19325_b200 as E
import synth
cfg = synth.ALL[sys.argv[1] if len(sys.argv) > 1 else "C5-large-planted"]
X = torch.empty(cfg.m, cfg.n, device="cuda")
synth.x_rows_device(cfg, 0, cfg.m, X, torch.cuda.current_stream().cuda_stream)
U = torch.empty(cfg.m, cfg.r, device="cuda"); V = torch.empty(cfg.n, cfg.r, device="cuda")
h = E.Enmf(cfg.m, cfg.n, cfg.r)
h.init(X, U, V)
for t in range(14):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    f, it = h.iterate(U, V, 1)
    b.record(); b.synchronize()
    print(t, it.get("pbcd_iters_u"), it.get("pbcd_iters_v"), it.get("ascent_sweeps"),
          f"{f[0]:.6e}", f"{a.elapsed_time(b):.2f} ms", flush=True)
