"""HALS-stage sweep time of the small BASELINE configs (C1-C4) at steady state.

usage: python tools/small_probe.py [sweeps] [cfg ...]
Each config: init, one iterate call that ends the ascent stage, then `sweeps` HALS sweeps timed
with CUDA events on the handle stream (twice: the second call is the steady state).  Run under
`ncu --metrics gpu__time_duration.sum` with a small sweep count for the per-kernel list.
"""
import sys
sys.path.insert(0, ".")
import torch
import synth
import paper_2605_19325_b200 as E

sweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
names = sys.argv[2:] or ["C1", "C2", "C3", "C4"]
stream = torch.cuda.current_stream()
for nm in names:
    cfg = getattr(synth, nm)
    X = torch.empty(cfg.m, cfg.n, device="cuda", dtype=torch.float32)
    synth.x_rows_device(cfg, 0, cfg.m, X, stream.cuda_stream)
    U = torch.empty(cfg.m, cfg.r, device="cuda")
    V = torch.empty(cfg.n, cfg.r, device="cuda")
    h = E.Enmf(cfg.m, cfg.n, cfg.r, stream=stream)
    h.init(X, U, V)
    f, info = h.iterate(U, V, 14)
    assert info["hals_sweeps"] > 0, info
    for rep in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = h.launch_count
        a.record(stream)
        f, info = h.iterate(U, V, sweeps)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"{cfg.name} rep {rep}: {sweeps} HALS sweeps {ms:.3f} ms = {1e3 * ms / sweeps:.1f} us/sweep, "
              f"{(h.launch_count - l0) / sweeps:.1f} launches/sweep, f {f[-1]:.9g}, path {h.precision}",
              flush=True)
    h.close()
    del X, U, V
