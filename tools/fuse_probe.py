"""HALS sweep time at C5 with the U block fused behind the X V pass (ENMF_FUSE_HALS=1) and
without (0), alternated A/B so that clock drift under the power cap hits both alike:
graph-replayed calls of 4 sweeps (median of 12 per arm), single-sweep calls, and the X-pass
times under enmf_set_profiling (events / kernel timestamps)."""
import os
import statistics
import sys
sys.path.insert(0, "/root/repo")
import torch
import paper_2605_19325_b200 as E
import synth
cfg = synth.ALL[sys.argv[1] if len(sys.argv) > 1 else "C5-large-planted"]
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
X = torch.empty(cfg.m, cfg.n, device="cuda")
synth.x_rows_device(cfg, 0, cfg.m, X, torch.cuda.current_stream().cuda_stream)
U = torch.empty(cfg.m, cfg.r, device="cuda"); V = torch.empty(cfg.n, cfg.r, device="cuda")
h = E.Enmf(cfg.m, cfg.n, cfg.r)
h.init(X, U, V)
U0, V0 = U.clone(), V.clone()
h.set_stage(1)
h.iterate(U, V, 3)


def timed(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b)


res = {"1": [], "0": []}
single = {"1": [], "0": []}
for rep in range(12):
    for fuse in ("1", "0"):
        os.environ["ENMF_FUSE_HALS"] = fuse
        res[fuse].append(timed(lambda: h.iterate(U, V, 4)) / 4)
        single[fuse].append(timed(lambda: h.iterate(U, V, 1)))
for fuse in ("1", "0"):
    os.environ["ENMF_FUSE_HALS"] = fuse
    h.set_profiling(True)
    prof_ms = timed(lambda: h.iterate(U, V, 6)) / 6
    p = h.profile()
    h.set_profiling(False)
    print(f"fuse={fuse}: graph median {statistics.median(res[fuse]):.3f} ms/sweep "
          f"(min {min(res[fuse]):.3f}), single median {statistics.median(single[fuse]):.3f}, "
          f"profiled {prof_ms:.3f} (xv {p['xv'][0] / max(1, p['xv'][1]):.3f} ms x {p['xv'][1]}, "
          f"xtu {p['xtu'][0] / max(1, p['xtu'][1]):.3f} ms)", flush=True)
print("pairs (fused - unfused, ms):", [round(a - b, 3) for a, b in zip(res["1"], res["0"])])
