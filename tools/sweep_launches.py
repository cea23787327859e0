"""Per-sweep kernel composition at C5 for the ncu launch list: 3 ascent sweeps from the
rotated point and 3 HALS sweeps, each group inside an NVTX range, so that
    ncu --nvtx --nvtx-include "ascent/" --nvtx-include "hals/" --metrics gpu__time_duration.sum
profiles exactly those sweeps (no init kernels)."""
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
h.iterate(U, V, 2)                    # ascent warm-up (the first U block stops at k* = 1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("ascent")
for _ in range(3):
    h.iterate(U, V, 1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
h.set_stage(1)
h.iterate(U, V, 2)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("hals")
for _ in range(3):
    h.iterate(U, V, 1)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done")
