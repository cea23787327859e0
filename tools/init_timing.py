"""Init phase timing at C5 (SVD, rotation) through the public API."""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2605_19325_b200 as E
import synth
cfg = synth.ALL["C5-large-planted"]
X = torch.empty(cfg.m, cfg.n, device="cuda")
synth.x_rows_device(cfg, 0, cfg.m, X, torch.cuda.current_stream().cuda_stream)
U = torch.empty(cfg.m, cfg.r, device="cuda"); V = torch.empty(cfg.n, cfg.r, device="cuda")
h = E.Enmf(cfg.m, cfg.n, cfg.r)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter(); h.set_data(X); torch.cuda.synchronize(); t1 = time.perf_counter()
    h.svd(U, V); torch.cuda.synchronize(); t2 = time.perf_counter()
    h.rotate(U, V); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"set_data {t1-t0:.3f} s  svd {t2-t1:.3f} s  rotate {t3-t2:.3f} s")
