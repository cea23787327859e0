"""Persistent HALS kernel vs separate launches at mid sizes (several waves of tiles, K splits,
multi-round row phases): 5 HALS sweeps from a feasible start, factors and objective compared."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2605_19325_b200 as E

rng = np.random.default_rng(1)
for (m, n, r) in ((3000, 5000, 128), (5000, 3000, 64), (700, 40000, 32), (20000, 1500, 20), (4097, 4099, 97)):
    X = torch.from_numpy((rng.random((m, 8)) @ rng.random((8, n))).astype(np.float32)).cuda()
    U0 = torch.from_numpy(rng.random((m, r)).astype(np.float32)).cuda()
    V0 = torch.from_numpy(rng.random((n, r)).astype(np.float32)).cuda()
    out = {}
    for fused in ("1", "0"):
        os.environ["ENMF_SMALL_FUSED"] = fused
        h = E.Enmf(m, n, r, precision=1)
        h.set_data(X)
        h.set_stage(1)
        U, V = U0.clone(), V0.clone()
        f, info = h.iterate(U, V, 5)
        U2, V2 = U.clone(), V.clone()                 # steady-state time: a second call
        torch.cuda.synchronize(); t0 = time.perf_counter()
        h.iterate(U2, V2, 5)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        out[fused] = (U.double().cpu().numpy(), V.double().cpu().numpy(), np.array(f), dt, h.objective(U, V, exact=True))
        h.close()
    a, b = out["1"], out["0"]
    eu = np.linalg.norm(a[0] - b[0]) / np.linalg.norm(b[0]); ev = np.linalg.norm(a[1] - b[1]) / np.linalg.norm(b[1])
    ef = np.max(np.abs(a[2] - b[2]) / np.abs(b[2])); ed = abs(a[2][-1] - a[4]) / a[4]
    print(f"{m}x{n} r{r}: fused vs separate U {eu:.2e} V {ev:.2e} f {ef:.2e}; trace vs direct {ed:.2e}; "
          f"5 more sweeps {1e3*a[3]:.2f} ms vs {1e3*b[3]:.2f} ms", flush=True)
    assert eu < 1e-6 and ev < 1e-6 and ef < 1e-8 and ed < 1e-6
print("ok")
