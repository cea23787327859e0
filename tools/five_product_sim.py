"""Design probe (CPU, numpy; not product code): accuracy of the X passes with 5 digit products
(2-digit, 15-bit factor) against the 6 used, at C5-recipe rows and several K.  The 5-product
form was 12 % faster in bench.py (a timing-only build that skipped A0 B2: 61.3 -> 68.6 sweeps/s, X passes
6.35 -> 5.42 ms at the power cap) but one HALS U update errs by 2.7e-5 at K = 16000 (bar
1e-5), so the passes keep 6 products.  Usage: python tools/five_product_sim.py 300 1000 4000"""
import numpy as np, sys
def pow2(mx, top):
    mx = np.maximum(mx, 1e-300); return 2.0 ** np.floor(np.log2(top / mx))
def dig3(t):   # mixed radix (8,8,7): n = rint(t 2^15)
    n = np.rint(t * 2.0**15).astype(np.int64)
    d2 = ((n + 64) & 127) - 64
    n = (n - d2) >> 7
    d1 = ((n + 128) & 255) - 128
    d0 = (n - d1) >> 8
    return [d0, d1, d2], [1.0, 2.0**-8, 2.0**-15]
def dig2(t):   # 2 digits base 2^8: n = rint(t 2^8)
    n = np.rint(t * 2.0**8).astype(np.int64)
    d1 = ((n + 128) & 255) - 128
    d0 = (n - d1) >> 8
    return [d0, d1], [1.0, 2.0**-8]
def contract(A, sa, F, sf, fdig, keep):
    # A: rows x K (X), scales per row sa; F: K x r, scales per column sf
    Ad, wa = dig3(A * sa[:, None]); Fd, wf = fdig(F * sf[None, :])
    acc = 0.0
    for i, a in enumerate(Ad):
        for j, b in enumerate(Fd):
            if (i, j) in keep:
                acc = acc + (a.astype(np.float64) @ b.astype(np.float64)) * wa[i] * wf[j]
    return acc / sa[:, None] / sf[None, :]
K6 = {(0,0),(0,1),(1,0),(1,1),(0,2),(2,0)}
K5 = {(0,0),(0,1),(1,0),(1,1),(2,0)}
def hals(F, C, G):
    F = F.copy()
    for k in range(F.shape[1]):
        F[:, k] = np.maximum(0.0, F[:, k] + (C[:, k] - F @ G[:, k]) / G[k, k])
    return F
g = np.random.default_rng(0)
r = 128
for K in [int(a) for a in sys.argv[1:]]:
    m = 1500
    U0 = g.random((m, r)); V0 = g.random((K, r))
    X = (U0 @ V0.T + 0.01 * np.abs(g.standard_normal((m, K)))).astype(np.float32).astype(np.float64)
    U = np.abs(U0 * (1 + 0.02 * g.standard_normal(U0.shape))).astype(np.float32).astype(np.float64)
    V = np.abs(V0 * (1 + 0.02 * g.standard_normal(V0.shape))).astype(np.float32).astype(np.float64)
    P = X @ V; G = V.T @ V
    sa = pow2(np.abs(X).max(1), 126.0); sf = pow2(np.abs(V).max(0), 126.0)
    Uref = hals(U, P, G)
    out = [f"K={K}:"]
    for name, fd, keep in (("6p", dig3, K6), ("5p", dig2, K5)):
        Pt = contract(X, sa, V, sf, fd, keep)
        # consistent Gram of the quantised factor for the 5p case (as the trace form would)
        Un = hals(U, Pt, G)
        out.append(f"{name}: P {np.linalg.norm(Pt-P)/np.linalg.norm(P):.2e} HALS-U {np.linalg.norm(Un-Uref)/np.linalg.norm(Uref):.2e}")
    print("  ".join(out), flush=True)
