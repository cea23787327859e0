"""Design probe (CPU, numpy): accuracy of int8-digit encodings for the two X passes.

Emulates, with exact integer arithmetic carried in fp64, the digit products the tensor-core
kernels accumulate in int32 TMEM, and compares P = X V, Q = X^T U, the trace-form cross term
and one HALS V-block update against fp64 on a C5-recipe matrix (planted, r = 128) at reduced
size.  Schemes:
  s7x4  -- round-1 encoding: one global X scale, 4 balanced base-2^7 digits (t*2^21), classes
           <= 3 (10 products) or <= 2 (6 products)
  s8x3  -- per-row (pass 1) / per-column (pass 2) X scales, 3 balanced base-2^8 digits
           (t*2^16, |t| < 127.4), classes <= 2 (6 products)
Not part of the product or the tests; the numbers it prints are quoted in DESIGN.md §5.1.
"""
import sys

import numpy as np


def pow2(mx, top):
    mx = np.maximum(mx, 1e-300)
    return 2.0 ** np.floor(np.log2(top / mx))


def digits(t, frac_bits, base_bits, nd):
    """Balanced digits of t (any shape): t ~ sum_k d_k 2^(-base_bits k), rounded at 2^-frac_bits."""
    n = np.rint(t * 2.0 ** frac_bits).astype(np.int64)
    half = 1 << (base_bits - 1)
    out = []
    for _ in range(nd - 1):
        d = ((n + half) & ((1 << base_bits) - 1)) - half
        out.append(d)
        n = (n - d) >> base_bits
    out.append(n)
    return out[::-1]       # d0 (top) first


def contract(Xd, Fd, classes, base_bits):
    acc = 0.0
    for i, a in enumerate(Xd):
        for j, b in enumerate(Fd):
            if i + j <= classes:
                acc = acc + (a.astype(np.float64) @ b.astype(np.float64)) * 2.0 ** (-base_bits * (i + j))
    return acc


def enc_s7(A, scale):
    return digits(A * scale, 21, 7, 4)


def enc_s8(A, scale):
    return digits(A * scale, 16, 8, 3)


def hals(F, C, G):
    F = F.copy()
    for k in range(F.shape[1]):
        if G[k, k] <= 0:
            continue
        F[:, k] = np.maximum(0.0, F[:, k] + (C[:, k] - F @ G[:, k]) / G[k, k])
    return F


def main(m=20000, n=5000, r=128):
    g = np.random.default_rng(0)
    U0 = g.random((m, r)).astype(np.float32).astype(np.float64)
    V0 = g.random((n, r)).astype(np.float32).astype(np.float64)
    X = (U0 @ V0.T + 0.01 * np.abs(g.standard_normal((m, n)))).astype(np.float32).astype(np.float64)
    # a HALS-stage state near the planted point
    U = np.abs(U0 * (1 + 0.02 * g.standard_normal(U0.shape))).astype(np.float32).astype(np.float64)
    V = np.abs(V0 * (1 + 0.02 * g.standard_normal(V0.shape))).astype(np.float32).astype(np.float64)
    P, Q = X @ V, X.T @ U
    GU = U.T @ U
    cross = float((Q * V).sum())
    f_true = float(((X - U @ V.T) ** 2).sum())
    xn2 = float((X * X).sum())
    Vnew = hals(V, Q, GU)
    print(f"m={m} n={n} r={r}: f={f_true:.6e} ||X||^2/f={xn2 / f_true:.2e}")

    def report(name, Pt, Qt, GUt, xn2t):
        ep = np.linalg.norm(Pt - P) / np.linalg.norm(P)
        eq = np.linalg.norm(Qt - Q) / np.linalg.norm(Q)
        ft = xn2t - 2 * float((Qt * V).sum()) + float((GUt * (V.T @ V)).sum())
        ev = np.linalg.norm(hals(V, Qt, GUt) - Vnew) / np.linalg.norm(Vnew)
        print(f"{name:34s} P {ep:.2e}  Q {eq:.2e}  f_trace {abs(ft - f_true) / f_true:.2e}  "
              f"HALS V {ev:.2e}")

    # round-1 scheme: global X scale, per-column factor scales, 4 x 7-bit
    sx = pow2(np.abs(X).max(), 63.99)
    su, sv = pow2(np.abs(U).max(0), 63.99), pow2(np.abs(V).max(0), 63.99)
    Xd = enc_s7(X, sx)
    Pt = contract(Xd, enc_s7(V, sv), 2, 7) / (sx * sv)
    Qt = contract([d.T for d in Xd], enc_s7(U, su), 3, 7) / (sx * su)
    report("s7x4 (P 6 products, Q 10)", Pt, Qt, GU, xn2)
    # new scheme: per-row / per-column X scales, 3 x 8-bit, 6 products each
    sr = pow2(np.abs(X).max(1), 127.4)[:, None]
    sc = pow2(np.abs(X).max(0), 127.4)[None, :]
    su8, sv8 = pow2(np.abs(U).max(0), 127.4), pow2(np.abs(V).max(0), 127.4)
    Pt = contract(enc_s8(X, sr), enc_s8(V, sv8), 2, 8) / (sr * sv8)
    Xc = enc_s8(X, sc)
    Qt = contract([d.T for d in Xc], enc_s8(U, su8), 2, 8) / (sc.T * su8)
    report("s8x3 (6 + 6 products)", Pt, Qt, GU, xn2)
    # the same with ||X~||^2 and the Gram of the quantised U in the trace form (consistent
    # objective of the quantised operands)
    Xq = sum(d * 2.0 ** (-8 * i) for i, d in enumerate(Xc)) / sc
    Uq = sum(d * 2.0 ** (-8 * i) for i, d in enumerate(enc_s8(U, su8))) / su8
    report("s8x3 + ||Xq||^2, Gram(Uq)", Pt, Qt, Uq.T @ Uq, float((Xq * Xq).sum()))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])


def digits_mixed(t):
    """Mixed radix (8, 8, 7): n = rint(t 2^15) = d0 2^15 + d1 2^7 + d2, d2 symmetric in
    [-64, 64] (a tie goes to +-64 so that the carry is even: mean 0), d1 in [-128, 127]."""
    n = np.rint(t * 2.0 ** 15).astype(np.int64)
    d2 = ((n + 64) & 127) - 64
    tie = (d2 == -64) & (((n + 64) & 128) != 0)
    d2 = np.where(tie, 64, d2)
    n = (n - d2) >> 7
    d1 = ((n + 128) & 255) - 128
    d0 = (n - d1) >> 8
    return [d0, d1, d2]


def contract_mixed(Ad, Bd):
    """acc0 + 2^-8 acc1 + 2^-15 (a0 b2 + a2 b0) + 2^-16 a1 b1 (the six kept products)."""
    mm = lambda a, b: a.astype(np.float64) @ b.astype(np.float64)
    return (mm(Ad[0], Bd[0]) + (mm(Ad[0], Bd[1]) + mm(Ad[1], Bd[0])) * 2.0 ** -8 +
            (mm(Ad[0], Bd[2]) + mm(Ad[2], Bd[0])) * 2.0 ** -15 + mm(Ad[1], Bd[1]) * 2.0 ** -16)


def value_mixed(d):
    return d[0] + d[1] * 2.0 ** -8 + d[2] * 2.0 ** -15
