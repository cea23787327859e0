"""Diagnostics of the tensor-core X passes: per-entry error of P = X V and Q = X^T U against the
oracle's fp64 products, normalised by the natural scale |X| |V| (resp. |X|^T |U|).

    ENMF_TC_PROMOTE=8 python tools/tc_diag.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2605_19325_b200 as E  # noqa: E402
import synth  # noqa: E402
from tests.gpu_common import rotated_point  # noqa: E402


def report(name, got, ref, scale):
    err = np.abs(got - ref) / np.maximum(scale, 1e-300)
    nrm = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    r = ref.shape[1]
    halves = [err[:, :64].max()] + ([err[:, 64:].max()] if r > 64 else [])
    print(f"  {name}: normwise {nrm:.2e}  max scaled {err.max():.2e}  by col half "
          f"{[f'{h:.1e}' for h in halves]}  worst (row, col) {np.unravel_index(err.argmax(), err.shape)}")


def main():
    print("promote =", os.environ.get("ENMF_TC_PROMOTE", "8"))
    cases = [synth.C5.scaled(400, 300, 128, 128), synth.C5.scaled(700, 650, 128, 128),
             synth.C2.scaled(150, 700, 49, 49), synth.C4.scaled(300, 250, 20, 0)]
    for cfg in cases:
        X = synth.x_full(cfg)
        Xd = torch.from_numpy(X).cuda()
        h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=E.PREC_TC)
        h.set_data(Xd)
        U0, V0, _, _ = rotated_point(X, cfg.r)
        g = np.random.default_rng(0)
        for label, (U, V) in {"random": (g.random(U0.shape), g.random(V0.shape)),
                              "|rotated|": (np.abs(U0), np.abs(V0)),
                              "rotated": (U0, V0)}.items():
            U = U.astype(np.float32).astype(np.float64)
            V = V.astype(np.float32).astype(np.float64)
            P, Q = h.cross_terms(torch.from_numpy(U.astype(np.float32)).cuda(),
                                 torch.from_numpy(V.astype(np.float32)).cuda())
            P, Q = P.cpu().numpy(), Q.cpu().numpy()
            Xa = np.abs(X.astype(np.float64))
            print(f"{cfg.name} {label}:")
            report("P = X V  ", P, oracle.xv(X, V), Xa @ np.abs(V))
            report("Q = X^T U", Q, oracle.xtu(X, U), Xa.T @ np.abs(U))
        h.close()


if __name__ == "__main__":
    main()
