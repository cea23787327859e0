"""The Gram of the quantised U on the tensor cores (tc_gemm.cu tc_gram_quantised) against the
fp64 SIMT Gram of the same quantised values (kernels_gram.cu with the factor scales,
ENMF_TC_GRAM=0).

On the tensor-core path G_U is the Gram of the U digits pass 2 multiplied: the
V update and the trace-form objective use it.  The tensor-core version sums every digit
product exactly (int32 classes, int64 totals) and rounds once to fp64; the SIMT version
accumulates the same quantised values in fp64.  They agree to the SIMT sum's rounding, and the
tensor-core Gram is
symmetric bitwise (exact integer sums).  A 1e-16 difference in G_U can flip the fp32 rounding
of a factor entry (R26: the state is stored in fp32), one ulp = 6e-8 of that entry, so the
sweeps are held to 1e-8; the objective of one fixed state to 1e-13."""
import os

import numpy as np
import pytest

import synth
from tests.gpu_common import make, to_dev, to_np

pytestmark = pytest.mark.gpu

TC = 2
CASES = [
    synth.C5.scaled(400, 300, 128, 128, name="C5-shape-r128"),
    synth.C2.scaled(361, 700, 49, 49),
    synth.C1.scaled(3000, 131, 33, 33, name="planted-3000x131-r33"),
]
IDS = [c.name for c in CASES]


def _run(cfg, X, U0, V0, tcgram):
    old = os.environ.get("ENMF_TC_GRAM")
    os.environ["ENMF_TC_GRAM"] = tcgram
    try:
        h, _, _ = make(X, cfg.r, precision=TC)
        U, V = to_dev(U0), to_dev(V0)
        f_obj = h.objective(U, V, exact=False)
        h.set_stage(1)
        l0 = h.launch_count
        f, _ = h.iterate(U, V, 3)
        launches = h.launch_count - l0
        h.close()
        return to_np(U), to_np(V), np.array(f), f_obj, launches
    finally:
        if old is None:
            del os.environ["ENMF_TC_GRAM"]
        else:
            os.environ["ENMF_TC_GRAM"] = old


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_tc_gram_matches_simt_gram_of_quantised_u(cfg):
    X = synth.x_full(cfg)
    g = np.random.default_rng(4)
    U0 = (0.5 + g.random((cfg.m, cfg.r))).astype(np.float32).astype(np.float64)
    V0 = (0.5 + g.random((cfg.n, cfg.r))).astype(np.float32).astype(np.float64)
    Ua, Va, fa, oa, la = _run(cfg, X, U0, V0, "1")
    Ub, Vb, fb, ob, lb = _run(cfg, X, U0, V0, "0")
    # (at these row counts the fp64 SIMT sums of the <= 44-bit digit products stay below 2^53,
    # so they are exact too and the two agree bitwise; at C5, 2e5 rows, they round, and the
    # tensor-core Gram is what test_gpu_fullsize.py's trace-form bar (1e-6 of the direct
    # objective) exercises.  Both paths issue 3 counted launches per Gram.)
    eu = np.linalg.norm(Ua - Ub) / np.linalg.norm(Ub)
    ev = np.linalg.norm(Va - Vb) / np.linalg.norm(Vb)
    ef = np.max(np.abs(fa - fb) / fb)
    eo = abs(oa - ob) / ob
    print(f"{cfg.name}: tc Gram vs SIMT Gram: U {eu:.1e} V {ev:.1e} f {ef:.1e} objective {eo:.1e} "
          f"(launches per 3 sweeps {la} / {lb})")
    assert eo < 1e-13
    assert eu < 1e-8 and ev < 1e-8 and ef < 1e-8
