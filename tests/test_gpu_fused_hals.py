"""The fused U block of the tensor-core path against the unfused one.

With ENMF_FUSE_HALS on (the default), sweep() enqueues the tensor-core HALS kernel right behind
the X V pass with programmatic dependent launch: the pass publishes each finished 128-row band
of P = X V and the HALS kernel takes bands in order as they are published (enmf_capi.cu
sweep(), tc_gemm.cu band_ready, tc_pbcd.cu next_band_tile).  Only the schedule changes -- which
CTA updates which rows and when -- so U, V and the objective trace must be BITWISE identical
to the unfused sequence (ENMF_FUSE_HALS=0), through the HALS stage, through the ascent stage
(where the HALS kernel exits at once and the PBCD stages that follow must still see the whole
pass, griddepcontrol.wait), and through CUDA-graph replay of the sweeps (iterate(n >= 3)).
"""
import os

import numpy as np
import pytest

import synth
from tests.gpu_common import make, to_dev, to_np
from tests.test_gpu_shadow import start_point

pytestmark = pytest.mark.gpu

TC = 2
CASES = [
    synth.C5.scaled(400, 300, 128, 128, name="C5-shape-r128"),
    synth.C2.scaled(361, 700, 49, 49),
    synth.C1.scaled(1000, 131, 33, 33, name="planted-ragged-1000x131-r33"),
]
IDS = [c.name for c in CASES]


def _run(cfg, X, U0, V0, stage, lu, lv, calls, fuse):
    old = os.environ.get("ENMF_FUSE_HALS")
    os.environ["ENMF_FUSE_HALS"] = fuse
    try:
        h, _, _ = make(X, cfg.r, precision=TC)
        assert h.precision.startswith("tc")
        U, V = to_dev(U0), to_dev(V0)
        h.set_stage(stage, lu, lv)
        fs, asc = [], 0
        for n in calls:
            f, info = h.iterate(U, V, n)
            fs.extend(list(f))
            asc += info["ascent_sweeps"]
        h.close()
        return to_np(U), to_np(V), np.array(fs), asc
    finally:
        if old is None:
            del os.environ["ENMF_FUSE_HALS"]
        else:
            os.environ["ENMF_FUSE_HALS"] = old


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_fused_hals_bitwise_equals_unfused(cfg):
    X = synth.x_full(cfg)
    # HALS stage from a feasible start: single sweeps, then graph-replayed runs
    g = np.random.default_rng(3)
    U0 = (0.5 + g.random((cfg.m, cfg.r))).astype(np.float32).astype(np.float64)
    V0 = (0.5 + g.random((cfg.n, cfg.r))).astype(np.float32).astype(np.float64)
    a = _run(cfg, X, U0, V0, 1, 0.0, 0.0, [1, 1, 5, 4], "1")
    b = _run(cfg, X, U0, V0, 1, 0.0, 0.0, [1, 1, 5, 4], "0")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])


@pytest.mark.parametrize("cfg", CASES[:2], ids=IDS[:2])
def test_fused_hals_through_ascent_stage(cfg):
    """From an infeasible start: ascent sweeps (the fused HALS kernel exits at once and the
    PBCD stages follow), the switch to HALS, then HALS sweeps -- one call with graph replay."""
    X = synth.x_full(cfg)
    U0, V0, lu, lv = start_point(X, cfg.r, want_infeasible=True)
    a = _run(cfg, X, U0, V0, 0, lu, lv, [1, 14], "1")
    b = _run(cfg, X, U0, V0, 0, lu, lv, [1, 14], "0")
    print(f"{cfg.name}: {a[3]} ascent sweeps of 15")
    assert a[3] == b[3] and a[3] >= 1
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])
