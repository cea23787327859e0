"""The persistent cache-resident HALS kernel (csrc/small_sweep.cu; C1-C4 are bound
by launch latency) against the fp64 oracle and against the separate-launch fp64 path.

Every HALS sweep of a single-rank dense fp64-path handle with m n <= 2^26 runs in the
cooperative kernel; ENMF_SMALL_FUSED=0 keeps the separate launches.  Checked here:
  * one HALS sweep from identical (U, V) against the oracle at BASELINE's 1e-5 per factor, the
    trace-form objective of the sweep against the oracle's direct objective (1e-9 here: fp64);
  * 30 sweeps shadowed sweep by sweep (the oracle restarted from the GPU's own state);
  * fused vs separate launches: factors to fp32 rounding flips (1e-7), traces to 1e-12, the
    same stage counters, feasibility flag and trace length, through the ascent -> HALS switch;
  * the result does not depend on how the caller chunks its calls (bitwise), nor on host-state
    calls (enmf_iterate_host) vs device-state calls (bitwise);
  * shapes: all four small BASELINE recipes, ranks 1, 5, 33 (ragged), 70 (three 32-column
    groups), 100 / 128 (four), rows and columns that are not multiples of the 64-row tiles.
"""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import make, rel_fro, rotated_point, to_dev, to_np

pytestmark = pytest.mark.gpu

CASES = [
    synth.C1,
    synth.C2.scaled(150, 700, 49, 49, name="C2-image@150x700"),
    synth.C3.scaled(160, 900, 32, 32, name="C3-spectro@160x900"),
    synth.C4.scaled(300, 250, 20, 20, name="C4-ratings@300x250"),
    synth.C1.scaled(131, 77, 33, 33, name="planted-ragged-r33"),
    synth.C1.scaled(64, 50, 1, 1, name="planted-r1"),
    synth.C5.scaled(200, 330, 70, 70, name="planted-r70"),
    synth.C5.scaled(257, 190, 100, 100, name="planted-r100"),
    synth.C5.scaled(400, 300, 128, 128, name="C5-shape-r128"),
]
IDS = [c.name for c in CASES]


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def oracle_hals_sweep(X, U, V):
    """One HALS sweep of the oracle (Alg. 3): the U block with V fixed, rounded
    to fp32 as the C-ABI stores it (reading R26), then the V block with the new U."""
    Un = f32(oracle.hals(U, oracle.xv(X, V), oracle.gram(V)))
    Vn = f32(oracle.hals(V, oracle.xtu(X, Un), oracle.gram(Un)))
    return Un, Vn


def feasible_start(X, r, seed=3):
    rng = np.random.default_rng(seed)
    m, n = X.shape
    s = np.sqrt(X.mean() / r)
    U = (s * (0.5 + rng.random((m, r)))).astype(np.float32).astype(np.float64)
    V = (s * (0.5 + rng.random((n, r)))).astype(np.float32).astype(np.float64)
    U[rng.random((m, r)) < 0.1] = 0.0          # some entries on the boundary
    V[rng.random((n, r)) < 0.1] = 0.0
    return U, V


def run(h, U0, V0, k, stage=None):
    U, V = to_dev(U0), to_dev(V0)
    if stage is not None:
        h.set_stage(*stage)
    f, info = h.iterate(U, V, k)
    return to_np(U), to_np(V), np.array(f), info


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_fused_hals_sweep_matches_oracle(cfg):
    h, X, _ = make(cfg, precision=1)
    U0, V0 = feasible_start(X, cfg.r)
    l0 = h.launch_count
    run(h, U0, V0, 6, stage=(1,))
    l1 = h.launch_count
    Ug, Vg, f, info = run(h, U0, V0, 1, stage=(1,))
    assert h.launch_count - l1 == l1 - l0, "all sweeps of a call run in ONE persistent kernel"
    Uo, Vo = oracle_hals_sweep(X, U0, V0)
    eu, ev = rel_fro(Ug, Uo), rel_fro(Vg, Vo)
    fo = oracle.frob2_direct(X, Uo, Vo)
    ef = abs(f[0] - fo) / fo
    print(f"{cfg.name}: fused HALS sweep U {eu:.2e} V {ev:.2e} f {ef:.2e}")
    assert eu < 1e-5 and ev < 1e-5
    assert ef < 1e-4 * max(1.0, 1e-12 * oracle.xnorm2(X) / fo)
    assert info["hals_sweeps"] == 1 and info["ascent_sweeps"] == 0 and info["feasible"]
    assert Ug.min() >= 0 and Vg.min() >= 0


@pytest.mark.parametrize("cfg", CASES[:5], ids=IDS[:5])
def test_fused_shadow_30_sweeps(cfg):
    """Sweep by sweep: the oracle's HALS sweep from the GPU's own state against the GPU's next
    state (1e-5 per factor per sweep; all 30 sweeps in ONE kernel launch are compared through
    a second handle that is stepped one sweep at a time -- bitwise the same states)."""
    h, X, _ = make(cfg, precision=1)
    U0, V0 = feasible_start(X, cfg.r)
    Ua, Va, fa, _ = run(h, U0, V0, 30, stage=(1,))
    h2, _, _ = make(cfg, precision=1)
    h2.set_stage(1)
    U, V = to_dev(U0), to_dev(V0)
    worst = 0.0
    fs = []
    for t in range(30):
        Up, Vp = to_np(U), to_np(V)
        f, _ = h2.iterate(U, V, 1)
        fs.append(f[0])
        Uo, Vo = oracle_hals_sweep(X, Up, Vp)
        worst = max(worst, rel_fro(to_np(U), Uo), rel_fro(to_np(V), Vo))
    print(f"{cfg.name}: 30 fused sweeps, worst per-sweep shadow error {worst:.2e}")
    assert worst < 1e-5
    assert np.array_equal(to_np(U), Ua) and np.array_equal(to_np(V), Va)
    assert np.array_equal(np.array(fs), fa)
    fd = h2.objective(U, V, exact=True)
    assert abs(fa[-1] - fd) / fd < 1e-4 * max(1.0, 1e-12 * oracle.xnorm2(X) / fd)


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_fused_equals_separate_launches(cfg, monkeypatch):
    """The method's schedule from the rotated point (ascent sweeps on separate launches, then
    HALS in the persistent kernel) against the same schedule with ENMF_SMALL_FUSED=0."""
    X = synth.x_full(cfg)
    U0, V0, lu, lv = rotated_point(X, cfg.r)
    out = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("ENMF_SMALL_FUSED", fused)
        h, _, _ = make(X, cfg.r, precision=1)
        l0 = h.launch_count
        out[fused] = run(h, U0, V0, 25, stage=(0, lu, lv)) + (h.launch_count - l0,)
        h.close()
    a, b = out["1"], out["0"]
    eu, ev = rel_fro(a[0], b[0]), rel_fro(a[1], b[1])
    ef = float(np.max(np.abs(a[2] - b[2]) / np.abs(b[2])))
    print(f"{cfg.name}: fused vs separate U {eu:.2e} V {ev:.2e} f {ef:.2e}, "
          f"sweeps {a[3]['ascent_sweeps']} + {a[3]['hals_sweeps']}, launches {a[4]} vs {b[4]}")
    assert len(a[2]) == len(b[2]) == 25
    for key in ("ascent_sweeps", "hals_sweeps", "feasible", "pbcd_iters_u", "pbcd_iters_v"):
        assert a[3][key] == b[3][key], key
    assert eu < 1e-6 and ev < 1e-6
    assert ef < 1e-9 * max(1.0, 1e-3 * oracle.xnorm2(X) / np.min(np.abs(b[2])))
    if a[3]["hals_sweeps"] > 2:
        assert a[4] < b[4]


@pytest.mark.parametrize("cfg", [CASES[0], CASES[3], CASES[4]], ids=[IDS[0], IDS[3], IDS[4]])
def test_fused_chunking_and_host_calls_bitwise(cfg):
    """20 sweeps in one call, in calls of 7 + 13, one by one, and through enmf_iterate_host:
    the same factors and objective trace bit for bit (which sweeps run in the persistent
    kernel does not depend on the call pattern)."""
    import torch
    X = synth.x_full(cfg)
    U0, V0, lu, lv = rotated_point(X, cfg.r)
    h, _, _ = make(X, cfg.r, precision=1)
    Ua, Va, fa, ia = run(h, U0, V0, 20, stage=(0, lu, lv))
    for chunks in ((7, 13), (1,) * 20):
        h2, _, _ = make(X, cfg.r, precision=1)
        h2.set_stage(0, lu, lv)
        U, V = to_dev(U0), to_dev(V0)
        fs = []
        for c in chunks:
            f, _ = h2.iterate(U, V, c)
            fs += list(f)
        assert np.array_equal(to_np(U), Ua) and np.array_equal(to_np(V), Va), chunks
        assert np.array_equal(np.array(fs), fa), chunks
    h3, _, _ = make(X, cfg.r, precision=1)
    h3.set_stage(0, lu, lv)
    Uh = torch.from_numpy(U0.astype(np.float32)).pin_memory()
    Vh = torch.from_numpy(V0.astype(np.float32)).pin_memory()
    fs = []
    for c in (5, 1, 14):
        f, _ = h3.iterate_host(Uh, Vh, c)
        fs += list(f)
    assert np.array_equal(Uh.numpy().astype(np.float64), Ua)
    assert np.array_equal(Vh.numpy().astype(np.float64), Va)
    assert np.array_equal(np.array(fs), fa)


def test_fused_zero_gram_column_and_empty_rows():
    """A zero column of V (G_kk = 0: HALS skips the column, PAPER.md:322-324 divides by G_kk)
    and all-zero rows of X."""
    cfg = synth.C1.scaled(90, 70, 6, 6, name="zero-column")
    X = synth.x_full(cfg)
    X[10:14] = 0.0
    h, _, _ = make(X, cfg.r, precision=1)
    U0, V0 = feasible_start(X, cfg.r)
    V0[:, 2] = 0.0
    Ug, Vg, f, _ = run(h, U0, V0, 1, stage=(1,))
    Uo, Vo = oracle_hals_sweep(X, U0, V0)
    print(f"zero column: U {rel_fro(Ug, Uo):.2e} V {rel_fro(Vg, Vo):.2e}")
    assert rel_fro(Ug, Uo) < 1e-5 and rel_fro(Vg, Vo) < 1e-5
    assert np.isfinite(f).all()
