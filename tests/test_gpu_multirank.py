"""The multi-rank C-ABI path (X and U row-sharded, V replicated, allreduce of
X^T U, the Grams, the PBCD stopping partials and the init collectives) exercised on ONE GPU:
two processes (gloo) share cuda:0 and the handle's collectives go through
enmf_set_host_allreduce -- stream-synchronous host staging, so no kernel of one rank ever waits
on the other's.  NCCL itself is not exercised here (one GPU); everything around it is:
  * V and the objective trace come out bitwise identical on both ranks;
  * HALS sweeps from a shared feasible point match a single-rank run (the sharded sums differ
    only in summation order);
  * the sharded randomised SVD matches the single-rank singular values."""
import multiprocessing as mp
import socket

import numpy as np
import pytest

from tests import multirank_worker

pytestmark = pytest.mark.gpu

FP64, TC = 1, 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(cfg_args, prec, mode, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=multirank_worker.run, args=(r, world, port, cfg_args, prec, mode, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=600) for _ in ps]
    for p in ps:
        p.join(timeout=120)
    errs = [r["error"] for r in res if "error" in r]
    assert not errs, errs[0]
    return sorted(res, key=lambda r: r["rank"])


def _single(cfg_args, prec, mode):
    import torch

    import paper_2605_19325_b200 as E
    import synth
    from tests.gpu_common import to_dev
    cfg = synth.ALL[cfg_args[0]].scaled(*cfg_args[1:]) if len(cfg_args) > 1 else \
        synth.ALL[cfg_args[0]]
    X = multirank_worker.load_x(cfg, 0, cfg.m) if cfg.recipe == synth.SPARSE else \
        to_dev(synth.x_full(cfg))
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=prec)
    if mode == "init":
        U = torch.empty(cfg.m, cfg.r, device="cuda")
        V = torch.empty(cfg.n, cfg.r, device="cuda")
        info = multirank_worker.init(h, X, U, V)
        f, _ = h.iterate(U, V, 12)
        return np.array(info["sigma"]), f, U.cpu().numpy(), V.cpu().numpy()
    if mode == "ascent":
        U0, V0, lu, lv = multirank_worker.ascent_point(cfg)
        multirank_worker.bind(h, X)
        U, V = torch.from_numpy(U0).cuda(), torch.from_numpy(V0).cuda()
        h.set_stage(0, lu, lv)
        f, _ = h.iterate(U, V, 3)
        return None, f, U.cpu().numpy(), V.cpu().numpy()
    g = np.random.default_rng(5)
    U0 = g.random((cfg.m, cfg.r)).astype(np.float32)
    V0 = g.random((cfg.n, cfg.r)).astype(np.float32)
    multirank_worker.bind(h, X)
    U, V = torch.from_numpy(U0).cuda(), torch.from_numpy(V0).cuda()
    h.set_stage(1)
    f, _ = h.iterate(U, V, 5)
    _single.kkt = h.kkt(U, V)
    _single.fx = h.objective(U, V, exact=True)
    return None, f, U.cpu().numpy(), V.cpu().numpy()


CASES = [(("C1-planted",), FP64), (("C5-large-planted", 400, 300, 128, 128), TC),
         (("C6-reuters-like", 400, 300, 24, 24, None, 0.05), TC)]


@pytest.mark.parametrize("cfg_args,prec", CASES, ids=["C1-fp64", "C5shape-tc", "C6shape-csr"])
def test_two_ranks_hals_match_single_rank(cfg_args, prec):
    r0, r1 = _spawn(cfg_args, prec, "hals")
    assert np.array_equal(r0["V"], r1["V"]), "V must be bitwise identical on all ranks"
    assert np.array_equal(r0["f"], r1["f"])
    _, f, U, V = _single(cfg_args, prec, "hals")
    Ug = np.vstack([r0["U"], r1["U"]])
    # tensor-core path: each rank packs its own digit scales (the X^T copy's column scales
    # and the factor's column maxima are per rank), so one rank and two ranks round the
    # operands differently at the path's ~2^-22 -- held to BASELINE's per-update 1e-5
    tol = 1e-9 if prec == FP64 else 1e-5
    eu = np.linalg.norm(Ug - U) / np.linalg.norm(U)
    ev = np.linalg.norm(r0["V"] - V) / np.linalg.norm(V)
    ef = np.max(np.abs(r0["f"] - f) / f)
    print(f"{cfg_args[0]} prec={prec}: U {eu:.2e} V {ev:.2e} f {ef:.2e}")
    assert eu < tol and ev < tol and ef < tol
    # the sharded KKT statistics and direct objective (rank-combined) match the single rank
    assert r0["kkt"] == r1["kkt"] and r0["fx"] == r1["fx"]
    assert abs(r0["fx"] - _single.fx) <= tol * _single.fx
    # TC: dual_viol / comp_max are maxima over entries of the gradient U G - P, whose relative
    # change is ~cond x the factor difference (tol above); 5 HALS sweeps from a random point
    # with the digit-grid coupling of tc_hals_kernel (2^-26 of a row's max) observed 1.1e-5
    rtol = 1e-9 if prec == FP64 else 5e-5
    for key in ("min_u", "min_v", "comp_max", "dual_viol"):
        a, b = r0["kkt"][key], _single.kkt[key]
        assert abs(a - b) <= rtol * max(abs(b), 1e-12 * _single.kkt["xnorm2"]), key


@pytest.mark.parametrize("cfg_args,prec", CASES, ids=["C1-fp64", "C5shape-tc", "C6shape-csr"])
def test_two_ranks_init_and_ascent_consistent(cfg_args, prec):
    r0, r1 = _spawn(cfg_args, prec, "init")
    assert np.array_equal(r0["V"], r1["V"])
    assert np.array_equal(r0["f"], r1["f"])
    assert np.array_equal(r0["sigma"], r1["sigma"])
    assert r0["it"] == r1["it"]        # same stage schedule (C1: 10 ascent sweeps, R9)
    if cfg_args[0] == "C1-planted":
        assert r0["it"]["ascent_sweeps"] == 10
    sigma, _, _, _ = _single(cfg_args, prec, "init")
    es = np.max(np.abs(r0["sigma"] - sigma) / sigma)
    print(f"{cfg_args[0]} prec={prec}: sigma {es:.2e}")
    assert es < (1e-10 if prec == FP64 else 1e-6)   # tc: the rtol of the SVD-vs-oracle test


@pytest.mark.parametrize("cfg_args,prec", CASES, ids=["C1-fp64", "C5shape-tc", "C6shape-csr"])
def test_two_ranks_ascent_sharded_v(cfg_args, prec):
    """Lift + PBCD sweeps with the V block sharded across the ranks (Alg. 2's stopping rule
    summed over both slices): V and f bitwise identical on the ranks; on the fp64 path the
    factors equal the single-rank run's up to the summation order of the stopping sums."""
    r0, r1 = _spawn(cfg_args, prec, "ascent")
    assert np.array_equal(r0["V"], r1["V"])
    assert np.array_equal(r0["f"], r1["f"])
    assert r0["it"] == r1["it"] and r0["it"]["ascent_sweeps"] == 3
    if prec == FP64:
        _, f, U, V = _single(cfg_args, prec, "ascent")
        Ug = np.vstack([r0["U"], r1["U"]])
        eu = np.linalg.norm(Ug - U) / np.linalg.norm(U)
        ev = np.linalg.norm(r0["V"] - V) / np.linalg.norm(V)
        print(f"{cfg_args[0]} ascent: U {eu:.2e} V {ev:.2e}")
        assert eu < 1e-12 and ev < 1e-12


@pytest.mark.parametrize("mode", ["hals", "ascent"])
def test_two_ranks_sliced_pass2_bitwise(mode, monkeypatch):
    """The tensor-core pass 2 of the sharded V block runs slice by slice (each V slice's band
    range, reduced to its owner while the next slice computes; here through the host
    collective) instead of one pass and one reduction: the per-slice K split differs, but every
    partial is an integer multiple of one power of two below 2^53, so the sums -- and U, V and
    the objective trace -- are bitwise those of the unsliced pass (ENMF_PASS2_SLICED=0).  The
    C5-shape case (n = 300) has 128-row-aligned slices of 256 and 44 rows."""
    cfg_args = ("C5-large-planted", 400, 300, 128, 128)
    monkeypatch.setenv("ENMF_PASS2_SLICED", "1")
    a = _spawn(cfg_args, TC, mode)
    monkeypatch.setenv("ENMF_PASS2_SLICED", "0")
    b = _spawn(cfg_args, TC, mode)
    for ra, rb in zip(a, b):
        assert np.array_equal(ra["U"], rb["U"]) and np.array_equal(ra["V"], rb["V"])
        assert np.array_equal(ra["f"], rb["f"])


def test_three_ranks_sliced_pass2_bitwise(monkeypatch):
    """Three ranks (host collectives on one GPU): n = 700 gives 128-row-aligned V slices of
    256, 256 and 188 rows, so the sliced pass 2 has a short last slice and three reductions;
    U, V and f bitwise equal to the unsliced pass, V and f identical on all ranks."""
    cfg_args = ("C2-image", 361, 700, 49, 49)
    monkeypatch.setenv("ENMF_PASS2_SLICED", "1")
    a = _spawn(cfg_args, TC, "hals", world=3)
    monkeypatch.setenv("ENMF_PASS2_SLICED", "0")
    b = _spawn(cfg_args, TC, "hals", world=3)
    for ra in a[1:]:
        assert np.array_equal(ra["V"], a[0]["V"]) and np.array_equal(ra["f"], a[0]["f"])
    for ra, rb in zip(a, b):
        assert np.array_equal(ra["U"], rb["U"]) and np.array_equal(ra["V"], rb["V"])
        assert np.array_equal(ra["f"], rb["f"])
