"""The NCCL code path on real hardware, at one rank.

gpurun gives one GPU per call and NCCL refuses two ranks on one device, so the multi-rank
tests (test_gpu_multirank.py) route their collectives through the host.  A handle given an
ncclUniqueId at world_size == 1 runs the sharded code path with a one-rank communicator
(include/enmf.h, enmf_problem_t.nccl_unique_id): dlopen of the NCCL torch loaded,
ncclCommInitRank, the in-place ncclAllReduce of the Grams / scalars / PBCD partials, the
V-slice layout with 128-row-aligned slices, the sliced pass 2 with its ncclReduce per slice on
the communication stream, the in-place all-gather of the V slices, and the init collectives.
At one rank every collective is an identity, so the sweeps -- from a shared state -- must
equal the plain single-rank handle's bitwise: factors, objective trace, PBCD k*, KKT.  The
init's singular values are bitwise equal too; its ADMM rotation forms W^T B as the rank's U
rows plus rank 0's V rows (fixed-order sum of two partials), so the rotation equals the plain
one to rounding: checked after 5 ADMM steps.  After the default 100 steps the ADMM can be
chaotic (the oracle's own C3-300x1100 rotation moves by 19 % under a 1e-15 perturbation of W
after 100 steps, 6e-15 after 5), so there only the invariant of a rotation is checked: U V^T
equals the plain handle's (both are U* R (V* R)^T = U* V*^T)."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import rel_fro, to_dev, to_np

pytestmark = pytest.mark.gpu

FP64, TC = 1, 2


def _handle(cfg, prec, uid, X, **opts):
    import torch
    import paper_2605_19325_b200 as E
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=prec, nccl_id=uid, **opts)
    U = torch.empty(cfg.m, cfg.r, device="cuda")
    V = torch.empty(cfg.n, cfg.r, device="cuda")
    info = h.init(X, U, V)
    return h, U, V, info


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [synth.C1, synth.C5.scaled(700, 650, 128, 128, name="C5-700x650"),
                                 synth.C3.scaled(300, 1100, 32, 32, name="C3-300x1100")],
                         ids=["C1", "C5-700x650", "C3-300x1100"])
def test_single_rank_nccl_path_bitwise(cfg, prec, monkeypatch):
    import torch
    import paper_2605_19325_b200 as E
    # the plain handle's HALS sweeps on the separate-launch path, which is the one the
    # collective path runs (the persistent small-problem kernel, small_sweep.cu, is a
    # single-rank specialisation with its own fixed summation order: test_gpu_small_fused.py)
    monkeypatch.setenv("ENMF_SMALL_FUSED", "0")
    uid = E.nccl_unique_id()
    assert len(uid) == 128
    X = to_dev(synth.x_full(cfg))
    hp, Up, Vp, ip = _handle(cfg, prec, None, X)
    hc, Uc, Vc, ic = _handle(cfg, prec, uid, X)
    assert hp.precision == hc.precision
    assert np.array_equal(np.array(ip["sigma"]), np.array(ic["sigma"]))
    duv = rel_fro(to_np(Uc) @ to_np(Vc).T, to_np(Up) @ to_np(Vp).T)
    assert duv < 1e-6, duv
    # (a fresh ncclUniqueId per communicator: an id bootstraps exactly one)
    h5 = [_handle(cfg, prec, u, X, admm_iters=5) for u in (None, E.nccl_unique_id())]
    du = rel_fro(to_np(h5[1][1]), to_np(h5[0][1]))
    dv = rel_fro(to_np(h5[1][2]), to_np(h5[0][2]))
    assert du < 1e-6 and dv < 1e-6, (du, dv)
    for h in h5:
        h[0].close()
    # sweeps from the plain handle's rotated point, then the ascent from the SVD point
    Uc.copy_(Up)
    Vc.copy_(Vp)
    hc.set_stage(*hp.get_stage())
    outs = []
    for h, U, V in ((hp, Up, Vp), (hc, Uc, Vc)):
        f, it = h.iterate(U, V, 14)
        kkt = h.kkt(U, V)
        h.svd(U, V)
        Us, Vs = to_np(U), to_np(V)
        h.set_stage(0, oracle.lift_constant(Us), oracle.lift_constant(Vs))
        f2, it2 = h.iterate(U, V, 3)
        torch.cuda.synchronize()
        outs.append((np.concatenate([f, f2]), to_np(U), to_np(V), kkt,
                     (it["ascent_sweeps"], it2["ascent_sweeps"], it2["pbcd_iters_u"],
                      it2["pbcd_iters_v"])))
    (fp, Ua, Va, kp, sp), (fc, Ub, Vb, kc, sc) = outs
    print(f"{cfg.name} {hp.precision}: rotation (5 steps) U {du:.1e} V {dv:.1e}, UV^T after 100 "
          f"{duv:.1e}; stages/k* {sp}; "
          f"f {fp[13]:.10e} -> {fp[-1]:.10e}")
    assert sp == sc and sp[1] >= 1                        # the ascent stage ran on both
    assert np.array_equal(fp, fc)                         # objective trace
    assert np.array_equal(Ua, Ub) and np.array_equal(Va, Vb)
    for k in kp:
        assert kp[k] == kc[k], k
    hp.close()
    hc.close()
