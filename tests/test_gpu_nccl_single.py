"""The NCCL code path on real hardware, at one rank.

gpurun gives one GPU per call and NCCL refuses two ranks on one device, so the multi-rank
tests (test_gpu_multirank.py) route their collectives through the host.  A handle given an
ncclUniqueId at world_size == 1 runs the sharded code path with a one-rank communicator
(include/enmf.h, enmf_problem_t.nccl_unique_id): dlopen of the NCCL torch loaded,
ncclCommInitRank, the in-place ncclAllReduce of the Grams / scalars / PBCD partials, the
V-slice layout with 128-row-aligned slices, the sliced pass 2 with its ncclReduce per slice on
the communication stream, the in-place all-gather of the V slices, and the init collectives.
At one rank every collective is an identity, so the factors, the objective trace and the
init's singular values must equal the plain single-rank handle's bitwise."""
import numpy as np
import pytest

import synth
from tests.gpu_common import to_dev

pytestmark = pytest.mark.gpu

FP64, TC = 1, 2


def _run(cfg, prec, uid, sweeps):
    import torch
    import paper_2605_19325_b200 as E
    X = to_dev(synth.x_full(cfg))
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=prec, nccl_id=uid)
    U = torch.empty(cfg.m, cfg.r, device="cuda")
    V = torch.empty(cfg.n, cfg.r, device="cuda")
    info = h.init(X, U, V)
    f, it = h.iterate(U, V, sweeps)
    kkt = h.kkt(U, V)
    torch.cuda.synchronize()
    out = (np.array(info["sigma"]), np.array(f), U.cpu().numpy(), V.cpu().numpy(), kkt,
           it["ascent_sweeps"], h.precision)
    h.close()
    return out


@pytest.mark.parametrize("prec", [FP64, TC], ids=["fp64", "tc"])
@pytest.mark.parametrize("cfg", [synth.C1, synth.C5.scaled(700, 650, 128, 128, name="C5-700x650"),
                                 synth.C3.scaled(300, 1100, 32, 32, name="C3-300x1100")],
                         ids=["C1", "C5-700x650", "C3-300x1100"])
def test_single_rank_nccl_path_bitwise(cfg, prec):
    import paper_2605_19325_b200 as E
    uid = E.nccl_unique_id()
    assert len(uid) == 128
    plain = _run(cfg, prec, None, 14)
    comm = _run(cfg, prec, uid, 14)
    assert plain[6] == comm[6]
    assert plain[5] == comm[5] and plain[5] >= 1          # the ascent stage ran on both
    print(f"{cfg.name} {plain[6]}: {plain[5]} ascent sweeps, f {plain[1][-1]:.10e}")
    assert np.array_equal(plain[0], comm[0])               # sigma of the init
    assert np.array_equal(plain[1], comm[1])               # objective trace
    assert np.array_equal(plain[2], comm[2])               # U
    assert np.array_equal(plain[3], comm[3])               # V
    for k in plain[4]:
        assert plain[4][k] == comm[4][k], k
