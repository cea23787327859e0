"""Heavy-tailed X on the tensor-core path (advisor, round 1): the precision policy and the
quantisation error bound the policy rests on.

The tensor-core X passes round every operand entry to the 2^-15 grid of a scale group whose
maximum lies in [63, 126) (per row of X for P = X V, per column of X for Q = X^T U, per column
of the factor), i.e. |dx| <= 2^-16 / 63 max_group|x| ~ 2^-22 max_group|x|, and
drop three digit products (weight <= 2^-23, unbiased).  On data with a wide dynamic range the
error is therefore bounded relative to the group maxima, not to each entry: for P

    |P_ik - (X V)_ik| <= 2^-22 ( max_j|x_ij| sum_j |v_jk| + max_j|v_jk| sum_j |x_ij| )

(the two operand roundings; the dropped products add an unbiased ~2^-23 max|x| max|v| sqrt(K),
below that at these shapes -- an exact numpy emulation of the digit scheme reaches 0.20 of the
bound on both cases), and the same with rows and columns exchanged for Q.  The entrywise error
relative to |X||V| then reaches ~2e-4 (emulation; planted data: ~7e-8), far from the 2e-6 of
test_tc_contractions_match_oracle: this is why ENMF_PREC_AUTO keeps such X on the fp64 path
(max|X| > 64 rms(X), enmf_capi.cu)."""
import numpy as np
import pytest

import oracle
from tests.gpu_common import rel_fro, to_dev, to_np

pytestmark = pytest.mark.gpu

FP64, TC = 1, 2


def heavy_x(m, n, sigma, seed):
    """Log-normal entries (sigma in log space), a fifth of them zero: a count / tf-idf-like
    dynamic range."""
    g = np.random.default_rng(seed)
    X = np.exp(sigma * g.standard_normal((m, n))) * (g.random((m, n)) >= 0.2)
    return X.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("shape", [(700, 650, 64), (257, 1031, 33)], ids=["700x650r64", "257x1031r33"])
def test_tc_contractions_heavy_tail_within_group_bound(shape):
    import paper_2605_19325_b200 as E
    m, n, r = shape
    X = heavy_x(m, n, 2.5, 11)
    g = np.random.default_rng(12)
    # factors with a range of their own: half of each column ~1e-3 of the rest
    U0 = g.random((m, r)) * np.where(g.random((m, r)) < 0.5, 1e-3, 1.0)
    V0 = g.random((n, r)) * np.where(g.random((n, r)) < 0.5, 1e-3, 1.0)
    U0 = U0.astype(np.float32).astype(np.float64)
    V0 = V0.astype(np.float32).astype(np.float64)
    h = E.Enmf(m, n, r, precision=TC)
    h.set_data(to_dev(X))
    assert h.precision.startswith("tc")
    P, Q = h.cross_terms(to_dev(U0), to_dev(V0))
    P, Q = to_np(P), to_np(Q)
    Pr, Qr = oracle.xv(X, V0), oracle.xtu(X, U0)
    Xa = np.abs(X)
    bp = 2.0 ** -22 * (Xa.max(1)[:, None] * np.abs(V0).sum(0)[None, :]
                       + np.abs(V0).max(0)[None, :] * Xa.sum(1)[:, None])
    bq = 2.0 ** -22 * (Xa.max(0)[:, None] * np.abs(U0).sum(0)[None, :]
                       + np.abs(U0).max(0)[None, :] * Xa.sum(0)[:, None])
    rp = np.abs(P - Pr) / bp
    rq = np.abs(Q - Qr) / bq
    ent = max((np.abs(P - Pr) / (Xa @ np.abs(V0))).max(), (np.abs(Q - Qr) / (Xa.T @ np.abs(U0))).max())
    print(f"heavy {m}x{n} r{r}: max|X|/rms {Xa.max() / np.sqrt((Xa ** 2).mean()):.0f}; error / "
          f"group bound P {rp.max():.3f} Q {rq.max():.3f}; entrywise rel {ent:.2e}; "
          f"normwise P {rel_fro(P, Pr):.2e} Q {rel_fro(Q, Qr):.2e}")
    assert rp.max() <= 1.0 and rq.max() <= 1.0


def test_auto_keeps_heavy_tailed_x_on_fp64():
    """ENMF_PREC_AUTO at a size where the tensor-core path is chosen for the planted recipe
    (m n >= 2.5e8): the same shape with log-normal entries stays on fp64."""
    import torch
    import paper_2605_19325_b200 as E
    m, n, r = 20000, 12500, 32
    gen = torch.Generator(device="cuda")
    gen.manual_seed(5)
    X = torch.rand(m, n, device="cuda", generator=gen)
    h = E.Enmf(m, n, r)
    h.set_data(X)
    assert h.precision.startswith("tc"), h.precision
    del h
    X.normal_(generator=gen).mul_(2.5).exp_()
    h = E.Enmf(m, n, r)
    h.set_data(X)
    assert h.precision.startswith("fp64"), h.precision
    del h, X
    torch.cuda.empty_cache()
