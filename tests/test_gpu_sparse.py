"""Sparse X (the paper's sparse Reuters experiment): the
CSR path (enmf_set_data_csr, fp64-accumulating SpMM X passes) against the fp64 oracle run on
the same X densified.  The oracle needs no sparse code: P = X V and Q = X^T U of a matrix
with stored zeros are the same numbers.  Inputs: the SPARSE recipe (planted product sampled
at a density, synth_core.h, reading R27) at sizes the oracle finishes in seconds, with ragged
row lengths and empty rows."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import rel_fro, rotated_point, to_dev, to_np

pytestmark = pytest.mark.gpu

FP64, AUTO = 1, 0
CASES = [
    synth.C6.scaled(300, 220, 12, 12, density=0.05, name="sparse-300x220-r12"),
    synth.C6.scaled(700, 650, 100, 100, density=0.02, name="sparse-700x650-r100"),
    synth.C6.scaled(257, 131, 33, 33, density=0.004, name="sparse-ragged-empty-rows"),
]
IDS = [c.name for c in CASES]
PRECS = [(FP64, "rows-fp64"), (AUTO, "rows-tc")]


def bind(cfg, precision=AUTO):
    import torch
    import paper_2605_19325_b200 as E
    rp, ci, v = synth.csr_rows(cfg)
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=precision)
    dev = (torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(), torch.from_numpy(v).cuda())
    h.set_data_csr(*dev)
    return h, synth.x_full(cfg), dev


def test_csr_device_generator_matches_host():
    cfg = CASES[1]
    rp, ci, v = synth.csr_rows(cfg, 100, 400)
    drp, dci, dv = synth.csr_rows_device(cfg, 100, 400)
    assert np.array_equal(drp.cpu().numpy(), rp)
    assert np.array_equal(dci.cpu().numpy(), ci) and np.array_equal(dv.cpu().numpy(), v)


@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_sparse_contractions_and_objective(cfg):
    """P = X V, Q = X^T U (CSR and CSC SpMM, fp64 accumulation of the fp32 products) entry by
    entry, and both objective forms, against the oracle on the densified X.  Only the
    summation order differs: bound 1e-12 of |X||F| per entry."""
    h, X, _ = bind(cfg)
    assert h.precision.startswith("csr")
    g = np.random.default_rng(2)
    U0 = g.random((cfg.m, cfg.r)).astype(np.float32).astype(np.float64)
    V0 = g.random((cfg.n, cfg.r)).astype(np.float32).astype(np.float64)
    P, Q = h.cross_terms(to_dev(U0), to_dev(V0))
    P, Q = to_np(P), to_np(Q)
    Xa = np.abs(X.astype(np.float64))
    ep = np.abs(P - oracle.xv(X, V0)) / np.maximum(Xa @ np.abs(V0), 1e-300)
    eq = np.abs(Q - oracle.xtu(X, U0)) / np.maximum(Xa.T @ np.abs(U0), 1e-300)
    print(f"{cfg.name}: nnz {int((X != 0).sum())}, P max {ep.max():.1e}, Q max {eq.max():.1e}")
    assert ep.max() < 1e-12 and eq.max() < 1e-12
    f_d = oracle.frob2_direct(X, U0, V0)
    for exact in (False, True):
        f = h.objective(to_dev(U0), to_dev(V0), exact=exact)
        assert abs(f - f_d) <= 1e-10 * f_d, (exact, f, f_d)


@pytest.mark.parametrize("prec,pid", PRECS, ids=[p[1] for p in PRECS])
@pytest.mark.parametrize("cfg", CASES, ids=IDS)
def test_sparse_svd_and_hals_sweep(cfg, prec, pid):
    """The randomised SVD (Alg. 3) through the SpMM passes against the same
    algorithm on the densified X through the dense fp64 passes (same seeded Omega; the
    range finder itself is pinned to the oracle's converged SVD by the dense tests -- a
    sampled planted product has no spectral gap, so q = 2 is not converged here): sigma and
    the balanced factors within 1e-8.  Then one HALS sweep from a shared feasible point
    against the oracle (BASELINE's 1e-5 per factor)."""
    import paper_2605_19325_b200 as E
    h, X, _ = bind(cfg, prec)
    U = to_dev(np.zeros((cfg.m, cfg.r)))
    V = to_dev(np.zeros((cfg.n, cfg.r)))
    sig = h.svd(U, V)
    hd = E.Enmf(cfg.m, cfg.n, cfg.r, precision=FP64)
    hd.set_data(to_dev(X))
    Ud = to_dev(np.zeros((cfg.m, cfg.r)))
    Vd = to_dev(np.zeros((cfg.n, cfg.r)))
    sig_d = hd.svd(Ud, Vd)
    print(f"{cfg.name}: sigma rel {np.max(np.abs(sig - sig_d) / sig_d[0]):.1e}, "
          f"U {rel_fro(to_np(U), to_np(Ud)):.1e}")
    assert np.max(np.abs(sig - sig_d)) <= 1e-8 * sig_d[0]
    assert rel_fro(to_np(U), to_np(Ud)) < 1e-6 and rel_fro(to_np(V), to_np(Vd)) < 1e-6
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U0, V0 = np.abs(U0), np.abs(V0)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    h.iterate(U, V, 1)
    Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1),
                                oracle.options(cfg.r, round_f32=1))
    eu, ev = rel_fro(to_np(U), Uo), rel_fro(to_np(V), Vo)
    print(f"{cfg.name} {h.precision}: HALS sweep U {eu:.2e} V {ev:.2e}")
    assert eu < 1e-5 and ev < 1e-5


@pytest.mark.parametrize("prec,pid", PRECS, ids=[p[1] for p in PRECS])
@pytest.mark.parametrize("cfg", [CASES[0], CASES[2]], ids=[IDS[0], IDS[2]])
def test_sparse_ascent_then_hals_trajectory(cfg, prec, pid):
    """20 sweeps from the oracle's rotated point (ascent stage, then HALS) in the well-posed
    form of tests/test_gpu_shadow.py: every ascent sweep repeated by the oracle from the GPU's
    own state with the GPU's k* (per-update 1e-5 on the well-conditioned rows, R20 flips
    counted, k* against the oracle's own eps rule), and from the GPU's first feasible point on
    the oracle's OWN HALS trajectory against the GPU's direct objective at 1e-4 per sweep."""
    from tests.test_gpu_shadow import FP64 as S_FP64, TC as S_TC, Shadow, oracle_block, \
        shadow_sweep
    h, X, _ = bind(cfg, prec)
    U0, V0, lu, lv = rotated_point(X, cfg.r)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(0, lu, lv)
    # arithmetic precision of the block updates: fp64 rows, or the tensor-core rows (2^-22)
    pk = S_FP64 if prec == FP64 else (S_TC if "tc" in h.precision else S_FP64)
    sh = Shadow(cfg.m, cfg.n, cfg.r)
    Ut, Vt = U0, V0
    Uo = Vo = None
    e_hals, n_asc, n_hals = 0.0, 0, 0
    for t in range(20):
        _, info = h.iterate(U, V, 1)
        Un, Vn = to_np(U), to_np(V)
        fg = h.objective(U, V, exact=True)
        if info["ascent_sweeps"] == 1:
            n_asc += 1
            shadow_sweep(sh, X, Ut, Vt, Un, Vn, info, lu, lv, pk, t)
        else:
            n_hals += 1
            if Uo is None:                       # the oracle's HALS trajectory starts here
                Uo, Vo = Ut, Vt
            Uo = oracle_block(X, Uo, Vo, True, False)[0]
            Vo = oracle_block(X, Vo, Uo, False, False)[0]
            fo = oracle.frob2_direct(X, Uo, Vo)
            e_hals = max(e_hals, abs(fg - fo) / fo)
        Ut, Vt = Un, Vn
    tol_margin = 1e-6 if pk == S_FP64 else 1e-3
    print(f"{cfg.name} {h.precision}: {n_asc} ascent (per-update U {sh.eu:.2e} V {sh.ev:.2e}, "
          f"flips {sh.flips}, ill-posed rows {sh.ill}, k* mismatches {sh.kmis}) + {n_hals} HALS "
          f"sweeps (oracle's own trajectory: direct f {e_hals:.2e})")
    assert n_hals >= 5
    assert sh.eu < 1e-5 and sh.ev < 1e-5
    assert sh.flips <= sh.limit_flips
    assert all(m[4] < tol_margin for m in sh.kmis), sh.kmis
    assert e_hals < 1e-4


def test_sparse_input_checks():
    import torch
    import paper_2605_19325_b200 as E
    cfg = CASES[0]
    rp, ci, v = synth.csr_rows(cfg)
    h = E.Enmf(cfg.m, cfg.n, cfg.r)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()   # noqa: E731
    bad = ci.copy()
    r0 = int(np.argmax(np.diff(rp) >= 2))            # a row with two entries: swap them
    bad[rp[r0]], bad[rp[r0] + 1] = bad[rp[r0] + 1], bad[rp[r0]]
    with pytest.raises(RuntimeError, match="-1"):
        h.set_data_csr(dev(rp), dev(bad), dev(v))
    neg = v.copy()
    neg[3] = -1.0
    with pytest.raises(RuntimeError, match="-3"):
        h.set_data_csr(dev(rp), dev(ci), dev(neg))
    # advisor (round 1): nnz larger than row_ptr[rows], and a rebased slice of a global CSR
    # (row_ptr[0] != 0) -- both rejected instead of sorting stray entries into the CSC
    ci1 = np.concatenate([ci, ci[:1]])
    v1 = np.concatenate([v, v[:1]])
    with pytest.raises(RuntimeError, match="-1"):
        h.set_data_csr(dev(rp), dev(ci1), dev(v1))
    with pytest.raises(RuntimeError, match="-1"):
        h.set_data_csr(dev(rp + 1), dev(ci1), dev(v1))
    h.set_data_csr(dev(rp), dev(ci), dev(v))        # and a valid bind afterwards works
    assert h.precision.startswith("csr")


def test_tc_hals_ill_conditioned_gram_hands_over_to_fp64():
    """The ragged sparse case is rank deficient: the rotated factors keep columns of size
    ~1e-36 that are still coupled to the others, so G_jj is ~2^-200 of its column sum and the
    tensor-core HALS (u on a per-row digit grid) would lose the update of u_j entirely.  The
    G-digit pass flags such a G and the SIMT fp64 kernel takes the sweep: one HALS sweep on the
    DENSE tensor-core path within BASELINE's 1e-5 of the oracle, no fallback rows."""
    import paper_2605_19325_b200 as E
    cfg = CASES[2]
    X = synth.x_full(cfg)
    h = E.Enmf(cfg.m, cfg.n, cfg.r, precision=2)
    h.set_data(to_dev(X))
    assert h.precision.startswith("tc")
    U0, V0, _, _ = rotated_point(X, cfg.r)
    U0, V0 = np.abs(U0), np.abs(V0)
    U, V = to_dev(U0), to_dev(V0)
    h.set_stage(1)
    _, info = h.iterate(U, V, 1)
    Uo, Vo, _, _ = oracle.sweep(X, U0, V0, oracle.SweepState(stage=1),
                                oracle.options(cfg.r, round_f32=1))
    eu, ev = rel_fro(to_np(U), Uo), rel_fro(to_np(V), Vo)
    print(f"ill-conditioned G, {h.precision}: U {eu:.2e} V {ev:.2e}, fallback rows "
          f"{info['hals_fallback_rows']}")
    assert eu < 1e-5 and ev < 1e-5


def _sparse_exact(m, n, r, k, seed):
    """X = A B^T with A (m x r), B (n x r) nonnegative and k nonzeros per row, so X is sparse
    (density ~ k^2 / r) and has rank r exactly: the randomised range finder's q = 2 power
    iterations then capture the range to rounding and the result is the converged truncated
    SVD, which the oracle computes by its own algorithm (block subspace iteration)."""
    g = np.random.default_rng(seed)

    def factor(rows):
        F = np.zeros((rows, r))
        for i in range(rows):
            F[i, g.choice(r, k, replace=False)] = 0.5 + g.random(k)
        return F

    X = (factor(m) @ factor(n).T).astype(np.float32)
    X[np.arange(0, m, 37)] = 0.0                       # a few empty rows
    rp = np.zeros(m + 1, np.int64)
    rows, cols = np.nonzero(X)
    np.add.at(rp, rows + 1, 1)
    return X.astype(np.float64), np.cumsum(rp), cols.astype(np.int32), X[rows, cols]


@pytest.mark.parametrize("shape", [(400, 350, 12, 2), (700, 650, 40, 2)],
                         ids=["400x350-r12", "700x650-r40"])
def test_sparse_svd_matches_oracle_on_exact_low_rank(shape):
    """The SpMM randomised SVD against the ORACLE's truncated SVD (not the dense GPU path):
    on an exactly rank-r sparse X (more rows removed, rank <= r) sigma within 1e-9 of sigma_1
    and the balanced factors within 1e-7 (the sign rule R5 fixes the singular vectors; a
    repeated sigma would not, the seeded input has none)."""
    import torch
    import paper_2605_19325_b200 as E
    m, n, r, k = shape
    X, rp, ci, v = _sparse_exact(m, n, r, k, 11)
    h = E.Enmf(m, n, r, precision=FP64)
    h.set_data_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                   torch.from_numpy(v.astype(np.float32)).cuda())
    assert h.precision.startswith("csr")
    U = to_dev(np.zeros((m, r)))
    V = to_dev(np.zeros((n, r)))
    sig = np.asarray(h.svd(U, V))
    Uo, Vo, so, _ = oracle.truncated_svd(X, r)
    gap = np.min(np.abs(np.diff(so))) / so[0]
    print(f"sparse exact rank {r}: density {len(v) / (m * n):.3f}, min sigma gap {gap:.1e}, "
          f"sigma {np.max(np.abs(sig - so)) / so[0]:.1e}, U {rel_fro(to_np(U), Uo):.1e}, "
          f"V {rel_fro(to_np(V), Vo):.1e}")
    assert gap > 1e-4
    assert np.max(np.abs(sig - so)) <= 1e-9 * so[0]
    assert rel_fro(to_np(U), Uo) < 1e-7 and rel_fro(to_np(V), Vo) < 1e-7
