"""Worker of tests/test_gpu_multirank.py (a module so that spawned processes can import it)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ascent_point(cfg):
    """A deterministic infeasible fp32 point and its lift constants 1.001 |min| / L (R9)."""
    import numpy as np
    g = np.random.default_rng(7)
    U0 = (g.random((cfg.m, cfg.r)) - 0.15).astype(np.float32)
    V0 = (g.random((cfg.n, cfg.r)) - 0.15).astype(np.float32)
    lam = lambda A: 1.001 * abs(min(float(A.min()), 0.0)) / 10.0   # noqa: E731
    return U0, V0, lam(U0), lam(V0)


def load_x(cfg, begin, count):
    """This rank's rows of X on the device: a dense tensor, or CSR tensors (SPARSE recipe)."""
    import torch

    import synth
    if cfg.recipe == synth.SPARSE:
        rp, ci, v = synth.csr_rows(cfg, begin, count)
        return tuple(torch.from_numpy(a).cuda() for a in (rp, ci, v))
    X = torch.empty(count, cfg.n, device="cuda")
    synth.x_rows_device(cfg, begin, count, X, torch.cuda.current_stream().cuda_stream)
    return X


def bind(h, X):
    if isinstance(X, tuple):
        h.set_data_csr(*X)
    else:
        h.set_data(X)


def init(h, X, U, V):
    """Alg. 3 lines 331-333 (enmf_init, or set_data_csr + svd + rotate for a sparse X)."""
    if not isinstance(X, tuple):
        return h.init(X, U, V)
    bind(h, X)
    sig = h.svd(U, V)
    info = h.rotate(U, V)
    info["sigma"] = sig
    return info


def run(rank, world, port, cfg_args, prec, mode, out_q):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2605_19325_b200 as E
    import synth
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                                world_size=world)
        cfg = synth.ALL[cfg_args[0]].scaled(*cfg_args[1:]) if len(cfg_args) > 1 else \
            synth.ALL[cfg_args[0]]
        begin, count = E.row_partition(cfg.m, world, rank)
        X = load_x(cfg, begin, count)
        h = E.Enmf(cfg.m, cfg.n, cfg.r, row_begin=begin, row_count=count, world_size=world,
                   rank=rank, precision=prec)
        rop = {"sum": dist.ReduceOp.SUM, "min": dist.ReduceOp.MIN, "max": dist.ReduceOp.MAX}

        def ar(buf, op):
            t = torch.from_numpy(buf)
            dist.all_reduce(t, op=rop[op])

        h.set_host_allreduce(ar)
        res = {"rank": rank, "begin": begin, "count": count}
        if mode == "init":
            U = torch.empty(count, cfg.r, device="cuda")
            V = torch.empty(cfg.n, cfg.r, device="cuda")
            info = init(h, X, U, V)
            f, it = h.iterate(U, V, 12)
            res.update(sigma=np.array(info["sigma"]), f=f, it=it)
        elif mode == "ascent":                  # lift + PBCD sweeps from a shared point
            U0, V0, lu, lv = ascent_point(cfg)
            bind(h, X)
            U = torch.from_numpy(U0[begin:begin + count]).cuda()
            V = torch.from_numpy(V0).cuda()
            h.set_stage(0, lu, lv)
            f, it = h.iterate(U, V, 3)
            res.update(f=f, it=it)
        else:                                   # HALS sweeps from a shared feasible point
            g = np.random.default_rng(5)
            U0 = g.random((cfg.m, cfg.r)).astype(np.float32)
            V0 = g.random((cfg.n, cfg.r)).astype(np.float32)
            bind(h, X)
            U = torch.from_numpy(U0[begin:begin + count]).cuda()
            V = torch.from_numpy(V0).cuda()
            h.set_stage(1)
            f, it = h.iterate(U, V, 5)
            res.update(f=f, it=it, kkt=h.kkt(U, V), fx=h.objective(U, V, exact=True))
        res.update(U=U.cpu().numpy(), V=V.cpu().numpy())
        out_q.put(res)
        dist.destroy_process_group()
    except Exception as e:                      # noqa: BLE001 -- reported to the parent
        import traceback
        out_q.put({"rank": rank, "error": f"{e}\n{traceback.format_exc()}"})
