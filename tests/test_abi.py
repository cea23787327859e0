"""CPU-only checks of the C-ABI boundary: the library loads, exports every function that
include/enmf.h declares, and the host-side helpers behave (no GPU compute here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "enmf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(enmf_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2605_19325_b200", "libenmf.so"))
    names = declared_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name


def test_binding_covers_the_header():
    import paper_2605_19325_b200 as E
    assert set(declared_functions()) <= set(E.EXPORTED)


def test_status_strings_and_defaults():
    import paper_2605_19325_b200 as E
    assert E._lib.enmf_status_string(-3) == b"X has a negative entry"
    o = E.default_options()
    assert (o.oversample, o.power_iters, o.admm_iters, o.lift_steps, o.pbcd_max_iter) == \
        (10, 2, 100, 10, 50)
    assert o.pbcd_eps == 1e-2 and o.admm_rho == 0.0
    with pytest.raises(TypeError):
        E.default_options(bogus=1)


def test_create_rejects_bad_shapes_without_gpu():
    """Shape validation happens before any device work (ENMF_ERR_SHAPE = -2)."""
    import paper_2605_19325_b200 as E
    prob = E.Problem(10, 5, 6, 0, 10, 1, 0, None, None)
    h = E._H()
    assert E._lib.enmf_create(ctypes.byref(prob), None, ctypes.byref(h)) == -2
    prob = E.Problem(10, 5, 2, 3, 10, 1, 0, None, None)     # row range outside m
    assert E._lib.enmf_create(ctypes.byref(prob), None, ctypes.byref(h)) == -2
    prob = E.Problem(10, 5, 2, 0, 5, 2, 2, None, None)      # rank outside the world
    assert E._lib.enmf_create(ctypes.byref(prob), None, ctypes.byref(h)) == -1
    # (world 2 without an NCCL id is valid: collectives then go through
    # enmf_set_host_allreduce -- tests/test_gpu_multirank.py)


@pytest.mark.parametrize("m,world", [(200000, 8), (10, 3), (7, 7), (5, 1)])
def test_row_partition_covers_rows_once(m, world):
    import paper_2605_19325_b200 as E
    spans = [E.row_partition(m, world, s) for s in range(world)]
    assert spans[0][0] == 0
    for (b0, c0), (b1, _) in zip(spans, spans[1:]):
        assert b0 + c0 == b1
    assert sum(c for _, c in spans) == m
    assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
