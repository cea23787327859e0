"""Seeded synthetic inputs shared by the oracle tests and the GPU product path.

This package holds no eNMF arithmetic: it only draws X (BASELINE.json:7-11)
with a counter-based Philox generator whose host (libsynth_cpu.so) and device
(libsynth_gpu.so) builds give bit-identical bytes for any row range.
"""
import ctypes
import os

import numpy as np

from .configs import (ALL, C1, C2, C3, C4, C5, C6, IMAGE, PLANTED, RATINGS, SPARSE,  # noqa: F401
                      SPECTRO, Config)

_HERE = os.path.dirname(os.path.abspath(__file__))
_cpu = None
_gpu = None


def _load_cpu():
    global _cpu
    if _cpu is None:
        path = os.path.join(_HERE, "libsynth_cpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python __graft_entry__.py build`")
        lib = ctypes.CDLL(path)
        i64, u64, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        lib.synth_x_rows.argtypes = [ctypes.c_int, u64, i64, i64, ctypes.c_int, dbl, dbl,
                                     i64, i64, ctypes.c_void_p, i64]
        lib.synth_x_rows.restype = ctypes.c_int
        lib.synth_x_block.argtypes = [ctypes.c_int, u64, i64, i64, ctypes.c_int, dbl, dbl,
                                      i64, i64, i64, i64, ctypes.c_void_p, i64]
        lib.synth_x_block.restype = ctypes.c_int
        lib.synth_smax.argtypes = [ctypes.c_int, u64, i64, i64, ctypes.c_int]
        lib.synth_smax.restype = dbl
        lib.synth_factor.argtypes = [ctypes.c_int, u64, ctypes.c_int, i64, i64, ctypes.c_int,
                                     ctypes.c_void_p]
        lib.synth_philox.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_csr_rows.argtypes = [u64, i64, i64, ctypes.c_int, dbl, dbl, i64, i64,
                                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, i64]
        lib.synth_csr_rows.restype = i64
        lib.synth_normal.argtypes = [u64, ctypes.c_uint32, u64]
        lib.synth_normal.restype = dbl
        lib.synth_log.argtypes = [dbl]
        lib.synth_log.restype = dbl
        lib.synth_cos2pi.argtypes = [dbl]
        lib.synth_cos2pi.restype = dbl
        _cpu = lib
    return _cpu


def _load_gpu():
    global _gpu
    if _gpu is None:
        path = os.path.join(_HERE, "libsynth_gpu.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python __graft_entry__.py build`")
        lib = ctypes.CDLL(path)
        i64, u64, dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
        lib.synth_gpu_x_rows.argtypes = [ctypes.c_int, u64, i64, i64, ctypes.c_int, dbl, dbl,
                                         i64, i64, ctypes.c_void_p, i64, ctypes.c_void_p]
        lib.synth_gpu_x_rows.restype = ctypes.c_int
        lib.synth_gpu_smax.argtypes = [ctypes.c_int, u64, i64, i64, ctypes.c_int,
                                       ctypes.POINTER(dbl), ctypes.c_void_p]
        lib.synth_gpu_smax.restype = ctypes.c_int
        lib.synth_gpu_csr_rows.argtypes = [u64, i64, i64, ctypes.c_int, dbl, dbl, i64, i64,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_gpu_csr_rows.restype = ctypes.c_int
        _gpu = lib
    return _gpu


def philox(ctr, key):
    lib = _load_cpu()
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib.synth_philox(c, k, o)
    return list(o)


def normal(seed, stream, idx):
    return _load_cpu().synth_normal(seed, stream, idx)


def _smax_cpu(cfg: Config) -> float:
    if cfg.recipe == SPARSE:
        return cfg.density          # SPARSE reads its density from the smax argument
    if cfg.recipe != IMAGE or not cfg.normalised:
        return 0.0
    return _load_cpu().synth_smax(cfg.recipe, cfg.seed, cfg.m, cfg.n, cfg.k)


def x_rows(cfg: Config, row_begin=0, row_count=None, smax=None) -> np.ndarray:
    """Rows [row_begin, row_begin+row_count) of X as a C-contiguous float32 array."""
    if row_count is None:
        row_count = cfg.m - row_begin
    if smax is None:
        smax = _smax_cpu(cfg)
    out = np.empty((row_count, cfg.n), dtype=np.float32)
    rc = _load_cpu().synth_x_rows(cfg.recipe, cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, smax,
                                  row_begin, row_count, out.ctypes.data, cfg.n)
    if rc != 0:
        raise ValueError("synth_x_rows: bad row range")
    return out


def x_block(cfg: Config, r0, rc, c0, cc, smax=None) -> np.ndarray:
    """X[r0:r0+rc, c0:c0+cc], bit-identical to the same entries of x_full(cfg)."""
    if smax is None:
        smax = _smax_cpu(cfg)
    out = np.empty((rc, cc), dtype=np.float32)
    rc_ = _load_cpu().synth_x_block(cfg.recipe, cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, smax,
                                    r0, rc, c0, cc, out.ctypes.data, cc)
    if rc_ != 0:
        raise ValueError("synth_x_block: bad block")
    return out


def x_full(cfg: Config) -> np.ndarray:
    return x_rows(cfg, 0, cfg.m)


def factors(cfg: Config, which: int, begin: int, count: int) -> np.ndarray:
    """Planted row (which=0) / column (which=1) factor rows, float32 (count x k)."""
    out = np.empty((count, cfg.k), dtype=np.float32)
    _load_cpu().synth_factor(cfg.recipe, cfg.seed, which, begin, count, cfg.k, out.ctypes.data)
    return out


def x_rows_device(cfg: Config, row_begin, row_count, out, stream_ptr=0):
    """Fill `out` (a CUDA tensor/pointer, row_count x n, fp32, row-major) on the GPU."""
    lib = _load_gpu()
    ptr = out.data_ptr() if hasattr(out, "data_ptr") else int(out)
    ld = out.stride(0) if hasattr(out, "stride") else cfg.n
    smax = cfg.density if cfg.recipe == SPARSE else 0.0
    if cfg.recipe == IMAGE and cfg.normalised:
        s = ctypes.c_double(0.0)
        rc = lib.synth_gpu_smax(cfg.recipe, cfg.seed, cfg.m, cfg.n, cfg.k, ctypes.byref(s),
                                stream_ptr)
        if rc:
            raise RuntimeError(f"synth_gpu_smax failed: cudaError {rc}")
        smax = s.value
    rc = lib.synth_gpu_x_rows(cfg.recipe, cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, smax,
                              row_begin, row_count, ptr, ld, stream_ptr)
    if rc:
        raise RuntimeError(f"synth_gpu_x_rows failed: cudaError {rc}")


def csr_rows(cfg: Config, row_begin=0, row_count=None):
    """SPARSE recipe rows as CSR numpy arrays (rowptr int64, colidx int32, vals float32),
    bit-identical to the stored entries of x_rows(cfg, ...)."""
    if row_count is None:
        row_count = cfg.m - row_begin
    lib = _load_cpu()
    nnz = lib.synth_csr_rows(cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, cfg.density, row_begin,
                             row_count, None, None, None, 0)
    if nnz < 0:
        raise ValueError("synth_csr_rows: bad row range")
    rowptr = np.empty(row_count + 1, dtype=np.int64)
    colidx = np.empty(max(nnz, 1), dtype=np.int32)
    vals = np.empty(max(nnz, 1), dtype=np.float32)
    lib.synth_csr_rows(cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, cfg.density, row_begin,
                       row_count, rowptr.ctypes.data, colidx.ctypes.data, vals.ctypes.data, nnz)
    return rowptr, colidx[:nnz], vals[:nnz]


def csr_rows_device(cfg: Config, row_begin, row_count, stream_ptr=0):
    """SPARSE recipe rows generated on the GPU: (rowptr int64, colidx int32, vals float32) CUDA
    tensors, bit-identical to csr_rows()."""
    import torch
    lib = _load_gpu()
    counts = torch.empty(max(row_count, 1), dtype=torch.int64, device="cuda")
    rc = lib.synth_gpu_csr_rows(cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, cfg.density, row_begin,
                                row_count, counts.data_ptr(), None, None, None, stream_ptr)
    if rc:
        raise RuntimeError(f"synth_gpu_csr_rows (count) failed: cudaError {rc}")
    rowptr = torch.zeros(row_count + 1, dtype=torch.int64, device="cuda")
    if row_count:
        rowptr[1:] = torch.cumsum(counts[:row_count], 0)
    nnz = int(rowptr[-1].item())
    colidx = torch.empty(max(nnz, 1), dtype=torch.int32, device="cuda")
    vals = torch.empty(max(nnz, 1), dtype=torch.float32, device="cuda")
    rc = lib.synth_gpu_csr_rows(cfg.seed, cfg.m, cfg.n, cfg.k, cfg.noise, cfg.density, row_begin,
                                row_count, None, rowptr.data_ptr(), colidx.data_ptr(),
                                vals.data_ptr(), stream_ptr)
    if rc:
        raise RuntimeError(f"synth_gpu_csr_rows (fill) failed: cudaError {rc}")
    return rowptr, colidx[:nnz], vals[:nnz]
