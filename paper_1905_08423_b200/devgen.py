"""Device-side construction of the BASELINE operands (config 1-3) as
row-block ``DistMatrix`` objects holding ``DeviceLocalMatrix`` locals.

The CSR rows are produced by the CUDA generators (csrc/ptap_gen.cu, bit-equal
to problems.py) for the rank's row block with global columns, then split into
the diag/offdiag blocks of the paper's MPI layout (src/partition.py:123-154).
The split is one-time setup plumbing and uses torch ops.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .device import DeviceCsr, DeviceLocalMatrix
from .partition import DistMatrix, make_partition
from .problems import CONFIGS


def _torch():
    import torch

    return torch


def _stream():
    return ctypes.c_void_p(_torch().cuda.current_stream().cuda_stream)


def gen_stencil_rows(n: int, points: int, kind: int, seed: int, lo: int, hi: int, device):
    torch = _torch()
    L = _lib.load()
    nr = hi - lo
    rp = torch.zeros(nr + 1, dtype=torch.int64, device=device)
    nnz = ctypes.c_int64()
    _lib.check(L.ptap_gen_stencil_rowptr(points, n, lo, hi, ctypes.c_void_p(rp.data_ptr()), ctypes.byref(nnz),
                                         _stream()), "gen rowptr")
    col = torch.empty(nnz.value, dtype=torch.int32, device=device)
    val = torch.empty(nnz.value, dtype=torch.float64, device=device)
    _lib.check(L.ptap_gen_stencil_fill(points, kind, seed, n, lo, hi, ctypes.c_void_p(rp.data_ptr()),
                                       ctypes.c_void_p(col.data_ptr()), ctypes.c_void_p(val.data_ptr()), _stream()),
               "gen fill")
    return rp, col, val


def gen_trilinear_rows(nc: int, lo: int, hi: int, device):
    torch = _torch()
    L = _lib.load()
    nr = hi - lo
    rp = torch.zeros(nr + 1, dtype=torch.int64, device=device)
    nnz = ctypes.c_int64()
    _lib.check(L.ptap_gen_trilinear_rowptr(nc, lo, hi, ctypes.c_void_p(rp.data_ptr()), ctypes.byref(nnz), _stream()),
               "gen rowptr")
    col = torch.empty(nnz.value, dtype=torch.int32, device=device)
    val = torch.empty(nnz.value, dtype=torch.float64, device=device)
    _lib.check(L.ptap_gen_trilinear_fill(nc, lo, hi, ctypes.c_void_p(rp.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                                         ctypes.c_void_p(val.data_ptr()), _stream()), "gen fill")
    return rp, col, val


def split_rows_device(rp, col, val, row_lo, row_hi, col_lo, col_hi, ncols_global) -> DeviceLocalMatrix:
    """Rows with global columns -> diag (local columns) + offdiag (compact)."""
    torch = _torch()
    dev = rp.device
    nr = row_hi - row_lo
    if col.numel() == 0 or (int(col.min().item()) >= col_lo and int(col.max().item()) < col_hi):
        diag = DeviceCsr(nr, col_hi - col_lo, rp, (col - col_lo).to(torch.int32) if col_lo else col, val)
        return DeviceLocalMatrix(row_lo, row_hi, col_lo, col_hi, diag, DeviceCsr.empty(nr, 0, dev),
                                 torch.zeros(0, dtype=torch.int32, device=dev))
    rowid = torch.repeat_interleave(torch.arange(nr, device=dev), rp[1:] - rp[:-1])
    inside = (col >= col_lo) & (col < col_hi)

    def block(mask, cols, ncols):
        cnt = torch.bincount(rowid[mask], minlength=nr)
        brp = torch.zeros(nr + 1, dtype=torch.int64, device=dev)
        torch.cumsum(cnt, 0, out=brp[1:])
        return DeviceCsr(nr, ncols, brp, cols.to(torch.int32), val[mask])

    diag = block(inside, col[inside] - col_lo, col_hi - col_lo)
    ocol = col[~inside].to(torch.int64)
    col_map = torch.unique(ocol)
    off = block(~inside, torch.searchsorted(col_map, ocol), col_map.numel())
    return DeviceLocalMatrix(row_lo, row_hi, col_lo, col_hi, diag, off, col_map.to(torch.int32))


def config_dist(name: str, nranks: int, rank: int, device, n_fine: int | None = None):
    """(A, P) DistMatrix pair of config ``name`` for one rank (z-slab rows)."""
    spec = CONFIGS[name]
    n = spec.n_fine if n_fine is None else n_fine
    nc = n // 2
    N, M = n ** 3, nc ** 3
    row_part = make_partition(N, nranks)
    col_part = make_partition(M, nranks)
    lo, hi = row_part.owned_range(rank)
    clo, chi = col_part.owned_range(rank)
    kind = 0 if spec.points == 7 else 1
    arp, acol, aval = gen_stencil_rows(n, spec.points, kind, spec.seed, lo, hi, device)
    prp, pcol, pval = gen_trilinear_rows(nc, lo, hi, device)
    a_loc = split_rows_device(arp, acol, aval, lo, hi, lo, hi, N)
    del acol, aval
    p_loc = split_rows_device(prp, pcol, pval, lo, hi, clo, chi, M)
    return (DistMatrix(row_part, row_part, rank, a_loc), DistMatrix(row_part, col_part, rank, p_loc))
