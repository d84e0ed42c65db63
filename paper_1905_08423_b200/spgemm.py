"""Row-wise SpGEMM C~ = A*P on the device (the two-step's first product).

Mirrors the reference's ``symbolic_ap`` / ``numeric_ap`` (src/spgemm.py:184-234):
the symbolic call gathers the remote rows of P and allocates the structure
of A*P (one row per local row of A, global columns, sorted); the numeric call
fills values in the reference's fold order (bit-identical AP rows).  Backed by
``ptap_spgemm_ap_symbolic`` / ``ptap_spgemm_ap_numeric`` of the C ABI.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .comm import RankContext, gather_remote_rows, refresh_remote_values
from .device import DeviceCsr, DeviceLocalMatrix, DeviceOperands
from .errors import PartitionMismatchError
from .partition import DistMatrix, LocalMatrix
from .sparse import CsrMatrix


def _torch():
    import torch

    return torch


class DeviceAP:
    """C~ = A*P rows of one rank on the device (global columns)."""

    def __init__(self, row_ptr, col, val, ncols, ops, remote):
        self.row_ptr, self.col, self.val, self.ncols = row_ptr, col, val, ncols
        self._ops, self._remote = ops, remote

    def to_host(self) -> CsrMatrix:
        return CsrMatrix(self.row_ptr.numel() - 1, self.ncols, self.row_ptr.cpu().numpy(),
                         self.col.cpu().numpy().astype(np.int64), self.val.cpu().numpy(), check=False)


def _ops_for(a: DistMatrix, p: DistMatrix, ctx: RankContext):
    if a.col_part != p.row_part:
        raise PartitionMismatchError("the column partition of A must equal the row partition of P")
    dev = ctx.device
    ad = a.local if isinstance(a.local, DeviceLocalMatrix) else DeviceLocalMatrix.from_local(a.local, dev)
    pd = p.local if isinstance(p.local, DeviceLocalMatrix) else DeviceLocalMatrix.from_local(p.local, dev)
    cmap = a.local.col_map if isinstance(a.local, LocalMatrix) else a.local.col_map.cpu().numpy().astype(np.int64)
    rr = gather_remote_rows(ctx, cmap, p.row_part, pd)
    m = p.col_part.nglobal
    c_lo, c_hi = p.col_part.owned_range(ctx.rank)
    remote = DeviceCsr(rr.source_cols.size, m, rr.row_ptr.to(dev), rr.col.to(dev), rr.val.to(dev))
    return DeviceOperands(ad, pd, m, c_lo, c_hi, remote), rr


def symbolic_ap(a: DistMatrix, p: DistMatrix, ctx: RankContext) -> DeviceAP:
    torch = _torch()
    L = _lib.load()
    ops, rr = _ops_for(a, p, ctx)
    st = ops.struct()
    nnz = ctypes.c_int64()
    rp_ptr, col_ptr = ctypes.c_void_p(), ctypes.c_void_p()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.ptap_spgemm_ap_symbolic(ctypes.byref(st), ctypes.byref(nnz), ctypes.byref(rp_ptr),
                                         ctypes.byref(col_ptr), stream), "symbolic_ap")
    n = ops.a.nrows
    # copy into torch-owned buffers and release the library allocations
    from .tripleproduct import _dev_view
    rp = _dev_view(rp_ptr.value, n + 1, "int64", ctx.device).clone()
    col = _dev_view(col_ptr.value, nnz.value, "int32", ctx.device).clone()
    torch.cuda.current_stream().synchronize()
    L.ptap_device_free(rp_ptr, stream)
    L.ptap_device_free(col_ptr, stream)
    val = torch.zeros(nnz.value, dtype=torch.float64, device=ctx.device)
    return DeviceAP(rp, col, val, p.col_part.nglobal, ops, rr)


def numeric_ap(a: DistMatrix, p: DistMatrix, c: DeviceAP, ctx: RankContext) -> DeviceAP:
    """Values of C~ = A*P into the symbolic structure (reference numeric_ap,
    src/spgemm.py:205-234): the operands' current values -- host operands
    are uploaded, device operands are used as given -- and, at several
    ranks, the gathered rows of P refreshed first (values only,
    update_remote_rows_numeric, src/spgemm.py:224-225)."""
    torch = _torch()
    L = _lib.load()
    ops = c._ops
    if isinstance(a.local, LocalMatrix):
        ops.a.refresh_values(a.local)
    else:
        ops.a = a.local
    if isinstance(p.local, LocalMatrix):
        ops.p.refresh_values(p.local)
    else:
        ops.p = p.local
    if ctx.nranks > 1:
        refresh_remote_values(ctx, c._remote, ops.p)
        ops.p_remote.val = c._remote.val
    st = ops.struct()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(L.ptap_spgemm_ap_numeric(ctypes.byref(st), ctypes.c_void_p(c.row_ptr.data_ptr()),
                                        ctypes.c_void_p(c.col.data_ptr() if c.col.numel() else 0),
                                        ctypes.c_void_p(c.val.data_ptr() if c.val.numel() else 0), stream),
               "numeric_ap")
    return c
