"""Device images of the CSR blocks (torch tensors as raw device buffers).

Layout in HBM: row offsets int64, column indices int32, values
fp64.  A rank's operands are the device image of its ``LocalMatrix`` of A and
of P (diag block, off-diagonal block, column map) plus the gathered remote
rows of P; ``DeviceOperands.struct()`` packs them into the C-ABI struct.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .partition import LocalMatrix
from .sparse import CsrMatrix


def _torch():
    import torch

    return torch


def _ptr(t) -> int | None:
    return None if t is None or t.numel() == 0 else int(t.data_ptr())


class DeviceCsr:
    """One CSR block on the device."""

    __slots__ = ("nrows", "ncols", "row_ptr", "col", "val")

    def __init__(self, nrows, ncols, row_ptr, col, val=None):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.row_ptr, self.col, self.val = row_ptr, col, val

    @property
    def nnz(self) -> int:
        return int(self.col.numel())

    @property
    def nbytes(self) -> int:
        n = self.row_ptr.numel() * 8 + self.col.numel() * 4
        return n + (0 if self.val is None else self.val.numel() * 8)

    @classmethod
    def from_host(cls, m: CsrMatrix, device, with_values=True) -> "DeviceCsr":
        torch = _torch()
        rp = torch.from_numpy(np.ascontiguousarray(m.row_offsets, np.int64)).to(device)
        col = torch.from_numpy(np.ascontiguousarray(m.col_indices, np.int32)).to(device)
        val = None
        if with_values and m.values is not None:
            val = torch.from_numpy(np.ascontiguousarray(m.values, np.float64)).to(device)
        return cls(m.nrows, m.ncols, rp, col, val)

    @classmethod
    def empty(cls, nrows, ncols, device) -> "DeviceCsr":
        torch = _torch()
        return cls(nrows, ncols, torch.zeros(nrows + 1, dtype=torch.int64, device=device),
                   torch.zeros(0, dtype=torch.int32, device=device),
                   torch.zeros(0, dtype=torch.float64, device=device))

    def set_values(self, values, non_blocking=False):
        torch = _torch()
        if isinstance(values, torch.Tensor):
            src = values
        else:
            src = torch.from_numpy(np.ascontiguousarray(values, np.float64))
        if self.val is None:
            self.val = src.to(self.row_ptr.device, non_blocking=non_blocking)
        elif self.val.numel() != src.numel():
            # a plan built on this block sized every map for its nnz
            from .errors import StructuralDriftError
            raise StructuralDriftError(
                f"value array has {src.numel()} entries, the block's structure has {self.val.numel()}")
        else:
            self.val.copy_(src, non_blocking=non_blocking)

    def to_host(self) -> CsrMatrix:
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr.cpu().numpy(),
                         self.col.cpu().numpy().astype(np.int64),
                         None if self.val is None else self.val.cpu().numpy(), check=False)

    def struct(self) -> _lib.Csr:
        return _lib.Csr(self.nrows, self.ncols, self.nnz, _ptr(self.row_ptr), _ptr(self.col), _ptr(self.val))

    def transpose_with_permutation(self):
        """Device transpose plus the permutation mapping this block's values
        to the transpose's (reference CsrMatrix.transpose_with_permutation,
        src/sparse.py:165-178: ``t.val[:] = self.val[perm]`` refreshes it).
        Runs ``ptap_transpose`` (count, scan, scatter, per-row sort)."""
        import ctypes

        torch = _torch()
        dev = self.row_ptr.device
        n = self.nnz
        t_rp = torch.zeros(self.ncols + 1, dtype=torch.int64, device=dev)
        t_col = torch.empty(n, dtype=torch.int32, device=dev)
        perm = torch.empty(n, dtype=torch.int64, device=dev)
        t_val = None if self.val is None else torch.empty(n, dtype=torch.float64, device=dev)
        L = _lib.load()
        _lib.check(L.ptap_transpose(self.nrows, self.ncols, _ptr(self.row_ptr), _ptr(self.col), _ptr(self.val), n,
                                    _ptr(t_rp), _ptr(t_col), _ptr(perm), _ptr(t_val),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)), "transpose")
        return DeviceCsr(self.ncols, self.nrows, t_rp, t_col, t_val), perm

    def transpose(self) -> "DeviceCsr":
        return self.transpose_with_permutation()[0]


class DeviceLocalMatrix:
    """Device image of a reference ``LocalMatrix``."""

    def __init__(self, row_lo, row_hi, col_lo, col_hi, diag: DeviceCsr, offdiag: DeviceCsr, col_map):
        self.row_lo, self.row_hi, self.col_lo, self.col_hi = int(row_lo), int(row_hi), int(col_lo), int(col_hi)
        self.diag, self.offdiag, self.col_map = diag, offdiag, col_map  # col_map: int32 device tensor

    @property
    def nrows(self) -> int:
        return self.row_hi - self.row_lo

    @property
    def nnz(self) -> int:
        return self.diag.nnz + self.offdiag.nnz

    @property
    def nbytes(self) -> int:
        return self.diag.nbytes + self.offdiag.nbytes + self.col_map.numel() * 4

    @classmethod
    def from_local(cls, lm: LocalMatrix, device) -> "DeviceLocalMatrix":
        torch = _torch()
        return cls(lm.row_lo, lm.row_hi, lm.col_lo, lm.col_hi,
                   DeviceCsr.from_host(lm.diag, device), DeviceCsr.from_host(lm.offdiag, device),
                   torch.from_numpy(np.ascontiguousarray(lm.col_map, np.int32)).to(device))

    def refresh_values(self, lm: LocalMatrix, non_blocking=False):
        self.diag.set_values(lm.diag.values, non_blocking)
        self.offdiag.set_values(lm.offdiag.values, non_blocking)

    def to_local(self) -> LocalMatrix:
        return LocalMatrix(self.row_lo, self.row_hi, self.col_lo, self.col_hi, self.diag.to_host(),
                           self.offdiag.to_host(), self.col_map.cpu().numpy().astype(np.int64))


def structure_token(lm: LocalMatrix) -> tuple:
    """Cheap identity of a host LocalMatrix's structure (the reference uses a
    CRC32 of the structure arrays, src/comm.py:517-524)."""
    import zlib

    d = zlib.crc32(lm.diag.row_offsets.tobytes())
    for arr in (lm.diag.col_indices, lm.offdiag.row_offsets, lm.offdiag.col_indices, lm.col_map):
        d = zlib.crc32(np.ascontiguousarray(arr).tobytes(), d)
    return (lm.nrows, lm.diag.nnz, lm.offdiag.nnz, d)


class DeviceOperands:
    """Everything one rank passes to the library for C = P^T A P."""

    def __init__(self, a: DeviceLocalMatrix, p: DeviceLocalMatrix, m_global: int, c_lo: int, c_hi: int,
                 p_remote: DeviceCsr):
        self.a, self.p, self.m, self.c_lo, self.c_hi, self.p_remote = a, p, int(m_global), int(c_lo), int(c_hi), p_remote

    def struct(self) -> _lib.Operands:
        return _lib.Operands(
            self.a.nrows, self.m, self.c_lo, self.c_hi,
            self.a.diag.struct(), self.a.offdiag.struct(), self.p.diag.struct(), self.p.offdiag.struct(),
            _ptr(self.p.col_map), int(self.p.col_map.numel()), self.p_remote.struct())
