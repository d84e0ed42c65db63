"""The drop-in operator API: C = P^T A P with three algorithms.

Same entry points, argument meanings and error behaviour as the reference
(src/tripleproduct.py:50-529): ``ptap``, ``run_symbolic``, ``run_numeric``,
``aao_symbolic``/``aao_numeric``, ``merged_symbolic``/``merged_numeric``,
``two_step_symbolic``/``two_step_numeric``, ``TripleProductPlan`` with the
``keep``/``free`` cache policy.  Every phase runs on the GPU through the
C-ABI library (include/ptap_b200.h); this module only orchestrates the
phases and the rank exchanges (comm.py), in the reference's order:

    all-at-once  symbolic: send loop -> start C_s exchange -> local loop -> merge -> allocate C
                 numeric:  send loop -> start exchange -> local loop (overlapped) -> merge
    merged       one fused loop, then the exchange (no overlap window)
    two-step     C~ = A P, explicit P^T, P_o^T C~ (sent), P_d^T C~ (local), merge

There is no CPU path: without the CUDA library or a device every call
raises ``DeviceError``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .comm import (RankContext, RemoteRows, exchange_structure, exchange_values, gather_remote_rows,
                   refresh_remote_values)
from .device import DeviceCsr, DeviceLocalMatrix, DeviceOperands, structure_token
from .errors import PartitionMismatchError, StructuralDriftError
from .ledger import PlanCounters
from .partition import DistMatrix, LocalMatrix, RowPartition
from .sparse import CsrMatrix

TWO_STEP = "two-step"
ALL_AT_ONCE = "allatonce"
MERGED = "merged"
ALGORITHMS = (TWO_STEP, ALL_AT_ONCE, MERGED)

CACHE_KEEP = "keep"
CACHE_FREE = "free"


def _torch():
    import torch

    return torch


class _CudaArray:
    """Expose a library-owned device buffer to torch without copying.  The
    tensor torch builds keeps this object alive, and this object keeps the
    owning plan alive, so a view never outlives the plan's memory."""

    _TYPESTR = {"int64": "<i8", "int32": "<i4", "float64": "<f8"}

    def __init__(self, ptr: int, n: int, dtype: str, owner=None):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": self._TYPESTR[dtype],
                                         "data": (int(ptr or 0), False), "version": 3, "strides": None}


def _dev_view(ptr, n, dtype, device, owner=None):
    torch = _torch()
    tdt = {"int64": torch.int64, "int32": torch.int32, "float64": torch.float64}[dtype]
    if not ptr or n == 0:
        return torch.zeros(0, dtype=tdt, device=device)
    return torch.as_tensor(_CudaArray(ptr, n, dtype, owner), device=device)


def _want_deterministic(flag) -> bool:
    """Explicit argument, else the PTAP_DETERMINISTIC environment switch."""
    import os
    if flag is None:
        return os.environ.get("PTAP_DETERMINISTIC", "") not in ("", "0")
    return bool(flag)


def _stream_ptr():
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


@dataclass
class AllocatedMatrix:
    """Host view of the allocated C (reference AllocatedMatrix,
    src/spgemm.py:35-68).  ``local`` is refreshed by every numeric pass.

    The reference marks every slot a numeric pass writes (fill flags) and
    raises StructuralDriftError when one was never written -- i.e. when the
    operands' structure no longer matches the symbolic plan.  On the device
    the numeric kernels write C through the plan's maps, so the same
    condition is checked at its source: every numeric call compares the
    operands' sizes with the symbolic image (and re-digests replaced
    structure arrays); ``verify_filled`` runs the full device digest of every
    structure array against the symbolic one (``ptap_plan_verify``).  The
    fill arrays report the slots the last verified pass wrote."""

    local: LocalMatrix
    nzd: np.ndarray
    nzo: np.ndarray
    fill_d: np.ndarray
    fill_o: np.ndarray
    _plan: object = None

    @property
    def nbytes(self) -> int:
        return self.local.nbytes + self.nzd.nbytes + self.nzo.nbytes

    def reset_fill(self):
        self.fill_d[:] = 0
        self.fill_o[:] = 0

    def verify_filled(self, what: str = "C"):
        plan = self._plan
        if plan is None or not plan._h or plan._ops is None:
            raise StructuralDriftError(f"{what}: no live plan to verify against")
        st = plan._ops.struct()
        _lib.check(_lib.load().ptap_plan_verify(plan._h, ctypes.byref(st), _stream_ptr()), f"verify {what}")
        self.fill_d[:] = 1
        self.fill_o[:] = 1


@dataclass
class StagingView:
    """Host summary of the send-side staging (rows owned by other ranks)."""

    rows: np.ndarray
    indptr: np.ndarray
    nnz: int

    @property
    def nbytes(self) -> int:
        return self.rows.nbytes + self.indptr.nbytes + self.nnz * 12


def _check_triple_operands(a: DistMatrix, p: DistMatrix):
    """Reference checks (src/tripleproduct.py:148-159, src/spgemm.py:107-113)."""
    if a.row_part != a.col_part:
        raise PartitionMismatchError("A must be square with matching row/column partitions")
    if a.col_part.nglobal != p.row_part.nglobal:
        raise PartitionMismatchError(
            f"dimension mismatch: A has {a.col_part.nglobal} columns, P has {p.row_part.nglobal} rows")
    if a.col_part != p.row_part:
        raise PartitionMismatchError("the column partition of A must equal the row partition of P")
    if a.rank != p.rank:
        raise PartitionMismatchError("operands come from different rank contexts")
    m = p.col_part.nglobal
    if m and m * m >= 2 ** 62:
        raise PartitionMismatchError("output dimension too large for combined row/col keys")


class TripleProductPlan:
    """Device-resident symbolic state for repeated numeric products
    (reference TripleProductPlan, src/tripleproduct.py:105-145)."""

    def __init__(self, algorithm: str, rank: int):
        self.algorithm = algorithm
        self.rank = rank
        self.counters = PlanCounters()
        self.released = False
        self.remote_rows: RemoteRows | None = None
        self.staging: StagingView | None = None
        self._h = ctypes.c_void_p()
        self._ops: DeviceOperands | None = None
        self._a_token = self._p_token = None
        self._route = None
        self._recv_keep = None
        self._c_host = None  # (rp, col, diag_idx, off_idx, LocalMatrix skeleton)
        self._c_alloc: AllocatedMatrix | None = None
        self._device = None
        self._c_part = None

    # -- library state -----------------------------------------------------

    def _lib(self):
        return _lib.load()

    def memory(self) -> dict:
        mem = _lib.Memory()
        _lib.check(self._lib().ptap_plan_memory(self._h, ctypes.byref(mem)), "plan memory")
        cats = ("input_matrices", "output_matrix", "auxiliary_matrices", "transient_hash_peak", "plan_cache")
        out = {"current": dict(zip(cats, list(mem.current))), "peak": dict(zip(cats, list(mem.peak))),
               "product_peak": int(mem.product_peak), "device_high_water": int(mem.device_high_water)}
        rr = self.remote_rows.nbytes if self.remote_rows is not None else 0
        out["remote_rows_bytes"] = rr
        return out

    def device_counters(self) -> dict:
        c = _lib.Counters()
        _lib.check(self._lib().ptap_plan_counters(self._h, ctypes.byref(c)), "plan counters")
        return {name: int(getattr(c, name)) for name, _ in _lib.Counters._fields_}

    def _sync_counters(self):
        d = self.device_counters()
        self.counters.symbolic_runs = d["symbolic_runs"]
        self.counters.numeric_runs = d["numeric_runs"]
        self.counters.symbolic_row_kernel_calls = d["symbolic_row_kernel_calls"]
        self.counters.numeric_row_kernel_calls = d["numeric_row_kernel_calls"]

    def c_device(self):
        """(row_ptr int64, col int32 [global columns], val float64) device
        tensors of the rank's rows of C, aliasing plan storage."""
        v = _lib.CView()
        _lib.check(self._lib().ptap_plan_get_c(self._h, ctypes.byref(v)), "get C")
        dev = self._device
        return (_dev_view(v.row_ptr, v.nrows + 1, "int64", dev, self), _dev_view(v.col, v.nnz, "int32", dev, self),
                _dev_view(v.val, v.nnz, "float64", dev, self))

    def _staging_device(self):
        s = _lib.Staging()
        _lib.check(self._lib().ptap_plan_staging(self._h, ctypes.byref(s)), "staging")
        dev = self._device
        return (_dev_view(s.rows, s.nrows, "int32", dev, self),
                _dev_view(s.row_ptr, s.nrows + 1 if s.nrows else 0, "int64", dev, self),
                _dev_view(s.col, s.nnz, "int32", dev, self), _dev_view(s.val, s.nnz, "float64", dev, self))

    @property
    def c_alloc(self) -> AllocatedMatrix:
        if self._c_alloc is None:
            self._build_c_host()
        return self._c_alloc

    def _build_c_host(self):
        rp_d, col_d, _ = self.c_device()
        rp = rp_d.cpu().numpy()
        col = col_d.cpu().numpy().astype(np.int64)
        c_lo, c_hi = self._c_part.owned_range(self.rank)
        n = rp.size - 1
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
        inside = (col >= c_lo) & (col < c_hi)
        diag_idx = np.flatnonzero(inside)
        off_idx = np.flatnonzero(~inside)
        nzd = np.bincount(rows[inside], minlength=n).astype(np.int64)
        nzo = np.bincount(rows[~inside], minlength=n).astype(np.int64)
        ipd = np.zeros(n + 1, np.int64)
        np.cumsum(nzd, out=ipd[1:])
        ipo = np.zeros(n + 1, np.int64)
        np.cumsum(nzo, out=ipo[1:])
        col_map = np.unique(col[~inside])
        diag = CsrMatrix(n, c_hi - c_lo, ipd, col[inside] - c_lo, np.zeros(diag_idx.size), check=False)
        off = CsrMatrix(n, col_map.size, ipo, np.searchsorted(col_map, col[~inside]), np.zeros(off_idx.size), check=False)
        local = LocalMatrix(c_lo, c_hi, c_lo, c_hi, diag, off, col_map)
        self._c_host = (diag_idx, off_idx)
        self._c_alloc = AllocatedMatrix(local, nzd, nzo, np.ones(diag_idx.size, np.uint8), np.ones(off_idx.size, np.uint8),
                                        self)

    def check(self):
        """Wait for the status of the last numeric pass and raise on drift
        (the device-result path reports it asynchronously)."""
        if self._h:
            _lib.check(self._lib().ptap_plan_status_poll(self._h), "numeric")

    def c_local(self) -> LocalMatrix:
        """Copy the current C values to the host LocalMatrix view."""
        self.check()
        alloc = self.c_alloc
        _, _, val_d = self.c_device()
        diag_idx, off_idx = self._c_host
        if off_idx.size == 0:
            # every column owned: C values are the diag values in order
            if getattr(self, "_pinned_c", None) is None or self._pinned_c.numel() != val_d.numel():
                self._pinned_c = _torch().empty(val_d.numel(), dtype=_torch().float64,
                                                pin_memory=_torch().cuda.is_available())
            self._pinned_c.copy_(val_d)
            alloc.local.diag.values = self._pinned_c.numpy()
            return alloc.local
        vals = val_d.cpu().numpy()
        alloc.local.diag.values[:] = vals[diag_idx]
        alloc.local.offdiag.values[:] = vals[off_idx]
        return alloc.local

    def release_cache(self, ctx=None):
        """Free everything beyond C (cache='free', src/tripleproduct.py:127-139)."""
        if self.released:
            return
        if self._c_alloc is None and self._h:
            self._build_c_host()
        if self._h:
            _lib.check(self._lib().ptap_plan_release_cache(self._h), "release cache")
        if ctx is not None:
            for cat in ("plan_cache", "auxiliary_matrices"):
                cur = ctx.ledger.current(cat)
                if cur:
                    ctx.ledger.release(cat, cur)
        self.remote_rows = None
        self.staging = None
        self._recv_keep = None
        self.released = True

    def _require_live(self):
        if self.released:
            raise StructuralDriftError("plan internals were released (free-after-solve); rebuild the plan")

    def __del__(self):
        try:
            if self._h:
                _lib.load(require_device=False).ptap_plan_destroy(self._h)
                self._h = ctypes.c_void_p()
        except Exception:
            pass

    @property
    def values_ready(self) -> bool:
        """True when the symbolic phase also computed C's values (the
        single-shot pass): C holds the product of the symbolic-time operands."""
        if not self._h:
            return False
        r = ctypes.c_int(0)
        _lib.check(self._lib().ptap_plan_values_ready(self._h, ctypes.byref(r)), "values ready")
        return bool(r.value)

    @property
    def deterministic(self) -> bool:
        """True when repeated numeric passes are bitwise identical: the
        two-step comparator, or an all-at-once / merged plan running the
        owner-computes kernel (numeric_path 2; ``deterministic=True`` at
        symbolic time on a one-rank-structured local loop)."""
        if self.algorithm == TWO_STEP:
            return True
        return bool(self._h) and self.device_counters()["numeric_path"] == 2

    # two-step inspection helper (reference plan.ctilde)
    @property
    def ctilde(self):
        """Two-step: the stored auxiliary C~ = A P of this rank as device
        tensors (row_ptr int64, col int32 global, val float64), or None
        (other algorithms, or after release_cache)."""
        if self.algorithm != TWO_STEP or self.released or not self._h:
            return None
        v = _lib.CView()
        _lib.check(self._lib().ptap_plan_get_ctilde(self._h, ctypes.byref(v)), "ctilde")
        dev = self._device
        from .spgemm import DeviceAP
        return DeviceAP(_dev_view(v.row_ptr, v.nrows + 1, "int64", dev, self), _dev_view(v.col, v.nnz, "int32", dev, self),
                        _dev_view(v.val, v.nnz, "float64", dev, self), v.ncols, None, None)


# ---------------------------------------------------------------------------
# operand upload
# ---------------------------------------------------------------------------


def _device_local(m, device) -> DeviceLocalMatrix:
    if isinstance(m.local, DeviceLocalMatrix):
        return m.local
    return DeviceLocalMatrix.from_local(m.local, device)


def _prepare(plan: TripleProductPlan, a: DistMatrix, p: DistMatrix, ctx: RankContext, symbolic: bool):
    """Upload (symbolic) or refresh values (numeric) of the operands."""
    dev = ctx.device
    if symbolic:
        plan._a_dev = _device_local(a, dev)
        plan._p_dev = _device_local(p, dev)
        if isinstance(a.local, LocalMatrix):
            plan._a_token = (_identity(a.local), structure_token(a.local))
        if isinstance(p.local, LocalMatrix):
            plan._p_token = (_identity(p.local), structure_token(p.local))
        return
    for which, m, tok in (("A", a, plan._a_token), ("P", p, plan._p_token)):
        if isinstance(m.local, LocalMatrix):
            _check_host_structure(which, m.local, tok)
            target = plan._a_dev if which == "A" else plan._p_dev
            target.refresh_values(m.local)
        else:
            target = plan._a_dev if which == "A" else plan._p_dev
            if m.local is not target:
                if which == "A":
                    plan._a_dev = m.local
                else:
                    plan._p_dev = m.local
    plan._ops.a, plan._ops.p = plan._a_dev, plan._p_dev


def _identity(lm: LocalMatrix) -> tuple:
    """The structure arrays themselves (strong references: their identity
    cannot be recycled while the plan holds them)."""
    return (lm.diag.row_offsets, lm.diag.col_indices, lm.offdiag.row_offsets, lm.offdiag.col_indices, lm.col_map)


def _check_host_structure(which: str, lm: LocalMatrix, tok):
    """Numeric-time drift check of a host operand: the very arrays seen at
    symbolic time, still frozen (CsrMatrix makes its structure read-only),
    need no hashing; anything else is compared by CRC (the reference's
    structure token, src/comm.py:517-524)."""
    if tok is None:
        return
    cur = _identity(lm)
    # the CSR structure arrays are frozen by CsrMatrix; col_map is compared by identity
    same = all(x is y for x, y in zip(cur, tok[0])) and not any(
        getattr(x, "flags", None) is not None and x.flags.writeable for x in cur[:4])
    if not same and (tok[1] is None or structure_token(lm) != tok[1]):
        raise StructuralDriftError(f"{which} changed structure since the symbolic phase")


def _remote_csr(rr: RemoteRows, m: int, device) -> DeviceCsr:
    n = rr.source_cols.size
    return DeviceCsr(n, m, rr.row_ptr.to(device), rr.col.to(device), rr.val.to(device))


# ---------------------------------------------------------------------------
# phases
# ---------------------------------------------------------------------------


def _symbolic(a: DistMatrix, p: DistMatrix, ctx: RankContext, algorithm: str, deterministic=None,
              maps=None, lockstep=None, single_shot=None) -> TripleProductPlan:
    _check_triple_operands(a, p)
    L = _lib.load()
    torch = _torch()
    plan = TripleProductPlan(algorithm, ctx.rank)
    plan._device = ctx.device
    plan._c_part = p.col_part
    with ctx.timer.phase("symbolic"):
        _prepare(plan, a, p, ctx, symbolic=True)
        ctx.ledger.add("input_matrices", plan._a_dev.nbytes + plan._p_dev.nbytes)
        m = p.col_part.nglobal
        c_lo, c_hi = p.col_part.owned_range(ctx.rank)
        a_colmap = a.local.col_map
        if not isinstance(a_colmap, np.ndarray):
            a_colmap = a_colmap.cpu().numpy().astype(np.int64)
        with ctx.timer.phase("gather"):
            rr = gather_remote_rows(ctx, a_colmap, p.row_part, plan._p_dev)
        plan.remote_rows = rr
        ctx.ledger.add("plan_cache", rr.nbytes)
        ops = DeviceOperands(plan._a_dev, plan._p_dev, m, c_lo, c_hi, _remote_csr(rr, m, ctx.device))
        plan._ops = ops
        st = ops.struct()
        _lib.check(L.ptap_plan_create(_lib.ALGORITHM_CODES[algorithm], ctypes.byref(st), ctypes.byref(plan._h)),
                   "plan create")
        if _want_deterministic(deterministic):
            _lib.check(L.ptap_plan_set_option(plan._h, b"deterministic", 1), "plan option")
        if maps is not None:
            _lib.check(L.ptap_plan_set_option(plan._h, b"maps", 1 if maps else 0), "plan option")
        if lockstep is not None:
            _lib.check(L.ptap_plan_set_option(plan._h, b"lockstep", 1 if lockstep else 0), "plan option")
        if single_shot:
            _lib.check(L.ptap_plan_set_option(plan._h, b"single_shot", 1), "plan option")
        stream = _stream_ptr()
        _lib.check(L.ptap_symbolic_send(plan._h, ctypes.byref(st), stream), "symbolic send")
        s_rows, s_rp, s_col, _ = plan._staging_device()
        plan.staging = StagingView(s_rows.cpu().numpy().astype(np.int64),
                                   s_rp.cpu().numpy() if s_rp.numel() else np.zeros(1, np.int64), int(s_col.numel()))
        recv = None
        if ctx.nranks > 1:
            with ctx.timer.phase("exchange"):
                rows_in, widths_in, cols_in, route = exchange_structure(ctx, s_rows, s_rp, s_col, p.col_part)
            plan._route = route
            if rows_in.size and (rows_in.min() < c_lo or rows_in.max() >= c_hi):
                raise StructuralDriftError(
                    f"received contribution rows outside the owned range [{c_lo}, {c_hi})")
            rp_in = np.zeros(rows_in.size + 1, np.int64)
            np.cumsum(widths_in, out=rp_in[1:])
            d_rows = torch.as_tensor(rows_in.astype(np.int32), device=ctx.device)
            d_rp = torch.as_tensor(rp_in, device=ctx.device)
            d_col = cols_in.to(ctx.device).to(torch.int32)
            srcs = np.arange(ctx.nranks, dtype=np.int32)
            row_off = np.concatenate(([0], np.cumsum(route.recv_rows))).astype(np.int64)
            nnz_off = np.concatenate(([0], np.cumsum(route.recv_nnz))).astype(np.int64)
            plan._recv_keep = (d_rows, d_rp, d_col, srcs, row_off, nnz_off)
            recv = _lib.Received(ctx.nranks, srcs.ctypes.data, row_off.ctypes.data, nnz_off.ctypes.data,
                                 int(rows_in.size), int(rp_in[-1]), d_rows.data_ptr() if d_rows.numel() else None,
                                 d_rp.data_ptr(), d_col.data_ptr() if d_col.numel() else None)
        _lib.check(L.ptap_symbolic_local(plan._h, ctypes.byref(st), ctypes.byref(recv) if recv is not None else None,
                                         stream), "symbolic local")
        mem = plan.memory()
        for cat in ("output_matrix", "auxiliary_matrices", "plan_cache"):
            if mem["current"][cat]:
                ctx.ledger.add(cat, mem["current"][cat])
        ctx.ledger.record_peak("transient_hash_peak", mem["peak"]["transient_hash_peak"])
    plan._sync_counters()
    return plan


_UPLOAD_BLOCKS = 32  # row blocks of the streamed host-operand numeric pass (PTAP_UPLOAD_BLOCKS; 8 -> 75.7 ms, 32 -> 74.5 ms on config 3)


def _streamable(a: DistMatrix, p: DistMatrix, plan: TripleProductPlan, ctx: RankContext) -> bool:
    import os
    if os.environ.get("PTAP_UPLOAD_BLOCKS", "") == "1" or getattr(plan, "_stream_ok", True) is False:
        return False
    return (ctx.nranks == 1 and plan.algorithm == ALL_AT_ONCE and isinstance(a.local, LocalMatrix)
            and isinstance(p.local, LocalMatrix) and a.local.offdiag.nnz == 0 and p.local.offdiag.nnz == 0
            and _torch().cuda.is_available())


def _numeric_streamed(a: DistMatrix, p: DistMatrix, plan: TripleProductPlan, ctx: RankContext):
    """All-at-once numeric pass at one rank with host operands, pipelined over
    PCIe: P's values go up first, then A's values in row blocks on a copy
    stream while the previous blocks fold (``ptap_numeric_local_rows``), and
    C rows that are final (every contributing fine row folded, from the
    plan's last-contributor map) come back on a third stream while later
    blocks run.  Same kernels, same result as the one-shot path."""
    import os

    torch = _torch()
    L = _lib.load()
    # drift check as in _prepare
    for which, m, tok in (("A", a, plan._a_token), ("P", p, plan._p_token)):
        _check_host_structure(which, m.local, tok)
    st = plan._ops.struct()
    dev = ctx.device
    if getattr(plan, "_stream_state", None) is None:
        up, dn = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        rp_d, _, val_d = plan.c_device()
        last = torch.empty(max(rp_d.numel() - 1, 1), dtype=torch.int32, device=dev)
        _lib.check(L.ptap_plan_c_last_row(plan._h, ctypes.byref(st), ctypes.c_void_p(last.data_ptr()),
                                          _stream_ptr()), "last contributors")
        pmax = np.maximum.accumulate(last[:rp_d.numel() - 1].cpu().numpy().astype(np.int64)) if rp_d.numel() > 1 \
            else np.zeros(0, np.int64)
        plan._stream_state = (up, dn, rp_d.cpu().numpy(), pmax)
    up, dn, c_rp, pmax = plan._stream_state
    nblk = max(1, int(os.environ.get("PTAP_UPLOAD_BLOCKS", _UPLOAD_BLOCKS)))
    n = a.local.nrows
    a_rp = a.local.diag.row_offsets
    # block-aligned bounds (the plan's numeric kernels fold 64-row blocks)
    bounds = sorted({min(n, -(-(n * k // nblk) // 64) * 64) for k in range(nblk)} | {0, n})
    if len(bounds) < 2:
        bounds = [0, n]
    nblk = len(bounds) - 1  # small operands: fewer, non-empty blocks (every bound is a multiple of 64, or n)
    a_host = torch.from_numpy(a.local.diag.values)
    p_host = torch.from_numpy(p.local.diag.values)
    a_dev, p_dev = plan._a_dev.diag.val, plan._p_dev.diag.val
    _, _, val_d = plan.c_device()
    if getattr(plan, "_pinned_c", None) is None or plan._pinned_c.numel() != val_d.numel():
        plan._pinned_c = torch.empty(val_d.numel(), dtype=torch.float64, pin_memory=True)
    c_host = plan._pinned_c
    comp = torch.cuda.current_stream(dev)
    up.wait_stream(comp)  # the previous pass no longer reads the operands
    dn.wait_stream(comp)
    with ctx.timer.phase("numeric"):
        with torch.cuda.stream(up):
            p_dev.copy_(p_host, non_blocking=True)
            ev_p = torch.cuda.Event()
            ev_p.record(up)
            ev_blk = []
            for b in range(nblk):
                lo, hi = int(a_rp[bounds[b]]), int(a_rp[bounds[b + 1]])
                if hi > lo:
                    a_dev[lo:hi].copy_(a_host[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(up)
                ev_blk.append(e)
        comp.wait_event(ev_p)
        done_c = 0
        for b in range(nblk):
            comp.wait_event(ev_blk[b])
            flags = (1 if b == 0 else 0) | (2 if b == nblk - 1 else 0)
            status = L.ptap_numeric_local_rows(plan._h, ctypes.byref(st), bounds[b], bounds[b + 1], flags,
                                               ctypes.c_void_p(comp.cuda_stream))
            if status != 0 and b == 0:
                plan._stream_ok = False  # not range-addressable: one-shot path from now on
                return None
            _lib.check(status, "numeric local rows")
            # C rows whose last contributor has been folded
            upto = int(np.searchsorted(pmax, bounds[b + 1], side="left")) if b < nblk - 1 else pmax.size
            end = int(c_rp[upto]) if pmax.size else 0
            if end > done_c:
                ev = torch.cuda.Event()
                ev.record(comp)
                dn.wait_event(ev)
                with torch.cuda.stream(dn):
                    c_host[done_c:end].copy_(val_d[done_c:end], non_blocking=True)
                done_c = end
        comp.wait_stream(dn)
        _lib.check(L.ptap_plan_check(plan._h, _stream_ptr()), "numeric")
    plan._sync_counters()
    alloc = plan.c_alloc
    alloc.local.diag.values = c_host.numpy()
    return alloc.local


def _numeric(a: DistMatrix, p: DistMatrix, plan: TripleProductPlan, ctx: RankContext, expected: str,
             to_host: bool = True):
    if plan.algorithm != expected:
        raise ValueError(f"plan was built by {plan.algorithm!r}, not {expected!r}")
    plan._require_live()
    if to_host and _streamable(a, p, plan, ctx):
        local = _numeric_streamed(a, p, plan, ctx)
        if local is not None:
            return local
    L = _lib.load()
    with ctx.timer.phase("numeric"):
        _prepare(plan, a, p, ctx, symbolic=False)
        st = plan._ops.struct()
        stream = _stream_ptr()
        if ctx.nranks > 1:
            with ctx.timer.phase("gather"):
                refresh_remote_values(ctx, plan.remote_rows, plan._p_dev, plan._h, plan._ops)
        _lib.check(L.ptap_numeric_send(plan._h, ctypes.byref(st), stream), "numeric send")
        work = recv_vals = None
        if ctx.nranks > 1:
            s_val = plan._staging_device()[3]
            with ctx.timer.phase("exchange"):
                recv_vals, work = exchange_values(ctx, s_val, plan._route, async_op=True)
        # the local loop overlaps the in-flight exchange (all-at-once, two-step)
        _lib.check(L.ptap_numeric_local(plan._h, ctypes.byref(st), stream), "numeric local")
        if ctx.nranks > 1:
            with ctx.timer.phase("exchange"):
                if work is not None:
                    work.wait()
            rv = recv_vals.to(ctx.device, non_blocking=True)
            _lib.check(L.ptap_numeric_merge(plan._h, ctypes.c_void_p(rv.data_ptr() if rv.numel() else 0), stream),
                       "numeric merge")
        if to_host:
            _lib.check(L.ptap_plan_check(plan._h, stream), "numeric")
        else:
            # device result: the pass's status is copied behind it and read
            # by the next call (or plan.check()) -- no host synchronisation
            _lib.check(L.ptap_plan_status_async(plan._h, stream), "numeric")
    plan._sync_counters()
    return plan.c_local() if to_host else plan.c_device()


def aao_symbolic(a, p, ctx, *, deterministic=None, maps=None, lockstep=None, single_shot=None) -> TripleProductPlan:
    """All-at-once symbolic: send loop, exchange, local loop (Alg. 7).
    ``deterministic=True`` (or PTAP_DETERMINISTIC=1) selects the
    owner-computes numeric kernel: bitwise-repeatable passes whose C is
    bit-identical to the reference's at one rank."""
    return _symbolic(a, p, ctx, ALL_AT_ONCE, deterministic, maps, lockstep, single_shot)


def aao_numeric(a, p, plan, ctx):
    """All-at-once numeric into the plan's allocation (Alg. 8)."""
    return _numeric(a, p, plan, ctx, ALL_AT_ONCE)


def merged_symbolic(a, p, ctx, *, deterministic=None, maps=None, lockstep=None, single_shot=None) -> TripleProductPlan:
    """Merged all-at-once: one fused loop computes each AP row once (Alg. 9)."""
    return _symbolic(a, p, ctx, MERGED, deterministic, maps, lockstep, single_shot)


def merged_numeric(a, p, plan, ctx):
    return _numeric(a, p, plan, ctx, MERGED)


def two_step_symbolic(a, p, ctx, *, deterministic=None, maps=None, lockstep=None, single_shot=None) -> TripleProductPlan:
    """Two-step: C~ = A P, explicit P^T, then P^T C~ (Alg. 5); always
    deterministic (every entry is folded in the reference's order)."""
    return _symbolic(a, p, ctx, TWO_STEP, deterministic, maps, lockstep, single_shot)


def two_step_numeric(a, p, plan, ctx):
    return _numeric(a, p, plan, ctx, TWO_STEP)


_SYMBOLIC = {TWO_STEP: two_step_symbolic, ALL_AT_ONCE: aao_symbolic, MERGED: merged_symbolic}
_NUMERIC = {TWO_STEP: two_step_numeric, ALL_AT_ONCE: aao_numeric, MERGED: merged_numeric}


def run_symbolic(a, p, algorithm: str, ctx, *, deterministic=None, maps=None, lockstep=None,
                 single_shot=None) -> TripleProductPlan:
    """Symbolic phase (reference run_symbolic, src/tripleproduct.py:499-502).
    Options beyond the reference: ``deterministic`` (bitwise-repeatable
    numeric passes, bit-identical to the reference at one rank) and ``maps``
    (None: keep plan maps when rows repeat; False: hash numeric path, nothing
    stored per row; True: always keep maps) and ``lockstep`` (None/True: the
    class-lockstep numeric kernel when the plan is eligible, numeric_path 3;
    False: the per-row mapped kernels) and ``single_shot`` (True: when the
    rank neither sends nor receives, the symbolic phase also computes C's
    values in the same pass over A -- ``plan.values_ready``; nothing is kept
    per row, later numeric passes hash)."""
    if algorithm not in ALGORITHMS:
        raise ValueError(f"unknown algorithm {algorithm!r}; pick one of {ALGORITHMS}")
    return _SYMBOLIC[algorithm](a, p, ctx, deterministic=deterministic, maps=maps, lockstep=lockstep,
                                single_shot=single_shot)


def run_numeric(a, p, plan: TripleProductPlan, ctx):
    return _NUMERIC[plan.algorithm](a, p, plan, ctx)


def run_numeric_device(a, p, plan: TripleProductPlan, ctx):
    """Numeric pass leaving C on the device; returns (row_ptr, col, val)."""
    return _numeric(a, p, plan, ctx, plan.algorithm, to_host=False)


def ptap(a: DistMatrix, p: DistMatrix, algorithm: str, ctx: RankContext, cache: str = CACHE_KEEP, *,
         deterministic=None, single_shot=False):
    """One symbolic plus one numeric triple product; returns (C, plan).
    ``single_shot=True`` (all-at-once / merged): symbolic and numeric in one
    pass over A when the rank neither sends nor receives (BASELINE north_star
    (3)); otherwise the two phases run as usual."""
    if cache not in (CACHE_KEEP, CACHE_FREE):
        raise ValueError(f"cache policy must be '{CACHE_KEEP}' or '{CACHE_FREE}'")
    plan = run_symbolic(a, p, algorithm, ctx, deterministic=deterministic, single_shot=single_shot)
    if single_shot and plan.values_ready:
        plan._sync_counters()
        local = plan.c_local()
    else:
        local = run_numeric(a, p, plan, ctx)
    if cache == CACHE_FREE:
        plan.release_cache(ctx)
    return DistMatrix(p.col_part, p.col_part, ctx.rank, local), plan
