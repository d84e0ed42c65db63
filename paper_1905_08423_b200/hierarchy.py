"""Multigrid hierarchy driver: A_{l+1} = P_l^T A_l P_l, level after level,
with every coarse operator kept on the device.

The reference has no such driver -- chaining levels is caller composition
around ``ptap`` -- but config 3 asks for the
product at each level of a 3-level hierarchy.  Here level l+1's A is built
from level l's plan-owned C without a host round trip:

  * its structure comes from level l's symbolic phase (C's row offsets and
    global columns), split into the diag/offdiag blocks of the coarse row
    partition (``p_l.col_part``), so level l+1's symbolic phase can run before
    any numeric pass;
  * its values are C's values: at one rank they *are* C's value buffer (no
    copy); with several ranks a device gather through the split's index
    arrays refreshes them after each level-l numeric pass.

``numeric()`` re-runs every level in order (the 1 symbolic + many numeric
protocol of PAPER:434 applied to the whole hierarchy).
"""

from __future__ import annotations

from dataclasses import dataclass

from .comm import RankContext
from .device import DeviceCsr, DeviceLocalMatrix
from .partition import DistMatrix
from .tripleproduct import TripleProductPlan, run_numeric_device, run_symbolic


def _torch():
    import torch
    return torch


@dataclass
class HierarchyLevel:
    a: DistMatrix               # A_l (level 0: the caller's operand)
    p: DistMatrix               # P_l
    plan: TripleProductPlan     # plan of C_l = P_l^T A_l P_l
    _next_a: DistMatrix = None  # A_{l+1} (device, built from C_l)
    _diag_idx: object = None    # C_l value positions of A_{l+1}'s diag block (None: aliased)
    _off_idx: object = None     # ... and of its offdiag block


def _coarse_operator(plan: TripleProductPlan, p: DistMatrix):
    """A_{l+1} as a device DistMatrix over p.col_part, from C_l's structure;
    returns (DistMatrix, diag_idx, off_idx)."""
    torch = _torch()
    part = p.col_part
    rank = p.rank
    lo, hi = part.owned_range(rank)
    nr = hi - lo
    rp, col, val = plan.c_device()
    dev = rp.device
    if col.numel() == 0 or (int(col.min().item()) >= lo and int(col.max().item()) < hi):
        # every column owned (one rank): the diag block aliases C itself
        dcol = col if lo == 0 else (col - lo).to(torch.int32)
        diag = DeviceCsr(nr, nr, rp, dcol, val)
        loc = DeviceLocalMatrix(lo, hi, lo, hi, diag, DeviceCsr.empty(nr, 0, dev),
                                torch.zeros(0, dtype=torch.int32, device=dev))
        return DistMatrix(part, part, rank, loc), None, None
    rowid = torch.repeat_interleave(torch.arange(nr, device=dev), rp[1:] - rp[:-1])
    inside = (col >= lo) & (col < hi)
    diag_idx = torch.nonzero(inside).flatten()
    off_idx = torch.nonzero(~inside).flatten()

    def block(idx, cols, ncols):
        cnt = torch.bincount(rowid[idx], minlength=nr)
        brp = torch.zeros(nr + 1, dtype=torch.int64, device=dev)
        torch.cumsum(cnt, 0, out=brp[1:])
        return DeviceCsr(nr, ncols, brp, cols.to(torch.int32), val[idx].clone())

    diag = block(diag_idx, col[diag_idx] - lo, nr)
    ocol = col[off_idx].to(torch.int64)
    col_map = torch.unique(ocol)
    off = block(off_idx, torch.searchsorted(col_map, ocol), col_map.numel())
    loc = DeviceLocalMatrix(lo, hi, lo, hi, diag, off, col_map.to(torch.int32))
    return DistMatrix(part, part, rank, loc), diag_idx, off_idx


class GalerkinHierarchy:
    """Symbolic phases of every level at construction, numeric passes on
    demand.  ``prolongations[l]`` is P_l as a DistMatrix whose row partition
    is the column (and row) partition of A_l."""

    def __init__(self, a: DistMatrix, prolongations, algorithm: str, ctx: RankContext):
        self.ctx = ctx
        self.algorithm = algorithm
        self.levels: list[HierarchyLevel] = []
        cur = a
        for p in prolongations:
            if p.row_part.nglobal != cur.col_part.nglobal:
                from .errors import PartitionMismatchError
                raise PartitionMismatchError(
                    f"level {len(self.levels)}: P has {p.row_part.nglobal} rows, A has {cur.col_part.nglobal} columns")
            plan = run_symbolic(cur, p, algorithm, ctx)
            nxt, di, oi = _coarse_operator(plan, p)
            self.levels.append(HierarchyLevel(cur, p, plan, nxt, di, oi))
            cur = nxt

    @property
    def coarsest(self) -> DistMatrix:
        return self.levels[-1]._next_a

    def operators(self) -> list:
        """[A_0, A_1, ..., A_L]; A_{l>0} are device-resident DistMatrix."""
        return [self.levels[0].a] + [lv._next_a for lv in self.levels]

    def numeric(self):
        """One numeric pass per level, in order; returns the coarse operators'
        device C views [(row_ptr, col, val)] per level."""
        out = []
        for lv in self.levels:
            c = run_numeric_device(lv.a, lv.p, lv.plan, self.ctx)
            if lv._diag_idx is not None:
                loc = lv._next_a.local
                _torch().index_select(c[2], 0, lv._diag_idx, out=loc.diag.val)
                _torch().index_select(c[2], 0, lv._off_idx, out=loc.offdiag.val)
            out.append(c)
        return out

    def c_local(self, level: int):
        """Host LocalMatrix of level ``level``'s C (a copy of the current values)."""
        return self.levels[level].plan.c_local()

    def memory(self) -> list:
        return [lv.plan.memory() for lv in self.levels]
