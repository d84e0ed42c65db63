"""Rank contexts and the two exchange patterns of the triple product.

The reference simulates ranks as threads with an in-process message harness
(src/comm.py:97-344).  Here a rank is a process with one GPU, and the two
communication patterns of the algorithm run over ``torch.distributed``:

* the remote-row gather of P (symbolic: structure and values,
  src/comm.py:561-622; numeric: values only, src/comm.py:625-649), and
* the owner-directed exchange of the send-side contributions C_s
  (src/comm.py:452-486), an alltoallv that NCCL performs over NVLink.

NCCL has no alltoallv primitive; ``all_to_all_single`` with split sizes is
the grouped send/recv it lowers to.  Counts are exchanged once in the
symbolic phase and cached in the plan, so numeric passes move values only.
With the ``gloo`` backend (CPU tests, world_size 2) the same code runs on
host tensors.  Received batches are always consumed in ascending source rank.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from .errors import OwnershipError, StructuralDriftError
from .ledger import MemoryLedger, PhaseTimer


def _torch():
    import torch

    return torch


class RankContext:
    """One rank's handle: rank/world, device, ledger, timer, collectives."""

    def __init__(self, rank: int = 0, nranks: int = 1, device=None, group=None, backend: str = "single"):
        self.rank, self.nranks = int(rank), int(nranks)
        self.group = group
        self.backend = backend
        self.ledger = MemoryLedger()
        self.timer = PhaseTimer()
        if device is None:
            torch = _torch()
            device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
        self.device = device
        self.trace: list = []

    @property
    def comm_device(self):
        """Where collective buffers must live: the GPU for NCCL, host for gloo."""
        torch = _torch()
        return self.device if self.backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.nranks > 1:
            _torch().distributed.barrier(group=self.group)

    # -- alltoallv ---------------------------------------------------------

    def exchange_counts(self, counts: np.ndarray) -> np.ndarray:
        """counts[d] = elements this rank sends to rank d -> received[s]."""
        torch = _torch()
        if self.nranks == 1:
            return np.asarray(counts, np.int64).copy()
        t = torch.as_tensor(np.asarray(counts, np.int64), device=self.comm_device)
        out = torch.empty_like(t)
        torch.distributed.all_to_all_single(out, t, group=self.group)
        return out.cpu().numpy()

    def alltoallv(self, send, send_counts, recv_counts, async_op=False, out=None):
        """Flat alltoallv of one tensor: send[sum(send_counts)] grouped by
        destination, returns the flat receive buffer grouped by source
        (ascending).  With async_op, returns (buffer, work handle).  ``out``
        (on the communication device) receives in place."""
        torch = _torch()
        sc = [int(x) for x in send_counts]
        rc = [int(x) for x in recv_counts]
        dev = self.comm_device
        src = send.to(dev) if send.device != dev else send
        if out is None or out.device != dev or out.numel() != sum(rc):
            out = torch.empty(sum(rc), dtype=send.dtype, device=dev)
        if self.nranks == 1:
            out.copy_(src)
            return (out, None) if async_op else out
        work = torch.distributed.all_to_all_single(out, src.contiguous(), output_split_sizes=rc,
                                                   input_split_sizes=sc, group=self.group, async_op=async_op)
        self.trace.append(("alltoallv", self.rank, sc, str(send.dtype)))
        return (out, work) if async_op else out


def single_rank_context(device=None) -> RankContext:
    return RankContext(0, 1, device=device, backend="single")


def init_from_env(backend: str | None = None) -> RankContext:
    """Context for a torchrun / launched process (RANK, WORLD_SIZE, MASTER_*)."""
    torch = _torch()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    if world == 1:
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        return single_rank_context()
    if backend is None:
        # PTAP_BACKEND=gloo runs several ranks on one GPU (functional checks of
        # the multi-rank path when only one device is available)
        backend = os.environ.get("PTAP_BACKEND") or ("nccl" if torch.cuda.is_available() else "gloo")
    if torch.cuda.is_available():
        ndev = torch.cuda.device_count()
        torch.cuda.set_device(local % ndev)
    if not torch.distributed.is_initialized():
        torch.distributed.init_process_group(backend=backend, rank=rank, world_size=world)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    return RankContext(rank, world, device=dev, group=None, backend=backend)


# ---------------------------------------------------------------------------
# remote-row gather of P (src/comm.py:494-649)
# ---------------------------------------------------------------------------


@dataclass
class RemoteRows:
    """Rows of P owned elsewhere and needed here, in A's off-diagonal
    column-map order; ``serve_idx`` lets the owner push values only."""

    source_cols: np.ndarray
    row_ptr: object            # device int64
    col: object                # device int32 (global coarse columns)
    val: object                # device float64
    send_counts: np.ndarray    # values this rank serves to each rank
    recv_counts: np.ndarray    # values this rank receives from each rank
    serve_idx: object          # device int64: positions in [P_d.val, P_o.val] to serve, grouped by dest
    structure_token: tuple = ()
    nbytes: int = 0


def _served_rows_global(p_local, wanted_local: np.ndarray, device):
    """Owner side of the gather (src/comm.py:527-554): for each wanted local
    row, its global columns (diag + offdiag merged, sorted) and the position
    of each value in the concatenation [P_d.val, P_o.val]."""
    torch = _torch()
    d_rp = p_local.diag.row_ptr
    o_rp = p_local.offdiag.row_ptr
    w = torch.as_tensor(wanted_local, dtype=torch.int64, device=device)
    dn = d_rp[w + 1] - d_rp[w]
    on = o_rp[w + 1] - o_rp[w]
    widths = dn + on
    ip = torch.zeros(w.numel() + 1, dtype=torch.int64, device=device)
    torch.cumsum(widths, 0, out=ip[1:])
    tot = int(ip[-1].item()) if w.numel() else 0
    if tot == 0:
        return ip, torch.zeros(0, dtype=torch.int32, device=device), torch.zeros(0, dtype=torch.int64, device=device)
    r = torch.repeat_interleave(torch.arange(w.numel(), device=device), widths)
    k = torch.arange(tot, device=device) - ip[:-1][r]
    is_d = k < dn[r]
    dpos = d_rp[w][r] + k
    opos = o_rp[w][r] + (k - dn[r])
    ddiag_nnz = p_local.diag.nnz
    gcol = torch.empty(tot, dtype=torch.int64, device=device)
    src = torch.empty(tot, dtype=torch.int64, device=device)
    if p_local.diag.nnz:
        gcol[is_d] = p_local.diag.col[dpos[is_d]].to(torch.int64) + p_local.col_lo
    src[is_d] = dpos[is_d]
    if p_local.offdiag.nnz:
        gcol[~is_d] = p_local.col_map[p_local.offdiag.col[opos[~is_d]].to(torch.int64)].to(torch.int64)
    src[~is_d] = ddiag_nnz + opos[~is_d]
    order = torch.argsort(r * (int(gcol.max().item()) + 1) + gcol)
    return ip, gcol[order].to(torch.int32), src[order]


def _p_values_concat(p_local):
    torch = _torch()
    parts = [t for t in (p_local.diag.val, p_local.offdiag.val) if t is not None and t.numel()]
    if not parts:
        return torch.zeros(0, dtype=torch.float64, device=p_local.diag.row_ptr.device)
    return torch.cat(parts)


def gather_remote_rows(ctx: RankContext, a_col_map: np.ndarray, p_row_part, p_local) -> RemoteRows:
    """Collective symbolic gather of the rows of P indexed by A's
    off-diagonal column map (one request + one reply per neighbour)."""
    torch = _torch()
    dev = p_local.diag.row_ptr.device
    wanted = np.asarray(a_col_map, np.int64)
    if ctx.nranks == 1 or wanted.size == 0 and ctx.nranks == 1:
        return RemoteRows(wanted, torch.zeros(1, dtype=torch.int64, device=dev),
                          torch.zeros(0, dtype=torch.int32, device=dev), torch.zeros(0, dtype=torch.float64, device=dev),
                          np.zeros(ctx.nranks, np.int64), np.zeros(ctx.nranks, np.int64),
                          torch.zeros(0, dtype=torch.int64, device=dev))
    if wanted.size and (wanted.min() < 0 or wanted.max() >= p_row_part.nglobal):
        raise OwnershipError(f"requested P row outside the global range [0, {p_row_part.nglobal})")
    owners = p_row_part.owners(wanted) if wanted.size else np.zeros(0, np.int64)
    req_counts = np.bincount(owners, minlength=ctx.nranks).astype(np.int64)
    got_counts = ctx.exchange_counts(req_counts)
    requests = ctx.alltoallv(torch.as_tensor(wanted, dtype=torch.int64), req_counts, got_counts).cpu().numpy()
    lo, hi = p_row_part.owned_range(ctx.rank)
    if requests.size and (requests.min() < lo or requests.max() >= hi):
        raise OwnershipError(f"a rank requested P rows outside rank {ctx.rank}'s range [{lo}, {hi})")
    # serve: widths + columns + value positions, grouped by requester (ascending)
    ip, gcol, src = _served_rows_global(p_local, requests - lo, dev)
    widths = (ip[1:] - ip[:-1]).cpu().numpy()
    # per-destination counts
    edges = np.concatenate(([0], np.cumsum(got_counts)))
    serve_row_counts = got_counts
    serve_val_counts = np.array([widths[edges[d]:edges[d + 1]].sum() for d in range(ctx.nranks)], np.int64)
    recv_val_counts = ctx.exchange_counts(serve_val_counts)
    w_in = ctx.alltoallv(torch.as_tensor(widths, dtype=torch.int64), serve_row_counts, req_counts).cpu().numpy()
    cols_in = ctx.alltoallv(gcol, serve_val_counts, recv_val_counts)
    vcat = _p_values_concat(p_local)
    vals_in = ctx.alltoallv(vcat[src] if src.numel() else vcat[:0], serve_val_counts, recv_val_counts)
    rp = np.zeros(wanted.size + 1, np.int64)
    np.cumsum(w_in, out=rp[1:])
    return RemoteRows(wanted, torch.as_tensor(rp, device=dev), cols_in.to(dev).to(torch.int32),
                      vals_in.to(dev), serve_val_counts, recv_val_counts, src,
                      nbytes=int(rp.nbytes + cols_in.numel() * 4 + vals_in.numel() * 8 + src.numel() * 8))


def refresh_remote_values(ctx: RankContext, rr: RemoteRows, p_local, plan_handle=None, ops=None):
    """Numeric values-only refresh of the gathered rows (src/comm.py:625-649).

    With the plan's handle the owner-side gather is one device kernel
    (``ptap_pack_values``: the serve index into [P_d.val, P_o.val] read in
    place, out-of-range indices flag drift in the plan status) and the
    alltoallv receives straight into the gathered rows' value buffer: no
    concatenation, no host synchronisation.  Without it (the standalone
    SpGEMM) the same gather runs as a tensor index."""
    if ctx.nranks == 1:
        return
    torch = _torch()
    n = rr.serve_idx.numel()
    if plan_handle is not None:
        from . import _lib
        if getattr(rr, "send_buf", None) is None or rr.send_buf.numel() != n:
            rr.send_buf = torch.empty(n, dtype=torch.float64, device=rr.serve_idx.device)
        st = ops.struct()
        stream = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.load().ptap_pack_values(plan_handle, __import__("ctypes").byref(st),
                                                rr.serve_idx.data_ptr() if n else None, n,
                                                rr.send_buf.data_ptr() if n else None, stream), "pack values")
        send = rr.send_buf
    else:
        vcat = _p_values_concat(p_local)
        send = vcat[rr.serve_idx] if n else vcat[:0]
    vals = ctx.alltoallv(send, rr.send_counts, rr.recv_counts, out=rr.val)
    if vals.data_ptr() != rr.val.data_ptr():
        rr.val.copy_(vals.to(rr.val.device), non_blocking=True)


# ---------------------------------------------------------------------------
# C_s -> owner exchange (src/comm.py:452-486)
# ---------------------------------------------------------------------------


@dataclass
class ContributionRoute:
    """Cached routing of the send-side staging: per-destination row/entry
    counts (sending side) and per-source counts (receiving side)."""

    send_rows: np.ndarray
    send_nnz: np.ndarray
    recv_rows: np.ndarray
    recv_nnz: np.ndarray
    recv_src_ranks: list = field(default_factory=list)


def exchange_structure(ctx: RankContext, staging_rows, staging_rp, staging_col, c_part):
    """Symbolic exchange of the staged (row, column) structure; returns the
    received batches (concatenated, ascending source) and the route."""
    torch = _torch()
    rows_h = staging_rows.cpu().numpy().astype(np.int64) if staging_rows is not None else np.zeros(0, np.int64)
    rp_h = staging_rp.cpu().numpy() if staging_rp is not None else np.zeros(1, np.int64)
    owners = c_part.owners(rows_h) if rows_h.size else np.zeros(0, np.int64)
    if np.any(owners == ctx.rank):
        raise OwnershipError("staged rows must be owned by other ranks")
    send_rows = np.bincount(owners, minlength=ctx.nranks).astype(np.int64)
    widths = np.diff(rp_h)
    send_nnz = np.array([widths[owners == d].sum() for d in range(ctx.nranks)], np.int64)
    recv_rows = ctx.exchange_counts(send_rows)
    recv_nnz = ctx.exchange_counts(send_nnz)
    hdr = np.stack([rows_h, widths], axis=1).reshape(-1) if rows_h.size else np.zeros(0, np.int64)
    hdr_in = ctx.alltoallv(torch.as_tensor(hdr, dtype=torch.int64), 2 * send_rows, 2 * recv_rows).cpu().numpy()
    col_send = staging_col if staging_col is not None else torch.zeros(0, dtype=torch.int32)
    cols_in = ctx.alltoallv(col_send.to(torch.int32), send_nnz, recv_nnz)
    hdr_in = hdr_in.reshape(-1, 2)
    route = ContributionRoute(send_rows, send_nnz, recv_rows, recv_nnz,
                              [s for s in range(ctx.nranks) if recv_rows[s] > 0])
    return hdr_in[:, 0], hdr_in[:, 1], cols_in, route


def exchange_values(ctx: RankContext, staging_val, route: ContributionRoute, async_op=False):
    """Numeric exchange: values only, in the symbolic layout."""
    torch = _torch()
    send = staging_val if staging_val is not None else torch.zeros(0, dtype=torch.float64)
    return ctx.alltoallv(send, route.send_nnz, route.recv_nnz, async_op=async_op)


# ---------------------------------------------------------------------------
# test harness: spawn one process per rank (gloo) and collect results
# ---------------------------------------------------------------------------


def _rank_main(rank, nranks, port, program, queue, backend):
    if isinstance(program, bytes):
        import cloudpickle

        program = cloudpickle.loads(program)
    torch = _torch()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(nranks),
                      LOCAL_RANK="0")
    try:
        torch.distributed.init_process_group(backend=backend, rank=rank, world_size=nranks)
        dev = torch.device("cuda", 0) if torch.cuda.is_available() else torch.device("cpu")
        ctx = RankContext(rank, nranks, device=dev, backend=backend)
        res = program(ctx)
        queue.put((rank, "ok", res))
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    except BaseException as exc:  # report and let the parent re-raise
        import traceback

        queue.put((rank, "err", (repr(exc), traceback.format_exc(), exc)))


def spawn_ranks(nranks: int, program, *, backend: str = "gloo", timeout: float = 600.0, return_contexts=False,
                scheduler: str | None = None, trace=None):
    """Run ``program(ctx)`` on ``nranks`` ranks and return per-rank results
    (the reference's spawn_ranks contract, src/comm.py:325-344).  One rank
    runs inline; more ranks are forked processes joined over ``backend``
    (gloo on host tensors -- all ranks may share one GPU because no kernel
    ever waits on another rank)."""
    if nranks == 1:
        ctx = single_rank_context()
        res = program(ctx)
        return ([res], [ctx]) if return_contexts else [res]
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    # fresh interpreters (spawn): a forked child inherits the parent's CUDA
    # context and OpenMP thread-pool state, either of which can hang it; the
    # program (usually a closure) is shipped by value
    import cloudpickle

    mpctx = mp.get_context("spawn")
    payload = cloudpickle.dumps(program)
    q = mpctx.Queue()
    procs = [mpctx.Process(target=_rank_main, args=(r, nranks, port, payload, q, backend)) for r in range(nranks)]
    for p in procs:
        p.start()
    results = [None] * nranks
    errors = []
    for _ in range(nranks):
        rank, kind, payload = q.get(timeout=timeout)
        if kind == "ok":
            results[rank] = payload
        else:
            errors.append((rank, payload))
            break
    if errors:
        for p in procs:
            if p.is_alive():
                p.kill()
        rank, (msg, tb, exc) = errors[0]
        if isinstance(exc, BaseException):
            raise exc
        raise RuntimeError(f"rank {rank} failed: {msg}\n{tb}")
    for p in procs:
        p.join(timeout=60)
    return (results, None) if return_contexts else results
