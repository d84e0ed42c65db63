"""Device-side construction of the BASELINE operands (configs 1-5) as
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


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def gen_block_transport_rows(nn: int, lo: int, hi: int, device, ncomp: int = 10, seed: int = 20190520,
                             agg: int = 3, omega: float | None = None):
    """Config 4 on the device (problems_amg.block_transport): rows [lo, hi)
    of A and of the smoothed-aggregation P with global columns.  ``omega`` is
    (4/3) / lambda_max(D^-1 A) from 10 power iterations over the whole matrix
    started from numpy's default_rng(seed) vector, as in the host generator
    (computed here on the device when not given).  Returns
    ((a_rp, a_col, a_val), (p_rp, p_col, p_val), omega)."""
    torch = _torch()
    L = _lib.load()
    n = nn ** 3 * ncomp

    def rows(r_lo, r_hi, want_p=True):
        nr = r_hi - r_lo
        arp = torch.zeros(nr + 1, dtype=torch.int64, device=device)
        prp = torch.zeros(nr + 1, dtype=torch.int64, device=device)
        annz, pnnz = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.ptap_gen_block_transport_rowptr(nn, ncomp, agg, r_lo, r_hi, _ptr(arp), ctypes.byref(annz),
                                                     _ptr(prp), ctypes.byref(pnnz), _stream()), "gen rowptr")
        acol = torch.empty(annz.value, dtype=torch.int32, device=device)
        aval = torch.empty(annz.value, dtype=torch.float64, device=device)
        _lib.check(L.ptap_gen_block_transport_a(nn, ncomp, seed, r_lo, r_hi, _ptr(arp), _ptr(acol), _ptr(aval),
                                                _stream()), "gen A")
        return arp, acol, aval, prp, pnnz.value

    if omega is None:
        import numpy as np

        arp, acol, aval, _, _ = rows(0, n)
        v = torch.from_numpy(np.random.default_rng(seed).random(n)).to(device)
        w = torch.empty_like(v)
        lam = 0.0
        for _ in range(10):
            _lib.check(L.ptap_gen_spmv_dinv(n, _ptr(arp), _ptr(acol), _ptr(aval), _ptr(v), _ptr(w), _stream()),
                       "gen spmv")
            nw = torch.linalg.norm(w)
            lam = float(nw / torch.linalg.norm(v))
            v = w / nw
            w = torch.empty_like(v)
        omega = (4.0 / 3.0) / lam
        if (lo, hi) != (0, n):
            del arp, acol, aval
    arp, acol, aval, prp, pnnz = rows(lo, hi)
    pcol = torch.empty(pnnz, dtype=torch.int32, device=device)
    pval = torch.empty(pnnz, dtype=torch.float64, device=device)
    _lib.check(L.ptap_gen_block_transport_p(nn, ncomp, agg, float(omega), lo, hi, _ptr(arp), _ptr(aval), _ptr(prp),
                                            _ptr(pcol), _ptr(pval), _stream()), "gen P")
    return (arp, acol, aval), (prp, pcol, pval), omega


def block_transport_dist(nn: int, nranks: int, rank: int, device, ncomp: int = 10, seed: int = 20190520,
                         agg: int = 3, omega: float | None = None):
    """(A, P) DistMatrix pair of config 4 for one rank, generated on the
    device (row blocks of nodes x components; coarse columns in row blocks)."""
    n = nn ** 3 * ncomp
    na = -(-nn // agg)
    m = na ** 3 * ncomp
    row_part = make_partition(n, nranks)
    col_part = make_partition(m, nranks)
    lo, hi = row_part.owned_range(rank)
    clo, chi = col_part.owned_range(rank)
    (arp, acol, aval), (prp, pcol, pval), _ = gen_block_transport_rows(nn, lo, hi, device, ncomp, seed, agg, omega)
    a_loc = split_rows_device(arp, acol, aval, lo, hi, lo, hi, n)
    p_loc = split_rows_device(prp, pcol, pval, lo, hi, clo, chi, m)
    return DistMatrix(row_part, row_part, rank, a_loc), DistMatrix(row_part, col_part, rank, p_loc)


def _greedy_aggregate_device(rows, cols, n: int):
    """problems_amg._greedy_aggregate on the device.  Pass 1 (a point none of
    whose neighbours is aggregated roots an aggregate of itself and its
    neighbours, natural order) is the lexicographically first set of roots
    pairwise more than two edges apart: a point becomes a root once every
    lower-numbered point within two edges is known not to be one, and a
    non-root once a root lies within two edges (rounds of neighbourhood
    minima).  Pass 2 (a leftover joins the aggregate of its smallest-index
    aggregated neighbour, earlier leftovers included) is one neighbourhood
    minimum and pointer jumping along the chains of leftovers."""
    torch = _torch()
    dev = rows.device
    idx = torch.arange(n, device=dev)
    BIG = n
    U, R, N = 0, 1, 2
    state = torch.zeros(n, dtype=torch.int8, device=dev)

    def nbr_min(x):  # min over the closed neighbourhood
        out = x.clone()
        out.scatter_reduce_(0, rows, x[cols], reduce="amin", include_self=True)
        return out

    while True:
        cand = torch.where(state != N, idx, torch.full_like(idx, BIG))
        a2 = nbr_min(nbr_min(cand))
        state[(state == U) & (a2 == idx)] = R
        near = (state == R).to(torch.int64)
        near = -nbr_min(nbr_min(-near))  # max over two closed neighbourhoods
        state[(state == U) & (near > 0)] = N
        if not bool((state == U).any()):
            break
    root = state == R
    root_id = torch.cumsum(root.to(torch.int64), 0) - 1
    nagg = int(root_id[-1].item()) + 1 if n else 0
    agg = torch.where(root, root_id, torch.full_like(idx, -1))
    er = root[rows]
    agg[cols[er]] = root_id[rows[er]]  # roots are more than two edges apart: no point has two
    left = agg < 0
    if bool(left.any()):
        agg1 = agg.clone()
        ok = (agg1[cols] >= 0) | (cols < rows)
        cand = torch.where(ok & left[rows] & (cols != rows), cols, torch.full_like(cols, BIG))
        best = torch.full_like(idx, BIG)
        best.scatter_reduce_(0, rows, cand, reduce="amin", include_self=True)
        fresh = left & (best == BIG)  # no aggregated neighbour at all: a new aggregate, in index order
        agg[fresh] = nagg + torch.cumsum(fresh.to(torch.int64), 0)[fresh] - 1
        nagg += int(fresh.sum().item())
        todo = left & ~fresh
        while bool(todo.any()):
            b = best[todo]
            got = agg[b]
            ti = idx[todo]
            agg[ti] = got  # -1 where the chain's head is still unresolved
            todo = left & (agg < 0)
    return agg, nagg


def gen_knn_laplacian(npts: int, device, k: int = 26, seed: int = 20190520):
    """Config 5 on the device (problems_amg.knn_laplacian): the symmetric
    k-nearest-neighbour graph Laplacian and its smoothed-aggregation P as
    global CSR device tensors ((a_rp, a_col, a_val), (p_rp, p_col, p_val), nagg).
    The points come from numpy's default_rng(seed) as in the host generator;
    the neighbour search is the CUDA kernel k_knn_cells, the rest (edge union,
    aggregation, smoothing) device tensor operations."""
    import numpy as np

    torch = _torch()
    L = _lib.load()
    n = int(npts)
    pts = torch.from_numpy(np.random.default_rng(seed).random((n, 3))).to(device)
    # points sorted by cell of a G^3 grid, about 16 per cell
    G = max(1, int(round((n / 16.0) ** (1.0 / 3.0))))
    cc = torch.clamp((pts * G).to(torch.int64), max=G - 1)
    cell = cc[:, 0] + G * (cc[:, 1] + G * cc[:, 2])
    order = torch.argsort(cell, stable=True)
    spts = pts[order].contiguous()
    cnt = torch.bincount(cell, minlength=G ** 3)
    cstart = torch.zeros(G ** 3 + 1, dtype=torch.int64, device=device)
    torch.cumsum(cnt, 0, out=cstart[1:])
    del cc, cell, cnt
    kk = min(k, max(n - 1, 0))
    nbr = torch.empty(n * max(kk, 1), dtype=torch.int32, device=device)
    d2 = torch.empty(n * max(kk, 1), dtype=torch.float64, device=device)
    if kk > 0:
        _lib.check(L.ptap_gen_knn(n, _ptr(spts), _ptr(cstart), G, kk, _ptr(nbr), _ptr(d2), _stream()), "gen knn")
    del d2, spts, cstart
    # directed edges in original numbering, both directions plus the diagonal, unique
    src = order.repeat_interleave(kk)
    dst = order[nbr.to(torch.int64)] if kk > 0 else src
    del nbr
    keys = torch.cat((src * n + dst, dst * n + src, torch.arange(n, device=device) * (n + 1)))
    del src, dst, order
    keys = torch.unique(keys)
    rows = torch.div(keys, n, rounding_mode="floor")
    cols = keys - rows * n
    del keys
    # weights 1 / distance, the squared distance folded x, y, z in order
    dx = pts[rows, 0] - pts[cols, 0]
    dsq = dx * dx
    dx = pts[rows, 1] - pts[cols, 1]
    dsq = dsq + dx * dx
    dx = pts[rows, 2] - pts[cols, 2]
    dsq = dsq + dx * dx
    del dx
    offd = rows != cols
    w = torch.where(offd, 1.0 / torch.sqrt(dsq), torch.zeros_like(dsq))
    del dsq
    deg = torch.zeros(n, dtype=torch.float64, device=device).index_add_(0, rows, w)
    aval = torch.where(offd, -w, (deg + 1e-3)[rows])
    a_rp = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(torch.bincount(rows, minlength=n), 0, out=a_rp[1:])
    a_col = cols.to(torch.int32)
    # aggregation over the off-diagonal graph, then P = (I - omega D^-1 A) P_tent
    agg, nagg = _greedy_aggregate_device(rows[offd], cols[offd], n)
    diag = deg + 1e-3
    dinv = 1.0 / diag
    rowsum = torch.zeros(n, dtype=torch.float64, device=device).index_add_(0, rows, aval.abs()) * dinv
    omega = (2.0 / 3.0) / float(rowsum.max().item())
    da = dinv[rows] * aval
    pkey, inv = torch.unique(rows * nagg + agg[cols], return_inverse=True)
    sums = torch.zeros(pkey.numel(), dtype=torch.float64, device=device).index_add_(0, inv, da)
    del inv, da, w
    prow = torch.div(pkey, nagg, rounding_mode="floor")
    pcolv = pkey - prow * nagg
    tent = pcolv == agg[prow]
    pval = torch.where(tent, 1.0 - omega * sums, -(omega * sums))
    p_rp = torch.zeros(n + 1, dtype=torch.int64, device=device)
    torch.cumsum(torch.bincount(prow, minlength=n), 0, out=p_rp[1:])
    return (a_rp, a_col, aval), (p_rp, pcolv.to(torch.int32), pval), nagg


def _row_block(rp, col, val, lo, hi):
    e0, e1 = int(rp[lo].item()), int(rp[hi].item())
    return (rp[lo:hi + 1] - e0).contiguous(), col[e0:e1].contiguous(), val[e0:e1].contiguous()


def knn_laplacian_dist(npts: int, nranks: int, rank: int, device, k: int = 26, seed: int = 20190520):
    """(A, P) DistMatrix pair of config 5 for one rank, generated on the
    device (the graph is global: every rank builds it and keeps its rows)."""
    (arp, acol, aval), (prp, pcol, pval), nagg = gen_knn_laplacian(npts, device, k, seed)
    row_part = make_partition(npts, nranks)
    col_part = make_partition(nagg, nranks)
    lo, hi = row_part.owned_range(rank)
    clo, chi = col_part.owned_range(rank)
    a_loc = split_rows_device(*_row_block(arp, acol, aval, lo, hi), lo, hi, lo, hi, npts)
    p_loc = split_rows_device(*_row_block(prp, pcol, pval, lo, hi), lo, hi, clo, chi, nagg)
    return DistMatrix(row_part, row_part, rank, a_loc), DistMatrix(row_part, col_part, rank, p_loc)


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
