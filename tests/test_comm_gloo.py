"""Multi-rank host logic over torch.distributed/gloo (world_size 2, CPU).

Covers the two exchange patterns of the triple product with the code the
GPU path runs (comm.py), on host tensors: the remote-row gather of P with its
values-only refresh (reference src/comm.py:561-649; toy golden from
tests/test_comm.py:92-101), and the owner-directed C_s exchange with its
ascending-source ordering and ownership checks (src/comm.py:452-486).
"""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import comm
from paper_1905_08423_b200.device import DeviceLocalMatrix

TOY_A = [(0, 0, 1.0), (0, 1, 1.0), (0, 4, 1.0), (1, 1, 1.0), (1, 2, 1.0), (1, 4, 1.0),
         (2, 0, 1.0), (2, 3, 1.0), (2, 4, 1.0), (3, 1, 1.0), (3, 3, 1.0), (4, 3, 1.0),
         (4, 4, 1.0), (5, 1, 1.0), (5, 4, 1.0), (5, 5, 1.0)]
TOY_P = [(0, 0, 1.0), (0, 3, 1.0), (1, 1, 1.0), (2, 2, 1.0), (2, 3, 1.0), (3, 2, 1.0),
         (4, 1, 1.0), (4, 3, 1.0), (5, 2, 1.0)]


def _toy(nranks, rank):
    import torch
    a = pk.csr_from_triplets(6, 6, TOY_A)
    p = pk.csr_from_triplets(6, 4, TOY_P)
    ad, pd = pk.distribute(a, p, nranks, rank)
    return ad, pd, DeviceLocalMatrix.from_local(pd.local, torch.device("cpu"))


def test_alltoallv_roundtrip():
    def prog(ctx):
        import torch
        counts = np.array([ctx.rank + 1, 2], np.int64)  # to rank 0, to rank 1
        send = torch.arange(int(counts.sum()), dtype=torch.int64) + 100 * ctx.rank
        recv_counts = ctx.exchange_counts(counts)
        out = ctx.alltoallv(send, counts, recv_counts)
        return recv_counts.tolist(), out.tolist()

    r0, r1 = pk.spawn_ranks(2, prog)
    assert r0 == ([1, 2], [0, 100, 101])
    assert r1 == ([2, 2], [1, 2, 102, 103])


def test_gather_remote_rows_toy_golden():
    """3 ranks: rank 0 requests P rows [2, 4] -> [[2, 3], [1, 3]]."""
    def prog(ctx):
        ad, pd, pdev = _toy(ctx.nranks, ctx.rank)
        rr = comm.gather_remote_rows(ctx, ad.local.col_map, pd.row_part, pdev)
        rp = rr.row_ptr.numpy()
        cols = rr.col.numpy()
        rows = [cols[rp[k]:rp[k + 1]].tolist() for k in range(rp.size - 1)]
        return rr.source_cols.tolist(), rows, rr.val.numpy().tolist()

    res = pk.spawn_ranks(3, prog)
    assert res[0][0] == [2, 4]
    assert res[0][1] == [[2, 3], [1, 3]]
    assert all(v == 1.0 for v in res[0][2])


def test_values_refresh_equals_fresh_gather():
    def prog(ctx):
        import torch
        ad, pd, pdev = _toy(ctx.nranks, ctx.rank)
        rr = comm.gather_remote_rows(ctx, ad.local.col_map, pd.row_part, pdev)
        # scale P's values on every rank, refresh values only
        pdev.diag.val.mul_(3.0)
        pdev.offdiag.val.mul_(3.0)
        comm.refresh_remote_values(ctx, rr, pdev)
        fresh = comm.gather_remote_rows(ctx, ad.local.col_map, pd.row_part, pdev)
        return torch.equal(rr.val, fresh.val), torch.equal(rr.col, fresh.col)

    for eq_v, eq_c in pk.spawn_ranks(2, prog):
        assert eq_v and eq_c


def test_contribution_exchange_orders_by_source():
    """Every rank stages rows owned by the others; the receiver gets them
    concatenated in ascending source rank with values in the symbolic layout."""
    def prog(ctx):
        import torch
        cpart = pk.make_partition(9, ctx.nranks)
        mine = set(range(*cpart.owned_range(ctx.rank)))
        rows = np.array([r for r in range(9) if r not in mine], np.int32)
        widths = (rows % 3) + 1
        rp = np.concatenate(([0], np.cumsum(widths))).astype(np.int64)
        cols = np.concatenate([np.arange(w) + 10 * ctx.rank for w in widths]).astype(np.int32)
        r_in, w_in, c_in, route = comm.exchange_structure(
            ctx, torch.as_tensor(rows), torch.as_tensor(rp), torch.as_tensor(cols), cpart)
        vals = torch.arange(int(rp[-1]), dtype=torch.float64) + 1000 * ctx.rank
        v_in = comm.exchange_values(ctx, vals, route)
        return r_in.tolist(), w_in.tolist(), c_in.tolist(), v_in.tolist(), route.recv_src_ranks

    res = pk.spawn_ranks(3, prog)
    r_in, w_in, c_in, v_in, srcs = res[1]
    # rank 1 owns rows [3, 6); it receives them from rank 0 then rank 2
    assert srcs == [0, 2]
    assert r_in == [3, 4, 5, 3, 4, 5]
    assert w_in == [1, 2, 3, 1, 2, 3]
    assert c_in[:6] == [0, 0, 1, 0, 1, 2] and c_in[6:] == [20, 20, 21, 20, 21, 22]
    assert all(v < 1000 for v in v_in[:6]) and all(v >= 2000 for v in v_in[6:])


def test_staging_rows_owned_locally_are_rejected():
    def prog(ctx):
        import torch
        cpart = pk.make_partition(4, ctx.nranks)
        lo, _ = cpart.owned_range(ctx.rank)
        try:
            comm.exchange_structure(ctx, torch.tensor([lo], dtype=torch.int32),
                                    torch.tensor([0, 1], dtype=torch.int64),
                                    torch.tensor([0], dtype=torch.int32), cpart)
        except pk.OwnershipError:
            return "raised"
        return "no error"

    assert pk.spawn_ranks(2, prog) == ["raised", "raised"]


def test_rank_failure_propagates():
    def prog(ctx):
        if ctx.rank == 1:
            raise ValueError("boom")
        return 0

    with pytest.raises(ValueError, match="boom"):
        pk.spawn_ranks(2, prog, timeout=120)
