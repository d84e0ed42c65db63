"""Config 3 level 1 at full size (256^3, 450 M nonzeros) on the device,
checked through size-independent properties (the oracle would take minutes
here): C is symmetric (A is), C x = P^T (A (P x)) for random x, and the three
algorithms agree to a row-scaled 1e-12.  Reference products use torch's
sparse CSR kernels -- library code, used only as the checker."""

import pytest

pytestmark = pytest.mark.gpu


def _csr(rp, col, val, shape, torch):
    return torch.sparse_csr_tensor(rp, col.to(torch.int64), val, size=shape)


def test_cfg3_full_size_properties():
    import torch

    import paper_1905_08423_b200 as pk
    from paper_1905_08423_b200 import devgen
    ctx = pk.single_rank_context()
    dev = ctx.device
    a, p = devgen.config_dist("cfg3", 1, 0, dev)
    n, m = a.nrows, p.ncols
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    rp, col, val = pk.run_numeric_device(a, p, plan, ctx)
    rp, col, val = rp.clone(), col.clone(), val.clone()
    del plan
    rows = torch.repeat_interleave(torch.arange(m, device=dev), rp[1:] - rp[:-1])
    scale = torch.zeros(m, dtype=torch.float64, device=dev)
    scale.scatter_reduce_(0, rows, val.abs(), reduce="amax")
    # symmetry: the transposed entry list equals the entry list
    key = rows * m + col.to(torch.int64)
    tkey = col.to(torch.int64) * m + rows
    order = torch.argsort(tkey)
    assert torch.equal(tkey[order], key), "pattern symmetric"
    d = (val[order] - val).abs() / scale[rows]
    assert float(d.max()) <= 1e-12
    # C x = P^T (A (P x))
    A = _csr(a.local.diag.row_ptr, a.local.diag.col, a.local.diag.val, (n, n), torch)
    P = _csr(p.local.diag.row_ptr, p.local.diag.col, p.local.diag.val, (n, m), torch)
    C = _csr(rp, col, val, (m, m), torch)
    g = torch.Generator(device=dev).manual_seed(7)
    for _ in range(2):
        x = torch.rand(m, dtype=torch.float64, device=dev, generator=g) * 2 - 1
        direct = C @ x
        via = (P.t() @ (A @ (P @ x)))
        err = (direct - via).abs().max() / direct.abs().max()
        assert float(err) <= 1e-12
    del A, P, C
    # the other algorithms agree
    for alg in ("merged", "two-step"):
        plan = pk.run_symbolic(a, p, alg, ctx)
        rp2, col2, val2 = pk.run_numeric_device(a, p, plan, ctx)
        assert torch.equal(rp2, rp) and torch.equal(col2, col), alg
        assert float(((val2 - val).abs() / scale[rows]).max()) <= 1e-12, alg
        del plan
