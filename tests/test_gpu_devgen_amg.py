"""Device generators of BASELINE configs 4 and 5 (csrc/ptap_gen.cu,
devgen.py) against the host generators (problems_amg.py), and the triple
product on device-generated operands against the CPU oracle."""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen
from paper_1905_08423_b200 import problems_amg as amg
from tests.conftest import row_scaled_err

pytestmark = pytest.mark.gpu


def _dev():
    return pk.single_rank_context().device


def _host(t):
    return t.cpu().numpy()


def _rel(got, want):
    return float(np.abs(got - want).max(initial=0.0) / max(np.abs(want).max(initial=0.0), 1e-300))


@pytest.mark.parametrize("nn,ncomp", [(4, 3), (7, 10), (9, 4)])
def test_block_transport_device_matches_host(nn, ncomp):
    """A bit for bit; P's pattern exact and its values to 1e-14 given the
    host's omega (scipy folds the smoothing sums in its own order), to 1e-12
    with the omega of the device's own power iteration."""
    import scipy.sparse as sp

    A, P = amg.block_transport(nn, ncomp=ncomp)
    n = nn ** 3 * ncomp
    As = sp.csr_matrix((A.values, A.col_indices, A.row_offsets), shape=(n, n))
    omega = (4.0 / 3.0) / amg._power_lambda_max(sp.diags(1.0 / As.diagonal()) @ As, 20190520)
    (arp, acol, aval), (prp, pcol, pval), _ = devgen.gen_block_transport_rows(nn, 0, n, _dev(), ncomp=ncomp,
                                                                             omega=omega)
    a_pattern = np.array_equal(_host(arp), A.row_offsets) and np.array_equal(_host(acol), A.col_indices)
    a_bits = a_pattern and np.array_equal(_host(aval).view(np.uint64), A.values.view(np.uint64))
    assert a_pattern and a_bits
    p_pattern = np.array_equal(_host(prp), P.row_offsets) and np.array_equal(_host(pcol), P.col_indices)
    assert p_pattern
    assert _rel(_host(pval), P.values) <= 1e-14
    _, (prp2, pcol2, pval2), om2 = devgen.gen_block_transport_rows(nn, 0, n, _dev(), ncomp=ncomp)
    assert abs(om2 - omega) <= 1e-13 * omega
    p2_pattern = np.array_equal(_host(pcol2), P.col_indices)
    assert p2_pattern and _rel(_host(pval2), P.values) <= 1e-12


def test_block_transport_row_blocks_tile_the_matrix():
    nn, ncomp = 6, 5
    n = nn ** 3 * ncomp
    (arp, acol, aval), (prp, pcol, pval), om = devgen.gen_block_transport_rows(nn, 0, n, _dev(), ncomp=ncomp)
    cut = n // 3 + 1
    parts = [devgen.gen_block_transport_rows(nn, lo, hi, _dev(), ncomp=ncomp, omega=om)
             for lo, hi in ((0, cut), (cut, n))]
    same = [np.array_equal(np.concatenate([_host(x[0][1]) for x in parts]), _host(acol)),
            np.array_equal(np.concatenate([_host(x[0][2]) for x in parts]), _host(aval)),
            np.array_equal(np.concatenate([_host(x[1][1]) for x in parts]), _host(pcol)),
            np.array_equal(np.concatenate([_host(x[1][2]) for x in parts]), _host(pval))]
    assert same == [True] * 4


@pytest.mark.parametrize("npts", [400, 5000, 40000])
def test_knn_laplacian_device_matches_host(npts):
    """The same graph (pattern exact), weights to 1e-13, the same aggregates
    (so P's pattern is exact) and P's values to 1e-12."""
    A, P = amg.knn_laplacian(npts)
    (arp, acol, aval), (prp, pcol, pval), nagg = devgen.gen_knn_laplacian(npts, _dev())
    a_pattern = np.array_equal(_host(arp), A.row_offsets) and np.array_equal(_host(acol), A.col_indices)
    assert a_pattern
    assert _rel(_host(aval), A.values) <= 1e-13
    assert nagg == P.ncols
    p_pattern = np.array_equal(_host(prp), P.row_offsets) and np.array_equal(_host(pcol), P.col_indices)
    assert p_pattern
    assert _rel(_host(pval), P.values) <= 1e-12


@pytest.mark.parametrize("which", ["cfg4", "cfg5"])
def test_ptap_on_device_generated_amg_inputs(which):
    """All three algorithms on device-generated operands against the oracle
    run on a host copy of the same operands."""
    from oracle.oracle import oracle_ptap
    from paper_1905_08423_b200.sparse import CsrMatrix

    ctx = pk.single_rank_context()
    if which == "cfg4":
        a, p = devgen.block_transport_dist(8, 1, 0, ctx.device, ncomp=6)
    else:
        a, p = devgen.knn_laplacian_dist(20000, 1, 0, ctx.device)

    def down(d):
        return CsrMatrix(d.nrows, d.ncols, d.row_ptr.cpu().numpy(), d.col.cpu().numpy().astype(np.int64),
                         d.val.cpu().numpy(), check=False)

    A, P = down(a.local.diag), down(p.local.diag)
    want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                       P.values, nranks=1, algorithm="allatonce")
    for alg in pk.ALGORITHMS:
        plan = pk.run_symbolic(a, p, alg, ctx)
        rp, col, val = pk.run_numeric_device(a, p, plan, ctx)
        plan.check()
        pattern = np.array_equal(rp.cpu().numpy(), want.row_ptr) and np.array_equal(col.cpu().numpy(), want.col)
        assert pattern, alg
        assert row_scaled_err(want.row_ptr, val.cpu().numpy(), want.val) <= 1e-12
