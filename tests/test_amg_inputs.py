"""Configs 4 and 5 (smoothed-aggregation P) at reduced size: generator
invariants on the CPU, the oracle on them, and CUDA parity (``-m gpu``)."""

import numpy as np
import pytest

from paper_1905_08423_b200 import problems_amg as amg
from tests.conftest import row_scaled_err, run_ptap

TOL = 1e-12


def _dense(m):
    d = np.zeros((m.nrows, m.ncols))
    for i in range(m.nrows):
        d[i, m.row_cols(i)] = m.row_values(i)
    return d


@pytest.fixture(scope="module")
def cfg4():
    return amg.block_transport(6)


@pytest.fixture(scope="module")
def cfg5():
    return amg.knn_laplacian(3000)


@pytest.fixture(scope="module")
def cfg4_wide():
    """12^3 nodes: C rows up to ~270 entries, past the byte-map limit, so the
    hash numeric path runs."""
    return amg.block_transport(12)


@pytest.fixture(scope="module")
def cfg5_large():
    return amg.knn_laplacian(20000)


def test_cfg4_generator_invariants(cfg4):
    A, P = cfg4
    assert A.nrows == 6 ** 3 * 10 and P.ncols == 2 ** 3 * 10
    d = _dense(A)
    assert np.array_equal(d, d.T), "A symmetric"
    off = np.abs(d).sum(axis=1) - np.abs(np.diag(d))
    assert np.all(np.diag(d) > off), "strictly diagonally dominant"
    assert np.all(np.diff(P.row_offsets) > 0)
    A2, P2 = amg.block_transport(6)
    assert np.array_equal(A.values.view(np.uint64), A2.values.view(np.uint64))
    assert np.array_equal(P.values.view(np.uint64), P2.values.view(np.uint64))


def test_cfg5_generator_invariants(cfg5):
    A, P = cfg5
    d = _dense(A)
    assert np.allclose(d, d.T, rtol=0, atol=0), "A symmetric"
    assert np.all(np.abs(np.diag(d) - (-(d - np.diag(np.diag(d))).sum(axis=1)) - 1e-3) < 1e-9), "Laplacian + 1e-3"
    deg = np.diff(A.row_offsets) - 1
    assert deg.min() >= 26, "every point keeps its 26 nearest neighbours"
    assert 20 < A.nrows / P.ncols < 120, "aggregation coarsening"
    assert np.all(np.diff(P.row_offsets) > 0)


@pytest.mark.parametrize("which", ["cfg4", "cfg5"])
def test_oracle_on_amg_inputs_matches_dense(which, request):
    """The oracle (pinned on the reference's goldens) on these inputs agrees
    with a dense P^T A P; this is the check the GPU tests then lean on."""
    from oracle.oracle import oracle_ptap
    A, P = request.getfixturevalue(which)
    w = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets,
                    P.col_indices, P.values, nranks=2, algorithm="allatonce")
    dense = _dense(P).T @ _dense(A) @ _dense(P)
    got = np.zeros_like(dense)
    for i in range(P.ncols):
        got[i, w.col[w.row_ptr[i]:w.row_ptr[i + 1]]] = w.val[w.row_ptr[i]:w.row_ptr[i + 1]]
    assert np.max(np.abs(got - dense)) <= 1e-12 * np.max(np.abs(dense))


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["cfg4", "cfg5", "cfg4_wide", "cfg5_large"])
@pytest.mark.parametrize("nr", [1, 2])
@pytest.mark.parametrize("alg", ["two-step", "allatonce", "merged"])
def test_gpu_parity_amg_inputs(which, nr, alg, request):
    from oracle.oracle import oracle_ptap
    A, P = request.getfixturevalue(which)
    want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets,
                       P.col_indices, P.values, nranks=nr, algorithm=alg)
    c, _ = run_ptap(A, P, nr, alg)
    assert np.array_equal(c.row_offsets, want.row_ptr)
    assert np.array_equal(c.col_indices, want.col)
    if alg == "two-step":
        assert np.array_equal(c.values.view(np.uint64), want.val.view(np.uint64))
    assert row_scaled_err(want.row_ptr, c.values, want.val) <= TOL


@pytest.mark.gpu
def test_map_policy_structured_vs_unstructured(cfg5_large):
    """Plan maps are kept when sampled rows repeat (a stencil: a handful of
    structural classes) and skipped when they do not (the kNN graph): that
    plan runs the hash numeric path and keeps no per-row maps.  Forcing maps
    (PTAP_MAPS=1) on the unstructured input gives the same C."""
    import os

    import paper_1905_08423_b200 as pk
    from oracle.oracle import oracle_ptap
    from paper_1905_08423_b200 import problems as gen

    ctx = pk.single_rank_context()
    A3, P3 = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=24)
    # numeric_path: 3 = plan maps run by the class-lockstep kernel, 1 = plan maps, 0 = hash tables
    for (A, P), paths in (((A3, P3), (1, 3)), (cfg5_large, (0,))):
        a, p = pk.distribute(A, P, 1, 0)
        plan = pk.run_symbolic(a, p, "allatonce", ctx)
        d = plan.device_counters()
        assert d["numeric_path"] in paths, d
        assert (d["map_bytes"] > 0) == (0 not in paths)
        assert 0 <= d["row_structures_ppm"] <= 10 ** 6
    A, P = cfg5_large
    want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets,
                       P.col_indices, P.values, nranks=1, algorithm="allatonce")
    os.environ["PTAP_MAPS"] = "1"
    try:
        c, _ = run_ptap(A, P, 1, "allatonce")
    finally:
        del os.environ["PTAP_MAPS"]
    assert np.array_equal(c.row_offsets, want.row_ptr) and np.array_equal(c.col_indices, want.col)
    assert row_scaled_err(want.row_ptr, c.values, want.val) <= TOL


def test_greedy_aggregation_compiled_matches_reference_loops():
    """The numba-compiled aggregation (used at config-5 scale) gives the same
    aggregates as the numpy restatement of the two passes."""
    import scipy.sparse as sp
    from scipy.spatial import cKDTree

    rng = np.random.default_rng(7)
    pts = rng.random((4000, 3))
    _, nb = cKDTree(pts).query(pts, k=9)
    r = np.repeat(np.arange(4000), 8)
    W = sp.csr_matrix((np.ones(r.size), (r, nb[:, 1:].ravel())), shape=(4000, 4000))
    W = (W + W.T).tocsr()
    W.sort_indices()
    a = amg._greedy_aggregate_py(W.indptr, W.indices, 4000)
    b = amg._greedy_aggregate(W.indptr, W.indices, 4000)
    assert np.array_equal(a, b)
    assert a.min() == 0 and np.all(np.diff(np.unique(a)) == 1)


def test_parallel_greedy_aggregation_matches_sequential_loops():
    """devgen's rounds-of-neighbourhood-minima aggregation (the device
    generator of config 5, run here on CPU tensors) gives exactly the
    aggregates of the sequential two-pass loops."""
    import scipy.sparse as sp
    import torch
    from scipy.spatial import cKDTree

    from paper_1905_08423_b200 import problems_amg as amg
    from paper_1905_08423_b200.devgen import _greedy_aggregate_device

    for npts, k, seed in ((500, 26, 1), (4000, 26, 20190520), (3000, 6, 7)):
        pts = np.random.default_rng(seed).random((npts, 3))
        _, nbr = cKDTree(pts).query(pts, k=k + 1)
        indptr = np.arange(0, npts * k + 1, k, dtype=np.int64)
        wd = sp.csr_matrix((np.ones(npts * k), nbr[:, 1:].ravel().astype(np.int64), indptr), shape=(npts, npts))
        w = wd.maximum(wd.T.tocsr()).tocsr()
        w.sort_indices()
        want = amg._greedy_aggregate(w.indptr, w.indices, npts)
        rows = torch.from_numpy(np.repeat(np.arange(npts), np.diff(w.indptr)))
        cols = torch.from_numpy(w.indices.astype(np.int64))
        agg, nagg = _greedy_aggregate_device(rows, cols, npts)
        assert nagg == int(want.max()) + 1
        assert np.array_equal(agg.numpy(), want)
