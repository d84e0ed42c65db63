"""Reference behaviours of the operator API on the CUDA path (tests mirror
the reference's tests/test_tripleproduct.py and tests/test_spgemm.py)."""

import os

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems as gen
from tests.conftest import csr_from_arrays, load_golden, row_scaled_err, run_ptap

pytestmark = pytest.mark.gpu

# Two all-at-once passes sum each C entry's ~13 contributions in whatever order
# the fp64 reductions land, so repeated or rearranged passes agree to a few
# ulps of the row's largest entry, not bitwise (measured up to 1.1e-15).
RUN_TOL = 1e-14


def _cfg3(n=16):
    return gen.config_operands(gen.CONFIGS["cfg3"], n_fine=n)


def test_repeated_numeric_protocol_one_symbolic_eleven_numeric():
    """1 symbolic + 11 numeric: counters, and the two-step passes
    are bitwise identical (deterministic ordered folds); all-at-once passes
    agree to a row-scaled RUN_TOL (atomics order varies)."""
    A, P = _cfg3()
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    for alg in pk.ALGORITHMS:
        plan = pk.run_symbolic(a, p, alg, ctx)
        outs = [pk.run_numeric(a, p, plan, ctx).diag.values.copy() for _ in range(11)]
        assert plan.counters.symbolic_runs == 1 and plan.counters.numeric_runs == 11
        ip = plan.c_alloc.local.diag.row_offsets
        for o in outs[1:]:
            if alg == "two-step":
                assert np.array_equal(o.view(np.uint64), outs[0].view(np.uint64))
            else:
                assert row_scaled_err(ip, o, outs[0]) <= RUN_TOL


def test_values_change_structure_fixed_linearity():
    """A scaled by 3 with a cached plan gives C scaled by 3 (dyadic scale:
    exact); the plan re-reads values every pass."""
    A, P = _cfg3()
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    for alg in pk.ALGORITHMS:
        plan = pk.run_symbolic(a, p, alg, ctx)
        c0 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
        a.local.diag.values *= 4.0
        c4 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
        a.local.diag.values /= 4.0
        ip = plan.c_alloc.local.diag.row_offsets
        assert row_scaled_err(ip, c4, 4.0 * c0) <= RUN_TOL


def test_cache_free_releases_plan_keeps_c():
    A, P = _cfg3()
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    for alg in pk.ALGORITHMS:
        c, plan = pk.ptap(a, p, alg, ctx, cache="free")
        assert c.local.nnz > 0 and plan.released
        mem = plan.memory()
        assert mem["current"]["plan_cache"] == 0 and mem["current"]["auxiliary_matrices"] == 0
        assert mem["current"]["output_matrix"] > 0
        with pytest.raises(pk.StructuralDriftError):
            pk.run_numeric(a, p, plan, ctx)


def test_structure_change_is_drift():
    A, P = _cfg3()
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    A2, _ = _cfg3(18)
    A3 = pk.CsrMatrix(A.nrows, A.ncols, A2.row_offsets[:A.nrows + 1], A2.col_indices[:A2.row_offsets[A.nrows]] % A.ncols,
                      A2.values[:A2.row_offsets[A.nrows]], check=False)
    a3, _ = pk.distribute(A3, P, 1, 0)
    with pytest.raises(pk.StructuralDriftError):
        pk.run_numeric(a3, p, plan, ctx)


def test_zero_a_gives_stored_zeros_on_device():
    A, P = _cfg3()
    Z = pk.CsrMatrix(A.nrows, A.ncols, A.row_offsets, A.col_indices, np.zeros(A.nnz))
    for alg in pk.ALGORITHMS:
        cz, _ = run_ptap(Z, P, 1, alg)
        c, _ = run_ptap(A, P, 1, alg)
        assert cz.structure_equal(c) and np.all(cz.values == 0.0)


def test_memory_two_step_vs_all_at_once():
    """aux: the outer-product variants store no auxiliary matrix (ledger
    category 0, SPEC C4); two-step books C~ and P^T there."""
    A, P = _cfg3(24)
    for alg in pk.ALGORITHMS:
        _, res = run_ptap(A, P, 1, alg)
        snap = res[0][2]
        if alg == "two-step":
            assert snap.peak["auxiliary_matrices"] > 0
        else:
            assert snap.peak["auxiliary_matrices"] == 0


def test_mapped_and_hash_numeric_paths_agree():
    """The plan-mapped numeric pass (default) and the hash pass
    (PTAP_NO_MAPS=1) give the same C (row-scaled RUN_TOL)."""
    A, P = _cfg3(20)
    c_map, _ = run_ptap(A, P, 1, "allatonce")
    os.environ["PTAP_NO_MAPS"] = "1"
    try:
        c_hash, _ = run_ptap(A, P, 1, "allatonce")
    finally:
        del os.environ["PTAP_NO_MAPS"]
    assert c_map.structure_equal(c_hash)
    assert row_scaled_err(c_map.row_offsets, c_map.values, c_hash.values) <= RUN_TOL


def test_interned_maps_shrink_plan_and_match_private_maps():
    """Rows of one structural class share one interned slot/position map:
    the plan keeps a fraction of the per-row map bytes, and C equals the C of
    a plan with a private map per row (PTAP_NO_INTERN=1)."""
    A, P = _cfg3(32)
    ctx = pk.single_rank_context()

    def one():
        a, p = pk.distribute(A, P, 1, 0)
        plan = pk.run_symbolic(a, p, "allatonce", ctx)
        loc = pk.run_numeric(a, p, plan, ctx)
        return loc.diag.row_offsets.copy(), loc.diag.col_indices.copy(), loc.diag.values.copy(), \
            plan.memory()["current"]["plan_cache"]

    ip, j, v, shared = one()
    os.environ["PTAP_NO_INTERN"] = "1"
    try:
        ip2, j2, v2, private = one()
    finally:
        del os.environ["PTAP_NO_INTERN"]
    assert np.array_equal(ip, ip2) and np.array_equal(j, j2)
    assert row_scaled_err(ip, v, v2) <= RUN_TOL
    assert shared < 0.5 * private, (shared, private)


def test_device_generators_match_host_generators():
    import torch
    from paper_1905_08423_b200 import devgen
    for name, n in (("cfg1", 16), ("cfg3", 16)):
        spec = gen.CONFIGS[name]
        A, P = gen.config_operands(spec, n_fine=n)
        for (lo, hi) in ((0, n ** 3), (100, 2000)):
            rp, col, val = devgen.gen_stencil_rows(n, spec.points, 0 if spec.points == 7 else 1, spec.seed, lo, hi,
                                                   torch.device("cuda"))
            a0, a1 = A.row_offsets[lo], A.row_offsets[hi]
            assert np.array_equal(rp.cpu().numpy(), A.row_offsets[lo:hi + 1] - a0)
            assert np.array_equal(col.cpu().numpy(), A.col_indices[a0:a1])
            assert np.array_equal(val.cpu().numpy().view(np.uint64), A.values[a0:a1].view(np.uint64))
        rp, col, val = devgen.gen_trilinear_rows(n // 2, 0, n ** 3, torch.device("cuda"))
        assert np.array_equal(rp.cpu().numpy(), P.row_offsets)
        assert np.array_equal(col.cpu().numpy(), P.col_indices)
        assert np.array_equal(val.cpu().numpy(), P.values)


def test_two_level_hierarchy_level2_parity():
    """Config-3 style hierarchy: level-2 A is level-1 C (kept on the device
    path through the API); both levels against the oracle."""
    from oracle.oracle import oracle_ptap
    A, P = _cfg3(16)
    c1, _ = run_ptap(A, P, 1, "two-step")
    P2 = gen.trilinear(4)
    w1 = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                     P.values, algorithm="two-step")
    assert np.array_equal(c1.values.view(np.uint64), w1.val.view(np.uint64))
    for alg in pk.ALGORITHMS:
        c2, _ = run_ptap(c1, P2, 1, alg)
        w2 = oracle_ptap(c1.nrows, P2.ncols, c1.row_offsets, c1.col_indices, c1.values, P2.row_offsets,
                         P2.col_indices, P2.values, algorithm=alg)
        assert np.array_equal(c2.row_offsets, w2.row_ptr) and np.array_equal(c2.col_indices, w2.col)
        assert row_scaled_err(w2.row_ptr, c2.values, w2.val) <= 1e-12


def test_standalone_spgemm_matches_reference_golden():
    """symbolic_ap / numeric_ap (src/spgemm.py:184-234): AP rows bit-exact
    against a host product in the reference's fold order."""
    from paper_1905_08423_b200.spgemm import numeric_ap, symbolic_ap
    n, m, a, p, _ = load_golden("random_instance_s11")
    A = csr_from_arrays(n, n, *a)
    P = csr_from_arrays(n, m, *p)
    ctx = pk.single_rank_context()
    ad, pd = pk.distribute(A, P, 1, 0)
    c = numeric_ap(ad, pd, symbolic_ap(ad, pd, ctx), ctx).to_host()
    # host fold: for each row, A entries ascending, first product sets
    for i in range(n):
        acc = {}
        for t in range(A.row_offsets[i], A.row_offsets[i + 1]):
            k, av = A.col_indices[t], A.values[t]
            for u in range(P.row_offsets[k], P.row_offsets[k + 1]):
                g = P.col_indices[u]
                acc[g] = acc[g] + av * P.values[u] if g in acc else av * P.values[u]
        cols = sorted(acc)
        assert c.row_cols(i).tolist() == cols
        assert np.array_equal(np.array([acc[g] for g in cols]).view(np.uint64), c.row_values(i).view(np.uint64))


def test_streamed_host_numeric_matches_one_shot():
    """At one rank the all-at-once pass with host operands streams A's values
    up in row blocks and final C rows back; the result equals the one-shot
    path (same kernels) within the atomics' row-scaled RUN_TOL, for several
    block counts, and numeric_runs counts passes, not blocks."""
    A, P = _cfg3(20)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    os.environ["PTAP_UPLOAD_BLOCKS"] = "1"
    try:
        ref = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
    finally:
        del os.environ["PTAP_UPLOAD_BLOCKS"]
    ip = plan.c_alloc.local.diag.row_offsets
    for blocks in ("8", "3", "17"):
        os.environ["PTAP_UPLOAD_BLOCKS"] = blocks
        try:
            got = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
        finally:
            del os.environ["PTAP_UPLOAD_BLOCKS"]
        assert row_scaled_err(ip, got, ref) <= RUN_TOL
    assert plan.counters.numeric_runs == 4


def test_streamed_path_falls_back_when_rows_not_range_addressable():
    """Config-4 rows (wide P rows: > 128 fold pairs) take the generic mapped
    kernel, so the streamed host pass is declined on the first call and the
    one-shot path produces C (same values both calls)."""
    from paper_1905_08423_b200 import problems_amg as amg
    A, P = amg.block_transport(6)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    c1 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
    assert getattr(plan, "_stream_ok", True) is False
    c2 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
    ip = plan.c_alloc.local.diag.row_offsets
    assert row_scaled_err(ip, c2, c1) <= RUN_TOL
    assert plan.counters.numeric_runs == 2


def test_device_transpose_matches_reference_semantics():
    """DeviceCsr.transpose_with_permutation (ptap_transpose) against the
    host definition of the reference (stable argsort of the columns,
    src/sparse.py:165-178): identical structure, permutation and values."""
    from paper_1905_08423_b200.device import DeviceCsr
    rng = np.random.default_rng(3)
    for (n, m, dens) in ((40, 25, 0.2), (1000, 3000, 0.003), (5, 7, 0.0)):
        mask = rng.random((n, m)) < dens
        rows, cols = np.nonzero(mask)
        ip = np.zeros(n + 1, np.int64)
        np.add.at(ip, rows + 1, 1)
        ip = np.cumsum(ip)
        vals = rng.standard_normal(rows.size)
        A = pk.CsrMatrix(n, m, ip, cols, vals)
        d = DeviceCsr.from_host(A, "cuda")
        t, perm = d.transpose_with_permutation()
        want_perm = np.argsort(cols, kind="stable")
        want_ip = np.zeros(m + 1, np.int64)
        np.add.at(want_ip, cols + 1, 1)
        want_ip = np.cumsum(want_ip)
        assert np.array_equal(t.row_ptr.cpu().numpy(), want_ip)
        assert np.array_equal(t.col.cpu().numpy(), rows[want_perm])
        assert np.array_equal(perm.cpu().numpy(), want_perm)
        assert np.array_equal(t.val.cpu().numpy().view(np.uint64), vals[want_perm].view(np.uint64))
