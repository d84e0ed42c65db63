"""The class-lockstep numeric kernel (csrc/ptap_lock.cu) and the single-shot
pass (symbolic and numeric together, BASELINE north_star (3)) against the
reference's own golden outputs and the CPU oracle.

Gates: pattern (row_ptr, sorted columns) bit-exact; values
row-scaled <= 1e-12 (summation order differs: fused multiply-adds and a
slot-major fold in the lockstep kernel, atomics into the arena in the
single-shot pass)."""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems as gen
from tests.conftest import csr_from_arrays, golden_cases, load_golden, row_scaled_err

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _assemble(local, P):
    return pk.assemble_global([local], ncols=P.ncols)


def _oracle(A, P):
    from oracle.oracle import oracle_ptap

    return oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                       P.values, nranks=1, algorithm="allatonce")


@pytest.mark.parametrize("cfg,nf", [("cfg1", 16), ("cfg2", 32), ("cfg3", 8), ("cfg3", 24), ("cfg3", 40)])
@pytest.mark.parametrize("alg", ["allatonce", "merged"])
def test_lockstep_kernel_matches_oracle_and_per_row_kernels(cfg, nf, alg):
    """Structured grids take the lockstep kernel (numeric_path 3); its C has
    the oracle's pattern and values within the gate, and agrees with the
    per-row mapped kernels (lockstep=False, numeric_path 1) on the same plan
    inputs; eleven passes stay within the run-to-run tolerance."""
    A, P = gen.config_operands(gen.CONFIGS[cfg], n_fine=nf)
    want = _oracle(A, P)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, alg, ctx)
    assert plan.device_counters()["numeric_path"] == 3
    g = _assemble(pk.run_numeric(a, p, plan, ctx), P)
    assert np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
    assert row_scaled_err(want.row_ptr, g.values, want.val) <= TOL
    # per-entry relative error on the entries that are not cancellation-dominated
    rows = np.repeat(np.arange(want.row_ptr.size - 1), np.diff(want.row_ptr))
    rmax = np.zeros(want.row_ptr.size - 1)
    np.maximum.at(rmax, rows, np.abs(want.val))
    big = np.abs(want.val) >= 1e-3 * rmax[rows]
    per_entry = float((np.abs(g.values - want.val)[big] / np.abs(want.val)[big]).max(initial=0.0))
    assert per_entry <= TOL
    first = g.values.copy()
    for _ in range(10):
        again = pk.run_numeric(a, p, plan, ctx).diag.values
        assert row_scaled_err(want.row_ptr, again, first) <= 1e-14
    plan1 = pk.run_symbolic(a, p, alg, ctx, lockstep=False)
    assert plan1.device_counters()["numeric_path"] == 1
    g1 = _assemble(pk.run_numeric(a, p, plan1, ctx), P)
    assert np.array_equal(g1.col_indices, g.col_indices)
    assert row_scaled_err(want.row_ptr, g1.values, first) <= 1e-14


def test_lockstep_values_change_between_passes():
    """P's class-major copy (Q) is rebuilt every pass: scaling P by 2 scales C
    by 4 exactly (dyadic), scaling A back and forth returns the first C."""
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=16)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    assert plan.device_counters()["numeric_path"] == 3
    c0 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
    ip = plan.c_alloc.local.diag.row_offsets
    p.local.diag.values *= 2.0
    c4 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
    p.local.diag.values /= 2.0
    assert row_scaled_err(ip, c4, 4.0 * c0) <= 1e-14
    a.local.diag.values *= 8.0
    c8 = pk.run_numeric(a, p, plan, ctx).diag.values.copy()
    a.local.diag.values /= 8.0
    assert row_scaled_err(ip, c8, 8.0 * c0) <= 1e-14


@pytest.mark.parametrize("name", golden_cases())
@pytest.mark.parametrize("alg", ["allatonce", "merged"])
def test_single_shot_matches_reference_goldens(name, alg):
    """ptap(..., single_shot=True): C of the reference's own np=1 run, pattern
    bit-exact, values within the gate, with no numeric call made; the plan
    stays usable (a later numeric pass gives the same C through the hash
    path)."""
    n, m, (a_ip, a_j, a_v), (p_ip, p_j, p_v), results = load_golden(name)
    if (1, alg) not in results:
        pytest.skip("no np=1 result stored")
    A = csr_from_arrays(n, n, a_ip, a_j, a_v)
    P = csr_from_arrays(n, m, p_ip, p_j, p_v)
    w_ip, w_j, w_v = results[(1, alg)]
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    c, plan = pk.ptap(a, p, alg, ctx, single_shot=True)
    assert plan.values_ready
    assert plan.counters.numeric_runs == 0 and plan.counters.symbolic_runs == 1
    g = pk.assemble_global([c.local], ncols=m)
    assert np.array_equal(g.row_offsets, w_ip) and np.array_equal(g.col_indices, w_j)
    assert row_scaled_err(w_ip, g.values, w_v) <= TOL
    g2 = pk.assemble_global([pk.run_numeric(a, p, plan, ctx)], ncols=m)
    assert plan.device_counters()["numeric_path"] == 0
    assert row_scaled_err(w_ip, g2.values, w_v) <= TOL


def test_single_shot_falls_back_when_rows_are_exchanged():
    """With two ranks the rank sends and receives contributions: the option
    is ignored (values_ready False) and the usual two phases run."""
    from oracle.oracle import oracle_ptap

    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=12)
    want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                       P.values, nranks=2, algorithm="allatonce")

    def prog(ctx):
        a, p = pk.distribute(A, P, ctx.nranks, ctx.rank)
        c, plan = pk.ptap(a, p, "allatonce", ctx, single_shot=True)
        return c.local, plan.values_ready

    res = pk.spawn_ranks(2, prog)
    assert not any(r[1] for r in res)
    g = pk.assemble_global([r[0] for r in res], ncols=P.ncols)
    assert np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
    assert row_scaled_err(want.row_ptr, g.values, want.val) <= TOL


@pytest.mark.parametrize("nr", [2, 3])
def test_lockstep_runs_inside_rank_interiors(nr):
    """Several ranks (gloo, one GPU): the rows of a z-slab without off-rank
    parts form long runs; their whole 64-row tiles take the lockstep kernel
    (numeric_path 3), the slab faces and the runs' edges the per-row kernels.
    C matches the oracle at the same rank count; a second pass after scaling
    A scales C."""
    from oracle.oracle import oracle_ptap

    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=24)
    want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                       P.values, nranks=nr, algorithm="allatonce")

    def prog(ctx):
        import copy

        a, p = pk.distribute(A, P, ctx.nranks, ctx.rank)
        plan = pk.run_symbolic(a, p, "allatonce", ctx)
        pk.run_numeric(a, p, plan, ctx)
        path = plan.device_counters()["numeric_path"]
        a.local.diag.values *= 2.0
        a.local.offdiag.values *= 2.0
        c2 = copy.deepcopy(pk.run_numeric(a, p, plan, ctx))
        a.local.diag.values /= 2.0
        a.local.offdiag.values /= 2.0
        c3 = pk.run_numeric(a, p, plan, ctx)
        return c3, path, c2

    res = pk.spawn_ranks(nr, prog)
    assert all(r[1] == 3 for r in res), [r[1] for r in res]
    g = pk.assemble_global([r[0] for r in res], ncols=P.ncols)
    pattern = np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
    assert pattern
    assert row_scaled_err(want.row_ptr, g.values, want.val) <= TOL
    g2 = pk.assemble_global([r[2] for r in res], ncols=P.ncols)
    assert row_scaled_err(want.row_ptr, g2.values, 2.0 * want.val) <= TOL


def test_lockstep_kernel_flags_in_place_structure_edits():
    """The lockstep kernel trusts the plan's classes; a row whose length no
    longer matches its class (row offsets edited in place, sizes unchanged, so
    the host-side size checks pass) is reported as structural drift instead of
    reading past its staged row."""
    from paper_1905_08423_b200 import devgen
    from paper_1905_08423_b200.errors import StructuralDriftError

    ctx = pk.single_rank_context()
    a, p = devgen.config_dist("cfg3", 1, 0, ctx.device, n_fine=16)
    plan = pk.run_symbolic(a, p, "allatonce", ctx)
    assert plan.device_counters()["numeric_path"] == 3
    pk.run_numeric_device(a, p, plan, ctx)
    plan.check()
    rp = a.local.diag.row_ptr
    k = rp.numel() // 2
    rp[k] += 1  # row k-1 one entry longer, row k one shorter
    pk.run_numeric_device(a, p, plan, ctx)
    with pytest.raises(StructuralDriftError):
        plan.check()
    rp[k] -= 1


@pytest.mark.parametrize("single", [True, False])
def test_arena_growth_path(single, monkeypatch):
    """An undersized first arena (PTAP_ARENA_SHRINK) overflows and is grown:
    the single-shot pass recomputes its values into the grown arena, the
    arena symbolic phase re-runs its pass; C matches the oracle either way."""
    monkeypatch.setenv("PTAP_ARENA_SHRINK", "6")
    monkeypatch.setenv("PTAP_NO_UNION", "1")  # the arena path also without single_shot
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=12)
    want = _oracle(A, P)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    c, plan = pk.ptap(a, p, "allatonce", ctx, single_shot=single)
    assert plan.values_ready == single
    g = pk.assemble_global([c.local], ncols=P.ncols)
    pattern = np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
    assert pattern
    assert row_scaled_err(want.row_ptr, g.values, want.val) <= TOL
