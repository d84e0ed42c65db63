"""The deterministic numeric pass (plan option ``deterministic``: the
owner-computes kernel of csrc/ptap_tile.cu) reproduces the reference's
summation order exactly (src/tripleproduct.py:12-16, src/_kernels.py:446-515):
at one rank its C is BIT-IDENTICAL to the reference's -- checked against the
reference's own golden outputs and against the oracle -- and repeated
numeric passes are bitwise identical, as are all-at-once and merged
(tests/test_tripleproduct.py:74-79, 111-128; acceptance C5)."""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems as gen
from tests.conftest import csr_from_arrays, golden_cases, load_golden, row_scaled_err

pytestmark = pytest.mark.gpu


def _bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def _run(A, P, alg, reps=1):
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, alg, ctx, deterministic=True)
    outs = [pk.run_numeric(a, p, plan, ctx).diag.values.copy() for _ in range(reps)]
    g = pk.assemble_global([plan.c_local()], ncols=P.ncols)
    return g, outs, plan


@pytest.mark.parametrize("case", golden_cases())
def test_golden_bitwise_at_one_rank(case):
    """Every golden fixture the kernel takes (one-rank structure, AP rows <= 32,
    C rows <= 64): all-at-once and merged bit-identical to the reference's own
    np=1 output; fixtures outside its envelope fall back to the atomic pass
    (plan.deterministic False) and are held to the row-scaled gate."""
    n, m, a, p, results = load_golden(case)
    A = csr_from_arrays(n, n, *a)
    P = csr_from_arrays(n, m, *p)
    for alg in ("allatonce", "merged"):
        if (1, alg) not in results:
            continue
        g, _, plan = _run(A, P, alg)
        ip, j, v = results[(1, alg)]
        assert np.array_equal(g.row_offsets, ip) and np.array_equal(g.col_indices, j), (alg, "pattern")
        if plan.deterministic:
            assert np.array_equal(_bits(g.values), _bits(v)), (alg, "bit-exact against the reference")
        else:
            assert row_scaled_err(ip, g.values, v) <= 1e-12, alg


def test_structured_fixtures_take_the_deterministic_kernel():
    taken = []
    for case in ("random27_16", "poisson7_16", "model_4x4x4", "cfg1_full"):
        n, m, a, p, _ = load_golden(case)
        _, _, plan = _run(csr_from_arrays(n, n, *a), csr_from_arrays(n, m, *p), "allatonce")
        taken.append(plan.deterministic)
    assert all(taken), taken


@pytest.mark.parametrize("nf", [24, 40])
def test_cfg3_bitwise_vs_oracle_repeat_and_merged(nf):
    """Config 3 (27-point random, non-dyadic values) at reduced size: C
    bit-identical to the oracle's np=1 output, 11 numeric passes bitwise
    identical, merged == all-at-once bitwise."""
    from oracle.oracle import oracle_ptap
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=nf)
    want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                       P.values, nranks=1, algorithm="allatonce")
    g, outs, plan = _run(A, P, "allatonce", reps=11)
    assert plan.deterministic and plan.device_counters()["numeric_path"] == 2
    assert plan.counters.numeric_runs == 11
    assert np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
    assert np.array_equal(_bits(g.values), _bits(want.val))
    for o in outs[1:]:
        assert np.array_equal(_bits(o), _bits(outs[0]))
    gm, _, _ = _run(A, P, "merged")
    assert np.array_equal(_bits(gm.values), _bits(g.values))


def test_values_change_between_passes_and_streamed_host_pass():
    """New values through the same plan (host operands: the streamed
    row-block upload path): still bit-identical to the oracle."""
    from oracle.oracle import oracle_ptap
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=32)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, "allatonce", ctx, deterministic=True)
    rng = np.random.default_rng(5)
    for _ in range(2):
        av = A.values * (1.0 + rng.random(A.values.size))
        a.local.diag.values = av.copy()
        c = pk.run_numeric(a, p, plan, ctx)
        want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, av, P.row_offsets, P.col_indices,
                           P.values, nranks=1, algorithm="allatonce")
        assert np.array_equal(_bits(c.diag.values), _bits(want.val))


def test_drift_is_detected():
    """A structure swapped after symbolic (same sizes, other columns) is caught
    by the device digest (StructuralDriftError), as the reference's fill check
    does (src/spgemm.py:58-68)."""
    import torch
    from paper_1905_08423_b200.errors import StructuralDriftError
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=16)
    ctx = pk.single_rank_context()
    a, p = pk.distribute(A, P, 1, 0)
    plan = pk.run_symbolic(a, p, "allatonce", ctx, deterministic=True)
    pk.run_numeric(a, p, plan, ctx)
    plan.c_alloc.verify_filled("C")
    col = plan._a_dev.diag.col.clone()
    col[5], col[6] = col[6], col[5]  # a different structure behind a new buffer
    plan._a_dev.diag.col = col
    with pytest.raises(StructuralDriftError):
        pk.run_numeric_device(a, p, plan, ctx)
    torch.cuda.synchronize()
