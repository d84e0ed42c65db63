"""Galerkin invariants of C on the CUDA path (the reference's
tests/test_tripleproduct.py:313-351 and its partition-invariance checks):
zero row sums and symmetry on the model problem (graph Laplacian, constant-
preserving P) at 8 ranks, matvec consistency C x = P^T (A (P x)), and C at
np = 1 vs np = 5 within a row-scaled 1e-13."""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems as gen
from tests.conftest import row_scaled_err, run_ptap

pytestmark = pytest.mark.gpu


def test_model_16cube_row_sums_and_symmetry():
    A, P = gen.model_problem_global(16, 16, 16)
    c, _ = run_ptap(A, P, 8, "merged")
    scale = np.abs(c.values).max()
    assert np.abs(c.matvec(np.ones(P.ncols))).max() <= 1e-12 * scale
    t = c.transpose()
    assert t.structure_equal(c)
    assert np.abs(t.values - c.values).max() <= 1e-12 * scale


@pytest.mark.parametrize("alg", ["two-step", "allatonce", "merged"])
def test_galerkin_matvec_consistency(alg):
    A, P = gen.model_problem_global(4, 5, 3)
    c, _ = run_ptap(A, P, 2, alg)
    rng = np.random.default_rng(15)
    for _ in range(5):
        x = rng.uniform(-1, 1, P.ncols)
        via = P.transpose().matvec(A.matvec(P.matvec(x)))
        direct = c.matvec(x)
        assert np.abs(via - direct).max() <= 1e-12 * max(np.abs(direct).max(), 1e-300)


@pytest.mark.parametrize("alg", ["allatonce", "merged", "two-step"])
def test_partition_invariance(alg):
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=14)
    c1, _ = run_ptap(A, P, 1, alg)
    c5, _ = run_ptap(A, P, 5, alg)
    assert np.array_equal(c1.row_offsets, c5.row_offsets) and np.array_equal(c1.col_indices, c5.col_indices)
    assert row_scaled_err(c1.row_offsets, c5.values, c1.values) <= 1e-13
