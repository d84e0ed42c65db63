"""Pin the CPU oracle against fixtures produced by the reference itself.

The fixtures (tests/golden/*.npz) come from tests/golden/make_golden.py,
which runs the reference's public API.  The oracle must reproduce every one
of them bit for bit: pattern and values, each algorithm, each rank count.
"""

import numpy as np
import pytest

from oracle.oracle import oracle_ptap
from tests.conftest import golden_cases, load_golden


@pytest.mark.parametrize("case", golden_cases())
def test_oracle_matches_reference_bitwise(case):
    n, m, a, p, results = load_golden(case)
    for (nr, alg), (ip, j, v) in results.items():
        got = oracle_ptap(n, m, *a, *p, nranks=nr, algorithm=alg)
        assert np.array_equal(got.row_ptr, ip), (case, nr, alg)
        assert np.array_equal(got.col, j), (case, nr, alg)
        assert np.array_equal(got.val.view(np.uint64), v.view(np.uint64)), (case, nr, alg)


def test_reference_algorithms_agree_bitwise_at_fixed_np():
    """SURVEY.md §0 finding 1: the three algorithms are bitwise identical at
    a fixed rank count (checked on the reference's own outputs)."""
    for case in golden_cases():
        _, _, _, _, results = load_golden(case)
        for (nr, alg), (ip, j, v) in results.items():
            base = results[(nr, "two-step")]
            assert np.array_equal(ip, base[0]) and np.array_equal(j, base[1])
            assert np.array_equal(v.view(np.uint64), base[2].view(np.uint64)), (case, nr, alg)


def test_oracle_counters_match_reference_definitions():
    """merged computes each AP row once; all-at-once twice for rows with both
    P_d and P_o nonempty (tests/test_tripleproduct.py:149-171 in the reference)."""
    n, m, a, p, _ = load_golden("dense_random_s4")
    for nr in (1, 2, 5):
        aao = oracle_ptap(n, m, *a, *p, nranks=nr, algorithm="allatonce").stats
        mrg = oracle_ptap(n, m, *a, *p, nranks=nr, algorithm="merged").stats
        assert mrg["rows_sym"] <= aao["rows_sym"]
        if nr == 1:
            assert mrg["rows_sym"] == aao["rows_sym"]
