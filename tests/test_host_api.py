"""Host-side behaviour of the drop-in API (no GPU needed): the data model,
the partition layout and the operand checks that run before any device work,
mirroring the reference's tests (test_partition.py, test_sparse.py,
test_tripleproduct.py:379-428)."""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems as gen


def test_make_partition_golden_offsets():
    assert pk.make_partition(10, 3).offsets.tolist() == [0, 4, 7, 10]
    assert pk.make_partition(7, 7).offsets.tolist() == list(range(8))
    assert pk.make_partition(2, 4).offsets.tolist() == [0, 1, 2, 2, 2]
    with pytest.raises(pk.PartitionMismatchError):
        pk.make_partition(5, 0)


@pytest.mark.parametrize("nranks", [1, 2, 3, 5, 8])
def test_split_assemble_roundtrip(nranks):
    a, _ = gen.random_instance(40, 12, 0.2, seed=5)
    part = pk.make_partition(40, nranks)
    locs = [pk.dist_from_global(a, part, part, r).local for r in range(nranks)]
    back = pk.assemble_global(locs, ncols=40)
    assert back.structure_equal(a) and np.array_equal(back.values, a.values)
    for lm in locs:
        assert np.all(np.diff(lm.col_map) > 0)
        lo, hi = lm.col_lo, lm.col_hi
        assert not np.any((lm.col_map >= lo) & (lm.col_map < hi))


def test_from_triplets_sums_duplicates_and_sorts():
    m = pk.CsrMatrix.from_triplets(2, 3, [1, 0, 1, 0], [2, 1, 2, 0], [1.0, 2.0, 3.0, 4.0])
    assert m.row_offsets.tolist() == [0, 2, 3]
    assert m.col_indices.tolist() == [0, 1, 2]
    assert m.values.tolist() == [4.0, 2.0, 4.0]
    with pytest.raises(pk.AssemblyError):
        pk.CsrMatrix.from_triplets(2, 2, [0], [2], [1.0])


def test_transpose_with_permutation_is_stable():
    p = pk.csr_from_triplets(6, 4, [(0, 0, 1.0), (0, 3, 2.0), (1, 1, 3.0), (2, 2, 4.0), (2, 3, 5.0),
                                    (3, 2, 6.0), (4, 1, 7.0), (4, 3, 8.0), (5, 2, 9.0)])
    t, perm = p.transpose_with_permutation()
    assert t.row_cols(3).tolist() == [0, 2, 4]
    assert np.array_equal(t.values, p.values[perm])
    assert t.transpose().structure_equal(p)


def _toy_dist():
    a = pk.csr_from_triplets(4, 4, [(i, i, 2.0) for i in range(4)])
    p = pk.csr_from_triplets(4, 2, [(0, 0, 1.0), (1, 0, 1.0), (2, 1, 1.0), (3, 1, 1.0)])
    return pk.distribute(a, p, 1, 0)


def test_operand_checks_run_before_device_work():
    a, p = _toy_dist()
    ctx = pk.RankContext(0, 1, device="cpu")
    bad = pk.DistMatrix(pk.make_partition(5, 1), pk.make_partition(2, 1), 0, p.local)
    with pytest.raises(pk.PartitionMismatchError, match="dimension mismatch"):
        pk.run_symbolic(a, bad, "allatonce", ctx)
    with pytest.raises(ValueError, match="unknown algorithm"):
        pk.run_symbolic(a, p, "three-step", ctx)
    with pytest.raises(ValueError, match="cache policy"):
        pk.ptap(a, p, "merged", ctx, cache="sometimes")


def test_cpu_only_box_raises_device_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    a, p = _toy_dist()
    with pytest.raises(pk.DeviceError):
        pk.run_symbolic(a, p, "allatonce", pk.RankContext(0, 1, device="cpu"))


def test_generators_are_row_block_invariant():
    """Any row block of a generator equals the same rows of the whole matrix,
    so ranks can build their slabs independently (z-slab layout)."""
    a = gen.random27(8, 7)
    part = gen.random27(8, 7, 100, 300)
    assert np.array_equal(part.values, a.values[a.row_offsets[100]:a.row_offsets[300]])
    p = gen.trilinear(4)
    assert p.nnz == 11 ** 3  # 1D: 4 even points + 3 odd with 2 coarse neighbours + the last odd point
    sums = np.bincount(np.repeat(np.arange(p.nrows), np.diff(p.row_offsets)), weights=p.values)
    assert np.all(sums <= 1.0) and sums[0] == 1.0
    pp = gen.poisson7(32)
    assert pp.nnz == 223232
    tp = gen.trilinear(16)
    assert tp.nnz == 103823


def test_config3_values_are_symmetric_and_dominant():
    a = gen.random27(10, gen.CONFIGS["cfg3"].seed)
    d = a.to_dense()
    assert np.array_equal(d, d.T)
    off = np.abs(d).sum(axis=1) - np.abs(np.diag(d))
    assert np.all(np.diag(d) > off)


def test_ledger_categories_and_product_peak():
    led = pk.MemoryLedger()
    led.add("input_matrices", 100)
    led.add("output_matrix", 10)
    led.add("transient_hash_peak", 50)
    led.release("transient_hash_peak", 50)
    led.add("plan_cache", 5)
    assert led.product_peak == 60 and led.peak("input_matrices") == 100
    with pytest.raises(ValueError):
        led.release("plan_cache", 6)
