"""Matrix Market and .npz interchange (the reference's tests/test_mmio.py
contract: bit-exact round trip, duplicates summed, line-numbered errors)."""

import numpy as np
import pytest

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems as gen


def test_round_trip_bit_exact(tmp_path):
    A, P = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=6)
    for m in (A, P):
        f = tmp_path / "m.mtx"
        pk.write_matrix_market(f, m)
        r = pk.read_matrix_market(f)
        assert r.nrows == m.nrows and r.ncols == m.ncols
        assert np.array_equal(r.row_offsets, m.row_offsets) and np.array_equal(r.col_indices, m.col_indices)
        assert np.array_equal(r.values.view(np.uint64), m.values.view(np.uint64))
        g = tmp_path / "m.npz"
        pk.save_npz(g, m)
        q = pk.load_npz(g)
        assert np.array_equal(q.values.view(np.uint64), m.values.view(np.uint64))
        assert np.array_equal(q.col_indices, m.col_indices)


def test_duplicates_summed_and_comments(tmp_path):
    f = tmp_path / "d.mtx"
    f.write_text("%%MatrixMarket matrix coordinate real general\n% a comment\n2 3 3\n1 2 1.5\n1 2 2.5\n2 3 -1\n")
    m = pk.read_matrix_market(f)
    assert m.nnz == 2 and m.row_cols(0).tolist() == [1] and m.row_values(0).tolist() == [4.0]


@pytest.mark.parametrize("text,line", [
    ("%%MatrixMarket matrix array real general\n1 1\n1\n", 1),
    ("hello\n", 1),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", 2),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 3),
])
def test_errors_carry_line(tmp_path, text, line):
    f = tmp_path / "e.mtx"
    f.write_text(text)
    with pytest.raises(pk.MatrixMarketError) as ei:
        pk.read_matrix_market(f)
    assert ei.value.line == line
