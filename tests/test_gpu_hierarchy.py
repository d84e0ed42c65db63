"""Multigrid hierarchy driver (config 3 style, 3 levels): every level's C
against the oracle chained on its own C (end to end), at 1 and 2 ranks."""

import numpy as np
import pytest

from tests.conftest import row_scaled_err

pytestmark = pytest.mark.gpu


def _oracle_chain(A, Ps, nr, alg):
    from oracle.oracle import oracle_ptap
    from paper_1905_08423_b200 import CsrMatrix
    out = []
    cur = A
    for P in Ps:
        w = oracle_ptap(cur.nrows, P.ncols, cur.row_offsets, cur.col_indices, cur.values, P.row_offsets,
                        P.col_indices, P.values, nranks=nr, algorithm=alg)
        out.append(w)
        cur = CsrMatrix(P.ncols, P.ncols, w.row_ptr, w.col, w.val, check=False)
    return out


@pytest.mark.parametrize("nr", [1, 2])
@pytest.mark.parametrize("alg", ["two-step", "allatonce", "merged"])
def test_three_level_chain(nr, alg):
    import paper_1905_08423_b200 as pk
    from paper_1905_08423_b200 import problems as gen
    A, P1 = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=16)
    P2 = gen.trilinear(4)
    want = _oracle_chain(A, [P1, P2], nr, alg)

    def prog(ctx):
        a, p1 = pk.distribute(A, P1, ctx.nranks, ctx.rank)
        part1 = p1.col_part
        lo, hi = part1.owned_range(ctx.rank)
        p2 = pk.dist_from_global(P2, part1, pk.make_partition(P2.ncols, ctx.nranks), ctx.rank)
        h = pk.GalerkinHierarchy(a, [p1, p2], alg, ctx)
        res = []
        for _ in range(2):  # the second pass reuses every plan
            h.numeric()
            res = [h.c_local(0), h.c_local(1)]
        return [(r.row_lo, r.row_hi, r.diag.row_offsets.copy(), r.diag.col_indices.copy(), r.diag.values.copy(),
                 r.offdiag.row_offsets.copy(), r.offdiag.col_indices.copy(), r.offdiag.values.copy(),
                 r.col_map.copy(), r.col_lo) for r in res]

    results = pk.spawn_ranks(nr, prog)
    for lvl, P in enumerate([P1, P2]):
        locs = []
        for rk in results:
            lo, hi, drp, dcol, dval, orp, ocol, oval, cmap, clo = rk[lvl]
            locs.append(pk.LocalMatrix(lo, hi, clo, clo + (hi - lo), pk.CsrMatrix(hi - lo, hi - lo, drp, dcol, dval, check=False),
                                       pk.CsrMatrix(hi - lo, len(cmap), orp, ocol, oval, check=False), cmap))
        c = pk.assemble_global(locs, ncols=P.ncols)
        w = want[lvl]
        assert np.array_equal(c.row_offsets, w.row_ptr), f"level {lvl + 1} pattern"
        assert np.array_equal(c.col_indices, w.col), f"level {lvl + 1} columns"
        if alg == "two-step":
            assert np.array_equal(c.values.view(np.uint64), w.val.view(np.uint64)), f"level {lvl + 1} bitwise"
        assert row_scaled_err(w.row_ptr, c.values, w.val) <= 1e-12
