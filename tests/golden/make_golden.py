"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

For every case it runs the reference's own public API (``distribute``,
``spawn_ranks``, ``ptap``, ``assemble_global``; src/problems.py:147-154,
src/comm.py:325-344, src/tripleproduct.py:509-529, src/partition.py:215-234)
for each algorithm at several rank counts, and stores the assembled C
(row offsets, columns, values -- bit-exact) next to the inputs in
``tests/golden/<case>.npz``.  Inputs built by this repo's generators are
stored as a SHA-256 of their arrays instead of the arrays, to keep the
fixtures small; the tests rebuild them and check the digest first.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import ptap as ref  # noqa: E402  (the reference package)
from paper_1905_08423_b200 import problems as gen  # noqa: E402

ALGS = ("two-step", "allatonce", "merged")

TOY_A = [(0, 0, 1.0), (0, 1, 1.0), (0, 4, 1.0), (1, 1, 1.0), (1, 2, 1.0), (1, 4, 1.0),
         (2, 0, 1.0), (2, 3, 1.0), (2, 4, 1.0), (3, 1, 1.0), (3, 3, 1.0), (4, 3, 1.0),
         (4, 4, 1.0), (5, 1, 1.0), (5, 4, 1.0), (5, 5, 1.0)]
TOY_P = [(0, 0, 1.0), (0, 3, 1.0), (1, 1, 1.0), (2, 2, 1.0), (2, 3, 1.0), (3, 2, 1.0),
         (4, 1, 1.0), (4, 3, 1.0), (5, 2, 1.0)]


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def dense_random(n, m, density, seed):
    rng = np.random.default_rng(seed)
    ad = (rng.random((n, n)) < density) * rng.uniform(-1, 1, (n, n))
    np.fill_diagonal(ad, rng.uniform(0.5, 1.0, n))
    pd = (rng.random((n, m)) < density) * rng.uniform(-1, 1, (n, m))
    ar, ac = np.nonzero(ad)
    pr, pc = np.nonzero(pd)
    return (ref.CsrMatrix.from_triplets(n, n, ar, ac, ad[ar, ac]),
            ref.CsrMatrix.from_triplets(n, m, pr, pc, pd[pr, pc]))


def run_ref(a, p, nranks, alg):
    def prog(ctx):
        ad, pd = ref.distribute(a, p, ctx.nranks, ctx.rank)
        c, _ = ref.ptap(ad, pd, alg, ctx)
        return c.local

    locs = ref.spawn_ranks(nranks, prog)
    return ref.assemble_global(locs, ncols=p.ncols)


def to_ref(m):
    return ref.CsrMatrix(m.nrows, m.ncols, m.row_offsets, m.col_indices, m.values)


def save_case(name, a, p, ranks, store_inputs=True, meta=None):
    out = {"n": a.nrows, "m": p.ncols, "ranks": np.array(ranks)}
    if store_inputs:
        out.update(a_ip=a.row_offsets, a_j=a.col_indices, a_v=a.values,
                   p_ip=p.row_offsets, p_j=p.col_indices, p_v=p.values)
    else:
        out["input_digest"] = digest(a.row_offsets, a.col_indices, a.values,
                                     p.row_offsets, p.col_indices, p.values)
    for k, v in (meta or {}).items():
        out[k] = v
    for nr in ranks:
        for alg in ALGS:
            c = run_ref(a, p, nr, alg)
            tag = f"np{nr}_{alg}"
            out[tag + "_ip"] = c.row_offsets
            out[tag + "_j"] = c.col_indices
            out[tag + "_v"] = c.values
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print("wrote", name, {k: np.asarray(v).shape for k, v in out.items() if k.endswith("_v")})


def main():
    save_case("toy", ref.csr_from_triplets(6, 6, TOY_A), ref.csr_from_triplets(6, 4, TOY_P), [1, 2, 3])
    tri = ref.csr_from_triplets(3, 3, [(0, 0, 2.0), (0, 1, -1.0), (1, 0, -1.0), (1, 1, 2.0),
                                       (1, 2, -1.0), (2, 1, -1.0), (2, 2, 2.0)])
    save_case("tridiag", tri, ref.csr_from_triplets(3, 1, [(0, 0, 0.5), (1, 0, 1.0), (2, 0, 0.5)]), [1])
    save_case("identity_p", ref.csr_from_triplets(6, 6, TOY_A), ref.CsrMatrix.identity(6), [1, 3])
    for (n, m, d, s, ranks) in [(26, 14, 0.25, 3, [1, 2, 4]), (30, 18, 0.2, 4, [1, 2, 3, 5, 8]),
                                (28, 15, 0.3, 5, [1, 2, 4, 8]), (34, 21, 0.22, 6, [1, 3, 5])]:
        a, p = dense_random(n, m, d, s)
        save_case(f"dense_random_s{s}", a, p, ranks)
    a, p = dense_random(16, 9, 0.3, 8)
    za = ref.CsrMatrix(a.nrows, a.ncols, a.row_offsets, a.col_indices, np.zeros(a.nnz))
    save_case("zero_a", za, p, [1, 2])
    for seed in (11, 12):
        a, p = ref.random_instance(60, 20, 0.1, seed)
        save_case(f"random_instance_s{seed}", a, p, [1, 3, 7])
    for spec, ranks in [((4, 4, 4), [1, 3]), ((3, 4, 5), [2])]:
        def prog(ctx, spec=spec):
            a, p = ref.model_problem(ref.GridSpec(*spec), ctx.nranks, ctx.rank)
            return a.local, p.local
        res = ref.spawn_ranks(1, prog)
        nf, nc = ref.grid_dims(ref.GridSpec(*spec))
        a = ref.assemble_global([res[0][0]], ncols=nf)
        p = ref.assemble_global([res[0][1]], ncols=nc)
        save_case("model_%dx%dx%d" % spec, a, p, ranks)
    # this repo's config generators at reduced size (inputs stored by digest)
    a, p = gen.config_operands(gen.CONFIGS["cfg1"], n_fine=16)
    save_case("poisson7_16", to_ref(a), to_ref(p), [1, 4], store_inputs=False,
              meta={"gen": "cfg1", "n_fine": 16})
    a, p = gen.config_operands(gen.CONFIGS["cfg3"], n_fine=16)
    save_case("random27_16", to_ref(a), to_ref(p), [1, 3, 4], store_inputs=False,
              meta={"gen": "cfg3", "n_fine": 16})
    a, p = gen.config_operands(gen.CONFIGS["cfg1"], n_fine=32)
    save_case("cfg1_full", to_ref(a), to_ref(p), [1], store_inputs=False,
              meta={"gen": "cfg1", "n_fine": 32})


if __name__ == "__main__":
    main()
