"""Time the reference package itself (numba CPU, installed unmodified into
baseline/_ref) on one BASELINE configuration at np=1, through its own public
API (ptap.spawn_ranks + run_symbolic / run_numeric, src/tripleproduct.py:499-506),
and optionally check the oracle port (oracle/) against it bit for bit.

BENCH / TEST INFRASTRUCTURE ONLY (bench.py runs it in a subprocess):

    PYTHONPATH=baseline/_ref NUMBA_CACHE_DIR=... python tools/ref_numba.py cfg2 [--n-fine N] [--repeats R]
        [--check-oracle]

prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", default="cfg2", nargs="?")
    ap.add_argument("--n-fine", type=int, default=None)
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--check-oracle", action="store_true")
    args = ap.parse_args()
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if ref_dir not in sys.path:
        sys.path.insert(0, ref_dir)
    sys.path.insert(1, ROOT)
    import numpy as np

    import ptap  # the unmodified reference
    from ptap.comm import spawn_ranks
    from ptap.problems import distribute
    from ptap.sparse import CsrMatrix as RefCsr

    from paper_1905_08423_b200 import problems as gen

    t0 = time.perf_counter()
    A, P = gen.config_operands(gen.CONFIGS[args.config], n_fine=args.n_fine)
    gen_s = time.perf_counter() - t0
    Ar = RefCsr(A.nrows, A.ncols, A.row_offsets, A.col_indices, A.values, check=False)
    Pr = RefCsr(P.nrows, P.ncols, P.row_offsets, P.col_indices, P.values, check=False)
    out = {}

    def prog(ctx):
        a, p = distribute(Ar, Pr, 1, 0)
        t = time.perf_counter()
        plan = ptap.run_symbolic(a, p, "allatonce", ctx)
        out["symbolic_s"] = time.perf_counter() - t
        times = []
        loc = None
        for _ in range(max(1, args.repeats)):
            t = time.perf_counter()
            loc = ptap.run_numeric(a, p, plan, ctx)
            times.append(time.perf_counter() - t)
        out["numeric_s"] = times
        out["c_local"] = loc
        return None

    spawn_ranks(1, prog)
    loc = out.pop("c_local")
    # one rank: diag block holds every column
    ip = np.asarray(loc.diag.row_offsets)
    col = np.asarray(loc.diag.col_indices)
    val = np.asarray(loc.diag.values)
    res = {"config": args.config, "n_fine": args.n_fine or gen.CONFIGS[args.config].n_fine, "np": 1,
           "algorithm": "allatonce", "gen_s": gen_s, "symbolic_s": out["symbolic_s"], "numeric_s": out["numeric_s"],
           "nnz_c": int(col.size), "numba": __import__("numba").__version__, "threads": 1}
    if args.check_oracle:
        from oracle.oracle import OraclePlan
        plan = OraclePlan(A.nrows, P.ncols, A.row_offsets, A.col_indices, P.row_offsets, P.col_indices, nranks=1,
                          algorithm="allatonce")
        t = time.perf_counter()
        v = plan.numeric(A.values, P.values)
        res["port_numeric_s"] = time.perf_counter() - t
        st = plan.num_stats
        res["mac"] = int(st.mac_ap + st.mac_outer)
        res["port_bitwise_equal"] = bool(np.array_equal(plan.row_ptr, ip) and np.array_equal(plan.col, col)
                                         and np.array_equal(v.view(np.uint64), val.view(np.uint64)))
        tn = min(out["numeric_s"])
        res["gflops"] = 2.0 * res["mac"] / tn / 1e9
        res["port_gflops"] = 2.0 * res["mac"] / res["port_numeric_s"] / 1e9
        res["port_over_reference"] = res["port_gflops"] / res["gflops"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
