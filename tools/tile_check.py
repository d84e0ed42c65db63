"""GPU check of the deterministic tile numeric pass: bitwise parity with the
CPU oracle at np=1 on reduced config-3/config-2 grids, bitwise repeat, and
the full 256^3 timing.  python tools/tile_check.py [full]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_08423_b200 as pk
from oracle.oracle import oracle_ptap
from paper_1905_08423_b200 import devgen
from paper_1905_08423_b200 import problems as gen


def check_small():
    ctx = pk.single_rank_context()
    for cfg, nf in (("cfg3", 16), ("cfg3", 24), ("cfg2", 32), ("cfg3", 64)):
        A, P = gen.config_operands(gen.CONFIGS[cfg], n_fine=nf)
        want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                           P.values, nranks=1, algorithm="allatonce")
        for alg in ("allatonce", "merged"):
            a, p = pk.distribute(A, P, 1, 0)
            c, plan = pk.ptap(a, p, alg, ctx, deterministic=True)
            g = pk.assemble_global([c.local], ncols=P.ncols)
            path = plan.device_counters()["numeric_path"]
            pat = np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
            bits = pat and np.array_equal(g.values.view(np.uint64), want.val.view(np.uint64))
            nd = int((g.values.view(np.uint64) != want.val.view(np.uint64)).sum()) if pat else -1
            print(f"{cfg}@{nf} {alg}: path {path} pattern {pat} bitwise {bits} ndiff {nd}", flush=True)


def full(n=256, reps=11):
    ctx = pk.single_rank_context()
    a, p = devgen.config_dist("cfg3", 1, 0, ctx.device, n_fine=n)
    t = time.perf_counter()
    plan = pk.run_symbolic(a, p, "allatonce", ctx, deterministic=os.environ.get("PTAP_TILE_OFF") is None)
    torch.cuda.synchronize()
    print("symbolic s", time.perf_counter() - t, "counters", plan.device_counters(), flush=True)
    print("memory", plan.memory(), flush=True)
    vals = []
    for r in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _, _, v = pk.run_numeric_device(a, p, plan, ctx)
        e1.record()
        torch.cuda.synchronize()
        print("numeric ms", round(e0.elapsed_time(e1), 3), flush=True)
        vals.append(v.clone())
    same = all(torch.equal(vals[0].view(torch.int64), x.view(torch.int64)) for x in vals[1:])
    print("bitwise repeat over", reps, "passes:", same, flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "full":
        full(int(sys.argv[2]) if len(sys.argv) > 2 else 256)
    else:
        check_small()
