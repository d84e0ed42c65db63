"""Debug: deterministic pass vs oracle at full cfg3 after bench-like usage."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import devgen
from paper_1905_08423_b200.sparse import CsrMatrix
import bench
ctx = pk.single_rank_context()
a, p = devgen.config_dist("cfg3", 1, 0, ctx.device, n_fine=int(sys.argv[1]) if len(sys.argv) > 1 else 256)
dl, pl_ = a.local.diag, p.local.diag
A = CsrMatrix(dl.nrows, dl.ncols, dl.row_ptr.cpu().numpy(), dl.col.cpu().numpy(), dl.val.cpu().numpy(), check=False)
P = CsrMatrix(pl_.nrows, pl_.ncols, pl_.row_ptr.cpu().numpy(), pl_.col.cpu().numpy(), pl_.val.cpu().numpy(), check=False)
times, cmac, oplan, cval, csym = bench.oracle_run(A, P, 1, 1, 0)
for reps in (1, 12):
    plan = pk.run_symbolic(a, p, "allatonce", ctx, deterministic=True)
    for r in range(reps):
        bench.time_numeric(pk, a, p, plan, ctx, 1, 0, torch)
        _, _, v = plan.c_device()
        d = v.cpu().numpy()
        nb = int((d.view(np.uint64) != cval.view(np.uint64)).sum())
        print("reps", reps, "pass", r, "differing", nb, flush=True)
    del plan
