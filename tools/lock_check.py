"""GPU check of the class-lockstep numeric pass (csrc/ptap_lock.cu): parity
with the CPU oracle at np=1 on reduced grids (pattern exact, row-scaled
values), agreement with the q4a pass, and the full 256^3 timing.
python tools/lock_check.py [full [n]]"""
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


def row_scaled(rp, ref, got):
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    rmax = np.zeros(len(rp) - 1)
    np.maximum.at(rmax, rows, np.abs(ref))
    return float((np.abs(got - ref) / np.maximum(rmax[rows], 1e-300)).max(initial=0.0))


def check_small():
    ctx = pk.single_rank_context()
    for cfg, nf in (("cfg3", 8), ("cfg3", 16), ("cfg3", 24), ("cfg2", 32), ("cfg1", 32), ("cfg3", 64)):
        A, P = gen.config_operands(gen.CONFIGS[cfg], n_fine=nf)
        want = oracle_ptap(A.nrows, P.ncols, A.row_offsets, A.col_indices, A.values, P.row_offsets, P.col_indices,
                           P.values, nranks=1, algorithm="allatonce")
        for alg in ("allatonce", "merged"):
            a, p = pk.distribute(A, P, 1, 0)
            c, plan = pk.ptap(a, p, alg, ctx)
            g = pk.assemble_global([c.local], ncols=P.ncols)
            path = plan.device_counters()["numeric_path"]
            pat = np.array_equal(g.row_offsets, want.row_ptr) and np.array_equal(g.col_indices, want.col)
            err = row_scaled(want.row_ptr, want.val, g.values) if pat else -1.0
            # a second pass on the same plan
            c2 = pk.run_numeric(a, p, plan, ctx)
            err2 = row_scaled(want.row_ptr, want.val, pk.assemble_global([c2], ncols=P.ncols).values) if pat else -1.0
            print(f"{cfg}@{nf} {alg}: path {path} pattern {pat} row-scaled {err:.2e} second pass {err2:.2e}", flush=True)


def full(n=256, reps=11):
    ctx = pk.single_rank_context()
    a, p = devgen.config_dist("cfg3", 1, 0, ctx.device, n_fine=n)
    res = {}
    for name, env in (("lock", None), ("q4a", "PTAP_NO_LOCK")):
        if env:
            os.environ[env] = "1"
        t = time.perf_counter()
        plan = pk.run_symbolic(a, p, "allatonce", ctx)
        torch.cuda.synchronize()
        print(name, "symbolic s", round(time.perf_counter() - t, 4), "path", plan.device_counters()["numeric_path"], flush=True)
        print(name, "memory", plan.memory(), flush=True)
        ms = []
        for r in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rp, col, v = pk.run_numeric_device(a, p, plan, ctx)
            e1.record()
            torch.cuda.synchronize()
            ms.append(round(e0.elapsed_time(e1), 3))
        print(name, "numeric ms", ms, flush=True)
        res[name] = (rp.clone(), v.clone())
        if env:
            del os.environ[env]
        del plan
    rp, v0 = res["q4a"]
    v1 = res["lock"][1]
    rows = torch.repeat_interleave(torch.arange(rp.numel() - 1, device=rp.device), rp[1:] - rp[:-1])
    scale = torch.zeros(rp.numel() - 1, dtype=torch.float64, device=rp.device)
    scale.scatter_reduce_(0, rows, v0.abs(), reduce="amax")
    print("lock vs q4a row-scaled", float(((v0 - v1).abs() / scale[rows].clamp_min(1e-300)).max().item()), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "full":
        full(int(sys.argv[2]) if len(sys.argv) > 2 else 256)
    else:
        check_small()
