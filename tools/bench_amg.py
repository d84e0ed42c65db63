"""Numeric/symbolic timing of the config-4 and config-5 style inputs (host
generators, reduced sizes): which device path each takes and how fast.
usage: python tools/bench_amg.py [nn_cfg4] [npts_cfg5]"""
import json
import sys
import time

sys.path.insert(0, '/root/repo')
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems_amg as amg


def run(name, A, P, reps=5):
    ctx = pk.single_rank_context()
    t = time.perf_counter()
    a, p = pk.distribute(A, P, 1, 0)
    out = {"config": name, "n": A.nrows, "nnz_a": A.nnz, "nnz_p": P.nnz, "m": P.ncols}
    from paper_1905_08423_b200.devgen import split_rows_device
    dev = ctx.device
    # device-resident operands (same CSR), so the timing is the device pass
    def up(lm, ncols):
        rp = torch.as_tensor(lm.diag.row_offsets, device=dev)
        col = torch.as_tensor(lm.diag.col_indices.astype('int32'), device=dev)
        val = torch.as_tensor(lm.diag.values, device=dev)
        return split_rows_device(rp, col, val, 0, lm.nrows, 0, ncols, ncols)
    from paper_1905_08423_b200.partition import DistMatrix
    ad = DistMatrix(a.row_part, a.col_part, 0, up(a.local, A.ncols))
    pd = DistMatrix(p.row_part, p.col_part, 0, up(p.local, P.ncols))
    for alg in ("allatonce", "two-step"):
        plan = pk.run_symbolic(ad, pd, alg, ctx)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan = pk.run_symbolic(ad, pd, alg, ctx)
        torch.cuda.synchronize()
        sym = time.perf_counter() - t0
        pk.run_numeric_device(ad, pd, plan, ctx)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            pk.run_numeric_device(ad, pd, plan, ctx)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        cnt = plan.device_counters()
        mac = cnt["mac_ap"] + cnt["mac_outer"]
        mem = plan.memory()
        out[alg] = {"numeric_ms": ms, "symbolic_ms": sym * 1e3, "gflops": 2 * mac / ms / 1e6, "mac": mac,
                    "nnz_c": cnt["nnz_c"], "aux_peak_bytes": mem["device_high_water"] - mem["current"]["output_matrix"]}
        del plan
    return out


nn = int(sys.argv[1]) if len(sys.argv) > 1 else 48
npts = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
t = time.perf_counter()
A4, P4 = amg.block_transport(nn)
g4 = time.perf_counter() - t
r4 = run(f"cfg4 block transport {nn}^3 x 10 (smoothed aggregation)", A4, P4)
r4["gen_s"] = g4
print(json.dumps(r4), flush=True)
t = time.perf_counter()
A5, P5 = amg.knn_laplacian(npts)
g5 = time.perf_counter() - t
r5 = run(f"cfg5 kNN Laplacian {npts} points (greedy aggregation)", A5, P5)
r5["gen_s"] = g5
print(json.dumps(r5), flush=True)
