"""Numeric passes of config 5 (kNN Laplacian, hash path by policy) at a
reduced point count, for profiling: python tools/cfg5_numeric.py [npts] [reps] [variants]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1905_08423_b200 as pk
from paper_1905_08423_b200 import problems_amg as amg
from tools.bench_configs import upload

npts = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
variants = sys.argv[3].split(",") if len(sys.argv) > 3 else ["hash"]
ctx = pk.single_rank_context()
A, P = amg.knn_laplacian(npts)
a, p = upload(A, P, ctx.device)
for v in variants:
    alg = "two-step" if v == "two-step" else "allatonce"
    kw = {"maps": True} if v == "maps" else {}
    plan = pk.run_symbolic(a, p, alg, ctx, **kw)
    torch.cuda.synchronize()
    c = plan.device_counters()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        pk.run_numeric_device(a, p, plan, ctx)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    mac = c["mac_ap"] + c["mac_outer"]
    print(f"{v}: path {c['numeric_path']} numeric ms {sorted(ts)[len(ts) // 2]:.3f} GF/s "
          f"{2 * mac / (sorted(ts)[len(ts) // 2] * 1e-3) / 1e9:.1f} mem {plan.memory()['product_peak'] / 1e9:.2f} GB",
          flush=True)
    del plan
